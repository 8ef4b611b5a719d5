# robustness sweep of bench configurations (each re-checks sampled units of its own step against the reference)
run() {
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --dropin-units 0 --check 4 "$@" > gpurun_out/sweep.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/sweep.log').read().strip().splitlines()[-1]);print('$*', round(d['value']), round(d['ms_per_step'],3), d['parity_ok'], d['parity'].get('exact'), d['parity'].get('tie'), d['parity'].get('error'), round(d['kv_fraction_read'],4))" || tail -3 gpurun_out/sweep.log
}
run --total-requests 64
run --microbatch 4
run --eps 0.99
run --eps 0.8
run --eps 0.9 --dist iso
run --hkv 16
run --hkv 4 --hq 32
run --ctx 32768 --requests 1 --layers 1
run --ctx 100003
