run() {
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --check 4 "$@" > gpurun_out/sweep.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/sweep.log').read().strip().splitlines()[-1]);print('$*', round(d['value']), round(d['ms_per_step'],3), d['parity_ok'], d['parity'].get('exact'), d['parity'].get('tie'), d['parity'].get('error'), d['config'].get('layers_resident'), (d.get('e2e_dropin') or {}).get('value'))" || tail -5 gpurun_out/sweep.log
}
run --hkv 16 --dropin-units 0
run --ctx 100003 --dropin-units 2
run --ctx 100003 --dist iso --dropin-units 0
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 --ctx 100003 2>&1 | tail -1
