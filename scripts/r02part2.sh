mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_stream.py -q -x 2>&1 | tail -2
run() {
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --check 4 --dropin-units 0 "$@" > gpurun_out/part.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/part.log').read().strip().splitlines()[-1]);print('$*', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['stage_ms_per_step'].items()}, d['parity_ok'], d['parity'].get('exact'), d['parity'].get('tie'), d['parity'].get('error'))" || tail -5 gpurun_out/part.log
}
run --eps 0.99 --dense-partial 0
run --eps 0.99
run --eps 0.99 --dense-partial 1024
run --eps 0.99 --dense-partial 512
run
run --dist iso
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
   --log-file gpurun_out/launches_e99p.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --check 0 --dropin-units 0 --eps 0.99 \
   > gpurun_out/ncu_e99p.log 2>&1; echo "ncu rc=$?"
