mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_bench_parity.py tests/test_gpu_batch.py -q -x > gpurun_out/pytest_r02i.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r02i.log | cut -c1-300
for r in 1 2; do timeout 300 python bench.py --warmup 3 --steps 20 --no-cpu-baseline --check 4 > gpurun_out/bench_r02i.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_r02i.log').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],3), d['stage_ms_per_step'], d['parity_ok'], d['clocks']['sm_mhz'])"; done
PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_sprof.so timeout 300 python bench.py --warmup 3 --steps 5 --no-cpu-baseline --check 0 2>&1 | grep stream_prof
