mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_bench_parity.py tests/test_gpu_batch.py tests/test_gpu_dense.py -q -x > gpurun_out/pytest_r02m.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_r02m.log | cut -c1-400
for r in 1 2; do timeout 300 python bench.py --warmup 3 --steps 20 --no-cpu-baseline --check 4 --dropin-units 0 > gpurun_out/bench_r02m.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/bench_r02m.log').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],3), d['stage_ms_per_step'], d['parity_ok'], d['clocks']['sm_mhz'])"; done
PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_sprof.so timeout 300 python bench.py --warmup 3 --steps 5 --no-cpu-baseline --check 0 --dropin-units 0 2>&1 | grep stream_prof
timeout 600 python bench.py --dist iso --steps 5 --warmup 3 --no-cpu-baseline --check 2 --dropin-units 0 > gpurun_out/bench_iso_r02m.log 2>&1; echo "iso rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/bench_iso_r02m.log').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],3), d['stage_ms_per_step'], d['parity_ok'])"
