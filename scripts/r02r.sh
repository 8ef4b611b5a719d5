mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_dense.py tests/test_gpu_batch.py tests/test_gpu_bench_parity.py -q -x > gpurun_out/pytest_r02r.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r02r.log | cut -c1-300
bash scripts/ab_iso.sh main
bash scripts/ab_stream.sh main pfk2 pfk3 pfk4 2>&1 | grep -v "^pytest\|passed"
bash scripts/sanitize.sh
