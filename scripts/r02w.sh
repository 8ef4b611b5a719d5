timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_bench_parity.py -q -x > gpurun_out/pytest_r02w.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r02w.log | cut -c1-300
bash scripts/ab_stream.sh main k12 k12l3 e384 2>&1 | grep -v "^pytest\|passed"
