timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_stream.py tests/test_gpu_batch.py tests/test_gpu_tier.py -q -x > gpurun_out/pytest_r02t.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r02t.log | cut -c1-400
bash scripts/ab_iso.sh main
bash scripts/ab_stream.sh main w6 w6b 2>&1 | grep -v "^pytest\|passed"
