timeout 900 python -m pytest tests/test_gpu_tier.py tests/test_gpu_dense.py -q -x > gpurun_out/pytest_r02u.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r02u.log | cut -c1-300
bash scripts/ab_iso.sh main dvt
bash scripts/ab_stream.sh main w6 w6c w6l3 rv12 2>&1 | grep -v "^pytest\|passed"
