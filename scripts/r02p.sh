timeout 600 python -m pytest tests/test_gpu_capi.py tests/test_gpu_dense.py tests/test_gpu_cpp.py -q -x > gpurun_out/pytest_r02p.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r02p.log | cut -c1-300
bash scripts/ab_iso.sh main dpf3 dpf4 main
