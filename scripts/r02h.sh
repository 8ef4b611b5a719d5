mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_cpp.py -q -x -m gpu -s > gpurun_out/pytest_cpp_r02h.log 2>&1; echo "cpp rc=$?"; grep -a "pipeline overlap\|golden\|FAIL\|passed\|failed" gpurun_out/pytest_cpp_r02h.log | head
PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_sprof.so timeout 300 python bench.py --warmup 3 --steps 5 --no-cpu-baseline --check 0 2>&1 | grep stream_prof
PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_sprof.so timeout 300 python bench.py --warmup 3 --steps 5 --no-cpu-baseline --check 0 --dist iso 2>&1 | grep stream_prof
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02h.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu_r02h.log | cut -c1-300
