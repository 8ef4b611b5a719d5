timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_bench_parity.py tests/test_gpu_batch.py -q -x > gpurun_out/pytest_r02v.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r02v.log | cut -c1-300
PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_spl2.so timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_bench_parity.py -q -x -k "not counters" > gpurun_out/pytest_r02v_spl2.log 2>&1; echo "pytest spl2 rc=$?"; tail -2 gpurun_out/pytest_r02v_spl2.log | cut -c1-300
bash scripts/ab_stream.sh main spl2 spl2l1 2>&1 | grep -v "^pytest\|passed"
