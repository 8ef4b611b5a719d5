# ncu full captures of the three kernels of the planted step + the C++ API test (executors)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_cpp.py -q -x -m gpu -s > gpurun_out/pytest_cpp_r02g.log 2>&1; echo "cpp rc=$?"; grep -a "pipeline overlap\|FAIL\|passed\|failed" gpurun_out/pytest_cpp_r02g.log | head
for k in psa_stream_kernel score_kernel_tma first_tranche_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 -c 1 \
     -o gpurun_out/r02g_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --check 0 --graph 0 \
     > gpurun_out/ncu_full_${k}_r02g.log 2>&1; echo "ncu $k rc=$?"
done
