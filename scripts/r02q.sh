mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02q.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_r02q.log | cut -c1-300
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02q.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r02q.log
timeout 600 python bench.py > gpurun_out/bench_r02q.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r02q.log | cut -c1-600
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r02q.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_r02q.log | cut -c1-300
timeout 600 python bench.py --dist iso --steps 10 --no-cpu-baseline --check 4 > gpurun_out/bench_iso_r02q.log 2>&1; echo "iso rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
   --log-file gpurun_out/launches_r02q.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --check 0 --dropin-units 0 \
   > gpurun_out/ncu_launch_bench_r02q.log 2>&1; echo "ncu launches rc=$?"
for k in score_kernel_tma psa_stream_kernel first_tranche_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 -c 1 \
     -o gpurun_out/r02q_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --check 0 --graph 0 --dropin-units 0 \
     > gpurun_out/ncu_full_${k}_r02q.log 2>&1; echo "ncu $k rc=$?"
done
for k in dense_k_kernel dense_v_kernel dense_decide_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 1 -c 1 \
     -o gpurun_out/r02q_$k -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --dist iso --check 0 --graph 0 --dropin-units 0 \
     > gpurun_out/ncu_full_${k}_r02q.log 2>&1; echo "ncu $k rc=$?"
done
