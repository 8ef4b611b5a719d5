# final round-2 evidence: tests, smoke, bench lines, config-3 report, launch lists, full ncu captures, sanitizers
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02z.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_r02z.log | cut -c1-300
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02z.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r02z.log
timeout 600 python bench.py > gpurun_out/bench_r02z.log 2>&1; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r02z.log 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --dist iso --steps 10 --no-cpu-baseline --check 4 > gpurun_out/bench_iso_r02z.log 2>&1; echo "iso rc=$?"
timeout 600 python scripts/config3_report.py gpurun_out/config3_r02z.json > /dev/null 2>&1; echo "config3 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
   --log-file gpurun_out/launches_r02z.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --check 0 --dropin-units 0 --e2e-buffers 1 \
   > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:"psa|score|dense|first" --launch-skip 7 -c 7 --csv --log-file gpurun_out/launches_iso_r02z.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --dist iso --graph 0 --check 0 --dropin-units 0 --e2e-buffers 1 > /dev/null 2>&1; echo "ncu iso rc=$?"
for k in score_kernel_tma psa_stream_kernel first_tranche_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 3 -c 1 \
     -o gpurun_out/r02z_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --check 0 --graph 0 --dropin-units 0 --e2e-buffers 1 \
     > /dev/null 2>&1; echo "ncu $k rc=$?"
done
for k in dense_k_kernel dense_v_kernel dense_decide_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 1 -c 1 \
     -o gpurun_out/r02z_$k -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --dist iso --check 0 --graph 0 --dropin-units 0 --e2e-buffers 1 \
     > /dev/null 2>&1; echo "ncu $k rc=$?"
done
bash scripts/sanitize.sh
