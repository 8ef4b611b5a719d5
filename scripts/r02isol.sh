mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 30 --csv \
   --log-file gpurun_out/launches_iso_now.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --check 0 --dropin-units 0 --dist iso \
   > gpurun_out/ncu_iso_now.log 2>&1; echo "ncu rc=$?"
