timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_stream.py tests/test_gpu_batch.py -q -x > gpurun_out/pytest_r02s.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r02s.log | cut -c1-400
bash scripts/ab_iso.sh main dk3 oldk oldkv
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:"dense" --launch-skip 4 -c 4 --csv --log-file gpurun_out/launches_iso_r02s.csv \
     python bench.py --steps 1 --warmup 1 --no-cpu-baseline --dist iso --graph 0 --check 0 --dropin-units 0 > /dev/null 2>&1; echo "ncu iso rc=$?"
python scripts/launch_table.py gpurun_out/launches_iso_r02s.csv
