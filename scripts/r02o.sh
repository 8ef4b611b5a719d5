mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stream.py tests/test_gpu_bench_parity.py tests/test_gpu_batch.py tests/test_gpu_dense.py -q -x > gpurun_out/pytest_r02o.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r02o.log | cut -c1-400
timeout 600 python bench.py --dist iso --steps 5 --warmup 3 --no-cpu-baseline --check 2 --dropin-units 0 > gpurun_out/bench_iso_r02o.log 2>&1; echo "iso rc=$?"; python -c "import json;d=json.loads(open('gpurun_out/bench_iso_r02o.log').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],3), d['stage_ms_per_step'], d['parity_ok'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:"psa|score|dense|first" --launch-skip 7 -c 7 --csv --log-file gpurun_out/launches_iso_r02o.csv \
     python bench.py --steps 1 --warmup 3 --no-cpu-baseline --dist iso --graph 0 --check 0 --dropin-units 0 > /dev/null 2>&1; echo "ncu iso rc=$?"
python scripts/launch_table.py gpurun_out/launches_iso_r02o.csv
