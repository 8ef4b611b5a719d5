mkdir -p gpurun_out
PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_sprof.so timeout 300 python bench.py --warmup 3 --steps 5 --no-cpu-baseline --check 0 --dropin-units 0 2>&1 | grep stream_prof
timeout 600 python bench.py --warmup 3 --steps 10 --no-cpu-baseline --check 2 > gpurun_out/bench_r02j.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r02j.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d.get(k) for k in ('value','ms_per_step','stage_ms_per_step','e2e','e2e_dropin')})"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:"psa|score|dense|first" --launch-skip 7 -c 7 --csv --log-file gpurun_out/launches_iso_r02j.csv \
     python bench.py --steps 1 --warmup 3 --no-cpu-baseline --dist iso --graph 0 --check 0 --dropin-units 0 > /dev/null 2>&1; echo "ncu iso rc=$?"
python scripts/launch_table.py gpurun_out/launches_iso_r02j.csv
