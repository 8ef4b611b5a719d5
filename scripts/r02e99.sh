mkdir -p gpurun_out
for e in 0.95 0.99; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --check 4 --dropin-units 0 --eps $e > gpurun_out/e99.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/e99.log').read().strip().splitlines()[-1]);print('$e', d['ms_per_step'], d['stage_ms_per_step'], d['kv_fraction_read'], d.get('fetch'), d['mean_blocks_processed'])"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
   --log-file gpurun_out/launches_e99.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --check 0 --dropin-units 0 --eps 0.99 \
   > gpurun_out/ncu_e99.log 2>&1; echo "ncu rc=$?"
