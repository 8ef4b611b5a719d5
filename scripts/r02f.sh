# A/B of stream-kernel variants + per-kernel launch list (time + DRAM bytes) of one planted step
mkdir -p gpurun_out
for v in main look4 look6 rk12; do
  if [ $v = main ]; then export PSATTN_B200_LIB=; else export PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_$v.so; fi
  for r in 1 2; do
  timeout 200 python bench.py --warmup 3 --steps 20 --no-cpu-baseline --check 2 > gpurun_out/ab_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]);print('$v', round(d['value']), round(d['ms_per_step'],3), d['stage_ms_per_step'], d['parity_ok'], d['fetch']['waste_frac'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab_$v.log
  done
done
unset PSATTN_B200_LIB
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none \
   --launch-skip 12 -c 12 --csv --log-file gpurun_out/launches_r02f.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --check 0 --graph 0 > gpurun_out/ncu_r02f.log 2>&1; echo "ncu rc=$?"
python scripts/launch_table.py gpurun_out/launches_r02f.csv || true
