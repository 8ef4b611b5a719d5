# development A/B over library variants (stream kernel): bash scripts/ab_stream.sh <variant>... (main = product build)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_bench_parity.py -q -x > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ab_pytest.log
for v in "$@"; do
  if [ $v = main ]; then export PSATTN_B200_LIB=; else export PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_$v.so; fi
  for r in 1 2; do
  timeout 200 python bench.py --warmup 3 --steps 20 --no-cpu-baseline --check 2 --dropin-units 0 > gpurun_out/ab_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]);print('$v', round(d['value']), round(d['ms_per_step'],3), {k: round(x, 3) for k, x in d['stage_ms_per_step'].items()}, d['parity_ok'], round(d['fetch']['waste_frac'], 4), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab_$v.log
  done
done
