# development A/B over library variants: bash scripts/ab_libs.sh <variant>... (main = the product build)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q -m gpu 2>&1 | tail -2
for v in "$@"; do
  if [ $v = main ]; then export PSATTN_B200_LIB=; else export PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_$v.so; fi
  for r in 1 2; do
  timeout 200 python bench.py --warmup 3 --steps 20 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]);print('$v', round(d['value']), round(d['ms_per_step'],3), d['stage_ms_per_step'])" || tail -3 gpurun_out/ab_$v.log
  done
done
