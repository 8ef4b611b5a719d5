# development A/B on the iso workload (dense hand-over): bash scripts/ab_iso.sh <variant>... (main = product build)
for v in "$@"; do
  if [ $v = main ]; then export PSATTN_B200_LIB=; else export PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_$v.so; fi
  timeout 300 python bench.py --warmup 3 --steps 6 --no-cpu-baseline --check 1 --dropin-units 0 --dist iso | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v iso', round(d['value']), round(d['ms_per_step'],3), d['stage_ms_per_step'], d['parity_ok'])"
done
