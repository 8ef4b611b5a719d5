# development A/B on the iso workload only (dense hand-over kernels)
for v in "$@"; do
  if [ $v = main ]; then export PSATTN_B200_LIB=; else export PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_$v.so; fi
  timeout 300 python bench.py --warmup 3 --steps 10 --no-cpu-baseline --dist iso | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v iso', round(d['value']), round(d['ms_per_step'],3), d['stage_ms_per_step'])"
done
