# development A/B: GPU parity of the batch path, then the bench with the phase-timer build and the product build
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q -m gpu 2>&1 | tail -2
PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_prof.so timeout 200 python bench.py --warmup 3 --steps 10 --no-cpu-baseline 2>&1 | grep gqa_phase
for r in 1 2; do
timeout 200 python bench.py --warmup 3 --steps 20 --no-cpu-baseline > gpurun_out/ab.log 2>&1
python -c "import json;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],3), d['stage_ms_per_step'])"
done
