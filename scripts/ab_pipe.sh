# development A/B: score/progressive two-stream overlap (sub-batches x score smem floor)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_batch.py -x -q -m gpu -k pipelined 2>&1 | tail -2
PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_prof.so timeout 200 python bench.py --warmup 3 --steps 10 --no-cpu-baseline 2>&1 | grep gqa_phase
run() {
  timeout 200 python bench.py --warmup 3 --steps 20 --no-cpu-baseline "$@" > gpurun_out/ab.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]);print(sys.argv[1:], round(d['value']), round(d['ms_per_step'],3), d['stage_ms_per_step'])" "$@" "floor=$PSA_SCORE_SMEM_FLOOR"
}
run --pipeline 1
for k in 2 4 8 16; do run --pipeline $k; done
export PSA_SCORE_SMEM_FLOOR=0; run --pipeline 4
export PSA_SCORE_SMEM_FLOOR=80000; run --pipeline 4
