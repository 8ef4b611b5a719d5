mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stream.py tests/test_gpu_bench_parity.py tests/test_gpu_batch.py -q -x > gpurun_out/ab_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ab_pytest.log
run() {  # tag, env, args
  timeout 200 env $2 python bench.py --warmup 3 --steps 20 --no-cpu-baseline --check 4 --dropin-units 0 $3 > gpurun_out/ab_$1.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_$1.log').read().strip().splitlines()[-1]);print('$1', round(d['value']), round(d['ms_per_step'],3), {k: round(x, 3) for k, x in d['stage_ms_per_step'].items()}, d['parity_ok'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab_$1.log
}
for r in 1 2; do
run base X=1 "--pipeline 1"
run p2 X=1 "--pipeline 2"
run p4 X=1 "--pipeline 4"
run p2f0 PSA_SCORE_SMEM_FLOOR=0 "--pipeline 2"
run p4f0 PSA_SCORE_SMEM_FLOOR=0 "--pipeline 4"
run p8f0 PSA_SCORE_SMEM_FLOOR=0 "--pipeline 8"
done
PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_sprof.so timeout 300 python bench.py --warmup 3 --steps 5 --no-cpu-baseline --check 0 --dropin-units 0 2>&1 | grep stream_prof
