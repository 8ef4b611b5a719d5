set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02a.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_r02a.log
timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/bench_r02a.log 2>&1; tail -1 gpurun_out/bench_r02a.log
PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_prof.so timeout 200 python bench.py --warmup 3 --steps 10 --no-cpu-baseline 2>&1 | grep gqa_phase
