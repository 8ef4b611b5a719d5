set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02b.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_r02b.log
timeout 400 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02b.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r02b.log | cut -c1-3000
PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_prof.so timeout 300 python bench.py --warmup 3 --steps 10 --no-cpu-baseline --check 0 2>&1 | grep gqa_phase
timeout 600 python bench.py --total-requests 64 --steps 10 --warmup 3 --no-cpu-baseline --check 4 > gpurun_out/bench_c5_r02b.log 2>&1; echo "c5 rc=$?"; tail -1 gpurun_out/bench_c5_r02b.log | cut -c1-1500
