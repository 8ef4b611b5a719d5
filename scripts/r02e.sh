set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02e.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu_r02e.log | cut -c1-400
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02e.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_r02e.log
timeout 500 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02e.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r02e.log | cut -c1-4000
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --psa-kernel 2 --check 0 > gpurun_out/bench_r02e_round.log 2>&1; tail -1 gpurun_out/bench_r02e_round.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d.get(k) for k in ('value','ms_per_step','stage_ms_per_step')})"
timeout 600 python bench.py --dist iso --steps 5 --warmup 3 --no-cpu-baseline --check 4 > gpurun_out/bench_iso_r02e.log 2>&1; echo "iso rc=$?"; tail -1 gpurun_out/bench_iso_r02e.log | cut -c1-2500
