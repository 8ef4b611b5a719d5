mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02x.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_r02x.log | cut -c1-300
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02x.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r02x.log
timeout 600 python bench.py > gpurun_out/bench_r02x.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_r02x.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: d.get(k) for k in ('value','ms_per_step','stage_ms_per_step','e2e','e2e_serial','e2e_dropin','parity_ok','clocks','roofline')})"
