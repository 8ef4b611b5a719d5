#!/bin/bash
# One GPU session: parity tests, smoke, bench line, ncu launch list + full captures of the two hot kernels.
# usage (from the repo root, on the GPU box): bash scripts/gpu_round.sh <tag> [tests|bench|ncu|all]
tag=${1:-r01}; what=${2:-all}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$tag.txt 2>&1
if [[ $what == all || $what == tests ]]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/pytest_gpu_$tag.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"
  tail -2 gpurun_out/smoke_$tag.log
fi
if [[ $what == all || $what == bench ]]; then
  timeout 600 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?"
  tail -1 gpurun_out/bench_$tag.log
  timeout 600 python bench.py --dist iso --steps 10 --no-cpu-baseline > gpurun_out/bench_iso_$tag.log 2>&1; echo "bench iso rc=$?"
  timeout 600 python scripts/config3_report.py gpurun_out/config3_$tag.json > /dev/null 2>&1; echo "config3 rc=$?"
  timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.log 2>&1; echo "ref rc=$?"
  tail -1 gpurun_out/bench_ref_$tag.log | cut -c1-300
fi
if [[ $what == all || $what == ncu ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
     --log-file gpurun_out/launches_$tag.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --dropin-groups 0 --check 0 \
     > gpurun_out/ncu_launch_bench_$tag.log 2>&1; echo "ncu launches rc=$?"
  for k in score_kernel psa_stream_kernel first_tranche_kernel; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 2 -c 1 \
       -o gpurun_out/${tag}_$k -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --dropin-groups 0 --check 0 \
       > gpurun_out/ncu_full_${k}_$tag.log 2>&1; echo "ncu $k rc=$?"
  done
  # isotropic keys: the dense hand-over kernels carry the step
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:"psa|score|dense|first" --launch-skip 7 -c 7 --csv --log-file gpurun_out/launches_iso_$tag.csv \
     python bench.py --steps 1 --warmup 3 --no-cpu-baseline --dropin-groups 0 --check 0 --dist iso > /dev/null 2>&1; echo "ncu iso rc=$?"
  for k in dense_k_kernel dense_v_kernel dense_decide_kernel; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 1 -c 1 \
       -o gpurun_out/${tag}_$k -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --dropin-groups 0 --check 0 --dist iso \
       > gpurun_out/ncu_full_${k}_$tag.log 2>&1; echo "ncu $k rc=$?"
  done
fi
