mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:psa_stream_kernel --launch-skip 3 -c 1 \
     -o gpurun_out/r02k_stream -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --check 0 --graph 0 --dropin-units 0 \
     > gpurun_out/ncu_full_stream_r02k.log 2>&1; echo "ncu rc=$?"
