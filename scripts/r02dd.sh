mkdir -p gpurun_out
for k in dense_decide_kernel dense_k_kernel; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 1 -c 1 \
     -o gpurun_out/r02s_$k -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --dist iso --check 0 --graph 0 --dropin-units 0 \
     > gpurun_out/ncu_full_${k}_r02s.log 2>&1; echo "ncu $k rc=$?"
done
