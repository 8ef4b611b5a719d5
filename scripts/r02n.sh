bash scripts/ab_stream.sh main pf2 pf3 look3
PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_sprof.so timeout 300 python bench.py --warmup 3 --steps 5 --no-cpu-baseline --check 0 --dropin-units 0 2>&1 | grep stream_prof
