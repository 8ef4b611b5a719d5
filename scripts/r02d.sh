mkdir -p gpurun_out
PSATTN_B200_LIB=$PWD/paper_2503_00392_b200/_lib/libpsattn_b200_dbg.so REPS=60 timeout 600 python scripts/debug_stream.py > gpurun_out/debug_stream.log 2>&1; echo rc=$?
grep -v "^\s*$" gpurun_out/debug_stream.log | grep -v Warning | head -30 | cut -c1-300
bash scripts/r02c.sh
