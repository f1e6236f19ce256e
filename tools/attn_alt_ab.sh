mkdir -p gpurun_out/r3
export PYTHONUNBUFFERED=1
GS_LIB=paper_2604_04335_b200/libgs_alt.so timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k attention > gpurun_out/r3/alt_test.log 2>&1
echo "alt_test_rc=$?"; tail -2 gpurun_out/r3/alt_test.log
timeout -s KILL 180 python tools/attn_trace_alt.py > gpurun_out/r3/trace_alt.log 2>&1
echo "trace_rc=$?"; grep -A12 "tile period" gpurun_out/r3/trace_alt.log | head -14
for r in 1 2; do
  timeout -s KILL 200 python tools/kbench.py --attn --reps 5 > gpurun_out/r3/kb_v5_$r.log 2>&1
  timeout -s KILL 200 python tools/kbench.py --attn --reps 5 --lib paper_2604_04335_b200/libgs_alt.so > gpurun_out/r3/kb_alt_$r.log 2>&1
  grep "^attn" gpurun_out/r3/kb_v5_$r.log gpurun_out/r3/kb_alt_$r.log
done
