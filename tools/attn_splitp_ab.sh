# v5 with the P hand-off split in two 64-key halves (libgs_splitp.so, -DGS_ATTN_SPLITP=1) vs v5.
mkdir -p gpurun_out/sp
GS_LIB=paper_2604_04335_b200/libgs_splitp.so timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k attention > gpurun_out/sp/test.log 2>&1
echo "test_rc=$?"; tail -1 gpurun_out/sp/test.log
for r in 1 2; do
  timeout -s KILL 200 python tools/kbench.py --attn --reps 5 > gpurun_out/sp/kb_v5_$r.log 2>&1
  timeout -s KILL 200 python tools/kbench.py --attn --reps 5 --lib paper_2604_04335_b200/libgs_splitp.so > gpurun_out/sp/kb_split_$r.log 2>&1
  grep "^attn" gpurun_out/sp/kb_v5_$r.log gpurun_out/sp/kb_split_$r.log | grep -v tiny
done
