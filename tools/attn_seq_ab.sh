# v5 softmax-phase variants (cuDNN-SDPA-like structure, profiles/r01_notes.md): SEQ = named-barrier
# phase lock between the softmax warpgroups, LSUM = row sum after the P hand-off, SPLITP = P in two
# halves, POLY8 = polynomial exp2 for 2 of 8 pairs.  Parity of the full combination, then kbench.
mkdir -p gpurun_out/seq
for v in cud SEQ; do
  GS_LIB=paper_2604_04335_b200/libgs_$v.so timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k attention > gpurun_out/seq/test_$v.log 2>&1
  echo "test_$v rc=$?"; tail -1 gpurun_out/seq/test_$v.log
done
for r in 1 2; do
  for v in v5 SEQ seqlsum seqsplit seqpoly seqsplitpoly cud; do
    lib=paper_2604_04335_b200/libgs_$v.so; [ $v = v5 ] && lib=paper_2604_04335_b200/libgs.so
    timeout -s KILL 200 python tools/kbench.py --attn --reps 5 --lib $lib > gpurun_out/seq/kb_${v}_$r.log 2>&1
    echo "== $v $r"; grep "^attn" gpurun_out/seq/kb_${v}_$r.log | grep -v tiny
  done
done
