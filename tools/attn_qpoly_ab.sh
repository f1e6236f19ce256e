# v5 with the issuer's SMSP (TMEM lane quarter 1) softmax warps on the FMA-pipe exp2 (QPOLY of every 8
# pairs) vs v5: fewer MUFU instructions ahead of the issuer's mbarrier tests in that SMSP's MIO queue.
mkdir -p gpurun_out/qp
L=paper_2604_04335_b200
for v in GS_ATTN_QPOLY8 GS_ATTN_QPOLY4 GS_ATTN_QPOLY8GS_ATTN_QPQ5; do
  GS_LIB=$L/libgs_$v.so timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k attention > gpurun_out/qp/test_$v.log 2>&1
  echo "test_$v rc=$?"; tail -1 gpurun_out/qp/test_$v.log
done
for r in 1 2; do
  for v in v5 GS_ATTN_QPOLY8 GS_ATTN_QPOLY4 GS_ATTN_QPOLY8GS_ATTN_QPQ5; do
    lib=$L/libgs_$v.so; [ $v = v5 ] && lib=$L/libgs.so
    timeout -s KILL 200 python tools/kbench.py --attn --reps 5 --lib $lib > gpurun_out/qp/kb_${v}_$r.log 2>&1
    echo "== $v $r"; grep "^attn" gpurun_out/qp/kb_${v}_$r.log | grep -v tiny
  done
done
