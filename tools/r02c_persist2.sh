# Persistent attention: co-resident cluster count as reported, and grid = SMs / 2 pairs (libgs_nsm.so) vs np.
mkdir -p gpurun_out/pa2
export PYTHONUNBUFFERED=1
GS_DEBUG=1 timeout -s KILL 200 python tools/kbench.py --attn --reps 3 --only "c4 720p sp8" 2>&1 | grep -E "\[gs\] attention|^attn" 
GS_LIB=paper_2604_04335_b200/libgs_nsm.so timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k attention > gpurun_out/pa2/test_attn.log 2>&1
echo "test_attn rc=$?"; tail -1 gpurun_out/pa2/test_attn.log
for r in 1 2; do
  for v in np nsm pa; do
    lib=paper_2604_04335_b200/libgs_$v.so; [ $v = pa ] && lib=paper_2604_04335_b200/libgs.so
    GS_DEBUG=1 timeout -s KILL 200 python tools/kbench.py --attn --reps 5 --lib $lib > gpurun_out/pa2/kb_${v}_$r.log 2>&1
    echo "== $v $r"; grep "^attn\|co-resident" gpurun_out/pa2/kb_${v}_$r.log | grep -v tiny
  done
done
