# Persistent attention slowdown: the same kernel code with one unit per CTA pair (libgs_one.so) vs np vs pa.
mkdir -p gpurun_out/pa3
for r in 1 2; do
  for v in np one pa; do
    lib=paper_2604_04335_b200/libgs_$v.so; [ $v = pa ] && lib=paper_2604_04335_b200/libgs.so
    timeout -s KILL 200 python tools/kbench.py --attn --reps 5 --lib $lib > gpurun_out/pa3/kb_${v}_$r.log 2>&1
    echo "== $v $r"; grep "^attn" gpurun_out/pa3/kb_${v}_$r.log | grep -v tiny
  done
done
