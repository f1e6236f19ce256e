# Same-box A/B of attention variants: in-tree libgs.so vs scratch_old/libgs_*.so (interleaved rounds).
python paper_2604_04335_b200/build.py > /dev/null
for round in 1 2; do
  for lib in "" scratch_old/libgs_*.so; do
    echo "== ${lib:-in-tree} (round $round)"
    timeout 200 python tools/kbench.py --attn --reps 5 --only "${ONLY:-c4 720p sp}" ${lib:+--lib $lib} 2>&1 | tail -3
  done
done
