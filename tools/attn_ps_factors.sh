python paper_2604_04335_b200/build.py > /dev/null 2>&1
for r in 1 2; do
  echo "== default ($r)"; timeout 200 python tools/kbench.py --attn --reps 5 --only "c4 720p sp8" 2>&1 | grep "^attn"
  echo "== PS ($r)"; GS_ATTN_PS=1 timeout 200 python tools/kbench.py --attn --reps 5 --only "c4 720p sp8" 2>&1 | grep "^attn"
  echo "== ring 3/2, no PS ($r)"; timeout 200 python tools/kbench.py --attn --reps 5 --only "c4 720p sp8" --lib scratch_old/libgs_ring32.so 2>&1 | grep "^attn"
  echo "== PS without proxy fence ($r)"; GS_ATTN_PS=1 timeout 200 python tools/kbench.py --attn --reps 5 --only "c4 720p sp8" --lib scratch_old/libgs_psnofence.so 2>&1 | grep "^attn"
done
