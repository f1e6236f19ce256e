#!/bin/bash
# Timing-only: the PS schedule with the PV MMA reading P from TMEM (values wrong) vs the real PS
# variant vs v5 -- isolates the SS-PV MMA's in-situ cost.
python paper_2604_04335_b200/build.py > /dev/null 2>&1
for r in 1 2; do
  echo "== v5 ($r)"; timeout 200 python tools/kbench.py --attn --reps 5 --only "c4 720p sp8" 2>&1 | grep "^attn"
  echo "== PS ($r)"; GS_ATTN_PS=1 timeout 200 python tools/kbench.py --attn --reps 5 --only "c4 720p sp8" 2>&1 | grep "^attn"
  echo "== PS schedule, TS PV ($r)"; GS_ATTN_PS=1 timeout 200 python tools/kbench.py --attn --reps 5 --only "c4 720p sp8" --lib scratch_old/libgs_ps_tspv.so 2>&1 | grep "^attn"
done
