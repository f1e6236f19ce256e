python paper_2604_04335_b200/build.py >/dev/null
for P in 0 2 3 4; do
  echo "== POLY8=$P"
  GS_ATTN_POLY8=$P python tools/attn_trace.py 2>&1 | grep -E "period|T_s \(|Pdone -> issue|j=21 WG" 
  GS_ATTN_POLY8=$P python tools/kbench.py --attn --only "c4 720p sp" --reps 3 2>&1
done
python tools/kbench.py --attn --only "c4 720p sp8" --reps 3 --torch
