# v6 attention A/B sweep (GS_ATTN_FLAGS bits: 1 softmax try_wait, 2 issuer try_wait, 4 early S, 8 P try_wait)
python paper_2604_04335_b200/build.py > /dev/null 2>&1 || exit 1
for F in ${FLAGS:-0 2 4 6 8 10}; do for P in ${POLYS:-0 2}; do
  echo -n "POLY8=$P FLAGS=$F: "; GS_ATTN_POLY8=$P GS_ATTN_FLAGS=$F timeout 100 python tools/kbench.py --attn --reps 5 --only "c4 720p sp8" 2>&1 | tail -1
done; done
