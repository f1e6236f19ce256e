# In-step (power-capped) A/B of the attention variants on the config-4 step: default libgs.so (v5) vs
# libgs_alt.so (alternating-set variant, two MMA issuers).
mkdir -p gpurun_out/ia
for r in 1 2; do
  for L in v5 alt; do
    if [ $L = alt ]; then export GS_LIB=paper_2604_04335_b200/libgs_alt.so; else unset GS_LIB; fi
    timeout -s KILL 600 python bench.py --workload t2v720 --steps 2 --warmup 2 --prof-steps 1 --e2e-steps 1 \
      --no-cpu-baseline --no-secondary > gpurun_out/ia/t2v_${L}_$r.jsonl 2> gpurun_out/ia/t2v_${L}_$r.err
    python -c "import json; d=json.loads(open('gpurun_out/ia/t2v_${L}_$r.jsonl').read().strip().splitlines()[-1]); print('$L', $r, d['value'], 'attn', d['roofline']['achieved'], d['clocks']['sm_mhz'], d['clocks']['power_w'])"
  done
done
