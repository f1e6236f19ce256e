# Same-box A/B of the row kernels (libgs_prev.so = previous HEAD vs in-tree libgs.so) at the config-2 T2I
# step: step ms and the per-class breakdown (bench.py --workload t2i1024).
mkdir -p gpurun_out/rk
for r in 1 2; do
  for L in prev cur; do
    if [ $L = prev ]; then export GS_LIB=paper_2604_04335_b200/libgs_prev.so; else unset GS_LIB; fi
    timeout -s KILL 300 python bench.py --workload t2i1024 --steps 20 --warmup 3 --prof-steps 3 --no-cpu-baseline --no-secondary \
      > gpurun_out/rk/t2i_${L}_$r.jsonl 2> gpurun_out/rk/t2i_${L}_$r.err
    python -c "import json,sys; d=json.loads(open('gpurun_out/rk/t2i_${L}_$r.jsonl').read().strip().splitlines()[-1]); b=d['breakdown_ms_per_step']; print('$L', $r, d['value'], 'qk', b.get('qk_norm_rope'), 'ln', b.get('ln_mod'), 'attn', b.get('attention'))"
  done
done
unset GS_LIB
timeout -s KILL 600 python -m pytest tests/test_gpu_dit.py -m gpu -x -q -k "bit_exact or block_config2 or row_kernel" > gpurun_out/rk/tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/rk/tests.log
