# Persistent attention (CTA pairs walk units with a static stride) vs the one-unit-per-CTA build (libgs_np.so):
# attention parity tests, kbench A/B, the step / SP bit-exactness suites, then t2i / t2v720 bench lines.
mkdir -p gpurun_out/pa
export PYTHONUNBUFFERED=1
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q -k attention > gpurun_out/pa/test_attn.log 2>&1
rc=$?; echo "test_attn rc=$rc"; tail -2 gpurun_out/pa/test_attn.log
[ $rc = 0 ] || exit 1
for r in 1 2; do
  for v in np pa; do
    lib=paper_2604_04335_b200/libgs.so; [ $v = np ] && lib=paper_2604_04335_b200/libgs_np.so
    timeout -s KILL 200 python tools/kbench.py --attn --reps 5 --lib $lib > gpurun_out/pa/kb_${v}_$r.log 2>&1
    echo "== $v $r"; grep "^attn" gpurun_out/pa/kb_${v}_$r.log | grep -v tiny
  done
done
timeout -s KILL 1200 python -m pytest tests/test_gpu_dit.py tests/test_gpu_text.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/pa/test.log 2>&1
echo "test rc=$?"; tail -2 gpurun_out/pa/test.log
timeout -s KILL 400 python bench.py --workload t2i1024 --steps 20 --no-cpu-baseline --no-secondary > gpurun_out/pa/t2i.jsonl 2> gpurun_out/pa/t2i.err
timeout -s KILL 600 python bench.py --steps 3 --no-cpu-baseline --no-secondary > gpurun_out/pa/t2v.jsonl 2> gpurun_out/pa/t2v.err
python - <<'PY'
import json
for f in ['t2i','t2v']:
    try:
        d=json.loads(open(f'gpurun_out/pa/{f}.jsonl').read().strip().splitlines()[-1])
        b=d.get('breakdown_ms_per_step',{})
        print(f, d['value'], d['roofline']['frac'], {k:b.get(k) for k in ('attention','ln_mod','qk_norm_rope','_gaps')}, {k:(v.get('frac'),v.get('avg_launch_us')) for k,v in d.get('kernels',{}).items() if k in ('ln_mod','qk_norm_rope')}, d['clocks']['sm_mhz'])
    except Exception as e: print(f, 'ERR', e)
PY
