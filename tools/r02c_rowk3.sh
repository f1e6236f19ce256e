# qk streaming kernel with the pass-2 loads one chunk ahead: parity (kernels, dit), t2i / t2v720 bench lines.
mkdir -p gpurun_out/rk3
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dit.py -m gpu -x -q > gpurun_out/rk3/test.log 2>&1
echo "test_rc=$?"; tail -2 gpurun_out/rk3/test.log
timeout -s KILL 400 python bench.py --workload t2i1024 --steps 20 --no-cpu-baseline --no-secondary > gpurun_out/rk3/t2i.jsonl 2> gpurun_out/rk3/t2i.err
timeout -s KILL 600 python bench.py --steps 3 --no-cpu-baseline --no-secondary > gpurun_out/rk3/t2v.jsonl 2> gpurun_out/rk3/t2v.err
python - <<'PY'
import json
for f in ['t2i','t2v']:
    try:
        d=json.loads(open(f'gpurun_out/rk3/{f}.jsonl').read().strip().splitlines()[-1])
        b=d.get('breakdown_ms_per_step',{})
        print(f, d['value'], {k:b.get(k) for k in ('attention','ln_mod','qk_norm_rope','_gaps')}, {k:(v.get('frac'),v.get('avg_launch_us')) for k,v in d.get('kernels',{}).items() if k in ('ln_mod','qk_norm_rope')}, d['clocks']['sm_mhz'])
    except Exception as e: print(f, 'ERR', e)
PY
