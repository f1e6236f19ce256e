# qk v2 (grid-stride rows, packed math, V read in place at SP = 1): parity tests, then t2i / t2v720 bench lines.
mkdir -p gpurun_out/rk
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dit.py tests/test_gpu_text.py -m gpu -x -q > gpurun_out/rk/test.log 2>&1
echo "test_rc=$?"; tail -2 gpurun_out/rk/test.log
timeout -s KILL 400 python bench.py --workload t2i1024 --steps 20 --no-cpu-baseline --no-secondary > gpurun_out/rk/t2i.jsonl 2> gpurun_out/rk/t2i.err
echo "t2i_rc=$?"
timeout -s KILL 600 python bench.py --steps 3 --no-cpu-baseline --no-secondary > gpurun_out/rk/t2v.jsonl 2> gpurun_out/rk/t2v.err
echo "t2v_rc=$?"
python - <<'PY'
import json
for f in ['t2i','t2v']:
    try:
        d=json.loads(open(f'gpurun_out/rk/{f}.jsonl').read().strip().splitlines()[-1])
        print(f, d['value'], d.get('breakdown_ms_per_step'), {k:(v.get('frac'),v.get('avg_launch_us')) for k,v in d.get('kernels',{}).items()}, d['clocks'])
    except Exception as e: print(f, 'ERR', e)
PY
