# Streaming warp-per-row qk (D > 1024) + grid-stride LN: parity (kernels, dit, text, fullsize), then t2i / t2v720
# bench lines for the default build (U = 2) and the U = 4 variant.
mkdir -p gpurun_out/rk2
export PYTHONUNBUFFERED=1
timeout -s KILL 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dit.py tests/test_gpu_text.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/rk2/test.log 2>&1
echo "test_rc=$?"; tail -2 gpurun_out/rk2/test.log
for v in def qku4; do
  lib=paper_2604_04335_b200/libgs.so; [ $v = qku4 ] && lib=paper_2604_04335_b200/libgs_qku4.so
  GS_LIB=$lib timeout -s KILL 400 python bench.py --workload t2i1024 --steps 20 --no-cpu-baseline --no-secondary > gpurun_out/rk2/t2i_$v.jsonl 2> gpurun_out/rk2/t2i_$v.err
  echo "t2i_$v rc=$?"
  GS_LIB=$lib timeout -s KILL 600 python bench.py --steps 3 --no-cpu-baseline --no-secondary > gpurun_out/rk2/t2v_$v.jsonl 2> gpurun_out/rk2/t2v_$v.err
  echo "t2v_$v rc=$?"
done
python - <<'PY'
import json
for f in ['t2i_def','t2v_def','t2i_qku4','t2v_qku4']:
    try:
        d=json.loads(open(f'gpurun_out/rk2/{f}.jsonl').read().strip().splitlines()[-1])
        b=d.get('breakdown_ms_per_step',{})
        print(f, d['value'], {k:b.get(k) for k in ('attention','ln_mod','qk_norm_rope','_gaps')}, {k:(v.get('frac'),v.get('avg_launch_us')) for k,v in d.get('kernels',{}).items() if k in ('ln_mod','qk_norm_rope')}, d['clocks']['sm_mhz'])
    except Exception as e: print(f, 'ERR', e)
PY
