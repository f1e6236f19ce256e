# ssq only above D = 2048: config 2 back on the two-pass qk kernel (no QKV epilogue sums); parity + t2i / t2v lines.
mkdir -p gpurun_out/ssq3
export PYTHONUNBUFFERED=1
timeout -s KILL 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dit.py tests/test_gpu_text.py -m gpu -x -q > gpurun_out/ssq3/test.log 2>&1
echo "test rc=$?"; tail -1 gpurun_out/ssq3/test.log
timeout -s KILL 400 python bench.py --workload t2i1024 --steps 20 --no-cpu-baseline --no-secondary > gpurun_out/ssq3/t2i.jsonl 2>/dev/null
timeout -s KILL 600 python bench.py --steps 2 --no-cpu-baseline --no-secondary > gpurun_out/ssq3/t2v.jsonl 2>/dev/null
for w in t2i t2v; do python -c "
import json; d=json.loads(open('gpurun_out/ssq3/${w}.jsonl').read().strip().splitlines()[-1]); k=d['kernels']
print('$w', d['value'], {x:(k[x]['frac'],k[x]['avg_launch_us']) for x in ('ln_mod','qk_norm_rope','gemm_qkv')}, d['clocks']['sm_mhz'])"; done
