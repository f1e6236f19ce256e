# QKV GEMM epilogue sums of squares + single-pass qk kernel: parity (kernels, dit, text,
# fullsize), then t2v720 / t2i bench lines and an ncu of one qk launch + the QKV GEMM at config 4.
mkdir -p gpurun_out/ssq
export PYTHONUNBUFFERED=1
timeout -s KILL 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dit.py tests/test_gpu_text.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/ssq/test.log 2>&1
echo "test rc=$?"; tail -2 gpurun_out/ssq/test.log
timeout -s KILL 600 python bench.py --steps 2 --no-cpu-baseline --no-secondary > gpurun_out/ssq/t2v.jsonl 2>/dev/null
timeout -s KILL 400 python bench.py --workload t2i1024 --steps 20 --no-cpu-baseline --no-secondary > gpurun_out/ssq/t2i.jsonl 2>/dev/null
for w in t2v t2i; do python -c "
import json; d=json.loads(open('gpurun_out/ssq/${w}.jsonl').read().strip().splitlines()[-1]); k=d['kernels']
print('$w', d['value'], {x:(k[x]['frac'],k[x]['avg_launch_us']) for x in ('ln_mod','qk_norm_rope','gemm_qkv')}, d['clocks']['sm_mhz'])"; done
timeout -s KILL 600 /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:"qk_norm" -s 2 -c 1 \
  -o gpurun_out/ssq/qk_t2v720 -f python bench.py --workload t2v720 --steps 1 --warmup 0 --e2e-steps 1 --prof-steps 1 \
  --no-cpu-baseline --no-secondary > gpurun_out/ssq/ncu.log 2>&1
echo "ncu rc=$?"
