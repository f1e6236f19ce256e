# GEMM rasterisation band (GS_GEMM_GROUP_M development knob) at config 4: 16 (default) vs 8 vs 6, per-GEMM times
# from the bench kernels object (same box, interleaved).
mkdir -p gpurun_out/band
export PYTHONUNBUFFERED=1
for r in 1 2; do for g in 16 8 6; do
  GS_GEMM_GROUP_M=$g timeout -s KILL 600 python bench.py --steps 2 --no-cpu-baseline --no-secondary > gpurun_out/band/t2v_g${g}_$r.jsonl 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/band/t2v_g${g}_$r.jsonl').read().strip().splitlines()[-1]); k=d['kernels']
print('g$g r$r', d['value'], {x:k[x]['avg_launch_us'] for x in ('gemm_qkv','gemm_o','gemm_mlp_up','gemm_mlp_down')}, d['clocks']['sm_mhz'])"
done; done
