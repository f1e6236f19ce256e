# qk stream kernel as (row, tensor) units with L2 hints, 3 vs 4 CTAs per SM (libgs_qs3 / qs4), and the GEMM operand
# loads with L2 eviction hints on top (libgs_gh), vs the committed build: parity, then t2v720 / t2i bench lines.
mkdir -p gpurun_out/qs
export PYTHONUNBUFFERED=1
for v in qs4 gh; do
GS_LIB=paper_2604_04335_b200/libgs_$v.so timeout -s KILL 700 python -m pytest tests/test_gpu_dit.py tests/test_gpu_kernels.py -m gpu -x -q > gpurun_out/qs/test_$v.log 2>&1
echo "test $v rc=$?"; tail -1 gpurun_out/qs/test_$v.log
done
for v in def qs3 qs4 gh; do
  lib=paper_2604_04335_b200/libgs_$v.so; [ $v = def ] && lib=paper_2604_04335_b200/libgs.so
  GS_LIB=$lib timeout -s KILL 600 python bench.py --steps 2 --no-cpu-baseline --no-secondary > gpurun_out/qs/t2v_$v.jsonl 2>/dev/null
  GS_LIB=$lib timeout -s KILL 400 python bench.py --workload t2i1024 --steps 20 --no-cpu-baseline --no-secondary > gpurun_out/qs/t2i_$v.jsonl 2>/dev/null
  for w in t2v t2i; do python -c "
import json; d=json.loads(open('gpurun_out/qs/${w}_$v.jsonl').read().strip().splitlines()[-1]); k=d['kernels']
print('$w $v', d['value'], {x:(k[x]['frac'],k[x]['avg_launch_us']) for x in ('ln_mod','qk_norm_rope','gemm_qkv','gemm_mlp_down')}, d['clocks']['sm_mhz'], d['clocks']['power_w'])"; done
done
