# single-pass qk (GEMM sums of squares): 4 CTAs per SM (64 registers, default) vs 3 (libgs_m3.so), same box.
mkdir -p gpurun_out/ssq2
export PYTHONUNBUFFERED=1
timeout -s KILL 600 python -m pytest tests/test_gpu_dit.py -m gpu -x -q > gpurun_out/ssq2/test.log 2>&1
echo "test rc=$?"; tail -1 gpurun_out/ssq2/test.log
for r in 1 2; do for v in def m3; do
  lib=paper_2604_04335_b200/libgs.so; [ $v = m3 ] && lib=paper_2604_04335_b200/libgs_m3.so
  GS_LIB=$lib timeout -s KILL 600 python bench.py --steps 2 --no-cpu-baseline --no-secondary > gpurun_out/ssq2/t2v_${v}_$r.jsonl 2>/dev/null
  GS_LIB=$lib timeout -s KILL 400 python bench.py --workload t2i1024 --steps 20 --no-cpu-baseline --no-secondary > gpurun_out/ssq2/t2i_${v}_$r.jsonl 2>/dev/null
  for w in t2v t2i; do python -c "
import json; d=json.loads(open('gpurun_out/ssq2/${w}_${v}_$r.jsonl').read().strip().splitlines()[-1]); k=d['kernels']
print('$w $v $r', d['value'], {x:(k[x]['frac'],k[x]['avg_launch_us']) for x in ('ln_mod','qk_norm_rope','gemm_qkv')}, d['clocks']['sm_mhz'])"; done
done; done
