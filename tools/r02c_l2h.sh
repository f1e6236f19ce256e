# qk streaming kernel with L2 eviction-priority hints (pass 1 evict-last, pass 2 evict-first; libgs_l2h.so) vs the
# committed build: qk parity tests, bench kernel fractions at config 4 / config 2, ncu DRAM bytes of one qk launch.
mkdir -p gpurun_out/l2h
export PYTHONUNBUFFERED=1
GS_LIB=paper_2604_04335_b200/libgs_l2h.so timeout -s KILL 600 python -m pytest tests/test_gpu_dit.py -m gpu -x -q > gpurun_out/l2h/test.log 2>&1
echo "test rc=$?"; tail -1 gpurun_out/l2h/test.log
for v in def l2h; do
  lib=paper_2604_04335_b200/libgs.so; [ $v = l2h ] && lib=paper_2604_04335_b200/libgs_l2h.so
  GS_LIB=$lib timeout -s KILL 600 python bench.py --steps 2 --no-cpu-baseline --no-secondary > gpurun_out/l2h/t2v_$v.jsonl 2>/dev/null
  GS_LIB=$lib timeout -s KILL 400 python bench.py --workload t2i1024 --steps 20 --no-cpu-baseline --no-secondary > gpurun_out/l2h/t2i_$v.jsonl 2>/dev/null
  for w in t2v t2i; do python -c "
import json; d=json.loads(open('gpurun_out/l2h/${w}_$v.jsonl').read().strip().splitlines()[-1]); k=d['kernels']
print('$w $v', d['value'], {x:(k[x]['frac'],k[x]['avg_launch_us']) for x in ('ln_mod','qk_norm_rope')}, d['clocks']['sm_mhz'])"; done
done
GS_LIB=paper_2604_04335_b200/libgs_l2h.so timeout -s KILL 600 /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:"qk_norm" -s 2 -c 1 \
  -o gpurun_out/l2h/qk_t2v720 -f python bench.py --workload t2v720 --steps 1 --warmup 0 --e2e-steps 1 --prof-steps 1 \
  --no-cpu-baseline --no-secondary > gpurun_out/l2h/ncu.log 2>&1
echo "ncu rc=$?"
