# LN + modulate at D = 1536 (config 2): a warp per row (libgs_lnw.so) vs two warps per row (default).
mkdir -p gpurun_out/lnw
export PYTHONUNBUFFERED=1
GS_LIB=paper_2604_04335_b200/libgs_lnw.so timeout -s KILL 600 python -m pytest tests/test_gpu_dit.py -m gpu -x -q > gpurun_out/lnw/test.log 2>&1
echo "test rc=$?"; tail -1 gpurun_out/lnw/test.log
for r in 1 2; do for v in def lnw; do
  lib=paper_2604_04335_b200/libgs.so; [ $v = lnw ] && lib=paper_2604_04335_b200/libgs_lnw.so
  GS_LIB=$lib timeout -s KILL 400 python bench.py --workload t2i1024 --steps 20 --no-cpu-baseline --no-secondary > gpurun_out/lnw/t2i_${v}_$r.jsonl 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/lnw/t2i_${v}_$r.jsonl').read().strip().splitlines()[-1]); k=d['kernels']
print('$v $r', d['value'], {x:(k[x]['frac'],k[x]['avg_launch_us']) for x in ('ln_mod','qk_norm_rope')}, d['clocks']['sm_mhz'])"
done; done
