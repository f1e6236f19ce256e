#!/bin/bash
# Row-kernel A/B on one box: in-tree build (launch-bound variants via GS_ROWK_MINB_LN / _QK) vs
# scratch_old/libgs_head.so: bit identity of whole steps, t2i bench breakdowns.
set -x
TAG=${TAG:-r01h}
OLD=${OLD:-scratch_old/libgs_head.so}
python paper_2604_04335_b200/build.py > gpurun_out/${TAG}_build.log 2>&1
timeout 600 python tools/ab_step_bits.py dump /tmp/new.npz > gpurun_out/${TAG}_bits.log 2>&1
GS_LIB=$PWD/$OLD timeout 600 python tools/ab_step_bits.py dump /tmp/old.npz >> gpurun_out/${TAG}_bits.log 2>&1
python tools/ab_step_bits.py compare /tmp/new.npz /tmp/old.npz >> gpurun_out/${TAG}_bits.log 2>&1
for i in 1 2; do
  GS_LIB=$PWD/$OLD timeout 300 python bench.py --workload t2i1024 --no-cpu-baseline > gpurun_out/${TAG}_t2i_old_$i.jsonl 2>/dev/null
  for ln in 4 3; do for qk in 3 2; do
    GS_ROWK_MINB_LN=$ln GS_ROWK_MINB_QK=$qk timeout 300 python bench.py --workload t2i1024 --no-cpu-baseline > gpurun_out/${TAG}_t2i_ln${ln}qk${qk}_$i.jsonl 2>/dev/null
  done; done
done
