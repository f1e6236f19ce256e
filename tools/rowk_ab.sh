#!/bin/bash
# Row-kernel A/B on one box: in-tree build vs scratch_old/libgs_head.so (the previous commit):
# bit identity of whole steps (tools/ab_step_bits.py), bench breakdowns per workload.
set -x
TAG=${TAG:-r01j}
OLD=${OLD:-scratch_old/libgs_head.so}
python paper_2604_04335_b200/build.py > gpurun_out/${TAG}_build.log 2>&1
timeout 600 python tools/ab_step_bits.py dump /tmp/new.npz > gpurun_out/${TAG}_bits.log 2>&1
GS_LIB=$PWD/$OLD timeout 600 python tools/ab_step_bits.py dump /tmp/old.npz >> gpurun_out/${TAG}_bits.log 2>&1
python tools/ab_step_bits.py compare /tmp/new.npz /tmp/old.npz >> gpurun_out/${TAG}_bits.log 2>&1
for wl in ${WLS:-t2i1024 t2v480}; do
  for i in 1 2; do
    GS_LIB=$PWD/$OLD timeout 900 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/${TAG}_${wl}_old_$i.jsonl 2>/dev/null
    timeout 900 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/${TAG}_${wl}_new_$i.jsonl 2>/dev/null
  done
done
