#!/bin/bash
# Programmatic dependent launch A/B on one box: GS_PDL=0 vs default (on); bit identity of whole
# steps, full GPU test suite with PDL on, bench breakdowns.
set -x
TAG=${TAG:-r01l}
python paper_2604_04335_b200/build.py > gpurun_out/${TAG}_build.log 2>&1
timeout 600 python tools/ab_step_bits.py dump /tmp/on.npz > gpurun_out/${TAG}_bits.log 2>&1
GS_PDL=0 timeout 600 python tools/ab_step_bits.py dump /tmp/off.npz >> gpurun_out/${TAG}_bits.log 2>&1
python tools/ab_step_bits.py compare /tmp/on.npz /tmp/off.npz >> gpurun_out/${TAG}_bits.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
for wl in t2i1024 t2v480; do
  for i in 1 2; do
    GS_PDL=0 timeout 600 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/${TAG}_${wl}_off_$i.jsonl 2>/dev/null
    timeout 600 python bench.py --workload $wl --no-cpu-baseline > gpurun_out/${TAG}_${wl}_on_$i.jsonl 2>/dev/null
  done
done
