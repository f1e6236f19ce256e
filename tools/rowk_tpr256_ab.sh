#!/bin/bash
# Historical (kept for the record in profiles/r01_notes.md): the env knob it toggles was removed once
# the variant became the default, so today both arms run the same kernels.
# D > 2048 row kernels: 256 threads per row (GS_ROWK_TPR256=1) vs 128; GPU parity tests under 256,
# t2v720 bench breakdowns.
set -x
TAG=${TAG:-r01p}
python paper_2604_04335_b200/build.py > /dev/null 2>&1
GS_ROWK_TPR256=1 timeout 1200 python -m pytest tests/test_gpu_dit.py tests/test_gpu_text.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1
for i in 1 2; do
  timeout 600 python bench.py --workload t2v720 --no-cpu-baseline --steps 2 > gpurun_out/${TAG}_t2v720_t128_$i.jsonl 2>/dev/null
  GS_ROWK_TPR256=1 timeout 600 python bench.py --workload t2v720 --no-cpu-baseline --steps 2 > gpurun_out/${TAG}_t2v720_t256_$i.jsonl 2>/dev/null
done
