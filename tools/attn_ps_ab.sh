#!/bin/bash
# Round-2 experiment: attention with P in shared memory (GS_ATTN_PS=1) -- correctness on the GPU
# attention tests, then same-box kbench A/B against the default v5 kernel.
python paper_2604_04335_b200/build.py > /dev/null 2>&1
GS_ATTN_PS=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k attention > gpurun_out/ps_test.log 2>&1
echo "rc=$?" >> gpurun_out/ps_test.log
for r in 1 2; do
  timeout 200 python tools/kbench.py --attn --reps 5 --only "c" > gpurun_out/ps_kb_default_$r.log 2>&1
  GS_ATTN_PS=1 timeout 200 python tools/kbench.py --attn --reps 5 --only "c" > gpurun_out/ps_kb_ps_$r.log 2>&1
done
