#!/bin/bash
# Profiling pass run under gpurun (one GPU): launch list of one bench step + ncu --set full of
# the top kernels.  Outputs land in gpurun_out/ (scratch); summaries are copied to profiles/.
set -x
TAG=${TAG:-r01d}
python paper_2604_04335_b200/build.py >/dev/null
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:'gemm|attn|ln_modulate|qk_norm|gemv|sinusoid|f32_to_bf16' \
  --log-file gpurun_out/${TAG}_launches_${WL:-t2v720}.csv \
  python bench.py --workload ${WL:-t2v720} --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
  > gpurun_out/${TAG}_launches_bench.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn -s 1 -c 1 \
  -o gpurun_out/${TAG}_attn_c4sp8 -f python tools/kbench.py --attn --only "c4 720p sp8" --reps 1 \
  > gpurun_out/${TAG}_ncu_attn.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm -s 1 -c 1 \
  -o gpurun_out/${TAG}_gemm_c4sp8up -f python tools/kbench.py --gemm --only "c4 sp8 up" --reps 1 \
  > gpurun_out/${TAG}_ncu_gemm.log 2>&1
ls -la gpurun_out
# row kernels (LN + modulate, qk-RMSNorm + RoPE + pack) at the config-2 T2I and config-4 shapes
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:"ln_modulate|qk_norm" -s 4 -c 2 \
  -o gpurun_out/${TAG}_rowk_t2i -f python bench.py --workload t2i1024 --steps 1 --warmup 0 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/${TAG}_ncu_rowk_t2i.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:"ln_modulate|qk_norm" -s 4 -c 2 \
  -o gpurun_out/${TAG}_rowk_t2v720 -f python bench.py --workload t2v720 --steps 1 --warmup 0 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/${TAG}_ncu_rowk_t2v720.log 2>&1
ls -la gpurun_out
