python paper_2604_04335_b200/build.py >/dev/null
for e in bf16 resid; do python tools/kbench.py --gemm --only "c2 o" --epi $e --reps 20 > gpurun_out/go_kb_$e.log 2>&1; done
python tools/kbench.py --gemm --only "c2" --epi bf16 --reps 10 > gpurun_out/go_kb_c2.log 2>&1
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:gemm -s 1 -c 1 \
  -o gpurun_out/go_c2o_resid -f python tools/kbench.py --gemm --only "c2 o" --epi resid --reps 1 > gpurun_out/go_ncu.log 2>&1
