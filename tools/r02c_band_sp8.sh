# GEMM band at the config-4 SP = 8 shapes (M = 9450: A fits L2): 16 (default) vs the whole M range (64).
mkdir -p gpurun_out/bsp8
for r in 1 2; do for g in 16 64; do
  GS_GEMM_GROUP_M=$g timeout -s KILL 300 python tools/kbench.py --gemm --reps 10 --only "c4 sp8" > gpurun_out/bsp8/kb_g${g}_$r.log 2>&1
  echo "== g$g r$r"; grep -i "^gemm" gpurun_out/bsp8/kb_g${g}_$r.log
done; done
for g in 16 64; do
  GS_GEMM_GROUP_M=$g timeout -s KILL 300 /usr/local/cuda/bin/ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm -s 2 -c 4 python tools/kbench.py --gemm --reps 1 --only "c4 sp8" > gpurun_out/bsp8/ncu_g$g.log 2>&1
  echo "== ncu g$g"; grep -E "dram__bytes|gpu__time_duration" gpurun_out/bsp8/ncu_g$g.log | head -12
done
