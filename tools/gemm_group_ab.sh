#!/bin/bash
# GEMM rasterisation band A/B (GS_GEMM_GROUP_M): DRAM bytes per launch of the config-4 SP=1 QKV and
# MLP-up GEMMs under ncu, and bench step breakdowns.
set -x
TAG=${TAG:-r01n}
python paper_2604_04335_b200/build.py > /dev/null 2>&1
for g in 4 8 16 32; do
  for c in "c4 sp1 qkv" "c2 down"; do
    f=$(echo $c | tr " " _)
    GS_GEMM_GROUP_M=$g timeout 300 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
      --clock-control none --csv -k regex:gemm -s 1 -c 1 python tools/kbench.py --gemm --only "$c" --reps 1 > gpurun_out/${TAG}_g${g}_$f.csv 2>&1
  done
done
for g in 16 8 32; do
  GS_GEMM_GROUP_M=$g timeout 600 python bench.py --workload t2v720 --no-cpu-baseline --steps 2 > gpurun_out/${TAG}_t2v720_g$g.jsonl 2>/dev/null
  GS_GEMM_GROUP_M=$g timeout 300 python bench.py --workload t2i1024 --no-cpu-baseline > gpurun_out/${TAG}_t2i_g$g.jsonl 2>/dev/null
done
