#!/bin/bash
# ncu --set full captures of the attention kernel at the shapes bench.py times (one launch each);
# dram bytes per launch feed bench.py's roofline "traffic" via profiles/attention_traffic.json.
TAG=${TAG:-r01}
NCU=/usr/local/cuda/bin/ncu
python paper_2604_04335_b200/build.py >/dev/null
for case in "c4 720p sp1 40h" "c4 720p sp8 5h" "c2 4x4096 12h" "c3 480p sp1 12h"; do
  f=$(echo "$case" | tr ' ' '_')
  timeout 600 $NCU --set full --clock-control none -k regex:attn -s 1 -c 1 -o gpurun_out/${TAG}_traffic_$f -f \
    python tools/kbench.py --attn --only "$case" --reps 1 > /dev/null 2>&1
done
ls gpurun_out
