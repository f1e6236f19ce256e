# ncu --set full of the alternating-set attention variant (libgs_alt.so) at the c4 SP=8 shape.
mkdir -p gpurun_out/na
GS_LIB=paper_2604_04335_b200/libgs_alt.so timeout -s KILL 600 /usr/local/cuda/bin/ncu --set full --clock-control none \
  --import-source on -k regex:attn -s 1 -c 1 -o gpurun_out/na/attn_alt_c4sp8 -f \
  python tools/kbench.py --attn --only "c4 720p sp8" --reps 1 > gpurun_out/na/ncu.log 2>&1
echo "ncu rc=$?"
