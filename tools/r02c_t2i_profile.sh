# Config-2 (t2i1024) launch list of one step and an ncu --set full of its attention launch.
mkdir -p gpurun_out/t2ip
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:'gemm|attn|ln_modulate|qk_norm|gemv|sinusoid|f32_to_bf16' --log-file gpurun_out/t2ip/launches_t2i.csv \
  python bench.py --workload t2i1024 --steps 1 --warmup 1 --e2e-steps 1 --prof-steps 1 --no-cpu-baseline --no-secondary \
  > gpurun_out/t2ip/launches.log 2>&1
echo "launches rc=$?"
timeout -s KILL 600 $NCU --set full --clock-control none -k regex:attn -s 3 -c 1 -o gpurun_out/t2ip/attn_t2i -f \
  python bench.py --workload t2i1024 --steps 1 --warmup 0 --e2e-steps 1 --prof-steps 1 --no-cpu-baseline --no-secondary \
  > gpurun_out/t2ip/ncu.log 2>&1
echo "ncu rc=$?"
