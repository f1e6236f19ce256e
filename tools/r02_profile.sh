# Round-2 profiling pass (one GPU): launch list of one bench step (ncu gpu__time_duration, cold-cache,
# serialised), ncu --set full of the top kernels: attention (c4 SP=8), the row kernels (c2 and c4), the
# VAE conv at its largest stage shape.  Outputs in gpurun_out/p2; summaries go to profiles/.
mkdir -p gpurun_out/p2
export PYTHONUNBUFFERED=1
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:'gemm|attn|ln_modulate|qk_norm|gemv|sinusoid|f32_to_bf16|rng' \
  --log-file gpurun_out/p2/launches_t2v720.csv \
  python bench.py --workload t2v720 --steps 1 --warmup 3 --e2e-steps 1 --prof-steps 1 --no-cpu-baseline --no-secondary \
  > gpurun_out/p2/launches_bench.log 2>&1
echo "launches rc=$?"
timeout -s KILL 600 $NCU --set full --clock-control none --import-source on -k regex:"ln_modulate|qk_norm" -s 4 -c 2 \
  -o gpurun_out/p2/rowk_t2i -f python bench.py --workload t2i1024 --steps 1 --warmup 0 --e2e-steps 1 --prof-steps 1 \
  --no-cpu-baseline --no-secondary > gpurun_out/p2/ncu_rowk_t2i.log 2>&1
echo "rowk t2i rc=$?"
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on -k regex:"ln_modulate|qk_norm" -s 4 -c 2 \
  -o gpurun_out/p2/rowk_t2v720 -f python bench.py --workload t2v720 --steps 1 --warmup 0 --e2e-steps 1 --prof-steps 1 \
  --no-cpu-baseline --no-secondary > gpurun_out/p2/ncu_rowk_t2v720.log 2>&1
echo "rowk t2v rc=$?"
timeout -s KILL 600 python tools/vae_profile.py > gpurun_out/p2/vae_profile.log 2>&1
echo "vae prof rc=$?"; tail -30 gpurun_out/p2/vae_profile.log
timeout -s KILL 600 $NCU --set full --clock-control none --import-source on -k regex:"conv3d" -s 40 -c 1 \
  -o gpurun_out/p2/conv_vae -f python tools/vae_profile.py --once > gpurun_out/p2/ncu_conv.log 2>&1
echo "conv ncu rc=$?"
ls -la gpurun_out/p2
