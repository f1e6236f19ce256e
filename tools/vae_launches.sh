# Per-kernel launch list of one 720p/81f VAE decode (ncu duration only, cold serialised launches):
# which kernel classes the decode spends its time in.
mkdir -p gpurun_out/vl
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/vl/vae_launches.csv python tools/vae_profile.py --once > gpurun_out/vl/ncu.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/vl/ncu.log
