# VAE decode with the norm fused into the conv epilogues: parity (incl. the full-size 720p windows),
# decode time, launch list.
mkdir -p gpurun_out/vf
timeout -s KILL 900 python -m pytest tests/test_gpu_vae.py -m gpu -x -q -p no:cacheprovider > gpurun_out/vf/test.log 2>&1
echo "test rc=$?"; tail -3 gpurun_out/vf/test.log
for r in 1 2; do timeout -s KILL 300 python tools/vae_profile.py > gpurun_out/vf/prof_$r.log 2>&1; head -1 gpurun_out/vf/prof_$r.log; done
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/vf/vae_launches.csv python tools/vae_profile.py --once > gpurun_out/vf/ncu.log 2>&1
echo "ncu rc=$?"
