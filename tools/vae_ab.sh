# VAE: conv parity (incl. 32-channel K blocks) + decoders vs oracle, then the decode profile.
mkdir -p gpurun_out/va
export PYTHONUNBUFFERED=1
timeout -s KILL 900 python -m pytest tests/test_gpu_vae.py -m gpu -x -v -s -o faulthandler_timeout=240 > gpurun_out/va/vae.log 2>&1
echo "vae_rc=$?"; grep -E "rel-L2|passed|failed|Error" gpurun_out/va/vae.log | tail -12
timeout -s KILL 600 python tools/vae_profile.py > gpurun_out/va/vae_profile.log 2>&1
echo "prof rc=$?"; cat gpurun_out/va/vae_profile.log
