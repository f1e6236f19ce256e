# Round-2 GPU pass: VAE parity, the alternating-set attention trace and A/B, then the bench line.
mkdir -p gpurun_out/r2
export PYTHONUNBUFFERED=1
timeout -s KILL 600 python -m pytest tests/test_gpu_vae.py -m gpu -x -v -s -o faulthandler_timeout=240 > gpurun_out/r2/vae.log 2>&1
echo "vae_rc=$?"; grep -E "rel-L2|passed|failed" gpurun_out/r2/vae.log | tail -8
timeout -s KILL 180 python tools/attn_trace_alt.py > gpurun_out/r2/trace_alt.log 2>&1
echo "trace_rc=$?"
for r in 1 2; do
  timeout -s KILL 200 python tools/kbench.py --attn --reps 5 --only "c4 720p sp8" > gpurun_out/r2/kb_v5_$r.log 2>&1
  timeout -s KILL 200 python tools/kbench.py --attn --reps 5 --only "c4 720p sp8" --lib paper_2604_04335_b200/libgs_alt.so > gpurun_out/r2/kb_alt_$r.log 2>&1
  grep "^attn" gpurun_out/r2/kb_v5_$r.log gpurun_out/r2/kb_alt_$r.log
done
timeout -s KILL 900 python bench.py > gpurun_out/r2/bench.jsonl 2> gpurun_out/r2/bench.err
echo "bench_rc=$?"; tail -2 gpurun_out/r2/bench.err
