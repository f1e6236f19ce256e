python paper_2604_04335_b200/build.py > /dev/null 2>&1
# Historical (kept for the record in profiles/r01_notes.md): the env knob it toggles was removed once
# the variant became the default, so today both arms run the same kernels.
GS_ROWK_TPR64=1 timeout 900 python -m pytest tests/test_gpu_dit.py tests/test_gpu_text.py -m gpu -x -q > gpurun_out/t64_pytest.log 2>&1
for i in 1 2; do
  timeout 300 python bench.py --workload t2i1024 --no-cpu-baseline > gpurun_out/t64_t2i_w32_$i.jsonl 2>/dev/null
  GS_ROWK_TPR64=1 timeout 300 python bench.py --workload t2i1024 --no-cpu-baseline > gpurun_out/t64_t2i_w64_$i.jsonl 2>/dev/null
done
GS_ROWK_TPR64=1 timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:"ln_modulate|qk_norm" -s 4 -c 2 \
  -o gpurun_out/t64_rowk_t2i -f python bench.py --workload t2i1024 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/t64_ncu.log 2>&1
