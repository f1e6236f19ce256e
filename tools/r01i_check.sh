set -x
python paper_2604_04335_b200/build.py > gpurun_out/r01i_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_dit.py -m gpu -x -q -k degenerate > gpurun_out/r01i_degenerate.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r01i_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r01i_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01i_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r01i_bench.jsonl 2> gpurun_out/r01i_bench.err
timeout 600 python bench.py --workload t2i1024 > gpurun_out/r01i_bench_t2i.jsonl 2> gpurun_out/r01i_bench_t2i.err
timeout 600 python bench.py --workload t2v480 > gpurun_out/r01i_bench_t2v480.jsonl 2> gpurun_out/r01i_bench_t2v480.err
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:'gemm|attn|ln_modulate|qk_norm|gemv|sinusoid|f32_to_bf16' \
  --log-file gpurun_out/r01i_launches_t2i1024.csv \
  python bench.py --workload t2i1024 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r01i_launches_bench.log 2>&1
timeout 600 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"ln_modulate|qk_norm" -s 4 -c 2 \
  -o gpurun_out/r01i_rowk_t2i -f python bench.py --workload t2i1024 --steps 1 --warmup 0 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/r01i_ncu_rowk_t2i.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"ln_modulate|qk_norm" -s 4 -c 2 \
  -o gpurun_out/r01i_rowk_t2v720 -f python bench.py --workload t2v720 --steps 1 --warmup 0 --e2e-steps 0 \
  --no-cpu-baseline > gpurun_out/r01i_ncu_rowk_t2v720.log 2>&1
