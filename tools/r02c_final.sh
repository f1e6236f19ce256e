# Round-2 (session 3) check of the committed state: full -m gpu suite, smoke, default bench line, launch list of
# one t2v720 step, ncu --set full of the row kernels (t2i and t2v720 shapes).  Outputs in gpurun_out/f1.
mkdir -p gpurun_out/f1
export PYTHONUNBUFFERED=1
NCU=/usr/local/cuda/bin/ncu
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -o faulthandler_timeout=240 > gpurun_out/f1/pytest.log 2>&1
echo "pytest_rc=$?"; tail -2 gpurun_out/f1/pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1/smoke.log 2>&1
echo "smoke_rc=$?"; tail -1 gpurun_out/f1/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/f1/bench.jsonl 2> gpurun_out/f1/bench.err
echo "bench_rc=$?"
timeout -s KILL 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:'gemm|attn|ln_modulate|qk_norm|gemv|sinusoid|f32_to_bf16|rng' \
  --log-file gpurun_out/f1/launches_t2v720.csv \
  python bench.py --workload t2v720 --steps 1 --warmup 3 --e2e-steps 1 --prof-steps 1 --no-cpu-baseline --no-secondary \
  > gpurun_out/f1/launches_bench.log 2>&1
echo "launches rc=$?"
timeout -s KILL 600 $NCU --set full --clock-control none --import-source on -k regex:"ln_modulate|qk_norm" -s 4 -c 2 \
  -o gpurun_out/f1/rowk_t2i -f python bench.py --workload t2i1024 --steps 1 --warmup 0 --e2e-steps 1 --prof-steps 1 \
  --no-cpu-baseline --no-secondary > gpurun_out/f1/ncu_rowk_t2i.log 2>&1
echo "rowk t2i rc=$?"
timeout -s KILL 900 $NCU --set full --clock-control none --import-source on -k regex:"ln_modulate|qk_norm" -s 4 -c 2 \
  -o gpurun_out/f1/rowk_t2v720 -f python bench.py --workload t2v720 --steps 1 --warmup 0 --e2e-steps 1 --prof-steps 1 \
  --no-cpu-baseline --no-secondary > gpurun_out/f1/ncu_rowk_t2v720.log 2>&1
echo "rowk t2v rc=$?"
ls -la gpurun_out/f1
