#!/bin/bash
# Round validation at HEAD (TAG names the round): GPU tests, smoke, bench lines (all workloads + reference arm),
# the launch list of the default bench command, ncu --set full of attention and the top GEMM.
set -x
TAG=${TAG:-r01s}
NCU=/usr/local/cuda/bin/ncu
python paper_2604_04335_b200/build.py > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.jsonl 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py > gpurun_out/${TAG}_bench_repeat.jsonl 2> /dev/null
timeout 600 python bench.py --workload t2i1024 > gpurun_out/${TAG}_bench_t2i.jsonl 2> gpurun_out/${TAG}_bench_t2i.err
timeout 600 python bench.py --workload t2v480 > gpurun_out/${TAG}_bench_t2v480.jsonl 2> /dev/null
timeout 900 python bench.py --workload t2v720_text_cfg --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_t2v720_text_cfg.jsonl 2> /dev/null
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.jsonl 2> /dev/null
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  -k regex:'gemm|attn|ln_modulate|qk_norm|gemv|sinusoid|f32_to_bf16' \
  --log-file gpurun_out/${TAG}_launches_t2v720.csv \
  python bench.py --workload t2v720 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/${TAG}_launches_bench.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:attn -s 1 -c 1 \
  -o gpurun_out/${TAG}_attn_c4sp8 -f python tools/kbench.py --attn --only "c4 720p sp8" --reps 1 > gpurun_out/${TAG}_ncu_attn.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:gemm -s 1 -c 1 \
  -o gpurun_out/${TAG}_gemm_c4sp8up -f python tools/kbench.py --gemm --only "c4 sp8 up" --reps 1 > gpurun_out/${TAG}_ncu_gemm.log 2>&1
