# Round-2 GPU suite: the whole -m gpu test set (progress unbuffered, stack dump after 240 s in a test).
mkdir -p gpurun_out/s1
export PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,utilization.gpu --format=csv > gpurun_out/s1/smi.txt 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -x -v -o faulthandler_timeout=240 --durations=20 > gpurun_out/s1/pytest.log 2>&1
echo "pytest_rc=$?"
grep -E "passed|failed|error" gpurun_out/s1/pytest.log | tail -3
