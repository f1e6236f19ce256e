# Round-2 (session 3) HEAD check: the whole -m gpu suite, smoke, then the default bench line.
mkdir -p gpurun_out/c1
export PYTHONUNBUFFERED=1
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -o faulthandler_timeout=240 --durations=15 > gpurun_out/c1/pytest.log 2>&1
echo "pytest_rc=$?"; tail -3 gpurun_out/c1/pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c1/smoke.log 2>&1
echo "smoke_rc=$?"; tail -2 gpurun_out/c1/smoke.log
timeout -s KILL 900 python bench.py > gpurun_out/c1/bench.jsonl 2> gpurun_out/c1/bench.err
echo "bench_rc=$?"; tail -2 gpurun_out/c1/bench.err
