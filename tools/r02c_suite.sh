# Full -m gpu suite + smoke at HEAD.
mkdir -p gpurun_out/s2
export PYTHONUNBUFFERED=1
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -o faulthandler_timeout=240 > gpurun_out/s2/pytest.log 2>&1
echo "pytest_rc=$?"; tail -2 gpurun_out/s2/pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2/smoke.log 2>&1
echo "smoke_rc=$?"; tail -1 gpurun_out/s2/smoke.log
