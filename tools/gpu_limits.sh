mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_limits.py tests/test_harness.py -m gpu -x -q > gpurun_out/pytest_limits.log 2>&1; echo "limits tests rc=$?"; tail -15 gpurun_out/pytest_limits.log
timeout -s KILL 1200 python tools/convergence_study.py gpurun_out/convergence_study.json > gpurun_out/convergence.log 2>&1; echo "study rc=$?"; tail -20 gpurun_out/convergence.log
