mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_harness.py -m gpu -x -q > gpurun_out/pytest_harness.log 2>&1; echo "harness tests rc=$?"; tail -15 gpurun_out/pytest_harness.log
timeout -s KILL 900 python tools/complexity_study.py gpurun_out/complexity_study.json > gpurun_out/complexity.log 2>&1; echo "study rc=$?"; tail -45 gpurun_out/complexity.log
