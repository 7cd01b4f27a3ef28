timeout -s KILL 900 python -m pytest tests/test_gpu_deadlock.py -q -x > gpurun_out/pytest_dl.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_dl.log
timeout -s KILL 600 python tools/exp_deadlock.py --reps 2 2>&1 | tee gpurun_out/exp_dl.json
timeout -s KILL 600 python tools/exp_deadlock.py --reps 1 --untracked 2>&1 | tail -3
