timeout -s KILL 600 python -m pytest tests/test_gpu_configs.py -m gpu -x -q -k "page_locked or mirror or delta" > gpurun_out/pytest_delta.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_delta.log
python tools/exp_mirror.py > gpurun_out/e2e_delta3.log 2>&1; echo rc=$?; cat gpurun_out/e2e_delta3.log
