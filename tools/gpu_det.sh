timeout -s KILL 400 python -m pytest tests/test_gpu_detect.py -q -x --timeout=120 2>&1 | tail -15
