timeout -s KILL 900 python -m pytest tests/test_gpu_configs.py -q -x --timeout=600 -k "bench" 2>&1 | tail -20
