timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout=300 -k "seam or incremental" 2>&1 | tail -15
timeout -s KILL 1200 python -m pytest tests/ref_suite -q --timeout=600 2>&1 | tail -3
