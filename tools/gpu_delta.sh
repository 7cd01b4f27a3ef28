mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_configs.py -m gpu -x -q -k "delta or mirror or pinned or concurrent" > gpurun_out/pytest_delta.log 2>&1; echo "delta tests rc=$?"; tail -15 gpurun_out/pytest_delta.log
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout -s KILL 600 python bench.py --steps 50 > gpurun_out/bench_delta.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_delta.log").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"]); print(json.dumps(d["e2e"]))
PY
python tools/exp_mirror.py > gpurun_out/e2e_delta.log 2>&1; echo "exp_e2e rc=$?"; tail -30 gpurun_out/e2e_delta.log
