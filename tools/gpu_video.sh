mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_configs.py -m gpu -x -q -k "video_host" > gpurun_out/pytest_video.log 2>&1; echo "video tests rc=$?"; tail -15 gpurun_out/pytest_video.log
timeout -s KILL 600 python bench.py --steps 50 > gpurun_out/bench_video.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_video.log").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"]); print(json.dumps(d["e2e"]))
PY
