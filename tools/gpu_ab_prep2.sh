# A/B: prep guide loop two pixels per thread (new libgf_b200.so) vs one (libgf_b200_old.so).
mkdir -p gpurun_out
CMD="python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu --no-extras"
for rep in 1 2; do
  for v in old new; do
    if [ $v = old ]; then L=paper_1611_05319_b200/libgf_b200_old.so; else L=paper_1611_05319_b200/libgf_b200.so; fi
    GF_B200_LIB=$L timeout 300 $CMD > gpurun_out/ab_$v.log 2>&1
    python - "$v" <<'PY'
import json, sys
l = [x for x in open(f"gpurun_out/ab_{sys.argv[1]}.log") if x.startswith("{")][-1]
d = json.loads(l); c = d["config"]
print(sys.argv[1], round(d["ms_per_step"], 5), c["timeline"]["prep"], c["timeline"]["shells"]["start_us"], "c5", round(d["c5"]["ms_per_frame_per_gpu"] * 1e3, 2))
PY
  done
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_guide*.py tests/test_gpu_configs.py -x -q 2>&1 | tail -2
