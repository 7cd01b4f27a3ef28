# A/B of the prep/shell shared-memory carveout (GF_CARVEOUT, percent) on the C2 bench step.
mkdir -p gpurun_out
CMD="python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu --no-c5 --no-extras"
for rep in 1 2; do
  for c in none 58 100 75; do
    if [ "$c" = none ]; then env -u GF_CARVEOUT timeout 200 $CMD > gpurun_out/co_$c.log 2>&1
    else GF_CARVEOUT=$c timeout 200 $CMD > gpurun_out/co_$c.log 2>&1; fi
    python - "$c" <<'PY'
import json, sys
l = [x for x in open(f"gpurun_out/co_{sys.argv[1]}.log") if x.startswith("{")][-1]
d = json.loads(l); c = d["config"]
print(sys.argv[1], round(d["ms_per_step"], 5), c["timeline"])
PY
  done
done
