mkdir -p gpurun_out
for cfg in C1 C2 C3 C4; do
  timeout -s KILL 600 python bench.py --config $cfg --steps 50 --no-cpu --no-e2e > gpurun_out/bench_$cfg.log 2>&1; echo "$cfg rc=$?"
  python - $cfg <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/bench_{sys.argv[1]}.log").read().strip().splitlines()[-1])
c=d["config"]; r=d["roofline"]
print(sys.argv[1], "ms/frame %.4f" % d["ms_per_step"], "Mpx/s %.0f" % d["value"], "frac %.3f" % r["frac"], "shells", c["shells"], "timeline", {k:(round(v["start_us"]),round(v["end_us"])) for k,v in c["timeline"].items()})
PY
done
timeout -s KILL 600 python bench.py --untracked --steps 50 --no-cpu --no-e2e > gpurun_out/bench_untracked.log 2>&1; echo "untracked rc=$?"
tail -c 300 gpurun_out/bench_untracked.log | head -c 300; echo
python -c "import json; d=json.loads(open('gpurun_out/bench_untracked.log').read().strip().splitlines()[-1]); print('C2 untracked ms/frame %.4f' % d['ms_per_step'])"
