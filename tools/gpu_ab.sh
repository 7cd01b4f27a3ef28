mkdir -p gpurun_out
for lib in ${LIBS:-libgf_b200.so}; do
  GF_B200_LIB=$PWD/paper_1611_05319_b200/$lib timeout -s KILL 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench_$lib.log 2>&1; echo "$lib rc=$?"
  python - "$lib" <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/bench_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print(sys.argv[1], "ms/frame %.4f" % d["ms_per_step"], "min %.4f" % d["config"]["ms_step_min"], "Mpx/s %.1f" % d["value"])
print("  timeline", {k: (round(v["start_us"],1), round(v["end_us"],1)) for k, v in d["config"]["timeline"].items()})
for r in d["config"]["shell_trace"]: print("  items %6d fill %6.2f lat %6.2f rot %6.2f sync %5.2f" % (r["items"], r["fill_us"], r["lattice_item_max_us"], r["rotated_item_max_us"], r["sync_us"]))
PY
done
