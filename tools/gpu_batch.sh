mkdir -p gpurun_out
for lib in ${LIBS:-libgf_b200.so}; do
for nf in ${FRAMES:-8 32 64}; do
  GF_B200_LIB=$PWD/paper_1611_05319_b200/$lib timeout -s KILL 600 python bench.py --frames $nf --steps 20 --no-cpu --no-e2e > gpurun_out/bench_f$nf.log 2>&1; echo "frames $nf rc=$?"
  python - $nf $lib <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/bench_f{sys.argv[1]}.log").read().strip().splitlines()[-1])
c=d["config"]; r=d["roofline"]
print(sys.argv[2], "frames", c["frames_per_gpu"], "ms/step %.3f" % d["ms_per_step"], "ms/frame %.4f" % c["ms_per_frame"], "Mpx/s %.0f" % d["value"], "HBM %.0f GB/s frac %.3f" % (r["achieved"], r["frac"]), "timeline", {k:(round(v["start_us"]),round(v["end_us"])) for k,v in c["timeline"].items()})
PY
done
done
