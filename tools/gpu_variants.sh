mkdir -p gpurun_out
for lib in libgf_b200.so; do
 for nf in 1 32; do
  GF_B200_LIB=$PWD/paper_1611_05319_b200/$lib timeout -s KILL 600 python bench.py --frames $nf --steps 20 --no-cpu --no-e2e > gpurun_out/v_${lib}_$nf.log 2>&1
  python - $lib $nf <<'PY'
import json,sys
d=json.loads(open(f"gpurun_out/v_{sys.argv[1]}_{sys.argv[2]}.log").read().strip().splitlines()[-1])
c=d["config"]
print(sys.argv[1], "frames", c["frames_per_gpu"], "ms/frame %.4f" % c["ms_per_frame"], "timeline", {k:(round(v["start_us"]),round(v["end_us"])) for k,v in c["timeline"].items()})
PY
 done
done
