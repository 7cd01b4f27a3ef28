# numpy-convention C2 call: copy piece size x DMA chunk size (pageable upload through the result buffer)
for piece in 524288 1048576 2097152 4194304; do
  GF_COPY_PIECE=$piece timeout 200 python - <<'PY'
import os, sys, time
sys.path.insert(0, ".")
import torch
from paper_1611_05319_b200 import FillParams, Spline, scenes, tracker, _staging
sc = scenes.config("C2"); p = FillParams(**sc.params)
spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"], kind=s["kind"]) for s in sc.splines]
for ch in (8 << 20, 16 << 20, 4 << 20):
    _staging._CHUNK = ch
    ts = []
    for k in range(14):
        t0 = time.perf_counter(); tracker.run_tracked(sc.image, sc.labels, spl, p); torch.cuda.synchronize()
        if k >= 3: ts.append((time.perf_counter() - t0) * 1e3)
    print("piece", os.environ["GF_COPY_PIECE"], "chunk", ch >> 20, "ms", round(sorted(ts)[len(ts) // 2], 3), flush=True)
PY
done
