"""Experiment: where build_guide_field's host time goes (C2)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1611_05319_b200 import scenes, Spline, build_guide_field, _staging
from paper_1611_05319_b200._device import SegmentSet, guide_field_device
sc = scenes.config("C2"); dev = torch.device("cuda")
spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"], kind=s["kind"]) for s in sc.splines]
def tm(name, fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): r = fn()
    torch.cuda.synchronize(); print(f"{name:40s} {(time.perf_counter()-t0)/n*1e3:8.3f} ms", flush=True)
    return r
tm("build_guide_field", lambda: build_guide_field(spl, sc.labels))
tm("labels == INPAINT any", lambda: (sc.labels == 255).any())
tm("SegmentSet", lambda: SegmentSet(spl, dev))
tm("SegmentSet.cached", lambda: SegmentSet.cached(spl, dev))
d_lab = tm("labels upload (stager)", lambda: _staging.upload(np.ascontiguousarray(sc.labels, dtype=np.uint8), dev, "lab"))
tm("labels upload (.to)", lambda: torch.from_numpy(sc.labels).to(dev))
segs = SegmentSet(spl, dev)
f = tm("raster kernel", lambda: guide_field_device(d_lab, segs, 3.0))
tm("download field 33MB", lambda: _staging.download(f))
