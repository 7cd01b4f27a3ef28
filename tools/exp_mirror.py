"""Experiment: e2e run_tracked (C2) with the mirrored result path vs the full download."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1611_05319_b200 import scenes, Spline, FillParams, tracker, _staging
sc = scenes.config("C2"); dev = torch.device("cuda")
spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"], kind=s["kind"]) for s in sc.splines]
p = FillParams(**sc.params)
img_p = torch.from_numpy(sc.image).pin_memory(); lab_p = torch.from_numpy(sc.labels).pin_memory()
key = str(dev if dev.index is not None else torch.device("cuda", 0))
def tm(name, fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); print(f"{name:40s} {(time.perf_counter()-t0)/n*1e3:8.3f} ms", flush=True)
for chunk in (1 << 20, 2 << 20, 4 << 20, 8 << 20):
    _staging._CHUNK = chunk
    _staging._mirror_ok.pop(key, None)
    print("mirror supported:", _staging.mirror_supported(torch.device("cuda", 0)), "stage chunk MB", chunk >> 20, "threads", _staging._executor()._max_workers)
    tm("pinned tensors, mirrored", lambda: tracker.run_tracked(img_p, lab_p, spl, p))
    tm("numpy, mirrored", lambda: tracker.run_tracked(sc.image, sc.labels, spl, p))
_staging._mirror_ok[key] = False
tm("pinned tensors, full download", lambda: tracker.run_tracked(img_p, lab_p, spl, p))
tm("numpy, full download", lambda: tracker.run_tracked(sc.image, sc.labels, spl, p))

# raw link: H2D alone, D2H alone, both at once (two streams), 50 MB each
n = sc.image.nbytes
hA = torch.empty(n, dtype=torch.uint8, pin_memory=True); hB = torch.empty(n, dtype=torch.uint8, pin_memory=True)
dA = torch.empty(n, dtype=torch.uint8, device=dev); dB = torch.empty(n, dtype=torch.uint8, device=dev)
s2 = torch.cuda.Stream()
def both():
    dA.copy_(hA, non_blocking=True)
    with torch.cuda.stream(s2): hB.copy_(dB, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
tm("raw H2D 50MB", lambda: dA.copy_(hA, non_blocking=True))
tm("raw D2H 50MB", lambda: hB.copy_(dB, non_blocking=True))
tm("raw H2D + D2H 50MB concurrently", both)

from paper_1611_05319_b200 import build_guide_field
_staging._mirror_ok.pop(key, None)
def two_call():
    f = build_guide_field(spl, sc.labels)
    return tracker.run_tracked(sc.image, sc.labels, f, p)
tm("two-call drop-in (numpy)", two_call)
tm("build_guide_field alone", lambda: build_guide_field(spl, sc.labels))
f0 = build_guide_field(spl, sc.labels)
tm("run_tracked(numpy img, returned field)", lambda: tracker.run_tracked(sc.image, sc.labels, f0, p))
f1 = f0.copy()
tm("run_tracked(numpy img, pageable field)", lambda: tracker.run_tracked(sc.image, sc.labels, f1, p))
