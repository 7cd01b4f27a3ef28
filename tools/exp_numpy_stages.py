"""Stage times of the numpy-convention C2 call (pageable f64 in)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1611_05319_b200 import FillParams, Spline, scenes, tracker, _staging, engine

sc = scenes.config("C2")
p = FillParams(**sc.params)
spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"],
              kind=s["kind"]) for s in sc.splines]
img, lab = sc.image, sc.labels
dev = torch.device("cuda:0")


def med(fn, n=11):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return round(sorted(ts)[n // 2], 3)


keep = []
def up():
    keep.append(_staging.upload_mirrored(img, dev, False))
    if len(keep) > 2:
        keep.pop(0)
print("upload_mirrored numpy + sync ms", med(up))
def up_nosync():
    t0 = time.perf_counter()
    keep.append(_staging.upload_mirrored(img, dev, False))
    keep.pop(0)
    up_nosync.t.append((time.perf_counter() - t0) * 1e3)
up_nosync.t = []
med(up_nosync)
print("upload_mirrored host return ms", round(sorted(up_nosync.t)[len(up_nosync.t) // 2], 3))
print("labels numpy .to(dev) ms", med(lambda: torch.from_numpy(lab).to(dev)))
print("pool take ms", med(lambda: _staging._pool_out.take(img.shape, np.float64)))
print("run_tracked numpy ms", med(lambda: tracker.run_tracked(img, lab, spl, p)))
imgp = torch.from_numpy(img).pin_memory(); labp = torch.from_numpy(lab).pin_memory()
print("run_tracked pinned ms", med(lambda: tracker.run_tracked(imgp, labp, spl, p)))
print("run_tracked numpy img + pinned labels ms", med(lambda: tracker.run_tracked(img, labp, spl, p)))
