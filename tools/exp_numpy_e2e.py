"""The reference's calling convention (pageable numpy f64 in, numpy out) on
C2: host copy throughput into pinned memory by thread count, and the e2e
call by staging chunk size (_staging._CHUNK)."""
import sys, time
sys.path.insert(0, ".")
from concurrent.futures import ThreadPoolExecutor
import numpy as np
import torch
from paper_1611_05319_b200 import FillParams, Spline, scenes, tracker, _staging

sc = scenes.config("C2")
p = FillParams(**sc.params)
spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"],
              kind=s["kind"]) for s in sc.splines]
img, lab = sc.image, sc.labels


def med(fn, n=11):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return round(sorted(ts)[n // 2], 3)


src = img.reshape(-1).view(np.uint8)
dst = torch.empty(src.nbytes, dtype=torch.uint8, pin_memory=True).numpy()
import os
print("cpus", os.cpu_count())
for nt in (1, 2, 4, 8, 16):
    ex = ThreadPoolExecutor(nt)
    n = src.nbytes
    parts = [(o, min(n, o + (n + nt - 1) // nt)) for o in range(0, n, (n + nt - 1) // nt)]
    def cp():
        list(ex.map(lambda lh: np.copyto(dst[lh[0]:lh[1]], src[lh[0]:lh[1]]), parts))
    print("threads", nt, "copy 49.8MB ms", med(cp))
for ch in (8 << 20, 4 << 20, 16 << 20):
    _staging._CHUNK = ch
    print("chunk MB", ch >> 20, "run_tracked numpy ms", med(lambda: tracker.run_tracked(img, lab, spl, p)))
