"""Same-box A/B of the pageable upload: staging buffer + D2H mirror (round-2
code) vs copying into the result buffer (no mirror), interleaved."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1611_05319_b200 import FillParams, Spline, scenes, tracker, _staging as S

new = S.upload_mirrored


def old(src, device, as_tensor):
    a = np.ascontiguousarray(src)
    n = a.nbytes
    dst = torch.empty(a.shape, dtype=torch.from_numpy(a[:0].reshape(-1)).dtype, device=device)
    mir = S.Mirror(device, a.shape, dst.dtype, False)
    stage = S._staging(n, "img")
    srcb = a.reshape(-1).view(np.uint8)
    host = stage.numpy()
    parts = S._chunks_of(n, S._CHUNK)
    futs = [S._executor().submit(np.copyto, host[lo:hi], srcb[lo:hi]) for lo, hi in parts]
    for (lo, hi), fut in zip(parts, futs):
        fut.result()
        mir.upload(stage.data_ptr(), dst.data_ptr(), lo, hi)
    torch.cuda.current_stream().synchronize()
    return dst, mir


sc = scenes.config("C2"); p = FillParams(**sc.params)
spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"], kind=s["kind"]) for s in sc.splines]
ref = tracker.run_tracked(sc.image, sc.labels, spl, p)[0].copy()
res = {}
for rnd in range(4):
    for name, fn, piece in (("old", old, 8 << 20), ("new8", new, 8 << 20), ("new4", new, 4 << 20)):
        S.upload_mirrored = fn
        pass
        ts = []
        for k in range(12):
            t0 = time.perf_counter()
            u, _ = tracker.run_tracked(sc.image, sc.labels, spl, p)
            torch.cuda.synchronize()
            if k >= 2:
                ts.append((time.perf_counter() - t0) * 1e3)
        assert np.array_equal(u, ref), name
        res.setdefault(name, []).append(round(sorted(ts)[len(ts) // 2], 3))
for k, v in res.items():
    print(k, v, "median", sorted(v)[len(v) // 2])
