"""Stage times of the C2 end-to-end call (tracker.run_tracked on pinned host
tensors): labels upload, mirrored image upload, fill, delta, report read --
each followed by a synchronize, so the sum exceeds the pipelined call."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1611_05319_b200 import FillParams, Spline, scenes, tracker
from paper_1611_05319_b200 import _staging
from paper_1611_05319_b200._device import SegmentSet, fill_device

dev = torch.device("cuda:0")
sc = scenes.config("C2")
p = FillParams(**sc.params)
spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"],
              kind=s["kind"]) for s in sc.splines]
img_p = torch.from_numpy(sc.image).pin_memory()
lab_p = torch.from_numpy(sc.labels).pin_memory()
H, W = sc.labels.shape


def med(fn, n=15):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return round(sorted(ts)[n // 2], 4)


d = torch.empty(img_p.shape, dtype=torch.float64, device=dev)
back = torch.empty_like(img_p).pin_memory()
print("raw H2D 49.8MB ms", med(lambda: d.copy_(img_p, non_blocking=True)))
print("raw D2H 49.8MB ms", med(lambda: back.copy_(d, non_blocking=True)))
s2 = torch.cuda.Stream()
def duplex():
    d.copy_(img_p, non_blocking=True)
    with torch.cuda.stream(s2):
        back.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
d2 = torch.empty_like(d)
print("duplex H2D+D2H ms", med(duplex))
print("run_tracked pinned ms", med(lambda: tracker.run_tracked(img_p, lab_p, spl, p)))
segs = SegmentSet.cached(spl, dev)
print("labels upload ms", med(lambda: lab_p.to(dev, non_blocking=True)))
st = {}
def up():
    st["d"], st["m"] = _staging.upload_mirrored(img_p, dev, True)
print("upload_mirrored ms", med(up))
d_lab = lab_p.to(dev).reshape(1, H, W)
d_img = st["d"].reshape(1, H, W, 3)
def fill():
    st["res"] = fill_device(d_img, d_lab, None, p, tracked=True, rows_cap=H * W + 1, splines=segs,
                            want_fillshell=True)
print("fill_device (f64 image) ms", med(fill))
d_img32 = d_img.float()
print("fill_device (f32 image) ms", med(lambda: fill_device(d_img32, d_lab, None, p, tracked=True,
      rows_cap=H * W + 1, splines=segs, want_fillshell=True)))
def fin():
    st["m"].finish(d_img, st["res"]["out"])
print("mirror.finish ms", med(fin))
print("read_report ms", med(lambda: _staging.read_report(st["res"]["stats"][0], st["res"]["rows"][0])))
