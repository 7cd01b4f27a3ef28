import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1611_05319_b200 import scenes, Spline, FillParams, tracker, _staging
from paper_1611_05319_b200._device import SegmentSet, fill_device
sc = scenes.config("C2"); dev = torch.device("cuda")
spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"], kind=s["kind"]) for s in sc.splines]
p = FillParams(**sc.params)
H, W = sc.labels.shape
for _ in range(3): tracker.run_tracked(sc.image, sc.labels, spl, p)
torch.cuda.synchronize()
def tm(name, fn, n=10):
    fn(); torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(n): r=fn()
    torch.cuda.synchronize(); print(f"{name:30s} {(time.perf_counter()-t0)/n*1e3:8.3f} ms"); return r
d_img = tm("upload img f64 50MB", lambda: _staging.upload(sc.image, dev, "img"))
d_lab = tm("upload labels", lambda: _staging.upload(sc.labels, dev, "lab"))
segs = tm("SegmentSet", lambda: SegmentSet(spl, dev))
res = tm("fill_device", lambda: fill_device(d_img.reshape(1,H,W,3), d_lab.reshape(1,H,W), None, p, rows_cap=H*W+1, splines=segs, want_fillshell=True))
tm("stats+rows cpu", lambda: (res["stats"][0].cpu().numpy(), res["rows"][0,:11].cpu().numpy()))
tm("download out 50MB", lambda: _staging.download(res["out"][0]))
tm("run_tracked total", lambda: tracker.run_tracked(sc.image, sc.labels, spl, p))
tm("np.empty 50MB + touch", lambda: np.empty((H,W,3)).fill(0))
