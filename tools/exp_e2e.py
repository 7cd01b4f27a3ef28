"""Experiment: where the end-to-end run_tracked time goes (C2, float64 numpy in/out)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1611_05319_b200 import scenes, Spline, FillParams, tracker, _staging, grid
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
    torch.cuda.synchronize(); print(f"{name:34s} {(time.perf_counter()-t0)/n*1e3:8.3f} ms", flush=True); return r
tm("run_tracked total", lambda: tracker.run_tracked(sc.image, sc.labels, spl, p))
d_img = tm("upload img f64 50MB (staged)", lambda: _staging.upload(sc.image, dev, "img"))
d_lab = tm("upload labels 2MB", lambda: _staging.upload(sc.labels, dev, "lab"))
tm("validate labels (GPU + sync)", lambda: grid.validate_labels(sc.labels, d_lab))
segs = tm("SegmentSet (flatten + H2D)", lambda: SegmentSet(spl, dev))
res = tm("fill_device (eager)", lambda: fill_device(d_img.reshape(1,H,W,3), d_lab.reshape(1,H,W), None, p, rows_cap=H*W+1, splines=segs, want_fillshell=True))
tm("stats+rows .cpu()", lambda: (res["stats"][0].cpu().numpy(), res["rows"][0,:11].cpu().numpy()))
tm("download out 50MB (pinned pool)", lambda: _staging.download(res["out"][0]))
tm("np.copy 50MB (1 thread)", lambda: sc.image.copy())
tm("np.ascontiguousarray f64", lambda: np.ascontiguousarray(sc.image, dtype=np.float64))
x = torch.empty(H * W * 3, dtype=torch.float64, pin_memory=True)
tm("H2D 50MB pinned (raw DMA)", lambda: d_img.view(-1).copy_(x, non_blocking=True))
tm("D2H 50MB pinned (raw DMA)", lambda: x.copy_(d_img.view(-1), non_blocking=True))
print("cpus", os.cpu_count())

# step-by-step copy of engine._run_fill with timers
from paper_1611_05319_b200 import engine
from paper_1611_05319_b200 import _native as N
def run_timed():
    ts = [time.perf_counter()]
    def mark(): torch.cuda.synchronize(); ts.append(time.perf_counter())
    labels = sc.labels
    img = np.ascontiguousarray(sc.image, dtype=np.float64); mark()
    d_img = _staging.upload(img, dev, "img").reshape(1, H, W, 3); mark()
    d_lab = _staging.upload(np.ascontiguousarray(labels, dtype=np.uint8), dev, "lab").reshape(1, H, W); mark()
    grid.validate_labels(labels, d_lab); mark()
    segs = SegmentSet(list(spl), dev); mark()
    res = fill_device(d_img, d_lab, None, p, tracked=True, rows_cap=H * W + 1, splines=segs, want_fillshell=True); mark()
    stats = res["stats"][0].cpu().numpy(); iters = int(stats[N.STAT_ITERATIONS]); rows_dev = res["rows"][0, :iters + 1].cpu().numpy(); mark()
    u = _staging.download(res["out"][0]); mark()
    return np.diff(ts) * 1e3
for _ in range(3): run_timed()
acc = np.mean([run_timed() for _ in range(10)], axis=0)
print("steps ms: contig %.3f up_img %.3f up_lab %.3f validate %.3f segs %.3f fill %.3f stats %.3f down %.3f" % tuple(acc))
