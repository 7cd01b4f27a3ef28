"""Experiment: video.fill_video_host per-frame timing, repeated (flakiness hunt)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1611_05319_b200 import scenes, Spline, FillParams, video, tracker
vframes = [scenes.config("C5", frame=i) for i in range(8)]
p = FillParams(**vframes[0].params)
v_img = [torch.from_numpy(f.image).pin_memory() for f in vframes]
v_lab = [torch.from_numpy(f.labels).pin_memory() for f in vframes]
v_spl = [[Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"], kind=s["kind"]) for s in f.splines] for f in vframes]
stamps = []
def consume(f, u, rep):
    stamps.append(time.perf_counter())
for rep_i in range(6):
    stamps.clear()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    video.fill_video_host(v_img + v_img, v_lab + v_lab, v_spl + v_spl, p, on_frame=consume)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    gaps = np.diff([t0] + stamps) * 1e3
    print(f"run {rep_i}: {(t1 - t0) / 16 * 1e3:.3f} ms/frame; per-frame gaps ms", np.round(gaps, 2).tolist(), flush=True)
# single calls for comparison, then the pipeline again
for _ in range(5):
    tracker.run_tracked(v_img[0], v_lab[0], v_spl[0], p)
torch.cuda.synchronize(); t0 = time.perf_counter()
video.fill_video_host(v_img + v_img, v_lab + v_lab, v_spl + v_spl, p, on_frame=consume)
torch.cuda.synchronize(); print("after run_tracked calls: %.3f ms/frame" % ((time.perf_counter() - t0) / 16 * 1e3))
