"""A batched C5 fill (device-rendered frames) run twice: the ncu target for
the batched kernels.  python tools/prof_batch.py [frames]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]

import torch  # noqa: E402

from paper_1611_05319_b200 import FillParams, Spline, scenes  # noqa: E402
from paper_1611_05319_b200._device import SegmentSet, fill_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
dev = torch.device("cuda")
images, labels, spl = scenes.video_batch_device(range(n), dev)
segs = SegmentSet([[Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"],
                           kind=s["kind"]) for s in fs] for fs in spl], dev, per_frame=True)
p = FillParams(**scenes.config("C5").params)
ws = None
for _ in range(2):
    r = fill_device(images, labels, None, p, splines=segs, workspace=ws, rows_cap=256)
    ws = r["workspace"]
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
r = fill_device(images, labels, None, p, splines=segs, workspace=ws, rows_cap=256)
e1.record()
torch.cuda.synchronize()
print(n, "frames", e0.elapsed_time(e1) * 1e3 / n, "us/frame")
