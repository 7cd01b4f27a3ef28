"""torch.profiler breakdown of one C2 coherence-transport fill (device-resident)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
from paper_1611_05319_b200 import FillParams, scenes  # noqa: E402
from paper_1611_05319_b200.coherence import run_coherence_fill  # noqa: E402

sc = scenes.config("C2")
p = FillParams.coherence_transport()
d_img = torch.from_numpy(np.ascontiguousarray(sc.image, dtype=np.float64)).cuda()
d_lab = torch.from_numpy(sc.labels).cuda()
for _ in range(2):
    run_coherence_fill(d_img.clone(), d_lab, p, tracked=True)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    run_coherence_fill(d_img.clone(), d_lab, p, tracked=True)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
