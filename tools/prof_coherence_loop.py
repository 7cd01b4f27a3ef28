"""C2 coherence preset: time of the persistent kernel alone (events around the
gf_coherence_fill launch) vs the whole run_coherence_fill call; with --ncu,
one call for an ncu capture of k_ct_loop."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
from paper_1611_05319_b200 import FillParams, scenes  # noqa: E402
from paper_1611_05319_b200 import _native as N  # noqa: E402
from paper_1611_05319_b200._device import params_to_c  # noqa: E402
from paper_1611_05319_b200.coherence import run_coherence_fill  # noqa: E402

sc = scenes.config(os.environ.get("GF_CONFIG", "C2"))
p = FillParams.coherence_transport()
H, W = sc.labels.shape
C = sc.image.shape[2]
d_img = torch.from_numpy(np.ascontiguousarray(sc.image, dtype=np.float64)).cuda()
d_lab = torch.from_numpy(sc.labels).cuda()
lib = N.load()
n_inp = int((d_lab == 255).sum())
ws_bytes = lib.gf_coherence_fill_workspace_bytes(H, W, C, n_inp)
ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
rows = torch.zeros((n_inp + 1, 5), dtype=torch.int64, device="cuda")
report = torch.zeros(4, dtype=torch.int32, device="cuda")
pc = params_to_c(p, True, N.GF_G_FIELD)


def kernel_once(u, lab, fs):
    N.check(lib.gf_coherence_fill(H, W, C, N.ptr(u), N.ptr(lab), ctypes.byref(pc), float(p.sigma),
                                  float(p.rho), float(p.coherence_lambda), n_inp, N.ptr(fs), None,
                                  N.ptr(rows), n_inp + 1, N.ptr(report), N.ptr(ws), ws_bytes,
                                  N.stream_ptr()))


if "--ncu" in sys.argv:
    u, lab = d_img.clone(), d_lab.clone()
    fs = torch.full((H * W,), -1, dtype=torch.int32, device="cuda")
    kernel_once(u, lab, fs)
    torch.cuda.synchronize()
    sys.exit(0)
kt, at = [], []
for it in range(8):
    u, lab = d_img.clone(), d_lab.clone()
    fs = torch.full((H * W,), -1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    kernel_once(u, lab, fs)
    e1.record()
    torch.cuda.synchronize()
    kt.append(e0.elapsed_time(e1))
    u = d_img.clone()
    torch.cuda.synchronize()
    e0.record()
    run_coherence_fill(u, d_lab, p, tracked=True)
    e1.record()
    torch.cuda.synchronize()
    at.append(e0.elapsed_time(e1))
print(json.dumps(dict(kernel_ms=min(kt[2:]), kernel_all=kt, api_ms=min(at[2:]), api_all=at,
                      report=report.cpu().tolist())))
