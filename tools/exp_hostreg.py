"""Experiment: page-locking the caller's numpy buffer (cudaHostRegister) vs the pinned stager."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1611_05319_b200 import _staging
cr = torch.cuda.cudart()
dev = torch.device("cuda")
a = np.random.default_rng(0).random((1080, 1920, 3))
d = torch.empty(a.size, dtype=torch.float64, device=dev)
def tm(name, fn, n=10):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); print(f"{name:44s} {(time.perf_counter()-t0)/n*1e3:8.3f} ms", flush=True)
tm("stager upload 50MB", lambda: _staging.upload(a, dev, "img"))
def reg():
    p = a.ctypes.data
    r = cr.cudaHostRegister(p, a.nbytes, 0)
    d.copy_(torch.from_numpy(a.reshape(-1)), non_blocking=True)
    torch.cuda.synchronize()
    cr.cudaHostUnregister(p)
tm("register + DMA + unregister 50MB", reg)
def reg_only():
    p = a.ctypes.data
    cr.cudaHostRegister(p, a.nbytes, 0); cr.cudaHostUnregister(p)
tm("register + unregister only", reg_only)
tm("pageable .copy_ 50MB", lambda: d.copy_(torch.from_numpy(a.reshape(-1))))
