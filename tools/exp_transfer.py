"""Experiment: host->device staging variants for the 50 MB float64 frame."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1611_05319_b200 import scenes, _staging
sc = scenes.config("C2"); dev = torch.device("cuda")
def tm(name, fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); print(f"{name:40s} {(time.perf_counter()-t0)/n*1e3:8.3f} ms", flush=True)
for chunk in (8 << 20, 4 << 20, 2 << 20, 1 << 20):
    _staging._CHUNK = chunk
    tm(f"upload f64 chunk {chunk >> 20} MB", lambda: _staging.upload(sc.image, dev, "img"))
_staging._CHUNK = 8 << 20
tm("labels .to(dev) pageable", lambda: torch.from_numpy(sc.labels).to(dev))
tm("labels staged", lambda: _staging.upload(sc.labels, dev, "lab"))
tm("image .to(dev) pageable", lambda: torch.from_numpy(sc.image).to(dev))

# page-lock the caller's own buffer in place, DMA from it, unlock
cudart = torch.cuda.cudart()
def reg_upload():
    a = sc.image
    ptr, nb = a.ctypes.data, a.nbytes
    err = cudart.cudaHostRegister(ptr, nb, 0)
    assert int(err) == 0, err
    src = torch.from_numpy(a)
    dst = torch.empty(a.shape, dtype=torch.float64, device=dev)
    dst.copy_(src, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    cudart.cudaHostUnregister(ptr)
    return dst
tm("upload via cudaHostRegister (in place)", reg_upload)
def reg_only():
    a = sc.image
    cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    cudart.cudaHostUnregister(a.ctypes.data)
tm("register+unregister only", reg_only)
