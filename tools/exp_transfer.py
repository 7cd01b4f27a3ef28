import time, numpy as np, torch
dev = torch.device("cuda")
H, W = 1080, 1920
img = np.random.rand(H, W, 3)
out_dev = torch.rand(H, W, 3, dtype=torch.float64, device=dev)
torch.cuda.synchronize()

def t(fn, n=10):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3

print("pageable H2D 50MB ms", t(lambda: torch.from_numpy(img).to(dev)))
pin = torch.empty((H, W, 3), dtype=torch.float64, pin_memory=True)
def staged():
    pin.numpy()[...] = img
    return pin.to(dev, non_blocking=True)
print("memcpy->pinned + H2D ms", t(staged))
print("memcpy only ms", t(lambda: np.copyto(pin.numpy(), img)))
print("pinned H2D ms", t(lambda: pin.to(dev, non_blocking=True)))
cr = torch.cuda.cudart()
def registered():
    ptr = img.ctypes.data
    cr.cudaHostRegister(ptr, img.nbytes, 0)
    x = torch.from_numpy(img).to(dev, non_blocking=True)
    torch.cuda.synchronize()
    cr.cudaHostUnregister(ptr)
    return x
print("register + H2D + unregister ms", t(registered))
print("pageable D2H 50MB ms", t(lambda: out_dev.cpu()))
pin_out = torch.empty((H, W, 3), dtype=torch.float64, pin_memory=True)
print("pinned D2H ms", t(lambda: pin_out.copy_(out_dev, non_blocking=True)))
print("pinned alloc (cached) + D2H ms", t(lambda: torch.empty((H, W, 3), dtype=torch.float64, pin_memory=True).copy_(out_dev, non_blocking=True)))
print("np.ascontiguousarray f64 ms", t(lambda: np.ascontiguousarray(img, dtype=np.float64)))
print("labels copy 2MB H2D ms", t(lambda: torch.from_numpy(np.zeros((H,W),np.uint8)).to(dev)))
