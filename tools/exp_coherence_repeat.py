import gc, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_1611_05319_b200 import FillParams, scenes
from paper_1611_05319_b200.coherence import run_coherence_fill
sc = scenes.config("C2"); p = FillParams.coherence_transport()
d_img = torch.from_numpy(np.ascontiguousarray(sc.image, dtype=np.float64)).cuda()
d_lab = torch.from_numpy(sc.labels).cuda()
for mode in ("gc on", "gc off"):
    if mode == "gc off": gc.disable()
    ts = []
    for _ in range(12):
        u0 = d_img.clone(); torch.cuda.synchronize(); t0 = time.perf_counter()
        run_coherence_fill(u0, d_lab, p, tracked=True); torch.cuda.synchronize()
        ts.append(round((time.perf_counter() - t0) * 1e3, 2))
    print(mode, ts, "reserved MB", torch.cuda.memory_reserved() >> 20)
