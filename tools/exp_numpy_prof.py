"""cProfile of the numpy-convention C2 call (where the host time goes)."""
import sys, cProfile, pstats
sys.path.insert(0, ".")
import torch
from paper_1611_05319_b200 import FillParams, Spline, scenes, tracker

sc = scenes.config("C2")
p = FillParams(**sc.params)
spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"],
              kind=s["kind"]) for s in sc.splines]
for _ in range(3):
    tracker.run_tracked(sc.image, sc.labels, spl, p)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    tracker.run_tracked(sc.image, sc.labels, spl, p)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
