import sys, os, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1611_05319_b200 import scenes, Spline, FillParams, tracker
sc = scenes.config("C2")
spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"], kind=s["kind"]) for s in sc.splines]
p = FillParams(**sc.params)
for _ in range(3): tracker.run_tracked(sc.image, sc.labels, spl, p)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(20): u, m = tracker.run_tracked(sc.image, sc.labels, spl, p)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
