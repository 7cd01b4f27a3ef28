import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]
import numpy as np, torch
from paper_1611_05319_b200 import FillParams, scenes
from paper_1611_05319_b200._device import fill_device
dt = torch.float64 if sys.argv[1] == "f64" else torch.float32
sc = scenes.small_scene(96, 160, band=6, gx=4, gy=3, n_spl=3, seed=7)
img = torch.from_numpy(sc.image[None]).to(dt).cuda()
lab = torch.from_numpy(sc.labels[None]).cuda()
r = fill_device(img, lab, None, FillParams(**sc.params))
torch.cuda.synchronize()
print(sys.argv[1], os.environ.get("GF_NO_TMA"), r["stats"][0].tolist())
