"""Per-block timeline of the prep pass (experiment build -DGF_PREP_PROF).

GF_B200_LIB=paper_1611_05319_b200/libgf_b200_prof.so python tools/prof_prep_blocks.py
Runs the bench's C2 fill (spline raster fused into the prep) and prints the
distribution of block durations (tiles with / without Inpaint pixels near),
the kernel span and the per-SM busy time.
"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1611_05319_b200 import scenes, Spline, FillParams, _native
from paper_1611_05319_b200._device import fill_device, SegmentSet

sc = scenes.config(sys.argv[1] if len(sys.argv) > 1 else "C2")
dev = torch.device("cuda")
spl = [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"], kind=s["kind"]) for s in sc.splines]
img = torch.from_numpy(sc.image.astype(np.float32))[None].to(dev).contiguous()
lab = torch.from_numpy(sc.labels)[None].to(dev).contiguous()
segs = SegmentSet(spl, dev)
p = FillParams(**sc.params)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
H, W = sc.labels.shape
nt = ((H + 31) // 32) * ((W + 31) // 32)
lib = ctypes.CDLL(_native.LIB_PATH)
out = {}
for rep in range(6):
    sp = np.array([np.iinfo(np.int64).max] * 2 + [0], np.uint64)
    torch.cuda.synchronize()
    assert lib.gf_prep_prof_read(sp.ctypes.data_as(ctypes.c_void_p), -2) == 0
    flush.zero_()
    torch.cuda.synchronize()
    fill_device(img, lab, None, p, splines=segs, rows_cap=4096)
    torch.cuda.synchronize()
shp = np.zeros(3, np.uint64)
assert lib.gf_prep_prof_read(shp.ctypes.data_as(ctypes.c_void_p), -1) == 0
buf = np.zeros((nt, 12), np.uint64)
assert lib.gf_prep_prof_read(buf.ctypes.data_as(ctypes.c_void_p), nt) == 0
B = buf.astype(np.int64)
t0, t1 = B[:, 0], B[:, 10]
sm = B[:, 11] & 0xffffffff
fl = B[:, 11] >> 32
base = t0.min()
dur = (t1 - t0) / 1e3
d = (fl & 1) == 1
out["span_us"] = float((t1.max() - base) / 1e3)
out["shells_first_entry_us"] = float((int(shp[0]) - base) / 1e3) if shp[0] != 0 else None
out["shells_pdl_return_first_last_us"] = [float((int(shp[1]) - base) / 1e3), float((int(shp[2]) - base) / 1e3)]
out["first_start_last_start_us"] = [0.0, float((t0.max() - base) / 1e3)]
for name, m in (("copy_tiles", ~d), ("d_tiles", d)):
    if m.any():
        out[name] = dict(n=int(m.sum()), dur_us_mean=float(dur[m].mean()), p50=float(np.median(dur[m])),
                         p90=float(np.percentile(dur[m], 90)), max=float(dur[m].max()))
for name, m in (("copy_tiles", ~d), ("d_tiles", d)):
    st = {}
    prev = B[m, 0]
    for k in (1, 2, 3, 4, 5, 6, 7, 8, 10):
        if (B[m, k] == 0).all():
            continue
        st[f"->{k}"] = float(np.mean(B[m, k] - prev) / 1e3)
        prev = B[m, k]
    out[name]["stage_us"] = st
out["ncand_max"] = int((fl >> 1).max())
busy = np.zeros(148)
last = np.zeros(148)
for s_, a, b in zip(sm, t0, t1):
    busy[s_] += (b - a) / 1e3
    last[s_] = max(last[s_], (b - base) / 1e3)
out["sm_block_us_sum"] = dict(min=float(busy.min()), mean=float(busy.mean()), max=float(busy.max()))
out["sm_last_end_us"] = dict(min=float(last.min()), mean=float(last.mean()), max=float(last.max()))
# start-time histogram (µs buckets)
st = (t0 - base) / 1e3
out["start_hist_2us"] = np.bincount((st // 2).astype(int)).tolist()
en = (t1 - base) / 1e3
out["end_hist_2us"] = np.bincount((en // 2).astype(int)).tolist()
# longest blocks
idx = np.argsort(-dur)[:8]
out["longest"] = [[int(i), float(dur[i]), int(fl[i] & 1), int(fl[i] >> 1), float(st[i])] for i in idx]
def stages(i):
    ks = [k for k in (0, 1, 2, 3, 4, 5, 6, 7, 8, 10) if B[i, k] != 0]
    return {f"{a}->{b}": float((B[i, b] - B[i, a]) / 1e3) for a, b in zip(ks, ks[1:])}
out["longest_stages"] = [stages(int(i)) for i in idx]
print(json.dumps(out, indent=1))
