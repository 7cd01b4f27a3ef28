"""Full-size BASELINE.json configurations on the GPU vs the CPU oracle.

C1-C4 at their real sizes: fill order / frontier sets bit-exact, report rows
identical, values within 1e-4, guide field bit-exact; tracked == untracked;
a batched multi-frame launch is bit-identical to per-frame launches (the
property the frame-parallel video path relies on).
"""

import numpy as np
import pytest
import torch

from oracle import guidefill_oracle as orc
from paper_1611_05319_b200 import FillParams, Spline, build_guide_field, engine, scenes
from paper_1611_05319_b200 import _native as N
from paper_1611_05319_b200._device import fill_device

pytestmark = pytest.mark.gpu


def _splines(sc):
    return [Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"],
                   kind=s["kind"]) for s in sc.splines]


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_config_parity(name):
    sc = scenes.config(name)
    field = build_guide_field(_splines(sc), sc.labels)
    ref_field = orc.guide_field([orc.polyline(s["points"], s["kind"]) for s in sc.splines],
                                [s["direction"] for s in sc.splines], sc.labels)
    assert np.array_equal(field, ref_field)
    p = FillParams(**sc.params)
    ref = orc.fill(sc.image, sc.labels, ref_field, orc.Params.of(p), tracked=True)
    for tracked in (True, False):
        u, rep, maps = engine._run_fill(sc.image, sc.labels, field, p, tracked=tracked,
                                        order_log=True)
        assert np.array_equal(maps["fillshell"], ref["fillshell"])
        assert np.array_equal(maps["enter"], ref["enter"])
        assert rep.iterations == ref["iterations"] and rep.filled == ref["filled"]
        if tracked:
            assert [tuple(r) for r in rep.rows] == [tuple(r) for r in ref["rows"]]
        assert float(np.abs(u - ref["u"]).max()) <= 1e-4


def test_batched_frames_equal_single_frames():
    frames = [scenes.small_scene(270, 480, band=8, gx=5, gy=3, n_spl=4, seed=1611, frame=f)
              for f in range(6)]
    dev = torch.device("cuda")
    H, W = frames[0].labels.shape
    fields = [build_guide_field(_splines(sc), sc.labels) for sc in frames]
    p = FillParams(**frames[0].params)
    img = torch.from_numpy(np.stack([sc.image for sc in frames]).astype(np.float32)).to(dev)
    lab = torch.from_numpy(np.stack([sc.labels for sc in frames])).to(dev)
    gd = torch.from_numpy(np.stack(fields)).to(dev)
    for tracked in (True, False):
        batch = fill_device(img, lab, gd, p, tracked=tracked, order_log=True)
        for f in range(len(frames)):
            one = fill_device(img[f:f + 1].contiguous(), lab[f:f + 1].contiguous(),
                              gd[f:f + 1].contiguous(), p, tracked=tracked, order_log=True)
            assert torch.equal(batch["out"][f], one["out"][0])
            assert torch.equal(batch["fillshell"][f], one["fillshell"][0])
            assert torch.equal(batch["enter"][f], one["enter"][0])
            assert torch.equal(batch["stats"][f], one["stats"][0])
            it = int(one["stats"][0, N.STAT_ITERATIONS])
            assert torch.equal(batch["rows"][f, :it], one["rows"][0, :it])


def test_float32_device_path_matches_float64_order():
    sc = scenes.small_scene(200, 320, band=8, gx=4, gy=3, n_spl=3, seed=9)
    field = build_guide_field(_splines(sc), sc.labels)
    p = FillParams(**sc.params)
    dev = torch.device("cuda")
    r32 = fill_device(torch.from_numpy(sc.image.astype(np.float32))[None].to(dev),
                      torch.from_numpy(sc.labels)[None].to(dev),
                      torch.from_numpy(field)[None].to(dev), p, order_log=True)
    r64 = fill_device(torch.from_numpy(sc.image)[None].to(dev),
                      torch.from_numpy(sc.labels)[None].to(dev),
                      torch.from_numpy(field)[None].to(dev), p, order_log=True)
    assert torch.equal(r32["fillshell"], r64["fillshell"])
    assert (r32["out"].double() - r64["out"]).abs().max().item() <= 1e-6


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_fused_raster_fill_equals_two_pass(name):
    """gf_fill_splines (raster fused into the fill) == gf_guide_field + gf_fill."""
    from paper_1611_05319_b200._device import SegmentSet

    sc = scenes.config(name)
    dev = torch.device("cuda")
    p = FillParams(**sc.params)
    img = torch.from_numpy(sc.image.astype(np.float32))[None].to(dev)
    lab = torch.from_numpy(sc.labels)[None].to(dev)
    field = torch.from_numpy(build_guide_field(_splines(sc), sc.labels))[None].to(dev)
    two = fill_device(img, lab, field, p, order_log=True)
    one = fill_device(img, lab, None, p, order_log=True, splines=SegmentSet(_splines(sc), dev))
    assert torch.equal(one["fillshell"], two["fillshell"])
    assert torch.equal(one["enter"], two["enter"])
    assert torch.equal(one["out"], two["out"])
    assert torch.equal(one["stats"], two["stats"])


def _clip_scene(seed, H=150, W=230):
    """Readable values in [0.3, 0.6]; Bystanders hold 0.0 / 1.0 / in-hull
    values spread over many 32x32 tiles, so the shell loop's tile clip runs."""
    rng = np.random.default_rng(seed)
    img = 0.3 + 0.3 * rng.random((H, W, 3))
    lab = np.zeros((H, W), np.uint8)
    lab[40:48, 20:200] = 255
    lab[90:130, 100:108] = 255
    bys = rng.random((H, W)) < 0.08
    bys &= lab == 0
    lab[bys] = 128
    vals = rng.choice([0.0, 1.0, 0.45], size=(int(bys.sum()), 3))
    img[bys] = vals
    img[lab == 255] = 0.0
    return img, lab


@pytest.mark.parametrize("seed", [1, 2])
def test_bystander_clip_outside_hull(seed):
    img, lab = _clip_scene(seed)
    p = FillParams(r=3, mu=50.0, order="smart", neighborhood="rotated_ball")
    ref = orc.fill(img, lab, None, orc.Params.of(p), tracked=True)
    assert float(np.abs(ref["u"][lab == 128] - img[lab == 128]).max()) > 0.1  # clip does work
    for tracked in (True, False):
        u, rep, maps = engine._run_fill(img, lab, None, p, tracked=tracked, order_log=True)
        assert np.array_equal(maps["fillshell"], ref["fillshell"])
        assert np.array_equal(u[lab == 128], ref["u"][lab == 128])  # clip is exact
        assert np.array_equal(u[lab == 0], img[lab == 0])
        assert float(np.abs(u - ref["u"]).max()) <= 1e-4


def test_bystander_clip_batched_frames_own_hulls():
    scenes_ = [_clip_scene(s) for s in (3, 4, 5)]
    p = FillParams(r=3, mu=50.0, order="smart", neighborhood="rotated_ball")
    dev = torch.device("cuda")
    # frame 1 gets a wider hull: its Bystanders need no clip, the others do
    scenes_[1][0][0, 0] = (0.0, 1.0, 0.5)
    img = torch.from_numpy(np.stack([s[0] for s in scenes_])).to(dev)
    lab = torch.from_numpy(np.stack([s[1] for s in scenes_])).to(dev)
    res = fill_device(img, lab, None, p, order_log=True)
    for f, (im, lb) in enumerate(scenes_):
        ref = orc.fill(im, lb, None, orc.Params.of(p), tracked=True)
        out = res["out"][f].cpu().numpy()
        assert np.array_equal(res["fillshell"][f].cpu().numpy(), ref["fillshell"])
        assert np.array_equal(out[lb == 128], ref["u"][lb == 128])


def test_fill_graph_replay_matches_eager():
    from paper_1611_05319_b200._device import FillGraph, SegmentSet

    sc = scenes.config("C1")
    dev = torch.device("cuda")
    p = FillParams(**sc.params)
    img = torch.from_numpy(sc.image.astype(np.float32))[None].to(dev).contiguous()
    lab = torch.from_numpy(sc.labels)[None].to(dev).contiguous()
    segs = SegmentSet(_splines(sc), dev)
    g = FillGraph(img, lab, None, p, splines=segs, want_fillshell=True)
    for scale in (1.0, 0.5):  # a new frame written into the captured input
        img.copy_(torch.from_numpy((sc.image * scale).astype(np.float32))[None].to(dev))
        out = g.replay()
        eager = fill_device(img, lab, None, p, splines=segs, want_fillshell=True, rows_cap=4096)
        torch.cuda.synchronize()
        assert torch.equal(out["out"], eager["out"])
        assert torch.equal(out["fillshell"], eager["fillshell"])
        assert torch.equal(out["stats"], eager["stats"])


@pytest.mark.parametrize("r,order,nb", [(7, "smart", "rotated_ball"), (8, "onion", "axis_ball"),
                                        (9, "smart_with_data_term", "rotated_ball")])
def test_large_ball_generic_evaluator(r, order, nb):
    """r >= 7 (K > 128: several pairwise leaves) runs the runtime-K evaluator."""
    sc = scenes.small_scene(120, 200, band=10, gx=3, gy=2, n_spl=3, seed=31 + r)
    field = build_guide_field(_splines(sc), sc.labels)
    p = FillParams(r=r, mu=50.0, order=order, neighborhood=nb)
    ref = orc.fill(sc.image, sc.labels, field, orc.Params.of(p), tracked=True)
    for tracked in (True, False):
        u, rep, maps = engine._run_fill(sc.image, sc.labels, field, p, tracked=tracked,
                                        order_log=True)
        assert np.array_equal(maps["fillshell"], ref["fillshell"])
        assert np.array_equal(maps["enter"], ref["enter"])
        assert float(np.abs(u - ref["u"]).max()) <= 1e-4


@pytest.mark.parametrize("r", [2, 3, 5])
def test_fixed_guide_source(r):
    sc = scenes.small_scene(100, 160, band=8, gx=3, gy=2, n_spl=2, seed=5 + r)
    p = FillParams(r=r, mu=50.0, order="smart", neighborhood="rotated_ball", g_source="fixed",
                   g_fixed=(0.6, -0.8))
    ref = orc.fill(sc.image, sc.labels, None, orc.Params.of(p), tracked=True)
    u, rep, maps = engine._run_fill(sc.image, sc.labels, None, p, tracked=True, order_log=True)
    assert np.array_equal(maps["fillshell"], ref["fillshell"])
    assert float(np.abs(u - ref["u"]).max()) <= 1e-4


def test_run_tracked_accepts_pinned_tensors():
    """torch CPU tensors (pinned: DMA'd straight from the caller) and CUDA
    tensors give the numpy path's result; the result comes back as a tensor."""
    from paper_1611_05319_b200 import tracker

    sc = scenes.config("C1")
    spl = _splines(sc)
    p = FillParams(**sc.params)
    u_np, m_np = tracker.run_tracked(sc.image, sc.labels, spl, p)
    img_t = torch.from_numpy(sc.image).pin_memory()
    lab_t = torch.from_numpy(sc.labels).pin_memory()
    for img, lab in ((img_t, lab_t), (img_t.cuda(), sc.labels)):
        u_t, m_t = tracker.run_tracked(img, lab, spl, p)
        assert isinstance(u_t, torch.Tensor) and u_t.device.type == "cpu"
        assert np.array_equal(u_t.numpy(), u_np)
        assert m_t.rows == m_np.rows


def test_concurrent_host_threads():
    """Fills issued from several host threads (re-entrancy: service.py:28-104
    serialises per project, callers may still run projects in parallel)."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_1611_05319_b200 import tracker

    cases = [scenes.small_scene(90, 140, band=6, gx=3, gy=2, n_spl=2, seed=s) for s in range(4)]
    want = []
    for sc in cases:
        p = FillParams(**sc.params)
        want.append(tracker.run_tracked(sc.image, sc.labels, _splines(sc), p)[0])

    def job(i):
        sc = cases[i]
        return tracker.run_tracked(sc.image, sc.labels, _splines(sc), FillParams(**sc.params))[0]

    with ThreadPoolExecutor(4) as ex:
        got = list(ex.map(job, [0, 1, 2, 3, 0, 1, 2, 3]))
    for i, u in enumerate(got):
        assert np.array_equal(u, want[i % 4])


def test_c_abi_argument_errors():
    """The C ABI's status codes and messages (include/guidefill_b200.h:29-33)."""
    import ctypes

    lib = N.load()
    dev = torch.device("cuda")
    H, W = 40, 64
    img = torch.rand(1, H, W, 3, device=dev)
    lab = torch.zeros(1, H, W, dtype=torch.uint8, device=dev)
    lab[0, 10:20, 10:30] = 255
    out = torch.empty_like(img)
    stats = torch.zeros(1, N.GF_STATS, dtype=torch.int32, device=dev)
    rows = torch.zeros(1, 64, 2, dtype=torch.int32, device=dev)
    fr = N.FramesC(1, H, W, 3, N.GF_F32, img.data_ptr(), lab.data_ptr(), 0, out.data_ptr())
    from paper_1611_05319_b200._device import params_to_c

    pc = params_to_c(FillParams(r=3), True, N.GF_G_ZERO)
    oc = N.FillOutputsC(stats.data_ptr(), rows.data_ptr(), 64, 0, 0, 0, 0)
    need = lib.gf_fill_workspace_bytes(ctypes.byref(fr), ctypes.byref(pc))
    ws = torch.empty(need, dtype=torch.uint8, device=dev)
    stream = N.stream_ptr()
    # too small a workspace
    rc = lib.gf_fill(ctypes.byref(fr), ctypes.byref(pc), ctypes.byref(oc),
                     ctypes.c_void_p(ws.data_ptr()), need - 1, stream)
    assert rc == -3 and b"workspace" in lib.gf_last_error()
    # NULL outputs
    rc = lib.gf_fill(ctypes.byref(fr), ctypes.byref(pc), None, ctypes.c_void_p(ws.data_ptr()),
                     need, stream)
    assert rc == -1 and b"NULL" in lib.gf_last_error()
    # a ball beyond GF_MAX_RADIUS
    big = params_to_c(FillParams(r=3), True, N.GF_G_ZERO)
    big.r = 13
    rc = lib.gf_fill(ctypes.byref(fr), ctypes.byref(big), ctypes.byref(oc),
                     ctypes.c_void_p(ws.data_ptr()), need, stream)
    assert rc == -4
    # zero frames: nothing to do
    fr0 = N.FramesC(0, H, W, 3, N.GF_F32, img.data_ptr(), lab.data_ptr(), 0, out.data_ptr())
    assert lib.gf_fill(ctypes.byref(fr0), ctypes.byref(pc), ctypes.byref(oc),
                       ctypes.c_void_p(ws.data_ptr()), need, stream) == 0
    # and the valid call
    rc = lib.gf_fill(ctypes.byref(fr), ctypes.byref(pc), ctypes.byref(oc),
                     ctypes.c_void_p(ws.data_ptr()), need, stream)
    assert rc == 0
    torch.cuda.synchronize()
    assert int(stats[0, N.STAT_FILLED]) == 200 and int(stats[0, N.STAT_REMAINING]) == 0


def _force_mirror(on: bool):
    from paper_1611_05319_b200 import _staging

    key = str(torch.device("cuda", torch.cuda.current_device()))
    prev = _staging._mirror_ok.get(key)
    if on:
        _staging._mirror_ok.pop(key, None)
        assert _staging.mirror_supported(torch.device("cuda", torch.cuda.current_device()))
    else:
        _staging._mirror_ok[key] = False
    return key, prev


@pytest.mark.parametrize("dtype,C", [(torch.float64, 3), (torch.float32, 1), (torch.float32, 4),
                                     (torch.float64, 2)])
def test_output_delta_kernel(dtype, C):
    """gf_output_delta writes exactly the bitwise-changed pixels (incl. -0.0
    vs 0.0 and NaN payloads) into a mapped pinned buffer holding the input."""
    import ctypes

    gen = torch.Generator().manual_seed(C)
    n_px = 300_001
    a = torch.rand((n_px, C), generator=gen, dtype=torch.float64).to(dtype)
    b = a.clone()
    idx = torch.randperm(n_px, generator=gen)[:5000]
    b[idx, 0] = torch.rand(5000, generator=gen, dtype=torch.float64).to(dtype)
    b[7, C - 1] = float("nan")
    a[11, 0] = 0.0
    b[11, 0] = -0.0
    host = a.clone().pin_memory()
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    da, db = a.cuda(), b.cuda()
    lib = N.load()
    rc = lib.gf_output_delta(n_px, C, N.GF_F64 if dtype == torch.float64 else N.GF_F32,
                             ctypes.c_void_p(da.data_ptr()), ctypes.c_void_p(db.data_ptr()),
                             ctypes.c_void_p(host.data_ptr()), ctypes.c_void_p(cnt.data_ptr()),
                             N.stream_ptr())
    assert rc == N.GF_OK
    torch.cuda.synchronize()
    iv = torch.int64 if dtype == torch.float64 else torch.int32
    assert torch.equal(host.view(iv), b.view(iv))
    changed = int((a.view(iv) != b.view(iv)).any(dim=1).sum())
    assert int(cnt.item()) == changed
    # pageable memory is refused (not device-mapped), nothing is launched
    page = a.clone()
    rc = lib.gf_output_delta(n_px, C, N.GF_F64 if dtype == torch.float64 else N.GF_F32,
                             ctypes.c_void_p(da.data_ptr()), ctypes.c_void_p(db.data_ptr()),
                             ctypes.c_void_p(page.data_ptr()), None, N.stream_ptr())
    assert rc == N.GF_E_INVALID


@pytest.mark.parametrize("scene", ["C2", "clip"])
def test_mirrored_result_path_equals_full_download(scene):
    """The mirrored host result (input DMA'd back during the upload + changed
    pixels after the fill) equals the full-download result and the oracle,
    for numpy and pinned-tensor callers, including the Bystander clip."""
    from paper_1611_05319_b200 import _staging, tracker

    if scene == "C2":
        sc = scenes.config("C2")
        img, lab, guide = sc.image, sc.labels, _splines(sc)
        p = FillParams(**sc.params)
        field = build_guide_field(guide, lab)
    else:
        img, lab = _clip_scene(7, H=400, W=520)
        guide, field = None, None
        p = FillParams(r=3, mu=50.0, order="smart", neighborhood="rotated_ball")
    assert img.nbytes >= (1 << 20)
    ref = orc.fill(img, lab, field, orc.Params.of(p), tracked=True)
    key, prev = _force_mirror(False)
    try:
        u_full, m_full = tracker.run_tracked(img, lab, guide, p)
    finally:
        _staging._mirror_ok.pop(key, None)
    _force_mirror(True)
    u_np, m_np = tracker.run_tracked(img, lab, guide, p)
    u_t, m_t = tracker.run_tracked(torch.from_numpy(img).pin_memory(),
                                   torch.from_numpy(lab).pin_memory(), guide, p)
    assert np.array_equal(u_np, u_full)
    assert np.array_equal(u_t.numpy(), u_full)
    assert m_np.rows == m_full.rows == m_t.rows
    assert float(np.abs(u_np - ref["u"]).max()) <= 1e-4
    assert np.array_equal(u_np[lab == 0], img[lab == 0])
    if scene == "clip":
        assert np.array_equal(u_np[lab == 128], ref["u"][lab == 128])


def test_mirrored_path_concurrent_threads():
    """Several host threads on the mirrored path (per-thread side streams and
    result buffers) give the serial results."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_1611_05319_b200 import tracker

    cases = [scenes.small_scene(270, 480, band=8, gx=5, gy=3, n_spl=4, seed=40 + s)
             for s in range(3)]
    assert cases[0].image.nbytes >= (1 << 20)
    want = [tracker.run_tracked(sc.image, sc.labels, _splines(sc), FillParams(**sc.params))[0]
            for sc in cases]

    def job(i):
        sc = cases[i]
        return tracker.run_tracked(sc.image, sc.labels, _splines(sc), FillParams(**sc.params))[0]

    with ThreadPoolExecutor(3) as ex:
        got = list(ex.map(job, [0, 1, 2, 0, 1, 2]))
    for i, u in enumerate(got):
        assert np.array_equal(u, want[i % 3])


def test_pageable_staging_never_writes_a_live_result():
    """Pageable numpy frames are copied by host threads into a pooled pinned
    result buffer before the DMA: a result (or only a view of it) kept by
    the caller is never the buffer a later call of the same size stages
    into, and a released one is recycled without stale pixels."""
    import gc

    from paper_1611_05319_b200 import tracker

    cases = [scenes.small_scene(270, 480, band=8, gx=5, gy=3, n_spl=4, seed=70 + s)
             for s in range(3)]
    assert cases[0].image.nbytes >= (1 << 20)
    run = [lambda sc=sc: tracker.run_tracked(sc.image, sc.labels, _splines(sc),
                                             FillParams(**sc.params))[0] for sc in cases]
    first = run[0]()
    want0 = first.copy()
    view = first[..., 1]  # keep only a view of the first result
    del first
    gc.collect()
    second = run[1]()
    third = run[2]()
    assert np.array_equal(view, want0[..., 1])
    want2 = third.copy()
    del second, third
    gc.collect()
    again = run[2]()  # recycled buffer: fully rewritten
    assert np.array_equal(again, want2)
    assert np.array_equal(view, want0[..., 1])


def test_page_locked_numpy_inputs_take_the_direct_dma():
    """numpy arrays living in page-locked memory (a field returned by
    build_guide_field, a view of a pinned tensor) are DMA'd without the
    staging copy and give the same result as pageable arrays."""
    from paper_1611_05319_b200 import tracker

    sc = scenes.config("C2")
    spl = _splines(sc)
    p = FillParams(**sc.params)
    field = build_guide_field(spl, sc.labels)
    assert torch.from_numpy(field.reshape(-1).view(np.uint8)).is_pinned()
    img_locked = torch.from_numpy(sc.image).pin_memory().numpy()
    u_ref, m_ref = tracker.run_tracked(sc.image, sc.labels, field.copy(), p)
    u, m = tracker.run_tracked(img_locked, sc.labels, field, p)
    assert np.array_equal(u, u_ref) and m.rows == m_ref.rows
    u2, _ = tracker.run_tracked(sc.image, sc.labels, spl, p)
    assert np.array_equal(u2, u_ref)


@pytest.mark.parametrize("kind,depth", [("numpy", 2), ("pinned", 2), ("pinned", 1),
                                        ("numpy", 3)])
def test_fill_video_host_pipelined_equals_single_calls(kind, depth):
    """video.fill_video_host (uploads / fills / downloads on three streams)
    gives every frame's run_tracked result, with shared and per-frame masks
    and splines."""
    from paper_1611_05319_b200 import tracker, video

    frames = [scenes.small_scene(270, 480, band=8, gx=5, gy=3, n_spl=4, seed=1611, frame=f)
              for f in range(5)]
    p = FillParams(**frames[0].params)
    spl = [_splines(sc) for sc in frames]
    want = [tracker.run_tracked(sc.image, sc.labels, spl[i], p) for i, sc in enumerate(frames)]
    if kind == "pinned":
        imgs = [torch.from_numpy(sc.image).pin_memory() for sc in frames]
    else:
        imgs = [sc.image for sc in frames]
    got = video.fill_video_host(imgs, [sc.labels for sc in frames], spl, p, depth=depth)
    for (u, rep), (u_w, m_w) in zip(got, want):
        u = u.numpy() if isinstance(u, torch.Tensor) else u
        assert np.array_equal(u, u_w)
        assert rep.rows == m_w.rows and rep.iterations == m_w.iterations
    seen = []
    assert video.fill_video_host(imgs, [sc.labels for sc in frames], spl, p, depth=depth,
                                 on_frame=lambda f, u, rep: seen.append((f, rep.rows))) is None
    assert [f for f, _ in seen] == list(range(5))
    assert all(rows == want[f][1].rows for f, rows in seen)
    # one mask and one spline set for all frames
    got = video.fill_video_host(imgs[:3], frames[0].labels, spl[0], p, depth=depth)
    for i, (u, rep) in enumerate(got):
        u_w, m_w = tracker.run_tracked(frames[i].image, frames[0].labels, spl[0], p)
        u = u.numpy() if isinstance(u, torch.Tensor) else u
        assert np.array_equal(u, u_w) and rep.rows == m_w.rows


def test_fill_video_host_bad_labels_raise_and_drain():
    """A bad mask mid-stream raises the reference's ValueError (grid.py:36-46);
    the pipeline drains its in-flight copies, and the next call is clean."""
    from paper_1611_05319_b200 import tracker, video

    frames = [scenes.small_scene(270, 480, band=8, gx=5, gy=3, n_spl=4, seed=7, frame=f)
              for f in range(4)]
    p = FillParams(**frames[0].params)
    labs = [sc.labels.copy() for sc in frames]
    labs[2][5, 5] = 7
    with pytest.raises(ValueError):
        video.fill_video_host([sc.image for sc in frames], labs, [_splines(sc) for sc in frames], p)
    got = video.fill_video_host([sc.image for sc in frames[:2]], [sc.labels for sc in frames[:2]],
                                [_splines(sc) for sc in frames[:2]], p)
    for (u, rep), sc in zip(got, frames[:2]):
        u_w, m_w = tracker.run_tracked(sc.image, sc.labels, _splines(sc), p)
        assert np.array_equal(u, u_w) and rep.rows == m_w.rows


def _paint_reference(u, labels, fillshell):
    """engine.py:270-283 with scipy's EDT (test-side checker)."""
    from scipy import ndimage

    stranded = (labels == 255) & (fillshell < 0)
    readable = (labels == 0) | ((labels == 255) & (fillshell >= 0))
    u = u.copy()
    if readable.any():
        _, (jn, inn) = ndimage.distance_transform_edt(~readable, return_indices=True)
        jr, ir = np.nonzero(stranded)
        u[jr, ir] = u[jn[jr, ir], inn[jr, ir]]
    else:
        u[stranded] = 0.5
    return u, int(stranded.sum())


@pytest.mark.parametrize("seed", range(12))
def test_unfillable_paint_matches_scipy_edt(seed):
    """gf_paint_unfillable == scipy distance_transform_edt indices, ties
    included: sparse readable sets on lattices of many shapes (every pixel a
    distinct colour, so any wrong nearest pixel shows)."""
    from paper_1611_05319_b200.engine import _paint_unfillable_device

    rng = np.random.default_rng(seed)
    H, W = int(rng.integers(1, 90)), int(rng.integers(1, 130))
    C = int(rng.integers(1, 5))
    dtype = np.float64 if seed % 2 == 0 else np.float32
    labels = rng.choice(np.array([0, 128, 255], np.uint8), size=(H, W),
                        p=[0.02, 0.05, 0.93] if seed % 3 else [0.2, 0.3, 0.5])
    fillshell = np.where(rng.random((H, W)) < 0.03, 1, -1).astype(np.int32)
    fillshell[labels != 255] = -1
    if seed == 5:
        labels[labels == 0] = 128  # nothing Readable
        fillshell[:] = -1
    u = rng.random((H, W, C)).astype(dtype)
    want, n_want = _paint_reference(u, labels, fillshell)
    d_u = torch.from_numpy(u).cuda()
    n = _paint_unfillable_device(d_u, torch.from_numpy(labels).cuda(),
                                 torch.from_numpy(fillshell).cuda())
    assert n == n_want
    assert np.array_equal(d_u.cpu().numpy(), want)


def test_unfillable_paint_large_ties():
    """A 1080p lattice with three readable pixels: long equidistant ridges."""
    from paper_1611_05319_b200.engine import _paint_unfillable_device

    H, W = 1080, 1920
    labels = np.full((H, W), 255, np.uint8)
    for (r, c) in ((100, 100), (100, 1700), (900, 960)):
        labels[r, c] = 0
    fillshell = np.full((H, W), -1, np.int32)
    u = np.random.default_rng(3).random((H, W, 3))
    want, n_want = _paint_reference(u, labels, fillshell)
    d_u = torch.from_numpy(u).cuda()
    assert _paint_unfillable_device(d_u, torch.from_numpy(labels).cuda(),
                                    torch.from_numpy(fillshell).cuda()) == n_want
    assert np.array_equal(d_u.cpu().numpy(), want)


def test_fill_video_multi_equals_single_calls():
    """video.fill_video_multi (frame blocks over the devices, one host thread
    each) on the visible GPUs: every frame equals its run_tracked result,
    with per-frame masks as a list and as an (N, H, W) stack; a mask of the
    wrong shape is refused before anything runs."""
    from paper_1611_05319_b200 import tracker, video

    frames = [scenes.small_scene(270, 480, band=8, gx=5, gy=3, n_spl=4, seed=99, frame=f)
              for f in range(5)]
    p = FillParams(**frames[0].params)
    spl = [_splines(sc) for sc in frames]
    want = [tracker.run_tracked(sc.image, sc.labels, spl[i], p) for i, sc in enumerate(frames)]
    imgs = [sc.image for sc in frames]
    for labs in ([sc.labels for sc in frames], np.stack([sc.labels for sc in frames])):
        got = video.fill_video_multi(imgs, labs, spl, p)
        for (u, rep), (u_w, m_w) in zip(got, want):
            assert np.array_equal(u, u_w)
            assert rep.rows == m_w.rows
    seen = {}
    video.fill_video_multi(imgs, [sc.labels for sc in frames], spl, p, devices=[0],
                           on_frame=lambda f, u, rep: seen.__setitem__(f, rep.filled))
    assert seen == {f: want[f][1].report.filled for f in range(5)}
    with pytest.raises(ValueError, match="differ"):
        video.fill_video_multi(imgs, frames[0].labels[:-1], spl, p)
    with pytest.raises(ValueError):
        video.fill_video_host(imgs, np.stack([sc.labels for sc in frames])[:3], spl, p)


def test_device_rendered_video_matches_host_generator():
    """scenes.video_batch_device: labels and splines of the C5 frames are
    bit-identical to the host generator, so |D| and the fill order are the
    same work the CPU baseline measures."""
    frames = [0, 17, 255]
    images, labels, spl = scenes.video_batch_device(frames, torch.device("cuda"))
    for b, f in enumerate(frames):
        sc = scenes.config("C5", frame=f)
        assert np.array_equal(labels[b].cpu().numpy(), sc.labels)
        for a, c in zip(spl[b], sc.splines):
            assert np.array_equal(a["points"], c["points"]) and a["direction"] == c["direction"]
        img = images[b].cpu().numpy()
        assert float(np.abs(img - sc.image).max()) <= 0.05 + 1e-6  # noise differs only
        assert not img[sc.labels == 255].any()


def test_batch_graph_equals_per_frame_fills():
    """_device.BatchGraph (bench.py's C5 step: chunks of frames, one graph)
    gives each frame's single-frame fill."""
    from paper_1611_05319_b200._device import BatchGraph

    images, labels, spl = scenes.video_batch_device([3, 4, 5], torch.device("cuda"))
    splines = [[Spline(id=s["id"], source="user", direction=s["direction"], points=s["points"],
                       kind=s["kind"]) for s in fs] for fs in spl]
    p = FillParams(**scenes.config("C5").params)
    g = BatchGraph(images, labels, splines, p, chunk=2)
    assert g.launches_per_replay == 4  # k_prep + k_shells per chunk
    parts = g.replay()
    torch.cuda.synchronize()
    from paper_1611_05319_b200._device import SegmentSet

    for b in range(3):
        part = parts[b // 2]
        one = fill_device(images[b:b + 1], labels[b:b + 1], None, p,
                          splines=SegmentSet(splines[b], images.device))
        assert torch.equal(part["out"][b % 2], one["out"][0])
        assert torch.equal(part["stats"][b % 2], one["stats"][0])


def test_bench_line_single_gpu(tmp_path):
    """bench.py's own rank loop end to end (short): one JSON line with the C2
    value, the C5 block, launch counts from the library counter."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "3",
                          "--warmup", "3", "--c5-frames", "6", "--chunk", "4", "--no-cpu"],
                         capture_output=True, text=True, timeout=900, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["value"] > 0
    assert line["c5"]["frames_total"] == 6 and line["c5"]["value"] > 0
    assert line["gpu_launches"] == 2 * 3
    assert line["e2e"]["value"] > 0 and line["c5"]["e2e"]["value"] > 0


def test_bench_multi_rank_path_on_one_device(tmp_path):
    """bench.py --gpus 2 spawns its own ranks, splits the C5 batch into frame
    blocks and reduces over the ranks; on a one-GPU box both ranks share
    device 0 (gloo bookkeeping): a functional check of the N > 1 line, not a
    measurement."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GF_BENCH_ONE_DEVICE="1")
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps",
                          "3", "--warmup", "3", "--c5-frames", "6", "--chunk", "2", "--no-e2e"],
                         capture_output=True, text=True, timeout=900, cwd=root, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["global_batch"] == 6
    assert line["c5"]["frames_per_gpu"] == 3 and line["value"] == line["c5"]["value"]
    assert line["c5"]["inpaint_px_total"] > 0
