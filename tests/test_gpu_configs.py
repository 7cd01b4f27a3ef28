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
