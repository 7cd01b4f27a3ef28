"""Host-side API behaviour that needs no GPU: parameter validation, presets,
serialisation, report formulas and the reference's ValueError messages."""

import math

import numpy as np
import pytest

from oracle import guidefill_oracle as orc
from paper_1611_05319_b200 import FillParams, Spline, WorkMetrics, dumps, loads, engine, tracker
from paper_1611_05319_b200 import grid


def test_params_validation_and_serialization():
    with pytest.raises(ValueError):
        FillParams(order="random")
    with pytest.raises(ValueError):
        FillParams(r=0)
    with pytest.raises(ValueError):
        FillParams(neighborhood="square")
    with pytest.raises(ValueError):
        FillParams(mu=-1.0)
    assert FillParams(mu=math.inf).to_dict()["mu"] == "inf"
    assert FillParams.telea().g_fixed == (0.0, 0.0)
    assert FillParams.coherence_transport().r == 5


def test_dimension_mismatch_raises_before_touching_the_gpu():
    with pytest.raises(ValueError, match="differ"):
        engine.inpaint(np.zeros((4, 5, 3)), np.zeros((4, 4), dtype=np.uint8))
    with pytest.raises(ValueError, match="guide"):
        engine.inpaint(np.zeros((4, 4, 3)), np.zeros((4, 4), dtype=np.uint8), np.zeros((4, 5, 2)))
    with pytest.raises(ValueError, match="differ"):
        tracker.run_tracked(np.zeros((4, 5, 1)), np.zeros((4, 4), dtype=np.uint8))
    with pytest.raises(ValueError, match="allowed values"):
        engine.inpaint(np.zeros((4, 4, 1)), np.full((4, 4), 7, dtype=np.uint8))


def test_weight_frozen_value():
    w = engine.weight((0.0, 0.0), (1.0, -1.0), (0.0, 1.0), mu=10.0, eps=3.0)
    assert w == pytest.approx(0.0027336183461468657, rel=1e-15)
    assert engine.weight((0, 0), (3.0, 4.0), (0, 0), 50.0, 3.0) == pytest.approx(0.2, rel=1e-15)
    with pytest.raises(ValueError):
        engine.weight((1.0, 1.0), (1.0, 1.0), (0.0, 1.0), mu=10.0, eps=3.0)


def test_ready_predicates():
    assert engine.ready(0.0, (0, 0), FillParams(order="onion"))
    assert engine.ready(0.2, (0, 0), FillParams(order="smart"))
    assert not engine.ready(0.04, (0, 0), FillParams(order="smart"))
    p = FillParams(order="smart_with_data_term")
    assert not engine.ready(0.2, (0.0, 0.0), p)
    assert engine.ready(0.2, (0.0, 0.3), p)
    assert engine.ready(0.2, (0.0, 0.0), p, data_term_live=False)


def test_work_metrics_formulas():
    wm = WorkMetrics(rows=[(0, 10, 40, 10, 10), (1, 3, 5, 3, 3)])
    assert wm.work_total == 69 and wm.threads_max == 10 and wm.iterations == 2
    assert WorkMetrics(rows=[(0, 1, 1, 1, 1)]).work_total == 1
    text = wm.to_csv()
    assert text.splitlines()[0] == "iteration,frontier_size,candidates,threads_requested,filled"


def test_disk_offsets_match_reference_order():
    for r in range(1, 8):
        assert np.array_equal(grid.offsets_in_disk(r), orc.disk_offsets(r))


def test_spline_flattening_matches_oracle():
    rng = np.random.default_rng(3)
    for _ in range(50):
        pts = rng.uniform(-50, 150, size=(3 * int(rng.integers(1, 4)) + 1, 2))
        sp = Spline(id="b", source="user", direction=(0.1, 0.2), points=pts, kind="bezier")
        assert sp.polyline().tobytes() == orc.polyline(pts, "bezier").tobytes()


def test_spline_wire_format_round_trip():
    sp = [Spline(id="a", source="user", direction=(0.5, -0.25), points=[[0.0, 1.0], [2.5, 3.0]]),
          Spline(id="b", source="auto", direction=(0.0, 1.0), kind="bezier",
                 points=[[0, 0], [1, 2], [3, 4], [5, 6]])]
    text = dumps(sp)
    back = loads(text)
    assert dumps(back) == text
    with pytest.raises(ValueError):
        loads('{"version": 2, "splines": []}')


def test_pooled_result_buffers_outlive_their_views():
    """A view of a returned result keeps its pooled buffer out of the pool
    (the buffer used to be recycled when the first array died)."""
    import gc

    import torch

    from paper_1611_05319_b200 import _staging

    class Pool(_staging._PinnedPool):
        @staticmethod
        def _alloc(n):  # pageable stand-in: the lifetime logic is the same
            return torch.empty(max(n, 1), dtype=torch.uint8)

    pool = Pool()
    a, _ = pool.take((4, 5, 3), np.float64)
    a[...] = 1.0
    v, w = a[..., 0], a.reshape(-1, 3)
    del a
    gc.collect()
    b, _ = pool.take((4, 5, 3), np.float64)
    b[...] = 2.0
    assert float(v[0, 0]) == 1.0 and float(w[0, 0]) == 1.0
    del v, w, b
    gc.collect()
    assert len(pool.free[4 * 5 * 3 * 8]) == 2  # both buffers came back
    t, _ = pool.take_tensor((4, 5, 3), torch.float64)
    t.fill_(3.0)
    tv = t[..., 0]
    del t
    gc.collect()
    c, _ = pool.take((4, 5, 3), np.float64)
    c[...] = 4.0
    assert float(tv[0, 0]) == 3.0
