"""The exact-math primitives of the CUDA decision path match numpy bit for bit.

gf_math.cuh is compiled into libgf_b200.so for both the device kernels and
these host exports (gf_host_*), so checking the host build against numpy
pins the very source the kernels use.  SVML exp equality holds on AVX512_SKX
hosts (numpy's dispatch there); elsewhere numpy calls libm exp and the test
is skipped.
"""

import ctypes

import numpy as np
import pytest

from oracle import guidefill_oracle as orc
from paper_1611_05319_b200 import _native

lib = _native.load()
P = ctypes.c_void_p


def host_exp(x):
    y = np.empty_like(x)
    lib.gf_host_exp(x.ctypes.data_as(P), y.ctypes.data_as(P), x.size)
    return y


def host_hypot(x, y):
    o = np.empty_like(x)
    lib.gf_host_hypot(x.ctypes.data_as(P), y.ctypes.data_as(P), o.ctypes.data_as(P), x.size)
    return o


@pytest.mark.skipif(orc.numpy_exp_flavour() != "svml", reason="numpy uses libm exp on this host")
@pytest.mark.parametrize("lo,hi", [(-750, 0), (-1, 1), (-800, 710), (-746, -700), (-1e-12, 1e-12),
                                   (-708.5, -708.3), (-745.2, -744.0), (700, 720)])
def test_exp_matches_numpy(lo, hi):
    rng = np.random.default_rng(int(abs(lo) * 7 + hi))
    x = rng.uniform(lo, hi, 400_000)
    with np.errstate(over="ignore"):
        ref = np.exp(x)
    assert np.array_equal(host_exp(x).view(np.int64), ref.view(np.int64))


@pytest.mark.skipif(orc.numpy_exp_flavour() != "svml", reason="numpy uses libm exp on this host")
def test_exp_weight_arguments_and_specials():
    rng = np.random.default_rng(5)
    # the fill's arguments are coef * d * d with coef = -mu^2 / (2 r^2)
    coef = -(50.0 * 50.0) / (2.0 * 9.0)
    d = rng.uniform(-4, 4, 300_000)
    x = (coef * d) * d
    assert np.array_equal(host_exp(x).view(np.int64), np.exp(x).view(np.int64))
    sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 709.78, 709.79, -745.13, -745.14,
                   5e-324, -5e-324, -708.3964185322641, -707.7032713517042])
    with np.errstate(over="ignore", invalid="ignore"):
        ref = np.exp(sp)
    got = host_exp(sp)
    assert np.array_equal(np.isnan(ref), np.isnan(got))
    m = ~np.isnan(ref)
    assert np.array_equal(got[m].view(np.int64), ref[m].view(np.int64))


@pytest.mark.parametrize("scale", [1.0, 5.0, 1e-3, 1e300, 1e-300])
def test_hypot_matches_numpy(scale):
    rng = np.random.default_rng(int(scale * 1000) % 9973)
    x = rng.uniform(-scale, scale, 300_000)
    y = rng.uniform(-scale, scale, 300_000)
    assert np.array_equal(host_hypot(x, y).view(np.int64), np.hypot(x, y).view(np.int64))


def test_hypot_ball_offsets():
    # rotated ball points at arbitrary guide angles (engine.py:155-164)
    rng = np.random.default_rng(11)
    g = rng.uniform(-1, 1, size=(5000, 2))
    offs = orc.disk_offsets(6)[1:]
    rel = orc.ball_points(g, offs, True)
    x = np.ascontiguousarray(rel[..., 0]).ravel()
    y = np.ascontiguousarray(rel[..., 1]).ravel()
    assert np.array_equal(host_hypot(x, y), np.hypot(x, y))


@pytest.mark.parametrize("n", list(range(1, 40)) + [48, 80, 112, 127, 128, 129, 148, 196, 252,
                                                   316, 376, 440])
def test_pairwise_plan_matches_numpy_row_sum(n):
    # numpy's reduction over the last axis of an (F, K) array, engine.py:193-194
    rng = np.random.default_rng(n)
    a = rng.uniform(0, 1, size=(64, n)) * np.exp(rng.uniform(-40, 0, size=(64, n)))
    ref = a.sum(axis=1)
    got = np.array([lib.gf_host_pairwise_sum(np.ascontiguousarray(row).ctypes.data_as(P), n)
                    for row in a])
    assert np.array_equal(got.view(np.int64), ref.view(np.int64))


# ---- coherence directions: numpy arctan2 / tanh (SVML) and sin / cos (libm) ----
# guide.eigen_2x2 (guide.py:123-136): phi = 0.5 * arctan2(2b, a - c),
# v = (-sin phi, cos phi), coherence tanh((hi - lo) / lam).  gf_npmath.cuh.

def _bits_equal(got, ref):
    same = got.view(np.int64) == ref.view(np.int64)
    return bool(np.all(same | (np.isnan(got) & np.isnan(ref))))


def host_atan2(y, x):
    o = np.empty_like(x)
    lib.gf_host_atan2(y.ctypes.data_as(P), x.ctypes.data_as(P), o.ctypes.data_as(P), x.size)
    return o


def host_tanh(x):
    o = np.empty_like(x)
    lib.gf_host_tanh(x.ctypes.data_as(P), o.ctypes.data_as(P), x.size)
    return o


def host_sincos(x):
    s, c = np.empty_like(x), np.empty_like(x)
    lib.gf_host_sincos(x.ctypes.data_as(P), s.ctypes.data_as(P), c.ctypes.data_as(P), x.size)
    return s, c


N_EXACT = 10_000_000


@pytest.mark.skipif(orc.numpy_exp_flavour() != "svml", reason="numpy has no SVML on this host")
@pytest.mark.parametrize("span", [(0, 0), (-12, 8)])
def test_atan2_matches_numpy(span):
    # 10 M pairs: unit normals, then magnitudes spread over 1e-12 .. 1e8
    rng = np.random.default_rng(101 + span[0])
    y = rng.standard_normal(N_EXACT)
    x = rng.standard_normal(N_EXACT)
    if span != (0, 0):
        y *= 10.0 ** rng.uniform(*span, N_EXACT)
        x *= 10.0 ** rng.uniform(*span, N_EXACT)
    assert _bits_equal(host_atan2(y, x), np.arctan2(y, x))


@pytest.mark.skipif(orc.numpy_exp_flavour() != "svml", reason="numpy has no SVML on this host")
def test_atan2_structure_tensor_arguments_and_specials():
    # the coherence arguments (2 J12, J11 - J22) of smoothed squared gradients,
    # exact ties and near-axis directions included
    rng = np.random.default_rng(7)
    a = rng.uniform(0, 1, 2_000_000) ** 2
    c = rng.uniform(0, 1, 2_000_000) ** 2
    b = rng.uniform(-1, 1, 2_000_000) * np.sqrt(a * c)
    b[::7] = 0.0
    c[::11] = a[::11]
    y, x = 2.0 * b, a - c
    assert _bits_equal(host_atan2(y, x), np.arctan2(y, x))
    sp = np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 1e-310, -1e-310, 1e300,
                   -1e300, 5e-324, 1.7e308, -1.7e308, 2.0 ** -1021, 2.0 ** 993, 3e-308])
    Y, X = (v.ravel().copy() for v in np.meshgrid(sp, sp))
    assert _bits_equal(host_atan2(Y, X), np.arctan2(Y, X))


@pytest.mark.skipif(orc.numpy_exp_flavour() != "svml", reason="numpy has no SVML on this host")
def test_tanh_matches_numpy():
    rng = np.random.default_rng(13)
    z = rng.standard_normal(N_EXACT) * 10.0 ** rng.uniform(-8, 2.5, N_EXACT)
    assert _bits_equal(host_tanh(z), np.tanh(z))
    sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-310, 5e-324, 1e308, -1e308, 19.0,
                   19.1, 20.0, 0.125, 0.140625, 0.1249999, 1.7e308])
    assert _bits_equal(host_tanh(sp), np.tanh(sp))


@pytest.mark.parametrize("lo,hi,logspan", [(-np.pi / 2, np.pi / 2, 0), (-2.4262, 2.4262, 0),
                                           (-1.0, 1.0, 12)])
def test_sincos_match_numpy(lo, hi, logspan):
    # phi = 0.5 * arctan2(...) lies in [-pi/2, pi/2]; small angles exercise the
    # 2^-26 / 2^-27 shortcuts and the Taylor branch
    rng = np.random.default_rng(17 + logspan)
    p = rng.uniform(lo, hi, N_EXACT)
    if logspan:
        p *= 10.0 ** rng.uniform(-logspan, 0, N_EXACT)
    s, c = host_sincos(p)
    assert _bits_equal(s, np.sin(p))
    assert _bits_equal(c, np.cos(p))
