"""GPU parity of the post-processing chain (reference postprocess.cpp:40-197) against the
reference's smoothChain (oracle/_ref ref_smooth_chain): values and validity bit-exact."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl

from conftest import bits_equal, ref_render

pytestmark = pytest.mark.gpu

U8 = ctypes.POINTER(ctypes.c_uint8)
DP = ctypes.POINTER(ctypes.c_double)


def ref_chain(reference, values, valid, steps):
    H, W = values.shape
    kinds = (ctypes.c_int * len(steps))(*[s[0] for s in steps])
    radii = (ctypes.c_int * len(steps))(*[s[1] for s in steps])
    sig = (ctypes.c_double * len(steps))(*[float(s[2]) for s in steps])
    v = np.ascontiguousarray(values, dtype=np.float64)
    ok = np.ascontiguousarray(valid, dtype=np.uint8)
    vo, oo = np.empty_like(v), np.empty_like(ok)
    rc = reference.ref_smooth_chain(v.ctypes.data_as(DP), ok.ctypes.data_as(U8), W, H, kinds, radii, sig,
                                    len(steps), vo.ctypes.data_as(DP), oo.ctypes.data_as(U8))
    if rc != 0:
        raise pk.ReliefError(8, reference.ref_last_error().decode())
    return vo, oo


def _random_layer(rng, H, W, p_valid):
    values = rng.normal(0.0, 0.3, (H, W)).cumsum(axis=1) * 0.05
    valid = (rng.random((H, W)) < p_valid).astype(np.uint8)
    # carve invalid blobs so inpaint components have interiors and some lack borders
    for _ in range(6):
        r, c = rng.integers(0, H), rng.integers(0, W)
        valid[max(0, r - 4):r + 4, max(0, c - 6):c + 6] = 0
    values[valid == 0] = np.nan
    return values, valid


@pytest.mark.parametrize("steps", [
    wl.C5_CHAIN,
    [(2, 2, 1.0)],
    [(0, 3, 1.7), (1, 2, 1.0)],
    [(3, 0, 1.0)],
    [(3, 0, 1.0), (3, 0, 1.0), (2, 1, 1.0)],
])
def test_chain_matches_reference_random(gpu, reference, steps):
    rng = np.random.default_rng(len(steps))
    for p_valid in (0.9, 0.5, 0.1):
        values, valid = _random_layer(rng, 47, 63, p_valid)
        got_v, got_ok = pk.smooth_chain(gpu, values, valid, steps)
        want_v, want_ok = ref_chain(reference, values, valid, steps)
        assert np.array_equal(got_ok, want_ok)
        assert bits_equal(got_v, want_v).all(), np.nanmax(np.abs(got_v - want_v))


@pytest.mark.parametrize("radius", [1, 2])
def test_median_ties_zeros_and_nan(gpu, reference, radius):
    """Median windows with repeated values, +0 / -0 and NaN among the valid values: which of two
    equal-comparing values lands on the median rank is decided by the reference's stable insertion
    sort (std::sort on < 16 elements); the device's 3x3 network path defers such windows to the same
    insertion order, so values stay bit-exact."""
    rng = np.random.default_rng(7 + radius)
    H, W = 40, 70
    values = rng.integers(-3, 4, (H, W)).astype(np.float64) * 0.25   # many exact ties
    values[rng.random((H, W)) < 0.15] = -0.0
    values[rng.random((H, W)) < 0.02] = np.nan
    valid = (rng.random((H, W)) < 0.85).astype(np.uint8)
    steps = [(2, radius, 1.0)]
    got_v, got_ok = pk.smooth_chain(gpu, values, valid, steps)
    want_v, want_ok = ref_chain(reference, values, valid, steps)
    assert np.array_equal(got_ok, want_ok)
    assert bits_equal(got_v, want_v).all()
    # all-valid smooth layer: the network path on every interior cell
    smooth = rng.normal(1.0, 0.2, (H, W)).cumsum(axis=0)
    full = np.ones((H, W), dtype=np.uint8)
    got_v, _ = pk.smooth_chain(gpu, smooth, full, steps)
    want_v, _ = ref_chain(reference, smooth, full, steps)
    assert bits_equal(got_v, want_v).all()


def test_nothing_to_inpaint_status(gpu, reference):
    values = np.full((8, 9), np.nan)
    valid = np.zeros((8, 9), dtype=np.uint8)
    with pytest.raises(pk.ReliefError) as e:
        pk.smooth_chain(gpu, values, valid, [(3, 0, 1.0)])
    assert e.value.status == 8
    with pytest.raises(pk.ReliefError):
        ref_chain(reference, values, valid, [(3, 0, 1.0)])


def test_c5_chain_on_mapped_elevation(gpu, reference, tmp_path):
    """C5: the chain on the elevation layer of a map built from C3 LiDAR frames."""
    text = wl._map(0.04, 250, 250) + "noise.alpha_d = 0.0002\n" + wl.lidar(512, rings=64) + wl.SCENE_S0
    p = tmp_path / "c5.config"
    p.write_text(text)
    cfg = pk.Config.load(gpu, p)
    m = pk.ReliefMap.create(gpu, 0.04, 250, 250)
    for f in range(3):
        pose = wl.pose34(np.eye(3), (0.04 * f, 0.0, 1.0))
        m.integrate(ref_render(reference, p, pose, 0.1 * f, 5, f), pose, 0.1 * f, cfg)
    elev = m.layer("elevation")
    valid = m.layer("valid").astype(np.uint8)
    got_v, got_ok = m.smooth_chain("elevation", wl.C5_CHAIN)
    want_v, want_ok = ref_chain(reference, elev, valid, wl.C5_CHAIN)
    assert np.array_equal(got_ok, want_ok)
    assert bits_equal(got_v, want_v).all()
