"""Known-answer tests restated from the reference's own suites, run through the public C ABI
against every implementation: the product (GPU), the reference compiled in place and the C
restatement (CPU). Map states are injected with relief_map_load (crafted snapshots) where the
implementation supports it. Each case cites the reference test it restates."""
from __future__ import annotations

import ctypes
import math

import numpy as np
import pytest

import paper_2204_12876_b200 as pk

import snapshots as snap
from conftest import REF_LIB, RESTATE_LIB, bits_equal

QUIET = ("drift.enabled = false\ncleanup.enabled = false\ncleanup.upper_bound_enabled = false\n"
         "overlap.enabled = false\nexclusion.enabled = false\n")


@pytest.fixture(scope="module", params=[
    pytest.param("product", marks=pytest.mark.gpu), "reference", "restate"])
def impl(request, product, reference):
    if request.param == "product":
        if product.relief_gpu_device_count() <= 0:
            pytest.fail("GPU case needs a CUDA device")
        return product
    if request.param == "reference":
        return reference
    import subprocess
    from conftest import ROOT
    subprocess.run(["make", "-C", str(ROOT / "oracle"), "restate"], check=True, capture_output=True)
    return pk.load_library(RESTATE_LIB, gpu_api=False)


def _supports_load(lib):
    return "liboracle" not in lib._relief_path


def _map_from(lib, tmp_path, layers, res, center=(0.0, 0.0), name="m"):
    p = tmp_path / f"{name}.relief"
    p.write_text(snap.text(layers, res, center))
    return pk.ReliefMap.load(lib, p)


def _cfg(lib, tmp_path, text, name="c"):
    p = tmp_path / f"{name}.config"
    p.write_text(text)
    return pk.Config.load(lib, p)


def _point_above(cell_rc, res, W, H, z_map, sensor_z):
    """Sensor-frame point (identity rotation, sensor at (0.05,0.05,sensor_z)) landing in cell_rc."""
    r, c = cell_rc
    ox, oy = -0.5 * W * res, -0.5 * H * res
    x = ox + (c + 0.5) * res - 0.05
    y = oy + (r + 0.5) * res - 0.05
    return np.array([[x, y, z_map - sensor_z]])


POSE = pk.pose34(t=(0.05, 0.05, 3.0))


# ---- Kalman gates (reference test_integration.cpp:50-108) ---------------------------
@pytest.mark.parametrize("case", ["average", "outlier", "cap", "wall"])
def test_kalman_known_answers(impl, tmp_path, case):
    if not _supports_load(impl):
        pytest.skip("restatement has no snapshot loader")
    res, W, H = 0.1, 10, 10
    layers = snap.fresh(H, W)
    cfg_text = QUIET + "noise.alpha_d = 0\nupdate.max_range = 1000\n"
    if case == "average":       # h=0 var=1, z=2 sp=1 -> h=1 var=0.5
        snap.set_cell(layers, 5, 5, 0.0, 1.0)
        cfg_text += "noise.sigma_p_min2 = 1\n"
        pts = _point_above((5, 5), res, W, H, 2.0, 3.0)
    elif case == "outlier":     # |1-0|/0.1 = 10 > 2.5 -> var 0.01 + 0.01
        snap.set_cell(layers, 5, 5, 0.0, 0.01)
        cfg_text += "noise.sigma_p_min2 = 0.04\nupdate.sigma_outlier2 = 0.01\n"
        pts = _point_above((5, 5), res, W, H, 1.0, 3.0)
    elif case == "cap":         # inflation capped at sigma_max2
        snap.set_cell(layers, 5, 5, 0.0, 0.9)
        cfg_text += "noise.sigma_p_min2 = 0.04\nupdate.sigma_outlier2 = 50\nupdate.sigma_max2 = 1\n"
        pts = _point_above((5, 5), res, W, H, 100.0, 3.0)
    else:                       # 8 low points in a crowded cell: all ignored, state unchanged
        snap.set_cell(layers, 5, 5, 1.0, 0.01)
        cfg_text += "noise.sigma_p_min2 = 0.04\nupdate.wall_count_threshold = 5\n"
        pts = np.repeat(_point_above((5, 5), res, W, H, 0.2, 3.0), 8, axis=0)
    m = _map_from(impl, tmp_path, layers, res)
    st = m.integrate(pts, POSE, 0.0, _cfg(impl, tmp_path, cfg_text))
    h, v = m.layer("elevation")[5, 5], m.layer("variance")[5, 5]
    if case == "average":
        assert st.points_fused == 1 and h == 1.0 and v == 0.5
    elif case == "outlier":
        assert st.points_rejected_outlier == 1 and h == 0.0 and v == 0.02
    elif case == "cap":
        assert st.points_rejected_outlier == 1 and v == 1.0
    else:
        assert st.points_ignored_low == 8 and h == 1.0 and v == 0.01


# ---- harmonic-sum recursion (reference test_integration.cpp:110-131) ---------------
def test_repeated_fusion_follows_harmonic_sum(impl, tmp_path):
    res, W, H = 0.1, 10, 10
    cfg = _cfg(impl, tmp_path, QUIET + "noise.alpha_d = 0\nnoise.sigma_p_min2 = 0.04\n"
               "update.mahalanobis_threshold = 1e9\nupdate.sigma_t2 = 0\n")
    m = pk.ReliefMap.create(impl, res, W, H)
    pts = _point_above((5, 5), res, W, H, 5.0, 3.0)
    info = 1.0 / 100.0  # sigma_init2 prior term
    for k in range(31):
        m.integrate(pts, POSE, 0.1 * k, cfg)
        info += 1.0 / 0.04
        assert m.layer("variance")[5, 5] == pytest.approx(1.0 / info, rel=1e-12)
    assert m.layer("elevation")[5, 5] == pytest.approx(5.0)


# ---- single point over an invalid map (reference test_integration.cpp:190-214) -----
def test_single_point_creates_one_cell(impl, tmp_path):
    cfg = _cfg(impl, tmp_path, QUIET)
    m = pk.ReliefMap.create(impl, 0.04, 100, 100)
    st = m.integrate(np.array([[1.0, 0.0, -1.0]]), pk.pose34(t=(0.0, 0.0, 1.0)), 0.0, cfg)
    assert st.points_fused == 1 and st.cells_updated == 1
    valid = m.layer("valid")
    assert valid.sum() == 1
    r, c = np.argwhere(valid == 1)[0]
    assert (r, c) == (50, 75)
    assert abs(m.layer("elevation")[r, c]) < 1e-9
    assert m.layer("upper_bound")[r, c] == m.layer("elevation")[r, c]


# ---- DDA through the upper bound of an empty map (reference test_raycast.cpp:46-103) -
def test_single_ray_bounds_equal_reference_traversal(impl, reference, tmp_path):
    cfg = _cfg(impl, tmp_path, "drift.enabled = false\ncleanup.enabled = false\noverlap.enabled = false\n"
               "exclusion.enabled = false\n")
    rng = np.random.default_rng(4)
    res, W, H = 0.04, 125, 125
    I32 = ctypes.POINTER(ctypes.c_int32)
    DP = ctypes.POINTER(ctypes.c_double)
    for trial in range(24):
        o = np.array([rng.uniform(-2.4, 2.4), rng.uniform(-2.4, 2.4), rng.uniform(0.3, 2.0)])
        if trial % 4 == 0:
            o[:2] = np.round(o[:2] / res) * res  # origin on cell corners: tie handling
        e = np.array([rng.uniform(-3.2, 3.2), rng.uniform(-3.2, 3.2), rng.uniform(-0.5, 0.2)])
        if trial % 6 == 1:
            e[1] = o[1]  # axis-parallel ray
        m = pk.ReliefMap.create(impl, res, W, H, o[0], o[1])
        m.integrate((e - o)[None, :], pk.pose34(t=tuple(o)), 0.0, cfg)
        rows = np.zeros(1024, np.int32)
        cols = np.zeros(1024, np.int32)
        hts = np.zeros(1024)
        n = reference.ref_traverse_cells(o.ctypes.data_as(DP), e.ctypes.data_as(DP), res, W, H, o[0], o[1],
                                         rows.ctypes.data_as(I32), cols.ctypes.data_as(I32),
                                         hts.ctypes.data_as(DP), 1024)
        ub = m.layer("upper_bound")
        valid = m.layer("valid")
        want = np.full((H, W), np.nan)
        for k in range(n):
            want[rows[k], cols[k]] = hts[k]
        want[valid == 1] = m.layer("elevation")[valid == 1]
        assert bits_equal(ub, want).all(), f"trial {trial}: {np.argwhere(~bits_equal(ub, want))[:4]}"


# ---- recenter (reference test_grid.cpp:77-137) -------------------------------------
def test_recenter_survival_and_exposure(impl, tmp_path):
    if not _supports_load(impl):
        pytest.skip("restatement has no snapshot loader")
    res, W, H = 0.1, 12, 9
    layers = snap.fresh(H, W)
    rng = np.random.default_rng(2)
    for r in range(H):
        for c in range(W):
            if (r + c) % 3:
                snap.set_cell(layers, r, c, rng.normal(), 0.01 + rng.random(), 0.25, (0.1, -0.2, 0.97), 0.5)
    m = _map_from(impl, tmp_path, layers, res)
    before = m.layers()
    cfg = _cfg(impl, tmp_path, QUIET + "update.sigma_t2 = 0\n")
    m.integrate(np.zeros((0, 3)), pk.pose34(t=(0.04, -0.09, 1.0)), 0.0, cfg)  # sub-cell: no shift
    assert m.center() == (0.0, 0.0)
    m.integrate(np.zeros((0, 3)), pk.pose34(t=(0.31, -0.2, 1.0)), 0.0, cfg)   # +3 cols, -2 rows
    cx, cy = m.center()
    assert (round(cx / res), round(cy / res)) == (3, -2)
    after = m.layer("elevation")
    assert bits_equal(after[2:, :W - 3], before["elevation"][:H - 2, 3:]).all()
    assert np.isnan(after[:2, :]).all() and np.isnan(after[:, W - 3:]).all()
    m.integrate(np.zeros((0, 3)), pk.pose34(t=(5.0, 5.0, 1.0)), 0.0, cfg)     # beyond the extent
    assert (m.layer("valid") == 0).all()


# ---- time variance (reference test_grid.cpp:139-173) ------------------------------
def test_time_variance_growth_cap_and_skip(impl, tmp_path):
    if not _supports_load(impl):
        pytest.skip("restatement has no snapshot loader")
    res, W, H = 0.1, 10, 10
    layers = snap.fresh(H, W)
    snap.set_cell(layers, 1, 1, 0.0, 0.5)
    snap.set_cell(layers, 1, 2, 0.0, 99.995)
    snap.set_cell(layers, 5, 5, 0.0, 0.5)
    m = _map_from(impl, tmp_path, layers, res)
    cfg = _cfg(impl, tmp_path, QUIET + "update.sigma_t2 = 0.01\nupdate.nominal_period = 0.1\n"
               "update.mahalanobis_threshold = 1e9\n")
    m.integrate(np.zeros((0, 3)), POSE, 0.0, cfg)          # first scan: dt = 0
    m.integrate(_point_above((5, 5), res, W, H, 0.0, 3.0), POSE, 0.1, cfg)  # dt = 0.1
    v = m.layer("variance")
    assert v[1, 1] == pytest.approx(0.51, rel=1e-12)
    assert v[1, 2] == 100.0
    assert v[5, 5] < 0.5  # touched this scan: fused, no time growth
    assert np.isnan(v[0, 0])


# ---- normals and traversability (reference test_analysis.cpp:46-144) --------------
def test_normals_flat_ramp_isolated(impl, tmp_path):
    if not _supports_load(impl):
        pytest.skip("restatement has no snapshot loader")
    res, W, H = 0.1, 16, 12
    layers = snap.fresh(H, W)
    for r in range(H):
        for c in range(0, 6):
            snap.set_cell(layers, r, c, 0.0, 0.01)               # flat
        for c in range(8, 14):
            snap.set_cell(layers, r, c, 0.1 * c, 0.01)           # 45 degree ramp along x
    snap.set_cell(layers, 0, 15, 0.3, 0.01)                      # isolated (no x neighbour)
    m = _map_from(impl, tmp_path, layers, res)
    m.integrate(np.zeros((0, 3)), POSE, 0.0, _cfg(impl, tmp_path, QUIET))
    nx, ny, nz, t = (m.layer(n) for n in ("normal_x", "normal_y", "normal_z", "traversability"))
    assert np.allclose(nz[3:9, 1:5], 1.0) and np.allclose(nx[3:9, 1:5], 0.0)
    assert np.allclose(t[3:9, 2:4], 1.0)
    assert np.allclose(nx[3:9, 9:13], -1 / math.sqrt(2), atol=1e-6)
    assert np.allclose(nz[3:9, 9:13], 1 / math.sqrt(2), atol=1e-6)
    assert nx[0, 15] == 0.0 and ny[0, 15] == 0.0 and nz[0, 15] == 0.0 and t[0, 15] == 0.0


# ---- exclusion ramp boundary (reference test_sensing.cpp:84-143) ------------------
def test_exclusion_boundary(impl, tmp_path):
    cfg = _cfg(impl, tmp_path, "drift.enabled = false\ncleanup.enabled = false\n"
               "cleanup.upper_bound_enabled = false\noverlap.enabled = false\n"
               "exclusion.b = 0.5\nexclusion.c = 0.2\nexclusion.d_max = 1.0\n")
    tan_a = math.tan(0.785398163397448)
    pts = []
    for r in (0.1, 0.3, 0.55, 0.75, 2.0):
        ramp = 0.5 + max(0.0, r - 0.2) * tan_a
        lim = min(1.0, ramp)
        pts += [[r, 0.0, lim], [r, 0.0, np.nextafter(lim, 10.0)], [r, 0.0, lim - 0.01]]
    m = pk.ReliefMap.create(impl, 0.04, 100, 100)
    st = m.integrate(np.array(pts), pk.pose34(t=(0.0, 0.0, 0.0)), 0.0, cfg)
    assert st.points_excluded == 5


# ---- drift vote and clamp (reference test_integration.cpp:313-470) ----------------
@pytest.mark.parametrize("err,applied", [(0.05, 0.05), (1.0, 0.1), (-0.3, -0.1)])
def test_drift_offset_and_clamp(impl, tmp_path, err, applied):
    if not _supports_load(impl):
        pytest.skip("restatement has no snapshot loader")
    res, W, H = 0.1, 10, 10
    layers = snap.fresh(H, W)
    for r in range(2, 8):
        for c in range(2, 8):
            snap.set_cell(layers, r, c, 0.2, 0.01, 0.0, (0.0, 0.0, 1.0), 0.9)
    m = _map_from(impl, tmp_path, layers, res)
    cfg = _cfg(impl, tmp_path, "cleanup.enabled = false\ncleanup.upper_bound_enabled = false\n"
               "overlap.enabled = false\nexclusion.enabled = false\nupdate.mahalanobis_threshold = 1e9\n")
    pts = np.concatenate([_point_above((r, c), res, W, H, 0.2 + err, 3.0)
                          for r in range(2, 8) for c in range(2, 8)])
    st = m.integrate(pts, POSE, 0.0, cfg)
    assert st.drift_offset_applied == pytest.approx(applied, abs=1e-12)
