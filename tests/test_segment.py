"""Plane segmentation runner (reference runner.cpp:349-362, postprocess.cpp:
199-545). Host code in both libraries, so these run on CPU: the region file written by the
product must equal the reference's byte for byte, on snapshots the reference itself produced and
on synthetic ones (with and without stored normals, several parameter sets)."""
from __future__ import annotations

import numpy as np
import pytest

import snapshots as snap

SIM = """map.resolution = 0.04
map.width = {W}
map.height = {H}
noise.alpha_d = 0.0002
update.sigma_outlier2 = 0.00001
update.wall_count_threshold = 40
sensor.ring_elevations_deg = -80 -72 -64 -57 -51 -45 -40 -36 -32 -29 -26 -24
sensor.azimuth_steps = 360
sensor.max_range = 10
sensor.rate = 10
scene.ground = 0.0
scene.box = 1.5 0.5 0.25 0.6 0.6 0.5
scene.stairs = -2.0 -0.6 0 0.18 0.28 4 1.2 -x
traj.waypoint = 0 0 0 1
traj.waypoint = 8 1.0 0.5 1
run.scans = {scans}
run.publish_every = 100
run.seed = 1
run.mode = det
"""

PARAMS = {
    "default": "",
    "tight": "segmentation.normal_angle_max_deg = 8\nsegmentation.dist_max = 0.015\n"
             "segmentation.min_region_cells = 10\n",
    "simplify": "segmentation.simplify_tol = 0.05\nsegmentation.min_region_cells = 20\n",
}


def _segment(lib, snapshot, cfg, out):
    import ctypes
    n = ctypes.c_size_t(0)
    st = lib.relief_run_segment(str(snapshot).encode(), str(cfg).encode() if cfg else None,
                                str(out).encode(), ctypes.byref(n))
    return st, n.value, (out.read_text() if st == 0 else lib.relief_last_error().decode())


def _compare(product, reference, snapshot, tmp_path, params=""):
    cfg = None
    if params:
        cfg = tmp_path / "seg.config"
        cfg.write_text(params)
    got = _segment(product, snapshot, cfg, tmp_path / "got.txt")
    want = _segment(reference, snapshot, cfg, tmp_path / "want.txt")
    assert got[0] == want[0], (got[0], want[0], got[2][:200], want[2][:200])
    assert got[1] == want[1]
    assert got[2] == want[2]
    return got


@pytest.fixture(scope="module")
def simulated(reference, tmp_path_factory):
    """final.relief of a short reference simulation (ground, box, stairs)."""
    d = tmp_path_factory.mktemp("segsim")
    cfg = d / "sim.config"
    cfg.write_text(SIM.format(W=200, H=200, scans=6))
    st = reference.relief_run_simulate(str(cfg).encode(), str(d / "out").encode(), 0, 0, None)
    assert st == 0, reference.relief_last_error()
    return d / "out" / "final.relief"


@pytest.mark.parametrize("which", sorted(PARAMS))
def test_segment_simulated_snapshot_matches_reference(product, reference, simulated, tmp_path, which):
    st, n, text = _compare(product, reference, simulated, tmp_path, PARAMS[which])
    assert st == 0
    assert n >= 1 and text.startswith("region: 0"), which


def _synthetic(seed, with_normals):
    rng = np.random.default_rng(seed)
    H, W = 48, 56
    L = snap.fresh(H, W)
    yy, xx = np.mgrid[0:H, 0:W]
    h = np.where(xx < 20, 0.0, np.where(yy < 24, 0.3 + 0.01 * (xx - 20), 0.6))  # floor, ramp, shelf
    h = h + 1e-4 * rng.standard_normal((H, W))
    holes = rng.random((H, W)) < 0.05
    for r in range(H):
        for c in range(W):
            if holes[r, c]:
                continue
            n = (0.0, 0.0, 0.0)
            if with_normals:
                n = (-0.01 if (xx[r, c] >= 20 and yy[r, c] < 24) else 0.0, 0.0, 1.0)
                ln = float(np.sqrt(n[0] ** 2 + 1.0))
                n = (n[0] / ln, 0.0, 1.0 / ln)
            snap.set_cell(L, r, c, float(h[r, c]), 0.001, normal=n)
    return snap.text(L, 0.04)


@pytest.mark.parametrize("with_normals", [True, False])
@pytest.mark.parametrize("seed", [1, 2])
def test_segment_synthetic_matches_reference(product, reference, tmp_path, seed, with_normals):
    path = tmp_path / "syn.relief"
    path.write_text(_synthetic(seed, with_normals))
    for which in sorted(PARAMS):
        _compare(product, reference, path, tmp_path, PARAMS[which])


def test_segment_errors_match_reference(product, reference, tmp_path, simulated):
    bad = tmp_path / "bad.config"
    bad.write_text("segmentation.dist_max = -1\n")
    for snapshot, cfg in [(tmp_path / "absent.relief", None), (simulated, bad)]:
        got = _segment(product, snapshot, cfg, tmp_path / "g.txt")
        want = _segment(reference, snapshot, cfg, tmp_path / "w.txt")
        assert got[0] == want[0] != 0, (got, want)
