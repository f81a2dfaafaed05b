"""Pins the C restatement oracle (oracle/relief_oracle.c) against the reference compiled in
place (oracle/_ref): identical stats and bit-identical layers on the same scans.
CPU only (both oracles are host code)."""
from __future__ import annotations

import subprocess

import numpy as np
import pytest

import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl

from conftest import ROOT, RESTATE_LIB, assert_layers_match, assert_stats_match, ref_render


@pytest.fixture(scope="module")
def restate():
    subprocess.run(["make", "-C", str(ROOT / "oracle"), "restate"], check=True, capture_output=True)
    return pk.load_library(RESTATE_LIB, gpu_api=False)


def _run(libs, cfg_text, tmp_path, res, W, H, frames):
    p = tmp_path / "r.config"
    p.write_text(cfg_text)
    cfgs = [pk.Config.load(l, p) for l in libs]
    maps = [pk.ReliefMap.create(l, res, W, H) for l in libs]
    return p, cfgs, maps


@pytest.mark.parametrize("drift", [False, True])
def test_restatement_matches_reference_lidar(restate, reference, tmp_path, drift):
    text = wl._map(0.04, 160, 160) + "noise.alpha_d = 0.0002\n" + wl.lidar(360, rings=32) + wl.SCENE_S0
    if not drift:
        text += "drift.enabled = false\n"
    p, cfgs, maps = _run((restate, reference), text, tmp_path, 0.04, 160, 160, 6)
    for f in range(6):
        pose = wl.pose34(np.eye(3), (0.05 * f, 0.02 * f, 1.0))
        xyz = ref_render(reference, p, pose, 0.1 * f, 9, f)
        a = maps[0].integrate(xyz, pose, 0.25 * f, cfgs[0])
        b = maps[1].integrate(xyz, pose, 0.25 * f, cfgs[1])
        assert_stats_match(a, b, context=f"frame {f}")
        assert_layers_match(maps[0].layers(), maps[1].layers(), tol_trav=0.0, context=f"frame {f}")


def test_restatement_matches_reference_moving_box(restate, reference, tmp_path):
    import math
    text = (wl._map(0.04, 80, 80) +
            "noise.alpha_d = 0.005\nupdate.sigma_outlier2 = 0.0001\ndrift.enabled = false\n"
            "overlap.enabled = false\nexclusion.enabled = false\n"
            "sensor.pattern = grid\nsensor.h_fov_deg = 70\nsensor.v_fov_deg = 60\n"
            "sensor.cols = 80\nsensor.rows = 70\nsensor.max_range = 10\n"
            "scene.ground = 0.0\nscene.moving_box = 1.2 0.0 0.3 0.8 0.8 0.6 0 0 0 -1 2.95\n")
    p, cfgs, maps = _run((restate, reference), text, tmp_path, 0.04, 80, 80, 0)
    pose = wl.pose34(wl.rot_y(math.radians(35.0)), (0.0, 0.0, 1.2))
    removed = 0
    for s in range(45):
        xyz = ref_render(reference, p, pose, 0.1 * s, 4, s)
        a = maps[0].integrate(xyz, pose, 0.1 * s, cfgs[0])
        b = maps[1].integrate(xyz, pose, 0.1 * s, cfgs[1])
        assert_stats_match(a, b, context=f"scan {s}")
        removed += a.cells_removed_by_cleanup
    assert removed > 0
    assert_layers_match(maps[0].layers(), maps[1].layers(), tol_trav=0.0)


def test_restatement_random_edge_cases(restate, reference, tmp_path):
    text = "exclusion.b = 0.2\nexclusion.c = 0.1\nupdate.max_range = 3.0\nupdate.wall_count_threshold = 2\n"
    p, cfgs, maps = _run((restate, reference), text, tmp_path, 0.05, 70, 50, 0)
    rng = np.random.default_rng(1)
    for s in range(5):
        xyz = np.column_stack([rng.normal(0, 1.5, 4000), rng.normal(0, 1.5, 4000), rng.normal(-0.5, 0.6, 4000)])
        xyz[::53] = np.nan
        pose = wl.pose34(wl.rot_z(0.3 * s), (0.07 * s, 0.0, 0.6))
        a = maps[0].integrate(xyz, pose, 0.4 * s, cfgs[0])
        b = maps[1].integrate(xyz, pose, 0.4 * s, cfgs[1])
        assert_stats_match(a, b, context=f"scan {s}")
        assert_layers_match(maps[0].layers(), maps[1].layers(), tol_trav=0.0, context=f"scan {s}")
