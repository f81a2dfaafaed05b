"""The library's scene simulator (input generator for tests and bench.py) renders clouds
bit-identical to the reference's renderScan (reference sim.cpp:241-262) for every workload."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl

from conftest import ref_render


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "headline"])
def test_workload_clouds_bit_identical(product, reference, tmp_path, name):
    w = wl.ALL[name]()
    p = tmp_path / "w.config"
    p.write_text(w.config_text)
    for f in (0, 3):
        for c in w.calls(f)[:2]:
            a = pk.sim_render(product, p, c.pose, c.time, c.seed, c.scan_index)
            b = ref_render(reference, p, c.pose, c.time, c.seed, c.scan_index)
            assert a.shape == b.shape
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_point_counts_match_survey(product, tmp_path):
    expect = {"C1": 19477, "C3": 262144, "headline": 1000064}
    for name, n in expect.items():
        w = wl.ALL[name]()
        p = tmp_path / f"{name}.config"
        p.write_text(w.config_text)
        c = w.calls(0)[0]
        assert len(pk.sim_render(product, p, c.pose, c.time, c.seed, c.scan_index)) == n


def test_moving_box_and_trajectory_scene(product, reference, tmp_path):
    text = ("sensor.pattern = grid\nsensor.cols = 64\nsensor.rows = 48\nnoise.alpha_d = 0.005\n"
            "scene.ground = 0\nscene.moving_box = 1.2 0 0.3 0.8 0.8 0.6 0.1 0 0 -1 2.95\n"
            "scene.ramp = -2 -1 -1 1 0 0.3 -x\nscene.wall = 0 2 3 2 1.0 0.1\n"
            "scene.slab_overhang = -1 -3 1 -2 1.5\nscene.floor2 = 2 -3 4 -1 0.8 2.5 -2.5 3.5 -1.5\n")
    p = tmp_path / "s.config"
    p.write_text(text)
    pose = wl.pose34(wl.rot_z(0.7) @ wl.rot_y(0.4), (0.1, -0.2, 1.1))
    for t in (0.0, 1.5, 3.0):
        a = pk.sim_render(product, p, pose, t, 9, 3)
        b = ref_render(reference, p, pose, t, 9, 3)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
