"""Parity at BASELINE.json's full sizes: the reference
(oracle/_ref) and the B200 library integrate the same rendered frames through the same C ABI.

C4 is the 1,000,064-point frame on the 1000x1000 map that `bench.py` measures. With drift
compensation off every layer is compared bit for bit; with the defaults (drift on) heights are
compared within 1e-9 relative, the drift mean being a fixed-order parallel sum.
Stamps 1.2 s apart make every cell observed in an earlier frame stale, so the removal-candidate
path of the ray pass runs at full size too.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl

from conftest import assert_layers_match, assert_stats_match, ref_render

pytestmark = pytest.mark.gpu


def _run(product, reference, tmp_path, w, frames, extra="", stamp_step=None, drift_tol=0.0,
         height_tol=0.0):
    cfg_path = tmp_path / f"{w.name}.config"
    cfg_path.write_text(w.config_text + extra)
    libs = (product, reference)
    cfgs = [pk.Config.load(lib, cfg_path) for lib in libs]
    maps = [pk.ReliefMap.create(lib, w.resolution, w.width, w.height) for lib in libs]
    totals = {}
    for f in range(frames):
        for call in w.calls(f):
            xyz = ref_render(reference, cfg_path, call.pose, call.time, call.seed, call.scan_index)
            stamp = call.stamp if stamp_step is None else stamp_step * f
            got = maps[0].integrate(xyz, call.pose, stamp, cfgs[0])
            want = maps[1].integrate(xyz, call.pose, stamp, cfgs[1])
            ctx = f"{w.name} frame {f} call {call.scan_index}"
            assert_stats_match(got, want, drift_tol=drift_tol, context=ctx)
            for k in ("points_fused", "cells_removed_by_cleanup"):
                totals[k] = totals.get(k, 0) + getattr(got, k)
        assert_layers_match(maps[0].layers(), maps[1].layers(), height_tol=height_tol,
                            context=f"{w.name} after frame {f}")
    return totals


def test_c4_full_size_bit_exact(gpu, reference, tmp_path):
    t = _run(gpu, reference, tmp_path, wl.c4(), 3, extra="drift.enabled = false\n", stamp_step=1.2)
    assert t["points_fused"] > 1_000_000


def test_c4_full_size_defaults(gpu, reference, tmp_path):
    _run(gpu, reference, tmp_path, wl.c4(), 2, drift_tol=1e-12, height_tol=1e-9)


def test_c3_recenter_full_size(gpu, reference, tmp_path):
    _run(gpu, reference, tmp_path, wl.c3(), 4, drift_tol=1e-12, height_tol=1e-9)


def test_c2_four_cameras_per_frame(gpu, reference, tmp_path):
    _run(gpu, reference, tmp_path, wl.c2(), 2, drift_tol=1e-12, height_tol=1e-9)


def test_c2_four_cameras_bit_exact_with_removals(gpu, reference, tmp_path):
    t = _run(gpu, reference, tmp_path, wl.c2(), 3, extra="drift.enabled = false\n", stamp_step=1.2)
    assert t["points_fused"] > 0


def test_headline_full_size_bit_exact(gpu, reference, tmp_path):
    """The north star's own config: 1,000,064 points into 500x500 (rays clipped at the map border
    at full density), drift off, stamps 1.2 s apart so removal candidates are live."""
    t = _run(gpu, reference, tmp_path, wl.headline(), 3, extra="drift.enabled = false\n", stamp_step=1.2)
    assert t["points_fused"] > 1_000_000


def test_headline_full_size_defaults(gpu, reference, tmp_path):
    _run(gpu, reference, tmp_path, wl.headline(), 2, drift_tol=1e-12, height_tol=1e-9)


def test_overlap_clearance_fires_full_size(gpu, reference, tmp_path):
    """Overlap clearance (analysis.cpp:296-317) must actually clear cells: C3 frames with the
    sensor at 1 m build the map, then the robot rises to 3.2 m (a second floor / elevator), so
    valid ground cells within the (2 m) radius sit more than 1.5 m below it and are invalidated."""
    w = wl.c3()
    cfg_path = tmp_path / "ov.config"
    cfg_path.write_text(w.config_text + "drift.enabled = false\noverlap.radius = 2.0\n")
    libs = (gpu, reference)
    cfgs = [pk.Config.load(lib, cfg_path) for lib in libs]
    maps = [pk.ReliefMap.create(lib, w.resolution, w.width, w.height) for lib in libs]
    cleared = 0
    for f in range(4):
        z = 1.0 if f < 3 else 3.2
        pose = wl.pose34(np.eye(3), (0.0, 0.0, z))
        xyz = ref_render(reference, cfg_path, pose, 0.1 * f, 3, f)
        got = maps[0].integrate(xyz, pose, 0.1 * f, cfgs[0])
        want = maps[1].integrate(xyz, pose, 0.1 * f, cfgs[1])
        assert_stats_match(got, want, context=f"frame {f}")
        assert_layers_match(maps[0].layers(), maps[1].layers(), context=f"frame {f}")
        cleared += got.cells_cleared_by_overlap
    assert cleared > 100, cleared


# Steady state at full size: the bench's C4 sequence (stamps 0.1 s apart) for 40 frames, where
# the ray pass's jumps clear most of the DDA cells; every frame's counters and every 8th frame's
# layers against the reference (~30 s per config: the reference's frames take ~0.7 s each).
# RELIEF_FULL_STEADY=0 skips them.
@pytest.mark.skipif(os.environ.get("RELIEF_FULL_STEADY") == "0", reason="RELIEF_FULL_STEADY=0")
@pytest.mark.parametrize("name", ["C4", "headline"])
def test_full_size_steady_state(gpu, reference, tmp_path, name):
    w = wl.ALL[name]()
    cfg_path = tmp_path / f"{w.name}.config"
    cfg_path.write_text(w.config_text + "drift.enabled = false\n")
    libs = (gpu, reference)
    cfgs = [pk.Config.load(lib, cfg_path) for lib in libs]
    maps = [pk.ReliefMap.create(lib, w.resolution, w.width, w.height) for lib in libs]
    clouds = [[(ref_render(reference, cfg_path, c.pose, c.time, c.seed, c.scan_index), c) for c in w.calls(f)]
              for f in range(8)]
    for s in range(40):
        for xyz, c in clouds[s % 8]:
            got = maps[0].integrate(xyz, c.pose, 0.1 * s, cfgs[0])
            want = maps[1].integrate(xyz, c.pose, 0.1 * s, cfgs[1])
            assert_stats_match(got, want, context=f"{name} step {s}")
        if s % 8 == 7:
            assert_layers_match(maps[0].layers(), maps[1].layers(), context=f"{name} after step {s}")
