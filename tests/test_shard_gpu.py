"""Exact point-batch sharding of one frame on one GPU.

G replicas run the relief_gpu_shard_* phases in lockstep in one process (multigpu.
integrate_sharded_lockstep); the exchanges between phases are done with torch ops on the
replicas' device buffers. After every frame each replica must equal the single-call
relief_map_integrate of the whole frame -- bit for bit (drift off), and the reference on the same
frames through the same comparison (transitively: the single-call path is the parity-tested one).
No rank ever waits on another rank's kernels: the phases run one after the other.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import multigpu as mg
from paper_2204_12876_b200 import workloads as wl

from conftest import assert_layers_match, assert_stats_match, ref_render

pytestmark = pytest.mark.gpu


class Sharded:
    def __init__(self, lib, tmp_path, text, res, W, H, G):
        self.cfg_path = tmp_path / "shard.config"
        self.cfg_path.write_text(text)
        self.cfg = pk.Config.load(lib, self.cfg_path)
        self.single = pk.ReliefMap.create(lib, res, W, H)
        self.reps = [pk.ReliefMap.create(lib, res, W, H) for _ in range(G)]
        self.apis = [mg.CudaShardAPI(lib, m, self.cfg) for m in self.reps]

    def frame(self, xyz, pose, stamp, height_tol=0.0, drift_tol=0.0, context=""):
        want = self.single.integrate(xyz, pose, stamp, self.cfg)
        got = mg.integrate_sharded_lockstep(self.apis, xyz, pose, stamp)
        ref_layers = self.single.layers()
        for g, (st, m) in enumerate(zip(got, self.reps)):
            assert_stats_match(st, want, drift_tol=drift_tol, context=f"{context} rank {g}")
            assert m.center() == self.single.center()
            assert_layers_match(m.layers(), ref_layers, height_tol=height_tol, context=f"{context} rank {g}")
        return want


@pytest.mark.parametrize("G", [2, 3])
def test_sharded_lidar_recenter_every_frame_bit_exact(gpu, reference, tmp_path, G):
    text = wl._map(0.04, 300, 300) + "noise.alpha_d = 0.0002\n" + wl.lidar(512, rings=64) + wl.SCENE_S0 + \
        "drift.enabled = false\n"
    sh = Sharded(gpu, tmp_path, text, 0.04, 300, 300, G)
    for f in range(6):
        pose = wl.pose34(np.eye(3), (0.04 * f + 0.013, -0.021 * f, 1.0))
        xyz = ref_render(reference, sh.cfg_path, pose, 0.1 * f, 3, f)
        st = sh.frame(xyz, pose, 0.15 * f, context=f"frame {f}")
        assert st.points_fused > 0


def test_sharded_moving_box_removals_bit_exact(gpu, reference, tmp_path):
    """Removals fire: k* (global ray ids) and the second upper-bound exchange are exercised."""
    text = (wl._map(0.04, 120, 120) +
            "noise.alpha_d = 0.005\nupdate.sigma_outlier2 = 0.0001\ndrift.enabled = false\n"
            "overlap.enabled = false\nexclusion.enabled = false\ncleanup.t_free = 1.0\n"
            "sensor.pattern = grid\nsensor.h_fov_deg = 70\nsensor.v_fov_deg = 60\n"
            "sensor.cols = 160\nsensor.rows = 140\nsensor.max_range = 10\n"
            "scene.ground = 0.0\nscene.moving_box = 1.2 0.0 0.3 0.8 0.8 0.6 0 0 0 -1 2.95\n")
    sh = Sharded(gpu, tmp_path, text, 0.04, 120, 120, 4)
    pose = wl.pose34(wl.rot_y(math.radians(35.0)), (0.0, 0.0, 1.2))
    removed = 0
    for s in range(45):
        xyz = ref_render(reference, sh.cfg_path, pose, s * 0.1, 4, s)
        removed += sh.frame(xyz, pose, s * 0.1, context=f"scan {s}").cells_removed_by_cleanup
    assert removed > 50, removed


def test_sharded_drift_and_uneven_batches(gpu, reference, tmp_path):
    """Drift on: the offset is the ranks' partial votes summed in rank order (tolerance);
    5 ranks over a frame whose size is not a multiple of 5."""
    text = wl._map(0.04, 250, 250) + "noise.alpha_d = 0.0002\n" + wl.lidar(721, rings=48) + wl.SCENE_S0
    sh = Sharded(gpu, tmp_path, text, 0.04, 250, 250, 5)
    applied = 0
    for f in range(6):
        pose = wl.pose34(np.eye(3), (0.02 * f, 0.0, 1.0 + 0.01 * f))
        xyz = ref_render(reference, sh.cfg_path, pose, 0.1 * f, 7, f)
        st = sh.frame(xyz, pose, 0.1 * f, height_tol=1e-9, drift_tol=1e-12, context=f"frame {f}")
        applied += st.drift_offset_applied != 0.0
    assert applied >= 2


def test_sharded_empty_and_tiny_batches(gpu, tmp_path):
    """More ranks than points, and an empty frame: every phase still runs on every rank."""
    text = wl._map(0.04, 60, 60) + "drift.enabled = false\n"
    sh = Sharded(gpu, tmp_path, text, 0.04, 60, 60, 4)
    rng = np.random.default_rng(3)
    pose = wl.pose34(np.eye(3), (0.0, 0.0, 1.0))
    for f, n in enumerate([3, 0, 7, 1]):
        xyz = np.stack([rng.normal(0, 0.5, n), rng.normal(0, 0.5, n), rng.normal(-1, 0.1, n)], axis=1)
        sh.frame(xyz, pose, 0.2 * f, context=f"n={n}")
