"""Streaming integrate (relief_gpu_map_integrate_async / relief_gpu_map_wait): two frames in
flight, the PCIe copy of frame k+1 overlapping frame k's kernels. Every frame's stats and the final
map must equal the synchronous relief_map_integrate sequence bit for bit (the single-call path is
the one parity-tested against the reference)."""
from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl

from conftest import assert_layers_match, assert_stats_match, ref_render

pytestmark = pytest.mark.gpu


def _run_both(gpu, cfg_path, res, W, H, frames):
    cfg = pk.Config.load(gpu, cfg_path)
    sync = pk.ReliefMap.create(gpu, res, W, H)
    stream = pk.ReliefMap.create(gpu, res, W, H)
    want = [sync.integrate(x, p, t, cfg) for x, p, t in frames]
    pinned = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy() for x, _, _ in frames]
    got = []
    for k, (x, (_, p, t)) in enumerate(zip(pinned, frames)):
        stream.integrate_async(x, p, t, cfg)
        if gpu.relief_gpu_map_in_flight(stream.handle) == 3:
            got.append(stream.wait())
    while gpu.relief_gpu_map_in_flight(stream.handle):
        got.append(stream.wait())
    assert len(got) == len(want)
    for k, (g, w) in enumerate(zip(got, want)):
        assert_stats_match(g, w, context=f"frame {k}")
    assert_layers_match(stream.layers(), sync.layers(), context="final map")
    return got


def test_stream_lidar_recenter_matches_sync(gpu, reference, tmp_path):
    text = wl._map(0.04, 300, 300) + "noise.alpha_d = 0.0002\n" + wl.lidar(512, rings=64) + wl.SCENE_S0
    cfg = tmp_path / "s.config"
    cfg.write_text(text)
    frames = []
    for f in range(7):
        pose = wl.pose34(np.eye(3), (0.04 * f + 0.013, -0.021 * f, 1.0))
        frames.append((ref_render(reference, cfg, pose, 0.1 * f, 3, f), pose, 0.15 * f))
    got = _run_both(gpu, cfg, 0.04, 300, 300, frames)
    assert sum(s.drift_offset_applied != 0.0 for s in got) >= 1  # drift on, device-side offset


def test_stream_removals_and_growing_frames(gpu, reference, tmp_path):
    text = (wl._map(0.04, 120, 120) +
            "noise.alpha_d = 0.005\nupdate.sigma_outlier2 = 0.0001\ndrift.enabled = false\n"
            "overlap.enabled = false\nexclusion.enabled = false\ncleanup.t_free = 1.0\n"
            "sensor.pattern = grid\nsensor.h_fov_deg = 70\nsensor.v_fov_deg = 60\n"
            "sensor.cols = 160\nsensor.rows = 140\nsensor.max_range = 10\n"
            "scene.ground = 0.0\nscene.moving_box = 1.2 0.0 0.3 0.8 0.8 0.6 0 0 0 -1 2.95\n")
    cfg = tmp_path / "m.config"
    cfg.write_text(text)
    pose = wl.pose34(wl.rot_y(math.radians(35.0)), (0.0, 0.0, 1.2))
    frames = []
    for s in range(40):
        x = ref_render(reference, cfg, pose, s * 0.1, 4, s)
        if s in (5, 6, 20):  # point-scratch growth while a frame is in flight
            x = np.concatenate([x] * (3 if s == 20 else 2))
        if s == 12:
            x = x[:0]
        frames.append((x, pose, s * 0.1))
    got = _run_both(gpu, cfg, 0.04, 120, 120, frames)
    assert sum(s.cells_removed_by_cleanup for s in got) > 50


def test_stream_usage_errors(gpu, tmp_path):
    m = pk.ReliefMap.create(gpu, 0.04, 50, 50)
    pose = wl.pose34(np.eye(3), (0.0, 0.0, 1.0))
    x = np.array([[0.1, 0.1, -1.0]] * 10)
    with pytest.raises(pk.ReliefError) as e:
        m.wait()
    assert e.value.status == 1
    for k in range(3):
        m.integrate_async(x, pose, 0.1 * k)
    with pytest.raises(pk.ReliefError) as e:
        m.integrate_async(x, pose, 0.3)
    assert e.value.status == 1
    with pytest.raises(pk.ReliefError) as e:
        m.integrate(x, pose, 0.3)
    assert e.value.status == 1
    assert m.wait().points_fused > 0 and m.wait().points_in == 10 and m.wait().points_in == 10
    m.integrate(x, pose, 0.4)  # allowed again
