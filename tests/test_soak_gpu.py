"""Randomised parity soak: many small scenarios, each driven through both libraries (the B200
build and the reference compiled in place) with identical maps, configs, clouds, poses and
stamps. Each scenario draws its own map geometry, pipeline switches and point mix, including
the geometric corner cases of the ray pass: points exactly on cell boundaries (identity
rotation, cell-aligned sensor), points straight below the sensor (vertical rays), duplicated
points, far points whose rays are clipped at the map border, non-finite coordinates, stamp gaps
that make observed cells stale (removals), and recentering by several cells.

Bar as in test_parity_gpu.py: counters exact, layers bit-exact with drift compensation off,
heights within 1e-9 relative with it on (fixed-order vote sum).
"""
from __future__ import annotations

import math
import os

import numpy as np
import pytest

import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl

from conftest import assert_layers_match, assert_stats_match

pytestmark = pytest.mark.gpu

# RELIEF_SOAK_SEEDS=N widens the sweep (a 2,000-scenario run was clean).
SEEDS = list(range(int(os.environ.get("RELIEF_SOAK_SEEDS", "48"))))


def _config(rng) -> tuple[str, bool]:
    drift = bool(rng.random() < 0.3)
    lines = [
        f"drift.enabled = {'true' if drift else 'false'}",
        f"cleanup.enabled = {'true' if rng.random() < 0.8 else 'false'}",
        f"cleanup.upper_bound_enabled = {'true' if rng.random() < 0.8 else 'false'}",
        f"cleanup.t_free = {rng.choice([0.3, 1.0, 5.0])}",
        f"overlap.enabled = {'true' if rng.random() < 0.5 else 'false'}",
        f"exclusion.enabled = {'true' if rng.random() < 0.5 else 'false'}",
        f"noise.alpha_d = {rng.choice([0.0002, 0.002, 0.02])}",
        f"update.sigma_outlier2 = {rng.choice([0.0001, 0.01, 0.05])}",
        f"update.wall_count_threshold = {int(rng.choice([2, 5, 40]))}",
        f"update.max_range = {rng.choice([4.0, 10.0, 30.0])}",
    ]
    return "\n".join(lines) + "\n", drift


def _cloud(rng, res, cell_aligned: bool, n: int) -> np.ndarray:
    parts = []
    # ground-like points around the sensor
    r = rng.uniform(0.05, 3.0, n)
    a = rng.uniform(0, 2 * math.pi, n)
    parts.append(np.column_stack([r * np.cos(a), r * np.sin(a), -1.0 + 0.05 * rng.standard_normal(n)]))
    # a box-like cluster (dense cells, wall rule, outliers)
    m = n // 4
    parts.append(np.column_stack([rng.uniform(0.4, 0.8, m), rng.uniform(-0.2, 0.2, m),
                                  rng.uniform(-1.0, -0.4, m)]))
    if cell_aligned:  # exactly on cell boundaries (sensor at a cell corner, identity rotation)
        k = rng.integers(-40, 40, (m, 2)).astype(np.float64)
        parts.append(np.column_stack([k[:, 0] * res, k[:, 1] * res, rng.uniform(-1.2, -0.6, m)]))
    # vertical rays, duplicates, far points
    parts.append(np.column_stack([np.zeros(5), np.zeros(5), rng.uniform(-1.5, -0.5, 5)]))
    dup = parts[0][: max(1, n // 50)]
    parts.append(np.repeat(dup, 3, axis=0))
    far = rng.standard_normal((max(1, n // 30), 3)) * 40.0
    parts.append(far)
    xyz = np.concatenate(parts)
    if rng.random() < 0.3:
        bad = rng.integers(0, len(xyz), 4)
        xyz[bad[0], 0] = np.nan
        xyz[bad[1], 1] = np.inf
        xyz[bad[2], 2] = -np.inf
        xyz[bad[3]] = [np.nan, np.nan, np.nan]
    return xyz[rng.permutation(len(xyz))] if rng.random() < 0.5 else xyz


@pytest.mark.parametrize("seed", SEEDS)
def test_randomised_scenarios_match_reference(gpu, reference, tmp_path, seed):
    rng = np.random.default_rng(1000 + seed)
    res = float(rng.choice([0.02, 0.04, 0.05, 0.1]))
    W, H = int(rng.integers(20, 300)), int(rng.integers(20, 300))
    cell_aligned = bool(rng.random() < 0.4)
    text, drift = _config(rng)
    cfg_path = tmp_path / "soak.config"
    cfg_path.write_text(wl._map(res, W, H) + text)
    libs = (gpu, reference)
    cfgs = [pk.Config.load(lib, cfg_path) for lib in libs]
    maps = [pk.ReliefMap.create(lib, res, W, H) for lib in libs]
    pos = np.zeros(3)
    stamp = 0.0
    for f in range(6):
        if cell_aligned:
            R = np.eye(3)
            step = rng.integers(-3, 4, 2) * res  # whole cells: boundaries stay exact
            pos = np.array([pos[0] + step[0], pos[1] + step[1], 1.0])
        else:
            yaw, pitch = rng.uniform(-math.pi, math.pi), rng.uniform(-0.3, 0.3)
            R = wl.rot_z(yaw) @ wl.rot_y(pitch)
            pos = pos + np.array([rng.normal(0, 3 * res), rng.normal(0, 3 * res), 0.0])
            pos[2] = rng.uniform(0.4, 1.8)
        pose = wl.pose34(R, tuple(pos))
        stamp += float(rng.choice([0.0, 0.1, 0.4, 1.5]))
        xyz = _cloud(rng, res, cell_aligned, int(rng.integers(200, 6000)))
        got = maps[0].integrate(xyz, pose, stamp, cfgs[0])
        want = maps[1].integrate(xyz, pose, stamp, cfgs[1])
        ctx = f"seed {seed} frame {f} ({W}x{H}@{res}, aligned={cell_aligned}, drift={drift})"
        assert_stats_match(got, want, drift_tol=1e-12 if drift else 0.0, context=ctx)
        assert_layers_match(maps[0].layers(), maps[1].layers(), height_tol=1e-9 if drift else 0.0,
                            context=ctx)


# Long sequences: the ray pass's jumps engage once the map's cells have been
# observed and their bounds settled, so these scenarios run 24 frames of a slowly moving sensor
# over the same ground (every 6th frame with a stamp gap that makes cells stale) and compare
# every frame. RELIEF_SOAK_LONG_SEEDS=N widens the sweep.
LONG_SEEDS = list(range(int(os.environ.get("RELIEF_SOAK_LONG_SEEDS", "6"))))


@pytest.mark.parametrize("seed", LONG_SEEDS)
def test_randomised_long_sequences_match_reference(gpu, reference, tmp_path, seed):
    rng = np.random.default_rng(7000 + seed)
    res = float(rng.choice([0.02, 0.04, 0.05]))
    W, H = int(rng.integers(60, 260)), int(rng.integers(60, 260))
    text, drift = _config(rng)
    cfg_path = tmp_path / "soak_long.config"
    cfg_path.write_text(wl._map(res, W, H) + text)
    libs = (gpu, reference)
    cfgs = [pk.Config.load(lib, cfg_path) for lib in libs]
    maps = [pk.ReliefMap.create(lib, res, W, H) for lib in libs]
    pos = np.array([0.0, 0.0, rng.uniform(0.5, 1.5)])
    base = _cloud(rng, res, False, int(rng.integers(2000, 8000)))
    stamp = 0.0
    for f in range(24):
        yaw = rng.uniform(-0.2, 0.2)
        R = wl.rot_z(yaw) @ wl.rot_y(rng.uniform(-0.05, 0.05))
        pos = pos + np.array([rng.normal(0, 0.5 * res), rng.normal(0, 0.5 * res), 0.0])
        pose = wl.pose34(R, tuple(pos))
        stamp += 1.5 if f % 6 == 5 else 0.1
        jitter = base + rng.normal(0, 0.3 * res, base.shape)  # the same scene, re-sampled
        xyz = np.concatenate([jitter, _cloud(rng, res, False, int(rng.integers(100, 600)))])
        got = maps[0].integrate(xyz, pose, stamp, cfgs[0])
        want = maps[1].integrate(xyz, pose, stamp, cfgs[1])
        ctx = f"long seed {seed} frame {f} ({W}x{H}@{res}, drift={drift})"
        assert_stats_match(got, want, drift_tol=1e-12 if drift else 0.0, context=ctx)
        assert_layers_match(maps[0].layers(), maps[1].layers(), height_tol=1e-9 if drift else 0.0,
                            context=ctx)


def _frames(rng, res, cell_aligned, n_frames):
    pos, stamp, out = np.zeros(3), 0.0, []
    for _ in range(n_frames):
        if cell_aligned:
            R = np.eye(3)
            step = rng.integers(-3, 4, 2) * res
            pos = np.array([pos[0] + step[0], pos[1] + step[1], 1.0])
        else:
            R = wl.rot_z(rng.uniform(-math.pi, math.pi)) @ wl.rot_y(rng.uniform(-0.3, 0.3))
            pos = pos + np.array([rng.normal(0, 3 * res), rng.normal(0, 3 * res), 0.0])
            pos[2] = rng.uniform(0.4, 1.8)
        stamp += float(rng.choice([0.0, 0.1, 0.4, 1.5]))
        out.append((_cloud(rng, res, cell_aligned, int(rng.integers(200, 6000))),
                    wl.pose34(R, tuple(pos)), stamp))
    return out


@pytest.mark.parametrize("seed", SEEDS[: max(1, len(SEEDS) // 4)])
def test_randomised_sharded_frames_match_single_call(gpu, tmp_path, seed):
    """G replicas integrating one frame as exact point-batch shards (multigpu.
    integrate_sharded_lockstep) equal the single relief_map_integrate call, which the scenarios
    above tie to the reference."""
    from paper_2204_12876_b200 import multigpu as mg
    rng = np.random.default_rng(5000 + seed)
    res = float(rng.choice([0.02, 0.04, 0.05, 0.1]))
    W, H = int(rng.integers(20, 300)), int(rng.integers(20, 300))
    cell_aligned = bool(rng.random() < 0.4)
    text, drift = _config(rng)
    G = int(rng.integers(2, 5))
    cfg_path = tmp_path / "shard_soak.config"
    cfg_path.write_text(wl._map(res, W, H) + text)
    cfg = pk.Config.load(gpu, cfg_path)
    single = pk.ReliefMap.create(gpu, res, W, H)
    reps = [pk.ReliefMap.create(gpu, res, W, H) for _ in range(G)]
    apis = [mg.CudaShardAPI(gpu, m, cfg) for m in reps]
    for f, (xyz, pose, stamp) in enumerate(_frames(rng, res, cell_aligned, 5)):
        want = single.integrate(xyz, pose, stamp, cfg)
        got = mg.integrate_sharded_lockstep(apis, xyz, pose, stamp)
        ctx = f"seed {seed} frame {f} G={G} ({W}x{H}@{res}, drift={drift})"
        for g, (st, m) in enumerate(zip(got, reps)):
            assert_stats_match(st, want, drift_tol=1e-12 if drift else 0.0, context=f"{ctx} rank {g}")
            assert_layers_match(m.layers(), single.layers(), height_tol=1e-9 if drift else 0.0,
                                context=f"{ctx} rank {g}")


@pytest.mark.parametrize("seed", SEEDS[: max(1, len(SEEDS) // 4)])
def test_randomised_streaming_matches_sync(gpu, tmp_path, seed):
    """Up to three frames in flight (relief_gpu_map_integrate_async / wait) from pinned memory
    equal the synchronous sequence bit for bit."""
    import torch
    rng = np.random.default_rng(9000 + seed)
    res = float(rng.choice([0.02, 0.04, 0.05, 0.1]))
    W, H = int(rng.integers(20, 300)), int(rng.integers(20, 300))
    text, _ = _config(rng)
    cfg_path = tmp_path / "stream_soak.config"
    cfg_path.write_text(wl._map(res, W, H) + text)
    cfg = pk.Config.load(gpu, cfg_path)
    sync = pk.ReliefMap.create(gpu, res, W, H)
    stream = pk.ReliefMap.create(gpu, res, W, H)
    frames = _frames(rng, res, bool(rng.random() < 0.4), 7)
    want = [sync.integrate(x, p, t, cfg) for x, p, t in frames]
    pinned = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy() for x, _, _ in frames]
    got = []
    for x, (_, p, t) in zip(pinned, frames):
        stream.integrate_async(x, p, t, cfg)
        if gpu.relief_gpu_map_in_flight(stream.handle) == 3:
            got.append(stream.wait())
    while gpu.relief_gpu_map_in_flight(stream.handle):
        got.append(stream.wait())
    for k, (g, w) in enumerate(zip(got, want)):
        assert_stats_match(g, w, context=f"seed {seed} frame {k}")
    assert_layers_match(stream.layers(), sync.layers(), context=f"seed {seed} final map")
