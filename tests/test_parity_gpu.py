"""GPU parity: librelief_b200.so against the reference implementation (oracle/_ref), both
driven through the same C ABI (relief.h) with identical configs, clouds, poses and stamps.

Bar: every ScanStats counter exact; elevation, variance, last_update,
upper_bound(+valid), normals and validity bit-exact; traversability within 1e-12 (device
acos vs libm acos). Runs with drift compensation enabled compare heights within 1e-9
relative because the drift mean is a parallel (fixed-order) sum.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl

from conftest import assert_layers_match, assert_stats_match, ref_render

pytestmark = pytest.mark.gpu


class Pair:
    """The same map driven through both libraries."""

    def __init__(self, product, reference, tmp_path, config_text, res, W, H, cx=0.0, cy=0.0):
        self.cfg_path = tmp_path / "run.config"
        self.cfg_path.write_text(config_text)
        self.libs = (product, reference)
        self.cfgs = [pk.Config.load(lib, self.cfg_path) for lib in self.libs]
        self.maps = [pk.ReliefMap.create(lib, res, W, H, cx, cy) for lib in self.libs]

    def integrate(self, xyz, pose, stamp, drift_tol=0.0, context=""):
        got = self.maps[0].integrate(xyz, pose, stamp, self.cfgs[0])
        want = self.maps[1].integrate(xyz, pose, stamp, self.cfgs[1])
        assert_stats_match(got, want, drift_tol=drift_tol, context=context)
        return got, want

    def compare(self, height_tol=0.0, context=""):
        assert self.maps[0].center() == self.maps[1].center()
        assert_layers_match(self.maps[0].layers(), self.maps[1].layers(), height_tol=height_tol,
                            context=context)


def _render(reference, pair, call):
    return ref_render(reference, pair.cfg_path, call.pose, call.time, call.seed, call.scan_index)


def test_c1_depth_camera_fusion_bit_exact(gpu, reference, tmp_path):
    w = wl.c1()
    pair = Pair(gpu, reference, tmp_path, w.config_text, w.resolution, w.width, w.height)
    for f in range(6):
        for call in w.calls(f):
            xyz = _render(reference, pair, call)
            got, _ = pair.integrate(xyz, call.pose, call.stamp, context=f"frame {f}")
            assert got.points_fused > 0
        pair.compare(context=f"C1 frame {f}")


def test_lidar_recenter_every_frame_bit_exact(gpu, reference, tmp_path):
    # C3 geometry at reduced azimuth count; defaults except drift (exact mean below).
    text = wl._map(0.04, 300, 300) + "noise.alpha_d = 0.0002\n" + wl.lidar(512, rings=64) + wl.SCENE_S0 + \
        "drift.enabled = false\n"
    pair = Pair(gpu, reference, tmp_path, text, 0.04, 300, 300)
    for f in range(8):
        pose = wl.pose34(np.eye(3), (0.04 * f + 0.013, -0.021 * f, 1.0))
        xyz = ref_render(reference, pair.cfg_path, pose, 0.1 * f, 3, f)
        pair.integrate(xyz, pose, 0.15 * f, context=f"frame {f}")
        pair.compare(context=f"lidar frame {f}")


def test_moving_box_cleanup_removals_bit_exact(gpu, reference, tmp_path):
    # Acceptance #4 scene (reference acceptance.cpp:275-357): the box vacates at 2.95 s and
    # rays through its stale top remove cells -> exercises k* ordering for upper bounds.
    text = (wl._map(0.04, 120, 120) +
            "noise.alpha_d = 0.005\nupdate.sigma_outlier2 = 0.0001\ndrift.enabled = false\n"
            "overlap.enabled = false\nexclusion.enabled = false\ncleanup.t_free = 1.0\n"
            "sensor.pattern = grid\nsensor.h_fov_deg = 70\nsensor.v_fov_deg = 60\n"
            "sensor.cols = 160\nsensor.rows = 140\nsensor.max_range = 10\n"
            "scene.ground = 0.0\nscene.moving_box = 1.2 0.0 0.3 0.8 0.8 0.6 0 0 0 -1 2.95\n")
    pair = Pair(gpu, reference, tmp_path, text, 0.04, 120, 120)
    pitch = math.radians(35.0)
    pose = wl.pose34(wl.rot_y(pitch), (0.0, 0.0, 1.2))
    removed = 0
    for s in range(50):
        xyz = ref_render(reference, pair.cfg_path, pose, s * 0.1, 4, s)
        got, _ = pair.integrate(xyz, pose, s * 0.1, context=f"scan {s}")
        removed += got.cells_removed_by_cleanup
        if s % 10 == 9 or got.cells_removed_by_cleanup:
            pair.compare(context=f"moving box scan {s}")
    assert removed > 50, removed


def test_defaults_with_drift_tolerance(gpu, reference, tmp_path):
    text = wl._map(0.04, 250, 250) + "noise.alpha_d = 0.0002\n" + wl.lidar(720, rings=48) + wl.SCENE_S0
    pair = Pair(gpu, reference, tmp_path, text, 0.04, 250, 250)
    applied = 0
    for f in range(8):
        pose = wl.pose34(np.eye(3), (0.02 * f, 0.0, 1.0 + 0.01 * f))
        xyz = ref_render(reference, pair.cfg_path, pose, 0.1 * f, 7, f)
        got, _ = pair.integrate(xyz, pose, 0.1 * f, drift_tol=1e-12, context=f"frame {f}")
        applied += got.drift_offset_applied != 0.0
        pair.compare(height_tol=1e-9, context=f"drift frame {f}")
    assert applied >= 3


def _random_cloud(rng, n, spread=2.0, zsd=0.8):
    return np.stack([rng.normal(0, spread, n), rng.normal(0, spread, n), rng.normal(0, zsd, n)], axis=1)


def test_random_clouds_counters_partition(gpu, reference, tmp_path):
    # reference test_integration.cpp:216-243 with all stages on (drift off for exactness).
    text = ("exclusion.b = 0.2\nexclusion.c = 0.1\nexclusion.theta_a_deg = 17.188733853924695\n"
            "update.max_range = 3.0\ndrift.enabled = false\n")
    pair = Pair(gpu, reference, tmp_path, text, 0.04, 100, 100)
    rng = np.random.default_rng(8)
    pose = wl.pose34(np.eye(3), (0.0, 0.0, 0.5))
    for scan in range(6):
        xyz = _random_cloud(rng, 3000)
        got, _ = pair.integrate(xyz, pose, scan * 0.1, context=f"scan {scan}")
        total = (got.points_excluded + got.points_out_of_range + got.points_out_of_map +
                 got.points_rejected_outlier + got.points_ignored_low + got.points_fused)
        assert got.points_in == 3000 == total
        assert got.points_excluded > 0 and got.points_out_of_range > 0
        pair.compare(context=f"random scan {scan}")


def test_dense_cells_wall_rule_and_outliers(gpu, reference, tmp_path):
    # Many points per cell in scan order exercises the order-dependent gated fold.
    pair = Pair(gpu, reference, tmp_path, "drift.enabled = false\nupdate.sigma_outlier2 = 0.02\n",
                0.04, 60, 60)
    rng = np.random.default_rng(3)
    pose = wl.pose34(np.eye(3), (0.0, 0.0, 1.0))
    for scan in range(5):
        n = 40000
        xy = rng.uniform(-0.6, 0.6, (n, 2))
        z = -1.0 + 0.05 * rng.standard_normal(n) + (rng.random(n) < 0.1) * rng.uniform(-0.5, 0.5, n)
        xyz = np.column_stack([xy, z])
        got, _ = pair.integrate(xyz, pose, 0.1 * scan, context=f"scan {scan}")
        assert got.points_ignored_low > 0 and got.points_rejected_outlier > 0
        pair.compare(context=f"dense scan {scan}")


def test_rotated_pose_and_far_points(gpu, reference, tmp_path):
    pair = Pair(gpu, reference, tmp_path, "drift.enabled = false\n", 0.05, 80, 64, 0.3, -0.2)
    rng = np.random.default_rng(11)
    q = np.array([0.3, -0.5, 0.8, 0.1])
    q /= np.linalg.norm(q)
    w, x, y, z = q
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
                  [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
                  [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)]])
    for scan in range(4):
        pose = wl.pose34(R, (0.1 * scan, -0.05 * scan, 0.7))
        xyz = _random_cloud(rng, 5000, spread=3.0, zsd=1.0)
        xyz[::97] *= 50.0  # far points: out of range / out of map / clipped rays
        pair.integrate(xyz, pose, 0.3 * scan, context=f"scan {scan}")
        pair.compare(context=f"rotated scan {scan}")


def test_empty_cloud_only_ages(gpu, reference, tmp_path):
    pair = Pair(gpu, reference, tmp_path, "drift.enabled = false\n", 0.04, 100, 100)
    pose = wl.pose34(np.eye(3), (0.0, 0.0, 1.0))
    pair.integrate(np.array([[0.5, 0.5, -1.0]]), pose, 0.0)
    got, _ = pair.integrate(np.zeros((0, 3)), pose, 1.0)
    assert got.points_in == 0 and got.points_fused == 0
    pair.compare(context="empty cloud")


def test_nan_and_inf_points(gpu, reference, tmp_path):
    pair = Pair(gpu, reference, tmp_path, "drift.enabled = false\nexclusion.enabled = false\n",
                0.04, 60, 60)
    pose = wl.pose34(np.eye(3), (0.0, 0.0, 1.0))
    rng = np.random.default_rng(5)
    xyz = _random_cloud(rng, 2000, spread=0.8, zsd=0.1) - np.array([0, 0, 1.0])
    xyz[7] = [np.inf, 0.0, -1.0]
    xyz[9] = [0.2, np.nan, -1.0]
    xyz[11] = [0.3, 0.1, np.nan]
    xyz[13] = [-np.inf, np.nan, np.inf]
    for s in range(3):
        pair.integrate(xyz, pose, 2.0 * s, context=f"nan scan {s}")
        pair.compare(context=f"nan scan {s}")


def test_error_statuses_match(gpu, reference, tmp_path):
    pair = Pair(gpu, reference, tmp_path, "update.sigma_init2 = 0\n", 0.1, 10, 10)
    bad = wl.pose34(np.diag([5.0, 1.0, 1.0]), (0, 0, 0))
    for m, c in zip(pair.maps, pair.cfgs):
        with pytest.raises(pk.ReliefError) as e:
            m.integrate(np.zeros((1, 3)), bad, 0.0, c)
        assert e.value.status == 4
        with pytest.raises(pk.ReliefError) as e:
            m.integrate(np.array([[0.1, 0.1, -1.0]]), wl.pose34(np.eye(3), (0, 0, 1)), 0.0, c)
        assert e.value.status == 5
        with pytest.raises(pk.ReliefError) as e:
            m.layer("bogus")
        assert e.value.status == 1 and "elevation" in e.value.message


def _sections(text):
    out, cur = {}, "header"
    out[cur] = []
    for line in text.splitlines():
        if line.startswith("layer: "):
            cur = line[7:]
            out[cur] = []
        else:
            out[cur].append(line)
    return out


def test_snapshot_cross_compatible(gpu, reference, tmp_path):
    w = wl.c1()
    pair = Pair(gpu, reference, tmp_path, w.config_text, w.resolution, w.width, w.height)
    for f in range(3):
        for call in w.calls(f):
            pair.integrate(_render(reference, pair, call), call.pose, call.stamp)
    pm, rm = pair.maps
    pm.save(tmp_path / "p.relief")
    rm.save(tmp_path / "r.relief")
    # Byte-identical files except the traversability block (device acos, 1e-12).
    ps = _sections((tmp_path / "p.relief").read_text())
    rs = _sections((tmp_path / "r.relief").read_text())
    assert ps.keys() == rs.keys()
    for name in ps:
        if name != "traversability":
            assert ps[name] == rs[name], name
    a = np.array([[float(v) for v in row.split()] for row in ps["traversability"]])
    b = np.array([[float(v) for v in row.split()] for row in rs["traversability"]])
    assert np.array_equal(np.isnan(a), np.isnan(b))
    assert np.nanmax(np.abs(a - b)) <= 1e-12
    loaded = pk.ReliefMap.load(gpu, tmp_path / "r.relief")
    assert_layers_match(loaded.layers(), rm.layers(), tol_trav=0.0, context="loaded snapshot")


def test_overlapped_fold_retry_path(gpu, reference, tmp_path):
    """A long cell (> 64 points) that fuses nothing and stays a removal candidate: the ray pass
    that ran concurrently with its fold treated it as class none, so the exact retry must run
    and reproduce the reference (removal + upper bound)."""
    import snapshots as snap
    res, W, H = 0.1, 40, 40
    layers = snap.fresh(H, W)
    for r in range(H):
        for c in range(W):
            snap.set_cell(layers, r, c, 0.0, 0.01, 5.0, (0.0, 0.0, 1.0), 0.9)
    snap.set_cell(layers, 20, 25, 1.0, 0.01, 0.0, (0.0, 0.0, 1.0), 0.9)  # stale tall cell at x=0.55
    text = ("drift.enabled = false\noverlap.enabled = false\nexclusion.enabled = false\n"
            "update.wall_count_threshold = 5\nupdate.sigma_t2 = 0\n")
    p = tmp_path / "r.config"
    p.write_text(text)
    maps, cfgs = [], []
    for i, lib in enumerate((gpu, reference)):
        f = tmp_path / f"m{i}.relief"
        f.write_text(snap.text(layers, res))
        maps.append(pk.ReliefMap.load(lib, f))
        cfgs.append(pk.Config.load(lib, p))
    sensor = (0.05, 0.05, 0.8)
    pose = wl.pose34(np.eye(3), sensor)
    # 100 low points inside the tall cell (all ignored by the wall rule) ...
    low = np.tile([0.55 - 0.05, 0.05 - 0.05, 0.2 - 0.8], (100, 1))
    # ... and rays passing through it below its surface towards the ground beyond.
    far = np.array([[1.45 - 0.05, 0.05 - 0.05, 0.0 - 0.8 + 0.01 * k] for k in range(8)])
    xyz = np.concatenate([low, far])
    got = maps[0].integrate(xyz, pose, 5.0, cfgs[0])
    want = maps[1].integrate(xyz, pose, 5.0, cfgs[1])
    assert_stats_match(got, want)
    assert got.points_ignored_low == 100 and got.cells_removed_by_cleanup >= 1
    assert_layers_match(maps[0].layers(), maps[1].layers())


@pytest.mark.parametrize("W,H", [(3, 3), (45, 46), (64, 32), (2100, 2100)])
def test_sort_pass_count_paths(gpu, reference, tmp_path, W, H):
    """The stable radix sort by cell runs 1 pass (<= 2^11 cells), 2 passes (<= 2^22) or 3 passes
    (more cells); every geometry must keep scan order within cells (fold parity)."""
    res = 0.04 if W * H > 10_000 else 0.05
    pair = Pair(gpu, reference, tmp_path, "drift.enabled = false\nupdate.sigma_outlier2 = 0.02\n",
                res, W, H)
    rng = np.random.default_rng(W)
    pose = wl.pose34(np.eye(3), (0.0, 0.0, 1.0))
    half_x, half_y = 0.5 * W * res, 0.5 * H * res
    n = 200_000 if W * H > 1_000_000 else 20_000
    for scan in range(2):
        xy = np.column_stack([rng.uniform(-half_x, half_x, n), rng.uniform(-half_y, half_y, n)])
        xy = xy * np.where(rng.random((n, 1)) < 0.5, 0.02, 1.0)  # dense centre: long cells too
        z = -1.0 + 0.05 * rng.standard_normal(n)
        pair.integrate(np.column_stack([xy, z]), pose, 0.1 * scan, context=f"{W}x{H} scan {scan}")
        pair.compare(context=f"{W}x{H} scan {scan}")


def test_frame_sizes_changing_between_scans(gpu, reference, tmp_path):
    """Scratch sized by the largest frame, sort tile counts reused across scans of different
    sizes (tile-count layout changes with N), empty scans in between."""
    pair = Pair(gpu, reference, tmp_path, "drift.enabled = false\nupdate.sigma_outlier2 = 0.02\n",
                0.04, 150, 150)
    rng = np.random.default_rng(21)
    pose = wl.pose34(np.eye(3), (0.0, 0.0, 1.0))
    for scan, n in enumerate([20000, 3, 0, 70000, 5000, 2048, 2049, 150000, 1]):
        xy = rng.normal(0.0, 1.2, (n, 2))
        z = -1.0 + 0.05 * rng.standard_normal(n)
        pair.integrate(np.column_stack([xy, z]), pose, 0.1 * scan, context=f"n={n}")
        pair.compare(context=f"n={n}")


def _raw_sections(path):
    """Snapshot sections as float arrays (raw layers: the snapshot stores unmasked values)."""
    secs = _sections(path.read_text())
    return {k: np.array([[float(v) for v in row.split()] for row in rows if row.strip()])
            for k, rows in secs.items() if k != "header"}


def test_invalid_cells_normals_traversability_rebuilt(gpu, reference, tmp_path):
    """The reference rebuilds the normal and traversability layers every scan, with 0 for
    invalid cells (analysis.cpp:44-48,93). A loaded snapshot whose invalid cells carry non-zero
    normals / traversability must come out of the next scan with those zeroed, like the
    reference's (raw layers compared through save, not the NaN-masked export)."""
    import snapshots as snap
    res, W, H = 0.05, 48, 40
    rng = np.random.default_rng(5)
    layers = snap.fresh(H, W)
    for r in range(H):
        for c in range(W):
            if (r + c) % 3:
                snap.set_cell(layers, r, c, 0.01 * rng.standard_normal(), 0.01, 0.0, (0.0, 0.0, 1.0), 0.8)
            else:  # invalid cell with stale normals / traversability
                layers["normal_x"][r, c], layers["normal_z"][r, c] = 0.3, 0.9
                layers["traversability"][r, c] = 0.7
    p = tmp_path / "r.config"
    p.write_text("drift.enabled = false\nupdate.sigma_t2 = 0\n")
    pose = wl.pose34(np.eye(3), (0.0, 0.0, 1.0))
    xyz = np.column_stack([rng.uniform(-1.0, 1.0, 3000), rng.uniform(-0.9, 0.9, 3000),
                           -1.0 + 0.01 * rng.standard_normal(3000)])
    saved = []
    for i, lib in enumerate((gpu, reference)):
        f = tmp_path / f"m{i}.relief"
        f.write_text(snap.text(layers, res))
        m = pk.ReliefMap.load(lib, f)
        cfg = pk.Config.load(lib, p)
        m.integrate(xyz, pose, 1.0, cfg)
        m.save(tmp_path / f"o{i}.relief")
        saved.append(_raw_sections(tmp_path / f"o{i}.relief"))
    a, b = saved
    for name in ("normal_x", "normal_y", "normal_z", "valid", "elevation", "variance"):
        assert np.array_equal(a[name], b[name], equal_nan=True), name
    assert np.array_equal(np.isnan(a["traversability"]), np.isnan(b["traversability"]))
    assert np.nanmax(np.abs(a["traversability"] - b["traversability"])) <= 1e-12


def test_traversability_window_larger_than_shared_memory(gpu, reference, tmp_path):
    """A window whose shared-memory tile would exceed the SM's capacity runs the global-memory
    variant of the cell pass (the reference accepts any odd window)."""
    pair = Pair(gpu, reference, tmp_path, "drift.enabled = false\ntraversability.window = 151\n",
                0.04, 180, 170)
    rng = np.random.default_rng(9)
    pose = wl.pose34(np.eye(3), (0.0, 0.0, 1.0))
    for scan in range(2):
        xy = rng.uniform(-3.4, 3.4, (40000, 2))
        z = -1.0 + 0.05 * np.sin(xy[:, 0]) + 0.01 * rng.standard_normal(40000)
        pair.integrate(np.column_stack([xy, z]), pose, 0.1 * scan, context=f"scan {scan}")
        pair.compare(context=f"window 151 scan {scan}")


def test_graph_and_direct_launches_identical(gpu, reference, tmp_path):
    """One CUDA graph per frame vs direct launches (the default) vs the reference: frames whose size,
    recenter and input kind (pinned host / pageable host / device) change from call to call, so
    cached graphs are updated, re-instantiated and reused."""
    import torch
    text = wl._map(0.04, 200, 200) + "noise.alpha_d = 0.0002\n" + wl.lidar(300, rings=48) + wl.SCENE_S0
    pair = Pair(gpu, reference, tmp_path, text, 0.04, 200, 200)
    pair.maps[0].set_graphs(True)
    direct = pk.ReliefMap.create(gpu, 0.04, 200, 200)
    direct.set_graphs(False)  # direct launches
    cfg = pair.cfgs[0]
    for f in range(12):
        pose = wl.pose34(np.eye(3), (0.05 * (f // 3), 0.0, 1.0))  # recenter on every third frame
        xyz = ref_render(reference, pair.cfg_path, pose, 0.1 * f, 9, f)
        xyz = xyz[: len(xyz) - 997 * (f % 4)]                      # sizes change
        kind = f % 3
        if kind == 0:
            got = pair.maps[0].integrate(torch.from_numpy(xyz.copy()).pin_memory().numpy(), pose, 0.1 * f, cfg)
        elif kind == 1:
            got = pair.maps[0].integrate(xyz, pose, 0.1 * f, cfg)
        else:
            t = torch.from_numpy(xyz.copy()).cuda()
            torch.cuda.synchronize()
            got = pair.maps[0].integrate_device(t.data_ptr(), len(xyz), pose, 0.1 * f, cfg)
        want = pair.maps[1].integrate(xyz, pose, 0.1 * f, pair.cfgs[1])
        d = direct.integrate(xyz, pose, 0.1 * f, cfg)
        assert_stats_match(got, want, drift_tol=1e-12, context=f"frame {f}")
        assert_stats_match(d, got, context=f"direct frame {f}")
        assert_layers_match(direct.layers(), pair.maps[0].layers(), tol_trav=0.0, context=f"direct {f}")
        pair.compare(height_tol=1e-9, context=f"frame {f}")
    inst, upd = pair.maps[0].graph_stats()
    assert inst >= 2 and upd >= 6, (inst, upd)
    assert direct.graph_stats() == (0, 0)


def test_graph_modes_large_frames(gpu, reference, tmp_path):
    """Graph mode 2 (the default) on frames above both thresholds (the head launched directly,
    the rest captured), mode 1 and direct launches agree bit for bit, and with the reference."""
    text = wl._map(0.04, 400, 400) + "noise.alpha_d = 0.0002\n" + wl.lidar(4400, rings=128) + wl.SCENE_S0
    pair = Pair(gpu, reference, tmp_path, text, 0.04, 400, 400)   # default mode 2
    forced = pk.ReliefMap.create(gpu, 0.04, 400, 400)
    forced.set_graphs(1)
    direct = pk.ReliefMap.create(gpu, 0.04, 400, 400)
    direct.set_graphs(0)
    cfg = pair.cfgs[0]
    with pytest.raises(pk.ReliefError):
        direct.set_graphs(3)
    for f in range(4):
        pose = wl.pose34(np.eye(3), (0.05 * f, 0.0, 1.0))
        xyz = ref_render(reference, pair.cfg_path, pose, 0.1 * f, 9, f)
        xyz = xyz[: len(xyz) - 40000 * (f % 2)]            # above / below 512Ki points
        got = pair.maps[0].integrate(xyz, pose, 0.1 * f, cfg)
        want = pair.maps[1].integrate(xyz, pose, 0.1 * f, pair.cfgs[1])
        a = forced.integrate(xyz, pose, 0.1 * f, cfg)
        d = direct.integrate(xyz, pose, 0.1 * f, cfg)
        assert_stats_match(got, want, drift_tol=1e-12, context=f"frame {f}")
        assert_stats_match(a, got, context=f"mode 1 frame {f}")
        assert_stats_match(d, got, context=f"direct frame {f}")
        assert_layers_match(forced.layers(), pair.maps[0].layers(), tol_trav=0.0, context=f"mode 1 {f}")
        assert_layers_match(direct.layers(), pair.maps[0].layers(), tol_trav=0.0, context=f"direct {f}")
        pair.compare(height_tol=1e-9, context=f"frame {f}")
    assert pair.maps[0].graph_stats()[0] >= 1 and forced.graph_stats()[0] >= 1
    assert direct.graph_stats() == (0, 0)
