"""Group frames (relief_gpu_group_*, SURVEY §8e exact variant) on one GPU.

One frame split across G ranks, exchanges inside the library on the maps' streams:
* the local transport drives G replicas of the map on the same GPU from one process (peer copies
  + reduction kernels), exactly the phase code the NCCL transport runs;
* the NCCL transport with one rank (a real NCCL communicator; several ranks need several GPUs,
  which bench.py --gpus N exercises and checks with a layer hash).
After every frame each replica must equal relief_map_integrate of the whole frame on one map --
bit for bit, drift compensation included (the gathered drift block partials are the single-GPU
ones), and every ScanStats counter exact.
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


class Grouped:
    def __init__(self, lib, tmp_path, text, res, W, H, G, nccl=False):
        self.cfg_path = tmp_path / "group.config"
        self.cfg_path.write_text(text)
        self.cfg = pk.Config.load(lib, self.cfg_path)
        self.single = pk.ReliefMap.create(lib, res, W, H)
        self.reps = [pk.ReliefMap.create(lib, res, W, H) for _ in range(G)]
        if nccl:
            assert G == 1
            self.group = mg.create_nccl_group(lib, self.reps[0])
        else:
            self.group = pk.Group.local(lib, self.reps)

    def frame(self, xyz, pose, stamp, context="", device=False):
        want = self.single.integrate(xyz, pose, stamp, self.cfg)
        n = len(xyz)
        if device:
            import torch
            t = torch.from_numpy(np.ascontiguousarray(xyz, dtype=np.float64)).cuda()
            torch.cuda.synchronize()
            got = self.group.integrate_device(t.data_ptr(), n, n, pose, stamp, self.cfg)
        else:
            got = self.group.integrate(xyz, n, pose, stamp, self.cfg)
        ref_layers = self.single.layers()
        assert_stats_match(got, want, context=context)
        for g, m in enumerate(self.reps):
            assert m.center() == self.single.center()
            assert_layers_match(m.layers(), ref_layers, context=f"{context} rank {g}")
        return want


@pytest.mark.parametrize("G", [2, 3, 4])
def test_group_lidar_recenter_drift_bit_exact(gpu, reference, tmp_path, G):
    """Defaults incl. drift compensation, recenter every frame: bit-exact at every G."""
    text = wl._map(0.04, 300, 300) + "noise.alpha_d = 0.0002\n" + wl.lidar(512, rings=64) + wl.SCENE_S0
    gr = Grouped(gpu, tmp_path, text, 0.04, 300, 300, G)
    applied = 0
    for f in range(6):
        pose = wl.pose34(np.eye(3), (0.04 * f + 0.013, -0.021 * f, 1.0 + 0.01 * f))
        xyz = ref_render(reference, gr.cfg_path, pose, 0.1 * f, 3, f)
        st = gr.frame(xyz, pose, 0.15 * f, context=f"G={G} frame {f}")
        assert st.points_fused > 0
        applied += st.drift_offset_applied != 0.0
    assert applied >= 2


def test_group_moving_box_removals_bit_exact(gpu, reference, tmp_path):
    """Removals fire: global ray ids in k*, the merged bounds of removed cells."""
    text = (wl._map(0.04, 120, 120) +
            "noise.alpha_d = 0.005\nupdate.sigma_outlier2 = 0.0001\ndrift.enabled = false\n"
            "overlap.enabled = false\nexclusion.enabled = false\ncleanup.t_free = 1.0\n"
            "sensor.pattern = grid\nsensor.h_fov_deg = 70\nsensor.v_fov_deg = 60\n"
            "sensor.cols = 160\nsensor.rows = 140\nsensor.max_range = 10\n"
            "scene.ground = 0.0\nscene.moving_box = 1.2 0.0 0.3 0.8 0.8 0.6 0 0 0 -1 2.95\n")
    gr = Grouped(gpu, tmp_path, text, 0.04, 120, 120, 4)
    pose = wl.pose34(wl.rot_y(math.radians(35.0)), (0.0, 0.0, 1.2))
    removed = 0
    for s in range(45):
        xyz = ref_render(reference, gr.cfg_path, pose, s * 0.1, 4, s)
        removed += gr.frame(xyz, pose, s * 0.1, context=f"scan {s}").cells_removed_by_cleanup
    assert removed > 50, removed


def test_group_empty_tiny_and_device_input(gpu, tmp_path):
    """More ranks than tiles, empty frames, device-resident input."""
    text = wl._map(0.04, 60, 60)
    gr = Grouped(gpu, tmp_path, text, 0.04, 60, 60, 3)
    rng = np.random.default_rng(3)
    pose = wl.pose34(np.eye(3), (0.0, 0.0, 1.0))
    for f, n in enumerate([3, 0, 5000, 1, 7000]):
        xyz = np.stack([rng.normal(0, 0.5, n), rng.normal(0, 0.5, n), rng.normal(-1, 0.1, n)], axis=1)
        gr.frame(xyz, pose, 0.2 * f, context=f"n={n}", device=bool(f % 2))


def test_group_nccl_single_rank_matches(gpu, reference, tmp_path):
    """The NCCL transport (real communicator, one rank) on the C3 workload with drift."""
    w = wl.c3()
    gr = Grouped(gpu, tmp_path, w.config_text, w.resolution, w.width, w.height, 1, nccl=True)
    assert gpu.relief_gpu_nccl_version() >= 21800
    for f in range(4):
        for c in w.calls(f):
            xyz = ref_render(reference, gr.cfg_path, c.pose, c.time, c.seed, c.scan_index)
            gr.frame(xyz, c.pose, c.stamp, context=f"C3 frame {f}", device=bool(f % 2))


def test_group_c4_full_size_four_ranks(gpu, reference, tmp_path):
    """The configured split at full size: C4 (1,000,064 points -> 1000x1000), 4 ranks."""
    w = wl.c4()
    gr = Grouped(gpu, tmp_path, w.config_text, w.resolution, w.width, w.height, 4)
    for f in range(2):
        for c in w.calls(f):
            xyz = ref_render(reference, gr.cfg_path, c.pose, c.time, c.seed, c.scan_index)
            gr.frame(xyz, c.pose, c.stamp, context=f"C4 frame {f}")


def test_shard_api_exchange_written_late_on_torch_stream(gpu, reference, tmp_path):
    """relief_gpu_shard_*: exchanges done by torch ops that land late (a sleep kernel queued
    before each one on torch's stream) must still be seen by the library (after_stream)."""
    import torch
    text = wl._map(0.04, 200, 200) + "noise.alpha_d = 0.0002\n" + wl.lidar(400, rings=48) + wl.SCENE_S0 + \
        "drift.enabled = false\n"
    cfgp = tmp_path / "late.config"
    cfgp.write_text(text)
    cfg = pk.Config.load(gpu, cfgp)
    single = pk.ReliefMap.create(gpu, 0.04, 200, 200)
    reps = [pk.ReliefMap.create(gpu, 0.04, 200, 200) for _ in range(2)]
    apis = [mg.CudaShardAPI(gpu, m, cfg) for m in reps]
    orig_cat, orig_amin = torch.cat, torch.Tensor.amin

    def slow_cat(*a, **k):
        torch.cuda._sleep(20_000_000)  # ~10 ms on torch's stream before the records land
        return orig_cat(*a, **k)

    def slow_amin(self, *a, **k):
        torch.cuda._sleep(20_000_000)
        return orig_amin(self, *a, **k)

    for f in range(3):
        pose = wl.pose34(np.eye(3), (0.03 * f, 0.0, 1.0))
        xyz = ref_render(reference, cfgp, pose, 0.1 * f, 5, f)
        want = single.integrate(xyz, pose, 0.2 * f, cfg)
        torch.cat, torch.Tensor.amin = slow_cat, slow_amin
        try:
            got = mg.integrate_sharded_lockstep(apis, xyz, pose, 0.2 * f)
        finally:
            torch.cat, torch.Tensor.amin = orig_cat, orig_amin
        for st, m in zip(got, reps):
            assert_stats_match(st, want, context=f"frame {f}")
            assert_layers_match(m.layers(), single.layers(), context=f"frame {f}")


# ------------------------------------------------ information-form group frames
# relief_gpu_group_set_fusion(RELIEF_GPU_GROUP_INFORMATION): each rank sums its own points per cell
# in information form and the sums are all-reduced. Checked against the
# reference's sequential Kalman fold run with its gates disabled (integration.cpp:40-55: the
# outlier gate cannot fire under mahalanobis_threshold = 1e12, the wall gate under 2^30 points),
# the configuration the mode requires; heights equal up to rounding (1e-9 relative here).
UNGATED = "update.mahalanobis_threshold = 1e12\nupdate.wall_count_threshold = 1073741824\n"


def _info_run(gpu, reference, tmp_path, text, res, W, H, G, frames, context):
    cfg_path = tmp_path / "info.config"
    cfg_path.write_text(text)
    cfg, cfg_ref = pk.Config.load(gpu, cfg_path), pk.Config.load(reference, cfg_path)
    ref_map = pk.ReliefMap.create(reference, res, W, H)
    reps = [pk.ReliefMap.create(gpu, res, W, H) for _ in range(G)]
    group = pk.Group.local(gpu, reps)
    group.set_fusion(pk.Group.INFORMATION)
    assert group.fusion == pk.Group.INFORMATION
    totals = {"points_fused": 0, "cells_removed_by_cleanup": 0}
    for f, (xyz, pose, stamp) in enumerate(frames(cfg_path)):
        want = ref_map.integrate(xyz, pose, stamp, cfg_ref)
        got = group.integrate(xyz, len(xyz), pose, stamp, cfg)
        ctx = f"{context} G={G} frame {f}"
        assert_stats_match(got, want, drift_tol=1e-12, context=ctx)
        for k in totals:
            totals[k] += getattr(got, k)
        ref_layers = ref_map.layers()
        for g, m in enumerate(reps):
            assert m.center() == ref_map.center()
            assert_layers_match(m.layers(), ref_layers, height_tol=1e-9, tol_trav=1e-9,
                                context=f"{ctx} rank {g}")
    group.close()
    return totals


@pytest.mark.parametrize("G", [1, 2, 3])
def test_group_information_form_vs_reference_ungated(gpu, reference, tmp_path, G):
    """Recenter every frame, drift compensation, cleanup + bounds (reference defaults otherwise)."""
    text = wl._map(0.04, 300, 300) + "noise.alpha_d = 0.0002\n" + wl.lidar(512, rings=64) + \
        wl.SCENE_S0 + UNGATED

    def frames(cfg_path):
        for f in range(6):
            pose = wl.pose34(np.eye(3), (0.04 * f + 0.013, -0.021 * f, 1.0 + 0.01 * f))
            yield ref_render(reference, cfg_path, pose, 0.1 * f, 3, f), pose, 0.15 * f

    t = _info_run(gpu, reference, tmp_path, text, 0.04, 300, 300, G, frames, "lidar")
    assert t["points_fused"] > 0


def test_group_information_form_removals(gpu, reference, tmp_path):
    """Removals fire under the information form (4 ranks): a box seen by beams 25-35 degrees
    down vanishes at 2.95 s; the beams then pass below its stale top cells to the ground behind
    (ungated fusion would average any point landing in them, so none may land there)."""
    text = (wl._map(0.04, 120, 120) +
            "noise.alpha_d = 0.005\nupdate.sigma_outlier2 = 0.0001\ndrift.enabled = false\n"
            "overlap.enabled = false\nexclusion.enabled = false\ncleanup.t_free = 0.3\n"
            "sensor.pattern = grid\nsensor.h_fov_deg = 70\nsensor.v_fov_deg = 10\n"
            "sensor.cols = 160\nsensor.rows = 30\nsensor.max_range = 10\n"
            "scene.ground = 0.0\nscene.moving_box = 1.2 0.0 0.3 0.8 0.8 0.6 0 0 0 -1 2.95\n" + UNGATED)
    pose = wl.pose34(wl.rot_y(math.radians(30.0)), (0.0, 0.0, 1.2))

    def frames(cfg_path):
        for s in range(60):
            yield ref_render(reference, cfg_path, pose, s * 0.1, 4, s), pose, s * 0.1

    t = _info_run(gpu, reference, tmp_path, text, 0.04, 120, 120, 4, frames, "moving box")
    assert t["cells_removed_by_cleanup"] > 50, t


def test_group_information_form_c4_full_size(gpu, reference, tmp_path):
    """The configured C4 split (1,000,064 points -> 1000x1000) over 4 ranks, information form."""
    w = wl.c4()

    def frames(cfg_path):
        for f in range(2):
            for c in w.calls(f):
                yield ref_render(reference, cfg_path, c.pose, c.time, c.seed, c.scan_index), c.pose, c.stamp

    t = _info_run(gpu, reference, tmp_path, w.config_text + UNGATED, w.resolution, w.width, w.height, 4,
                  frames, "C4")
    assert t["points_fused"] > 1_000_000


def test_group_information_form_needs_ungated_config(gpu, tmp_path):
    """The mode refuses a config whose gates can fire (RELIEF_ERROR_USAGE), and unknown modes."""
    cfg_path = tmp_path / "gated.config"
    cfg_path.write_text(wl._map(0.04, 60, 60))
    cfg = pk.Config.load(gpu, cfg_path)
    reps = [pk.ReliefMap.create(gpu, 0.04, 60, 60) for _ in range(2)]
    group = pk.Group.local(gpu, reps)
    with pytest.raises(pk.ReliefError):
        group.set_fusion(7)
    group.set_fusion(pk.Group.INFORMATION)
    xyz = np.stack([np.zeros(10), np.zeros(10), -np.ones(10)], axis=1)
    with pytest.raises(pk.ReliefError) as e:
        group.integrate(xyz, 10, wl.pose34(np.eye(3), (0.0, 0.0, 1.0)), 0.0, cfg)
    assert "information-form" in str(e.value)
    group.set_fusion(pk.Group.EXACT)
    group.integrate(xyz, 10, wl.pose34(np.eye(3), (0.0, 0.0, 1.0)), 0.0, cfg)
    group.close()
