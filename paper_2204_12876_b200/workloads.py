"""Synthetic workloads C1-C5 and the headline frame.

Each workload is a reliefmap config text (scene + sensor + map + pipeline keys, the
reference's own format) plus a pose / stamp schedule. Clouds are rendered by the
library's scene simulator (relief_gpu_sim_render), an independent implementation of
the reference simulator (reference sim.cpp:241-262) that reproduces its clouds bit for
bit, so the same config text drives the reference and this build identically.

Scene S0 = reference configs/flat_ground.config:20-22 (ground + box + 4-step stairs).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Tuple

import numpy as np

SCENE_S0 = """scene.ground = 0.0
scene.box = 1.5 0.5 0.25 0.6 0.6 0.5
scene.stairs = -2.0 -0.6 0 0.18 0.28 4 1.2 -x
"""

QUIET = """drift.enabled = false
cleanup.enabled = false
cleanup.upper_bound_enabled = false
overlap.enabled = false
"""


def ring_elevations_deg(n: int = 128, lo: float = -45.0, span: float = 39.0) -> List[float]:
    return [lo + span * k / (n - 1) for k in range(n)]


def depth_camera(cols: int, rows: int) -> str:
    return (f"sensor.pattern = grid\nsensor.h_fov_deg = 87\nsensor.v_fov_deg = 58\n"
            f"sensor.cols = {cols}\nsensor.rows = {rows}\nsensor.max_range = 10\n")


def lidar(azimuths: int, rings: int = 128) -> str:
    elev = " ".join(repr(e) for e in ring_elevations_deg(rings))
    return (f"sensor.pattern = rings\nsensor.ring_elevations_deg = {elev}\n"
            f"sensor.azimuth_steps = {azimuths}\nsensor.max_range = 10\n")


def rot_y(theta: float) -> np.ndarray:
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])


def rot_z(psi: float) -> np.ndarray:
    c, s = math.cos(psi), math.sin(psi)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def pose34(R: np.ndarray, t) -> np.ndarray:
    out = np.zeros((3, 4))
    out[:, :3] = R
    out[:, 3] = t
    return out.reshape(12).copy()


@dataclass
class Call:
    """One relief_map_integrate call of a frame."""
    pose: np.ndarray      # row-major 3x4 [R | t]
    stamp: float
    seed: int
    scan_index: int
    time: float


@dataclass
class Workload:
    name: str
    description: str
    config_text: str
    resolution: float
    width: int
    height: int
    calls: Callable[[int], List[Call]]   # frame -> integrate calls
    points_per_frame: int = 0            # nominal (filled after rendering)
    extra: dict = field(default_factory=dict)


def _map(res: float, w: int, h: int) -> str:
    return f"map.resolution = {res!r}\nmap.width = {w}\nmap.height = {h}\n"


def c1() -> Workload:
    text = _map(0.04, 200, 200) + "noise.alpha_d = 0.0002\n" + depth_camera(160, 125) + SCENE_S0 + QUIET
    R = rot_z(0.0) @ rot_y(0.6)
    return Workload("C1", "depth camera 160x125 (19,477 pts) -> 200x200 @0.04 m, fusion + time variance",
                    text, 0.04, 200, 200,
                    lambda f: [Call(pose34(R, (0.0, 0.0, 0.6)), 0.1 * f, 1, f, 0.1 * f)])


def c2() -> Workload:
    text = _map(0.02, 400, 400) + "noise.alpha_d = 0.0002\n" + depth_camera(320, 240) + SCENE_S0
    Rs = [rot_z(math.radians(a)) @ rot_y(0.6) for a in (0.0, 90.0, 180.0, 270.0)]
    return Workload("C2", "4 depth cameras 320x240 (~300k pts/frame, 4 calls) -> 400x400 @0.02 m, "
                    "cleanup + drift", text, 0.02, 400, 400,
                    lambda f: [Call(pose34(Rs[j], (0.0, 0.0, 0.6)), 0.1 * f, 2, 4 * f + j, 0.1 * f)
                               for j in range(4)])


def c3() -> Workload:
    text = _map(0.04, 500, 500) + "noise.alpha_d = 0.0002\n" + lidar(2048) + SCENE_S0
    return Workload("C3", "128-ring LiDAR x 2048 azimuths (262,144 pts) -> 500x500 @0.04 m, "
                    "1-cell recenter per frame", text, 0.04, 500, 500,
                    lambda f: [Call(pose34(np.eye(3), (0.04 * f, 0.0, 1.0)), 0.1 * f, 3, f, 0.1 * f)])


def c4() -> Workload:
    text = _map(0.04, 1000, 1000) + "noise.alpha_d = 0.0002\n" + lidar(7813) + SCENE_S0
    return Workload("C4", "128-ring LiDAR x 7813 azimuths (1,000,064 pts) -> 1000x1000 @0.04 m, "
                    "defaults incl. ray-cast cleanup", text, 0.04, 1000, 1000,
                    lambda f: [Call(pose34(np.eye(3), (0.0, 0.0, 1.0)), 0.1 * f, 4, f, 0.1 * f)])


def headline() -> Workload:
    text = _map(0.04, 500, 500) + "noise.alpha_d = 0.0002\n" + lidar(7813) + SCENE_S0
    return Workload("headline", "128-ring LiDAR x 7813 azimuths (1,000,064 pts) -> 500x500 @0.04 m, "
                    "defaults incl. ray-cast cleanup", text, 0.04, 500, 500,
                    lambda f: [Call(pose34(np.eye(3), (0.0, 0.0, 1.0)), 0.1 * f, 5, f, 0.1 * f)])


# C5 post-processing chain: min_inpaint, median r1,
# gaussian r2 sigma 1, box r1 -- as (kind, radius, sigma), kinds per relief_gpu.h.
C5_CHAIN: List[Tuple[int, int, float]] = [(3, 0, 1.0), (2, 1, 1.0), (0, 2, 1.0), (1, 1, 1.0)]

ALL = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "headline": headline}
