"""CPU-side checks of the drop-in boundary (no GPU needed).

* librelief_b200.so loads and exports exactly the symbols include/*.h declare;
* the relief.h surface matches the reference library's export list;
* configuration parsing (host code) agrees with the reference: accepted keys, rejected keys,
  error statuses and messages;
* without a CUDA device, map creation fails loudly (there is no CPU fallback).
"""
from __future__ import annotations

import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2204_12876_b200 as pk
from conftest import ROOT, REF_LIB


def _declared(header: Path):
    text = header.read_text()
    return set(re.findall(r"RELIEF_API[^;]*?\b(relief_\w+)\s*\(", text, flags=re.S))


def _exported(lib_path: Path):
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib_path)], capture_output=True, text=True,
                         check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_exports_match_headers(product):
    declared = _declared(ROOT / "include" / "relief.h") | _declared(ROOT / "include" / "relief_gpu.h")
    exported = _exported(Path(product._relief_path))
    assert len(_declared(ROOT / "include" / "relief.h")) == 22
    assert declared == exported, (declared ^ exported)


def test_relief_h_surface_equals_reference(product, reference):
    ours = _declared(ROOT / "include" / "relief.h")
    ref = {s for s in _exported(REF_LIB) if s.startswith("relief_")}
    assert ours == ref


def test_version_string(product, reference):
    assert product.relief_version().decode() == reference.relief_version().decode()


CONFIGS = {
    "ok_full": """map.resolution = 0.05
map.width = 120
map.height = 90
update.mahalanobis_threshold = 3
update.wall_count_threshold = 7
noise.alpha_d = 0.0002
exclusion.theta_a_deg = 30
drift.enabled = off
cleanup.alpha_n = 0.3
traversability.window = 7
traversability.weights = 0.5 0.25 0.25
overlap.radius = 0.8
sensor.ring_elevations_deg = -30 -20 -10
scene.ground = 0
scene.stairs = 1 1 0 0.1 0.2 3 1.0 +y
scene.floor2 = -2 -2 2 2 2.5 -0.5 -0.5 0.5 0.5
traj.waypoint = 0 0 0 1
traj.waypoint = 1 1 0 1 0.7071067811865476 0 0 0.7071067811865476
run.mode = par
""",
    "unknown_key": "map.width = 10\nbogus.key = 3\n",
    "bad_number": "map.resolution = abc\n",
    "trailing": "map.width = 10 20\n",
    "no_equals": "map.width 10\n",
    "bad_flag": "drift.enabled = maybe\n",
    "bad_axis": "scene.stairs = 0 0 0 0.1 0.2 3 1.0 +z\n",
    "bad_window": "traversability.window = 4\n",
    "bad_weights": "traversability.weights = 0.5 0.5 0.5\n",
    "bad_quat": "traj.waypoint = 0 0 0 1 2 0 0 0\n",
    "bad_mode": "run.mode = fast\n",
    "tiny_grid": "map.width = 2\n",
}


@pytest.mark.parametrize("name", sorted(CONFIGS))
def test_config_load_agrees_with_reference(product, reference, tmp_path, name):
    path = tmp_path / f"{name}.config"
    path.write_text(CONFIGS[name])
    outcomes = []
    for lib in (product, reference):
        h = lib.relief_config_load(str(path).encode())
        outcomes.append((bool(h), lib.relief_last_error().decode() if not h else ""))
        if h:
            assert lib.relief_config_set_mode(h, b"det") == 0
            assert lib.relief_config_set_mode(h, b"sideways") == 1
            lib.relief_config_free(h)
    assert outcomes[0] == outcomes[1]


def test_missing_files_fail_like_reference(product, reference):
    for lib in (product, reference):
        assert not lib.relief_config_load(b"/nonexistent/config")
        assert "cannot open" in lib.relief_last_error().decode()
        assert not lib.relief_map_load(b"/nonexistent/path.relief")


def test_null_arguments_are_usage_errors(product):
    pose = pk.pose34()
    assert product.relief_map_integrate(None, None, None, 0, pose.ctypes.data_as(pk._DP), 0.0, None) == 1
    assert product.relief_map_layer(None, b"elevation", None, 0) == 1
    assert product.relief_config_set_mode(None, b"det") == 1
    product.relief_map_free(None)
    product.relief_config_free(None)


def test_no_cpu_fallback_without_gpu(product):
    if product.relief_gpu_device_count() > 0:
        pytest.skip("a CUDA device is present")
    assert not product.relief_map_create(0.04, 10, 10, 0.0, 0.0)
    assert "CUDA" in product.relief_last_error().decode()


def test_invalid_geometry_rejected_before_device(product, reference):
    for lib in (product, reference):
        assert not lib.relief_map_create(-1.0, 10, 10, 0.0, 0.0)
        assert "resolution" in lib.relief_last_error().decode()
