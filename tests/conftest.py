"""Shared fixtures.

Libraries involved:
  * product   -- paper_2204_12876_b200/lib/librelief_b200.so (the thing under test)
  * reference -- oracle/_ref/librelief_ref.so: the reliefmap reference compiled in place
                 from /root/reference with oracle/Makefile (TEST INFRASTRUCTURE; built in the
                 dev container and shipped to the GPU box with the repo snapshot)
  * restate   -- oracle/_build/liboracle.so: the C restatement of the reference path
Only tests (and smoke()/bench.py's CPU legs) touch the oracle libraries.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

REF_LIB = ROOT / "oracle" / "_ref" / "librelief_ref.so"
RESTATE_LIB = ROOT / "oracle" / "_build" / "liboracle.so"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _cuda_available() -> bool:
    try:
        import paper_2204_12876_b200 as pk
        lib = pk.load_library()
        return lib.relief_gpu_device_count() > 0
    except Exception:
        return False


@pytest.fixture(scope="session")
def product():
    import paper_2204_12876_b200 as pk
    from paper_2204_12876_b200 import build as b
    b.build()
    return pk.load_library()


@pytest.fixture(scope="session")
def gpu(product):
    if product.relief_gpu_device_count() <= 0:
        pytest.fail("no CUDA device visible: GPU tests must run on a B200 box (no CPU fallback)")
    return product


@pytest.fixture(scope="session")
def reference():
    if not REF_LIB.exists():
        if Path("/root/reference/proj").exists():
            subprocess.run(["make", "-C", str(ROOT / "oracle"), "ref", "-j8"], check=True,
                           capture_output=True)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    import paper_2204_12876_b200 as pk
    lib = pk.load_library(REF_LIB, gpu_api=False)
    # reference-only extras (oracle/ref_extras.cpp)
    D, DP, I = ctypes.c_double, ctypes.POINTER(ctypes.c_double), ctypes.c_int
    lib.ref_last_error.restype = ctypes.c_char_p
    lib.ref_render_scan.restype = ctypes.c_int64
    lib.ref_render_scan.argtypes = [ctypes.c_char_p, DP, D, ctypes.c_uint64, ctypes.c_uint64, DP,
                                    ctypes.c_int64]
    lib.ref_traverse_cells.restype = ctypes.c_int64
    lib.ref_traverse_cells.argtypes = [DP, DP, D, I, I, D, D, ctypes.POINTER(ctypes.c_int32),
                                       ctypes.POINTER(ctypes.c_int32), DP, ctypes.c_int64]
    lib.ref_kalman_update.restype = I
    lib.ref_kalman_update.argtypes = [D, D, D, D, I, D, D, I, D, DP, DP]
    lib.ref_smooth_chain.restype = I
    lib.ref_smooth_chain.argtypes = [DP, ctypes.POINTER(ctypes.c_uint8), I, I, ctypes.POINTER(I),
                                     ctypes.POINTER(I), DP, I, DP, ctypes.POINTER(ctypes.c_uint8)]
    return lib


def ref_render(reference, config_path, pose, time, seed, scan_index, capacity=1 << 21):
    pose = np.ascontiguousarray(pose, dtype=np.float64)
    buf = np.empty(capacity * 3)
    n = reference.ref_render_scan(str(config_path).encode(), pose.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                  time, seed, scan_index, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                  capacity)
    assert n >= 0, reference.ref_last_error()
    if n > capacity:
        return ref_render(reference, config_path, pose, time, seed, scan_index, capacity=n)
    return buf[: 3 * n].reshape(n, 3).copy()


# ------------------------------------------------------------ comparison helpers
BIT_EXACT_LAYERS = ("elevation", "variance", "last_update", "upper_bound", "upper_bound_valid",
                    "normal_x", "normal_y", "normal_z", "valid")


def bits_equal(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Elementwise bit equality, any NaN equal to any NaN."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    same = a.view(np.uint64) == b.view(np.uint64)
    return same | (np.isnan(a) & np.isnan(b))


def assert_layers_match(got: dict, want: dict, tol_trav: float = 1e-12, height_tol: float = 0.0,
                        context: str = "") -> None:
    """Parity bar: bit-exact layers, traversability within tol_trav (device acos vs libm acos).

    height_tol > 0 relaxes elevation / upper_bound / variance to |d| <= tol (abs and rel)
    for runs whose drift offset is a parallel sum.
    """
    for name in BIT_EXACT_LAYERS:
        g, w = got[name], want[name]
        assert g.shape == w.shape, (name, g.shape, w.shape)
        if height_tol > 0 and name in ("elevation", "upper_bound", "variance", "normal_x", "normal_y",
                                       "normal_z"):
            nan_ok = np.isnan(g) == np.isnan(w)
            assert nan_ok.all(), f"{context} {name}: NaN masks differ at {np.argwhere(~nan_ok)[:5]}"
            fin = np.isfinite(w) & np.isfinite(g)
            d = np.abs(g[fin] - w[fin])
            lim = height_tol * np.maximum(1.0, np.abs(w[fin]))
            assert (d <= lim).all(), f"{context} {name}: max diff {d.max()}"
            inf_ok = (np.isinf(g) == np.isinf(w))
            assert inf_ok.all(), f"{context} {name}: inf masks differ"
            continue
        eq = bits_equal(g, w)
        if not eq.all():
            idx = np.argwhere(~eq)
            r, c = idx[0]
            raise AssertionError(
                f"{context} layer {name}: {len(idx)} cells differ; first ({r},{c}) got {g[r, c]!r} "
                f"want {w[r, c]!r}")
    g, w = got["traversability"], want["traversability"]
    assert (np.isnan(g) == np.isnan(w)).all(), f"{context} traversability NaN masks differ"
    fin = ~np.isnan(w)
    if fin.any():
        d = np.abs(g[fin] - w[fin])
        # a height difference of height_tol moves window statistics / slopes by O(height_tol/res)
        lim = max(tol_trav, 1e3 * height_tol)
        assert d.max() <= lim, f"{context} traversability max diff {d.max()}"


STAT_INT_FIELDS = ("points_in", "points_excluded", "points_out_of_range", "points_out_of_map",
                   "points_rejected_outlier", "points_ignored_low", "points_fused", "cells_updated",
                   "cells_removed_by_cleanup", "cells_cleared_by_overlap")


def assert_stats_match(got, want, drift_tol: float = 0.0, context: str = "") -> None:
    for f in STAT_INT_FIELDS:
        assert getattr(got, f) == getattr(want, f), f"{context} {f}: got {getattr(got, f)} want {getattr(want, f)}"
    gd, wd = got.drift_offset_applied, want.drift_offset_applied
    if drift_tol == 0.0:
        assert gd == wd, f"{context} drift offset {gd!r} vs {wd!r}"
    else:
        assert abs(gd - wd) <= drift_tol, f"{context} drift offset {gd!r} vs {wd!r}"
