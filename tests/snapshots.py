"""Builds reliefmap snapshot text (format of reference snapshot.cpp:79-120) from numpy layers,
so tests can load an exact map state into any library through relief_map_load."""
from __future__ import annotations

import numpy as np

LAYERS = ("elevation", "variance", "last_update", "upper_bound", "upper_bound_valid",
          "traversability", "normal_x", "normal_y", "normal_z", "valid")


def _fmt(v: float) -> str:
    if np.isnan(v):
        return "nan"
    return "%.17g" % v


def fresh(H: int, W: int) -> dict:
    z = np.zeros((H, W))
    return {"elevation": np.full((H, W), np.nan), "variance": np.full((H, W), np.nan),
            "last_update": z.copy(), "upper_bound": np.full((H, W), np.nan),
            "upper_bound_valid": z.copy(), "traversability": z.copy(), "normal_x": z.copy(),
            "normal_y": z.copy(), "normal_z": z.copy(), "valid": z.copy()}


def set_cell(layers: dict, r: int, c: int, h: float, var: float, stamp: float = 0.0,
             normal=(0.0, 0.0, 0.0), trav: float = 0.0) -> None:
    """A valid cell with an estimate (its bound equals the estimate, grid.cpp:139-147)."""
    layers["elevation"][r, c] = h
    layers["variance"][r, c] = var
    layers["last_update"][r, c] = stamp
    layers["upper_bound"][r, c] = h
    layers["upper_bound_valid"][r, c] = 1.0
    layers["valid"][r, c] = 1.0
    layers["normal_x"][r, c], layers["normal_y"][r, c], layers["normal_z"][r, c] = normal
    layers["traversability"][r, c] = trav


def text(layers: dict, resolution: float, center=(0.0, 0.0)) -> str:
    H, W = layers["valid"].shape
    out = ["reliefmap-snapshot v1", f"resolution: {_fmt(resolution)}", f"width: {W}", f"height: {H}",
           f"center_x: {_fmt(center[0])}", f"center_y: {_fmt(center[1])}", "layers: " + ",".join(LAYERS)]
    valid = layers["valid"] != 0
    ubv = layers["upper_bound_valid"] != 0
    for name in LAYERS:
        a = np.array(layers[name], dtype=np.float64)
        if name in ("elevation", "variance", "last_update", "traversability", "normal_x", "normal_y",
                    "normal_z"):
            a = np.where(valid, a, np.nan)
        elif name == "upper_bound":
            a = np.where(ubv, a, np.nan)
        out.append("layer: " + name)
        for r in range(H):
            out.append(" ".join(_fmt(v) for v in a[r]))
    return "\n".join(out) + "\n"
