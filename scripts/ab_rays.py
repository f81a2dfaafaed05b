"""A/B timing of the ray pass on the headline workload.

Usage: [RELIEF_B200_LIB=ab/NAME/librelief_b200.so] python scripts/ab_rays.py
Prints per-phase kernel time (mean of the last 10 frames) for the default
config and with the upper-bound / cleanup work disabled.
"""
import os, sys, tempfile
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl

lib = pk.load_library()
w = wl.ALL[os.environ.get("AB_WORKLOAD", "headline")]()
names = ["upload", "ingest", "drift", "sort", "fuse", "rays", "cells", "total"]
print("lib", os.environ.get("RELIEF_B200_LIB", "default"))
for extra in ["", "cleanup.upper_bound_enabled = false\n"]:
    p = Path(tempfile.mkdtemp()) / "w.config"; p.write_text(w.config_text + extra)
    cfg = pk.Config.load(lib, p)
    m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height)
    clouds = [pk.sim_render(lib, p, c.pose, c.time, c.seed, c.scan_index) for c in [w.calls(f)[0] for f in range(2)]]
    acc = []
    for f in range(16):
        c = w.calls(f)[0]
        m.integrate(clouds[f % 2], c.pose, 0.1 * f, cfg)
        if f >= 6:
            acc.append(m.kernel_seconds())
    a = np.mean(np.array(acc), axis=0) * 1e6
    print(repr(extra), " ".join(f"{n}={v:.1f}" for n, v in zip(names, a)), "visits", m.last_visits())
