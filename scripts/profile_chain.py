"""Builds a C4-sized map then runs the C5 chain a few times (ncu target; dev aid)."""
import sys, tempfile
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl
lib = pk.load_library()
w = wl.ALL[sys.argv[1] if len(sys.argv) > 1 else "C4"]()
p = Path(tempfile.mkdtemp()) / "w.config"; p.write_text(w.config_text)
cfg = pk.Config.load(lib, p)
m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height)
for f in range(2):
    for c in w.calls(f):
        m.integrate(pk.sim_render(lib, p, c.pose, c.time, c.seed, c.scan_index), c.pose, 0.1 * f, cfg)
ts = []
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    v, ok = m.smooth_chain("elevation", wl.C5_CHAIN)
    ts.append(lib.relief_gpu_map_chain_seconds(m.handle) * 1e3)
print("chain ms", " ".join(f"{t:.4f}" for t in ts[:3]), "median", f"{np.median(ts[1:] or ts):.4f}")
