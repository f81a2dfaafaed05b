"""Post-processing chain timings on a mapped C4 elevation layer (C5 chain and single steps).
Usage: [RELIEF_B200_LIB=...] python scripts/chain_ab.py"""
import sys, os, tempfile, statistics
from pathlib import Path
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl
lib = pk.load_library()
w = wl.c4()
p = Path(tempfile.mkdtemp())/"w.config"; p.write_text(w.config_text)
cfg = pk.Config.load(lib, p)
m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height)
for f in range(3):
    c = w.calls(f)[0]
    m.integrate(pk.sim_render(lib, p, c.pose, c.time, c.seed, c.scan_index), c.pose, c.stamp, cfg)
cells = w.width * w.height
dv = torch.empty(cells, dtype=torch.float64, device="cuda"); do = torch.empty(cells, dtype=torch.uint8, device="cuda")
for chain, name in [(wl.C5_CHAIN, "C5"), ([(2, 1, 1.0)], "median r1"), ([(0, 2, 1.0)], "gauss r2"), ([(1, 1, 1.0)], "box r1"), ([(2, 2, 1.0)], "median r2"), ([(0, 3, 1.5)], "gauss r3")]:
    t = [m.smooth_chain_device("elevation", chain, dv.data_ptr(), do.data_ptr()) for _ in range(12)]
    print(os.environ.get("RELIEF_B200_LIB", "default")[:12], name, f"{statistics.median(t[2:]) * 1e6:.1f} us")
