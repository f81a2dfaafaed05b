"""Where the e2e time of relief_map_integrate goes (C4, pinned host input).

Prints per call: host wall, device upload (H2D, ev0->ev1), device compute (ev1->end)."""
import sys, time, tempfile
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl

lib = pk.load_library()
w = wl.c4()
p = Path(tempfile.mkdtemp()) / "w.config"
p.write_text(w.config_text)
cfg = pk.Config.load(lib, p)
m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height)
calls = [w.calls(f)[0] for f in range(2)]
frames = [torch.from_numpy(pk.sim_render(lib, p, c.pose, c.time, c.seed, c.scan_index)).pin_memory() for c in calls]
walls, ks = [], []
for s in range(12):
    c = calls[s % 2]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m.integrate(frames[s % 2], c.pose, 0.1 * s, cfg)
    walls.append(time.perf_counter() - t0)
    ks.append(m.kernel_seconds())
walls = np.array(walls[4:]) * 1e3
k = np.array(ks[4:]) * 1e3
print(f"wall {walls.mean():.3f} ms  upload(H2D) {k[:,0].mean():.3f}  compute {k[:,7].mean():.3f}  "
      f"unaccounted {walls.mean() - k[:,0].mean() - k[:,7].mean():.3f}")
