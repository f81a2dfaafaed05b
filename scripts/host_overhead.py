import sys, time, tempfile
from pathlib import Path
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl
lib = pk.load_library()
w = wl.c4()
p = Path(tempfile.mkdtemp())/"w.config"; p.write_text(w.config_text)
cfg = pk.Config.load(lib, p)
m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height)
c = w.calls(0)[0]
empty = np.zeros((0, 3))
small = torch.from_numpy(pk.sim_render(lib, p, c.pose, c.time, c.seed, c.scan_index)[:1000].copy()).pin_memory().numpy()
full = torch.from_numpy(pk.sim_render(lib, p, c.pose, c.time, c.seed, c.scan_index)).pin_memory().numpy()
for name, x in [("empty", empty), ("1k", small), ("full", full)]:
    ws, ks = [], []
    for s in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); m.integrate(x, c.pose, 0.1 * s, cfg); ws.append(time.perf_counter() - t0)
        ks.append(m.kernel_seconds())
    ws = np.array(ws[5:]) * 1e6; k = np.array(ks[5:]) * 1e6
    print(f"{name}: wall {ws.mean():.1f} us (min {ws.min():.1f})  upload {k[:,0].mean():.1f}  device total {k[:,7].mean():.1f}")
