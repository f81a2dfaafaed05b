"""e2e wall time of relief_map_integrate on C4 from pinned memory (median / mean / min over ITERS calls),
with the upload / post-copy device split. Usage: [RELIEF_B200_LIB=...] [ITERS=N] python scripts/e2e_ab.py"""
import sys, time, tempfile, os
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
calls = [w.calls(f)[0] for f in range(4)]
fr = [torch.from_numpy(pk.sim_render(lib, p, c.pose, c.time, c.seed, c.scan_index)).pin_memory().numpy() for c in calls]
ws, ks = [], []
for s in range(int(os.environ.get("ITERS", "40"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); m.integrate(fr[s % 4], calls[s % 4].pose, 0.1 * s, cfg); ws.append(time.perf_counter() - t0)
    ks.append(m.kernel_seconds())
ws = np.array(ws[8:]) * 1e6; k = np.array(ks[8:]) * 1e6
print(os.environ.get("RELIEF_B200_LIB", "default"), f"wall median {np.median(ws):.1f} mean {ws.mean():.1f} min {ws.min():.1f} | upload {k[:,0].mean():.1f} ingest {k[:,1].mean():.1f} device {k[:,7].mean():.1f}")
