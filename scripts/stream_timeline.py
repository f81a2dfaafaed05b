"""Host-side timeline of the streaming API on C4: enqueue and wait durations per frame."""
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
frames = [torch.from_numpy(pk.sim_render(lib, p, c.pose, c.time, c.seed, c.scan_index)).pin_memory().numpy()
          for c in calls]
for s in range(4):
    m.integrate(frames[s % 2], calls[s % 2].pose, 0.1 * s, cfg)
torch.cuda.synchronize()
enq, wt, ks = [], [], []
t_start = time.perf_counter()
pending = 0
for s in range(4, 24):
    t0 = time.perf_counter()
    m.integrate_async(frames[s % 2], calls[s % 2].pose, 0.1 * s, cfg)
    enq.append(time.perf_counter() - t0)
    pending += 1
    if pending == 3:
        t0 = time.perf_counter()
        m.wait()
        wt.append(time.perf_counter() - t0)
        ks.append(m.kernel_seconds())
        pending -= 1
while pending:
    m.wait()
    pending -= 1
total = time.perf_counter() - t_start
print(f"per frame {total / 20 * 1e3:.3f} ms; enqueue mean {np.mean(enq)*1e6:.0f} us (max {np.max(enq)*1e6:.0f}); "
      f"wait mean {np.mean(wt)*1e6:.0f} us; device copy {np.mean([k[0] for k in ks])*1e3:.3f} ms, "
      f"frame kernels {np.mean([k[7] for k in ks])*1e3:.3f} ms")
