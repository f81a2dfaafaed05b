import sys, time, tempfile, threading
from pathlib import Path
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl
lib = pk.load_library()
w = wl.c4()
p = Path(tempfile.mkdtemp()) / "w.config"; p.write_text(w.config_text)
cfg = pk.Config.load(lib, p)
m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height)
c = w.calls(0)[0]
x = torch.from_numpy(pk.sim_render(lib, p, c.pose, c.time, c.seed, c.scan_index)).cuda()
host = torch.empty(x.numel(), dtype=torch.float64).pin_memory()
dev = torch.empty_like(x)
cs = torch.cuda.Stream()
def compute(nf):
    ks = []
    for s in range(nf):
        m.integrate_device(x.data_ptr(), x.numel() // 3, c.pose, 0.1 * s, cfg)
        ks.append(m.kernel_seconds()[7])
    return np.mean(ks[2:]) * 1e3
print("compute alone ms/frame", compute(12))
# concurrent copies
stop = False
def copier():
    with torch.cuda.stream(cs):
        while not stop:
            dev.view(-1).copy_(host, non_blocking=True)
            cs.synchronize()
t = threading.Thread(target=copier); t.start()
time.sleep(0.05)
print("compute with concurrent H2D ms/frame", compute(12))
stop = True; t.join()
torch.cuda.synchronize()
# copy alone
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(cs):
    ev0.record(cs)
    for _ in range(10): dev.view(-1).copy_(host, non_blocking=True)
    ev1.record(cs)
cs.synchronize()
print("copy alone ms", ev0.elapsed_time(ev1) / 10)
