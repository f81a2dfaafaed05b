"""Device time per frame of the first 12 frames of a fresh map (C4, headline): the map's transient
(frame 0 also pays the lazy loading of the kernels). Usage (GPU box): python scripts/first_frames.py"""
import sys, tempfile
sys.path.insert(0, '/root/repo')
from pathlib import Path
import torch, paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl
lib = pk.load_library()
for name in ["C4", "headline"]:
    w = wl.ALL[name]()
    p = Path(tempfile.mkdtemp())/"w.config"; p.write_text(w.config_text)
    cfg = pk.Config.load(lib, p)
    frames = [[(torch.from_numpy(pk.sim_render(lib, p, c.pose, c.time, c.seed, c.scan_index)).cuda(), c) for c in w.calls(f)] for f in range(8)]
    m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height)
    out = []
    for s in range(12):
        for t, c in frames[s % 8]:
            m.integrate_device(t.data_ptr(), t.shape[0], c.pose, 0.1 * s, cfg)
            out.append(m.kernel_seconds()[7] * 1e3)
    print(name, " ".join(f"{x:.3f}" for x in out))
