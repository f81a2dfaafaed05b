"""A/B of whole-frame device time across library builds (no phase events, L2 flushed per frame).

Usage (GPU box): python scripts/ab_frame.py default ab/NAME ... [--workloads C4,headline,C3,C1]
Prints, per build and workload, the median device ms per frame over the last 20 of AB_FRAMES
frames (default 25) and the stats of the last frame (which must agree across builds).
"""
import os
import statistics
import subprocess
import sys
import json

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, os, sys, tempfile, statistics
from pathlib import Path
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl
lib = pk.load_library()
out = {}
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for name in WL:
    w = wl.ALL[name]()
    p = Path(tempfile.mkdtemp()) / "w.config"; p.write_text(w.config_text)
    cfg = pk.Config.load(lib, p)
    frames = [[(torch.from_numpy(pk.sim_render(lib, p, c.pose, c.time, c.seed, c.scan_index)).cuda(), c)
               for c in w.calls(f)] for f in range(8)]
    torch.cuda.synchronize()
    m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height)
    ts = []
    for s in range(NFR):
        flush.zero_(); torch.cuda.synchronize()
        dev = 0.0
        for t, c in frames[s % 8]:
            st = m.integrate_device(t.data_ptr(), t.shape[0], c.pose, 0.1 * s, cfg)
            dev += m.kernel_seconds()[7]
        if s >= NFR - 20:
            ts.append(dev)
    out[name] = {"ms": statistics.median(ts) * 1e3, "min": min(ts) * 1e3,
                 "stats": [st.points_fused, st.cells_updated, st.cells_removed_by_cleanup, st.points_rejected_outlier]}
print("RESULT" + json.dumps(out))
'''


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    wl = "C4,headline,C3,C1"
    for a in sys.argv[1:]:
        if a.startswith("--workloads="):
            wl = a.split("=", 1)[1]
    res = {}
    for rnd in range(2):  # interleaved rounds
        for v in args:
            env = dict(os.environ)
            if v != "default":
                env["RELIEF_B200_LIB"] = os.path.join(ROOT, v, "librelief_b200.so")
            code = CHILD.replace("ROOT", repr(ROOT), 1).replace("WL", repr(wl.split(",")), 1)
            code = code.replace("NFR", os.environ.get("AB_FRAMES", "25"))  # median over the last 20
            r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
            if os.environ.get("AB_DUMP"):  # keep the child's output (e.g. a diag build's counters)
                with open(os.environ["AB_DUMP"], "a") as fh:
                    fh.write(f"== {v} round {rnd}\n" + r.stdout)
            line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
            if not line:
                print(v, "FAILED", r.stderr[-2000:])
                continue
            d = json.loads(line[0][6:])
            for k, x in d.items():
                res.setdefault((v, k), []).append(x)
    for (v, k), xs in sorted(res.items(), key=lambda t: (t[0][1], t[0][0])):
        print(f"{k:9s} {v:24s} ms/frame " + " ".join(f"{x['ms']:.4f}" for x in xs) + f"  stats {xs[-1]['stats']}")


if __name__ == "__main__":
    main()
