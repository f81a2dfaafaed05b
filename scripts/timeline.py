"""Device timeline of a steady-state frame from a RB_TIMELINE build.

Usage (GPU box): python scripts/build_variant.py tl -DRB_TIMELINE=1   (here)
                 python scripts/timeline.py [C4] [frames=40] [graphs]  (GPU box)
Runs the workload's synchronous frames (device-resident input, as scripts/ab_frame.py) through ab/tl/librelief_b200.so; that
build prints, after each frame, the first block start and last block end
(%globaltimer) of every kernel slot. Prints the median over the last 10
frames of each slot's [start, end] relative to the ingest's start, in us.
"""
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SLOTS = ["shift", "ingest", "sort rowscan (both)", "sort scatter 0", "sort scatter 1", "drift vote (s2)",
         "side sweep / offset (s2)", "short fold", "long fold (s2)", "long fold: warp-per-cell end", "long fold: lane-per-cell end",
         "jump grid", "ray pass 1", "ray pass 1 retry", "ray tail", "cells"]

CHILD = r'''
import sys, tempfile
from pathlib import Path
sys.path.insert(0, ROOT)
import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl
lib = pk.load_library()
w = wl.ALL[NAME]()
p = Path(tempfile.mkdtemp()) / "w.config"; p.write_text(w.config_text)
cfg = pk.Config.load(lib, p)
m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height)
if GRAPHS >= 0:
    m.set_graphs(GRAPHS)
import torch
frames = [[(c, torch.from_numpy(pk.sim_render(lib, p, c.pose, c.time, c.seed, c.scan_index)).cuda())
           for c in w.calls(f)] for f in range(8)]
for s in range(FRAMES):
    for c, t in frames[s % len(frames)]:
        m.integrate_device(t.data_ptr(), t.shape[0], c.pose, 0.1 * s, cfg)
'''


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    lib = os.environ.get("TL_BUILD", "tl")  # ab/<TL_BUILD>: any RB_TIMELINE build
    env = dict(os.environ, RELIEF_B200_LIB=os.path.join(ROOT, "ab", lib, "librelief_b200.so"))
    graphs = int(sys.argv[3]) if len(sys.argv) > 3 else -1  # relief_gpu_map_set_graphs mode (-1: default)
    code = CHILD.replace("ROOT", repr(ROOT), 1).replace("NAME", repr(name)).replace("FRAMES", str(frames))
    code = code.replace("GRAPHS", str(graphs))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
    lines = [l.split()[1:] for l in r.stderr.splitlines() if l.startswith("TL ")]
    if not lines:
        print("no timeline lines", r.stderr[-3000:])
        return
    rows = []
    for l in lines[-10:]:
        v = [int(x) for x in l]
        t0 = v[2]  # ingest start
        # (slots recorded at their end only have no start: shown as starting at their end)
        rows.append([((v[2 * k] if v[2 * k] != 2**64 - 1 else v[2 * k + 1]) - t0, v[2 * k + 1] - t0)
                     if v[2 * k + 1] else None for k in range(len(SLOTS))])
    print(f"{name}: median over the last {len(rows)} frames (us from the ingest start)")
    counts = [l for l in r.stderr.splitlines() if l.startswith("TLC ")]
    if counts:
        print("  last frame's lists:", counts[-1][4:])
    for k, label in enumerate(SLOTS):
        vals = [r[k] for r in rows if r[k] is not None]
        if not vals:
            continue
        a = statistics.median(v[0] for v in vals) / 1e3
        b = statistics.median(v[1] for v in vals) / 1e3
        print(f"  {label:28s} {a:8.1f} {b:8.1f}  ({b - a:6.1f})")


if __name__ == "__main__":
    main()
