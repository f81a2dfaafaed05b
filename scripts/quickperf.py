"""Quick per-kernel timing of the product on a workload (development aid, not the bench)."""
from __future__ import annotations

import sys
import tempfile
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2204_12876_b200 as pk  # noqa: E402
from paper_2204_12876_b200 import workloads as wl  # noqa: E402

LABELS = ("upload", "ingest", "drift", "sort", "fuse", "rays", "cells", "total")


def main(name: str = "headline", frames: int = 6) -> None:
    lib = pk.load_library()
    w = wl.ALL[name]()
    d = Path(tempfile.mkdtemp())
    cfgp = d / "w.config"
    cfgp.write_text(w.config_text)
    cfg = pk.Config.load(lib, cfgp)
    m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height)
    t0 = time.time()
    clouds = []
    for f in range(min(frames, 3)):
        clouds.append([(pk.sim_render(lib, cfgp, c.pose, c.time, c.seed, c.scan_index), c) for c in w.calls(f)])
    print(f"{name}: rendered {sum(len(x) for x, _ in clouds[0])} pts/frame in {time.time() - t0:.2f}s", flush=True)
    for f in range(frames):
        calls = clouds[f % len(clouds)]
        t = time.perf_counter()
        tot = np.zeros(8)
        for xyz, c in calls:
            st = m.integrate(xyz, c.pose, 0.1 * f, cfg)
            tot += m.kernel_seconds()
        wall = time.perf_counter() - t
        npts = sum(len(x) for x, _ in calls)
        parts = " ".join(f"{l} {v * 1e6:.0f}" for l, v in zip(LABELS, tot))
        print(f"frame {f}: wall {wall * 1e3:.2f} ms | us: {parts} | {npts / tot[7] / 1e9:.2f} Gpts/s device "
              f"| launches {m.last_launches()} fused {st.points_fused} removed {st.cells_removed_by_cleanup}",
              flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["headline"]), *([int(sys.argv[2])] if len(sys.argv) > 2 else []))
