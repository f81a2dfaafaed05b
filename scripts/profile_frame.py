"""Runs `warm` untimed frames of a workload then `frames` more, for ncu capture
(development aid). Kernel launches per frame: see relief_gpu_map_last_launches."""
from __future__ import annotations

import sys
import tempfile
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2204_12876_b200 as pk  # noqa: E402
from paper_2204_12876_b200 import workloads as wl  # noqa: E402


def main(name: str = "headline", warm: int = 3, frames: int = 1, distinct: int = 2) -> None:
    lib = pk.load_library()
    w = wl.ALL[name]()
    d = Path(tempfile.mkdtemp())
    cfgp = d / "w.config"
    cfgp.write_text(w.config_text)
    cfg = pk.Config.load(lib, cfgp)
    m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height)
    clouds = [[(pk.sim_render(lib, cfgp, c.pose, c.time, c.seed, c.scan_index), c) for c in w.calls(f)]
              for f in range(distinct)]
    for f in range(warm + frames):
        for xyz, c in clouds[f % distinct]:
            m.integrate(xyz, c.pose, 0.1 * f, cfg)
    print("launches/frame", m.last_launches(), "kernel_seconds", list(m.kernel_seconds()))


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "headline", int(a[1]) if len(a) > 1 else 3, int(a[2]) if len(a) > 2 else 1,
         int(a[3]) if len(a) > 3 else 2)
