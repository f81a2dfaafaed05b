"""Host overhead of synchronous frames across library builds.

Usage (GPU box): python scripts/host_ab.py default ab/NAME default:g ... [--workloads=C1,C4]
(suffix ":g" = relief_gpu_map_set_graphs(1), ":d" = (0) direct launches; none = the default mode)
Per build and workload, over 200 frames after 20 warm-up frames (no L2 flush): the
library's in-call wall time (ScanStats.total_seconds, its own clock around the C call),
the device time of the frame (kernel_seconds()[7], events on the library stream) and
their difference, for device-resident input (relief_gpu_map_integrate_device) and for
pinned host input (relief_map_integrate, device time then includes the upload).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys, tempfile, statistics, time
from pathlib import Path
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl
lib = pk.load_library()
out = {}
for name in WL:
    w = wl.ALL[name]()
    p = Path(tempfile.mkdtemp()) / "w.config"; p.write_text(w.config_text)
    cfg = pk.Config.load(lib, p)
    c = w.calls(0)[0]
    host = pk.sim_render(lib, p, c.pose, c.time, c.seed, c.scan_index)
    dev = torch.from_numpy(host).cuda()
    pin = torch.from_numpy(host).pin_memory().numpy()
    torch.cuda.synchronize()
    res = {}
    for leg in ("device", "pinned"):
        m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height)
        if GRAPHS is not None:
            m.set_graphs(GRAPHS)
        inc, devt, wall = [], [], []
        for s in range(220):
            t0 = time.perf_counter()
            if leg == "device":
                st = m.integrate_device(dev.data_ptr(), dev.shape[0], c.pose, 0.1 * s, cfg)
            else:
                st = m.integrate(pin, c.pose, 0.1 * s, cfg)
            t1 = time.perf_counter()
            ks = m.kernel_seconds()
            if s >= 20:
                wall.append(t1 - t0)
                inc.append(st.total_seconds)
                devt.append(ks[7] + (ks[0] if leg == "pinned" else 0.0))
        med = lambda v: statistics.median(v) * 1e6
        res[leg] = {"python_wall_us": med(wall), "in_call_us": med(inc), "device_us": med(devt),
                    "overhead_us": statistics.median([a - b for a, b in zip(inc, devt)]) * 1e6}
    out[name] = res
print("RESULT" + json.dumps(out))
'''


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    wl = "C1,C4"
    for a in sys.argv[1:]:
        if a.startswith("--workloads="):
            wl = a.split("=", 1)[1]
    for rnd in range(2):
        for v in args:
            env = dict(os.environ)
            lib, _, opt = v.partition(":")
            if lib != "default":
                env["RELIEF_B200_LIB"] = os.path.join(ROOT, lib, "librelief_b200.so")
            code = CHILD.replace("ROOT", repr(ROOT), 1).replace("WL", repr(wl.split(",")), 1)
            code = code.replace("GRAPHS", {"g": "1", "d": "0"}.get(opt, "None"))
            r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
            diag = [l for l in r.stderr.splitlines() if l.startswith("HOSTDIAG")]
            line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")]
            if not line:
                print(v, "FAILED", r.stderr[-2000:])
                continue
            for k, legs in json.loads(line[0][6:]).items():
                for leg, x in legs.items():
                    print(f"r{rnd} {k:9s} {v:16s} {leg:7s} in-call {x['in_call_us']:8.1f} us  device "
                          f"{x['device_us']:8.1f}  overhead {x['overhead_us']:6.1f}  python wall "
                          f"{x['python_wall_us']:8.1f}")
            for d in diag[-6:]:
                print("   ", v, d)


if __name__ == "__main__":
    main()
