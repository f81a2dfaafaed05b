"""Conv-net traversability cost inside the frame (C4 workload, acceptance #12's model shape:
5 x 11x11 relu + 3x3 sigmoid), and the reference's convFilterInference on the same layer.

Usage: python scripts/convnet_perf.py
"""
import ctypes, sys, tempfile, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2204_12876_b200 as pk
from paper_2204_12876_b200 import workloads as wl

tmp = Path(tempfile.mkdtemp())
rng = np.random.default_rng(99)
rows = ["layers: 6"]
for k, act in [(11, "relu")] * 5 + [(3, "sigmoid")]:
    rows.append(f"kernel: {k}")
    w = 0.05 * rng.standard_normal((k, k))
    rows += [" ".join("%.17g" % v for v in r) for r in w]
    rows += ["bias: 0.01", f"activation: {act}"]
model = tmp / "acc12.weights"
model.write_text("\n".join(rows) + "\n")

lib = pk.load_library()
w = wl.c4()
cfgp = tmp / "w.config"
cfgp.write_text(w.config_text)
cfg = pk.Config.load(lib, cfgp)
cfg.load_convnet(model)
m = pk.ReliefMap.create(lib, w.resolution, w.width, w.height)
m.set_phase_timing(True)  # per-phase split (phase events on)
calls = [w.calls(f)[0] for f in range(2)]
clouds = [pk.sim_render(lib, cfgp, c.pose, c.time, c.seed, c.scan_index) for c in calls]
names = ["transform", "drift", "update+rays", "overlap+normals", "traversability", "normals", "total"]
acc = []
for f in range(8):
    m.integrate(clouds[f % 2], calls[f % 2].pose, 0.1 * f, cfg)
    if f >= 3:
        acc.append(m.phase_seconds())
a = np.mean(np.array(acc), axis=0) * 1e3
print("C4 + conv-net phases (ms):", " ".join(f"{n}={v:.3f}" for n, v in zip(names, a)))

ref_path = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "librelief_ref.so"
if ref_path.exists():
    ref = ctypes.CDLL(str(ref_path))
    DP, U8P = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_uint8)
    ref.ref_convnet_infer.argtypes = [ctypes.c_char_p, DP, U8P, ctypes.c_int, ctypes.c_int, DP]
    L = m.layers()
    elev = np.ascontiguousarray(L["elevation"])
    valid = np.ascontiguousarray(L["valid"].astype(np.uint8))
    out = np.empty_like(elev)
    t0 = time.perf_counter()
    rc = ref.ref_convnet_infer(str(model).encode(), elev.ctypes.data_as(DP), valid.ctypes.data_as(U8P),
                               w.width, w.height, out.ctypes.data_as(DP))
    dt = time.perf_counter() - t0
    print(f"reference convFilterInference (1 core) on the same {w.width}x{w.height} layer: {dt*1e3:.1f} ms rc={rc}")
    got = pk.convnet_infer(lib, cfg, elev, valid)
    print("max |gpu - ref| =", float(np.abs(got - out).max()))
