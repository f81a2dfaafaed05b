"""Conv-net traversability (reference analysis.cpp:138-290, runner.cpp:53-60).

CPU: the C restatement (oracle/relief_oracle.c) against the reference compiled in place, the
reference's own known-answer cases, and the weight-file reader of the product (host code) against
the reference's reader. GPU: relief_gpu_convnet_infer and the whole pipeline through the runners
against the reference.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np
import pytest

from conftest import RESTATE_LIB, assert_layers_match

DP = ctypes.POINTER(ctypes.c_double)
U8P = ctypes.POINTER(ctypes.c_uint8)
IP = ctypes.POINTER(ctypes.c_int)
ACTS = {"relu": 0, "sigmoid": 1, "identity": 2}
# reference ErrorCode (types.hpp:34-45) -> relief_status (capi.cpp:43-58)
CODE_TO_STATUS = {0: 3, 1: 4, 2: 5, 3: 6, 4: 7, 5: 8, 6: 9, 7: 10, 8: 11, 9: 1}


def model_text(layers) -> str:
    """layers: (k, weights[k*k], bias, activation) tuples -> weight-file text (%.17g)."""
    out = [f"layers: {len(layers)}"]
    for k, w, b, act in layers:
        w = np.asarray(w, dtype=np.float64).reshape(k, k)
        out.append(f"# layer\nkernel: {k}")
        out += [" ".join("%.17g" % v for v in row) for row in w]
        out += ["bias: %.17g" % b, f"activation: {act}"]
    return "\n".join(out) + "\n"


def random_model(rng, n_layers, sizes=(1, 3, 5), acts=("relu", "sigmoid", "identity"), scale=0.4):
    layers = []
    for _ in range(n_layers):
        k = int(rng.choice(sizes))
        layers.append((k, scale * rng.standard_normal(k * k), 0.2 * rng.standard_normal(),
                       str(rng.choice(acts))))
    return layers


def random_layer(rng, H, W, p_valid):
    layer = rng.standard_normal((H, W))
    valid = (rng.random((H, W)) < p_valid).astype(np.uint8)
    layer[valid == 0] = np.nan  # the map's invalid cells carry NaN elevation
    return layer, valid


@pytest.fixture(scope="module")
def refcn(reference):
    reference.ref_convnet_infer.restype = ctypes.c_int
    reference.ref_convnet_infer.argtypes = [ctypes.c_char_p, DP, U8P, ctypes.c_int, ctypes.c_int, DP]
    return reference


@pytest.fixture(scope="module")
def restate():
    if not RESTATE_LIB.exists():
        pytest.skip("oracle/_build/liboracle.so not built")
    lib = ctypes.CDLL(str(RESTATE_LIB))
    lib.oracle_convnet_infer.restype = ctypes.c_int
    lib.oracle_convnet_infer.argtypes = [ctypes.c_int, IP, DP, DP, IP, DP, U8P, ctypes.c_int, ctypes.c_int,
                                         DP]
    lib.relief_last_error.restype = ctypes.c_char_p
    return lib


def ref_infer(refcn, model_path, layer, valid):
    layer = np.ascontiguousarray(layer, dtype=np.float64)
    valid = np.ascontiguousarray(valid, dtype=np.uint8)
    H, W = layer.shape
    out = np.empty_like(layer)
    rc = refcn.ref_convnet_infer(str(model_path).encode(), layer.ctypes.data_as(DP),
                                 valid.ctypes.data_as(U8P), W, H, out.ctypes.data_as(DP))
    return rc, out, refcn.ref_last_error().decode()


def restate_infer(lib, layers, layer, valid):
    layer = np.ascontiguousarray(layer, dtype=np.float64)
    valid = np.ascontiguousarray(valid, dtype=np.uint8)
    H, W = layer.shape
    n = len(layers)
    ks = (ctypes.c_int * n)(*[l[0] for l in layers])
    ws = np.ascontiguousarray(np.concatenate([np.asarray(l[1], dtype=np.float64).ravel() for l in layers]))
    bs = (ctypes.c_double * n)(*[float(l[2]) for l in layers])
    acts = (ctypes.c_int * n)(*[ACTS[l[3]] for l in layers])
    out = np.empty_like(layer)
    rc = lib.oracle_convnet_infer(n, ks, ws.ctypes.data_as(DP), bs, acts, layer.ctypes.data_as(DP),
                                  valid.ctypes.data_as(U8P), W, H, out.ctypes.data_as(DP))
    assert rc == 0, lib.relief_last_error()
    return out


def same_bits(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint64), np.ascontiguousarray(b).view(np.uint64))


# ----------------------------------------------------------------- CPU: oracle pinning
@pytest.mark.parametrize("seed", range(12))
def test_restatement_matches_reference(refcn, restate, tmp_path, seed):
    rng = np.random.default_rng(1000 + seed)
    H, W = int(rng.integers(3, 40)), int(rng.integers(3, 40))
    p_valid = [0.0, 0.02, 0.3, 0.9, 1.0][seed % 5]
    layer, valid = random_layer(rng, H, W, p_valid)
    layers = random_model(rng, 1 + seed % 3)
    path = tmp_path / "m.weights"
    path.write_text(model_text(layers))
    rc, want, err = ref_infer(refcn, path, layer, valid)
    assert rc == 0, err
    got = restate_infer(restate, layers, layer, valid)
    assert same_bits(got, want)


def test_fill_ties_follow_bfs_queue_order(refcn, restate, tmp_path):
    """Sparse sources with many equidistant cells: the value a hole takes is decided by the
    BFS queue order; identity model exposes the fill itself."""
    rng = np.random.default_rng(7)
    H, W = 37, 41
    valid = np.zeros((H, W), np.uint8)
    for r, c in [(0, 0), (0, 40), (36, 0), (36, 40), (18, 20), (5, 9), (5, 11), (30, 30), (30, 32)]:
        valid[r, c] = 1
    layer = np.where(valid == 1, rng.standard_normal((H, W)), np.nan)
    layers = [(1, [1.0], 0.0, "identity")]
    path = tmp_path / "id.weights"
    path.write_text(model_text(layers))
    rc, want, err = ref_infer(refcn, path, layer * 0.1 + 0.5, valid)
    assert rc == 0, err
    got = restate_infer(restate, layers, layer * 0.1 + 0.5, valid)
    assert same_bits(got, want)


# Reference known-answer cases (test_analysis.cpp:146-184).
def test_known_answers_reference_tests(refcn, restate, tmp_path):
    rng = np.random.default_rng(3)
    n = 8
    layer = rng.random((n, n))
    valid = np.ones((n, n), np.uint8)
    ident = [(1, [1.0], 0.0, "identity")]
    assert np.allclose(restate_infer(restate, ident, layer, valid), layer)
    const = np.full((n, n), 0.25)
    mean3 = [(3, [1.0 / 9.0] * 9, 0.0, "identity")]
    assert np.allclose(restate_infer(restate, mean3, const, valid), 0.25)
    zero_sig = [(3, [0.0] * 9, 0.0, "sigmoid")]
    assert np.allclose(restate_infer(restate, zero_sig, layer, valid), 0.5)
    for layers in (ident, mean3, zero_sig):
        path = tmp_path / "k.weights"
        path.write_text(model_text(layers))
        rc, want, err = ref_infer(refcn, path, layer, valid)
        assert rc == 0, err
        assert same_bits(restate_infer(restate, layers, layer, valid), want)


# ----------------------------------------------------------------- CPU: weight-file reader
MODEL_FILES = {
    "two_layer": "layers: 2\nkernel: 3\n0 0.5 0\n0.5 1 0.5\n0 0.5 0\nbias: -0.25\nactivation: relu\n"
                 "kernel: 1\n2\nbias: 0\nactivation: sigmoid\n",
    "comments": "# model\n\n  layers: 1  \n# k\nkernel: 1\n  3.5 extra\nbias: 1e-3trailing\nactivation:  identity \t\n",
    "even": "layers: 1\nkernel: 2\n1 1\n1 1\nbias: 0\nactivation: relu\n",
    "bad_act": "layers: 1\nkernel: 1\n1\nbias: 0\nactivation: tanh\n",
    "truncated": "layers: 2\nkernel: 1\n1\nbias: 0\nactivation: relu\n",
    "zero_layers": "layers: 0\n",
    "no_tag": "kernel: 1\n",
    "bad_number": "layers: x\n",
    "short_row": "layers: 1\nkernel: 3\n1 2 3\n1 2\n1 2 3\nbias: 0\nactivation: relu\n",
    "nonfinite": "layers: 1\nkernel: 1\ninf\nbias: 0\nactivation: relu\n",
    "nan_bias": "layers: 1\nkernel: 1\n1\nbias: nan\nactivation: relu\n",
    "huge_bias": "layers: 1\nkernel: 1\n1\nbias: 1e999\nactivation: relu\n",
    "missing_act": "layers: 1\nkernel: 1\n1\nbias: 0\nactive: relu\n",
    "empty": "",
}


@pytest.mark.parametrize("name", sorted(MODEL_FILES))
def test_weight_file_reader_agrees_with_reference(product, refcn, tmp_path, name):
    import paper_2204_12876_b200 as pk
    path = tmp_path / f"{name}.weights"
    path.write_text(MODEL_FILES[name])
    rc, _, err = ref_infer(refcn, path, np.zeros((3, 3)), np.ones((3, 3), np.uint8))
    want_status = 0 if rc == 0 else CODE_TO_STATUS[-rc - 1]
    cfg = pk.Config.default(product)
    st = product.relief_gpu_config_load_convnet(cfg.handle, str(path).encode())
    assert st == want_status, (st, product.relief_last_error(), want_status, err)
    if st != 0:
        assert product.relief_last_error().decode() == err


def test_missing_model_file_is_io_error(product, refcn, tmp_path):
    import paper_2204_12876_b200 as pk
    path = tmp_path / "absent.weights"
    rc, _, err = ref_infer(refcn, path, np.zeros((3, 3)), np.ones((3, 3), np.uint8))
    cfg = pk.Config.default(product)
    st = product.relief_gpu_config_load_convnet(cfg.handle, str(path).encode())
    assert st == CODE_TO_STATUS[-rc - 1] == 11
    assert product.relief_last_error().decode() == err


# ----------------------------------------------------------------- GPU
def gpu_infer(gpu, layers, layer, valid, tmp_path):
    import paper_2204_12876_b200 as pk
    path = tmp_path / "g.weights"
    path.write_text(model_text(layers))
    cfg = pk.Config.default(gpu)
    cfg.load_convnet(path)
    return pk.convnet_infer(gpu, cfg, layer, valid), path


def assert_close_to_reference(got, want, layers):
    if any(l[3] == "sigmoid" for l in layers):
        # device exp vs glibc exp: <= 1 ulp per sigmoid, propagated through the stack
        assert np.abs(got - want).max() <= 1e-12
    else:
        assert same_bits(got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(16))
def test_gpu_convnet_matches_reference_random(gpu, refcn, tmp_path, seed):
    rng = np.random.default_rng(5000 + seed)
    H, W = int(rng.integers(3, 90)), int(rng.integers(3, 90))
    p_valid = [0.0, 0.01, 0.2, 0.7, 1.0][seed % 5]
    layer, valid = random_layer(rng, H, W, p_valid)
    layers = random_model(rng, 1 + seed % 4, sizes=(1, 3, 5, 7, 11))
    got, path = gpu_infer(gpu, layers, layer, valid, tmp_path)
    rc, want, err = ref_infer(refcn, path, layer, valid)
    assert rc == 0, err
    assert_close_to_reference(got, want, layers)


@pytest.mark.gpu
def test_gpu_fill_ties_and_large_holes(gpu, refcn, tmp_path):
    """Identity model: the output is the nearest-valid fill itself, bit for bit, on a map whose
    holes are hundreds of BFS levels deep with many equidistant sources."""
    rng = np.random.default_rng(11)
    H, W = 300, 257
    valid = np.zeros((H, W), np.uint8)
    valid[rng.integers(0, H, 40), rng.integers(0, W, 40)] = 1
    valid[140:150, 100:180] = 1
    layer = np.where(valid == 1, 0.5 + 0.1 * rng.standard_normal((H, W)), np.nan)
    layers = [(1, [1.0], 0.0, "identity")]
    got, path = gpu_infer(gpu, layers, layer, valid, tmp_path)
    rc, want, err = ref_infer(refcn, path, layer, valid)
    assert rc == 0, err
    assert same_bits(got, want)


@pytest.mark.gpu
def test_gpu_acceptance12_model_and_kernel_wider_than_map(gpu, refcn, tmp_path):
    """Acceptance #12's model shape (5 x 11x11 relu + 3x3 sigmoid), then a kernel wider than the
    map and one whose halo tile exceeds shared memory (global-memory path)."""
    rng = np.random.default_rng(99)
    layer, valid = random_layer(rng, 120, 140, 0.6)
    layers = [(11, 0.05 * rng.standard_normal(121), 0.01, "relu") for _ in range(5)]
    layers.append((3, 0.05 * rng.standard_normal(9), 0.01, "sigmoid"))
    got, path = gpu_infer(gpu, layers, layer, valid, tmp_path)
    rc, want, err = ref_infer(refcn, path, layer, valid)
    assert rc == 0, err
    assert_close_to_reference(got, want, layers)
    small, sv = random_layer(rng, 9, 7, 0.5)
    for k in (15, 203):
        layers = [(k, 0.01 * rng.standard_normal(k * k), 0.1, "identity")]
        got, path = gpu_infer(gpu, layers, small, sv, tmp_path)
        rc, want, err = ref_infer(refcn, path, small, sv)
        assert rc == 0, err
        assert np.abs(got - want).max() <= 1e-12  # identical sums; exact unless clamped edge cases
        assert same_bits(got, want)


SIM_CONFIG = """map.resolution = 0.04
map.width = 160
map.height = 140
noise.alpha_d = 0.0002
drift.enabled = false
sensor.ring_elevations_deg = -80 -72 -64 -57 -51 -45 -40 -36 -32 -29 -26 -24
sensor.azimuth_steps = 240
sensor.max_range = 10
sensor.rate = 10
scene.ground = 0.0
scene.box = 1.5 0.5 0.25 0.6 0.6 0.5
scene.stairs = -2.0 -0.6 0 0.18 0.28 4 1.2 -x
traj.waypoint = 0 0 0 1
traj.waypoint = 8 1.0 0.5 1
run.scans = 4
run.publish_every = 2
run.seed = 3
run.mode = det
traversability.convnet = {model}
"""


@pytest.mark.gpu
def test_runner_simulate_with_convnet_matches_reference(gpu, reference, tmp_path):
    import paper_2204_12876_b200 as pk
    rng = np.random.default_rng(12)
    layers = [(5, 0.04 * rng.standard_normal(25), 0.05, "relu"),
              (3, 0.3 * rng.standard_normal(9), 0.1, "sigmoid")]
    model = tmp_path / "model.weights"
    model.write_text(model_text(layers))
    cfg = tmp_path / "sim.config"
    cfg.write_text(SIM_CONFIG.format(model=model))
    outs = {}
    for name, lib in (("b200", gpu), ("ref", reference)):
        out = tmp_path / name
        st = lib.relief_run_simulate(str(cfg).encode(), str(out).encode(), 0, 0, None)
        assert st == 0, lib.relief_last_error()
        m = pk.ReliefMap.load(lib, out / "final.relief")
        outs[name] = m.layers()
        m.close()
    assert_layers_match(outs["b200"], outs["ref"], tol_trav=1e-12, context="convnet simulate")
    t = outs["b200"]["traversability"]
    assert np.isfinite(t[outs["b200"]["valid"] == 1]).all()


@pytest.mark.gpu
def test_c_api_integrate_with_attached_model(gpu, tmp_path):
    """relief_config_load alone leaves the model unloaded -> INVALID_MODEL (reference behaviour);
    after relief_gpu_config_load_convnet the integrate call runs the learned filter."""
    import paper_2204_12876_b200 as pk
    model = tmp_path / "c.weights"
    model.write_text("layers: 1\nkernel: 1\n0\nbias: 0.75\nactivation: identity\n")
    text = "map.width = 40\nmap.height = 40\ntraversability.convnet = %s\nscene.ground = 0.0\n" % model
    cfg = pk.Config.from_text(gpu, text, tmp_path / "c.config")
    m = pk.ReliefMap.create(gpu, 0.04, 40, 40)
    pts = np.array([[0.1 + 0.001 * k, 0.0, -1.0] for k in range(400)])
    with pytest.raises(pk.ReliefError) as e:
        m.integrate(pts, pk.pose34(t=(0, 0, 1.0)), 0.0, cfg)
    assert e.value.status == 6
    cfg.load_convnet(model)
    m.integrate(pts, pk.pose34(t=(0, 0, 1.0)), 0.0, cfg)
    trav = m.layers()["traversability"]
    v = m.layers()["valid"] == 1
    assert v.any() and (trav[v] == 0.75).all()  # test_io.cpp:216-238
