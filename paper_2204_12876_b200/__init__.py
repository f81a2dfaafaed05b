"""B200-native elevation-map update path of arXiv 2204.12876 (reliefmap drop-in).

The product is ``lib/librelief_b200.so``: the reference's C ABI (``include/relief.h``)
implemented as host C++ over hand-written sm_100a CUDA kernels, plus the additive
``include/relief_gpu.h`` entry points. This module is a thin ctypes mirror of that ABI
for Python callers (tests, bench.py); it mirrors the reference C API names, argument
meaning and error behaviour (reference proj/include/relief/relief.h:37-129):

    lib = load_library()
    m = ReliefMap.create(lib, resolution=0.04, width=500, height=500)
    stats = m.integrate(xyz, pose34, stamp, config=None)   # relief_map_integrate
    elev = m.layer("elevation")                            # relief_map_layer

There is no CPU fallback: loading fails loudly when the shared library is missing,
and map creation fails when no CUDA device is present.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
DEFAULT_LIB = PKG_DIR / "lib" / "librelief_b200.so"

LAYER_NAMES = (
    "elevation", "variance", "last_update", "upper_bound", "upper_bound_valid",
    "traversability", "normal_x", "normal_y", "normal_z", "valid",
)

STATUS_NAMES = {
    0: "OK", 1: "USAGE", 2: "DATA", 3: "OUT_OF_MAP", 4: "INVALID_POSE", 5: "INVALID_VARIANCE",
    6: "INVALID_MODEL", 7: "DEGENERATE_PLANE", 8: "NOTHING_TO_INPAINT", 9: "OUT_OF_TRAJECTORY",
    10: "PARSE", 11: "IO",
}

# Post-processing chain step kinds (relief_gpu.h).
GAUSSIAN, BOX, MEDIAN, MIN_INPAINT = 0, 1, 2, 3


class ScanStats(ctypes.Structure):
    """relief_scan_stats (reference relief.h:89-102), ABI-fixed layout."""

    _fields_ = [
        ("points_in", ctypes.c_int64),
        ("points_excluded", ctypes.c_int64),
        ("points_out_of_range", ctypes.c_int64),
        ("points_out_of_map", ctypes.c_int64),
        ("points_rejected_outlier", ctypes.c_int64),
        ("points_ignored_low", ctypes.c_int64),
        ("points_fused", ctypes.c_int64),
        ("cells_updated", ctypes.c_int64),
        ("cells_removed_by_cleanup", ctypes.c_int64),
        ("cells_cleared_by_overlap", ctypes.c_int64),
        ("drift_offset_applied", ctypes.c_double),
        ("total_seconds", ctypes.c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class ReliefError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {message}")
        self.status = status
        self.message = message


_P = ctypes.c_void_p
_D = ctypes.c_double
_DP = ctypes.POINTER(ctypes.c_double)
_I = ctypes.c_int
_SZ = ctypes.c_size_t
_CS = ctypes.c_char_p

# Symbols of relief.h (the drop-in ABI) and their ctypes signatures.
RELIEF_H_SIGNATURES = {
    "relief_last_error": (_CS, []),
    "relief_version": (_CS, []),
    "relief_config_default": (_P, []),
    "relief_config_load": (_P, [_CS]),
    "relief_config_free": (None, [_P]),
    "relief_config_set_mode": (_I, [_P, _CS]),
    "relief_config_set_seed": (_I, [_P, ctypes.c_uint64]),
    "relief_map_create": (_P, [_D, _I, _I, _D, _D]),
    "relief_map_load": (_P, [_CS]),
    "relief_map_save": (_I, [_P, _CS]),
    "relief_map_free": (None, [_P]),
    "relief_map_width": (_I, [_P]),
    "relief_map_height": (_I, [_P]),
    "relief_map_resolution": (_D, [_P]),
    "relief_map_center": (_I, [_P, _DP, _DP]),
    "relief_map_layer": (_I, [_P, _CS, _DP, _SZ]),
    "relief_map_integrate": (_I, [_P, _P, _DP, _SZ, _DP, _D, ctypes.POINTER(ScanStats)]),
    "relief_run_simulate": (_I, [_CS, _CS, ctypes.c_uint64, _I, _CS]),
    "relief_run_replay": (_I, [_CS, ctypes.POINTER(_CS), _SZ, _CS, _CS, _CS]),
    "relief_run_bench": (_I, [_CS, ctypes.POINTER(_SZ), _SZ, _I, _CS, _CS]),
    "relief_run_export": (_I, [_CS, _CS, _CS, _CS]),
    "relief_run_segment": (_I, [_CS, _CS, _CS, ctypes.POINTER(_SZ)]),
}

# Additive relief_gpu.h symbols.
class ShardIO(ctypes.Structure):
    """relief_gpu_shard_io (include/relief_gpu.h)."""
    _fields_ = [("n_records", ctypes.c_int64), ("drift", ctypes.c_double * 2), ("counters", ctypes.c_int64 * 3),
                ("rec_cell", ctypes.c_void_p), ("rec_z", ctypes.c_void_p), ("rec_var", ctypes.c_void_p),
                ("kstar", ctypes.c_void_p), ("upper_bound", ctypes.c_void_p),
                ("upper_bound_valid", ctypes.c_void_p), ("cells", ctypes.c_size_t)]


RELIEF_GPU_H_SIGNATURES = {
    "relief_gpu_device_count": (_I, []),
    "relief_gpu_map_create_on": (_P, [_I, _D, _I, _I, _D, _D]),
    "relief_gpu_map_device": (_I, [_P]),
    "relief_gpu_map_integrate_device": (_I, [_P, _P, ctypes.c_void_p, _SZ, _DP, _D, ctypes.POINTER(ScanStats)]),
    "relief_gpu_map_phase_seconds": (_I, [_P, _DP]),
    "relief_gpu_map_kernel_seconds": (_I, [_P, _DP]),
    "relief_gpu_map_set_phase_timing": (_I, [_P, ctypes.c_int]),
    "relief_gpu_map_last_launches": (ctypes.c_int64, [_P]),
    "relief_gpu_map_last_visits": (ctypes.c_int64, [_P]),
    "relief_gpu_map_layer_device": (_I, [_P, _CS, ctypes.c_void_p, _SZ]),
    "relief_gpu_map_smooth_chain": (_I, [_P, _CS, ctypes.POINTER(_I), ctypes.POINTER(_I), _DP, _I, _DP,
                                         ctypes.POINTER(ctypes.c_uint8)]),
    "relief_gpu_map_smooth_chain_device": (_I, [_P, _CS, ctypes.POINTER(_I), ctypes.POINTER(_I), _DP, _I,
                                                ctypes.c_void_p, ctypes.c_void_p]),
    "relief_gpu_map_chain_seconds": (_D, [_P]),
    "relief_gpu_smooth_chain": (_I, [_DP, ctypes.POINTER(ctypes.c_uint8), _I, _I, ctypes.POINTER(_I),
                                     ctypes.POINTER(_I), _DP, _I, _DP, ctypes.POINTER(ctypes.c_uint8)]),
    "relief_gpu_host_alloc": (ctypes.c_void_p, [_SZ]),
    "relief_gpu_host_free": (None, [ctypes.c_void_p]),
    "relief_gpu_map_integrate_async": (_I, [_P, _P, ctypes.c_void_p, _SZ, _DP, _D]),
    "relief_gpu_map_wait": (_I, [_P, ctypes.POINTER(ScanStats)]),
    "relief_gpu_map_in_flight": (_I, [_P]),
    "relief_gpu_config_load_convnet": (_I, [_P, _CS]),
    "relief_gpu_convnet_infer": (_I, [_P, _DP, ctypes.POINTER(ctypes.c_uint8), _I, _I, _DP]),
    "relief_gpu_shard_ingest": (_I, [_P, _P, ctypes.c_void_p, _SZ, _I, ctypes.c_uint64, ctypes.c_uint64, _DP, _D,
                                     ctypes.c_void_p]),
    "relief_gpu_shard_update": (_I, [_P, _DP, _I, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, _SZ,
                                     ctypes.c_void_p]),
    "relief_gpu_shard_remove": (_I, [_P, ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p]),
    "relief_gpu_shard_finish": (_I, [_P, ctypes.POINTER(ctypes.c_int64), ctypes.c_uint64,
                                     ctypes.POINTER(ScanStats)]),
    "relief_gpu_sim_render": (ctypes.c_int64, [_CS, _DP, _D, ctypes.c_uint64, ctypes.c_uint64, _DP,
                                               ctypes.c_int64]),
    "relief_gpu_map_after_stream": (_I, [_P, ctypes.c_void_p]),
    "relief_gpu_map_set_graphs": (_I, [_P, _I]),
    "relief_gpu_map_graph_stats": (_I, [_P, ctypes.POINTER(ctypes.c_int64)]),
    "relief_gpu_group_unique_id": (_I, [ctypes.c_void_p]),
    "relief_gpu_group_create": (_P, [_P, ctypes.c_void_p, _I, _I]),
    "relief_gpu_group_create_local": (_P, [ctypes.POINTER(_P), _I]),
    "relief_gpu_group_free": (None, [_P]),
    "relief_gpu_group_set_fusion": (_I, [_P, _I]),
    "relief_gpu_group_fusion": (_I, [_P]),
    "relief_gpu_group_bounds": (_I, [ctypes.c_uint64, _I, _I, ctypes.POINTER(ctypes.c_uint64),
                                     ctypes.POINTER(ctypes.c_uint64)]),
    "relief_gpu_group_integrate": (_I, [_P, _P, ctypes.c_void_p, _SZ, _I, ctypes.c_uint64, _DP, _D,
                                        ctypes.POINTER(ScanStats)]),
    "relief_gpu_nccl_version": (_I, []),
}


def _bind(lib: ctypes.CDLL, table: dict) -> None:
    for name, (res, args) in table.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def load_library(path: Optional[os.PathLike] = None, gpu_api: Optional[bool] = None) -> ctypes.CDLL:
    """Loads a library exporting relief.h (this repo's product by default).

    ``gpu_api`` binds relief_gpu.h too; it defaults to True for the product library.
    Raises FileNotFoundError when the library is missing -- there is no fallback.
    """
    if path is None and os.environ.get("RELIEF_B200_LIB"):
        path = os.environ["RELIEF_B200_LIB"]  # development override (A/B builds)
        gpu_api = True if gpu_api is None else gpu_api
    p = Path(path) if path is not None else DEFAULT_LIB
    if not p.exists():
        raise FileNotFoundError(
            f"{p} not found: build it with `python -m paper_2204_12876_b200.build` "
            "(the B200 path has no CPU fallback)")
    lib = ctypes.CDLL(str(p), mode=ctypes.RTLD_LOCAL)
    _bind(lib, RELIEF_H_SIGNATURES)
    if gpu_api if gpu_api is not None else path is None:
        _bind(lib, RELIEF_GPU_H_SIGNATURES)
    lib._relief_path = str(p)
    return lib


def _check(lib, status: int) -> None:
    if status != 0:
        raise ReliefError(status, lib.relief_last_error().decode())


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_DP)


def pose34(R=None, t=(0.0, 0.0, 0.0)) -> np.ndarray:
    """Row-major 3x4 [R | t] as relief_map_integrate expects."""
    R = np.eye(3) if R is None else np.asarray(R, dtype=np.float64)
    out = np.zeros((3, 4), dtype=np.float64)
    out[:, :3] = R
    out[:, 3] = t
    return np.ascontiguousarray(out.reshape(12))


class Config:
    """relief_config handle (reference relief.h:61-66)."""

    def __init__(self, lib, handle):
        self.lib = lib
        self.handle = handle

    @classmethod
    def default(cls, lib) -> "Config":
        h = lib.relief_config_default()
        if not h:
            raise ReliefError(2, lib.relief_last_error().decode())
        return cls(lib, h)

    @classmethod
    def load(cls, lib, path) -> "Config":
        h = lib.relief_config_load(str(path).encode())
        if not h:
            raise ReliefError(10, lib.relief_last_error().decode())
        return cls(lib, h)

    @classmethod
    def from_text(cls, lib, text: str, path) -> "Config":
        Path(path).write_text(text)
        return cls.load(lib, path)

    def set_mode(self, mode: str) -> None:
        _check(self.lib, self.lib.relief_config_set_mode(self.handle, mode.encode()))

    def set_seed(self, seed: int) -> None:
        _check(self.lib, self.lib.relief_config_set_seed(self.handle, seed))

    def load_convnet(self, model_path) -> None:
        """Attach a conv-net weight file; the pipeline then uses the learned filter."""
        _check(self.lib, self.lib.relief_gpu_config_load_convnet(self.handle, str(model_path).encode()))

    def close(self) -> None:
        if self.handle:
            self.lib.relief_config_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ReliefMap:
    """relief_map handle: the device-resident elevation map."""

    def __init__(self, lib, handle):
        self.lib = lib
        self.handle = handle

    @classmethod
    def create(cls, lib, resolution=0.04, width=250, height=250, center_x=0.0, center_y=0.0,
               device: Optional[int] = None) -> "ReliefMap":
        if device is None:
            h = lib.relief_map_create(resolution, width, height, center_x, center_y)
        else:
            h = lib.relief_gpu_map_create_on(device, resolution, width, height, center_x, center_y)
        if not h:
            raise ReliefError(1, lib.relief_last_error().decode())
        return cls(lib, h)

    @classmethod
    def load(cls, lib, path) -> "ReliefMap":
        h = lib.relief_map_load(str(path).encode())
        if not h:
            raise ReliefError(10, lib.relief_last_error().decode())
        return cls(lib, h)

    def save(self, path) -> None:
        _check(self.lib, self.lib.relief_map_save(self.handle, str(path).encode()))

    @property
    def width(self) -> int:
        return self.lib.relief_map_width(self.handle)

    @property
    def height(self) -> int:
        return self.lib.relief_map_height(self.handle)

    @property
    def resolution(self) -> float:
        return self.lib.relief_map_resolution(self.handle)

    def center(self):
        x, y = ctypes.c_double(), ctypes.c_double()
        _check(self.lib, self.lib.relief_map_center(self.handle, ctypes.byref(x), ctypes.byref(y)))
        return x.value, y.value

    def layer(self, name: str) -> np.ndarray:
        out = np.empty(self.width * self.height, dtype=np.float64)
        _check(self.lib, self.lib.relief_map_layer(self.handle, name.encode(), _dptr(out), out.size))
        return out.reshape(self.height, self.width)

    def layers(self) -> dict:
        return {n: self.layer(n) for n in LAYER_NAMES}

    def integrate(self, xyz, pose, stamp: float, config: Optional[Config] = None) -> ScanStats:
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1)
        pose = np.ascontiguousarray(pose, dtype=np.float64).reshape(12)
        st = ScanStats()
        status = self.lib.relief_map_integrate(
            self.handle, config.handle if config is not None else None,
            _dptr(xyz) if xyz.size else None, xyz.size // 3, _dptr(pose), stamp, ctypes.byref(st))
        _check(self.lib, status)
        return st

    def integrate_async(self, xyz, pose, stamp: float, config: Optional[Config] = None) -> None:
        """relief_gpu_map_integrate_async: enqueue a frame (keep xyz alive until its wait())."""
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1)
        pose = np.ascontiguousarray(pose, dtype=np.float64).reshape(12)
        _check(self.lib, self.lib.relief_gpu_map_integrate_async(
            self.handle, config.handle if config else None, xyz.ctypes.data_as(ctypes.c_void_p),
            xyz.size // 3, _dptr(pose), stamp))

    def wait(self) -> ScanStats:
        """relief_gpu_map_wait: stats of the oldest frame in flight."""
        st = ScanStats()
        _check(self.lib, self.lib.relief_gpu_map_wait(self.handle, ctypes.byref(st)))
        return st

    def integrate_device(self, d_xyz_ptr: int, n: int, pose, stamp: float,
                         config: Optional[Config] = None) -> ScanStats:
        """relief_gpu_map_integrate_device: points already in device memory."""
        pose = np.ascontiguousarray(pose, dtype=np.float64).reshape(12)
        st = ScanStats()
        status = self.lib.relief_gpu_map_integrate_device(
            self.handle, config.handle if config is not None else None, ctypes.c_void_p(d_xyz_ptr), n,
            _dptr(pose), stamp, ctypes.byref(st))
        _check(self.lib, status)
        return st

    def phase_seconds(self) -> np.ndarray:
        out = np.zeros(7, dtype=np.float64)
        _check(self.lib, self.lib.relief_gpu_map_phase_seconds(self.handle, _dptr(out)))
        return out

    def set_phase_timing(self, on: bool) -> None:
        """relief_gpu_map_set_phase_timing: record per-phase events (costs the overlap of the
        kernels at the phase boundaries; off by default)."""
        _check(self.lib, self.lib.relief_gpu_map_set_phase_timing(self.handle, 1 if on else 0))

    def kernel_seconds(self) -> np.ndarray:
        """[upload, ingest, drift, sort, fusion, rays, cell phases, total excl. upload]."""
        out = np.zeros(8, dtype=np.float64)
        _check(self.lib, self.lib.relief_gpu_map_kernel_seconds(self.handle, _dptr(out)))
        return out

    def last_launches(self) -> int:
        return int(self.lib.relief_gpu_map_last_launches(self.handle))

    def last_visits(self) -> int:
        return int(self.lib.relief_gpu_map_last_visits(self.handle))

    def smooth_chain(self, layer: str, steps: Sequence[tuple]):
        """steps: (kind, radius, sigma) tuples; returns (values, valid)."""
        n = self.width * self.height
        kinds = (ctypes.c_int * len(steps))(*[s[0] for s in steps])
        radii = (ctypes.c_int * len(steps))(*[s[1] for s in steps])
        sig = (ctypes.c_double * len(steps))(*[float(s[2]) for s in steps])
        vals = np.empty(n, dtype=np.float64)
        ok = np.empty(n, dtype=np.uint8)
        _check(self.lib, self.lib.relief_gpu_map_smooth_chain(
            self.handle, layer.encode(), kinds, radii, sig, len(steps), _dptr(vals),
            ok.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
        return vals.reshape(self.height, self.width), ok.reshape(self.height, self.width)

    def smooth_chain_device(self, layer: str, steps: Sequence[tuple], d_values: int, d_valid: int) -> float:
        """Chain with device outputs (raw device pointers); returns its device seconds."""
        kinds = (ctypes.c_int * len(steps))(*[s[0] for s in steps])
        radii = (ctypes.c_int * len(steps))(*[s[1] for s in steps])
        sig = (ctypes.c_double * len(steps))(*[float(s[2]) for s in steps])
        _check(self.lib, self.lib.relief_gpu_map_smooth_chain_device(
            self.handle, layer.encode(), kinds, radii, sig, len(steps), ctypes.c_void_p(d_values),
            ctypes.c_void_p(d_valid)))
        return float(self.lib.relief_gpu_map_chain_seconds(self.handle))

    def set_graphs(self, on) -> None:
        """relief_gpu_map_set_graphs: True / 1 one CUDA graph per synchronous frame, False / 0 direct
        launches, 2 (the default) graphs for frames of at least 32Ki points."""
        _check(self.lib, self.lib.relief_gpu_map_set_graphs(self.handle, int(on)))

    def graph_stats(self):
        """(graphs instantiated, frames that updated a cached graph)."""
        out = (ctypes.c_int64 * 2)()
        _check(self.lib, self.lib.relief_gpu_map_graph_stats(self.handle, out))
        return int(out[0]), int(out[1])

    def after_stream(self, stream_handle: int) -> None:
        """relief_gpu_map_after_stream: order the map's next device work after everything
        already enqueued on that cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream)."""
        _check(self.lib, self.lib.relief_gpu_map_after_stream(self.handle, ctypes.c_void_p(stream_handle)))

    def close(self) -> None:
        if self.handle:
            self.lib.relief_map_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def group_bounds(lib, n_total: int, ranks: int, rank: int):
    """relief_gpu_group_bounds: rank's batch [lo, hi) of an n_total-point frame."""
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    _check(lib, lib.relief_gpu_group_bounds(n_total, ranks, rank, ctypes.byref(lo), ctypes.byref(hi)))
    return int(lo.value), int(hi.value)


def group_unique_id(lib) -> bytes:
    """relief_gpu_group_unique_id: the 128-byte NCCL id rank 0 broadcasts."""
    buf = (ctypes.c_uint8 * 128)()
    _check(lib, lib.relief_gpu_group_unique_id(buf))
    return bytes(buf)


class Group:
    """relief_gpu_group: one frame split across the ranks of a group (include/relief_gpu.h).

    nccl(lib, map, uid, ranks, rank): one process per GPU, NCCL transport -- integrate() takes
    this rank's batch. local(lib, maps): one process drives every map -- integrate() takes the
    whole frame."""

    def __init__(self, lib, handle, maps, ranks: int, rank: int, local: bool):
        self.lib, self.handle, self.maps = lib, handle, maps
        self.ranks, self.rank, self.local = ranks, rank, local

    @classmethod
    def nccl(cls, lib, rmap: ReliefMap, uid: bytes, ranks: int, rank: int) -> "Group":
        if len(uid) != 128:
            raise ValueError("the NCCL unique id is 128 bytes")
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        h = lib.relief_gpu_group_create(rmap.handle, buf, ranks, rank)
        if not h:
            raise ReliefError(2, lib.relief_last_error().decode())
        return cls(lib, h, [rmap], ranks, rank, False)

    @classmethod
    def local(cls, lib, maps: Sequence[ReliefMap]) -> "Group":
        arr = (_P * len(maps))(*[m.handle for m in maps])
        h = lib.relief_gpu_group_create_local(arr, len(maps))
        if not h:
            raise ReliefError(1, lib.relief_last_error().decode())
        return cls(lib, h, list(maps), len(maps), 0, True)

    EXACT, INFORMATION = 0, 1

    def set_fusion(self, mode: int) -> None:
        """relief_gpu_group_set_fusion: Group.EXACT (gated, bit-identical to one GPU) or
        Group.INFORMATION (ungated information-form partial sums, all-reduced)."""
        _check(self.lib, self.lib.relief_gpu_group_set_fusion(self.handle, int(mode)))

    @property
    def fusion(self) -> int:
        return int(self.lib.relief_gpu_group_fusion(self.handle))

    def bounds(self, n_total: int, rank: Optional[int] = None):
        return group_bounds(self.lib, n_total, self.ranks, self.rank if rank is None else rank)

    def integrate(self, xyz, n_total: int, pose, stamp: float, config: Optional[Config] = None) -> ScanStats:
        """Host points: this rank's batch (NCCL) or the whole frame (local)."""
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1)
        pose = np.ascontiguousarray(pose, dtype=np.float64).reshape(12)
        st = ScanStats()
        _check(self.lib, self.lib.relief_gpu_group_integrate(
            self.handle, config.handle if config is not None else None,
            xyz.ctypes.data_as(ctypes.c_void_p) if xyz.size else None, xyz.size // 3, 0, n_total,
            _dptr(pose), stamp, ctypes.byref(st)))
        return st

    def integrate_device(self, d_xyz_ptr: int, n: int, n_total: int, pose, stamp: float,
                         config: Optional[Config] = None) -> ScanStats:
        pose = np.ascontiguousarray(pose, dtype=np.float64).reshape(12)
        st = ScanStats()
        _check(self.lib, self.lib.relief_gpu_group_integrate(
            self.handle, config.handle if config is not None else None, ctypes.c_void_p(d_xyz_ptr), n, 1,
            n_total, _dptr(pose), stamp, ctypes.byref(st)))
        return st

    def close(self) -> None:
        if self.handle:
            self.lib.relief_gpu_group_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def smooth_chain(lib, values: np.ndarray, valid: np.ndarray, steps: Sequence[tuple]):
    """relief_gpu_smooth_chain on host arrays; returns (values, valid)."""
    values = np.ascontiguousarray(values, dtype=np.float64)
    valid = np.ascontiguousarray(valid, dtype=np.uint8)
    H, W = values.shape
    kinds = (ctypes.c_int * len(steps))(*[s[0] for s in steps])
    radii = (ctypes.c_int * len(steps))(*[s[1] for s in steps])
    sig = (ctypes.c_double * len(steps))(*[float(s[2]) for s in steps])
    vo = np.empty_like(values)
    ko = np.empty_like(valid)
    u8 = ctypes.POINTER(ctypes.c_uint8)
    _check(lib, lib.relief_gpu_smooth_chain(_dptr(values), valid.ctypes.data_as(u8), W, H, kinds, radii,
                                            sig, len(steps), _dptr(vo), ko.ctypes.data_as(u8)))
    return vo, ko


def convnet_infer(lib, config: "Config", layer: np.ndarray, valid: np.ndarray) -> np.ndarray:
    """relief_gpu_convnet_infer: the config's conv-net over a host layer (H, W)."""
    layer = np.ascontiguousarray(layer, dtype=np.float64)
    valid = np.ascontiguousarray(valid, dtype=np.uint8)
    H, W = layer.shape
    out = np.empty_like(layer)
    _check(lib, lib.relief_gpu_convnet_infer(config.handle, _dptr(layer),
                                             valid.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), W, H,
                                             _dptr(out)))
    return out


class PinnedArray:
    """(n, 3) float64 points in page-locked memory from relief_gpu_host_alloc."""

    def __init__(self, lib, src: np.ndarray):
        src = np.ascontiguousarray(src, dtype=np.float64)
        self.lib = lib
        self.ptr = lib.relief_gpu_host_alloc(max(src.nbytes, 8))
        if not self.ptr:
            raise ReliefError(2, lib.relief_last_error().decode())
        buf = (ctypes.c_double * max(src.size, 1)).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=np.float64, count=src.size).reshape(src.shape)
        self.array[...] = src

    def __del__(self):
        try:
            if self.ptr:
                self.lib.relief_gpu_host_free(self.ptr)
                self.ptr = None
        except Exception:
            pass


def sim_render(lib, config_path, pose, time: float, seed: int, scan_index: int,
               capacity: int = 1 << 22) -> np.ndarray:
    """Synthetic scan from a reliefmap config (relief_gpu_sim_render); (n, 3) float64."""
    pose = np.ascontiguousarray(pose, dtype=np.float64).reshape(12)
    buf = np.empty(capacity * 3, dtype=np.float64)
    n = lib.relief_gpu_sim_render(str(config_path).encode(), _dptr(pose), time, seed, scan_index,
                                  _dptr(buf), capacity)
    if n < 0:
        raise ReliefError(2, lib.relief_last_error().decode())
    if n > capacity:
        return sim_render(lib, config_path, pose, time, seed, scan_index, capacity=int(n))
    return buf[: 3 * n].reshape(n, 3).copy()
