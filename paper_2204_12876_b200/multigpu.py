"""Multi-GPU host plumbing (torch.distributed): one process per GPU.

Two modes:

* replicas -- every rank owns an independent map and frame stream on its own device; collectives
  only carry the barrier and the max-over-ranks reduction of device timings (bench.py).
* exact point-batch sharding of ONE frame through the library's group API (relief_gpu_group_*,
  `create_nccl_group`): the frame's exchanges (all-gathers of the records, min / max all-reduces
  of k* and the bounds) run inside the library over NCCL on the map's own stream; Python only
  broadcasts the 128-byte NCCL id once. This is the production path (bench.py --gpus N).
* the same split with host-driven exchanges (relief_gpu_shard_*), for embedders with their own
  transport -- every rank keeps a full map
  replica and takes the contiguous batch [g*N/G, (g+1)*N/G) of the frame (`shard_bounds`), so the
  global point index stays the ray id used for k*. `integrate_sharded` drives the library's
  relief_gpu_shard_* phases and the exchanges between them: all-gather of the drift votes and of
  the fusion records (rank order = scan order), sum of the fate counters, min all-reduce of k* and
  of the upper bounds, max all-reduce of their validity. `DistExchange` does those with
  torch.distributed (NCCL on device buffers in production, gloo on host buffers in the CPU tests);
  `integrate_sharded_lockstep` runs G replicas in one process for the single-GPU parity tests.
"""
from __future__ import annotations

import os
from typing import Tuple


def rank_env() -> Tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_bounds(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, scan-order-preserving batch of n points for `rank` of `world`."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    return (n * rank) // world, (n * (rank + 1)) // world


def _device_for(dist):
    import torch
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def max_over_ranks(value: float, dist=None) -> float:
    """Max of a per-rank scalar (the timing reduction of bench.py); identity without dist."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device_for(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, dist=None) -> float:
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=_device_for(dist))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def weak_scaling_value(points_per_rank_per_step: int, steps: int, world: int, max_seconds: float) -> float:
    """Whole-job points/s: every rank integrates its own frames; time = slowest rank."""
    return world * points_per_rank_per_step * steps / max_seconds


# ------------------------------------------------------------------ sharded frames
def cuda_view(ptr: int, n: int, dtype):
    """Zero-copy torch CUDA tensor over n elements of a library-owned device buffer."""
    import numpy as np
    import torch

    class _Buf:
        pass

    b = _Buf()
    b.__cuda_array_interface__ = {"shape": (int(n),), "typestr": np.dtype(dtype).str,
                                  "data": (int(ptr), False), "version": 3, "strides": None}
    return torch.as_tensor(b, device=torch.device("cuda", torch.cuda.current_device()))


class CudaShardAPI:
    """One map's relief_gpu_shard_* phases; device buffers come back as torch CUDA views."""

    def __init__(self, lib, rmap, config=None):
        import ctypes
        from . import ShardIO
        self.lib, self.map, self.config = lib, rmap, config
        self.io = ShardIO()
        self._ct = ctypes

    def _check(self, st):
        from . import _check
        _check(self.lib, st)

    def _after_caller(self):
        """The library works on its own stream: order it after the caller's pending torch work
        (the exchanged records / k* / bounds written by NCCL or torch ops on that stream)."""
        import torch
        self._check(self.lib.relief_gpu_map_after_stream(
            self.map.handle, self._ct.c_void_p(torch.cuda.current_stream().cuda_stream)))

    def ingest(self, xyz, ray_offset: int, n_total: int, pose, stamp: float) -> dict:
        import numpy as np
        ct = self._ct
        xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1)
        pose = np.ascontiguousarray(pose, dtype=np.float64).reshape(12)
        n = xyz.size // 3
        self._check(self.lib.relief_gpu_shard_ingest(
            self.map.handle, self.config.handle if self.config else None,
            xyz.ctypes.data_as(ct.c_void_p) if n else None, n, 0, ray_offset, n_total,
            pose.ctypes.data_as(ct.POINTER(ct.c_double)), stamp, ct.byref(self.io)))
        io = self.io
        m = int(io.n_records)
        return {"drift": np.array(io.drift[:], dtype=np.float64),
                "counters": np.array(io.counters[:], dtype=np.int64),
                "records": (cuda_view(io.rec_cell, m, np.int32), cuda_view(io.rec_z, m, np.float64),
                            cuda_view(io.rec_var, m, np.float64))}

    def update(self, drift_pairs, cells, z, var) -> dict:
        import numpy as np
        ct = self._ct
        pairs = np.ascontiguousarray(drift_pairs, dtype=np.float64).reshape(-1)
        m = int(cells.numel())
        self._after_caller()
        self._check(self.lib.relief_gpu_shard_update(
            self.map.handle, pairs.ctypes.data_as(ct.POINTER(ct.c_double)), pairs.size // 2,
            cells.data_ptr() if m else None, z.data_ptr() if m else None, var.data_ptr() if m else None,
            m, ct.byref(self.io)))
        return self._bounds(with_kstar=True)

    def _bounds(self, with_kstar: bool) -> dict:
        import numpy as np
        io = self.io
        out = {"ub": cuda_view(io.upper_bound, io.cells, np.float64),
               "ubv": cuda_view(io.upper_bound_valid, io.cells, np.uint8)}
        if with_kstar:
            out["kstar"] = cuda_view(io.kstar, io.cells, np.int32)
        return out

    def remove(self):
        ct = self._ct
        removed = ct.c_int64(0)
        self._after_caller()
        self._check(self.lib.relief_gpu_shard_remove(self.map.handle, ct.byref(removed), ct.byref(self.io)))
        return int(removed.value), self._bounds(with_kstar=False)

    def finish(self, counters, n_total: int):
        import numpy as np
        from . import ScanStats
        ct = self._ct
        c = np.ascontiguousarray(counters, dtype=np.int64)
        st = ScanStats()
        self._after_caller()
        self._check(self.lib.relief_gpu_shard_finish(self.map.handle, c.ctypes.data_as(ct.POINTER(ct.c_int64)),
                                                     n_total, ct.byref(st)))
        return st


class DistExchange:
    """The sharded frame's exchanges over torch.distributed (tensors live where the API put them)."""

    def __init__(self, dist, group=None):
        self.dist, self.group = dist, group

    def world(self) -> int:
        return self.dist.get_world_size(self.group)

    def gather_pairs(self, pair):
        import numpy as np
        import torch
        dev = _device_for(self.dist)
        t = torch.as_tensor(np.asarray(pair, dtype=np.float64), device=dev)
        out = [torch.empty_like(t) for _ in range(self.world())]
        self.dist.all_gather(out, t, group=self.group)
        return np.stack([o.cpu().numpy() for o in out])

    def sum_counters(self, counters):
        import numpy as np
        import torch
        t = torch.as_tensor(np.asarray(counters, dtype=np.int64), device=_device_for(self.dist))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy()

    def gather_records(self, records):
        """All-gather of variable-length record arrays, concatenated in rank order (scan order)."""
        import torch
        G = self.world()
        n = torch.tensor([records[0].numel()], dtype=torch.int64, device=records[0].device)
        ns = [torch.empty_like(n) for _ in range(G)]
        self.dist.all_gather(ns, n, group=self.group)
        ns = [int(x.item()) for x in ns]
        mx = max(ns) if ns else 0
        out = []
        for a in records:
            pad = torch.zeros(mx, dtype=a.dtype, device=a.device)
            pad[: a.numel()] = a
            parts = [torch.empty_like(pad) for _ in range(G)]
            self.dist.all_gather(parts, pad, group=self.group)
            out.append(torch.cat([p[:k] for p, k in zip(parts, ns)]) if mx else pad[:0])
        return tuple(out)

    def reduce_min(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)

    def reduce_max(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)


def create_nccl_group(lib, rmap, dist=None, group=None):
    """relief_gpu_group over NCCL for this process's map: rank 0 makes the 128-byte NCCL id, the
    torch.distributed process group broadcasts it, every rank creates its end collectively. The
    frame's exchanges then run inside the library on the map's stream (no torch ops per frame)."""
    from . import Group
    uid, ranks, rank = broadcast_unique_id(lib, dist, group)
    return Group.nccl(lib, rmap, uid, ranks, rank)


def broadcast_unique_id(lib, dist=None, group=None):
    """(id, ranks, rank): rank 0's relief_gpu_group_unique_id, broadcast over torch.distributed."""
    import numpy as np
    import torch
    from . import group_unique_id
    if dist is None or not dist.is_initialized():
        return group_unique_id(lib), 1, 0
    ranks, rank = dist.get_world_size(group), dist.get_rank(group)
    uid = group_unique_id(lib) if rank == 0 else bytes(128)
    t = torch.tensor(np.frombuffer(uid, dtype=np.uint8).copy(), device=_device_for(dist))
    dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(t.cpu().numpy().tobytes()), ranks, rank


def integrate_sharded(api, ex, xyz_local, ray_offset: int, n_total: int, pose, stamp: float):
    """One frame, this rank's batch; identical maps and stats on every rank afterwards."""
    a = api.ingest(xyz_local, ray_offset, n_total, pose, stamp)
    pairs = ex.gather_pairs(a["drift"])
    counters = ex.sum_counters(a["counters"])
    cells, z, var = ex.gather_records(a["records"])
    b = api.update(pairs, cells, z, var)
    ex.reduce_min(b["kstar"])
    ex.reduce_min(b["ub"])
    ex.reduce_max(b["ubv"])
    removed, c = api.remove()
    if removed > 0:
        ex.reduce_min(c["ub"])
        ex.reduce_max(c["ubv"])
    return api.finish(counters, n_total)


def integrate_sharded_lockstep(apis, xyz, pose, stamp: float):
    """All G ranks of one sharded frame in one process (replicas on the current GPU), phase by
    phase, with the exchanges done by torch ops. Used by the single-GPU parity tests."""
    import numpy as np
    import torch
    xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3)
    N, G = xyz.shape[0], len(apis)
    outs = []
    for g, api in enumerate(apis):
        lo, hi = shard_bounds(N, G, g)
        outs.append(api.ingest(xyz[lo:hi], lo, N, pose, stamp))
    pairs = np.stack([o["drift"] for o in outs])
    counters = np.sum([o["counters"] for o in outs], axis=0)
    recs = [torch.cat([o["records"][k] for o in outs]) for k in range(3)]
    bs = [api.update(pairs, *recs) for api in apis]

    def reduce(key, fn):
        r = fn(torch.stack([b[key] for b in bs]))
        for b in bs:
            b[key].copy_(r)

    reduce("kstar", lambda t: t.amin(0))
    reduce("ub", lambda t: t.amin(0))
    reduce("ubv", lambda t: t.amax(0))
    rem = [api.remove() for api in apis]
    if len({r for r, _ in rem}) != 1:
        raise RuntimeError("ranks disagree on the removal count")
    if rem[0][0] > 0:
        bs = [c for _, c in rem]
        reduce("ub", lambda t: t.amin(0))
        reduce("ubv", lambda t: t.amax(0))
    return [api.finish(counters, N) for api in apis]

