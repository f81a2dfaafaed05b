"""N>1 host path on CPU: world_size-2 gloo processes exercise the reductions and the batch split
bench.py / the sharded mode rely on (the GPU legs run one process per B200 over NCCL)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from paper_2204_12876_b200 import multigpu as mg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, lr = mg.rank_env()
        t_rank = 0.010 + 0.005 * rank          # per-rank device time of the timed steps
        mx = mg.max_over_ranks(t_rank, dist)
        total = mg.sum_over_ranks(1000 * (rank + 1), dist)
        lo, hi = mg.shard_bounds(1_000_064, w, r)
        q.put((r, w, lr, mx, total, lo, hi))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_reductions_and_shards():
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, w0, l0, mx0, tot0, lo0, hi0), (r1, w1, l1, mx1, tot1, lo1, hi1) = out
    assert (r0, r1, w0, w1) == (0, 1, 2, 2)
    assert mx0 == mx1 == pytest.approx(0.015)
    assert tot0 == tot1 == 3000
    assert (lo0, hi1) == (0, 1_000_064) and hi0 == lo1
    assert mg.weak_scaling_value(1_000_064, 20, 2, mx0 * 20) == pytest.approx(2 * 1_000_064 / 0.015)


def test_shard_bounds_cover_in_order():
    for n in (0, 1, 7, 1_000_064):
        for world in (1, 2, 3, 8):
            spans = [mg.shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


# ----------------------------------------------------------------- sharded-frame plumbing
# A host-memory stand-in for CudaShardAPI with deterministic per-rank outputs, so each gloo
# worker can check that integrate_sharded moved exactly the right data between the phases.
CELLS = 64
BIG = np.iinfo(np.int32).max


def _rank_data(rank, n_local):
    rng = np.random.default_rng(100 + rank)
    m = n_local // 2 + rank
    return {"cells": rng.integers(0, CELLS, m).astype(np.uint32),
            "z": rng.normal(size=m), "var": rng.random(m) + 0.1,
            "drift": np.array([0.25 * (rank + 1), 10.0 + rank]),
            "counters": np.array([rank + 1, 2 * rank, 7], dtype=np.int64),
            "kstar": np.where(rng.random(CELLS) < 0.3, rng.integers(0, 1000, CELLS), BIG).astype(np.int32),
            "ub": np.where(rng.random(CELLS) < 0.5, rng.normal(size=CELLS), np.inf),
            "ubv": (rng.random(CELLS) < 0.4).astype(np.uint8),
            "ub2": rng.normal(size=CELLS) - 5.0,
            "ubv2": (rng.random(CELLS) < 0.2).astype(np.uint8)}


class MockShardAPI:
    def __init__(self, rank):
        self.rank = rank
        self.seen = {}

    def ingest(self, xyz, ray_offset, n_total, pose, stamp):
        import torch
        self.d = _rank_data(self.rank, len(xyz))
        self.seen["ingest"] = (len(xyz), ray_offset, n_total)
        return {"drift": self.d["drift"], "counters": self.d["counters"],
                "records": (torch.from_numpy(self.d["cells"].astype(np.int64)), torch.from_numpy(self.d["z"]),
                            torch.from_numpy(self.d["var"]))}

    def update(self, pairs, cells, z, var):
        import torch
        self.seen["update"] = (np.array(pairs), cells.numpy().copy(), z.numpy().copy(), var.numpy().copy())
        self.b = {"kstar": torch.from_numpy(self.d["kstar"].copy()), "ub": torch.from_numpy(self.d["ub"].copy()),
                  "ubv": torch.from_numpy(self.d["ubv"].copy())}
        return self.b

    def remove(self):
        import torch
        ks = self.b["kstar"].numpy()
        self.seen["kstar"] = ks.copy()
        self.seen["ub1"] = self.b["ub"].numpy().copy()
        self.seen["ubv1"] = self.b["ubv"].numpy().copy()
        removed = int((ks < BIG).sum())
        ub = self.b["ub"].numpy()
        ub[ks < BIG] = self.d["ub2"][ks < BIG]   # pass-2 bounds of removed cells from local rays
        self.b["ubv"].numpy()[ks < BIG] = self.d["ubv2"][ks < BIG]
        return removed, {"ub": self.b["ub"], "ubv": self.b["ubv"]}

    def finish(self, counters, n_total):
        self.seen["finish"] = (np.array(counters), n_total, self.b["ub"].numpy().copy(),
                               self.b["ubv"].numpy().copy())
        return "stats"


def _shard_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = 101
        lo, hi = mg.shard_bounds(N, world, rank)
        api = MockShardAPI(rank)
        out = mg.integrate_sharded(api, mg.DistExchange(dist), np.zeros((hi - lo, 3)), lo, N, None, 0.5)
        q.put((rank, out, api.seen))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_frame_exchanges():
    import torch.multiprocessing as tmp
    world, N = 2, 101
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=180) for _ in procs), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    data = [_rank_data(r, mg.shard_bounds(N, world, r)[1] - mg.shard_bounds(N, world, r)[0]) for r in range(world)]
    kmin = np.minimum.reduce([d["kstar"] for d in data])
    ub1 = np.minimum.reduce([d["ub"] for d in data])
    ubv1 = np.maximum.reduce([d["ubv"] for d in data])
    rem = kmin < BIG
    ub2 = np.minimum.reduce([np.where(rem, d["ub2"], ub1) for d in data])
    ubv2 = np.maximum.reduce([np.where(rem, d["ubv2"], ubv1) for d in data])
    for rank, out, seen in res:
        assert out == "stats"
        lo, hi = mg.shard_bounds(N, world, rank)
        assert seen["ingest"] == (hi - lo, lo, N)
        pairs, cells, z, var = seen["update"]
        assert np.array_equal(pairs, np.stack([d["drift"] for d in data]))          # rank order
        assert np.array_equal(cells, np.concatenate([d["cells"] for d in data]))    # scan order
        assert np.array_equal(z, np.concatenate([d["z"] for d in data]))
        assert np.array_equal(var, np.concatenate([d["var"] for d in data]))
        assert np.array_equal(seen["kstar"], kmin)                                   # MIN k*
        assert np.array_equal(seen["ub1"], ub1) and np.array_equal(seen["ubv1"], ubv1)
        counters, n_total, ub_f, ubv_f = seen["finish"]
        assert np.array_equal(counters, np.sum([d["counters"] for d in data], axis=0)) and n_total == N
        assert np.array_equal(ub_f, ub2) and np.array_equal(ubv_f, ubv2)             # 2nd exchange


# ----------------------------------------------------------------- group API (host side)
def test_group_bounds_whole_tiles_in_scan_order(product):
    """relief_gpu_group_bounds: contiguous batches in rank order, every batch but the tail a whole
    number of 2048-point radix tiles (so the gathered arrays equal the single-GPU ones)."""
    import paper_2204_12876_b200 as pk
    for n in (0, 1, 2047, 2048, 2049, 19_477, 262_144, 1_000_064):
        for G in (1, 2, 3, 4, 5, 8):
            spans = [pk.group_bounds(product, n, G, r) for r in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            for lo, hi in spans:
                assert lo % 2048 == 0 or lo == hi == n  # trailing ranks of a short frame are empty
                assert hi == n or (hi - lo) % 2048 == 0
    with pytest.raises(pk.ReliefError):
        pk.group_bounds(product, 10, 2, 2)


def _id_worker(rank, world, port, q, lib_path):
    import torch.distributed as dist
    import paper_2204_12876_b200 as pk
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lib = pk.load_library(lib_path, gpu_api=True)
        uid, ranks, r = mg.broadcast_unique_id(lib, dist)
        q.put((rank, ranks, r, uid))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_nccl_id_broadcast(product):
    """create_nccl_group's id exchange: every rank receives rank 0's 128-byte NCCL id."""
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_worker, args=(r, 2, port, q, product._relief_path)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, n0, g0, u0), (r1, n1, g1, u1) = out
    assert (n0, n1, g0, g1) == (2, 2, 0, 1)
    assert len(u0) == 128 and u0 == u1 and any(u0)
