"""N>1 host path on CPU: world_size-2 gloo processes exercise the reductions and the batch split
bench.py / the sharded mode rely on (the GPU legs run one process per B200 over NCCL)."""
from __future__ import annotations

import os
import socket

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
