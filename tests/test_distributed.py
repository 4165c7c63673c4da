"""Multi-process host logic over gloo (world_size 2, CPU): sharding, the
variable-length database all-gather, and the bench's max-over-ranks timing."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2112_10258_b200.distributed import gather_database, gather_rows, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(rank)
        # rank r holds subjects [2r, 2r+1] with different row counts
        ids = [2 * rank, 2 * rank + 1]
        counts = [3 + rank, 5 - rank]
        rows = [rng.integers(-5, 60, size=(c, 64)).astype(np.int8) for c in counts]
        desc = torch.from_numpy(np.concatenate(rows))
        subj = torch.from_numpy(np.concatenate([np.full(c, i, np.int32) for i, c in zip(ids, counts)]))
        db, s, ranges = gather_database(desc, subj)
        # max-over-ranks timing as bench.py does it
        t = torch.tensor([10.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        g, cnt = gather_rows(torch.arange(rank + 1, dtype=torch.int64).reshape(-1, 1))
        q.put((rank, db.numpy(), s.numpy(), ranges, float(t.item()), g.numpy().ravel().tolist(), cnt))
    finally:
        dist.destroy_process_group()


def test_shard_range_partitions():
    for n in (0, 1, 7, 512):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


def test_gather_database_gloo_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda r: r[0])
    (_, db0, s0, r0, t0, g0, c0), (_, db1, s1, r1, t1, g1, c1) = res
    assert np.array_equal(db0, db1) and np.array_equal(s0, s1) and r0 == r1
    assert t0 == t1 == 11.0
    assert g0 == g1 == [0, 0, 1] and c0 == [1, 2]
    # subject order and ranges: rank 0 -> subjects 0 (3 rows), 1 (5 rows); rank 1 -> 2 (4 rows), 3 (4 rows)
    assert r0 == {0: (0, 3), 1: (3, 8), 2: (8, 12), 3: (12, 16)}
    r = np.random.default_rng(0)
    expect0 = np.concatenate([r.integers(-5, 60, size=(c, 64)) for c in (3, 5)])
    assert np.array_equal(db0[:8], expect0.astype(np.int8))
