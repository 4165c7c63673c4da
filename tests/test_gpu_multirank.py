"""Multi-rank code paths on ONE GPU (the only hardware this run has): two
processes share cuda:0 over a gloo process group.

* bench.py's sharded run (torchrun, 2 ranks): each rank extracts its own
  shard, the timing is the max over ranks, and the cross-rank parity block
  shows both ranks' digests equal to each other AND to the unmodified
  reference's (tests/golden/bench.npz).
* distributed.match_database at world 2 == the oracle composition of
  match.py:81-121 (nearest_neighbor_matches(desc_i, concat_{j != i} desc_j)),
  including an empty subject."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_on_one_gpu():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--backend", "gloo", "--steps", "2", "--warmup", "3", "--batch", "4", "--streams", "2",
           "--no-cpu-baseline", "--no-matching", "--no-extras"]
    res = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-4000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    rp = d["rank_parity"]
    assert rp["ranks"] == 2 and rp["all_ranks_equal"], rp
    assert rp["matches_reference"], rp
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 4 * 145 * 174 * 145 * 4


def _db_worker(rank, world, port, subjects, q):
    import torch
    import torch.distributed as dist

    from paper_2112_10258_b200.distributed import match_database, shard_range

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ids = sorted(subjects)
        lo, hi = shard_range(len(ids), rank, world)
        local = {i: subjects[i] for i in ids[lo:hi]}
        out = match_database(local, 0.9, "euclidean")
        q.put((rank, {i: tuple(np.asarray(x) for x in v) for i, v in out.items()}))
    finally:
        dist.destroy_process_group()


def test_match_database_world2_equals_oracle_composition():
    import torch.multiprocessing as mp

    from oracle import volkey_oracle as O

    rng = np.random.default_rng(5)
    subjects = {i: np.stack([rng.permutation(64) for _ in range(int(rng.integers(20, 60)))]).astype(np.int64)
                for i in range(9)}
    subjects[9] = np.zeros((0, 64), np.int64)  # no descriptors
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_db_worker, args=(r, 2, port, subjects, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        _, part = q.get(timeout=300)
        got.update(part)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sorted(got) == sorted(subjects)
    assert len(got[9][0]) == 0
    for i, a in subjects.items():
        if not len(a):
            continue
        others = np.concatenate([subjects[j] for j in sorted(subjects) if j != i])
        ref = O.nn_match(a, others, 0.9, "euclidean")
        best, d1, d2, keep = got[i]
        mine = [(qq, int(best[qq]), float(d1[qq]), float(d2[qq])) for qq in np.flatnonzero(keep)]
        assert mine == ref, f"subject {i}"
