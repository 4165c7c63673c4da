"""Multi-GPU plumbing: one process per GPU over torch.distributed.

Detect + describe needs no exchange (independent volumes):
ranks take contiguous shards of the volume / subject list (`shard_range`).
Database matching (configs[4]) has exactly one exchange: the descriptor
tables of all ranks are all-gathered (NCCL over NVLink on GPUs, gloo in the CPU
tests) into one database, then every rank matches its own subjects against
it, excluding each query subject's own rows -- the composition
``nearest_neighbor_matches(desc_i, concat_{j != i} desc_j)`` of the reference
API (match.py:81-121) for every subject i.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ParameterError


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of range(n) for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ParameterError(f"bad rank {rank} / world {world}")
    return n * rank // world, n * (rank + 1) // world


def gather_rows(local, group=None):
    """All-gather a (n_local, ...) tensor with per-rank n_local; returns the
    concatenation in rank order (same tensor on every rank) and the counts."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if local.is_cuda and dist.get_backend(group) != "nccl":
        # gloo has no CUDA all-gather: stage through the host (multi-rank tests on one GPU)
        db, counts = gather_rows(local.cpu(), group)
        return db.to(local.device), counts
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    counts = [int(s.item()) for s in sizes]
    m = max(counts) if counts else 0
    pad = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)]), counts


def gather_database(desc, subjects, group=None):
    """All-gather descriptor rows and their subject ids.  Each rank must hold
    whole subjects, sorted by id, and ranks must hold increasing id ranges, so
    the database is in subject-id order.  Returns (db, subject_of_row,
    {subject: (lo, hi)})."""
    db, _ = gather_rows(desc, group)
    subj, _ = gather_rows(subjects.to(desc.device) if hasattr(subjects, "to") else subjects, group)
    s = subj.cpu().numpy()
    if len(s) and np.any(np.diff(s) < 0):
        raise ParameterError("database rows are not grouped by increasing subject id across ranks")
    ranges = {}
    if len(s):
        cuts = np.flatnonzero(np.diff(s)) + 1
        starts = np.concatenate([[0], cuts])
        ends = np.concatenate([cuts, [len(s)]])
        for a, b in zip(starts, ends):
            ranges[int(s[a])] = (int(a), int(b))
    return db, subj, ranges


def match_database(local: dict, ratio_max: float = 0.9, metric: str = "euclidean", group=None) -> dict:
    """{subject: descriptor array} for this rank's subjects -> {subject:
    (best_index, d1, d2, keep)} against all other subjects' descriptors (indices
    into concat of the other subjects in id order).  Rank descriptors whose
    values all fit in int8 (every rank decides the same way: the min / max are
    all-reduced) travel as int8 and run on the tensor-core kernel; any other
    integer or float rows go through the fp64 kernel (nearest_neighbor_matches'
    own choice, match.py _prepare).  Packed BRIEF bits travel as uint8.  A
    subject with no descriptors gets empty arrays (the reference composition
    returns no matches for an empty query)."""
    t = _lib.torch()
    ids = sorted(local)
    if metric not in ("hamming", "euclidean"):
        raise ParameterError(f"unknown metric {metric!r}")
    arrs = [np.asarray(local[i]) for i in ids]
    width = next((a.shape[1] for a in arrs if a.ndim == 2 and a.size), None)
    if width is None:
        width = 8 if metric == "hamming" else 64
    arrs = [a.reshape(len(a), width) if a.size else np.zeros((0, width), a.dtype if a.size else np.int64) for a in arrs]
    if metric == "hamming":
        rows = np.concatenate([a.astype(np.uint8) for a in arrs]) if arrs else np.zeros((0, width), np.uint8)
        pad = (-rows.shape[1]) % 8
        code = 0
    else:
        # range test per subject array, then one concatenation straight into the transfer dtype (the
        # configs[4] database is ~211 MB on the host: every extra pass over it is tens of ms)
        nonempty = [a for a in arrs if a.size]
        integral = all(a.dtype.kind in "iub" for a in nonempty)
        lo_hi = np.array([min((a.min() for a in nonempty), default=0), max((a.max() for a in nonempty), default=0),
                          0 if integral else 1], dtype=np.float64)
        lo_hi = _allreduce_minmax(lo_hi, group)
        if lo_hi[2] == 0 and lo_hi[0] >= -128 and lo_hi[1] <= 127:
            rows = np.concatenate([a.astype(np.int8, copy=False) for a in arrs]) if arrs else np.zeros((0, width), np.int8)
            pad = (-rows.shape[1]) % 32 if rows.shape[1] <= 128 else (-rows.shape[1]) % 4
            code = 1
        else:
            rows = (np.concatenate([a.astype(np.float64, copy=False) for a in arrs]) if arrs
                    else np.zeros((0, width), np.float64))
            pad = 0
            code = 2
    if pad:
        rows = np.pad(rows, ((0, 0), (0, pad)))
    subj = np.concatenate([np.full(len(a), i, np.int32) for i, a in zip(ids, arrs)]) if arrs else np.zeros(0, np.int32)
    d_rows = t.from_numpy(np.ascontiguousarray(rows)).cuda()
    db, _, ranges = gather_database(d_rows, t.from_numpy(subj).cuda(), group)
    out = {}
    dim = db.shape[1]
    empty = (np.zeros(0, np.int32), np.zeros(0), np.zeros(0), np.zeros(0, np.uint8))
    if code == 1 and dim % 32 == 0 and dim <= 128 and len(rows):
        # one tensor-core launch for every local query row, each excluding its
        # own subject's rows (vk_match_rows_excluding)
        n = len(rows)
        ex = np.empty((n, 2), dtype=np.int32)
        off = 0
        for i, a in zip(ids, arrs):
            ex[off: off + len(a)] = ranges.get(i, (0, 0))
            off += len(a)
        row_ex = t.from_numpy(ex).cuda()
        best = t.empty(n, dtype=t.int32, device="cuda")
        d1 = t.empty(n, dtype=t.float64, device="cuda")
        d2 = t.empty(n, dtype=t.float64, device="cuda")
        keep = t.empty(n, dtype=t.uint8, device="cuda")
        _lib.call("vk_match_rows_excluding", d_rows.data_ptr(), n, db.data_ptr(), db.shape[0], dim, float(ratio_max),
                  row_ex.data_ptr(), best.data_ptr(), d1.data_ptr(), d2.data_ptr(), keep.data_ptr(), _lib.stream_ptr())
        hb, h1, h2, hk = best.cpu().numpy(), d1.cpu().numpy(), d2.cpu().numpy(), keep.cpu().numpy()
        off = 0
        for i, a in zip(ids, arrs):
            sl = slice(off, off + len(a))
            out[i] = (hb[sl], h1[sl], h2[sl], hk[sl])
            off += len(a)
        return out
    off = 0
    for i, a in zip(ids, arrs):
        n = len(a)
        q = d_rows[off: off + n]
        off += n
        if n == 0:
            out[i] = empty
            continue
        lo, hi = ranges[i]
        best = t.empty(n, dtype=t.int32, device="cuda")
        d1 = t.empty(n, dtype=t.float64, device="cuda")
        d2 = t.empty(n, dtype=t.float64, device="cuda")
        keep = t.empty(n, dtype=t.uint8, device="cuda")
        _lib.call("vk_match_excluding", code, q.data_ptr(), n, db.data_ptr(), db.shape[0], db.shape[1],
                  float(ratio_max), lo, hi, best.data_ptr(), d1.data_ptr(), d2.data_ptr(), keep.data_ptr(),
                  _lib.stream_ptr())
        out[i] = (best.cpu().numpy(), d1.cpu().numpy(), d2.cpu().numpy(), keep.cpu().numpy())
    return out


def _allreduce_minmax(v: np.ndarray, group=None) -> np.ndarray:
    """[min, max, any_float] reduced over the ranks (identity without a process group)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return v
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    lo = torch.tensor([v[0]], dtype=torch.float64, device=dev)
    hi = torch.tensor([v[1], v[2]], dtype=torch.float64, device=dev)
    dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
    return np.array([lo.item(), hi[0].item(), hi[1].item()])
