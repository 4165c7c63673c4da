"""Nearest-neighbour descriptor matching on the GPU -- drop-in for the
in-scope part of volkey match.py (match.py:19-27, 64-121, 362-370).

``nearest_neighbor_matches`` runs ``vk_match``: exact integer arithmetic for
rank (int8, tcgen05 tensor cores) and packed-bit (popcount) descriptors, fp64
for anything else.  The 7-DOF Hough consensus (match.py:124-359) and
``match_records`` live in consensus.py; ``match_descriptors`` is
match_records without the consensus step.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ParameterError

_POPCOUNT = np.array([bin(i).count("1") for i in range(256)], dtype=np.uint8)


@dataclass(frozen=True)
class Match:
    index_a: int
    index_b: int
    distance: float
    second_distance: float


def hamming_distances(a_packed: np.ndarray, b_packed: np.ndarray) -> np.ndarray:
    """match.py:64-67: pairwise popcount distances (full matrix, on the GPU)."""
    t = _lib.torch()
    a = t.from_numpy(np.ascontiguousarray(a_packed, dtype=np.uint8)).cuda()
    b = t.from_numpy(np.ascontiguousarray(b_packed, dtype=np.uint8)).cuda()
    lut = t.from_numpy(_POPCOUNT).cuda().long()
    x = t.bitwise_xor(a[:, None, :], b[None, :, :]).long()
    return lut[x].sum(dim=2).double().cpu().numpy()


def euclidean_distances(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """match.py:70-78 (full matrix, fp64 on the GPU).  Integer-valued rows
    (ranks, int8 values) give the reference's matrix bit for bit (every product
    and sum is an exact fp64 integer); non-integer float rows follow cuBLAS's
    summation order rather than OpenBLAS's (last-ulp differences)."""
    t = _lib.torch()
    A = t.from_numpy(np.asarray(a, dtype=np.float64)).cuda()
    B = t.from_numpy(np.asarray(b, dtype=np.float64)).cuda()
    d2 = (A * A).sum(1)[:, None] + (B * B).sum(1)[None, :] - 2.0 * (A @ B.T)
    return t.sqrt(t.clamp(d2, min=0.0)).cpu().numpy()


def _prepare(a: np.ndarray, b: np.ndarray, metric: str):
    """Pick the kernel variant and lay the rows out for it."""
    t = _lib.torch()
    if metric == "hamming":
        a8, b8 = np.asarray(a, dtype=np.uint8), np.asarray(b, dtype=np.uint8)
        nbytes = a8.shape[1]
        pad = (-nbytes) % 8
        a8 = np.pad(a8, ((0, 0), (0, pad)))
        b8 = np.pad(b8, ((0, 0), (0, pad)))
        return 0, t.from_numpy(np.ascontiguousarray(a8)).cuda(), t.from_numpy(np.ascontiguousarray(b8)).cuda(), nbytes + pad
    a_, b_ = np.asarray(a), np.asarray(b)
    if a_.dtype.kind in "iub" and b_.dtype.kind in "iub" and a_.size and b_.size \
            and min(a_.min(), b_.min()) >= -128 and max(a_.max(), b_.max()) <= 127:
        dim = a_.shape[1]
        pad = (-dim) % 32 if dim <= 128 else (-dim) % 4  # zero columns: same dots and norms
        a8 = np.pad(a_.astype(np.int8), ((0, 0), (0, pad)))
        b8 = np.pad(b_.astype(np.int8), ((0, 0), (0, pad)))
        return 1, t.from_numpy(np.ascontiguousarray(a8)).cuda(), t.from_numpy(np.ascontiguousarray(b8)).cuda(), dim + pad
    a64 = np.ascontiguousarray(a_, dtype=np.float64)
    b64 = np.ascontiguousarray(b_, dtype=np.float64)
    return 2, t.from_numpy(a64).cuda(), t.from_numpy(b64).cuda(), a64.shape[1]


def nn_device(a: np.ndarray, b: np.ndarray, ratio_max: float, metric: str):
    """Raw per-query (best, d1, d2, keep) arrays from vk_match."""
    t = _lib.torch()
    code, A, B, dim = _prepare(a, b, metric)
    na, nb = A.shape[0], B.shape[0]
    best = t.empty(max(na, 1), dtype=t.int32, device="cuda")
    d1 = t.empty(max(na, 1), dtype=t.float64, device="cuda")
    d2 = t.empty(max(na, 1), dtype=t.float64, device="cuda")
    keep = t.empty(max(na, 1), dtype=t.uint8, device="cuda")
    _lib.call("vk_match", code, A.data_ptr(), na, B.data_ptr(), nb, dim, float(ratio_max), best.data_ptr(),
              d1.data_ptr(), d2.data_ptr(), keep.data_ptr(), _lib.stream_ptr())
    return best[:na].cpu().numpy(), d1[:na].cpu().numpy(), d2[:na].cpu().numpy(), keep[:na].cpu().numpy()


def nearest_neighbor_matches(a: np.ndarray, b: np.ndarray, ratio_max: float = 0.9, metric: str = "euclidean",
                             workers: int = 1) -> list[Match]:
    """match.py:81-121: nearest + second nearest, ratio test, ties to the lower index."""
    if metric not in ("hamming", "euclidean"):
        raise ParameterError(f"unknown metric {metric!r}")
    if not 0 < ratio_max <= 1:
        raise ParameterError(f"ratio_max must be in (0, 1], got {ratio_max}")
    if len(b) < 2:
        raise ParameterError(f"need at least 2 reference descriptors, got {len(b)}")
    if workers < 1:
        raise ParameterError(f"workers must be >= 1, got {workers}")
    if len(a) == 0:
        return []
    best, d1, d2, keep = nn_device(a, b, ratio_max, metric)
    idx = np.nonzero(keep)[0]
    bl, d1l, d2l = best[idx].tolist(), d1[idx].tolist(), d2[idx].tolist()
    return [Match(int(i), bl[k], d1l[k], d2l[k]) for k, i in enumerate(idx.tolist())]


def match_descriptors(records_a, records_b, config):
    """match_records (match.py:362-370) up to the consensus step: (matches, kind)."""
    from .descriptor import descriptor_array

    kind = config.descriptor
    metric = "hamming" if kind == "brief" else "euclidean"
    a = descriptor_array(records_a, kind)
    b = descriptor_array(records_b, kind)
    return nearest_neighbor_matches(a, b, config.ratio_max, metric, config.workers), kind


_CONSENSUS = ("SimilarityTransform7DOF", "rotation_angle_deg", "HoughSettings", "ConsensusResult", "vote_transform",
              "similarity_from_correspondences", "hough_consensus", "settings_from_config", "match_records",
              "count_inlier_matches")


def __getattr__(name):
    """volkey.match also holds the consensus API (match.py:31-401): re-export
    it lazily from consensus.py (which imports this module)."""
    if name in _CONSENSUS:
        from . import consensus

        return getattr(consensus, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
