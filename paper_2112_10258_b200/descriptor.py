"""Keypoint descriptors on the GPU -- drop-in for volkey descriptor.py.

Same names and semantics as descriptor.py:30-316.  ``describe_all`` and
``sift_rank_descriptor`` run ``vk_describe_siftrank``; BRIEF / RRIEF run
``vk_describe_patch`` (patch extraction, pre-blur and pair sampling fused in
one CTA per frame).  ``sample_point_pairs`` is the reference's host RNG draw
(a per-run constant table, uploaded once).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Literal, Sequence

import numpy as np

from . import tables as T
from .errors import ParameterError

Kind = Literal["siftrank", "brief", "rrief"]
KINDS = ("siftrank", "brief", "rrief")
SIFT_RANK_LENGTH = 64
PAIR_SUPPORT_RADIUS = T.PAIR_SUPPORT_RADIUS


@dataclass(frozen=True)
class PointPairSet:
    method: int
    n: int
    sigma_unit: float
    seed: int
    p1: np.ndarray
    p2: np.ndarray


@dataclass(frozen=True)
class SiftRankDescriptor:
    ranks: np.ndarray


@dataclass(frozen=True)
class BriefDescriptor:
    bits: np.ndarray


@dataclass(frozen=True)
class RriefDescriptor:
    ranks: np.ndarray


@dataclass(frozen=True)
class DescriptorRecord:
    keypoint: object
    frame: object
    descriptor: SiftRankDescriptor | BriefDescriptor | RriefDescriptor


def rank_vector(values) -> np.ndarray:
    """Stable ranks (descriptor.py:77-83).  Host helper for callers; the GPU
    kernels compute the same ranks in-kernel (csrc/vk_describe.cu)."""
    v = np.asarray(values)
    r = np.empty(len(v), dtype=np.int64)
    r[np.argsort(v, kind="stable")] = np.arange(len(v))
    return r


def _patch_grid(side: int) -> np.ndarray:
    a = T.patch_axis(side)
    g = np.stack([x.ravel() for x in np.meshgrid(a, a, a, indexing="ij")], axis=1)
    g.setflags(write=False)
    return g


def sample_point_pairs(method: int, n: int, sigma_unit: float = 1.0, seed: int = 0) -> PointPairSet:
    """descriptor.py:145-193: five deterministic point-pair strategies."""
    if method not in (1, 2, 3, 4, 5):
        raise ParameterError(f"point-pair method must be 1..5, got {method}")
    if n < 1:
        raise ParameterError(f"pair count must be >= 1, got {n}")
    if sigma_unit <= 0:
        raise ParameterError(f"sigma_unit must be > 0, got {sigma_unit}")
    rng = np.random.default_rng(seed)
    radius = PAIR_SUPPORT_RADIUS * sigma_unit
    zeros = np.zeros((n, 3))

    def redraw(draw):
        pts = draw()
        while True:
            bad = np.linalg.norm(pts, axis=1) > radius
            if not bad.any():
                return pts
            pts[bad] = draw()[bad]

    def uniform():
        return redraw(lambda: rng.uniform(-radius, radius, size=(n, 3)))

    def normal(center):
        return redraw(lambda: center + rng.normal(0.0, sigma_unit, size=(n, 3)))

    if method == 1:
        p1 = uniform()
        p2 = uniform()
    elif method == 2:
        p1 = normal(zeros)
        p2 = normal(zeros)
    elif method == 3:
        p1 = normal(zeros)
        p2 = normal(p1)
    elif method == 4:
        p1, p2 = zeros, normal(zeros)
    else:
        verts = []
        for axis in range(3):
            for s in (1.0, -1.0):
                v = [0.0, 0.0, 0.0]
                v[axis] = s
                verts.append(v)
        for i in range(3):
            for j in range(i + 1, 3):
                for si in (1.0, -1.0):
                    for sj in (1.0, -1.0):
                        v = [0.0, 0.0, 0.0]
                        v[i], v[j] = si, sj
                        verts.append([c / math.sqrt(2.0) for c in v])
        octa = np.array(verts)
        grid = np.array([r * d for r in np.array([0.5, 1.0, 1.5, 2.0]) * sigma_unit for d in octa])
        p1, p2 = zeros, grid[np.arange(n) % len(grid)]
    p1.setflags(write=False)
    p2.setflags(write=False)
    return PointPairSet(method, n, float(sigma_unit), int(seed), p1, p2)


def sift_rank_descriptor(pyr, kp, frame, radius_factor: float = 4.0) -> SiftRankDescriptor:
    """descriptor.py:227-263 for one (keypoint, frame) on the GPU."""
    from .stages import run_descriptors

    out = run_descriptors(pyr, [kp], [(0, frame.rotation)], "siftrank", radius_factor=radius_factor)
    return SiftRankDescriptor(out[0].astype(np.int64))


def describe_all(pyr, oriented: Sequence, kind: Kind = "siftrank", pairs: PointPairSet | None = None,
                 patch_side: int = 15, blur_sigma: float = 0.95, radius_factor: float = 4.0,
                 workers: int = 1) -> tuple[list[DescriptorRecord], int]:
    """descriptor.py:266-306: one descriptor per (keypoint, frame), input order."""
    from .stages import run_descriptors

    if kind not in KINDS:
        raise ParameterError(f"unknown descriptor kind {kind!r}")
    if kind != "siftrank" and pairs is None:
        raise ParameterError(f"descriptor kind {kind!r} needs a PointPairSet")
    if workers < 1:
        raise ParameterError(f"workers must be >= 1, got {workers}")
    if not oriented:
        return [], 0
    index, kps, rots = {}, [], []
    for kp, frame in oriented:
        if id(kp) not in index:
            index[id(kp)] = len(kps)
            kps.append(kp)
        rots.append((index[id(kp)], frame.rotation))
    out = run_descriptors(pyr, kps, rots, kind, pairs, patch_side, blur_sigma, radius_factor)
    return records_from(oriented, out, kind, pairs.n if pairs is not None else 64), 0


def records_from(oriented, out: np.ndarray, kind: str, npairs: int = 64) -> list[DescriptorRecord]:
    recs = []
    if kind == "siftrank":
        ranks = out.astype(np.int64)
        for (kp, fr), r in zip(oriented, ranks):
            recs.append(DescriptorRecord(kp, fr, SiftRankDescriptor(r)))
    elif kind == "brief":
        bits = np.unpackbits(out, axis=1, bitorder="big")[:, :npairs]
        for (kp, fr), b in zip(oriented, bits):
            recs.append(DescriptorRecord(kp, fr, BriefDescriptor(b)))
    else:
        ranks = out.astype(np.int64)
        for (kp, fr), r in zip(oriented, ranks):
            recs.append(DescriptorRecord(kp, fr, RriefDescriptor(r)))
    return recs


def descriptor_array(records: Sequence[DescriptorRecord], kind: Kind) -> np.ndarray:
    """descriptor.py:309-316: packed bits for brief, int64 ranks otherwise."""
    if not records:
        return np.zeros((0, 0), dtype=np.uint8 if kind == "brief" else np.int64)
    if kind == "brief":
        return np.packbits(np.stack([r.descriptor.bits for r in records]), axis=1, bitorder="big")
    return np.stack([r.descriptor.ranks for r in records])
