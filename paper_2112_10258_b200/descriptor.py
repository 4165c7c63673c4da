"""Keypoint descriptors on the GPU -- drop-in for volkey descriptor.py.

Same names and semantics as descriptor.py:30-316.  ``describe_all`` and
``sift_rank_descriptor`` run ``vk_describe_siftrank``; BRIEF / RRIEF run
``vk_describe_patch`` (patch extraction, pre-blur and pair sampling fused in
one CTA per frame).  The per-record building blocks the reference exposes
(``extract_patch``, ``preblur_patch``, ``brief_descriptor``,
``rrief_descriptor``) run the same device code one stage at a time
(``vk_extract_patches``, the pyramid blur, ``vk_sample_trilinear``).
``sample_point_pairs`` is the reference's host RNG draw (a per-run constant
table, uploaded once); ``pack_bits`` / ``pack_ranks`` and their inverses are
host byte helpers.
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
class Patch:
    """descriptor.py:37-42: (side, side, side) fp32 resample, [x, y, z]."""

    side: int
    data: np.ndarray


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


def extract_patch(pyr, kp, frame, side: int = 15) -> Patch:
    """descriptor.py:96-111 on the GPU: side^3 fp64 trilinear samples of the
    unblurred source spanning +-2 sigma along the frame axes, cast to fp32."""
    from .stages import run_patches

    if side < 1 or side % 2 == 0:
        raise ParameterError(f"patch side must be odd and >= 1, got {side}")
    if pyr.source is None:
        raise ParameterError("pyramid carries no source volume for patch extraction")
    data = run_patches(pyr, [kp], [(0, frame.rotation)], side)[0]
    data.setflags(write=False)
    return Patch(side, data)


def preblur_patch(p: Patch, blur_sigma: float) -> Patch:
    """descriptor.py:196-202: separable Gaussian blur of the patch (the
    pyramid's blur kernels, replicate borders); 0 returns the patch."""
    from .scalespace import convolve_array

    if blur_sigma < 0:
        raise ParameterError(f"blur_sigma must be >= 0, got {blur_sigma}")
    if blur_sigma == 0:
        return p
    return Patch(p.side, convolve_array(p.data, T.gaussian_kernel(blur_sigma)))


def _pair_samples(patch: Patch, pairs: PointPairSet) -> tuple[np.ndarray, np.ndarray]:
    """descriptor.py:205-212: fp64 trilinear samples of the pair endpoints."""
    from .volume import sample_trilinear_array

    center = (patch.side - 1) / 2.0
    scale = (patch.side - 1) / (2.0 * PAIR_SUPPORT_RADIUS) / pairs.sigma_unit
    return (sample_trilinear_array(patch.data, center + pairs.p1 * scale),
            sample_trilinear_array(patch.data, center + pairs.p2 * scale))


def brief_descriptor(p: Patch, pairs: PointPairSet) -> BriefDescriptor:
    """descriptor.py:215-218: bit k = sample(p1_k) - sample(p2_k) > 0."""
    s1, s2 = _pair_samples(p, pairs)
    return BriefDescriptor((s1 - s2 > 0).astype(np.uint8))


def rrief_descriptor(p: Patch, pairs: PointPairSet) -> RriefDescriptor:
    """descriptor.py:221-224: stable ranks of the pair differences."""
    s1, s2 = _pair_samples(p, pairs)
    return RriefDescriptor(rank_vector(s1 - s2))


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


def pack_bits(bits: np.ndarray) -> bytes:
    """descriptor.py:319-321: 0/1 bits MSB-first into bytes."""
    return np.packbits(np.asarray(bits, dtype=np.uint8), bitorder="big").tobytes()


def unpack_bits(blob: bytes, n: int) -> np.ndarray:
    """descriptor.py:324-325."""
    return np.unpackbits(np.frombuffer(blob, dtype=np.uint8), bitorder="big")[:n]


def _bit_weights(bits_per_rank: int) -> np.ndarray:
    return np.left_shift(1, np.arange(bits_per_rank - 1, -1, -1, dtype=np.int64))


def pack_ranks(ranks: np.ndarray, bits_per_rank: int = 6) -> bytes:
    """descriptor.py:328-334: each rank as ``bits_per_rank`` bits, MSB first,
    concatenated and packed big-endian (64 ranks -> 48 bytes)."""
    r = np.asarray(ranks, dtype=np.int64)
    if r.min() < 0 or r.max() >= (1 << bits_per_rank):
        raise ParameterError(f"ranks out of range for {bits_per_rank}-bit packing")
    bits = (r[:, None] & _bit_weights(bits_per_rank)[None, :]) != 0
    return np.packbits(bits.reshape(-1).astype(np.uint8), bitorder="big").tobytes()


def unpack_ranks(blob: bytes, n: int, bits_per_rank: int = 6) -> np.ndarray:
    """descriptor.py:337-340."""
    bits = np.unpackbits(np.frombuffer(blob, dtype=np.uint8), bitorder="big")[: n * bits_per_rank]
    return bits.reshape(n, bits_per_rank).astype(np.int64) @ _bit_weights(bits_per_rank)
