"""Host-side constant tables uploaded to the GPU.

These are the small per-configuration constants the reference also computes
on the host: Gaussian taps, the icosphere, integer balls and their Gaussian
windows, the 42 x 42 frame table, the patch grid and the BRIEF point pairs.
They are evaluated with the same numpy expressions as the reference (same
ufuncs, same evaluation order), so every table is bit-identical to the values
the reference uses -- including numpy's SIMD ``exp`` and OpenBLAS's ``dot``,
which a device re-implementation would not reproduce.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .errors import ParameterError


# ---------------------------------------------------------------- Gaussians
@dataclass(frozen=True)
class GaussianKernel1D:
    """Sampled normalised 1-D Gaussian, radius ceil(3 sigma) (scalespace.py:35-42)."""

    sigma: float
    radius: int
    weights: np.ndarray


@lru_cache(maxsize=256)
def gaussian_kernel(sigma: float) -> GaussianKernel1D:
    if sigma <= 0:
        raise ParameterError(f"sigma must be > 0, got {sigma}")
    radius = max(1, math.ceil(3.0 * sigma))
    k = np.arange(-radius, radius + 1, dtype=np.float64)
    w = np.exp(-(k ** 2) / (2.0 * sigma * sigma))
    w /= w.sum()
    w = w.astype(np.float32)
    w.setflags(write=False)
    return GaussianKernel1D(float(sigma), radius, w)


def incremental_sigma(current: float, target: float) -> float:
    """scalespace.py:154-155."""
    return math.sqrt(max(target * target - current * current, 0.0))


def octave_sigmas(base_sigma: float, levels: int):
    """kappa and octave-local sigmas (scalespace.py:179-181)."""
    kappa = 2.0 ** (1.0 / (levels - 3))
    return kappa, [base_sigma * kappa ** i for i in range(levels)]


# --------------------------------------------------------------- directions
@lru_cache(maxsize=1)
def icosphere_directions() -> np.ndarray:
    """42 lexsorted unit vectors: icosahedron vertices + edge midpoints (orient.py:34-60)."""
    phi = (1.0 + math.sqrt(5.0)) / 2.0
    pts = []
    for a in (-1.0, 1.0):
        for b in (-phi, phi):
            pts += [(0.0, a, b), (a, b, 0.0), (b, 0.0, a)]
    v = np.array(pts, dtype=np.float64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    d2 = np.sum((v[:, None, :] - v[None, :, :]) ** 2, axis=2)
    edge = np.min(d2[d2 > 1e-9])
    mids = []
    for i in range(len(v)):
        for j in range(i + 1, len(v)):
            if abs(d2[i, j] - edge) < 1e-9:
                m = v[i] + v[j]
                mids.append(m / np.linalg.norm(m))
    allv = np.vstack([v, np.array(mids)])
    allv = allv[np.lexsort((allv[:, 2].round(9), allv[:, 1].round(9), allv[:, 0].round(9)))]
    allv.setflags(write=False)
    return allv


@lru_cache(maxsize=1)
def icosphere_structure() -> np.ndarray:
    """int32[12 + 60 + 60]: indices (into icosphere_directions()) of the 12
    icosahedron vertices, then for each vertex the 5 edge midpoints around it,
    then for each vertex the same 5 midpoints by neighbour kind for the fast
    argmax of csrc/vk_orient.cu: vertex (p: +-1, q: +-phi, r: 0) in its group's
    (p, q, r) axes meets (p: s_p phi, r: +1), (p: s_p phi, r: -1),
    (q: s_q, r: +phi), (q: s_q, r: -phi), (p: -s_p, q: s_q phi)."""
    dirs = icosphere_directions()
    phi = (1.0 + math.sqrt(5.0)) / 2.0
    pts = []
    for a in (-1.0, 1.0):
        for b in (-phi, phi):
            pts += [(0.0, a, b), (a, b, 0.0), (b, 0.0, a)]
    v = np.array(pts, dtype=np.float64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    vidx = [int(np.argmin(np.linalg.norm(dirs - p, axis=1))) for p in v]
    d2 = np.sum((v[:, None, :] - v[None, :, :]) ** 2, axis=2)
    edge = np.min(d2[d2 > 1e-9])
    adj = []
    for i in range(12):
        mids = []
        for j in range(12):
            if j != i and abs(d2[i, j] - edge) < 1e-9:
                m = v[i] + v[j]
                mids.append(int(np.argmin(np.linalg.norm(dirs - m / np.linalg.norm(m), axis=1))))
        assert len(mids) == 5
        adj.append(sorted(mids))
    fast = []
    axes = {0: (1, 2, 0), 1: (0, 1, 2), 2: (2, 0, 1)}  # group -> (p, q, r) axes (+-1, +-phi, 0 coordinates)
    for s in range(12):
        grp = s % 3
        pa, qa, ra = axes[grp]
        V = np.array(pts[s])
        sp, sq = np.sign(V[pa]), np.sign(V[qa])
        kinds = []
        for coef in ((sp * phi, 0.0, 1.0), (sp * phi, 0.0, -1.0), (0.0, sq, phi), (0.0, sq, -phi), (-sp, sq * phi, 0.0)):
            W = np.zeros(3)
            W[pa], W[qa], W[ra] = coef
            assert abs(np.sum((V - W) ** 2) - 4.0) < 1e-9  # an icosahedron edge
            m = V / np.linalg.norm(V) + W / np.linalg.norm(W)
            k = int(np.argmin(np.linalg.norm(dirs - m / np.linalg.norm(m), axis=1)))
            assert k in adj[s]
            kinds.append(k)
        fast += kinds
    out = np.array(vidx + [m for a in adj for m in a] + fast, dtype=np.int32)
    assert len(set(vidx)) == 12
    out.setflags(write=False)
    return out


ICO_LUT_N = 128          # cells per axis of the canonical face
ICO_LUT_DILATE = 2.0 ** -14  # cell dilation in (u, v): >> fp32 gradient / division error (~1e-6)
ICO_LUT_MARGIN = 1e-9    # required dot lead at every dilated corner: >> fp64 dot error (~1e-15)


def _ico_canonical(a: np.ndarray):
    """Canonical (p, q, r) of |g| components (r the largest; cyclic order
    kept) and the permutation id, exactly as csrc/vk_orient.cu computes them."""
    ax, ay, az = a[..., 0], a[..., 1], a[..., 2]
    perm = np.where((az >= ax) & (az >= ay), 0, np.where(ax >= ay, 1, 2))
    p = np.choose(perm, [ax, ay, az])
    q = np.choose(perm, [ay, az, ax])
    r = np.choose(perm, [az, ax, ay])
    return p, q, r, perm


def icosphere_lut() -> np.ndarray:
    """uint8[N*N + 42*24]: exact-argmax lookup for orientation binning.

    The 42 icosphere directions are invariant under axis sign flips and cyclic
    axis permutations, so np.argmax(g @ dirs.T) follows from the canonical
    point (u, v) = (p / r, q / r) in [0, 1]^2 of |g| (gnomonic projection onto
    the face of its largest component).  Voronoi boundaries are great circles,
    i.e. straight lines in (u, v), so a cell whose four corners, dilated by
    ICO_LUT_DILATE, all have the same nearest direction with a lead above
    ICO_LUT_MARGIN has that direction at every point within the dilation --
    including every gradient whose fp32 canonical coordinates land in it.
    Table entry = canonical direction index, or 255 for the ~2.7% of cells a
    boundary crosses (the kernel then takes its screened path).  The trailing
    42 x 3 x 8 map turns (canonical index, permutation, sign bits of g) into
    the index of the actual direction."""
    dirs = icosphere_directions()
    N, d = ICO_LUT_N, ICO_LUT_DILATE
    i = np.arange(N)
    lo, hi = i / N - d, (i + 1) / N + d
    best, pure = None, np.ones((N, N), bool)
    for uu, vv in ((lo[None, :], lo[:, None]), (hi[None, :], lo[:, None]), (lo[None, :], hi[:, None]),
                   (hi[None, :], hi[:, None])):
        uu, vv = np.broadcast_arrays(uu, vv)
        x = np.stack([uu, vv, np.ones_like(uu)], -1)  # (iv, iu) rows
        dots = x @ dirs.T
        top2 = np.sort(dots, -1)[..., -2:]
        a = np.argmax(dots, -1)
        pure &= (top2[..., 1] - top2[..., 0]) > ICO_LUT_MARGIN
        pure &= a == (a if best is None else best)
        best = a if best is None else best
    table = np.where(pure, best, 255).astype(np.uint8).reshape(-1)
    lmap = np.zeros(42 * 24, dtype=np.uint8)
    for c in range(42):
        C = dirs[c]
        for perm, A in enumerate(((C[0], C[1], C[2]), (C[2], C[0], C[1]), (C[1], C[2], C[0]))):
            for sb in range(8):
                D = np.array([-A[k] if (sb >> k) & 1 else A[k] for k in range(3)])
                k = int(np.argmin(np.linalg.norm(dirs - D, axis=1)))
                assert np.linalg.norm(dirs[k] - D) < 1e-12
                lmap[c * 24 + perm * 8 + sb] = k
    out = np.concatenate([table, lmap])
    out.setflags(write=False)
    return out


def frame_tables(dirs: np.ndarray):
    """For every (primary p, candidate secondary q): whether q's projection
    orthogonal to p is usable (norm > 1e-6) and the resulting right-handed
    frame [a1, a2, a1 x a2] (orient.py:151-167), evaluated with the reference's
    own numpy calls so the rotations are bit-identical."""
    dirs = np.asarray(dirs, dtype=np.float64)
    K = len(dirs)
    ok = np.zeros((K, K), dtype=np.uint8)
    rot = np.zeros((K, K, 3, 3), dtype=np.float64)
    for p in range(K):
        a1 = dirs[p]
        for q in range(K):
            if q == p:
                continue
            proj = dirs[q] - np.dot(dirs[q], a1) * a1
            nrm = np.linalg.norm(proj)
            if nrm > 1e-6:
                a2 = proj / nrm
                ok[p, q] = 1
                rot[p, q] = np.column_stack([a1, a2, np.cross(a1, a2)])
    return ok, rot


@lru_cache(maxsize=4)
def default_frame_tables():
    return frame_tables(icosphere_directions())


# -------------------------------------------------------------------- balls
@lru_cache(maxsize=256)
def ball_offsets(radius_q: int) -> np.ndarray:
    """Integer offsets with |o| <= radius_q/1024, x-major / z-minor (orient.py:63-74)."""
    rad = radius_q / 1024.0
    r = int(math.floor(rad))
    ax = np.arange(-r, r + 1)
    g = np.stack([a.ravel() for a in np.meshgrid(ax, ax, ax, indexing="ij")], axis=1)
    out = g[np.sum(g * g, axis=1) <= rad * rad].astype(np.intp)
    out.setflags(write=False)
    return out


def pack_offsets(offs: np.ndarray) -> np.ndarray:
    """10 bits per axis, biased by 512 (vk_common.cuh unpack_off)."""
    o = np.asarray(offs, dtype=np.int64)
    if len(o) and np.abs(o).max() > 511:
        raise ParameterError("neighbourhood radius above 511 voxels is not supported")
    return (((o[:, 0] + 512) << 20) | ((o[:, 1] + 512) << 10) | (o[:, 2] + 512)).astype(np.int32)


def window_table(radius: float, max_d2: int) -> np.ndarray:
    """Orientation window exp(-|o|^2 / (2 (radius/2)^2)) for |o|^2 = 0..max_d2,
    the exact numpy expression of orient.py:116-117 (host numpy exp)."""
    window_sd = radius / 2.0
    d2 = np.arange(max_d2 + 1, dtype=np.float64)
    return np.exp(-d2 / (2.0 * window_sd * window_sd))


class BallTable:
    """Concatenated balls for a set of radii, as uploaded to the device.

    Each ball contributes its offsets twice: in the reference's x-major order
    (exact-order accumulation) and z-major with per-plane start indices (the
    slab-staged fast path walks the ball plane by plane)."""

    def __init__(self):
        self.radii: list[float] = []
        self._index: dict[float, int] = {}
        self.records: list[tuple] = []
        self._off: list[np.ndarray] = []
        self._win: list[np.ndarray] = []
        self._planes: list[np.ndarray] = []
        self._noff = 0
        self._nwin = 0
        self._nplanes = 0

    def index(self, radius: float) -> int:
        """Ball id for an orientation / SIFT-Rank radius (radius_factor * sigma_local)."""
        key = float(radius)
        if key in self._index:
            return self._index[key]
        rq = int(round(radius * 1024))
        offs = ball_offsets(rq)
        r = int(math.floor(rq / 1024.0))
        max_d2 = int(np.max(np.sum(offs * offs, axis=1))) if len(offs) else 0
        zorder = np.lexsort((offs[:, 0], offs[:, 1], offs[:, 2])) if len(offs) else np.zeros(0, np.int64)
        zoffs = offs[zorder]
        counts = np.bincount(zoffs[:, 2] + r, minlength=2 * r + 1) if len(offs) else np.zeros(2 * r + 1, np.int64)
        planes = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
        self._index[key] = len(self.records)
        n = len(offs)
        self.records.append((self._noff, n, self._nwin, max_d2, self._noff + n, self._nplanes, r, 0))
        self._off.append(pack_offsets(offs))
        self._off.append(pack_offsets(zoffs))
        self._win.append(window_table(radius, max_d2))
        self._planes.append(planes)
        self._noff += 2 * n
        self._nwin += max_d2 + 1
        self._nplanes += len(planes)
        self.radii.append(key)
        return self._index[key]

    def arrays(self):
        """(ball records, packed offsets, windows, plane starts)."""
        from ._lib import BALL_DTYPE

        rec = np.array(self.records, dtype=np.int32).reshape(-1, len(BALL_DTYPE.names))
        balls = np.zeros(len(rec), dtype=BALL_DTYPE)
        for i, name in enumerate(BALL_DTYPE.names):
            balls[name] = rec[:, i] if len(rec) else 0
        off = np.concatenate(self._off) if self._off else np.zeros(1, np.int32)
        win = np.concatenate(self._win) if self._win else np.zeros(1, np.float64)
        planes = np.concatenate(self._planes) if self._planes else np.zeros(1, np.int32)
        # the plane starts ride at the end of the offset table (the kernels read them at
        # ball_offsets + pstart); pstart becomes relative to the table's start
        if len(rec):
            balls["pstart"] += len(off)
        off = np.concatenate([off, planes]).astype(np.int32)
        return balls, off, win, planes


def ball_sphere(radius: float):
    """Compact shared-memory layout of a ball and its gradient stencil for the
    fused orientation + SIFT-Rank kernel (csrc/vk_orsr.cu).

    The stencil set S = ball + the six axis neighbours of every ball voxel.
    Each (y, z) row of S is a symmetric x interval [-m, m] (every contributing
    row interval is centred at 0), so S is stored row after row, x fastest.
    Returns (rows, entries, size):
      rows    (n_rows, 4) int32: dy, dz, m, first compact index of the row
      entries (n, 4) int32, one per ball voxel in the z-major walk order:
              packed offset, c | yh << 16, yl | zh << 16, zl -- the compact
              index of the voxel (its x neighbours are c -+ 1) and of its
              y / z neighbours
      size    compact floats."""
    rq = int(round(radius * 1024))
    offs = ball_offsets(rq)
    if not len(offs):
        return np.zeros((0, 4), np.int32), np.zeros((0, 4), np.int32), 0
    zoffs = offs[np.lexsort((offs[:, 0], offs[:, 1], offs[:, 2]))]
    half: dict[tuple[int, int], int] = {}
    for x, y, z in offs.tolist():
        for dy, dz, dx in ((0, 0, 1), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0)):
            key = (y + dy, z + dz)
            half[key] = max(half.get(key, -1), abs(x) + dx)
    rows, start, pos = [], 0, {}
    for (y, z) in sorted(half, key=lambda k: (k[1], k[0])):
        m = half[(y, z)]
        rows.append((y, z, m, start))
        pos[(y, z)] = (start, m)
        start += 2 * m + 1
    if start > 65535:
        raise ParameterError("neighbourhood too large for the compact sphere layout")

    def idx(x, y, z):
        s0, m = pos[(y, z)]
        assert -m <= x <= m
        return s0 + x + m

    ent = np.zeros((len(zoffs), 4), dtype=np.int64)
    ent[:, 0] = pack_offsets(zoffs)
    for k, (x, y, z) in enumerate(zoffs.tolist()):
        c = idx(x, y, z)
        assert idx(x + 1, y, z) == c + 1 and idx(x - 1, y, z) == c - 1
        ent[k, 1] = c | (idx(x, y + 1, z) << 16)
        ent[k, 2] = idx(x, y - 1, z) | (idx(x, y, z + 1) << 16)
        ent[k, 3] = idx(x, y, z - 1)
    return np.array(rows, dtype=np.int32), ent.astype(np.uint32).view(np.int32), start


def sphere_tables(radii) -> tuple[np.ndarray, np.ndarray, np.ndarray, int]:
    """ball_sphere for every ball of a BallTable (same ids): per ball
    (rows start, n_rows, compact size, entries start) int32x4, the
    concatenated rows and entries, and the largest compact size."""
    recs, rows, ents = [], [], []
    nr = ne = 0
    biggest = 0
    for radius in radii:
        r, e, size = ball_sphere(radius)
        recs.append((nr, len(r), size, ne))
        rows.append(r)
        ents.append(e)
        nr += len(r)
        ne += len(e)
        biggest = max(biggest, size)
    rec = np.array(recs, dtype=np.int32).reshape(-1, 4)
    row = np.concatenate(rows) if rows else np.zeros((1, 4), np.int32)
    ent = np.concatenate(ents) if ents else np.zeros((1, 4), np.int32)
    return rec, np.ascontiguousarray(row), np.ascontiguousarray(ent), biggest


# ------------------------------------------------------------ patch & pairs
PAIR_SUPPORT_RADIUS = 2.0  # descriptor.py:34


@lru_cache(maxsize=32)
def patch_axis(side: int) -> np.ndarray:
    """One axis of descriptor.py:86-93's grid (linspace(-1, 1, side))."""
    a = np.linspace(-1.0, 1.0, side) if side > 1 else np.zeros(1)
    a.setflags(write=False)
    return a


def pair_points(p1: np.ndarray, p2: np.ndarray, side: int, sigma_unit: float) -> np.ndarray:
    """Pair sample positions in patch index space (descriptor.py:205-212)."""
    center = (side - 1) / 2.0
    scale = (side - 1) / (2.0 * PAIR_SUPPORT_RADIUS) / sigma_unit
    return np.stack([center + p1 * scale, center + p2 * scale]).astype(np.float64)
