"""numpy restatement of the volkey hot path -- TEST INFRASTRUCTURE ONLY.

Every function names the reference file:line it restates (paths relative to
``/root/reference/pkg/src/volkey``).  Arrays follow the reference convention:
float32 ``[x, y, z]`` C-order (z fastest).  The restatement reproduces the
reference bit for bit on the same host (same numpy + OpenBLAS build); that is
checked against the committed golden vectors in ``tests/golden``.

Keypoints are ``OKp`` tuples, frames are (3, 3) float64 rotation matrices,
descriptors are ``("siftrank"|"brief"|"rrief", ndarray)``.
"""

from __future__ import annotations

import itertools
import math
from typing import NamedTuple

import numpy as np

SIFT_LEN = 64                 # descriptor.py:33
PAIR_RADIUS = 2.0             # descriptor.py:34
CALIB = math.sqrt(1.5)        # detect.py:26


class OracleParameterError(ValueError):
    """Mirrors errors.ParameterError (errors.py:32-36)."""


class OracleDataError(ValueError):
    """Mirrors errors.DataError (errors.py:46-50)."""


class OKp(NamedTuple):
    """detect.Keypoint (detect.py:36-45)."""

    position: tuple
    sigma: float
    octave: int
    level: int
    dog_value: float
    sign: str


# --------------------------------------------------------------------------
# scale space (scalespace.py)
# --------------------------------------------------------------------------

def gauss_taps(sigma: float):
    """scalespace.py:35-42 -> (radius, float32 taps)."""
    if sigma <= 0:
        raise OracleParameterError(f"sigma must be > 0, got {sigma}")
    r = max(1, math.ceil(3.0 * sigma))
    k = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-(k ** 2) / (2.0 * sigma * sigma))
    w /= w.sum()
    return r, w.astype(np.float32)


def _axis_pass(a: np.ndarray, w: np.ndarray, axis: int) -> np.ndarray:
    """One 1-D replicate-padded pass (scalespace.py:63-82): products rounded
    to fp32, then added in tap order -r..+r (no fused multiply-add)."""
    r = (len(w) - 1) // 2
    widths = [(0, 0)] * 3
    widths[axis] = (r, r)
    p = np.pad(a, widths, mode="edge")
    n = a.shape[axis]

    def window(t):
        idx = [slice(None)] * 3
        idx[axis] = slice(t, t + n)
        return p[tuple(idx)]

    out = w[0] * window(0)
    for t in range(1, len(w)):
        out += w[t] * window(t)
    return out


def blur3(a: np.ndarray, w: np.ndarray) -> np.ndarray:
    """convolve_array (scalespace.py:45-60): x, then y, then z."""
    out = np.asarray(a, dtype=np.float32)
    for axis in (0, 1, 2):
        out = _axis_pass(out, w, axis)
    return out


def half(a: np.ndarray) -> np.ndarray:
    """subsample_half (scalespace.py:95-109): floor-crop, ordered 8-sum, /8."""
    nx, ny, nz = a.shape
    if min(nx, ny, nz) < 2:
        raise OracleParameterError(f"cannot subsample dims {a.shape}")
    c = a[: nx - nx % 2, : ny - ny % 2, : nz - nz % 2]
    s = c[0::2, 0::2, 0::2].astype(np.float32).copy()
    for dx, dy, dz in list(itertools.product((0, 1), repeat=3))[1:]:
        s += c[dx::2, dy::2, dz::2]
    s /= 8.0
    return s


def octave_schedule(base_sigma: float, levels: int):
    """kappa, octave-local sigmas and the incremental blur sigmas
    (scalespace.py:154-155, 207-209, 223)."""
    kappa = 2.0 ** (1.0 / (levels - 3))
    local = [base_sigma * kappa ** i for i in range(levels)]
    inc = [math.sqrt(max(local[i] * local[i] - local[i - 1] * local[i - 1], 0.0))
           for i in range(1, levels)]
    return kappa, local, inc


def pyramid(vol: np.ndarray, base_sigma=1.6, levels=6, num_octaves=6, min_octave_dim=4):
    """build_gaussian_pyramid (scalespace.py:158-206).

    Returns dict(octaves=[[level arrays]], sigmas=[[abs sigma]], kappa, source).
    """
    if base_sigma <= 0 or levels < 4 or num_octaves < 1:
        raise OracleParameterError("bad pyramid parameters")
    kappa, local, inc = octave_schedule(base_sigma, levels)
    handoff = levels - 3
    octs, sig = [], []
    cur = np.asarray(vol, dtype=np.float32)
    for o in range(num_octaves):
        lv = [blur3(cur, gauss_taps(local[0])[1])] if o == 0 else [cur]
        for i in range(1, levels):
            lv.append(blur3(lv[-1], gauss_taps(inc[i - 1])[1]))
        octs.append(lv)
        sig.append([s * 2.0 ** o for s in local])
        if o + 1 == num_octaves:
            break
        nxt = tuple(d // 2 for d in cur.shape)
        if min(nxt) < min_octave_dim or min(cur.shape) < 2:
            break
        cur = half(lv[handoff])
    return dict(octaves=octs, sigmas=sig, kappa=kappa, levels=levels, source=vol)


def dog(pyr):
    """build_dog_pyramid (scalespace.py:209-223)."""
    octs = [[lv[i] - lv[i + 1] for i in range(len(lv) - 1)] for lv in pyr["octaves"]]
    return dict(octaves=octs, sigmas=[s[:-1] for s in pyr["sigmas"]], kappa=pyr["kappa"])


# --------------------------------------------------------------------------
# detection (detect.py)
# --------------------------------------------------------------------------

_NB = [d for d in itertools.product((-1, 0, 1), repeat=3)]


def sos_map(prev, cur, nxt) -> np.ndarray:
    """sum_of_signs_map (detect.py:48-79): int16, interior only."""
    nx, ny, nz = cur.shape
    out = np.zeros((nx, ny, nz), dtype=np.int16)
    if min(nx, ny, nz) < 3:
        return out
    c = cur[1:-1, 1:-1, 1:-1]
    acc = out[1:-1, 1:-1, 1:-1]
    for vol, skip in ((prev, False), (cur, True), (nxt, False)):
        for dx, dy, dz in _NB:
            if skip and dx == dy == dz == 0:
                continue
            nb = vol[1 + dx: nx - 1 + dx, 1 + dy: ny - 1 + dy, 1 + dz: nz - 1 + dz]
            acc += (c > nb).astype(np.int16)
            acc -= (c < nb).astype(np.int16)
    return out


def extrema(m, dcur, band, contrast_min, octave, level, sigma_local):
    """extract_extrema (detect.py:82-140)."""
    if not 0 <= band <= 80:
        raise OracleParameterError("threshold_band outside [0, 80]")
    nx, ny, nz = dcur.shape
    if min(nx, ny, nz) < 3:
        return []
    mi = m[1:-1, 1:-1, 1:-1]
    ok = np.abs(dcur[1:-1, 1:-1, 1:-1]) >= contrast_min
    scale = 2.0 ** octave
    off = (scale - 1.0) / 2.0
    sigma = sigma_local * scale
    kps = []
    for name, mask in (("peak", (mi >= 80 - band) & (mi > 0) & ok),
                       ("valley", (mi <= -80 + band) & (mi < 0) & ok)):
        for ix, iy, iz in np.argwhere(mask) + 1:
            kps.append(OKp((float(ix * scale + off), float(iy * scale + off), float(iz * scale + off)),
                           sigma, octave, level, float(dcur[ix, iy, iz]), name))
    kps.sort(key=lambda k: (k.position[2], k.position[1], k.position[0], k.sign == "valley"))
    return kps


def level_sigma(dg, octave, level):
    """level_sigma_local (detect.py:143-146)."""
    return dg["sigmas"][octave][level] / (2.0 ** octave) * math.sqrt(dg["kappa"]) * CALIB


def detect(dg, band=0, contrast_min=0.0):
    """detect_keypoints (detect.py:149-182)."""
    kps = []
    for o, lv in enumerate(dg["octaves"]):
        if len(lv) < 3:
            raise OracleParameterError("octave needs >= 3 DoG levels")
        for i in range(1, len(lv) - 1):
            m = sos_map(lv[i - 1], lv[i], lv[i + 1])
            kps.extend(extrema(m, lv[i], band, contrast_min, o, i, level_sigma(dg, o, i)))
    kps.sort(key=lambda k: (k.octave, k.level, k.position[2], k.position[1], k.position[0],
                            k.sign == "valley"))
    return kps


# --------------------------------------------------------------------------
# sampling helpers (volume.py)
# --------------------------------------------------------------------------

def trilinear(data: np.ndarray, pts: np.ndarray) -> np.ndarray:
    """sample_trilinear_array (volume.py:203-236): clamped, fp64 arithmetic."""
    p = np.atleast_2d(np.asarray(pts, dtype=np.float64))
    shape = np.array(data.shape)
    p = np.clip(p, 0.0, shape.astype(np.float64) - 1.0)
    i0 = np.minimum(np.floor(p).astype(np.intp), np.maximum(shape - 2, 0))
    f = p - i0
    i1 = np.minimum(i0 + 1, shape - 1)
    x0, y0, z0 = i0.T
    x1, y1, z1 = i1.T
    fx, fy, fz = f.T

    def lerp(a, b, t):
        return a * (1 - t) + b * t

    c00 = lerp(data[x0, y0, z0], data[x1, y0, z0], fx)
    c10 = lerp(data[x0, y1, z0], data[x1, y1, z0], fx)
    c01 = lerp(data[x0, y0, z1], data[x1, y0, z1], fx)
    c11 = lerp(data[x0, y1, z1], data[x1, y1, z1], fx)
    return lerp(lerp(c00, c10, fy), lerp(c01, c11, fy), fz)


def grads_at(data: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """gradients_at (volume.py:244-264): central, one-sided at borders."""
    idx = np.atleast_2d(np.asarray(idx, dtype=np.intp))
    g = np.empty((len(idx), 3), dtype=np.float64)
    for ax in range(3):
        n = data.shape[ax]
        hi = np.minimum(idx[:, ax] + 1, n - 1)
        lo = np.maximum(idx[:, ax] - 1, 0)
        den = np.maximum(hi - lo, 1).astype(np.float64)
        up, dn = idx.copy(), idx.copy()
        up[:, ax] = hi
        dn[:, ax] = lo
        g[:, ax] = (data[up[:, 0], up[:, 1], up[:, 2]].astype(np.float64)
                    - data[dn[:, 0], dn[:, 1], dn[:, 2]].astype(np.float64)) / den
    return g


# --------------------------------------------------------------------------
# orientation (orient.py)
# --------------------------------------------------------------------------

def icosphere() -> np.ndarray:
    """icosphere_directions (orient.py:34-60): 42 lexsorted unit vectors."""
    phi = (1.0 + math.sqrt(5.0)) / 2.0
    v = []
    for a in (-1.0, 1.0):
        for b in (-phi, phi):
            v += [(0.0, a, b), (a, b, 0.0), (b, 0.0, a)]
    v = np.array(v, dtype=np.float64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    d2 = np.sum((v[:, None, :] - v[None, :, :]) ** 2, axis=2)
    edge = np.min(d2[d2 > 1e-9])
    mids = []
    for i in range(len(v)):
        for j in range(i + 1, len(v)):
            if abs(d2[i, j] - edge) < 1e-9:
                s = v[i] + v[j]
                mids.append(s / np.linalg.norm(s))
    d = np.vstack([v, np.array(mids)])
    order = np.lexsort((d[:, 2].round(9), d[:, 1].round(9), d[:, 0].round(9)))
    return d[order]


def ball(radius_q: int) -> np.ndarray:
    """_ball_offsets (orient.py:63-74): x-major, z-minor integer offsets."""
    rad = radius_q / 1024.0
    r = int(math.floor(rad))
    ax = np.arange(-r, r + 1)
    g = np.stack([a.ravel() for a in np.meshgrid(ax, ax, ax, indexing="ij")], axis=1)
    return g[np.sum(g * g, axis=1) <= rad * rad].astype(np.intp)


def lattice(kp: OKp):
    """keypoint_local (orient.py:76-86) without the level lookup."""
    scale = 2.0 ** kp.octave
    off = (scale - 1.0) / 2.0
    return np.array([round((c - off) / scale) for c in kp.position], dtype=np.intp), kp.sigma / scale


def _level(pyr, kp):
    if not (0 <= kp.octave < len(pyr["octaves"])) or not (0 <= kp.level < len(pyr["octaves"][kp.octave])):
        raise OracleParameterError("keypoint outside pyramid")
    return pyr["octaves"][kp.octave][kp.level]


def orient_hist(pyr, kp, radius_factor=4.0, dirs=None) -> np.ndarray:
    """gradient_histogram (orient.py:89-125) -> (K,) fp64 weights."""
    if radius_factor <= 0:
        raise OracleParameterError("radius_factor must be > 0")
    dirs = icosphere() if dirs is None else np.asarray(dirs, dtype=np.float64)
    data = _level(pyr, kp)
    c, s = lattice(kp)
    rad = radius_factor * s
    offs = ball(int(round(rad * 1024)))
    vox = c[None, :] + offs
    inside = np.all((vox >= 0) & (vox < np.array(data.shape)[None, :]), axis=1)
    if not inside.any():
        raise OracleDataError("orientation neighbourhood outside the volume")
    vox, of = vox[inside], offs[inside].astype(np.float64)
    g = grads_at(data, vox)
    mag = np.linalg.norm(g, axis=1)
    sd = rad / 2.0
    votes = mag * np.exp(-np.sum(of * of, axis=1) / (2.0 * sd * sd))
    w = np.zeros(len(dirs), dtype=np.float64)
    nz = mag > 0
    if nz.any():
        np.add.at(w, np.argmax(g[nz] @ dirs.T, axis=1), votes[nz])
    return w


def frames_from_hist(w, dirs=None, secondary_ratio=0.8, max_frames=4):
    """dominant_orientations (orient.py:128-168) -> list of (3,3) rotations."""
    if not 0 < secondary_ratio <= 1 or max_frames < 1:
        raise OracleParameterError("bad frame parameters")
    dirs = icosphere() if dirs is None else np.asarray(dirs, dtype=np.float64)
    w = np.asarray(w, dtype=np.float64)
    top = w.max() if len(w) else 0.0
    if top <= 0:
        return []
    rank = sorted(range(len(w)), key=lambda i: (-w[i], i))
    prim = [i for i in rank if w[i] >= secondary_ratio * top][:max_frames]
    out = []
    for p in prim:
        a1 = dirs[p]
        a2 = None
        for q in rank:
            if q == p:
                continue
            pr = dirs[q] - np.dot(dirs[q], a1) * a1
            nrm = np.linalg.norm(pr)
            if nrm > 1e-6:
                a2 = pr / nrm
                break
        if a2 is None:
            continue
        out.append(np.column_stack([a1, a2, np.cross(a1, a2)]))
    return out


def frame_pairs_from_hist(w, secondary_ratio=0.8, max_frames=4):
    """Same selection as frames_from_hist but returns (primary, secondary)
    direction indices (used to check the device frame indices)."""
    dirs = icosphere()
    top = w.max() if len(w) else 0.0
    if top <= 0:
        return []
    rank = sorted(range(len(w)), key=lambda i: (-w[i], i))
    prim = [i for i in rank if w[i] >= secondary_ratio * top][:max_frames]
    out = []
    for p in prim:
        for q in rank:
            if q == p:
                continue
            pr = dirs[q] - np.dot(dirs[q], dirs[p]) * dirs[p]
            if np.linalg.norm(pr) > 1e-6:
                out.append((p, q))
                break
    return out


def orient_all(pyr, kps, radius_factor=4.0, secondary_ratio=0.8, max_frames=4):
    """assign_orientations (pipeline.py:41-67) -> ([(kp, R)], dropped)."""
    groups = {}
    for i, kp in enumerate(kps):
        groups.setdefault((kp.octave, kp.level), []).append(i)
    got, dropped = {}, 0
    for key in sorted(groups):
        for i in groups[key]:
            fr = frames_from_hist(orient_hist(pyr, kps[i], radius_factor), None, secondary_ratio, max_frames)
            if not fr:
                dropped += 1
                continue
            got[i] = [(kps[i], r) for r in fr]
    flat = []
    for i in sorted(got):
        flat.extend(got[i])
    return flat, dropped


# --------------------------------------------------------------------------
# descriptors (descriptor.py)
# --------------------------------------------------------------------------

def ranks(v) -> np.ndarray:
    """rank_vector (descriptor.py:77-83): stable ranks."""
    v = np.asarray(v)
    r = np.empty(len(v), dtype=np.int64)
    r[np.argsort(v, kind="stable")] = np.arange(len(v))
    return r


def patch_grid(side: int) -> np.ndarray:
    """_patch_grid (descriptor.py:86-93)."""
    c = np.linspace(-1.0, 1.0, side) if side > 1 else np.zeros(1)
    return np.stack([a.ravel() for a in np.meshgrid(c, c, c, indexing="ij")], axis=1)


def patch(pyr, kp: OKp, R: np.ndarray, side=15) -> np.ndarray:
    """extract_patch (descriptor.py:96-111) -> (side,)*3 float32."""
    if side < 1 or side % 2 == 0:
        raise OracleParameterError("patch side must be odd and >= 1")
    if pyr.get("source") is None:
        raise OracleParameterError("pyramid carries no source volume")
    pts = np.asarray(kp.position, dtype=np.float64)[None, :] + (patch_grid(side) * (PAIR_RADIUS * kp.sigma)) @ R.T
    return trilinear(pyr["source"], pts).astype(np.float32).reshape(side, side, side)


def point_pairs(method: int, n: int, sigma_unit=1.0, seed=0):
    """sample_point_pairs (descriptor.py:114-193) -> (p1, p2) fp64 (n, 3)."""
    if method not in (1, 2, 3, 4, 5) or n < 1 or sigma_unit <= 0:
        raise OracleParameterError("bad point-pair parameters")
    rng = np.random.default_rng(seed)
    rad = PAIR_RADIUS * sigma_unit

    def redraw(draw):
        pts = draw()
        while True:
            bad = np.linalg.norm(pts, axis=1) > rad
            if not bad.any():
                return pts
            pts[bad] = draw()[bad]

    def uni():
        return redraw(lambda: rng.uniform(-rad, rad, size=(n, 3)))

    def nrm(c):
        return redraw(lambda: c + rng.normal(0.0, sigma_unit, size=(n, 3)))

    zero = np.zeros((n, 3))
    if method == 1:
        p1 = uni()
        p2 = uni()
    elif method == 2:
        p1 = nrm(zero)
        p2 = nrm(zero)
    elif method == 3:
        p1 = nrm(zero)
        p2 = nrm(p1)
    elif method == 4:
        p1, p2 = zero, nrm(zero)
    else:
        octa = [np.eye(3)[a] * s for a in range(3) for s in (1.0, -1.0)]
        for i in range(3):
            for j in range(i + 1, 3):
                for si in (1.0, -1.0):
                    for sj in (1.0, -1.0):
                        e = np.zeros(3)
                        e[i], e[j] = si, sj
                        octa.append(np.array([c / math.sqrt(2.0) for c in e]))
        octa = np.array(octa)
        grid = np.array([r * d for r in np.array([0.5, 1.0, 1.5, 2.0]) * sigma_unit for d in octa])
        p1, p2 = zero, grid[np.arange(n) % len(grid)]
    return p1, p2


def preblur(p: np.ndarray, blur_sigma: float) -> np.ndarray:
    """preblur_patch (descriptor.py:196-202)."""
    if blur_sigma < 0:
        raise OracleParameterError("blur_sigma must be >= 0")
    return p if blur_sigma == 0 else blur3(p, gauss_taps(blur_sigma)[1])


def pair_diffs(p: np.ndarray, pairs, sigma_unit=1.0) -> np.ndarray:
    """_pair_samples (descriptor.py:205-212), returns s1 - s2."""
    side = p.shape[0]
    c = (side - 1) / 2.0
    sc = (side - 1) / (2.0 * PAIR_RADIUS) / sigma_unit
    return trilinear(p, c + pairs[0] * sc) - trilinear(p, c + pairs[1] * sc)


def siftrank(pyr, kp: OKp, R: np.ndarray, radius_factor=4.0) -> np.ndarray:
    """sift_rank_descriptor (descriptor.py:227-263) -> (64,) int64 ranks."""
    data = _level(pyr, kp)
    c, s = lattice(kp)
    offs = ball(int(round(radius_factor * s * 1024)))
    vox = c[None, :] + offs
    inside = np.all((vox >= 0) & (vox < np.array(data.shape)[None, :]), axis=1)
    b = np.zeros(SIFT_LEN, dtype=np.float64)
    if inside.any():
        g = grads_at(data, vox[inside])
        ro = offs[inside].astype(np.float64) @ R
        rg = g @ R
        sp = (ro[:, 0] > 0).astype(np.int64) + 2 * (ro[:, 1] > 0) + 4 * (ro[:, 2] > 0)
        orr = (rg[:, 0] > 0).astype(np.int64) + 2 * (rg[:, 1] > 0) + 4 * (rg[:, 2] > 0)
        np.add.at(b, sp * 8 + orr, np.linalg.norm(rg, axis=1))
    return ranks(b)


def describe(pyr, oriented, kind="siftrank", pairs=None, patch_side=15, blur_sigma=0.95,
             radius_factor=4.0):
    """describe_all (descriptor.py:266-306) -> (list of (kp, R, desc), dropped)."""
    if kind not in ("siftrank", "brief", "rrief"):
        raise OracleParameterError(f"unknown descriptor kind {kind!r}")
    if kind != "siftrank" and pairs is None:
        raise OracleParameterError("point-pair kinds need pairs")
    out, dropped = [], 0
    for kp, R in oriented:
        try:
            if kind == "siftrank":
                d = siftrank(pyr, kp, R, radius_factor)
            else:
                diff = pair_diffs(preblur(patch(pyr, kp, R, patch_side), blur_sigma), pairs)
                d = (diff > 0).astype(np.uint8) if kind == "brief" else ranks(diff)
            out.append((kp, R, d))
        except OracleParameterError:
            raise
        except Exception:
            dropped += 1
    return out, dropped


def desc_array(recs, kind) -> np.ndarray:
    """descriptor_array (descriptor.py:309-316)."""
    if not recs:
        return np.zeros((0, 0), dtype=np.uint8 if kind == "brief" else np.int64)
    m = np.stack([r[2] for r in recs])
    return np.packbits(m, axis=1, bitorder="big") if kind == "brief" else m


# --------------------------------------------------------------------------
# matching (match.py:64-121)
# --------------------------------------------------------------------------

_POP = np.array([bin(i).count("1") for i in range(256)], dtype=np.uint16)


def hamming(a, b):
    """hamming_distances (match.py:64-67)."""
    return _POP[np.bitwise_xor(a[:, None, :], b[None, :, :])].sum(axis=2).astype(np.float64)


def euclid(a, b):
    """euclidean_distances (match.py:70-78)."""
    a, b = a.astype(np.float64), b.astype(np.float64)
    d2 = np.sum(a * a, axis=1)[:, None] + np.sum(b * b, axis=1)[None, :] - 2.0 * (a @ b.T)
    return np.sqrt(np.maximum(d2, 0.0))


def nn_match(a, b, ratio_max=0.9, metric="euclidean"):
    """nearest_neighbor_matches (match.py:81-121) -> list of
    (index_a, index_b, distance, second_distance)."""
    if metric not in ("hamming", "euclidean") or not 0 < ratio_max <= 1 or len(b) < 2:
        raise OracleParameterError("bad match parameters")
    if len(a) == 0:
        return []
    d = (hamming if metric == "hamming" else euclid)(a, b)
    j = np.argmin(d, axis=1)
    rows = np.arange(len(a))
    d1 = d[rows, j]
    two = np.partition(d, 1, axis=1)[:, :2]
    d2 = np.maximum(np.where(two[:, 0] == d1, two[:, 1], two[:, 0]), d1)
    return [(int(i), int(j[i]), float(d1[i]), float(d2[i])) for i in rows if d1[i] <= ratio_max * d2[i]]


# --------------------------------------------------------------------------
# end to end (pipeline.py:70-102)
# --------------------------------------------------------------------------

DEFAULTS = dict(base_sigma=1.6, levels_per_octave=6, num_octaves=6, min_octave_dim=4,
                threshold_band=0, contrast_min=0.0, radius_factor=4.0, secondary_ratio=0.8,
                max_frames=4, descriptor="siftrank", pairs=64, method=3, patch_side=15,
                blur_sigma=0.95, seed=13, ratio_max=0.9)


def extract(vol: np.ndarray, **overrides):
    """extract_features (pipeline.py:70-102) -> dict."""
    c = dict(DEFAULTS, **overrides)
    pyr = pyramid(vol, c["base_sigma"], c["levels_per_octave"], c["num_octaves"], c["min_octave_dim"])
    dg = dog(pyr)
    kps = detect(dg, c["threshold_band"], c["contrast_min"])
    oriented, d_or = orient_all(pyr, kps, c["radius_factor"], c["secondary_ratio"], c["max_frames"])
    pairs = None if c["descriptor"] == "siftrank" else point_pairs(c["method"], c["pairs"], 1.0, c["seed"])
    recs, d_de = describe(pyr, oriented, c["descriptor"], pairs, c["patch_side"], c["blur_sigma"],
                          c["radius_factor"])
    return dict(pyramid=pyr, dog=dg, keypoints=kps, oriented=oriented, records=recs,
                dropped_orientation=d_or, dropped_descriptor=d_de)
