"""CPU: host-side logic of the device path (no GPU needed)."""

import math

import numpy as np
import pytest

from paper_2112_10258_b200 import tables as T
from paper_2112_10258_b200.config import PipelineConfig
from paper_2112_10258_b200.engine import Plan


def test_icosphere_screening_claim():
    """The nearest of the 42 directions is the nearest icosahedron vertex or one
    of its 5 edge midpoints (what csrc/vk_orient.cu's screened argmax relies on;
    the kernel additionally keeps every vertex within a margin)."""
    d = T.icosphere_directions()
    st = T.icosphere_structure()
    vert, adj = st[:12], st[12:72].reshape(12, 5)
    rng = np.random.default_rng(0)
    g = rng.normal(size=(400000, 3))
    # plus directions near Voronoi boundaries: midpoints of random direction pairs
    i, j = rng.integers(0, 42, size=(2, 50000))
    g = np.vstack([g, d[i] + d[j] + 1e-9 * rng.normal(size=(50000, 3))])
    best = np.argmax(g @ d.T, axis=1)
    vb = np.argmax(g @ d[vert].T, axis=1)
    cand = np.concatenate([vert[vb][:, None], adj[vb]], axis=1)
    assert (cand == best[:, None]).any(axis=1).all()


def test_icosphere_fast_kind_table():
    """The fast argmax of csrc/vk_orient.cu (nearest_dir_fast), restated in
    fp64 numpy: the winning vertex group, its (p, q, r) axes, the six scores
    (vertex + 5 midpoints by neighbour kind) and the kind table of
    tables.icosphere_structure give np.argmax(g @ dirs.T) whenever the top two
    scores are separated."""
    d = T.icosphere_directions()
    st = T.icosphere_structure()
    vert, kind = st[:12], st[72:].reshape(12, 5)
    phi = (1.0 + 5 ** 0.5) / 2.0
    rng = np.random.default_rng(1)
    g = rng.normal(size=(200000, 3))
    ax, ay, az = np.abs(g).T
    vA, vB, vC = ay + phi * az, ax + phi * ay, az + phi * ax
    grp = np.argmax(np.stack([vA, vB, vC], axis=1), axis=1)
    perm = {0: (1, 2, 0), 1: (0, 1, 2), 2: (2, 0, 1)}
    pqr = np.stack([np.abs(g)[np.arange(len(g)), [perm[k][i] for k in grp]] for i in range(3)], axis=1)
    sg = np.stack([g[np.arange(len(g)), [perm[k][i] for k in grp]] for i in range(3)], axis=1)
    p, q, r = pqr.T
    best = p + phi * q
    cv, cm = 1.0 / np.sqrt(2.0 + phi), 1.0 / (2.0 * phi)
    sc = np.stack([cv * best, cm * (best + phi * p + r), cm * (best + phi * p - r), cm * (best + q + phi * r),
                   cm * (best + q - phi * r), cm * (best + phi * q - p)], axis=1)
    w = np.argmax(sc, axis=1)
    srt = np.sort(sc, axis=1)
    clear = srt[:, -1] - srt[:, -2] > 1e-9
    slot = 6 * (sg[:, 0] > 0) + 3 * (sg[:, 1] > 0) + grp
    rp = sg[:, 2] > 0
    k = np.select([w == 0, w == 1, w == 2, w == 3, w == 4], [0, np.where(rp, 1, 2), np.where(rp, 2, 1),
                                                             np.where(rp, 3, 4), np.where(rp, 4, 3)], 5)
    fk = np.concatenate([vert[:, None], kind], axis=1)
    got = fk[slot, k]
    want = np.argmax(g @ d.T, axis=1)
    assert clear.mean() > 0.99
    assert np.array_equal(got[clear], want[clear])


def test_plan_matches_reference_schedule():
    p = Plan.build((145, 174, 145), PipelineConfig())
    assert p.octave_dims == [(145, 174, 145), (72, 87, 72), (36, 43, 36), (18, 21, 18), (9, 10, 9), (4, 5, 4)]
    assert [k.radius for k in p.taps] == [5, 4, 5, 6, 8, 10]
    assert p.kappa == 2 ** (1 / 3)
    assert p.sigmas[0][3] == 1.6 * (2 ** (1 / 3)) ** 3
    # detection segments: octave o, DoG levels 1..3, sigma = level_sigma_local * 2^o
    L = 6
    for o in range(6):
        for i in (1, 2, 3):
            s = o * L + i
            oo, ii, lvl, ball = p.seg_info[s]
            assert (oo, ii, lvl) == (o, i, o * L + i)
            want = p.sigmas[o][i] / 2.0 ** o * math.sqrt(p.kappa) * math.sqrt(1.5) * 2.0 ** o
            assert p.seg_sigma[s] == want
    # octave truncation rule (scalespace.py:199-203): 20 -> 10 -> 5 -> (2 < 4)
    assert len(Plan.build((20, 20, 20), PipelineConfig()).octave_dims) == 3


def test_ball_table_and_windows():
    bt = T.BallTable()
    i0 = bt.index(4.0 * 1.6)
    assert bt.index(4.0 * 1.6) == i0
    balls, off, win, planes = bt.arrays()
    n = balls[i0]["count"]
    offs = T.ball_offsets(int(round(4.0 * 1.6 * 1024)))
    assert n == len(offs)
    unpacked = np.stack([((off[:n] >> s) & 1023) - 512 for s in (20, 10, 0)], axis=1)
    assert np.array_equal(unpacked, offs)
    sd = 4.0 * 1.6 / 2.0
    d2 = np.sum(offs * offs, axis=1).astype(np.float64)
    assert np.array_equal(win[balls[i0]["window_start"] + d2.astype(int)], np.exp(-d2 / (2.0 * sd * sd)))
    # z-major copy: same point set, sorted by (oz, oy, ox), with per-plane starts
    z0 = balls[i0]["zstart"]
    zo = np.stack([((off[z0:z0 + n] >> s) & 1023) - 512 for s in (20, 10, 0)], axis=1)
    assert sorted(map(tuple, zo)) == sorted(map(tuple, offs))
    assert np.all(np.diff(zo[:, 2] * 10**6 + zo[:, 1] * 10**3 + zo[:, 0]) > 0)
    r = balls[i0]["r"]
    # plane starts travel at the end of the offset table: pstart indexes `off`
    ps = off[balls[i0]["pstart"]: balls[i0]["pstart"] + 2 * r + 2]
    assert np.array_equal(ps, planes[: 2 * r + 2])
    for oz in range(-r, r + 1):
        assert np.all(zo[ps[oz + r]: ps[oz + r + 1], 2] == oz)


def test_pack_helpers_round_trip():
    """pack_bits / unpack_bits / pack_ranks / unpack_ranks (descriptor.py:319-340):
    MSB-first packing, 64 six-bit ranks -> 48 bytes, out-of-range ranks rejected."""
    from paper_2112_10258_b200 import descriptor as D
    from paper_2112_10258_b200.errors import ParameterError

    rng = np.random.default_rng(3)
    bits = rng.integers(0, 2, 64).astype(np.uint8)
    blob = D.pack_bits(bits)
    assert len(blob) == 8 and blob[0] == int("".join(map(str, bits[:8])), 2)
    assert np.array_equal(D.unpack_bits(blob, 64), bits)
    ranks = rng.permutation(64)
    blob = D.pack_ranks(ranks)
    assert len(blob) == 48
    assert np.array_equal(D.unpack_ranks(blob, 64), ranks)
    stream = "".join(format(int(r), "06b") for r in ranks)
    assert blob == int(stream, 2).to_bytes(48, "big")
    assert np.array_equal(D.unpack_ranks(D.pack_ranks([5, 1, 7], 3), 3, 3), [5, 1, 7])
    with pytest.raises(ParameterError):
        D.pack_ranks([64])
    with pytest.raises(ParameterError):
        D.pack_ranks([-1])


def test_icosphere_lut_is_exact_argmax():
    """tables.icosphere_lut: every pure cell's lookup (canonical face point of
    |g|, permutation, sign bits) equals np.argmax(g @ dirs.T), for random
    gradients and for gradients pushed onto Voronoi boundaries and the
    canonical-face edges (ties between |g| components, zero components)."""
    N = T.ICO_LUT_N
    lut = T.icosphere_lut()
    tab, lmap = lut[: N * N], lut[N * N:]
    assert len(lmap) == 42 * 24 and 0.96 < np.mean(tab != 255) < 0.99
    dirs = T.icosphere_directions()
    rng = np.random.default_rng(5)
    g = rng.standard_normal((200000, 3))
    # near-boundary cases: midpoints of direction pairs, plus tiny noise
    i, j = rng.integers(0, 42, (2, 20000))
    near = (dirs[i] + dirs[j]) / 2 + 1e-7 * rng.standard_normal((20000, 3))
    edges = rng.standard_normal((6000, 3))
    edges[:2000, 0] = edges[:2000, 2]                # |gx| == |gz|
    edges[2000:4000, 1] = 0.0                        # zero component
    edges[4000:, 0] = -edges[4000:, 1]               # |gx| == |gy|
    g = np.concatenate([g, near, edges]).astype(np.float32)
    a = np.abs(g)
    p, q, r, perm = T._ico_canonical(a)
    iu = np.minimum((p / r * N).astype(np.float32).astype(int), N - 1)
    iv = np.minimum((q / r * N).astype(np.float32).astype(int), N - 1)
    c = tab[iv * N + iu]
    sb = (g[:, 0] < 0) + 2 * (g[:, 1] < 0) + 4 * (g[:, 2] < 0)
    hit = c != 255
    got = lmap[c[hit].astype(int) * 24 + perm[hit] * 8 + sb[hit]]
    assert np.array_equal(got, np.argmax(g[hit].astype(np.float64) @ dirs.T, axis=1))
