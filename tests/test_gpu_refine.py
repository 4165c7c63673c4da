"""GPU: the optional sub-voxel / sub-level keypoint refinement
(vk_refine_keypoints, extract_features(..., refine=True)) against a plain
Python restatement of the same fixed-order fp64 algorithm, and the guarantee
that it leaves every reference (parity) field unchanged."""

import math

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

vk = pytest.importorskip("paper_2112_10258_b200")
from paper_2112_10258_b200 import synthetic  # noqa: E402
from paper_2112_10258_b200.config import PipelineConfig  # noqa: E402


def refine_one(dogs, kp, kappa):
    """The documented algorithm (csrc/vk_detect.cu refine_kernel), operation for
    operation in Python floats; dogs = [D_{l-1}, D_l, D_{l+1}] as [x, y, z] arrays."""
    scale = 2.0 ** kp.octave
    off = (scale - 1.0) / 2.0
    ix, iy, iz = (int(round((c - off) / scale)) for c in kp.position)
    nx, ny, nz = dogs[1].shape

    def at(L, dx, dy, dz):
        x = min(max(ix + dx, 0), nx - 1)
        y = min(max(iy + dy, 0), ny - 1)
        z = min(max(iz + dz, 0), nz - 1)
        return float(dogs[L][x, y, z])

    def s1(a, o):
        if a == 3:
            return at(1 + o, 0, 0, 0)
        d = [0, 0, 0]
        d[a] = o
        return at(1, *d)

    def s2(a, oa, b, ob):
        L = 1 + ob if b == 3 else 1
        d = [0, 0, 0]
        d[a] = oa
        if b < 3:
            d[b] = ob
        return at(L, *d)

    c = s1(0, 0)
    g = [0.0] * 4
    H = [[0.0] * 4 for _ in range(4)]
    for a in range(4):
        p, m = s1(a, 1), s1(a, -1)
        g[a] = (p - m) * 0.5
        H[a][a] = (p + m) - 2.0 * c
    for a in range(4):
        for b in range(a + 1, 4):
            v = (s2(a, 1, b, 1) - s2(a, 1, b, -1)) - (s2(a, -1, b, 1) - s2(a, -1, b, -1))
            H[a][b] = H[b][a] = v * 0.25
    A = [H[i][:] + [-g[i]] for i in range(4)]
    status = 0
    for col in range(4):
        piv = col
        for r in range(col + 1, 4):
            if abs(A[r][col]) > abs(A[piv][col]):
                piv = r
        if not abs(A[piv][col]) > 0.0:
            status = 2
            break
        A[col], A[piv] = A[piv], A[col]
        for r in range(col + 1, 4):
            f = A[r][col] / A[col][col]
            for j in range(col, 5):
                A[r][j] = A[r][j] - f * A[col][j]
    d = [0.0] * 4
    if status == 0:
        for i in range(3, -1, -1):
            acc = A[i][4]
            for j in range(i + 1, 4):
                acc = acc - A[i][j] * d[j]
            d[i] = acc / A[i][i]
        if any(abs(v) > 0.5 for v in d):
            status = 1
    gd = 0.0
    for i in range(4):
        gd = gd + g[i] * d[i]
    pos = [((ix + d[0]) * scale) + off, ((iy + d[1]) * scale) + off, ((iz + d[2]) * scale) + off]
    return pos, kp.sigma * math.pow(kappa, d[3]), c + 0.5 * gd, status


@pytest.mark.parametrize("name", ["small0.npz", "small2.npz"])
def test_refinement_matches_restatement_and_keeps_parity_fields(name):
    g = load_golden(name)
    dims = tuple(int(d) for d in g["dims"])
    vol = synthetic.random_blob_phantom(dims, np.random.default_rng(int(g["seed"])), n_blobs=10, margin=6, noise=0.02)
    cfg = PipelineConfig()
    plain = vk.extract_features(vk.Volume(vol), cfg)
    res = vk.extract_features(vk.Volume(vol), cfg, refine=True)
    assert plain.refined is None
    # parity fields unchanged (and still the reference's)
    assert np.array_equal(np.array([k.position for k in res.keypoints]).reshape(-1, 3), g["kp_pos"])
    assert [k.sigma for k in res.keypoints] == [k.sigma for k in plain.keypoints]
    assert np.array_equal(vk.descriptor.descriptor_array(res.records, "siftrank"), g["desc_siftrank"])
    R = res.refined
    assert R.shape == (len(res.keypoints), 6) and len(R) > 10
    kappa = 2.0 ** (1.0 / (cfg.levels_per_octave - 3))
    st = np.zeros(3, int)
    for k, kp in enumerate(res.keypoints):
        o, l = kp.octave, kp.level
        dogs = [res.dog.octaves[o].levels[l + j].data for j in (-1, 0, 1)]
        pos, sigma, dogv, status = refine_one(dogs, kp, kappa)
        assert list(R[k, :3]) == pos, k
        assert R[k, 4] == dogv and int(R[k, 5]) == status, k
        assert math.isclose(R[k, 3], sigma, rel_tol=1e-14), k  # device pow vs libm pow
        st[status] += 1
        if status == 0:  # a converged refinement stays within half a sample of the lattice point
            assert max(abs(a - b) for a, b in zip(R[k, :3], kp.position)) <= 0.5 * 2 ** o + 1e-9
    assert st[0] > 0  # (blob phantoms: many extrema sit nearer a neighbouring level than their own)
