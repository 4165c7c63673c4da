"""Stage-level behaviour of orientation and descriptors on caller-built
pyramids (the reference's test_orient.py / test_descriptor.py scenarios:
ramps, constants, custom direction sets, frame construction, patches,
BRIEF / RRIEF / SIFT-Rank semantics), run on the GPU path and checked
against the oracle bit for bit where the reference states an exact value."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

vk = pytest.importorskip("paper_2112_10258_b200")
from paper_2112_10258_b200.descriptor import (Patch, brief_descriptor, describe_all, extract_patch,  # noqa: E402
                                              rank_vector, rrief_descriptor, sample_point_pairs,
                                              sift_rank_descriptor)
from paper_2112_10258_b200.detect import Keypoint  # noqa: E402
from paper_2112_10258_b200.errors import ParameterError  # noqa: E402
from paper_2112_10258_b200.orient import (OrientationFrame, SphericalHistogram,  # noqa: E402
                                          dominant_orientations, gradient_histogram, icosphere_directions)
from paper_2112_10258_b200.scalespace import GaussianPyramid, PyramidOctave  # noqa: E402
from paper_2112_10258_b200.synthetic import rotation_from_axis_angle  # noqa: E402

AXES = np.array([[1.0, 0, 0], [-1.0, 0, 0], [0, 1.0, 0], [0, -1.0, 0], [0, 0, 1.0], [0, 0, -1.0]])
IDENTITY = OrientationFrame(np.eye(3))


@pytest.fixture
def rng():
    return np.random.default_rng(17)


def one_level(arr, sigma=2.0):
    v = vk.Volume(np.asarray(arr, dtype=np.float32))
    return GaussianPyramid([PyramidOctave([v], [sigma])], sigma, 2 ** (1 / 3), 1, source=v)


def centre_kp(n, sigma=2.0):
    return Keypoint((float(n // 2),) * 3, sigma, 0, 0, 1.0, "peak")


def ramp(n, axis, gain=1.0):
    return (gain * np.meshgrid(*[np.arange(n)] * 3, indexing="ij")[axis]).astype(np.float32)


def okp(kp):
    from oracle import volkey_oracle as O

    return O.OKp(tuple(kp.position), kp.sigma, kp.octave, kp.level, kp.dog_value, kp.sign)


# ------------------------------------------------------------- orientation
def test_x_ramp_votes_only_nearest_x_direction():
    h = gradient_histogram(one_level(ramp(17, 0)), centre_kp(17))
    best = int(np.argmax(icosphere_directions() @ np.array([1.0, 0, 0])))
    assert int(np.argmax(h.weights)) == best and h.weights[best] > 0
    assert h.weights.sum() - h.weights[best] == 0.0


def test_constant_level_gives_zero_histogram():
    assert not np.any(gradient_histogram(one_level(np.full((15, 15, 15), 3.0)), centre_kp(15)).weights)


def test_two_mode_histogram_equals_oracle_loop():
    from oracle import volkey_oracle as O

    n, c = 21, 10
    gx, gy, _ = np.meshgrid(*[np.arange(n)] * 3, indexing="ij")
    arr = np.where(gx < c, 100.0 + 3.0 * gy, 1000.0 + 3.0 * gx).astype(np.float32)
    kp = centre_kp(n)
    h = gradient_histogram(one_level(arr), kp)
    assert np.array_equal(h.weights, O.orient_hist({"octaves": [[arr]]}, okp(kp)))
    dirs = icosphere_directions()
    want = {int(np.argmax(dirs @ np.array([1.0, 0, 0]))), int(np.argmax(dirs @ np.array([0, 1.0, 0])))}
    assert set(np.argsort(h.weights)[-2:]) == want


def test_custom_axis_directions_permute_under_rotation():
    kp = centre_kp(17)
    hx = gradient_histogram(one_level(ramp(17, 0, 2.0)), kp, directions=AXES)
    hy = gradient_histogram(one_level(ramp(17, 1, 2.0)), kp, directions=AXES)
    assert hx.weights[0] > 0 and hx.weights[0] == hy.weights[2]


def test_dominant_orientations_frame_construction():
    w = np.zeros(6)
    w[0], w[2] = 1.0, 0.9
    frames = dominant_orientations(SphericalHistogram(AXES, w))
    assert len(frames) == 2 and np.allclose(frames[0].rotation, np.eye(3), atol=1e-12)
    w = np.zeros(6)
    w[0] = w[2] = 1.0
    w[4] = 0.1
    frames = dominant_orientations(SphericalHistogram(AXES, w), secondary_ratio=1.0)
    assert len(frames) == 2
    assert np.allclose(frames[0].rotation[:, 0], [1, 0, 0]) and np.allclose(frames[1].rotation[:, 0], [0, 1, 0])
    assert dominant_orientations(SphericalHistogram(AXES, np.zeros(6))) == []
    with pytest.raises(ParameterError):
        dominant_orientations(SphericalHistogram(AXES, np.ones(6)), secondary_ratio=0.0)
    with pytest.raises(ParameterError):
        dominant_orientations(SphericalHistogram(AXES, np.ones(6)), max_frames=0)


def test_random_histograms_give_valid_frames(rng):
    from oracle import volkey_oracle as O

    dirs = icosphere_directions()
    for _ in range(25):
        w = rng.random(len(dirs))
        frames = dominant_orientations(SphericalHistogram(dirs, w))
        want = O.frames_from_hist(w)
        assert 1 <= len(frames) <= 4 and len(frames) == len(want)
        for f, r in zip(frames, want):
            assert np.array_equal(f.rotation, r)
            assert np.allclose(f.rotation.T @ f.rotation, np.eye(3), atol=1e-5)
        a = dominant_orientations(SphericalHistogram(dirs, 7.3 * w))
        assert [f.rotation.tolist() for f in a] == [f.rotation.tolist() for f in frames]


# ------------------------------------------------------------- descriptors
def test_patch_side_one_and_rotation_covariance(rng):
    arr = rng.random((17, 17, 17), dtype=np.float32)
    p = extract_patch(one_level(arr), centre_kp(17), IDENTITY, side=1)
    assert p.data.shape == (1, 1, 1) and p.data[0, 0, 0] == arr[8, 8, 8]
    kp = centre_kp(25)
    rot = OrientationFrame(rotation_from_axis_angle([0, 0, 1], 90.0))
    a = extract_patch(one_level(ramp(25, 1)), kp, rot, side=9).data
    b = extract_patch(one_level(ramp(25, 0)), kp, IDENTITY, side=9).data
    assert np.allclose(a - a.mean(), b - b.mean(), atol=1e-4)
    with pytest.raises(ParameterError):
        extract_patch(one_level(arr), centre_kp(17), IDENTITY, side=4)


def test_brief_and_rrief_semantics(rng):
    pairs = sample_point_pairs(2, 64, seed=1)
    assert not np.any(brief_descriptor(Patch(5, np.full((5, 5, 5), 1.0, dtype=np.float32)), pairs).bits)
    assert rrief_descriptor(Patch(5, np.zeros((5, 5, 5), dtype=np.float32)),
                            sample_point_pairs(2, 16, seed=2)).ranks.tolist() == list(range(16))
    patch = Patch(9, rng.random((9, 9, 9), dtype=np.float32))
    pairs = sample_point_pairs(3, 64, seed=34)
    bits, ranks = brief_descriptor(patch, pairs).bits, rrief_descriptor(patch, pairs).ranks
    scaled = Patch(9, 2.0 * patch.data)  # power-of-two gain: exact
    assert np.array_equal(bits, brief_descriptor(scaled, pairs).bits)
    assert np.array_equal(ranks, rrief_descriptor(scaled, pairs).ranks)
    from oracle import volkey_oracle as O

    d = O.pair_diffs(patch.data, (pairs.p1, pairs.p2))
    assert np.array_equal(bits == 1, d > 0) and np.array_equal(ranks, O.ranks(d))
    assert rank_vector(np.array([3.1, -2.0, 7.4])).tolist() == [1, 0, 2]


def test_siftrank_edge_cases_match_oracle(rng):
    from oracle import volkey_oracle as O

    arr = rng.random((19, 19, 19), dtype=np.float32)
    d = sift_rank_descriptor(one_level(arr), centre_kp(19), IDENTITY)
    assert sorted(d.ranks.tolist()) == list(range(64))
    assert np.array_equal(d.ranks, O.siftrank({"octaves": [[arr]]}, okp(centre_kp(19)), np.eye(3)))
    flat = sift_rank_descriptor(one_level(np.zeros((19, 19, 19))), centre_kp(19), IDENTITY)
    assert flat.ranks.tolist() == list(range(64))
    xr = ramp(21, 0, 2.0)
    d = sift_rank_descriptor(one_level(xr), centre_kp(21), IDENTITY)
    assert np.array_equal(d.ranks, O.siftrank({"octaves": [[xr]]}, okp(centre_kp(21)), np.eye(3)))
    arr = rng.random((21, 21, 21), dtype=np.float32)
    a = sift_rank_descriptor(one_level(arr), centre_kp(21), IDENTITY)
    b = sift_rank_descriptor(one_level(2.0 * arr), centre_kp(21), IDENTITY)
    assert np.array_equal(a.ranks, b.ranks)


def test_describe_all_bookkeeping(rng):
    pyr = one_level(rng.random((19, 19, 19), dtype=np.float32))
    assert describe_all(pyr, []) == ([], 0)
    kp = centre_kp(19)
    recs, dropped = describe_all(pyr, [(kp, IDENTITY), (kp, OrientationFrame(rotation_from_axis_angle([0, 0, 1], 90.0)))])
    assert len(recs) == 2 and dropped == 0
    with pytest.raises(ParameterError):
        describe_all(pyr, [(kp, IDENTITY)], kind="brief")
