"""Behavioural properties of matching (match.py:64-121, GPU kernels) and the
7-DOF consensus (match.py:124-359, host stage): brute-force agreement,
self-matching, ratio semantics, scale invariance, parameter errors, transform
recovery -- the reference's test_match.py checks, on this package."""

import numpy as np
import pytest

from paper_2112_10258_b200.consensus import (SimilarityTransform7DOF, hough_consensus, rotation_angle_deg,
                                             similarity_from_correspondences, vote_transform)
from paper_2112_10258_b200.detect import Keypoint
from paper_2112_10258_b200.errors import ParameterError
from paper_2112_10258_b200.match import Match, hamming_distances, nearest_neighbor_matches
from paper_2112_10258_b200.orient import OrientationFrame
from paper_2112_10258_b200.synthetic import rotation_from_axis_angle


@pytest.fixture
def rng():
    return np.random.default_rng(31)


def _kp(pos, sigma=2.0):
    return Keypoint(tuple(float(p) for p in pos), float(sigma), 0, 1, 0.1, "peak")


def _rand_rot(rng):
    q = np.linalg.qr(rng.normal(size=(3, 3)))[0]
    if np.linalg.det(q) < 0:
        q[:, 2] *= -1
    return q


# --------------------------------------------------------------- GPU matching
@pytest.mark.gpu
def test_identical_rank_sets_self_match(rng):
    a = rng.integers(0, 64, size=(20, 64))
    got = nearest_neighbor_matches(a, a, ratio_max=1.0)
    assert len(got) == 20 and all(m.index_a == m.index_b and m.distance == 0.0 for m in got)


@pytest.mark.gpu
def test_ratio_semantics(rng):
    a, b = rng.random((40, 8)), rng.random((60, 8))
    loose = nearest_neighbor_matches(a, b, ratio_max=1.0)
    tight = nearest_neighbor_matches(a, b, ratio_max=0.5)
    assert len(loose) == 40 and len(tight) <= len(loose)
    assert all(m.distance <= 0.5 * m.second_distance for m in tight)


@pytest.mark.gpu
def test_hamming_matches_brute_force(rng):
    bits_a = (rng.random((50, 64)) > 0.5).astype(np.uint8)
    bits_b = (rng.random((50, 64)) > 0.5).astype(np.uint8)
    got = nearest_neighbor_matches(np.packbits(bits_a, axis=1), np.packbits(bits_b, axis=1), ratio_max=1.0,
                                   metric="hamming")
    d = (bits_a[:, None, :] != bits_b[None, :, :]).sum(axis=2).astype(float)
    assert len(got) == 50
    for m in got:
        assert m.index_b == int(np.argmin(d[m.index_a])) and m.distance == d[m.index_a].min()


@pytest.mark.gpu
def test_euclidean_matches_brute_force_and_is_scale_invariant(rng):
    a, b = rng.random((25, 16)), rng.random((40, 16))
    got = nearest_neighbor_matches(a, b, ratio_max=1.0)
    for m in got:
        dist = np.linalg.norm(b - a[m.index_a], axis=1)
        assert m.index_b == int(np.argmin(dist)) and m.distance == pytest.approx(dist.min(), rel=1e-9)
    base = nearest_neighbor_matches(a, b, ratio_max=0.8)
    scaled = nearest_neighbor_matches(3.0 * a, 3.0 * b, ratio_max=0.8)
    assert [(m.index_a, m.index_b) for m in base] == [(m.index_a, m.index_b) for m in scaled]


@pytest.mark.gpu
def test_small_reference_set_rejected(rng):
    with pytest.raises(ParameterError):
        nearest_neighbor_matches(rng.random((5, 8)), rng.random((1, 8)))


@pytest.mark.gpu
def test_hamming_distance_popcount():
    a = np.array([[0xFF, 0x00]], dtype=np.uint8)
    b = np.array([[0x0F, 0x00], [0xFF, 0xFF]], dtype=np.uint8)
    assert hamming_distances(a, b).tolist() == [[4.0, 8.0]]


# ------------------------------------------------------------ host consensus
def test_vote_transform_identity_scale_and_round_trip(rng):
    eye = OrientationFrame(np.eye(3))
    t = vote_transform(_kp((5, 6, 7)), eye, _kp((5, 6, 7)), eye)
    assert t.scale == pytest.approx(1.0) and np.allclose(t.rotation, np.eye(3)) and np.allclose(t.translation, 0.0)
    t = vote_transform(_kp((0, 0, 0), 2.0), eye, _kp((0, 0, 0), 4.0), eye)
    assert t.scale == pytest.approx(2.0) and np.allclose(t.translation, 0.0)
    for _ in range(20):
        a = _kp(rng.uniform(0, 50, 3), rng.uniform(1, 4))
        b = _kp(rng.uniform(0, 50, 3), rng.uniform(1, 4))
        t = vote_transform(a, OrientationFrame(_rand_rot(rng)), b, OrientationFrame(_rand_rot(rng)))
        assert np.allclose(t.apply(np.array(a.position)), b.position, atol=1e-6)


def test_similarity_from_correspondences_recovers_truth(rng):
    truth = SimilarityTransform7DOF(1.3, rotation_from_axis_angle([1, 2, 0.5], 25.0), np.array([4.0, -2.0, 7.0]))
    src = rng.uniform(0, 40, size=(30, 3))
    got = similarity_from_correspondences(src, truth.apply(src))
    assert got.scale == pytest.approx(1.3, rel=1e-9)
    assert np.allclose(got.rotation, truth.rotation, atol=1e-9)
    assert np.allclose(got.translation, truth.translation, atol=1e-7)
    with pytest.raises(ParameterError):
        similarity_from_correspondences(np.zeros((2, 3)), np.zeros((2, 3)))


def test_hough_consensus_recovers_exact_transform(rng):
    truth = SimilarityTransform7DOF(1.05, rotation_from_axis_angle([0, 0, 1], 12.0), np.array([3.0, -4.0, 2.0]))
    pairs_a, pairs_b, matches = [], [], []
    for i in range(12):
        pos, sigma, q = rng.uniform(10, 54, 3), rng.uniform(1.5, 4.0), _rand_rot(rng)
        pairs_a.append((_kp(pos, sigma), OrientationFrame(q)))
        pairs_b.append((_kp(truth.apply(pos), truth.scale * sigma), OrientationFrame(truth.rotation @ q)))
        matches.append(Match(i, i, 0.0, 1.0))
    res = hough_consensus(matches, pairs_a, pairs_b)
    assert len(res.inliers) == len(matches)
    assert res.transform.scale == pytest.approx(truth.scale, rel=1e-6)
    assert rotation_angle_deg(res.transform.rotation @ truth.rotation.T) < 1e-4
    assert np.allclose(res.transform.translation, truth.translation, atol=1e-5)
