"""Known answers of the reference suite, checked on
the GPU path: Gaussian tap ratio, 2x2x2 mean, DoG impulse centre, strict
maximum scores 80, octave rescaling of keypoint position / sigma, band
monotonicity, rank examples, flat SIFT-Rank, popcount."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

vk = pytest.importorskip("paper_2112_10258_b200")
from paper_2112_10258_b200.descriptor import rank_vector  # noqa: E402
from paper_2112_10258_b200.detect import extract_extrema, sum_of_signs_map  # noqa: E402
from paper_2112_10258_b200.scalespace import (build_dog_pyramid, build_gaussian_pyramid, gaussian_kernel,  # noqa: E402
                                              subsample_half)


def test_gaussian_tap_ratio_and_symmetry():
    k = gaussian_kernel(1.0)
    assert k.weights[k.radius] / k.weights[k.radius + 1] == pytest.approx(math.exp(0.5), rel=1e-5)
    k = gaussian_kernel(1.7)
    assert np.array_equal(k.weights, k.weights[::-1]) and len(k.weights) == 2 * k.radius + 1


def test_subsample_mean_of_eight():
    out = subsample_half(vk.Volume(np.arange(8, dtype=np.float32).reshape(2, 2, 2)))
    assert out.dims == (1, 1, 1) and out.data[0, 0, 0] == 3.5 and tuple(out.spacing) == (2.0, 2.0, 2.0)


def test_dog_impulse_centre():
    base, n = 1.6, 65
    arr = np.zeros((n, n, n), dtype=np.float32)
    arr[n // 2, n // 2, n // 2] = 1.0
    dog = build_dog_pyramid(build_gaussian_pyramid(vk.Volume(arr), base, 6, 1))
    k0 = gaussian_kernel(base)
    k_inc = gaussian_kernel(((base * 2 ** (1 / 3)) ** 2 - base ** 2) ** 0.5)
    c0 = float(k0.weights[k0.radius]) ** 3
    g1 = np.convolve(k0.weights.astype(np.float64), k_inc.weights.astype(np.float64))
    c1 = float(g1[len(g1) // 2]) ** 3
    assert float(dog.octaves[0].levels[0].data[n // 2, n // 2, n // 2]) == pytest.approx(c0 - c1, abs=1e-5)


def test_strict_maximum_scores_80_and_octave_rescaling():
    arr = np.zeros((5, 5, 5), dtype=np.float32)
    arr[2, 2, 2] = 1.0
    cur, flat = vk.Volume(arr), vk.Volume(np.zeros((5, 5, 5), dtype=np.float32))
    m = sum_of_signs_map(flat, cur, flat)
    assert m[2, 2, 2] == 80 and np.abs(m).max() <= 80
    (kp,) = extract_extrema(m, cur, 0, 0.0, octave=2, level=1, sigma_local=2.0)
    assert kp.position == (9.5, 9.5, 9.5) and kp.sigma == pytest.approx(8.0)
    const = vk.Volume(np.full((6, 6, 6), 2.0, dtype=np.float32))
    assert not np.any(sum_of_signs_map(const, const, const))


def test_band_monotonicity():
    rng = np.random.default_rng(5)
    prev, cur, nxt = (vk.Volume(rng.random((9, 9, 9), dtype=np.float32)) for _ in range(3))
    m = sum_of_signs_map(prev, cur, nxt)
    got_prev = set()
    for band in (0, 4, 12, 30):
        got = {(k.position, k.sign) for k in extract_extrema(m, cur, band, 0.0)}
        assert got_prev <= got
        got_prev = got


def test_rank_and_popcount_examples():
    assert rank_vector(np.array([3.1, -2.0, 7.4])).tolist() == [1, 0, 2]
    assert rank_vector(np.array([5, 5, 5, 1])).tolist() == [1, 2, 3, 0]
    from paper_2112_10258_b200.match import hamming_distances

    a = np.array([[0xFF, 0x00]], dtype=np.uint8)
    b = np.array([[0x0F, 0x00], [0xFF, 0xFF]], dtype=np.uint8)
    assert hamming_distances(a, b).tolist() == [[4.0, 8.0]]
