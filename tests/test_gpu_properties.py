"""Size-independent properties of the GPU path (the covariance / invariance
checks of the reference's acceptance and scale-space suites, run on this
package): integer translation, polarity, power-of-two gain, constant and
impulse inputs, octave handoff and truncation, monotone smoothing.  They hold
for the reference by construction and must hold bit for bit here too."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

vk = pytest.importorskip("paper_2112_10258_b200")
from paper_2112_10258_b200 import synthetic  # noqa: E402
from paper_2112_10258_b200.config import PipelineConfig  # noqa: E402
from paper_2112_10258_b200.descriptor import descriptor_array  # noqa: E402
from paper_2112_10258_b200.scalespace import (build_gaussian_pyramid, convolve_separable,  # noqa: E402
                                              gaussian_kernel, subsample_half)


@pytest.fixture
def rng():
    return np.random.default_rng(7)


def test_integer_translation_shifts_octave0_keypoints(rng):
    """A cyclic shift by whole voxels moves every interior octave-0 keypoint by
    exactly that shift (same level, same polarity)."""
    vol = synthetic.random_blob_phantom((56, 56, 56), rng, n_blobs=6, margin=20, sigma_range=(2.0, 3.5))
    shift = (3, 2, 1)
    cfg = PipelineConfig(num_octaves=1)
    kp0 = [k for k in vk.extract_features(vk.Volume(vol), cfg).keypoints
           if all(18 <= c < 38 for c in k.position)]
    moved = {(k.position, k.level, k.sign)
             for k in vk.extract_features(vk.Volume(np.roll(vol, shift, axis=(0, 1, 2))), cfg).keypoints}
    assert kp0
    for k in kp0:
        assert (tuple(p + s for p, s in zip(k.position, shift)), k.level, k.sign) in moved


def test_negation_swaps_polarity(rng):
    vol = synthetic.random_blob_phantom((40, 40, 40), rng, n_blobs=6, margin=8)
    cfg = PipelineConfig(num_octaves=2)
    pos = vk.extract_features(vk.Volume(vol), cfg).keypoints
    neg = vk.extract_features(vk.Volume(-vol), cfg).keypoints
    assert len(pos) == len(neg) > 0
    flip = {"peak": "valley", "valley": "peak"}
    for a, b in zip(pos, neg):
        assert a.position == b.position and a.sigma == b.sigma and flip[a.sign] == b.sign


@pytest.mark.parametrize("kind", ["siftrank", "brief", "rrief"])
def test_power_of_two_gain_is_exact(rng, kind):
    """x2 gain is exact in float arithmetic end to end: same keypoints, DoG
    values doubled exactly, descriptors bit-identical."""
    vol = synthetic.soup_volume((48, 48, 48), rng)
    cfg = PipelineConfig(num_octaves=2, descriptor=kind)
    a = vk.extract_features(vk.Volume(vol), cfg)
    b = vk.extract_features(vk.Volume(2.0 * vol), cfg)
    assert len(a.keypoints) == len(b.keypoints) > 0
    for ka, kb in zip(a.keypoints, b.keypoints):
        assert (ka.position, ka.sigma, ka.octave, ka.level, ka.sign) == (kb.position, kb.sigma, kb.octave, kb.level,
                                                                         kb.sign)
        assert kb.dog_value == 2.0 * ka.dog_value
    assert np.array_equal(descriptor_array(a.records, kind), descriptor_array(b.records, kind))


def test_constant_volume_has_no_keypoints():
    res = vk.extract_features(vk.Volume(np.full((24, 24, 24), 3.0, dtype=np.float32)), PipelineConfig(num_octaves=2))
    assert res.keypoints == [] and res.records == []
    for oc in res.dog.octaves:  # every voxel sums the same taps in the same order: each level is constant
        for lv in oc.levels:
            assert np.ptp(lv.data) == 0.0


def test_impulse_response_is_outer_product_of_taps():
    k = gaussian_kernel(1.0)
    n = 4 * k.radius + 3
    arr = np.zeros((n, n, n), dtype=np.float32)
    c = n // 2
    arr[c, c, c] = 1.0
    out = convolve_separable(vk.Volume(arr), k).data
    w = k.weights.astype(np.float64)
    want = np.zeros((n, n, n))
    s = slice(c - k.radius, c + k.radius + 1)
    want[s, s, s] = w[:, None, None] * w[None, :, None] * w[None, None, :]
    assert np.allclose(out, want, atol=1e-6)


def test_octave_handoff_equals_explicit_subsample(rng):
    vol = vk.Volume(rng.random((40, 40, 40), dtype=np.float32))
    pyr = build_gaussian_pyramid(vol, 1.6, 6, 2)
    assert np.array_equal(pyr.octaves[1].levels[0].data, subsample_half(pyr.octaves[0].levels[3]).data)


def test_octave_truncation_and_brain_octave_count(rng):
    assert build_gaussian_pyramid(vk.Volume(rng.random((20, 20, 20), dtype=np.float32)), num_octaves=6).num_octaves == 3
    assert build_gaussian_pyramid(vk.Volume(rng.random((145, 174, 145), dtype=np.float32)), 1.6, 6, 6).num_octaves == 6


def test_smoothing_is_monotone(rng):
    pyr = build_gaussian_pyramid(vk.Volume(rng.random((24, 24, 24), dtype=np.float32)), num_octaves=1)
    hi = [float(lv.data.max()) for lv in pyr.octaves[0].levels]
    lo = [float(lv.data.min()) for lv in pyr.octaves[0].levels]
    assert all(b <= a + 1e-6 for a, b in zip(hi, hi[1:]))
    assert all(b >= a - 1e-6 for a, b in zip(lo, lo[1:]))
