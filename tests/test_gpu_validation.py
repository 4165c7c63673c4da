"""Parameter validation of the drop-in API matches the reference's errors
(scalespace.py:172-177, detect.py:96-97,163-164, match.py:93-98,
descriptor.py:99-100,145-160, orient.py:128-138): ParameterError with the
offending value, raised before any device work."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

vk = pytest.importorskip("paper_2112_10258_b200")
from paper_2112_10258_b200.descriptor import describe_all, sample_point_pairs  # noqa: E402
from paper_2112_10258_b200.detect import detect_keypoints  # noqa: E402
from paper_2112_10258_b200.errors import ParameterError  # noqa: E402
from paper_2112_10258_b200.match import nearest_neighbor_matches  # noqa: E402
from paper_2112_10258_b200.scalespace import build_dog_pyramid, build_gaussian_pyramid  # noqa: E402


@pytest.fixture(scope="module")
def vol():
    return vk.Volume(np.random.default_rng(3).random((20, 18, 16), dtype=np.float32))


@pytest.mark.parametrize("kw", [dict(base_sigma=0.0), dict(base_sigma=-1.0), dict(levels_per_octave=3),
                                dict(num_octaves=0), dict(workers=0), dict(chunk=0)])
def test_pyramid_parameters(vol, kw):
    with pytest.raises(ParameterError):
        build_gaussian_pyramid(vol, **kw)


def test_detection_parameters(vol):
    dog = build_dog_pyramid(build_gaussian_pyramid(vol, num_octaves=1))
    for band in (-1, 81):
        with pytest.raises(ParameterError):
            detect_keypoints(dog, threshold_band=band)
    assert isinstance(detect_keypoints(dog, threshold_band=80), list)


def test_matching_parameters():
    a = np.random.default_rng(1).random((4, 8))
    with pytest.raises(ParameterError):
        nearest_neighbor_matches(a, a, metric="cosine")
    for r in (0.0, 1.5):
        with pytest.raises(ParameterError):
            nearest_neighbor_matches(a, a, ratio_max=r)
    with pytest.raises(ParameterError):
        nearest_neighbor_matches(a, a[:1])
    assert nearest_neighbor_matches(a[:0], a) == []


def test_descriptor_parameters(vol):
    pyr = build_gaussian_pyramid(vol, num_octaves=1)
    with pytest.raises(ParameterError):
        sample_point_pairs(6, 64)
    with pytest.raises(ParameterError):
        sample_point_pairs(3, 0)
    with pytest.raises(ParameterError):
        sample_point_pairs(3, 64, sigma_unit=0.0)
    with pytest.raises(ParameterError):
        describe_all(pyr, [], kind="orb")


def test_config_validation():
    with pytest.raises(Exception):
        vk.PipelineConfig(descriptor="orb")
    with pytest.raises(Exception):
        vk.PipelineConfig(patch_side=14)
