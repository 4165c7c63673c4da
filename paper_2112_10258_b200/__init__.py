"""B200-native volkey: 3-D SIFT-Rank / BRIEF / RRIEF detect + describe + match.

Drop-in for the reference package's public API (volkey/__init__.py:5-28,
hot path only): the same names, signatures, dataclasses and errors, computed
by hand-written sm_100a kernels in ``libvolkey_b200.so`` (C ABI:
include/volkey_b200.h).  There is no CPU fallback: compute entry points raise
``DeviceError`` without a CUDA device.
"""

__version__ = "0.1.0"

from .config import PipelineConfig
from .consensus import (ConsensusResult, HoughSettings, SimilarityTransform7DOF, count_inlier_matches, hough_consensus,
                        match_records, similarity_from_correspondences, vote_transform)
from .detect import Keypoint, detect_keypoints
from .engine import Extractor
from .ingest import load_nifti_subset, load_raw, load_volume, read_raw_header, save_raw
from .errors import DataError, DeviceError, NoConsensusError, ParameterError, VolkeyError
from .match import Match, nearest_neighbor_matches
from .pipeline import ExtractionResult, assign_orientations, extract_batch, extract_features
from .scalespace import build_dog_pyramid, build_gaussian_pyramid
from .volume import DeviceVolume, Volume

__all__ = [
    "__version__",
    "PipelineConfig",
    "Keypoint",
    "detect_keypoints",
    "Extractor",
    "ExtractionResult",
    "extract_features",
    "extract_batch",
    "assign_orientations",
    "build_dog_pyramid",
    "build_gaussian_pyramid",
    "Volume",
    "load_raw",
    "save_raw",
    "read_raw_header",
    "load_nifti_subset",
    "load_volume",
    "DeviceVolume",
    "Match",
    "nearest_neighbor_matches",
    "hough_consensus",
    "match_records",
    "count_inlier_matches",
    "vote_transform",
    "similarity_from_correspondences",
    "HoughSettings",
    "ConsensusResult",
    "SimilarityTransform7DOF",
    "NoConsensusError",
    "VolkeyError",
    "ParameterError",
    "DataError",
    "DeviceError",
]
