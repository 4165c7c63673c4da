"""Orientation frames on the GPU -- drop-in for volkey orient.py.

Same names and semantics as orient.py:22-168.  ``gradient_histogram`` runs
``vk_orient`` in exact mode (votes accumulated in the reference order, so the
returned weights are bit-identical); ``dominant_orientations`` runs
``vk_frames_from_weights``.  The direction set, integer balls and frame
tables are host constants (tables.py), exactly as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from . import tables as T
from .errors import ParameterError


@dataclass(frozen=True)
class SphericalHistogram:
    directions: np.ndarray
    weights: np.ndarray


@dataclass(frozen=True)
class OrientationFrame:
    rotation: np.ndarray  # (3, 3), columns are the frame axes


icosphere_directions = T.icosphere_directions
_ball_offsets = T.ball_offsets


def keypoint_local(pyr, kp):
    """orient.py:76-86 (host bookkeeping; the level data is downloaded)."""
    if not (0 <= kp.octave < len(pyr.octaves)):
        raise ParameterError(f"keypoint octave {kp.octave} outside pyramid")
    octave = pyr.octaves[kp.octave]
    if not (0 <= kp.level < len(octave.levels)):
        raise ParameterError(f"keypoint level {kp.level} outside octave {kp.octave}")
    scale = 2.0 ** kp.octave
    offset = (scale - 1.0) / 2.0
    center = np.array([round((c - offset) / scale) for c in kp.position], dtype=np.intp)
    return center, kp.sigma / scale, octave.levels[kp.level].data


def gradient_histogram(pyr, kp, radius_factor: float = 4.0, directions: np.ndarray | None = None) -> SphericalHistogram:
    """orient.py:89-125 on the GPU (exact accumulation order)."""
    from .stages import run_orientation

    dirs = icosphere_directions() if directions is None else np.asarray(directions, dtype=np.float64)
    out = run_orientation(pyr, [kp], radius_factor, 0.8, 1, directions=directions, exact=True, want_weights=True)
    return SphericalHistogram(dirs, out["weights"][0])


def _frames(dirs, prim, sec, n) -> list[OrientationFrame]:
    if dirs is None:
        _, rot = T.default_frame_tables()
    else:
        _, rot = T.frame_tables(dirs)
    frames = []
    for f in range(n):
        r = rot[prim[f], sec[f]].copy()
        r.setflags(write=False)
        frames.append(OrientationFrame(r))
    return frames


def dominant_orientations(h: SphericalHistogram, secondary_ratio: float = 0.8, max_frames: int = 4) -> list[OrientationFrame]:
    """orient.py:128-168: frames for every direction reaching secondary_ratio * max."""
    if not 0 < secondary_ratio <= 1:
        raise ParameterError(f"secondary_ratio must be in (0, 1], got {secondary_ratio}")
    if max_frames < 1:
        raise ParameterError(f"max_frames must be >= 1, got {max_frames}")
    t = _lib.torch()
    w = np.ascontiguousarray(h.weights, dtype=np.float64)
    dirs = np.ascontiguousarray(h.directions, dtype=np.float64)
    K = len(w)
    if K == 0:
        return []
    default = dirs.shape == (42, 3) and np.array_equal(dirs, icosphere_directions())
    ok, _ = T.default_frame_tables() if default else T.frame_tables(dirs)
    mf = min(int(max_frames), 8) if K else 1
    d_w = t.from_numpy(w.copy()).cuda()
    d_ok = t.from_numpy(np.ascontiguousarray(ok).copy()).cuda()
    nf = t.zeros(1, dtype=t.int32, device="cuda")
    pr = t.zeros(mf, dtype=t.int32, device="cuda")
    se = t.zeros(mf, dtype=t.int32, device="cuda")
    _lib.call("vk_frames_from_weights", d_w.data_ptr(), 1, K, d_ok.data_ptr(), float(secondary_ratio), mf,
              nf.data_ptr(), pr.data_ptr(), se.data_ptr(), _lib.stream_ptr())
    n = int(nf.item())
    return _frames(None if default else dirs, pr.cpu().numpy(), se.cpu().numpy(), n)
