"""Device records for caller-built pyramids, keypoints and frames.

The stage functions of the drop-in API (``assign_orientations``,
``describe_all``, ``gradient_histogram``, ``sift_rank_descriptor``) accept
arbitrary ``GaussianPyramid`` / ``Keypoint`` / ``OrientationFrame`` objects --
the reference tests hand-build all three.  This module turns them into the
device records of include/volkey_b200.h (level table, vk_kp, vk_ball,
vk_frame + rotations) and runs the orientation / descriptor kernels on them.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from . import tables as T
from .engine import KIND_CODE, level_records
from .errors import DataError, ParameterError
from .volume import device_of


class PyramidView:
    """Level table of a GaussianPyramid (uploads host-resident levels once)."""

    def __init__(self, pyr, need_source: bool = False):
        self.pyr = pyr
        tensors, dims = [], []
        self.index = {}
        for o, oc in enumerate(pyr.octaves):
            for i, lv in enumerate(oc.levels):
                self.index[(o, i)] = len(tensors)
                tensors.append(device_of(lv))
                dims.append(tuple(lv.dims))
        self._keep = tensors
        self.dims = dims
        self.table = _lib.to_device_records(level_records(tensors, dims))
        self.source = None
        if need_source:
            if pyr.source is None:
                raise ParameterError("pyramid carries no source volume for patch extraction")
            src = device_of(pyr.source)
            self._keep.append(src)
            self.source = _lib.to_device_records(level_records([src], [tuple(pyr.source.dims)]))


def keypoint_records(view: PyramidView, keypoints, radius_factor: float, balls: T.BallTable):
    """vk_kp records via keypoint_local (orient.py:76-86) + ball ids."""
    if radius_factor <= 0:
        raise ParameterError(f"radius_factor must be > 0, got {radius_factor}")
    n = len(keypoints)
    rec = np.zeros(n, dtype=_lib.KP_DTYPE)
    pos = np.zeros((n, 3), dtype=np.float64)
    sig = np.zeros(n, dtype=np.float64)
    for j, kp in enumerate(keypoints):
        if not (0 <= kp.octave < len(view.pyr.octaves)):
            raise ParameterError(f"keypoint octave {kp.octave} outside pyramid")
        if not (0 <= kp.level < len(view.pyr.octaves[kp.octave].levels)):
            raise ParameterError(f"keypoint level {kp.level} outside octave {kp.octave}")
        scale = 2.0 ** kp.octave
        offset = (scale - 1.0) / 2.0
        c = [round((p - offset) / scale) for p in kp.position]
        radius = radius_factor * (kp.sigma / scale)
        rec[j] = (0, view.index[(kp.octave, kp.level)], c[0], c[1], c[2], balls.index(radius), kp.octave, kp.level)
        pos[j] = kp.position
        sig[j] = kp.sigma
    return rec, pos, sig


_LUT = {}


def _ico_lut(t):
    """Device copy of tables.icosphere_lut (per device, built once)."""
    dev = t.cuda.current_device()
    if dev not in _LUT:
        _LUT[dev] = t.from_numpy(T.icosphere_lut().copy()).cuda()
    return _LUT[dev]


def run_orientation(pyr, keypoints, radius_factor=4.0, secondary_ratio=0.8, max_frames=4, directions=None,
                    exact=False, want_weights=False):
    """Histograms (+ frames) for a list of keypoints.  Returns dict with
    nframes, prim, sec (int arrays) and optionally weights (n, K)."""
    t = _lib.torch()
    if not 0 < secondary_ratio <= 1:
        raise ParameterError(f"secondary_ratio must be in (0, 1], got {secondary_ratio}")
    if max_frames < 1:
        raise ParameterError(f"max_frames must be >= 1, got {max_frames}")
    mf = min(int(max_frames), 8)
    dirs = T.icosphere_directions() if directions is None else np.ascontiguousarray(directions, dtype=np.float64)
    if dirs.ndim != 2 or dirs.shape[1] != 3 or not 1 <= len(dirs) <= 64:
        raise ParameterError("directions must be a (K, 3) array with 1 <= K <= 64")
    ok, _ = T.default_frame_tables() if directions is None else T.frame_tables(dirs)
    n = len(keypoints)
    view = PyramidView(pyr)
    balls = T.BallTable()
    rec, _, _ = keypoint_records(view, keypoints, radius_factor, balls)
    if n == 0:
        return dict(nframes=np.zeros(0, np.int32), prim=np.zeros((0, mf), np.int32),
                    sec=np.zeros((0, mf), np.int32), weights=np.zeros((0, len(dirs))))
    b, off, win, planes = balls.arrays()
    d_kps = _lib.to_device_records(rec)
    d_balls = _lib.to_device_records(b)
    d_off = t.from_numpy(off.copy()).cuda()
    d_win = t.from_numpy(win.copy()).cuda()
    d_win32 = t.from_numpy(win.astype(np.float32)).cuda()
    d_dirs = t.from_numpy(dirs.copy()).cuda()
    d_ok = t.from_numpy(np.ascontiguousarray(ok).copy()).cuda()
    K = len(dirs)
    weights = t.empty(n * K, dtype=t.float64, device="cuda") if want_weights else None
    nframes = t.zeros(n, dtype=t.int32, device="cuda")
    prim = t.zeros(n * mf, dtype=t.int32, device="cuda")
    sec = t.zeros(n * mf, dtype=t.int32, device="cuda")
    status = t.zeros(4, dtype=t.int32, device="cuda")
    ico = np.ascontiguousarray(T.icosphere_structure()) if directions is None else None
    _lib.call("vk_orient", d_kps.data_ptr(), None, n, view.table.data_ptr(), d_balls.data_ptr(), d_off.data_ptr(),
              d_win.data_ptr(), d_win32.data_ptr(), d_dirs.data_ptr(), K, d_ok.data_ptr(), float(secondary_ratio), mf, _lib.ptr(weights),
              nframes.data_ptr(), prim.data_ptr(), sec.data_ptr(), status.data_ptr(), int(bool(exact)),
              None if ico is None else ico.ctypes.data, None if ico is None else _ico_lut(t).data_ptr(), None,
              _lib.accum_work().data_ptr(), _lib.stream_ptr())
    if int(status[0].item()) & 1:
        raise DataError("orientation neighborhood lies entirely outside the volume")
    out = dict(nframes=nframes.cpu().numpy(), prim=prim.cpu().numpy().reshape(n, mf),
               sec=sec.cpu().numpy().reshape(n, mf))
    if want_weights:
        out["weights"] = weights.cpu().numpy().reshape(n, K)
    return out


def run_descriptors(pyr, keypoints, rotations, kind="siftrank", pairs=None, patch_side=15, blur_sigma=0.95,
                    radius_factor=4.0, exact=False) -> np.ndarray:
    """Descriptors for (keypoint, rotation) pairs.  ``keypoints`` are the
    distinct keypoints, ``rotations`` a list of (keypoint index, 3x3 array)."""
    t = _lib.torch()
    m = len(rotations)
    view = PyramidView(pyr, need_source=kind != "siftrank")
    balls = T.BallTable()
    rec, pos, sig = keypoint_records(view, keypoints, radius_factor, balls)
    fr = np.zeros(m, dtype=_lib.FRAME_DTYPE)
    rot = np.zeros((m, 9), dtype=np.float64)
    for j, (ki, R) in enumerate(rotations):
        fr[j] = (ki, -1, -1, 0)
        rot[j] = np.asarray(R, dtype=np.float64).reshape(9)
    if kind == "siftrank":
        out = t.empty((max(m, 1), 64), dtype=t.uint8, device="cuda")
    elif kind == "brief":
        out = t.empty((max(m, 1), (pairs.n + 7) // 8), dtype=t.uint8, device="cuda")
    else:
        out = t.empty((max(m, 1), pairs.n), dtype=t.int16, device="cuda")
    if m == 0:
        return out[:0].cpu().numpy()
    b, off, win, planes = balls.arrays()
    d_kps = _lib.to_device_records(rec)
    d_fr = _lib.to_device_records(fr)
    d_rot = t.from_numpy(rot.reshape(-1).copy()).cuda()
    s = _lib.stream_ptr()
    if kind == "siftrank":
        d_balls = _lib.to_device_records(b)
        d_off = t.from_numpy(off.copy()).cuda()
        first = t.arange(m, dtype=t.int32, device="cuda")
        count = t.ones(m, dtype=t.int32, device="cuda")
        _lib.call("vk_describe_siftrank", d_fr.data_ptr(), d_rot.data_ptr(), first.data_ptr(), count.data_ptr(), None,
                  m, 1, d_kps.data_ptr(), view.table.data_ptr(), d_balls.data_ptr(), d_off.data_ptr(),
                  out.data_ptr(), int(bool(exact)), None, None, _lib.accum_work().data_ptr(), s)
    else:
        if patch_side < 1 or patch_side % 2 == 0:
            raise ParameterError(f"patch side must be odd and >= 1, got {patch_side}")
        if blur_sigma < 0:
            raise ParameterError(f"blur_sigma must be >= 0, got {blur_sigma}")
        grid = np.ascontiguousarray(T.patch_axis(patch_side), dtype=np.float64)
        if blur_sigma > 0:
            k = T.gaussian_kernel(blur_sigma)
            taps, radius = np.ascontiguousarray(k.weights), k.radius
        else:
            taps, radius = np.zeros(1, np.float32), 0
        pts = T.pair_points(pairs.p1, pairs.p2, patch_side, pairs.sigma_unit)
        d_pts = t.from_numpy(np.ascontiguousarray(pts).reshape(-1).copy()).cuda()
        d_pos = t.from_numpy(pos.reshape(-1).copy()).cuda()
        d_sig = t.from_numpy(sig.copy()).cuda()
        code = KIND_CODE[kind]
        _lib.call("vk_describe_patch", code, d_fr.data_ptr(), d_rot.data_ptr(), None, m, d_kps.data_ptr(),
                  d_pos.data_ptr(), d_sig.data_ptr(), view.source.data_ptr(), patch_side, grid.ctypes.data,
                  taps.ctypes.data, radius, d_pts.data_ptr(), pairs.n, out.data_ptr() if code == 1 else None,
                  out.data_ptr() if code == 2 else None, s)
    return out[:m].cpu().numpy()


def run_patches(pyr, keypoints, rotations, side=15, blur_sigma=0.0) -> np.ndarray:
    """(m, side, side, side) fp32 patches for (keypoint index, rotation) pairs:
    extract_patch (descriptor.py:96-111), pre-blurred when blur_sigma > 0."""
    t = _lib.torch()
    if side < 1 or side % 2 == 0:
        raise ParameterError(f"patch side must be odd and >= 1, got {side}")
    if blur_sigma < 0:
        raise ParameterError(f"blur_sigma must be >= 0, got {blur_sigma}")
    m = len(rotations)
    view = PyramidView(pyr, need_source=True)
    rec, pos, sig = keypoint_records(view, keypoints, 4.0, T.BallTable())
    out = t.empty((max(m, 1), side, side, side), dtype=t.float32, device="cuda")
    if m == 0:
        return out[:0].cpu().numpy()
    fr = np.zeros(m, dtype=_lib.FRAME_DTYPE)
    rot = np.zeros((m, 9), dtype=np.float64)
    for j, (ki, R) in enumerate(rotations):
        fr[j] = (ki, -1, -1, 0)
        rot[j] = np.asarray(R, dtype=np.float64).reshape(9)
    grid = np.ascontiguousarray(T.patch_axis(side), dtype=np.float64)
    if blur_sigma > 0:
        k = T.gaussian_kernel(blur_sigma)
        taps, radius = np.ascontiguousarray(k.weights), k.radius
    else:
        taps, radius = np.zeros(1, np.float32), 0
    d_kps, d_fr = _lib.to_device_records(rec), _lib.to_device_records(fr)
    d_rot = t.from_numpy(rot.reshape(-1).copy()).cuda()
    d_pos = t.from_numpy(pos.reshape(-1).copy()).cuda()
    d_sig = t.from_numpy(sig.copy()).cuda()
    _lib.call("vk_extract_patches", d_fr.data_ptr(), d_rot.data_ptr(), None, m, d_kps.data_ptr(), d_pos.data_ptr(),
              d_sig.data_ptr(), view.source.data_ptr(), side, grid.ctypes.data, taps.ctypes.data, radius,
              out.data_ptr(), _lib.stream_ptr())
    return out[:m].cpu().numpy()
