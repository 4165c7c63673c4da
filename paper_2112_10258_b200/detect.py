"""4-D scale-space extrema on the GPU -- drop-in for volkey detect.py.

Same names and semantics as detect.py:23-182.  ``detect_keypoints`` runs
``vk_detect_octave`` (early-exit 80-neighbour test, no map materialised) and
``vk_order_keypoints`` (reference order); ``sum_of_signs_map`` and
``extract_extrema`` expose the two halves separately for parity tests.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Literal

import numpy as np

from . import _lib
from .engine import level_records
from .errors import ParameterError
from .scalespace import DoGPyramid, _stage
from .volume import Volume, device_of

SCALE_CALIBRATION = math.sqrt(1.5)  # detect.py:26


@dataclass(frozen=True)
class Keypoint:
    """Scale-space extremum in base-volume voxel coordinates (detect.py:36-45)."""

    position: tuple[float, float, float]
    sigma: float
    octave: int
    level: int
    dog_value: float
    sign: Literal["peak", "valley"]


def sum_of_signs_map(dog_prev: Volume, dog_cur: Volume, dog_next: Volume, workers: int = 1) -> np.ndarray:
    """detect.py:48-79 -> int16 map ``[x, y, z]``."""
    if not (dog_prev.dims == dog_cur.dims == dog_next.dims):
        raise ParameterError(f"DoG triple dims differ: {dog_prev.dims}, {dog_cur.dims}, {dog_next.dims}")
    if workers < 1:
        raise ParameterError(f"workers must be >= 1, got {workers}")
    t = _lib.torch()
    nx, ny, nz = dog_cur.dims
    a, b, c = device_of(dog_prev), device_of(dog_cur), device_of(dog_next)
    out = t.empty((nz, ny, nx), dtype=t.int16, device="cuda")
    _lib.call("vk_sum_of_signs", a.data_ptr(), b.data_ptr(), c.data_ptr(), out.data_ptr(), 1, nx, ny, nz,
              _lib.stream_ptr())
    return out.permute(2, 1, 0).contiguous().cpu().numpy()


def level_sigma_local(dog: DoGPyramid, octave: int, level: int) -> float:
    """detect.py:143-146."""
    finer = dog.octaves[octave].sigmas[level] / (2.0 ** octave)
    return finer * math.sqrt(dog.kappa) * SCALE_CALIBRATION


def _keypoints_from(cand_keys, cand_count, cap, seg_info, seg_sigma, dog_tensors, dims_list) -> list[Keypoint]:
    """vk_order_keypoints + host Keypoint objects (one volume)."""
    t = _lib.torch()
    dog_table = _lib.to_device_records(level_records(dog_tensors, dims_list))
    kp_cap = cap
    kps = t.empty(kp_cap * 32, dtype=t.uint8, device="cuda")
    pos = t.empty(kp_cap * 3, dtype=t.float64, device="cuda")
    sig = t.empty(kp_cap, dtype=t.float64, device="cuda")
    dg = t.empty(kp_cap, dtype=t.float32, device="cuda")
    sg = t.empty(kp_cap, dtype=t.int8, device="cuda")
    voff = t.zeros(1, dtype=t.int32, device="cuda")
    total = t.zeros(2, dtype=t.int32, device="cuda")
    si = np.ascontiguousarray(seg_info, dtype=np.int32)
    ss = np.ascontiguousarray(seg_sigma, dtype=np.float64)
    _lib.call("vk_order_keypoints", cand_keys.data_ptr(), cand_count.data_ptr(), 1, cap, si.ctypes.data,
              ss.ctypes.data, len(ss), dog_table.data_ptr(), kps.data_ptr(), pos.data_ptr(), sig.data_ptr(),
              dg.data_ptr(), sg.data_ptr(), voff.data_ptr(), total.data_ptr(), kp_cap, _lib.stream_ptr())
    n, over = (int(v) for v in total.cpu())
    if over:
        return None  # caller retries with a larger capacity
    rec = kps[: 32 * n].cpu().numpy().view(_lib.KP_DTYPE)
    P = pos[: 3 * n].cpu().numpy().reshape(n, 3).tolist()
    S = sig[:n].cpu().numpy().tolist()
    D = dg[:n].cpu().numpy().astype(np.float64).tolist()
    G = sg[:n].cpu().numpy().tolist()
    octs, levs = rec["octave"].tolist(), rec["level"].tolist()
    return [Keypoint(tuple(P[i]), S[i], octs[i], levs[i], D[i], "peak" if G[i] > 0 else "valley") for i in range(n)]


def extract_extrema(extremum_map: np.ndarray, dog_cur: Volume, threshold_band: int, contrast_min: float,
                    octave: int = 0, level: int = 0, sigma_local: float = 1.0) -> list[Keypoint]:
    """detect.py:82-140 from a caller-supplied map."""
    if not 0 <= threshold_band <= 80:
        raise ParameterError(f"threshold_band must be in [0, 80], got {threshold_band}")
    nx, ny, nz = dog_cur.dims
    if min(nx, ny, nz) < 3:
        return []
    t = _lib.torch()
    m = t.from_numpy(np.ascontiguousarray(np.asarray(extremum_map, dtype=np.int16).transpose(2, 1, 0))).cuda()
    d = device_of(dog_cur)
    cap = max(1024, nx * ny * nz // 64)
    while True:
        keys = t.empty(cap, dtype=t.int64, device="cuda")
        cnt = t.zeros(1, dtype=t.int32, device="cuda")
        _lib.call("vk_extrema_from_map", m.data_ptr(), d.data_ptr(), nx, ny, nz, 0, threshold_band,
                  float(np.float32(contrast_min)), keys.data_ptr(), cnt.data_ptr(), cap, _lib.stream_ptr())
        seg_info = np.array([[octave, level, -1, -1]], dtype=np.int32)
        seg_sigma = np.array([sigma_local * 2.0 ** octave])
        out = _keypoints_from(keys, cnt, cap, seg_info, seg_sigma, [d], [dog_cur.dims])
        if out is not None:
            return out
        cap = int(cnt.item()) + 1


def detect_keypoints(dog: DoGPyramid, threshold_band: int = 0, contrast_min: float = 0.0, workers: int = 1,
                     recorder=None) -> list[Keypoint]:
    """detect.py:149-182: every consecutive DoG triple, reference order."""
    if not 0 <= threshold_band <= 80:
        raise ParameterError(f"threshold_band must be in [0, 80], got {threshold_band}")
    if workers < 1:
        raise ParameterError(f"workers must be >= 1, got {workers}")
    t = _lib.torch()
    rec = _stage(recorder)
    nlev = max(len(o.levels) for o in dog.octaves) if dog.octaves else 0
    for o, oc in enumerate(dog.octaves):
        if len(oc.levels) < 3:
            raise ParameterError(f"octave {o} has {len(oc.levels)} DoG levels; need >= 3")
    nseg = max(1, len(dog.octaves) * nlev)
    if nseg > 128 or nlev > 32:
        raise ParameterError("too many DoG levels for the device detector")
    devs = [[device_of(lv) for lv in oc.levels] for oc in dog.octaves]
    seg_info = np.full((nseg, 4), -1, dtype=np.int32)
    seg_sigma = np.zeros(nseg)
    dog_t, dims_l = [None] * nseg, [None] * nseg
    vox = max((int(np.prod(oc.levels[0].dims)) for oc in dog.octaves), default=1)
    cap = max(4096, vox // 64)
    while True:
        keys = t.empty(cap, dtype=t.int64, device="cuda")
        cnt = t.zeros(1, dtype=t.int32, device="cuda")
        for o, oc in enumerate(dog.octaves):
            nx, ny, nz = oc.levels[0].dims
            for i in range(len(oc.levels)):
                dog_t[o * nlev + i] = devs[o][i]
                dims_l[o * nlev + i] = oc.levels[i].dims
            for i in range(1, len(oc.levels) - 1):
                seg_info[o * nlev + i] = (o, i, -1, -1)
                seg_sigma[o * nlev + i] = level_sigma_local(dog, o, i) * 2.0 ** o
            ptrs = (C.c_void_p * len(oc.levels))(*[d.data_ptr() for d in devs[o]])
            with rec("peak_detect", o, 0):
                _lib.call("vk_detect_octave", C.cast(ptrs, C.c_void_p), len(oc.levels), 1, nx, ny, nz, o * nlev,
                          threshold_band, float(np.float32(contrast_min)), keys.data_ptr(), cnt.data_ptr(), cap,
                          _lib.stream_ptr())
        out = _keypoints_from(keys, cnt, cap, seg_info, seg_sigma, dog_t, dims_l)
        if out is not None:
            return out
        cap = int(cnt.item()) + 1
