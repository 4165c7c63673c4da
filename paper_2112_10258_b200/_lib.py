"""ctypes binding of ``libvolkey_b200.so`` (the C ABI in include/volkey_b200.h).

This is the reference-side binding a maintainer would add to volkey (see
INTEGRATION.md).  Loading the library needs no GPU; every compute entry point
needs one, and there is deliberately no CPU fallback: ``device()`` raises
``DeviceError`` when CUDA or the library is unavailable.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import DataError, DeviceError, ParameterError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VK_LIB_PATH") or os.path.join(_HERE, "libvolkey_b200.so")  # override: A/B variants

P = C.c_void_p
I = C.c_int
LL = C.c_longlong
D = C.c_double
F = C.c_float

# name -> argtypes (restype is int unless listed in _RESTYPE)
SIGNATURES = {
    "vk_last_error": [],
    "vk_abi_version": [],
    "vk_device_sm_count": [I],
    "vk_memset_async": [P, LL, P],
    "vk_launch_count": [],
    "vk_accum_work_bytes": [I],
    "vk_transpose_zfast_to_xfast": [P, P, I, I, I, I, P],
    "vk_transpose_xfast_to_zfast": [P, P, I, I, I, I, P],
    "vk_blur3d": [P, P, P, P, I, I, I, I, P, I, P],
    "vk_blur3d_ws": [P, P, P, P, I, I, I, I, P, I, P, LL, P],
    "vk_blur3d_ws2": [P, P, P, P, P, P, I, I, I, I, P, I, P, LL, P],
    "vk_set_blur_path": [I],
    "vk_set_xy_kernel": [I],
    "vk_set_z_kernel": [I],
    "vk_blur3d_chunked": [P, P, I, I, I, I, P, I, I, P],
    "vk_subsample_half": [P, P, I, I, I, I, P],
    "vk_small_octaves": [I, I, I, P, P, P, P, P, I, P],
    "vk_difference": [P, P, P, LL, P],
    "vk_sum_of_signs": [P, P, P, P, I, I, I, I, P],
    "vk_detect_octave": [P, I, I, I, I, I, I, I, F, P, P, I, P],
    "vk_extrema_from_map": [P, P, I, I, I, I, I, F, P, P, I, P],
    "vk_order_keypoints": [P, P, I, I, P, P, I, P, P, P, P, P, P, P, P, I, P],
    "vk_orient": [P, P, I, P, P, P, P, P, P, I, P, D, I, P, P, P, P, P, I, P, P, P, P, P],
    "vk_frames_from_weights": [P, I, I, P, D, I, P, P, P, P],
    "vk_expand_frames": [P, P, P, P, I, I, P, I, P, P, P, P, I, P, P],
    "vk_describe_siftrank": [P, P, P, P, P, I, I, P, P, P, P, P, I, P, P, P, P],
    "vk_gradient_volume": [P, P, P, I, I, I, I, P, P, P],
    "vk_describe_patch": [I, P, P, P, I, P, P, P, P, I, P, P, I, P, I, P, P, P],
    "vk_extract_patches": [P, P, P, I, P, P, P, P, I, P, P, I, P, P],
    "vk_orient_field": [P, P, P, I, I, I, I, P, P, P, P],
    "vk_match": [I, P, I, P, I, I, D, P, P, P, P, P],
    "vk_match_excluding": [I, P, I, P, I, I, D, I, I, P, P, P, P, P],
    "vk_set_match_path": [I],
    "vk_set_match_tc_kernel": [I],
    "vk_format_records": [LL, P, P, P, P, P, P, P, P, I, I, P, LL],
    "vk_gradients_at": [P, I, I, I, P, LL, P, P],
    "vk_sample_trilinear": [P, I, I, I, P, LL, P, P],
    "vk_match_rows_excluding": [P, I, P, I, I, D, P, P, P, P, P, P],
    "vk_orient_siftrank": [P, P, I, P, P, P, P, P, P, I, P, D, I, P, P, P, P, P, P, P, P, P, P, P, I, P, P],
    "vk_scatter_frame_rows": [P, P, P, I, I, P, P, P],
    "vk_refine_keypoints": [P, P, I, P, I, D, P, P, P],
    "vk_hough_init": [C.c_char_p],
    "vk_hough_dots": [I, P, P, P, I, P],
    "vk_hough_consensus": [I, P, P, P, P, P, P, P, P, P, P, P, I, P, I, P, P, P, P, P, P],
}
_RESTYPE = {"vk_last_error": C.c_char_p, "vk_launch_count": C.c_longlong, "vk_accum_work_bytes": C.c_longlong,
            "vk_format_records": C.c_longlong}

# device record layouts (must match include/volkey_b200.h)
LEVEL_DTYPE = np.dtype([("base", "<u8"), ("vol_stride", "<i8"), ("nx", "<i4"), ("ny", "<i4"), ("nz", "<i4"),
                        ("pad", "<i4")])
KP_DTYPE = np.dtype([(n, "<i4") for n in ("vol", "lvl", "ix", "iy", "iz", "ball", "octave", "level")])
BALL_DTYPE = np.dtype([(n, "<i4") for n in ("start", "count", "window_start", "max_d2", "zstart", "pstart", "r", "pad")])
GRADLEVEL_DTYPE = np.dtype([("g4", "<u8"), ("bin", "<u8"), ("vol_stride", "<i8"), ("nx", "<i4"), ("ny", "<i4"),
                            ("nz", "<i4"), ("kind", "<i4")])
FRAME_DTYPE = np.dtype([(n, "<i4") for n in ("kp", "prim", "sec", "pad")])

_lock = threading.Lock()
_lib = None


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load (building first if needed) the shared library; no GPU required."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            if not build_if_missing:
                raise DeviceError(f"{LIB_PATH} is missing; run python -m paper_2112_10258_b200.build")
            from . import build

            build.build()
        lib = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, I)
        _lib = lib
        return lib


def last_error() -> str:
    return (load().vk_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc == 0:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == 5:
        raise ParameterError(msg)
    if rc == 7:
        raise DataError(msg)
    raise DeviceError(f"libvolkey_b200 status {rc}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def accum_work():
    """Device scratch for vk_orient / vk_describe_siftrank (one per stream that
    runs them concurrently)."""
    t = torch()
    n = load().vk_accum_work_bytes(t.cuda.current_device())
    if n <= 0:
        raise DeviceError(f"vk_accum_work_bytes: {last_error()}")
    return t.empty(n // 8, dtype=t.float64, device="cuda")


_torch = None


def torch():
    """torch with a usable CUDA device, or DeviceError (no CPU fallback)."""
    global _torch
    if _torch is None:
        import torch as t

        if not t.cuda.is_available():
            raise DeviceError("no CUDA device: the B200 volkey path has no CPU fallback")
        load()
        _torch = t
    return _torch


def stream_ptr(stream=None) -> int:
    t = torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return s.cuda_stream


def ptr(t) -> int:
    return 0 if t is None else t.data_ptr()


def to_device_records(arr: np.ndarray):
    """Upload a numpy structured record array as a device byte tensor."""
    t = torch()
    raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
    if raw.size == 0:
        return t.empty(16, dtype=t.uint8, device="cuda")
    return t.from_numpy(raw.copy()).to("cuda", non_blocking=False)
