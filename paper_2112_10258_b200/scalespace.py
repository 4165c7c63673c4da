"""Gaussian scale space on the GPU -- drop-in for volkey scalespace.py.

Same names, signatures, dataclasses and errors as the reference
(scalespace.py:35-235); every voxel is computed by ``vk_blur3d`` /
``vk_subsample_half`` / ``vk_difference`` (csrc/vk_pyramid.cu).  Levels are
returned as ``DeviceVolume`` (a ``Volume`` whose ``.data`` downloads lazily).
``workers`` / ``chunk`` are accepted for API compatibility and validated like
the reference (parallel.py:20-32); they do not change results there either.
"""

from __future__ import annotations

from contextlib import nullcontext
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ParameterError
from .tables import GaussianKernel1D, gaussian_kernel, incremental_sigma  # noqa: F401 (re-exported)
from .volume import DeviceVolume, Volume, device_of, to_device, to_host

MIN_OCTAVE_DIM = 4
DEFAULT_CHUNK = 32


def _check_exec(workers: int, chunk: int) -> None:
    if workers < 1:
        raise ParameterError(f"workers must be >= 1, got {workers}")
    if chunk < 1:
        raise ParameterError(f"chunk must be >= 1, got {chunk}")


def _stage(recorder):
    """recorder.stage(...) that also waits for the GPU, so wall time = device
    time; recorders that time with CUDA events (``device = True``,
    timing.DeviceStageRecorder) are used as they are, without synchronising."""
    if recorder is None:
        return lambda *a: nullcontext()
    if getattr(recorder, "device", False):
        return recorder.stage

    def ctx(name, octave, level):
        inner = recorder.stage(name, octave, level)

        class _C:
            def __enter__(self):
                _lib.torch().cuda.synchronize()
                return inner.__enter__()

            def __exit__(self, *exc):
                _lib.torch().cuda.synchronize()
                return inner.__exit__(*exc)

        return _C()

    return ctx


def blur_device(src, kernel: GaussianKernel1D, dog=None, half=None, stream=None):
    """Blur an x-fastest (nz, ny, nx) tensor; optional fused DoG / subsample outputs."""
    t = _lib.torch()
    nz, ny, nx = src.shape[-3:]
    nb = src.numel() // (nx * ny * nz)
    dst = t.empty_like(src)
    w = np.ascontiguousarray(kernel.weights, dtype=np.float32)
    _lib.call("vk_blur3d", src.data_ptr(), dst.data_ptr(), _lib.ptr(dog), _lib.ptr(half), nb, nx, ny, nz,
              w.ctypes.data, kernel.radius, _lib.stream_ptr(stream))
    return dst


def blur_device_chunked(src, kernel: GaussianKernel1D, chunk: int, stream=None):
    """blur_device with the work granularity set by `chunk`: the z pass runs
    `chunk` output planes per CTA (vk_blur3d_chunked) -- the GPU analogue of
    the reference's k^3-voxel tasks (finer = more warm-up re-reads and CTAs).
    The result does not depend on `chunk`."""
    t = _lib.torch()
    nz, ny, nx = src.shape[-3:]
    nb = src.numel() // (nx * ny * nz)
    dst = t.empty_like(src)
    w = np.ascontiguousarray(kernel.weights, dtype=np.float32)
    _lib.call("vk_blur3d_chunked", src.data_ptr(), dst.data_ptr(), nb, nx, ny, nz, w.ctypes.data, kernel.radius,
              int(chunk), _lib.stream_ptr(stream))
    return dst


def convolve_array(arr: np.ndarray, kernel: GaussianKernel1D, workers: int = 1, chunk: int = DEFAULT_CHUNK) -> np.ndarray:
    """scalespace.py:45-70 on the GPU; returns a float32 numpy array."""
    _check_exec(workers, chunk)
    a = np.asarray(arr, dtype=np.float32)
    return np.array(to_host(blur_device_chunked(to_device(a), kernel, chunk)))


def convolve_separable(v: Volume, kernel: GaussianKernel1D, workers: int = 1, chunk: int = DEFAULT_CHUNK) -> Volume:
    """scalespace.py:45-64 (chunk = z planes per CTA of the z pass)."""
    _check_exec(workers, chunk)
    return DeviceVolume(blur_device_chunked(device_of(v), kernel, chunk), v.spacing)


def subsample_half(v: Volume) -> Volume:
    """scalespace.py:95-109."""
    nx, ny, nz = v.dims
    if min(nx, ny, nz) < 2:
        raise ParameterError(f"cannot subsample dims {v.dims}: every dim must be >= 2")
    t = _lib.torch()
    src = device_of(v)
    dst = t.empty((nz // 2, ny // 2, nx // 2), dtype=t.float32, device="cuda")
    _lib.call("vk_subsample_half", src.data_ptr(), dst.data_ptr(), 1, nx, ny, nz, _lib.stream_ptr())
    return DeviceVolume(dst, tuple(2.0 * s for s in v.spacing))


@dataclass
class PyramidOctave:
    levels: list
    sigmas: list


@dataclass
class GaussianPyramid:
    octaves: list
    base_sigma: float
    kappa: float
    levels_per_octave: int
    source: Volume | None = None

    @property
    def num_octaves(self) -> int:
        return len(self.octaves)

    def local_sigma(self, octave: int, level: int) -> float:
        return self.octaves[octave].sigmas[level] / (2.0 ** octave)


@dataclass
class DoGOctave:
    levels: list
    sigmas: list


@dataclass
class DoGPyramid:
    octaves: list
    kappa: float
    levels_per_octave: int = 0

    @property
    def num_octaves(self) -> int:
        return len(self.octaves)


def build_gaussian_pyramid(v: Volume, base_sigma: float = 1.6, levels_per_octave: int = 6, num_octaves: int = 6,
                           workers: int = 1, chunk: int = DEFAULT_CHUNK, min_octave_dim: int = MIN_OCTAVE_DIM,
                           recorder=None) -> GaussianPyramid:
    """scalespace.py:158-206; the handoff subsample is fused into the blur that
    produces the handoff level (recorded under that level's "convolution")."""
    from .config import PipelineConfig
    from .engine import Plan

    if base_sigma <= 0:
        raise ParameterError(f"base_sigma must be > 0, got {base_sigma}")
    if levels_per_octave < 4:
        raise ParameterError(f"levels_per_octave must be >= 4, got {levels_per_octave}")
    if num_octaves < 1:
        raise ParameterError(f"num_octaves must be >= 1, got {num_octaves}")
    _check_exec(workers, chunk)
    plan = Plan.build(v.dims, PipelineConfig.model_construct(
        base_sigma=base_sigma, levels_per_octave=levels_per_octave, num_octaves=num_octaves,
        min_octave_dim=min_octave_dim, radius_factor=4.0), segments=False)
    rec = _stage(recorder)
    t = _lib.torch()
    handoff = levels_per_octave - 3
    src = device_of(v)
    octaves = []
    cur_dev, spacing = src, v.spacing
    nxt_dev = None
    for o, (nx, ny, nz) in enumerate(plan.octave_dims):
        levels = []
        if o == 0:
            with rec("convolution", o, 0):
                cur_dev = blur_device(src, plan.taps[0])
        else:
            cur_dev = nxt_dev
        levels.append(DeviceVolume(cur_dev, spacing))
        prev = cur_dev
        for i in range(1, levels_per_octave):
            half = None
            if i == handoff and o + 1 < plan.n_octaves:
                half = nxt_dev = t.empty((nz // 2, ny // 2, nx // 2), dtype=t.float32, device="cuda")
            with rec("convolution", o, i):
                prev = blur_device(prev, plan.taps[i], half=half)
            levels.append(DeviceVolume(prev, spacing))
        octaves.append(PyramidOctave(levels, plan.sigmas[o]))
        spacing = tuple(2.0 * s for s in spacing)
    return GaussianPyramid(octaves, base_sigma, plan.kappa, levels_per_octave, source=v)


def build_dog_pyramid(g: GaussianPyramid, recorder=None) -> DoGPyramid:
    """scalespace.py:209-223 (finer minus coarser, per octave)."""
    if g.levels_per_octave < 2:
        raise ParameterError("pyramid needs at least 2 levels per octave")
    rec = _stage(recorder)
    t = _lib.torch()
    octaves = []
    for o, oc in enumerate(g.octaves):
        devs = [device_of(lv) for lv in oc.levels]
        diffs = []
        for i in range(len(devs) - 1):
            out = t.empty_like(devs[i])
            with rec("dog", o, i):
                _lib.call("vk_difference", devs[i].data_ptr(), devs[i + 1].data_ptr(), out.data_ptr(), out.numel(),
                          _lib.stream_ptr())
            diffs.append(DeviceVolume(out, oc.levels[i].spacing))
        octaves.append(DoGOctave(diffs, list(oc.sigmas[:-1])))
    return DoGPyramid(octaves, g.kappa, g.levels_per_octave)


_incremental_sigma = incremental_sigma  # scalespace.py:154-155


def dump_pyramid(g: GaussianPyramid, directory) -> list[str]:
    """scalespace.py:226-235: every level as ``oct{o}_lvl{i}_sigma{s:.4g}.f32``
    (+ header sidecar); device levels are written straight from their
    x-fastest layout.  Returns the data paths."""
    import os

    from .ingest import save_raw

    os.makedirs(directory, exist_ok=True)
    written = []
    for o, oc in enumerate(g.octaves):
        for i, (lv, sigma) in enumerate(zip(oc.levels, oc.sigmas)):
            path, _ = save_raw(lv, os.path.join(str(directory), f"oct{o}_lvl{i}_sigma{sigma:.4g}"))
            written.append(path)
    return written
