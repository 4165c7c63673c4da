"""Dense 3-D volumes at the drop-in boundary (volkey volume.py:23-46).

``Volume`` keeps the reference's contract: float32, C-contiguous, read-only
``data[x, y, z]`` (z fastest), ``spacing`` metadata.  ``DeviceVolume`` is the
same type backed by an x-fastest CUDA tensor (the layout every kernel uses);
its ``.data`` is materialised lazily, so pyramids returned by the GPU path cost
nothing until a caller actually looks at a level.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import FormatError

Triple = tuple[float, float, float]


@dataclass(frozen=True)
class Volume:
    data: np.ndarray
    spacing: Triple = (1.0, 1.0, 1.0)

    def __post_init__(self) -> None:
        arr = np.asarray(self.data, dtype=np.float32)
        if arr.ndim != 3:
            raise FormatError(f"volume data must be 3D, got {arr.ndim}D")
        if min(arr.shape) < 1:
            raise FormatError(f"all dims must be >= 1, got {arr.shape}")
        sp = tuple(float(s) for s in self.spacing)
        if len(sp) != 3 or min(sp) <= 0:
            raise FormatError(f"spacing components must be > 0, got {self.spacing}")
        arr = np.ascontiguousarray(arr)
        arr.setflags(write=False)
        object.__setattr__(self, "data", arr)
        object.__setattr__(self, "spacing", sp)

    @property
    def dims(self):
        return self.data.shape


class DeviceVolume(Volume):
    """A Volume whose voxels live in HBM as an x-fastest (nz, ny, nx) tensor."""

    def __init__(self, dev, spacing: Triple = (1.0, 1.0, 1.0)):  # noqa: D107 (frozen: set via object)
        object.__setattr__(self, "_dev", dev)
        object.__setattr__(self, "_host", None)
        object.__setattr__(self, "spacing", tuple(float(s) for s in spacing))

    @property
    def device(self):
        return self._dev

    @property
    def dims(self):
        nz, ny, nx = self._dev.shape
        return (int(nx), int(ny), int(nz))

    @property
    def data(self) -> np.ndarray:  # type: ignore[override]
        if self._host is None:
            object.__setattr__(self, "_host", to_host(self._dev))
        return self._host

    def __repr__(self) -> str:
        return f"DeviceVolume(dims={self.dims}, spacing={self.spacing})"


def to_device(arr: np.ndarray, stream=None):
    """numpy data[x, y, z] -> CUDA tensor (nz, ny, nx), x fastest (vk_transpose)."""
    t = _lib.torch()
    a = np.ascontiguousarray(arr, dtype=np.float32)
    if not a.flags.writeable:
        a = a.copy()
    nx, ny, nz = a.shape
    src = t.from_numpy(a).to("cuda", non_blocking=False)
    dst = t.empty((nz, ny, nx), dtype=t.float32, device="cuda")
    _lib.call("vk_transpose_zfast_to_xfast", _lib.ptr(src), _lib.ptr(dst), 1, nx, ny, nz, _lib.stream_ptr(stream))
    return dst


def to_host(dev, stream=None) -> np.ndarray:
    """CUDA tensor (..., nz, ny, nx) x fastest -> numpy (..., nx, ny, nz) z fastest."""
    t = _lib.torch()
    shape = tuple(dev.shape)
    nz, ny, nx = shape[-3:]
    nb = int(np.prod(shape[:-3])) if len(shape) > 3 else 1
    out = t.empty(shape[:-3] + (nx, ny, nz), dtype=t.float32, device="cuda")
    _lib.call("vk_transpose_xfast_to_zfast", _lib.ptr(dev.contiguous()), _lib.ptr(out), nb, nx, ny, nz,
              _lib.stream_ptr(stream))
    host = out.cpu().numpy()
    host.setflags(write=False)
    return host


def device_of(v: Volume):
    """x-fastest device tensor for any Volume (uploads host volumes)."""
    if isinstance(v, DeviceVolume):
        return v.device
    return to_device(v.data)


@dataclass(frozen=True)
class VoxelIndex:
    """volume.py:49-56."""

    x: int
    y: int
    z: int

    def within(self, dims) -> bool:
        return 0 <= self.x < dims[0] and 0 <= self.y < dims[1] and 0 <= self.z < dims[2]


def _dev_data(data):
    """x-fastest device tensor for a numpy data[x, y, z] array or a Volume."""
    if isinstance(data, Volume):
        return device_of(data), data.dims
    a = np.asarray(data, dtype=np.float32)
    return to_device(a), a.shape


def gradients_at(data, indices) -> np.ndarray:
    """volume.py:244-264 on the GPU: fp64 central differences in the interior,
    one-sided at borders, at integer voxel indices (N, 3) -> (N, 3)."""
    t = _lib.torch()
    dev, (nx, ny, nz) = _dev_data(data)
    idx = np.ascontiguousarray(np.atleast_2d(np.asarray(indices, dtype=np.int64)))
    n = len(idx)
    if n and (idx.shape[1] != 3 or (idx < 0).any() or (idx >= np.array([nx, ny, nz])).any()):
        raise IndexError("gradients_at: voxel index outside the volume")
    d_idx = t.from_numpy(idx).cuda()
    out = t.empty((max(n, 1), 3), dtype=t.float64, device="cuda")
    _lib.call("vk_gradients_at", _lib.ptr(dev), nx, ny, nz, d_idx.data_ptr(), n, out.data_ptr(), _lib.stream_ptr())
    return out[:n].cpu().numpy()


def central_gradient(volume: Volume, idx: VoxelIndex) -> np.ndarray:
    """volume.py:267-269: gradient at one voxel."""
    return gradients_at(volume, np.array([[idx.x, idx.y, idx.z]]))[0]


def sample_trilinear_array(data, points) -> np.ndarray:
    """volume.py:203-236 on the GPU: clamped trilinear interpolation in fp64 at
    continuous points (N, 3) or (3,), index units."""
    t = _lib.torch()
    dev, (nx, ny, nz) = _dev_data(data)
    pts = np.asarray(points, dtype=np.float64)
    single = pts.ndim == 1
    pts = np.ascontiguousarray(np.atleast_2d(pts))
    n = len(pts)
    d_pts = t.from_numpy(pts).cuda()
    out = t.empty(max(n, 1), dtype=t.float64, device="cuda")
    _lib.call("vk_sample_trilinear", _lib.ptr(dev), nx, ny, nz, d_pts.data_ptr(), n, out.data_ptr(), _lib.stream_ptr())
    res = out[:n].cpu().numpy()
    return res[0] if single else res


def trilinear_sample(volume: Volume, point) -> float:
    """volume.py:239-241."""
    return float(sample_trilinear_array(volume, np.asarray(point, dtype=np.float64)))


_INGEST = ("load_raw", "save_raw", "read_raw_header", "load_nifti_subset", "load_volume")


def __getattr__(name):
    """volkey.volume also holds the loaders (volume.py:73-200): re-export them
    lazily from ingest.py (which imports this module)."""
    if name in _INGEST:
        from . import ingest

        return getattr(ingest, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
