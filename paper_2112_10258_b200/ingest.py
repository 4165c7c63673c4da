"""Volume ingest -- drop-in for volkey volume.py:73-200 (``load_raw``,
``save_raw``, ``read_raw_header``, ``load_nifti_subset``, ``load_volume``)
plus a batched reader for throughput runs (SURVEY.md §8(f) "next" #2).

Both on-disk formats store voxels x-fastest, which is exactly the device
layout of every kernel here, so a file goes disk -> pinned host buffer ->
HBM with no host-side transpose (the reference transposes every volume to
``data[x, y, z]`` on the host).  Loaders return a ``DeviceVolume``; its
``.data`` (the reference's ``[x, y, z]`` array) is produced lazily on the
GPU.  Finiteness is checked on the device; errors are the reference's:
``InputOutputError`` (unreadable), ``FormatError`` (size / header),
``DataError`` (non-finite voxels).

``RawBatchReader`` fills a (B, nz, ny, nx) pinned buffer from B ``.f32``
files with a thread pool and copies it asynchronously into an Extractor's
input slot, so ingest of batch k+1 overlaps the extraction of batch k.
"""

from __future__ import annotations

import gzip
import os
import struct
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib
from .errors import DataError, FormatError, InputOutputError
from .volume import DeviceVolume, Volume

Dims = tuple[int, int, int]
Triple = tuple[float, float, float]


# ----------------------------------------------------------------- helpers
def _read_bytes(path) -> bytes:
    try:
        with open(path, "rb") as fh:
            return fh.read()
    except OSError as exc:
        raise InputOutputError(f"cannot read {path}: {exc}") from exc


def _device_from_xfast(flat: np.ndarray, dims: Dims, source: str):
    """x-fastest float32 voxels -> (nz, ny, nx) CUDA tensor, finiteness checked on the device."""
    t = _lib.torch()
    nx, ny, nz = dims
    host = t.from_numpy(np.ascontiguousarray(flat, dtype=np.float32).reshape(nz, ny, nx))
    dev = host.pin_memory().to("cuda", non_blocking=True)
    if not bool(t.isfinite(dev).all().item()):
        raise DataError(f"{source}: non-finite voxel values")
    return dev


# ------------------------------------------------------------------- .f32
def load_raw(path, dims: Dims, spacing: Triple = (1.0, 1.0, 1.0)) -> DeviceVolume:
    """volume.py:73-87: headerless little-endian float32, x fastest."""
    nx, ny, nz = (int(d) for d in dims)
    need = 4 * nx * ny * nz
    try:
        size = os.path.getsize(path)
    except OSError as exc:
        raise InputOutputError(f"cannot read {path}: {exc}") from exc
    if size != need:
        raise FormatError(f"{path}: file is {size} bytes, dims {tuple(dims)} require {need}")
    flat = np.frombuffer(_read_bytes(path), dtype="<f4")
    return DeviceVolume(_device_from_xfast(flat, (nx, ny, nz), str(path)), spacing)


def save_raw(volume: Volume, path) -> tuple[str, str]:
    """volume.py:90-105: ``<name>.f32`` (x fastest) + ``<name>.hdr.txt`` sidecar."""
    stem = str(path)
    if stem.endswith(".f32"):
        stem = stem[:-4]
    data_path, hdr_path = stem + ".f32", stem + ".hdr.txt"
    if isinstance(volume, DeviceVolume):
        xfast = volume.device.contiguous().cpu().numpy()          # already (nz, ny, nx)
    else:
        xfast = np.ascontiguousarray(np.asarray(volume.data, dtype=np.float32).transpose(2, 1, 0))
    nx, ny, nz = volume.dims
    try:
        with open(data_path, "wb") as fh:
            fh.write(xfast.astype("<f4", copy=False).tobytes())
        with open(hdr_path, "w") as fh:
            fh.write("dims: %d %d %d\n" % (nx, ny, nz))
            fh.write("spacing: %.9g %.9g %.9g\n" % tuple(volume.spacing))
    except OSError as exc:
        raise InputOutputError(f"cannot write {data_path}: {exc}") from exc
    return data_path, hdr_path


def read_raw_header(path) -> tuple[Dims, Triple]:
    """volume.py:108-130: ``dims: nx ny nz`` / ``spacing: sx sy sz`` sidecar."""
    try:
        with open(path) as fh:
            text = fh.read()
    except OSError as exc:
        raise InputOutputError(f"cannot read {path}: {exc}") from exc
    fields = {}
    for line in text.splitlines():
        key, sep, rest = line.partition(":")
        if sep:
            fields[key.strip()] = rest.split()
    try:
        dims = tuple(int(v) for v in fields["dims"])
        spacing = tuple(float(v) for v in fields["spacing"])
    except (KeyError, ValueError) as exc:
        raise FormatError(f"{path}: malformed raw header") from exc
    if len(dims) != 3 or len(spacing) != 3:
        raise FormatError(f"{path}: expected 3 dims and 3 spacing values")
    return dims, spacing


# ------------------------------------------------------------------ NIfTI
_NIFTI_TYPES = {2: np.uint8, 4: np.int16, 16: np.float32}


def load_nifti_subset(path) -> DeviceVolume:
    """volume.py:134-186: single-frame 3-D NIfTI-1 (uint8 / int16 / float32,
    optional gzip) honouring dim, datatype, pixdim, scl_slope / scl_inter and
    vox_offset.  The voxel conversion (cast, then slope / intercept in
    float32) runs on the device."""
    raw = _read_bytes(path)
    if raw[:2] == b"\x1f\x8b":
        raw = gzip.decompress(raw)
    if len(raw) < 352:
        raise FormatError(f"{path}: too short for a NIfTI-1 header")
    endian = next((e for e in "<>" if struct.unpack_from(e + "i", raw, 0)[0] == 348), None)
    if endian is None:
        raise FormatError(f"{path}: sizeof_hdr is not 348 in either byte order")
    magic = raw[344:348]
    if magic[:3] == b"ni1":
        raise FormatError(f"{path}: detached .hdr/.img NIfTI pairs are not supported")
    if magic[:3] != b"n+1":
        raise FormatError(f"{path}: bad NIfTI magic {magic!r}")
    dim = struct.unpack_from(endian + "8h", raw, 40)
    datatype = struct.unpack_from(endian + "h", raw, 70)[0]
    pixdim = struct.unpack_from(endian + "8f", raw, 76)
    vox_offset = struct.unpack_from(endian + "f", raw, 108)[0]
    slope, inter = struct.unpack_from(endian + "2f", raw, 112)
    ndim = dim[0]
    if ndim < 3 or any(d > 1 for d in dim[4: ndim + 1]):
        raise FormatError(f"{path}: expected a single 3D frame, got dim={dim[: ndim + 1]}")
    if datatype not in _NIFTI_TYPES:
        raise FormatError(f"{path}: unsupported NIfTI datatype code {datatype}")
    nx, ny, nz = (max(int(d), 1) for d in dim[1:4])
    dtype = np.dtype(_NIFTI_TYPES[datatype]).newbyteorder(endian)
    count, offset = nx * ny * nz, int(vox_offset)
    if offset < 348 or len(raw) < offset + count * dtype.itemsize:
        raise FormatError(f"{path}: data section truncated")
    t = _lib.torch()
    native = np.frombuffer(raw, dtype=dtype, count=count, offset=offset).astype(dtype.newbyteorder("="))
    dev = t.from_numpy(native.reshape(nz, ny, nx)).pin_memory().to("cuda", non_blocking=True).to(t.float32)
    if slope != 0.0 and (slope != 1.0 or inter != 0.0):
        dev = dev * slope + inter          # float32 product, then float32 sum (two roundings, as numpy)
    if not bool(t.isfinite(dev).all().item()):
        raise DataError(f"{path}: non-finite voxel values")
    spacing = tuple(float(p) if p > 0 else 1.0 for p in pixdim[1:4])
    return DeviceVolume(dev.contiguous(), spacing)


def load_volume(path, dims: Dims | None = None, spacing: Triple | None = None) -> DeviceVolume:
    """volume.py:189-200: dispatch on ``.nii`` / ``.nii.gz`` / ``.f32`` (+ sidecar)."""
    name = str(path)
    if name.endswith((".nii", ".nii.gz")):
        return load_nifti_subset(path)
    if name.endswith(".f32"):
        if dims is None:
            dims, hdr_spacing = read_raw_header(name[:-4] + ".hdr.txt")
            spacing = spacing or hdr_spacing
        return load_raw(path, dims, spacing or (1.0, 1.0, 1.0))
    raise FormatError(f"{name}: unrecognized volume format (expected .f32, .nii or .nii.gz)")


# ------------------------------------------------------------ batch reader
class RawBatchReader:
    """Read batches of B same-size ``.f32`` volumes into a pinned
    (B, nz, ny, nx) host buffer (thread pool, ``readinto`` straight into the
    pinned pages) and copy them into a device tensor on a side stream.

        reader = RawBatchReader(dims, B)
        reader.submit(paths_0)                      # starts reading batch 0
        for k in range(n):
            ev = reader.to_device(ex.input)         # H2D of batch k (async)
            if k + 1 < n: reader.submit(paths_k1)   # disk reads of batch k+1 overlap ...
            torch.cuda.current_stream().wait_event(ev)
            ex.run()                                # ... the extraction of batch k
    """

    def __init__(self, dims: Dims, batch: int, workers: int = 8):
        t = _lib.torch()
        self.dims = tuple(int(d) for d in dims)
        nx, ny, nz = self.dims
        self.B = int(batch)
        self.bytes = 4 * nx * ny * nz
        self.host = [t.empty((self.B, nz, ny, nx), dtype=t.float32).pin_memory() for _ in range(2)]
        self.pool = ThreadPoolExecutor(max_workers=workers)
        self.stream = t.cuda.Stream()
        self.copied = [t.cuda.Event(), t.cuda.Event()]
        self.pending = None
        self.slot = 0
        self.paths = None

    def _read_one(self, path, view: memoryview) -> None:
        try:
            size = os.path.getsize(path)
        except OSError as exc:
            raise InputOutputError(f"cannot read {path}: {exc}") from exc
        if size != self.bytes:
            raise FormatError(f"{path}: file is {size} bytes, dims {self.dims} require {self.bytes}")
        try:
            with open(path, "rb", buffering=0) as fh:
                got = fh.readinto(view)
        except OSError as exc:
            raise InputOutputError(f"cannot read {path}: {exc}") from exc
        if got != self.bytes:
            raise InputOutputError(f"{path}: short read")

    def submit(self, paths) -> None:
        """Start reading up to B files into the next pinned slot."""
        if len(paths) > self.B:
            raise FormatError(f"batch holds {self.B} volumes, got {len(paths)} paths")
        slot = self.slot
        self.copied[slot].synchronize()     # the previous H2D out of this slot is done
        buf = self.host[slot].numpy().reshape(self.B, -1).view(np.uint8)
        self.pending = [self.pool.submit(self._read_one, p, memoryview(buf[i])) for i, p in enumerate(paths)]
        self.paths = list(paths)

    def to_device(self, dst):
        """Wait for the submitted reads, copy the slot into `dst` (B, nz, ny, nx)
        on the side stream, check finiteness there; returns the event that
        marks the copy (make the compute stream wait on it)."""
        t = _lib.torch()
        for f in self.pending or []:
            f.result()
        slot, n = self.slot, len(self.paths or [])
        with t.cuda.stream(self.stream):
            self.stream.wait_stream(t.cuda.current_stream())
            dst[:n].copy_(self.host[slot][:n], non_blocking=True)
            bad = (~t.isfinite(dst[:n])).flatten(1).any(dim=1)
            self.copied[slot].record(self.stream)
        bad = bad.cpu()  # one small D2H per batch (waits for this batch's copy only)
        if bool(bad.any()):
            raise DataError(f"{self.paths[int(bad.nonzero()[0])]}: non-finite voxel values")
        self.slot ^= 1
        return self.copied[slot]
