"""Golden vectors for volume ingest (volume.py:73-200) from the REAL reference:
small .f32 / NIfTI-1 files (uint8, int16 with scl_slope/scl_inter, big-endian
float32, gzip) written here, and the arrays the reference loaders return.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_ingest_golden.py
"""

from __future__ import annotations

import gzip
import os
import struct
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
from volkey import volume as rvol  # noqa: E402


def nifti_bytes(data_xfast: np.ndarray, dims, dtype_code, endian="<", slope=0.0, inter=0.0, pixdim=(1.0, 1.0, 1.0)):
    hdr = bytearray(352)
    struct.pack_into(endian + "i", hdr, 0, 348)
    struct.pack_into(endian + "8h", hdr, 40, 3, *dims, 1, 1, 1, 1)
    bitpix = {2: 8, 4: 16, 16: 32}[dtype_code]
    struct.pack_into(endian + "2h", hdr, 70, dtype_code, bitpix)
    struct.pack_into(endian + "8f", hdr, 76, 1.0, *pixdim, 0, 0, 0, 0)
    struct.pack_into(endian + "f", hdr, 108, 352.0)
    struct.pack_into(endian + "2f", hdr, 112, slope, inter)
    hdr[344:348] = b"n+1\0"
    return bytes(hdr) + data_xfast.tobytes()


def main():
    rng = np.random.default_rng(31)
    dims = (10, 9, 8)
    n = int(np.prod(dims))
    out = {"dims": np.array(dims)}
    cases = {
        "f32": rng.standard_normal(n).astype("<f4").tobytes(),
        "u8": nifti_bytes(rng.integers(0, 256, n).astype(np.uint8), dims, 2, pixdim=(0.9, 1.1, 1.25)),
        "i16": nifti_bytes(rng.integers(-3000, 3000, n).astype("<i2"), dims, 4, slope=0.37, inter=-12.5),
        "f32be": nifti_bytes(rng.standard_normal(n).astype(">f4"), dims, 16, endian=">"),
        "i16gz": gzip.compress(nifti_bytes(rng.integers(-300, 300, n).astype("<i2"), dims, 4, slope=2.0, inter=1.0)),
    }
    with tempfile.TemporaryDirectory() as td:
        for name, blob in cases.items():
            out[f"{name}_bytes"] = np.frombuffer(blob, dtype=np.uint8)
            path = os.path.join(td, name + (".f32" if name == "f32" else ".nii.gz" if name.endswith("gz") else ".nii"))
            with open(path, "wb") as fh:
                fh.write(blob)
            v = rvol.load_raw(path, dims) if name == "f32" else rvol.load_nifti_subset(path)
            out[f"{name}_data"] = v.data
            out[f"{name}_spacing"] = np.array(v.spacing)
    np.savez_compressed(os.path.join(HERE, "ingest.npz"), **out)
    print("ok", list(cases))


if __name__ == "__main__":
    main()
