"""Per-volume digests of an extraction, shared by the golden generator
(``make_bench_golden.py``, run on the unmodified reference) and the GPU tests
(run on ``Extractor.results()``).  One sha256 over the keypoint fields, one
over the frames, one over the descriptors -- so full-size (145x174x145)
volumes can be pinned without shipping megabytes of fixtures."""

from __future__ import annotations

import hashlib

import numpy as np


def _h(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def digest(pos, sigma, octave, level, dog, sign, fr_kp, rot, desc) -> dict:
    """pos (n,3) f64, sigma/dog (n,) f64, octave/level (n,) int, sign (n,) +-1,
    fr_kp (m,) keypoint index within the volume, rot (m,3,3) f64, desc (m,k)."""
    n = len(sigma)
    return dict(
        n_kp=n,
        n_fr=len(fr_kp),
        kp=_h(np.asarray(pos, np.float64).reshape(n, 3), np.asarray(sigma, np.float64),
              np.asarray(octave, np.int32), np.asarray(level, np.int32), np.asarray(dog, np.float64),
              np.asarray(sign, np.int8)),
        fr=_h(np.asarray(fr_kp, np.int32), np.asarray(rot, np.float64).reshape(-1, 3, 3)),
        desc=_h(np.asarray(desc, np.int64)),
    )


def digest_results(r: dict, v: int) -> dict:
    """Digest of volume v of an ``Extractor.results()`` dict."""
    off = r["vol_offset"]  # first keypoint of each volume
    a = int(off[v])
    b = int(off[v + 1]) if v + 1 < len(off) else int(r["n_keypoints"])
    kp = r["kp"][a:b]
    sel = (r["frame_kp"] >= a) & (r["frame_kp"] < b)
    return digest(r["pos"][a:b], r["sigma"][a:b], kp["octave"], kp["level"], r["dog"][a:b],
                  np.where(r["sign"][a:b] > 0, 1, -1), r["frame_kp"][sel] - a, r["rot"][sel], r["desc"][sel])
