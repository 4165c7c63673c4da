"""Keypoint / descriptor text files -- drop-in for volkey keyfiles.py
(SURVEY.md §8(f) "next" #3), same formats byte for byte:

* ``# volkey keypoints v1``: ``x y z sigma octave level dog_value sign`` per
  keypoint, optionally followed by the 9 row-major reals of its frame;
* ``# volkey descriptors v1 kind=<k> n=<n> seed=<s>``: keypoint fields, frame,
  then 64 / n decimal ranks (siftrank / rrief) or the hex-packed bits (brief);
* inlier CSV ``idx_a,idx_b,distance``.

The lines are produced by the library's native formatter
(``vk_format_records``, C ``%.9g`` == CPython ``%.9g``: both correctly
rounded) from flat arrays, so writing the output of a batch never builds
per-record Python objects (``write_soa`` takes the structure-of-arrays of
``Extractor.results()`` directly).  Readers parse with numpy.
"""

from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _lib
from .descriptor import BriefDescriptor, DescriptorRecord, RriefDescriptor, SiftRankDescriptor
from .detect import Keypoint
from .errors import FormatError, InputOutputError
from .orient import OrientationFrame

KEYPOINT_HEADER = "# volkey keypoints v1"
DESCRIPTOR_HEADER = "# volkey descriptors v1"


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def format_lines(pos, sigma, octave, level, dog, sign, rot=None, payload=None, payload_kind: int = 0) -> bytes:
    """Text lines for n records from flat arrays (native formatter)."""
    n = len(sigma)
    pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(n, 3)
    sigma = np.ascontiguousarray(sigma, dtype=np.float64)
    octave = np.ascontiguousarray(octave, dtype=np.int32)
    level = np.ascontiguousarray(level, dtype=np.int32)
    dog = np.ascontiguousarray(dog, dtype=np.float64)
    sign = np.ascontiguousarray(sign, dtype=np.int8)
    rot = None if rot is None else np.ascontiguousarray(rot, dtype=np.float64).reshape(n, 9)
    plen = 0
    if payload is not None:
        payload = np.ascontiguousarray(payload, dtype=np.uint8).reshape(n, -1)
        plen = payload.shape[1]
    lib = _lib.load()
    args = (n, _ptr(pos), _ptr(sigma), _ptr(octave), _ptr(level), _ptr(dog), _ptr(sign), _ptr(rot), _ptr(payload),
            payload_kind if payload is not None else 0, plen)
    cap = max(1024, n * (160 + (150 if rot is not None else 0) + 4 * plen))
    while True:
        buf = C.create_string_buffer(cap)
        need = lib.vk_format_records(*args, buf, cap)
        if need < 0:
            raise FormatError(f"vk_format_records: {_lib.last_error()}")
        if need <= cap:
            return buf.raw[:need]
        cap = need


def _keypoint_arrays(kps):
    return dict(pos=np.array([k.position for k in kps], dtype=np.float64).reshape(-1, 3),
                sigma=np.array([k.sigma for k in kps], dtype=np.float64),
                octave=np.array([k.octave for k in kps], dtype=np.int32),
                level=np.array([k.level for k in kps], dtype=np.int32),
                dog=np.array([k.dog_value for k in kps], dtype=np.float64),
                sign=np.array([1 if k.sign == "peak" else -1 for k in kps], dtype=np.int8))


def _write(path, header: str, body: bytes) -> None:
    try:
        with open(path, "wb") as fh:
            fh.write(header.encode() + b"\n" + body)
    except OSError as exc:
        raise InputOutputError(f"cannot write {path}: {exc}") from exc


def _lines(path):
    try:
        with open(path) as fh:
            return fh.read().splitlines()
    except OSError as exc:
        raise InputOutputError(f"cannot read {path}: {exc}") from exc


# ----------------------------------------------------------------- keypoints
def write_keypoints(path, keypoints: Sequence[Keypoint] | None = None,
                    oriented: Sequence[tuple[Keypoint, OrientationFrame]] | None = None) -> None:
    """keyfiles.py:60-76: bare keypoints, or one line per (keypoint, frame)."""
    if oriented is not None:
        kps = [k for k, _ in oriented]
        rot = np.array([np.asarray(f.rotation, dtype=np.float64).reshape(9) for _, f in oriented]).reshape(-1, 9)
        body = format_lines(**_keypoint_arrays(kps), rot=rot)
    else:
        body = format_lines(**_keypoint_arrays(list(keypoints or [])))
    _write(path, KEYPOINT_HEADER, body)


def _parse_kp(p) -> Keypoint:
    if p[7] not in ("peak", "valley"):
        raise FormatError(f"bad keypoint sign {p[7]!r}")
    return Keypoint((float(p[0]), float(p[1]), float(p[2])), float(p[3]), int(p[4]), int(p[5]), float(p[6]), p[7])


def read_keypoints(path) -> list[tuple[Keypoint, OrientationFrame | None]]:
    """keyfiles.py:79-97."""
    lines = _lines(path)
    if not lines or lines[0].strip() != KEYPOINT_HEADER:
        raise FormatError(f"{path}: missing header {KEYPOINT_HEADER!r}")
    out = []
    for i, line in enumerate(lines[1:], 2):
        p = line.split()
        if not p:
            continue
        if len(p) == 8:
            out.append((_parse_kp(p), None))
        elif len(p) == 17:
            out.append((_parse_kp(p[:8]), OrientationFrame(np.array([float(v) for v in p[8:]]).reshape(3, 3))))
        else:
            raise FormatError(f"{path}:{i}: expected 8 or 17 fields, got {len(p)}")
    return out


# --------------------------------------------------------------- descriptors
def write_descriptors(path, records: Sequence[DescriptorRecord], kind: str, n: int, seed: int) -> None:
    """keyfiles.py:107-122."""
    kps = [r.keypoint for r in records]
    rot = np.array([np.asarray(r.frame.rotation, dtype=np.float64).reshape(9) for r in records]).reshape(-1, 9)
    if kind == "brief":
        payload = np.packbits(np.array([r.descriptor.bits for r in records], dtype=np.uint8).reshape(len(records), -1),
                              axis=1, bitorder="big")
        pk = 2
    else:
        payload = np.array([r.descriptor.ranks for r in records], dtype=np.int64).reshape(len(records), -1)
        if payload.size and (payload.min() < 0 or payload.max() > 255):
            raise FormatError("ranks outside 0..255 cannot use the byte payload path")
        pk = 1
    body = format_lines(**_keypoint_arrays(kps), rot=rot, payload=payload.astype(np.uint8), payload_kind=pk)
    _write(path, f"{DESCRIPTOR_HEADER} kind={kind} n={n} seed={seed}", body)


def write_soa(path, soa: dict, kind: str, n: int, seed: int, volume: int | None = None) -> int:
    """Descriptor file straight from ``Extractor.results()`` (structure of
    arrays, volume-major); ``volume`` selects one volume of a batch.  Returns
    the number of records written."""
    kp = soa["kp"]
    fk_all = np.asarray(soa["frame_kp"], dtype=np.int64)
    sel = np.arange(len(fk_all)) if volume is None else np.flatnonzero(kp["vol"][fk_all] == volume)
    fk = fk_all[sel]
    desc = np.asarray(soa["desc"])[sel]
    payload = desc[:, : (n + 7) // 8] if kind == "brief" else desc[:, :n]
    body = format_lines(soa["pos"][fk], soa["sigma"][fk], kp["octave"][fk], kp["level"][fk], soa["dog"][fk],
                        soa["sign"][fk], rot=np.asarray(soa["rot"])[sel].reshape(-1, 9), payload=payload,
                        payload_kind=2 if kind == "brief" else 1)
    _write(path, f"{DESCRIPTOR_HEADER} kind={kind} n={n} seed={seed}", body)
    return len(sel)


def read_descriptors(path) -> tuple[str, int, int, list[DescriptorRecord]]:
    """keyfiles.py:125-162 -> (kind, n, seed, records)."""
    lines = _lines(path)
    if not lines or not lines[0].startswith(DESCRIPTOR_HEADER):
        raise FormatError(f"{path}: missing header {DESCRIPTOR_HEADER!r}")
    meta = dict(t.split("=", 1) for t in lines[0][len(DESCRIPTOR_HEADER):].split() if "=" in t)
    try:
        kind, n, seed = meta["kind"], int(meta["n"]), int(meta["seed"])
    except (KeyError, ValueError) as exc:
        raise FormatError(f"{path}: malformed descriptor header") from exc
    if kind not in ("siftrank", "brief", "rrief"):
        raise FormatError(f"{path}: unknown descriptor kind {kind!r}")
    want = 18 if kind == "brief" else 17 + n
    recs = []
    for i, line in enumerate(lines[1:], 2):
        p = line.split()
        if not p:
            continue
        if len(p) != want:
            raise FormatError(f"{path}:{i}: expected {want} fields, got {len(p)}")
        frame = OrientationFrame(np.array([float(v) for v in p[8:17]]).reshape(3, 3))
        if kind == "brief":
            d = BriefDescriptor(np.unpackbits(np.frombuffer(bytes.fromhex(p[17]), dtype=np.uint8), bitorder="big")[:n])
        else:
            ranks = np.array([int(v) for v in p[17:]], dtype=np.int64)
            d = SiftRankDescriptor(ranks) if kind == "siftrank" else RriefDescriptor(ranks)
        recs.append(DescriptorRecord(_parse_kp(p[:8]), frame, d))
    return kind, n, seed, recs


def write_inlier_csv(path, inliers) -> None:
    """keyfiles.py:165-174."""
    body = "".join(f"{m.index_a},{m.index_b},{m.distance:.9g}\n" for m in inliers)
    try:
        with open(path, "w") as fh:
            fh.write("idx_a,idx_b,distance\n" + body)
    except OSError as exc:
        raise InputOutputError(f"cannot write {path}: {exc}") from exc
