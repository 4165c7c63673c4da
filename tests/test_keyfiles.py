"""CPU: key / descriptor text files are byte-identical to the reference
writers' (tests/golden/keyfiles.npz, made by tests/golden/make_keyfile_golden.py)
and read back losslessly."""

import hashlib

import numpy as np
import pytest

from conftest import load_golden
from paper_2112_10258_b200 import keyfiles as kf
from paper_2112_10258_b200.descriptor import BriefDescriptor, DescriptorRecord, RriefDescriptor, SiftRankDescriptor
from paper_2112_10258_b200.match import Match
from test_consensus import _pairs


def _sha(p):
    return hashlib.sha256(open(p, "rb").read()).hexdigest()


def test_keypoint_files_match_reference(tmp_path):
    g, h = load_golden("pair.npz"), load_golden("keyfiles.npz")
    pairs = _pairs(g, "a_")
    kps, seen = [], set()
    for k, _ in pairs:
        if id(k) not in seen:
            seen.add(id(k))
            kps.append(k)
    p = tmp_path / "k.txt"
    kf.write_keypoints(p, keypoints=kps)
    assert _sha(p) == str(h["keypoints_sha"])
    kf.write_keypoints(p, oriented=pairs)
    assert _sha(p) == str(h["oriented_sha"])
    back = kf.read_keypoints(p)
    assert len(back) == len(pairs)
    # %.9g text is lossy by design (keyfiles.py:35-40): values agree to 9 significant digits
    assert all(np.allclose(k2.position, k.position, rtol=1e-8) and np.isclose(k2.sigma, k.sigma, rtol=1e-8) and
               np.allclose(f2.rotation, f.rotation, rtol=1e-8, atol=1e-9) and k2.sign == k.sign
               for (k, f), (k2, f2) in zip(pairs, back))


@pytest.mark.parametrize("kind", ["siftrank", "brief", "rrief"])
def test_descriptor_files_match_reference(tmp_path, kind):
    g, h = load_golden("pair.npz"), load_golden("keyfiles.npz")
    pairs = _pairs(g, "a_")
    arr = g[f"a_desc_{kind}"]
    recs = []
    for (k, f), row in zip(pairs, arr):
        d = (BriefDescriptor(np.unpackbits(row, bitorder="big")[:64]) if kind == "brief" else
             SiftRankDescriptor(row.astype(np.int64)) if kind == "siftrank" else RriefDescriptor(row.astype(np.int64)))
        recs.append(DescriptorRecord(k, f, d))
    p = tmp_path / "d.txt"
    kf.write_descriptors(p, recs, kind, 64, 13)
    assert _sha(p) == str(h[f"desc_{kind}_sha"])
    k2, n2, s2, back = kf.read_descriptors(p)
    assert (k2, n2, s2, len(back)) == (kind, 64, 13, len(recs))
    field = "bits" if kind == "brief" else "ranks"
    assert all(np.array_equal(getattr(a.descriptor, field), getattr(b.descriptor, field)) for a, b in zip(recs, back))


def test_inlier_csv_matches_reference(tmp_path):
    g, h = load_golden("pair.npz"), load_golden("keyfiles.npz")
    p = tmp_path / "i.csv"
    kf.write_inlier_csv(p, [Match(int(r[0]), int(r[1]), float(r[2]), float(r[3])) for r in g["nn_siftrank"]])
    assert _sha(p) == str(h["inlier_csv_sha"])
