"""Golden key / descriptor files from the REAL reference writers (keyfiles.py)
on the configs[1] volume-A records pinned in pair.npz: their sha256 and sizes.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_keyfile_golden.py
"""

from __future__ import annotations

import hashlib
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)
from make_hough_golden import pairs_from  # noqa: E402
from volkey import descriptor as rdesc  # noqa: E402
from volkey import keyfiles as rkf  # noqa: E402
from volkey import match as rmatch  # noqa: E402


def sha_file(p):
    with open(p, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def main():
    g = np.load(os.path.join(HERE, "pair.npz"))
    pairs = pairs_from(g, "a_")
    out = {}
    with tempfile.TemporaryDirectory() as td:
        kps = []
        seen = set()
        for k, _ in pairs:
            if id(k) not in seen:
                seen.add(id(k))
                kps.append(k)
        p = os.path.join(td, "k.txt")
        rkf.write_keypoints(p, keypoints=kps)
        out["keypoints_sha"] = sha_file(p)
        rkf.write_keypoints(p, oriented=pairs)
        out["oriented_sha"] = sha_file(p)
        for kind in ("siftrank", "brief", "rrief"):
            arr = g[f"a_desc_{kind}"]
            recs = []
            for (k, f), row in zip(pairs, arr):
                if kind == "brief":
                    d = rdesc.BriefDescriptor(np.unpackbits(row, bitorder="big")[:64])
                elif kind == "siftrank":
                    d = rdesc.SiftRankDescriptor(row.astype(np.int64))
                else:
                    d = rdesc.RriefDescriptor(row.astype(np.int64))
                recs.append(rdesc.DescriptorRecord(k, f, d))
            rkf.write_descriptors(p, recs, kind, 64, 13)
            out[f"desc_{kind}_sha"] = sha_file(p)
        nn = g["nn_siftrank"]
        rkf.write_inlier_csv(p, [rmatch.Match(int(r[0]), int(r[1]), float(r[2]), float(r[3])) for r in nn])
        out["inlier_csv_sha"] = sha_file(p)
    np.savez_compressed(os.path.join(HERE, "keyfiles.npz"), **{k: np.array(v) for k, v in out.items()})
    print(out)


if __name__ == "__main__":
    main()
