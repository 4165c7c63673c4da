"""Golden vectors for the 7-DOF Hough consensus (match.py:124-359), from the
REAL reference.  Run in the build container (``/root/reference`` present):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_hough_golden.py

Inputs are the reference's own outputs already pinned in ``pair.npz``
(keypoints, frame rotations, nearest-neighbour matches of the configs[1]
volume pair for all three descriptor kinds); they are turned back into the
reference's ``Keypoint`` / ``OrientationFrame`` / ``Match`` objects and
``volkey.match.hough_consensus`` is called unmodified.  Stores, per kind, the
inlier match indices, the cell vote count, the consensus transform and the
reference's wall time.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from volkey import match as rmatch  # noqa: E402
from volkey.detect import Keypoint  # noqa: E402
from volkey.orient import OrientationFrame  # noqa: E402


def pairs_from(g, p):
    kps = [Keypoint(tuple(float(c) for c in pos), float(s), int(o), int(l), float(d), "peak" if sg > 0 else "valley")
           for pos, s, o, l, d, sg in zip(g[p + "kp_pos"], g[p + "kp_sigma"], g[p + "kp_octave"], g[p + "kp_level"],
                                          g[p + "kp_dog"], g[p + "kp_sign"])]
    return [(kps[int(k)], OrientationFrame(np.array(r))) for k, r in zip(g[p + "fr_kp"], g[p + "fr_rot"])]


def main():
    g = np.load(os.path.join(HERE, "pair.npz"))
    pa, pb = pairs_from(g, "a_"), pairs_from(g, "b_")
    out = {}
    for kind in ("siftrank", "brief", "rrief"):
        nn = g[f"nn_{kind}"]
        matches = [rmatch.Match(int(r[0]), int(r[1]), float(r[2]), float(r[3])) for r in nn]
        t0 = time.time()
        res = rmatch.hough_consensus(matches, pa, pb, rmatch.HoughSettings())
        dt = time.time() - t0
        pos = {(m.index_a, m.index_b, m.distance, m.second_distance): i for i, m in enumerate(matches)}
        inl = np.array([pos[(m.index_a, m.index_b, m.distance, m.second_distance)] for m in res.inliers], np.int32)
        out[f"{kind}_inliers"] = inl
        out[f"{kind}_cell_votes"] = np.int64(res.cell_votes)
        out[f"{kind}_scale"] = np.float64(res.transform.scale)
        out[f"{kind}_rotation"] = np.asarray(res.transform.rotation)
        out[f"{kind}_translation"] = np.asarray(res.transform.translation)
        out[f"{kind}_ref_seconds"] = np.float64(dt)
        print(kind, len(matches), "matches ->", len(inl), "inliers, cell", res.cell_votes, f"{dt:.3f} s", flush=True)
    np.savez_compressed(os.path.join(HERE, "hough.npz"), **out)


if __name__ == "__main__":
    main()
