"""configs[3] golden hashes from the REAL reference: 256^3 soup volume (seed
20240817, N(0, 0.01) noise), num_octaves=4, SIFT-Rank.  Run in the build
container (``/root/reference`` present):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_large_golden.py

The arrays are large, so only their sha256 (and counts) are stored; the GPU
test recomputes the same hashes from its own outputs.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)
sys.path.insert(0, REPO)

from make_golden import full_case, sha  # noqa: E402
from volkey.config import PipelineConfig  # noqa: E402

from paper_2112_10258_b200 import synthetic  # noqa: E402


def main():
    dims = (256, 256, 256)
    vol = synthetic.soup_volume(dims, np.random.default_rng(synthetic.BRAIN_SEED), noise=0.01)
    cfg = PipelineConfig(num_octaves=4)
    t0 = time.time()
    out, _, kps, oriented = full_case(vol, cfg)
    dt = time.time() - t0
    keep = {k: out[k] for k in ("input_sha", "pyr_dims", "pyr_sha", "dog_sha", "dropped_orientation")}
    for k in ("kp_pos", "kp_sigma", "kp_octave", "kp_level", "kp_dog", "kp_sign", "fr_kp", "fr_rot",
              "desc_siftrank", "desc_brief", "desc_rrief"):
        keep[k + "_sha"] = sha(out[k])
        keep[k + "_len"] = np.int64(len(out[k]))
    keep["ref_seconds"] = np.float64(dt)
    np.savez_compressed(os.path.join(HERE, "large256.npz"), **keep)
    print(f"{len(kps)} keypoints, {len(oriented)} frames, {dt:.1f} s")


if __name__ == "__main__":
    main()
