"""Golden digests for the volumes the benchmark and the sharded configs use,
made by the REAL reference (run in the build container, where
``/root/reference`` exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_bench_golden.py

* ``bench.npz``: SIFT-Rank extraction (default PipelineConfig) of
  - the first 4 volumes bench.py rank 0 extracts
    (``synthetic.batch_from(brain_volume(), n, seed=1000)``, bench.py run_ours);
  - SURVEY §8(d) C3 volumes, seeds 0..3 (``soup_params`` + N(0, 0.01) with
    ``default_rng(seed)``, /root/reference/pkg/tests/phantoms.py:97-103 as
    restated by ``synthetic.brain_volume(seed)``);
  stored as per-volume sha256 digests (tests/golden/digest.py) + counts.
* ``zeroback.npz``: full results (all three descriptor kinds) of kernel-soup
  phantoms set to exactly 0 outside a sphere (skull-stripped-MRI-like), one of
  them scaled by 1e-22 so every gradient's fp32 sum of squares underflows --
  the inputs where a fast fp32 |g| could differ from the reference's fp64 one.

Inputs are regenerated from seeds on the GPU box and checked against the
input hashes stored here.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as MG  # noqa: E402  (puts the reference on sys.path)
from digest import digest  # noqa: E402

from volkey.config import PipelineConfig  # noqa: E402
from volkey.pipeline import extract_features  # noqa: E402

from paper_2112_10258_b200 import synthetic  # noqa: E402

BENCH_SEED = 1000   # bench.py: synthetic.batch_from(base, B * S, seed=1000 + rank)
C3_SEEDS = (0, 1, 2, 3)


def bench_volumes():
    base = synthetic.brain_volume()
    return synthetic.batch_from(base, 4, seed=BENCH_SEED)


def c3_volume(seed: int) -> np.ndarray:
    return synthetic.brain_volume(seed=seed)


def zeroback_volume(dims, seed, radius_frac=0.42, scale=1.0):
    return synthetic.zero_background_volume(dims, seed, radius_frac, scale)


ZEROBACK = [((80, 80, 80), 31, 1.0), ((96, 88, 90), 32, 1.0), ((64, 70, 60), 33, 1e-22)]


def ref_digest(vol: np.ndarray) -> dict:
    res = extract_features(MG.rvol.Volume(vol), PipelineConfig())
    kps = res.keypoints
    index = {id(k): i for i, k in enumerate(kps)}
    arr = MG.rdesc.descriptor_array(res.records, "siftrank")
    return digest([k.position for k in kps], [k.sigma for k in kps], [k.octave for k in kps],
                  [k.level for k in kps], [k.dog_value for k in kps],
                  [1 if k.sign == "peak" else -1 for k in kps],
                  [index[id(k)] for k, _ in res.oriented], [f.rotation for _, f in res.oriented], arr)


def main():
    t0 = time.time()
    out = {}
    vols = [("bench", i, v) for i, v in enumerate(bench_volumes())] + [("c3", s, c3_volume(s)) for s in C3_SEEDS]
    for tag, i, v in vols:
        d = ref_digest(v)
        for k, val in d.items():
            out[f"{tag}{i}_{k}"] = val
        out[f"{tag}{i}_input_sha"] = MG.sha(v)
        print(f"  {tag}{i}: {d['n_kp']} keypoints, {d['n_fr']} frames, {time.time() - t0:.0f}s", flush=True)
    np.savez_compressed(os.path.join(HERE, "bench.npz"), **out)

    zb = {}
    cfg = PipelineConfig()
    for j, (dims, seed, scale) in enumerate(ZEROBACK):
        v = zeroback_volume(dims, seed, scale=scale)
        case, _, _, _ = MG.full_case(v, cfg, with_hist=True)
        for k, val in case.items():
            zb[f"z{j}_{k}"] = val
        zb[f"z{j}_dims"], zb[f"z{j}_seed"], zb[f"z{j}_scale"] = np.array(dims), seed, scale
    np.savez_compressed(os.path.join(HERE, "zeroback.npz"), **zb)
    print(f"done {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
