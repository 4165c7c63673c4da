"""Generate the golden vectors in this directory from the REAL reference.

Run in the build container (where ``/root/reference`` exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the unmodified reference package (``/root/reference/pkg/src``) and
the reference's own phantom generators (``/root/reference/pkg/tests/
phantoms.py``), runs the hot path on seeded inputs and stores the results as
compressed ``.npz`` fixtures.  Inputs are NOT stored: they are regenerated on
any box by ``paper_2112_10258_b200.synthetic`` (the restated generators) and
checked against the sha256 recorded here.  The GPU box never runs this
script; it only reads the ``.npz`` files.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
sys.path.insert(0, REPO)

import phantoms as ref_phantoms  # noqa: E402  (reference test generators)
from volkey import descriptor as rdesc  # noqa: E402
from volkey import detect as rdet  # noqa: E402
from volkey import match as rmatch  # noqa: E402
from volkey import orient as rori  # noqa: E402
from volkey import scalespace as rss  # noqa: E402
from volkey import volume as rvol  # noqa: E402
from volkey.config import PipelineConfig  # noqa: E402
from volkey.pipeline import assign_orientations, extract_features  # noqa: E402

from paper_2112_10258_b200 import synthetic  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def kp_arrays(kps):
    return dict(
        kp_pos=np.array([k.position for k in kps], dtype=np.float64).reshape(-1, 3),
        kp_sigma=np.array([k.sigma for k in kps], dtype=np.float64),
        kp_octave=np.array([k.octave for k in kps], dtype=np.int32),
        kp_level=np.array([k.level for k in kps], dtype=np.int32),
        kp_dog=np.array([k.dog_value for k in kps], dtype=np.float64),
        kp_sign=np.array([1 if k.sign == "peak" else -1 for k in kps], dtype=np.int8),
    )


def frame_arrays(keypoints, oriented):
    index = {id(k): i for i, k in enumerate(keypoints)}
    return dict(
        fr_kp=np.array([index[id(k)] for k, _ in oriented], dtype=np.int32),
        fr_rot=np.array([f.rotation for _, f in oriented], dtype=np.float64).reshape(-1, 3, 3),
    )


def pyramid_hashes(pyr, dog):
    out = {}
    out["pyr_dims"] = np.array([o.levels[0].dims for o in pyr.octaves], dtype=np.int32)
    out["pyr_sha"] = np.array([[sha(l.data) for l in o.levels] for o in pyr.octaves])
    out["dog_sha"] = np.array([[sha(l.data) for l in o.levels] for o in dog.octaves])
    out["pyr_sigmas"] = np.array([o.sigmas for o in pyr.octaves], dtype=np.float64)
    return out


def describe(pyr, oriented, kind, cfg):
    pairs = None if kind == "siftrank" else rdesc.sample_point_pairs(cfg.method, cfg.pairs, 1.0, cfg.seed)
    recs, dropped = rdesc.describe_all(pyr, oriented, kind=kind, pairs=pairs, patch_side=cfg.patch_side,
                                       blur_sigma=cfg.blur_sigma, radius_factor=cfg.radius_factor)
    arr = rdesc.descriptor_array(recs, kind)
    return arr.astype(np.uint8), dropped, len(recs)


def full_case(vol_arr, cfg, with_hist=False):
    """Pyramid + detection + orientation once, then all three descriptor kinds."""
    t0 = time.time()
    vol = rvol.Volume(vol_arr)
    pyr = rss.build_gaussian_pyramid(vol, cfg.base_sigma, cfg.levels_per_octave, cfg.num_octaves,
                                     min_octave_dim=cfg.min_octave_dim)
    dog = rss.build_dog_pyramid(pyr)
    kps = rdet.detect_keypoints(dog, cfg.threshold_band, cfg.contrast_min)
    oriented, dropped_or = assign_orientations(pyr, kps, cfg)
    out = dict(input_sha=sha(vol.data), dropped_orientation=dropped_or)
    out.update(pyramid_hashes(pyr, dog))
    out.update(kp_arrays(kps))
    out.update(frame_arrays(kps, oriented))
    if with_hist:
        out["hist"] = np.array([rori.gradient_histogram(pyr, k, cfg.radius_factor).weights for k in kps])
    for kind in ("siftrank", "brief", "rrief"):
        arr, dropped, n = describe(pyr, oriented, kind, cfg)
        out[f"desc_{kind}"] = arr
        out[f"dropped_{kind}"] = dropped
    print(f"  case: {len(kps)} keypoints, {len(oriented)} frames, {time.time() - t0:.1f}s", flush=True)
    return out, pyr, kps, oriented


def unit_vectors():
    rng = np.random.default_rng(20240817)
    out = {}
    sigmas = [0.5, 0.8, 0.95, 1.2, 1.6, 2.0, 2.4, 3.2, 4.0]
    sig_sched = []
    kappa = 2.0 ** (1.0 / 3)
    local = [1.6 * kappa ** i for i in range(6)]
    for i in range(1, 6):
        sig_sched.append(rss._incremental_sigma(local[i - 1], local[i]))
    sigmas += sig_sched
    out["taps_sigmas"] = np.array(sigmas)
    out["taps"] = np.array([np.pad(rss.gaussian_kernel(s).weights, (0, 41 - len(rss.gaussian_kernel(s).weights)))
                            for s in sigmas], dtype=np.float32)
    out["taps_radius"] = np.array([rss.gaussian_kernel(s).radius for s in sigmas], dtype=np.int32)
    # separable blur on seeded random arrays: (seed, dims, sigma) -> output
    blur_cases = [((13, 11, 9), 1.6), ((16, 15, 14), 0.8), ((12, 10, 17), 2.4), ((1, 5, 7), 1.6),
                  ((2, 2, 2), 1.2), ((40, 33, 21), 3.0902), ((7, 40, 3), 1.9466)]
    for i, (dims, s) in enumerate(blur_cases):
        a = np.random.default_rng(100 + i).random(dims, dtype=np.float32)
        out[f"blur{i}_dims"] = np.array(dims)
        out[f"blur{i}_sigma"] = s
        out[f"blur{i}_out"] = rss.convolve_array(a, rss.gaussian_kernel(s))
    for i, dims in enumerate([(7, 6, 5), (2, 2, 2), (5, 4, 7), (33, 20, 18)]):
        a = np.random.default_rng(200 + i).random(dims, dtype=np.float32)
        out[f"sub{i}_dims"] = np.array(dims)
        out[f"sub{i}_out"] = rss.subsample_half(rvol.Volume(a)).data
    for i, dims in enumerate([(12, 11, 10), (3, 3, 3), (20, 9, 14)]):
        r = np.random.default_rng(300 + i)
        tri = [rvol.Volume(r.random(dims, dtype=np.float32)) for _ in range(3)]
        out[f"sos{i}_dims"] = np.array(dims)
        out[f"sos{i}_map"] = rdet.sum_of_signs_map(*tri)
    out["icosphere"] = rori.icosphere_directions().copy()
    rq = [1024, 2048, 4915, 11351, 14302, 18019, 9000, 15011]
    out["ball_rq"] = np.array(rq)
    out["ball_len"] = np.array([len(rori._ball_offsets(q)) for q in rq])
    out["ball_sha"] = np.array([sha(rori._ball_offsets(q).astype(np.int64)) for q in rq])
    for m in (1, 2, 3, 4, 5):
        for seed in (0, 13):
            p = rdesc.sample_point_pairs(m, 64, 1.0, seed)
            out[f"pairs_m{m}_s{seed}_p1"] = p.p1
            out[f"pairs_m{m}_s{seed}_p2"] = p.p2
    p = rdesc.sample_point_pairs(3, 100, 0.7, 5)
    out["pairs_odd_p1"], out["pairs_odd_p2"] = p.p1, p.p2
    out["patch_grid15"] = rdesc._patch_grid(15).copy()
    data = rng.random((9, 8, 7), dtype=np.float32)
    pts = rng.uniform(-2, 11, size=(500, 3))
    out["tri_pts"] = pts
    out["tri_out"] = rvol.sample_trilinear_array(data, pts)
    out["tri_seed_dims"] = np.array([9, 8, 7])
    # nearest-neighbour matching on seeded integer/binary descriptors
    r = np.random.default_rng(400)
    a = r.integers(0, 64, size=(300, 64))
    b = r.integers(0, 64, size=(280, 64))
    ms = rmatch.nearest_neighbor_matches(a, b, 0.9, "euclidean")
    out["nn_eu_a"], out["nn_eu_b"] = a.astype(np.int8), b.astype(np.int8)
    out["nn_eu"] = np.array([(m.index_a, m.index_b, m.distance, m.second_distance) for m in ms])
    ba = np.packbits((r.random((300, 64)) > 0.5).astype(np.uint8), axis=1)
    bb = np.packbits((r.random((310, 64)) > 0.5).astype(np.uint8), axis=1)
    ms = rmatch.nearest_neighbor_matches(ba, bb, 0.9, "hamming")
    out["nn_ha_a"], out["nn_ha_b"] = ba, bb
    out["nn_ha"] = np.array([(m.index_a, m.index_b, m.distance, m.second_distance) for m in ms])
    return out


def main():
    t0 = time.time()
    np.savez_compressed(os.path.join(HERE, "unit.npz"), **unit_vectors())
    print(f"unit vectors done {time.time() - t0:.1f}s", flush=True)

    cfg = PipelineConfig()
    # small phantoms (reference tests/phantoms.py:36-52 with noise)
    small = {}
    for i, (dims, seed) in enumerate([((40, 44, 36), 7), ((33, 30, 41), 11), ((48, 48, 48), 3)]):
        ref = ref_phantoms.random_blob_phantom(dims, np.random.default_rng(seed), n_blobs=10, margin=6,
                                              noise=0.02).data
        mine = synthetic.random_blob_phantom(dims, np.random.default_rng(seed), n_blobs=10, margin=6,
                                             noise=0.02)
        assert np.array_equal(ref, mine), "restated phantom generator diverged"
        out, _, _, _ = full_case(ref, cfg, with_hist=True)
        out["dims"] = np.array(dims)
        out["seed"] = seed
        small[i] = out
        np.savez_compressed(os.path.join(HERE, f"small{i}.npz"), **out)
    # a soup phantom with a non-default configuration (band, contrast, 5 levels)
    dims = (50, 46, 38)
    vol = synthetic.soup_volume(dims, np.random.default_rng(5), noise=0.01)
    cfg2 = PipelineConfig(levels_per_octave=5, threshold_band=2, contrast_min=0.003, num_octaves=3,
                          secondary_ratio=0.7, max_frames=3, pairs=48, method=1, blur_sigma=1.3, seed=4)
    out, _, _, _ = full_case(vol, cfg2, with_hist=True)
    out["dims"] = np.array(dims)
    np.savez_compressed(os.path.join(HERE, "soup_cfg2.npz"), **out)
    print(f"small cases done {time.time() - t0:.1f}s", flush=True)

    # configs[0]: the brain-scale volume
    rng = np.random.default_rng(20240817)
    c, s, a = ref_phantoms.soup_params((145, 174, 145), rng)
    ref_vol = ref_phantoms.kernel_soup_field((145, 174, 145), c, s, a)
    ref_vol = ref_vol + rng.normal(0, 0.01, (145, 174, 145)).astype(np.float32)
    mine = synthetic.brain_volume()
    assert np.array_equal(ref_vol, mine), "restated brain volume diverged"
    out, _, _, _ = full_case(mine, cfg)
    np.savez_compressed(os.path.join(HERE, "brain.npz"), **out)
    print(f"brain case done {time.time() - t0:.1f}s", flush=True)

    # configs[1]: two-volume matching pair
    rot = ref_phantoms.rotation_from_axis_angle((0.3, 1.0, 0.2), 10.0)
    tr = rmatch.SimilarityTransform7DOF(1.0, rot, np.array([2.0, -1.0, 1.5]))
    va, vb = ref_phantoms.transformed_pair((145, 174, 145), np.random.default_rng(20240817), tr, noise=0.01)
    ma, mb = synthetic.match_pair()
    assert np.array_equal(va.data, ma) and np.array_equal(vb.data, mb), "restated pair diverged"
    res = {}
    for tag, arr in (("a", ma), ("b", mb)):
        o, _, _, _ = full_case(arr, cfg)
        for k, v in o.items():
            res[f"{tag}_{k}"] = v
    for kind, metric in (("siftrank", "euclidean"), ("brief", "hamming"), ("rrief", "euclidean")):
        a = res[f"a_desc_{kind}"].astype(np.int64) if kind != "brief" else res[f"a_desc_{kind}"]
        b = res[f"b_desc_{kind}"].astype(np.int64) if kind != "brief" else res[f"b_desc_{kind}"]
        ms = rmatch.nearest_neighbor_matches(a, b, cfg.ratio_max, metric)
        res[f"nn_{kind}"] = np.array([(m.index_a, m.index_b, m.distance, m.second_distance) for m in ms])
        print(f"  nn {kind}: {len(ms)} matches", flush=True)
    np.savez_compressed(os.path.join(HERE, "pair.npz"), **res)
    print(f"all done {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
