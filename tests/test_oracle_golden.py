"""CPU: pin the oracle restatement (and the product's host tables) to the
golden vectors generated from the real reference (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from conftest import load_golden, sha
from oracle import volkey_oracle as O
from paper_2112_10258_b200 import synthetic
from paper_2112_10258_b200 import tables as T

CFG2 = dict(levels_per_octave=5, threshold_band=2, contrast_min=0.003, num_octaves=3, secondary_ratio=0.7,
            max_frames=3, pairs=48, method=1, blur_sigma=1.3, seed=4)


def test_gaussian_taps(golden_unit):
    g = golden_unit
    for s, w, r in zip(g["taps_sigmas"], g["taps"], g["taps_radius"]):
        ro, wo = O.gauss_taps(float(s))
        k = T.gaussian_kernel(float(s))
        assert ro == r == k.radius
        assert np.array_equal(wo, w[: 2 * r + 1]) and np.array_equal(k.weights, w[: 2 * r + 1])


def test_blur_subsample_sos(golden_unit):
    g = golden_unit
    i = 0
    while f"blur{i}_dims" in g:
        dims = tuple(int(d) for d in g[f"blur{i}_dims"])
        a = np.random.default_rng(100 + i).random(dims, dtype=np.float32)
        assert np.array_equal(O.blur3(a, O.gauss_taps(float(g[f"blur{i}_sigma"]))[1]), g[f"blur{i}_out"])
        i += 1
    for i in range(4):
        dims = tuple(int(d) for d in g[f"sub{i}_dims"])
        a = np.random.default_rng(200 + i).random(dims, dtype=np.float32)
        assert np.array_equal(O.half(a), g[f"sub{i}_out"])
    for i in range(3):
        dims = tuple(int(d) for d in g[f"sos{i}_dims"])
        r = np.random.default_rng(300 + i)
        tri = [r.random(dims, dtype=np.float32) for _ in range(3)]
        assert np.array_equal(O.sos_map(*tri), g[f"sos{i}_map"])


def test_known_answers():
    # reference tests: 2x2x2 {0..7} -> 3.5; isolated max scores 80; stable ranks
    assert O.half(np.arange(8, dtype=np.float32).reshape(2, 2, 2))[0, 0, 0] == 3.5
    a = np.zeros((3, 3, 3), np.float32)
    a[1, 1, 1] = 1.0
    assert O.sos_map(np.zeros_like(a), a, np.zeros_like(a))[1, 1, 1] == 80
    assert O.ranks([3.1, -2.0, 7.4]).tolist() == [1, 0, 2]
    assert O.ranks([5.0, 5.0, 5.0, 1.0]).tolist() == [1, 2, 3, 0]
    assert O.hamming(np.array([[0xFF, 0x00]], np.uint8), np.array([[0x0F, 0x00], [0xFF, 0xFF]], np.uint8)).tolist() == [[4.0, 8.0]]
    k = O.gauss_taps(1.6)[1]
    assert k[len(k) // 2] / k[len(k) // 2 + 1] == pytest.approx(np.exp(0.5 / 1.6 ** 2), rel=1e-6)


def test_host_tables(golden_unit):
    g = golden_unit
    assert np.array_equal(O.icosphere(), g["icosphere"]) and np.array_equal(T.icosphere_directions(), g["icosphere"])
    for q, n, h in zip(g["ball_rq"], g["ball_len"], g["ball_sha"]):
        assert len(T.ball_offsets(int(q))) == n and sha(T.ball_offsets(int(q)).astype(np.int64)) == str(h)
        assert sha(O.ball(int(q)).astype(np.int64)) == str(h)
    from paper_2112_10258_b200.descriptor import _patch_grid, sample_point_pairs

    for m in (1, 2, 3, 4, 5):
        for seed in (0, 13):
            p = sample_point_pairs(m, 64, 1.0, seed)
            q1, q2 = O.point_pairs(m, 64, 1.0, seed)
            assert np.array_equal(p.p1, g[f"pairs_m{m}_s{seed}_p1"]) and np.array_equal(p.p2, g[f"pairs_m{m}_s{seed}_p2"])
            assert np.array_equal(q1, p.p1) and np.array_equal(q2, p.p2)
    p = sample_point_pairs(3, 100, 0.7, 5)
    assert np.array_equal(p.p1, g["pairs_odd_p1"]) and np.array_equal(p.p2, g["pairs_odd_p2"])
    assert np.array_equal(_patch_grid(15), g["patch_grid15"]) and np.array_equal(O.patch_grid(15), g["patch_grid15"])
    data = np.random.default_rng(20240817).random((9, 8, 7), dtype=np.float32)
    pts = np.random.default_rng(20240817)
    pts.random((9, 8, 7), dtype=np.float32)
    pts = pts.uniform(-2, 11, size=(500, 3))
    assert np.array_equal(pts, g["tri_pts"]) and np.array_equal(O.trilinear(data, pts), g["tri_out"])


def test_frame_table_matches_reference_rotations():
    """Rotations from the host frame table equal the reference's
    dominant_orientations for the same (primary, secondary) pair."""
    ok, rot = T.default_frame_tables()
    dirs = T.icosphere_directions()
    rng = np.random.default_rng(0)
    for _ in range(50):
        w = rng.random(42)
        got = O.frames_from_hist(w, dirs, 0.8, 4)
        pairs = O.frame_pairs_from_hist(w, 0.8, 4)
        assert len(got) == len(pairs)
        for R, (p, q) in zip(got, pairs):
            assert ok[p, q] and np.array_equal(R, rot[p, q])


def test_nn_golden(golden_unit):
    g = golden_unit
    got = np.array(O.nn_match(g["nn_eu_a"].astype(np.int64), g["nn_eu_b"].astype(np.int64), 0.9, "euclidean"))
    assert np.array_equal(got, g["nn_eu"])
    got = np.array(O.nn_match(g["nn_ha_a"], g["nn_ha_b"], 0.9, "hamming"))
    assert np.array_equal(got, g["nn_ha"])


def _check_case(g, vol, cfg):
    assert sha(vol) == str(g["input_sha"])
    kinds = ("siftrank", "brief", "rrief")
    res = O.extract(vol, **dict(cfg, descriptor="siftrank"))
    pyr, dg = res["pyramid"], res["dog"]
    assert np.array_equal(np.array([[sha(l) for l in o] for o in pyr["octaves"]]), g["pyr_sha"])
    assert np.array_equal(np.array([[sha(l) for l in o] for o in dg["octaves"]]), g["dog_sha"])
    kps = res["keypoints"]
    assert np.array_equal(np.array([k.position for k in kps]).reshape(-1, 3), g["kp_pos"])
    assert np.array_equal(np.array([k.sigma for k in kps]), g["kp_sigma"])
    assert np.array_equal(np.array([k.dog_value for k in kps]), g["kp_dog"])
    assert np.array_equal(np.array([np.asarray(R) for _, R in res["oriented"]]).reshape(-1, 3, 3), g["fr_rot"])
    if "hist" in g:
        for i, k in enumerate(kps):
            assert np.array_equal(O.orient_hist(pyr, k, cfg.get("radius_factor", 4.0)), g["hist"][i])
    for kind in kinds:
        pairs = None if kind == "siftrank" else O.point_pairs(cfg.get("method", 3), cfg.get("pairs", 64), 1.0,
                                                             cfg.get("seed", 13))
        recs, _ = O.describe(pyr, res["oriented"], kind, pairs, 15, cfg.get("blur_sigma", 0.95))
        assert np.array_equal(O.desc_array(recs, kind).astype(np.int64), g[f"desc_{kind}"].astype(np.int64)), kind


@pytest.mark.parametrize("i", [0, 1, 2])
def test_small_cases(i):
    g = load_golden(f"small{i}.npz")
    dims = tuple(int(d) for d in g["dims"])
    vol = synthetic.random_blob_phantom(dims, np.random.default_rng(int(g["seed"])), n_blobs=10, margin=6, noise=0.02)
    _check_case(g, vol, {})


def test_soup_cfg2():
    g = load_golden("soup_cfg2.npz")
    vol = synthetic.soup_volume(tuple(int(d) for d in g["dims"]), np.random.default_rng(5), noise=0.01)
    _check_case(g, vol, CFG2)


def test_brain_pyramid_and_keypoints():
    """configs[0] input regenerates bit-exactly; oracle pyramid + detection
    equal the reference's (1924 keypoints)."""
    g = load_golden("brain.npz")
    vol = synthetic.brain_volume()
    assert sha(vol) == str(g["input_sha"])
    pyr = O.pyramid(vol)
    dg = O.dog(pyr)
    assert np.array_equal(np.array([[sha(l) for l in o] for o in pyr["octaves"]]), g["pyr_sha"])
    kps = O.detect(dg)
    assert len(kps) == 1924
    assert np.array_equal(np.array([k.position for k in kps]), g["kp_pos"])


def test_brain_frames_and_siftrank():
    """configs[0] end to end through the oracle: orientation frames (3400) and
    SIFT-Rank descriptors equal the reference's (the GPU path is checked against
    the same golden in test_gpu_parity.test_brain_volume)."""
    g = load_golden("brain.npz")
    vol = synthetic.brain_volume()
    res = O.extract(vol, descriptor="siftrank")
    assert len(res["oriented"]) == len(g["fr_rot"]) == 3400
    assert np.array_equal(np.array([np.asarray(R) for _, R in res["oriented"]]).reshape(-1, 3, 3), g["fr_rot"])
    recs, _ = O.describe(res["pyramid"], res["oriented"], "siftrank")
    assert np.array_equal(O.desc_array(recs, "siftrank").astype(np.int64), g["desc_siftrank"].astype(np.int64))
