"""GPU parity: the CUDA path against golden vectors made by the real reference.

Every comparison is exact (np.array_equal / sha256 of float32 bytes): the
hot path is integer / fixed-order IEEE arithmetic and the kernels reproduce
the reference's rounding sequence.  Inputs are
regenerated from seeds with ``paper_2112_10258_b200.synthetic`` and checked
against the input hash stored in the fixture.
"""

import numpy as np
import pytest

from conftest import load_golden, sha

pytestmark = pytest.mark.gpu

vk = pytest.importorskip("paper_2112_10258_b200")
from paper_2112_10258_b200 import synthetic  # noqa: E402
from paper_2112_10258_b200.config import PipelineConfig  # noqa: E402

CFG2 = dict(levels_per_octave=5, threshold_band=2, contrast_min=0.003, num_octaves=3, secondary_ratio=0.7,
            max_frames=3, pairs=48, method=1, blur_sigma=1.3, seed=4)
KINDS = ("siftrank", "brief", "rrief")


def small_volume(g):
    dims = tuple(int(d) for d in g["dims"])
    return synthetic.random_blob_phantom(dims, np.random.default_rng(int(g["seed"])), n_blobs=10, margin=6, noise=0.02)


def case_inputs(name):
    g = load_golden(name)
    if name.startswith("small"):
        vol = small_volume(g)
        cfg = PipelineConfig()
    elif name == "soup_cfg2.npz":
        vol = synthetic.soup_volume(tuple(int(d) for d in g["dims"]), np.random.default_rng(5), noise=0.01)
        cfg = PipelineConfig(**CFG2)
    else:
        vol = synthetic.brain_volume()
        cfg = PipelineConfig()
    assert sha(vol) == str(g["input_sha"]), "synthetic input generator diverged from the golden input"
    return g, vol, cfg


def check_extraction(g, vol, cfg, prefix=""):
    for kind in KINDS:
        res = vk.extract_features(vk.Volume(vol), cfg.model_copy(update={"descriptor": kind}))
        if kind == "siftrank":
            dims = [o.levels[0].dims for o in res.pyramid.octaves]
            assert np.array_equal(np.array(dims), g[prefix + "pyr_dims"])
            got = np.array([[sha(lv.data) for lv in o.levels] for o in res.pyramid.octaves])
            assert np.array_equal(got, g[prefix + "pyr_sha"]), "gaussian pyramid differs"
            got = np.array([[sha(lv.data) for lv in o.levels] for o in res.dog.octaves])
            assert np.array_equal(got, g[prefix + "dog_sha"]), "DoG pyramid differs"
            kps = res.keypoints
            assert len(kps) == len(g[prefix + "kp_sigma"])
            assert np.array_equal(np.array([k.position for k in kps]).reshape(-1, 3), g[prefix + "kp_pos"])
            assert np.array_equal(np.array([k.sigma for k in kps]), g[prefix + "kp_sigma"])
            assert np.array_equal(np.array([k.octave for k in kps]), g[prefix + "kp_octave"])
            assert np.array_equal(np.array([k.level for k in kps]), g[prefix + "kp_level"])
            assert np.array_equal(np.array([k.dog_value for k in kps]), g[prefix + "kp_dog"])
            assert np.array_equal(np.array([1 if k.sign == "peak" else -1 for k in kps]), g[prefix + "kp_sign"])
            idx = {id(k): i for i, k in enumerate(kps)}
            assert np.array_equal(np.array([idx[id(k)] for k, _ in res.oriented]), g[prefix + "fr_kp"])
            assert np.array_equal(np.array([f.rotation for _, f in res.oriented]).reshape(-1, 3, 3), g[prefix + "fr_rot"])
            assert res.dropped_orientation == int(g[prefix + "dropped_orientation"])
        arr = vk.descriptor.descriptor_array(res.records, kind)
        want = g[prefix + f"desc_{kind}"]
        assert arr.shape == want.shape, kind
        assert np.array_equal(arr.astype(np.int64), want.astype(np.int64)), f"{kind} descriptors differ"


# ------------------------------------------------------------------- units
def test_blur_units(golden_unit):
    g = golden_unit
    i = 0
    while f"blur{i}_dims" in g:
        dims = tuple(int(d) for d in g[f"blur{i}_dims"])
        a = np.random.default_rng(100 + i).random(dims, dtype=np.float32)
        k = vk.scalespace.gaussian_kernel(float(g[f"blur{i}_sigma"]))
        out = vk.scalespace.convolve_array(a, k)
        assert np.array_equal(out, g[f"blur{i}_out"]), f"blur case {i} {dims}"
        i += 1
    assert i >= 7


def test_blur_all_radii_match_oracle():
    """Every radius the ring kernel instantiates (1..10) plus the generic path."""
    from oracle import volkey_oracle as O

    rng = np.random.default_rng(7)
    for sigma in (0.3, 0.6, 0.9, 1.2, 1.5, 1.9, 2.2, 2.6, 2.9, 3.2, 3.6, 4.5, 6.0):
        dims = tuple(int(d) for d in rng.integers(3, 40, size=3))
        a = rng.random(dims, dtype=np.float32)
        r, w = O.gauss_taps(sigma)
        want = O.blur3(a, w)
        got = vk.scalespace.convolve_array(a, vk.scalespace.gaussian_kernel(sigma))
        assert np.array_equal(got, want), f"sigma {sigma} radius {r} dims {dims}"


def test_blur_fused_epilogues_batched():
    """vk_blur3d with the DoG and 2x-subsample epilogues on a batch of odd-sized
    volumes (partial tiles, z-chunking, clamped borders) for every radius the
    streaming kernel instantiates: bit-equal to the oracle's blur3 / difference
    / half (scalespace.py:63-82, 137-151)."""
    import torch

    from oracle import volkey_oracle as O
    from paper_2112_10258_b200 import _lib

    rng = np.random.default_rng(11)
    for sigma, dims in ((0.3, (37, 9, 70)), (0.6, (33, 35, 64)), (0.9, (66, 40, 34)), (1.2, (45, 71, 40)),
                        (1.5, (64, 64, 33)), (1.9, (35, 38, 90)), (2.2, (71, 33, 36)), (2.6, (40, 40, 47)),
                        (2.9, (97, 65, 34)), (3.2, (33, 100, 41)), (3.6, (50, 37, 96))):
        nb = 3
        r, w = O.gauss_taps(sigma)
        a = rng.standard_normal((nb,) + dims).astype(np.float32)  # numpy [b][x][y][z]
        xf = np.ascontiguousarray(a.transpose(0, 3, 2, 1))         # x-fastest [b][z][y][x]
        src = torch.from_numpy(xf).cuda()
        dst = torch.empty_like(src)
        dog = torch.empty_like(src)
        hs = tuple(d // 2 for d in dims)
        half = torch.empty((nb,) + hs[::-1], dtype=torch.float32, device="cuda")
        wt = np.ascontiguousarray(w, dtype=np.float32)
        _lib.call("vk_blur3d", src.data_ptr(), dst.data_ptr(), dog.data_ptr(), half.data_ptr(), nb, *dims,
                  wt.ctypes.data, r, _lib.stream_ptr())
        torch.cuda.synchronize()
        got = dst.cpu().numpy().transpose(0, 3, 2, 1)
        gdog = dog.cpu().numpy().transpose(0, 3, 2, 1)
        ghalf = half.cpu().numpy().transpose(0, 3, 2, 1)
        for i in range(nb):
            want = O.blur3(a[i], w)
            assert np.array_equal(got[i], want), f"blur sigma {sigma} radius {r} dims {dims} volume {i}"
            assert np.array_equal(gdog[i], a[i] - want), f"dog sigma {sigma} radius {r}"
            assert np.array_equal(ghalf[i], O.half(want)), f"half sigma {sigma} radius {r}"


def test_xy_kernels_with_previous_pair_dog():
    """Every (x, y) kernel of the split blur (vk_set_xy_kernel 0 = plane, 1 =
    tile, 2 = persistent two-group plane kernel) with the previous pair's DoG
    fused in (vk_blur3d_ws2): level, DoG of the blurred pair and the previous
    pair's DoG bit-equal to the oracle (scalespace.py:63-82, 137-151)."""
    import torch

    from oracle import volkey_oracle as O
    from paper_2112_10258_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(23)
    try:
        for k in (0, 1, 2):
            assert lib.vk_set_xy_kernel(k) == 0
            for sigma, dims in ((0.9, (145, 37, 19)), (2.2, (61, 174, 23)), (3.6, (33, 50, 41))):
                nb = 3
                r, w = O.gauss_taps(sigma)
                a = rng.standard_normal((nb,) + dims).astype(np.float32)  # [b][x][y][z]
                p = rng.standard_normal((nb,) + dims).astype(np.float32)
                tx = lambda v: torch.from_numpy(np.ascontiguousarray(v.transpose(0, 3, 2, 1))).cuda()  # noqa: E731
                src, prev = tx(a), tx(p)
                dst, dog, pdog = torch.empty_like(src), torch.empty_like(src), torch.empty_like(src)
                wt = np.ascontiguousarray(w, dtype=np.float32)
                _lib.call("vk_blur3d_ws2", src.data_ptr(), dst.data_ptr(), dog.data_ptr(), None, prev.data_ptr(),
                          pdog.data_ptr(), nb, *dims, wt.ctypes.data, r, None, 0, _lib.stream_ptr())
                torch.cuda.synchronize()
                back = lambda t: t.cpu().numpy().transpose(0, 3, 2, 1)  # noqa: E731
                got, gdog, gp = back(dst), back(dog), back(pdog)
                for i in range(nb):
                    want = O.blur3(a[i], w)
                    assert np.array_equal(got[i], want), f"xy kernel {k} sigma {sigma} dims {dims}"
                    assert np.array_equal(gdog[i], a[i] - want), f"xy kernel {k} dog sigma {sigma}"
                    assert np.array_equal(gp[i], p[i] - a[i]), f"xy kernel {k} previous-pair dog sigma {sigma}"
    finally:
        lib.vk_set_xy_kernel(0)


def test_subsample_units(golden_unit):
    g = golden_unit
    for i in range(4):
        dims = tuple(int(d) for d in g[f"sub{i}_dims"])
        a = np.random.default_rng(200 + i).random(dims, dtype=np.float32)
        out = vk.scalespace.subsample_half(vk.Volume(a))
        assert np.array_equal(out.data, g[f"sub{i}_out"])


def test_sum_of_signs_units(golden_unit):
    g = golden_unit
    for i in range(3):
        dims = tuple(int(d) for d in g[f"sos{i}_dims"])
        r = np.random.default_rng(300 + i)
        tri = [vk.Volume(r.random(dims, dtype=np.float32)) for _ in range(3)]
        assert np.array_equal(vk.detect.sum_of_signs_map(*tri), g[f"sos{i}_map"])


def test_nn_units(golden_unit):
    g = golden_unit
    for metric, a, b, want in (("euclidean", g["nn_eu_a"].astype(np.int64), g["nn_eu_b"].astype(np.int64), g["nn_eu"]),
                               ("hamming", g["nn_ha_a"], g["nn_ha_b"], g["nn_ha"])):
        ms = vk.nearest_neighbor_matches(a, b, 0.9, metric)
        got = np.array([(m.index_a, m.index_b, m.distance, m.second_distance) for m in ms])
        assert np.array_equal(got, want), metric


def test_nn_float_and_ties():
    from oracle import volkey_oracle as O

    rng = np.random.default_rng(3)
    a, b = rng.random((40, 16)), rng.random((55, 16))
    ms = vk.nearest_neighbor_matches(a, b, 1.0)
    ref = O.nn_match(a, b, 1.0)
    assert [(m.index_a, m.index_b) for m in ms] == [(r[0], r[1]) for r in ref]
    np.testing.assert_allclose([m.distance for m in ms], [r[2] for r in ref], rtol=1e-9)
    # identical rows: ties keep the lower index and d2 == d1
    c = rng.integers(0, 64, size=(10, 64))
    b2 = np.concatenate([c, c])
    ms = vk.nearest_neighbor_matches(c, b2, 1.0)
    assert [(m.index_a, m.index_b, m.distance, m.second_distance) for m in ms] == [(i, i, 0.0, 0.0) for i in range(10)]


def _nn_raw(a8, b8, ratio, ex_lo=0, ex_hi=0, path=0):
    import torch

    from paper_2112_10258_b200 import _lib

    _lib.call("vk_set_match_path", path)
    try:
        A = torch.from_numpy(np.ascontiguousarray(a8)).cuda()
        B = torch.from_numpy(np.ascontiguousarray(b8)).cuda()
        n = len(a8)
        best = torch.empty(n, dtype=torch.int32, device="cuda")
        d1 = torch.empty(n, dtype=torch.float64, device="cuda")
        d2 = torch.empty(n, dtype=torch.float64, device="cuda")
        keep = torch.empty(n, dtype=torch.uint8, device="cuda")
        _lib.call("vk_match_excluding", 1, A.data_ptr(), n, B.data_ptr(), len(b8), a8.shape[1], float(ratio), ex_lo,
                  ex_hi, best.data_ptr(), d1.data_ptr(), d2.data_ptr(), keep.data_ptr(), _lib.stream_ptr())
        return best.cpu().numpy(), d1.cpu().numpy(), d2.cpu().numpy(), keep.cpu().numpy()
    finally:
        _lib.call("vk_set_match_path", 0)


def test_nn_tensor_core_path_matches_oracle():
    """tcgen05 kind::i8 matcher == dp4a matcher == oracle (match.py:70-121):
    full-range int8 rows (not only rank permutations), duplicate rows (ties
    keep the first index), ragged tile edges, 32..128-byte rows, and an
    excluded row range straddling tile boundaries."""
    from oracle import volkey_oracle as O

    rng = np.random.default_rng(21)
    for na, nb, dim, ex in ((300, 700, 64, (0, 0)), (129, 513, 32, (250, 300)), (77, 1030, 128, (0, 256)),
                            (256, 257, 96, (0, 0)), (5, 3, 64, (0, 0))):
        a = rng.integers(-128, 128, size=(na, dim)).astype(np.int8)
        b = rng.integers(-128, 128, size=(nb, dim)).astype(np.int8)
        b[nb // 2] = b[nb // 3]                     # a tie
        a[0] = b[nb // 3]                           # ... that is the exact nearest neighbour of row 0
        lo, hi = ex
        got_tc = _nn_raw(a, b, 0.9, lo, hi, path=0)
        got_dp = _nn_raw(a, b, 0.9, lo, hi, path=1)
        for x, y in zip(got_tc, got_dp):
            assert np.array_equal(x, y), (na, nb, dim, ex)
        from paper_2112_10258_b200 import _lib as L

        lib = L.load()
        lib.vk_set_match_tc_kernel(1)  # the barrier-synchronised N = 128 kernel agrees too
        try:
            got_t1 = _nn_raw(a, b, 0.9, lo, hi, path=0)
        finally:
            lib.vk_set_match_tc_kernel(0)
        for x, y in zip(got_tc, got_t1):
            assert np.array_equal(x, y), (na, nb, dim, ex)
        bb = np.concatenate([b[:lo], b[hi:]]).astype(np.int64)
        ref = O.nn_match(a.astype(np.int64), bb, 1.0)
        assert [int(i) for i in got_tc[0]] == [r[1] for r in ref]
        assert np.array_equal(got_tc[1], np.array([r[2] for r in ref])), (na, nb, dim)
        assert np.array_equal(got_tc[2], np.array([r[3] for r in ref])), (na, nb, dim)
    # rank permutations (SIFT-Rank rows), configs[1]-sized
    a = np.stack([rng.permutation(64) for _ in range(3333)]).astype(np.int8)
    b = np.stack([rng.permutation(64) for _ in range(3290)]).astype(np.int8)
    for x, y in zip(_nn_raw(a, b, 0.9, path=0), _nn_raw(a, b, 0.9, path=1)):
        assert np.array_equal(x, y)


# ------------------------------------------------------------ end to end
@pytest.mark.parametrize("name", ["small0.npz", "small1.npz", "small2.npz", "soup_cfg2.npz"])
def test_small_cases(name):
    g, vol, cfg = case_inputs(name)
    check_extraction(g, vol, cfg)


@pytest.mark.parametrize("name", ["small0.npz", "small2.npz", "soup_cfg2.npz"])
def test_gradient_histograms_exact(name):
    g, vol, cfg = case_inputs(name)
    pyr = vk.build_gaussian_pyramid(vk.Volume(vol), cfg.base_sigma, cfg.levels_per_octave, cfg.num_octaves,
                                    min_octave_dim=cfg.min_octave_dim)
    for i in range(len(g["kp_sigma"])):
        kp = vk.Keypoint(tuple(g["kp_pos"][i]), float(g["kp_sigma"][i]), int(g["kp_octave"][i]), int(g["kp_level"][i]),
                         float(g["kp_dog"][i]), "peak" if g["kp_sign"][i] > 0 else "valley")
        h = vk.orient.gradient_histogram(pyr, kp, cfg.radius_factor)
        assert np.array_equal(h.weights, g["hist"][i]), f"keypoint {i}"


def test_nearest_direction_exact_on_dense_gradients():
    """The screened / fast icosphere argmax (csrc/vk_orient.cu) on every voxel
    of blurred random and quantised volumes (millions of gradients, incl.
    exact ties and axis-aligned gradients) == np.argmax of the reference's
    fp64 dots g @ dirs.T (orient.py:89-125), zero gradients -> 255."""
    import torch

    from oracle import volkey_oracle as O
    from paper_2112_10258_b200 import _lib, tables

    dirs = tables.icosphere_directions()
    ico = np.ascontiguousarray(tables.icosphere_structure())
    d_dirs = torch.from_numpy(np.ascontiguousarray(dirs)).cuda()
    rng = np.random.default_rng(17)
    r, w = O.gauss_taps(1.2)
    smooth = O.blur3(rng.standard_normal((48, 40, 36)).astype(np.float32), w)
    for vol in (smooth, np.round(smooth * 64.0).astype(np.float32) / 64.0,
                (rng.integers(0, 3, size=(40, 40, 40)) * 0.5).astype(np.float32)):
        nx, ny, nz = vol.shape
        xf = torch.from_numpy(np.ascontiguousarray(vol.transpose(2, 1, 0))).cuda()
        g4 = torch.empty((nz, ny, nx, 4), dtype=torch.float32, device="cuda")
        bins = torch.empty((nz, ny, nx), dtype=torch.uint8, device="cuda")
        _lib.call("vk_gradient_volume", xf.data_ptr(), g4.data_ptr(), bins.data_ptr(), 1, nx, ny, nz,
                  d_dirs.data_ptr(), ico.ctypes.data, _lib.stream_ptr())
        got = bins.cpu().numpy().transpose(2, 1, 0).reshape(-1)
        idx = np.indices(vol.shape).reshape(3, -1).T
        g = O.grads_at(vol, idx)
        want = np.argmax(g @ dirs.T, axis=1)
        want[np.all(g == 0.0, axis=1)] = 255
        assert np.array_equal(got, want)


def test_stage_api_composition():
    """build_gaussian_pyramid -> build_dog_pyramid -> detect_keypoints ->
    assign_orientations -> describe_all, the composition of
    tests/test_acceptance.py:53-89, equals the fused pipeline."""
    g, vol, cfg = case_inputs("small2.npz")
    v = vk.Volume(vol)
    pyr = vk.build_gaussian_pyramid(v)
    dog = vk.build_dog_pyramid(pyr)
    assert np.array_equal(np.array([[sha(lv.data) for lv in o.levels] for o in dog.octaves]), g["dog_sha"])
    kps = vk.detect_keypoints(dog)
    assert np.array_equal(np.array([k.position for k in kps]), g["kp_pos"])
    oriented, dropped = vk.assign_orientations(pyr, kps, cfg)
    assert np.array_equal(np.array([f.rotation for _, f in oriented]), g["fr_rot"])
    for kind in KINDS:
        pairs = None if kind == "siftrank" else vk.descriptor.sample_point_pairs(cfg.method, cfg.pairs, 1.0, cfg.seed)
        recs, dd = vk.descriptor.describe_all(pyr, oriented, kind, pairs)
        assert dd == 0
        assert np.array_equal(vk.descriptor.descriptor_array(recs, kind).astype(np.int64),
                              g[f"desc_{kind}"].astype(np.int64)), kind


@pytest.mark.slow
def test_brain_volume():
    """configs[0]: 145x174x145 soup phantom -> 1924 keypoints / 3400 frames, all exact."""
    g, vol, cfg = case_inputs("brain.npz")
    assert len(g["kp_sigma"]) == 1924 and len(g["fr_kp"]) == 3400
    check_extraction(g, vol, cfg)


@pytest.mark.slow
@pytest.mark.slow
def test_large_volume_configs3():
    """configs[3]: 256^3 soup volume, num_octaves=4 -> 9228 keypoints / 16509
    frames; every keypoint field, frame rotation and descriptor of all three
    kinds hash-equal to the reference's (tests/golden/large256.npz)."""
    g = load_golden("large256.npz")
    vol = synthetic.soup_volume((256, 256, 256), np.random.default_rng(synthetic.BRAIN_SEED), noise=0.01)
    assert sha(vol) == str(g["input_sha"])
    for kind in ("siftrank", "brief", "rrief"):
        res = vk.extract_features(vk.Volume(vol), PipelineConfig(num_octaves=4, descriptor=kind))
        kps = res.keypoints
        if kind == "siftrank":
            arrays = dict(
                kp_pos=np.array([k.position for k in kps], dtype=np.float64).reshape(-1, 3),
                kp_sigma=np.array([k.sigma for k in kps], dtype=np.float64),
                kp_octave=np.array([k.octave for k in kps], dtype=np.int32),
                kp_level=np.array([k.level for k in kps], dtype=np.int32),
                kp_dog=np.array([k.dog_value for k in kps], dtype=np.float64),
                kp_sign=np.array([1 if k.sign == "peak" else -1 for k in kps], dtype=np.int8))
            idx = {id(k): i for i, k in enumerate(kps)}
            arrays["fr_kp"] = np.array([idx[id(k)] for k, _ in res.oriented], dtype=np.int32)
            arrays["fr_rot"] = np.array([f.rotation for _, f in res.oriented], dtype=np.float64).reshape(-1, 3, 3)
            for k, v in arrays.items():
                assert len(v) == int(g[k + "_len"]) and sha(v) == str(g[k + "_sha"]), k
            got = np.array([[sha(lv.data) for lv in o.levels] for o in res.pyramid.octaves])
            assert np.array_equal(got, g["pyr_sha"]), "gaussian pyramid differs"
            got = np.array([[sha(lv.data) for lv in o.levels] for o in res.dog.octaves])
            assert np.array_equal(got, g["dog_sha"]), "DoG pyramid differs"
        desc = vk.descriptor.descriptor_array(res.records, kind).astype(np.uint8)
        assert len(desc) == int(g[f"desc_{kind}_len"]) and sha(desc) == str(g[f"desc_{kind}_sha"]), kind


def test_fast_and_exact_accumulation_agree():
    """The bounded parallel accumulation must give the same frames and ranks
    as forcing the reference-order accumulation everywhere."""
    g, vol, cfg = case_inputs("brain.npz")
    outs = []
    for exact in (False, True):
        ex = vk.Extractor(vol.shape, cfg, batch=1, exact_only=exact)
        ex.input[0].copy_(vk.volume.to_device(vol))
        ex.enqueue()
        outs.append(ex.results())
    a, b = outs
    assert np.array_equal(a["frame_prim"], b["frame_prim"]) and np.array_equal(a["frame_sec"], b["frame_sec"])
    assert np.array_equal(a["desc"], b["desc"])
    assert np.array_equal(a["desc"], g["desc_siftrank"])


@pytest.mark.slow
def test_pair_matching():
    """configs[1]: two-volume matching, all three descriptor kinds."""
    g = load_golden("pair.npz")
    va, vb = synthetic.match_pair()
    assert sha(va) == str(g["a_input_sha"]) and sha(vb) == str(g["b_input_sha"])
    cfg = PipelineConfig()
    for kind, metric in (("siftrank", "euclidean"), ("brief", "hamming"), ("rrief", "euclidean")):
        c = cfg.model_copy(update={"descriptor": kind})
        ra = vk.extract_features(vk.Volume(va), c)
        rb = vk.extract_features(vk.Volume(vb), c)
        da = vk.descriptor.descriptor_array(ra.records, kind)
        db = vk.descriptor.descriptor_array(rb.records, kind)
        assert np.array_equal(da.astype(np.int64), g[f"a_desc_{kind}"].astype(np.int64))
        assert np.array_equal(db.astype(np.int64), g[f"b_desc_{kind}"].astype(np.int64))
        ms = vk.nearest_neighbor_matches(da, db, cfg.ratio_max, metric)
        got = np.array([(m.index_a, m.index_b, m.distance, m.second_distance) for m in ms])
        assert np.array_equal(got, g[f"nn_{kind}"]), kind


def test_count_inlier_matches_end_to_end():
    """configs[1] accuracy metric end to end: GPU extraction of both volumes,
    GPU nearest neighbours, host Hough consensus == the reference's inliers
    (tests/golden/hough.npz)."""
    h = load_golden("hough.npz")
    va, vb = synthetic.match_pair()
    for kind in ("siftrank", "brief", "rrief"):
        n, rep = vk.count_inlier_matches(vk.Volume(va), vk.Volume(vb), PipelineConfig(descriptor=kind))
        assert n == len(h[f"{kind}_inliers"]), kind
        assert rep["transform"].scale == float(h[f"{kind}_scale"])
        assert np.array_equal(rep["transform"].translation, h[f"{kind}_translation"])


def test_write_soa_equals_record_writer(tmp_path):
    """keyfiles.write_soa straight from Extractor.results() == the record-based
    writer on the same extraction (both byte-identical to the reference format)."""
    from paper_2112_10258_b200 import keyfiles as kf

    vols = [small_volume(load_golden(f"small{i}.npz"))[:40, :44, :36] for i in (0, 2)]
    for kind in ("siftrank", "brief"):
        cfg = PipelineConfig(descriptor=kind)
        soa = vk.extract_batch(np.stack(vols), cfg)
        for b, v in enumerate(vols):
            kf.write_soa(tmp_path / "soa.txt", soa, kind, 64, cfg.seed, volume=b)
            res = vk.extract_features(vk.Volume(v), cfg)
            kf.write_descriptors(tmp_path / "rec.txt", res.records, kind, 64, cfg.seed)
            assert (tmp_path / "soa.txt").read_bytes() == (tmp_path / "rec.txt").read_bytes(), (kind, b)


def test_batch_equals_single():
    """Batched extraction (volume-major SoA) equals one-volume extraction."""
    vols = [small_volume(load_golden(f"small{i}.npz")) for i in (0, 2)]
    vols = [v[:40, :44, :36] for v in vols]
    batch = np.stack(vols)
    res = vk.extract_batch(batch, PipelineConfig())
    off = list(res["vol_offset"]) + [res["n_keypoints"]]
    for b, v in enumerate(vols):
        single = vk.extract_features(vk.Volume(v))
        n = off[b + 1] - off[b]
        assert n == len(single.keypoints)
        assert np.array_equal(res["pos"][off[b]:off[b + 1]], np.array([k.position for k in single.keypoints]).reshape(-1, 3))
        sel = (res["frame_kp"] >= off[b]) & (res["frame_kp"] < off[b + 1])
        assert np.array_equal(res["desc"][sel].astype(np.int64),
                              vk.descriptor.descriptor_array(single.records, "siftrank"))


def test_edge_cases():
    # tiny volumes: octave truncation, no keypoints, 1-voxel dims
    for dims in ((1, 1, 1), (2, 3, 2), (5, 5, 5), (9, 3, 12)):
        a = np.random.default_rng(1).random(dims, dtype=np.float32)
        from oracle import volkey_oracle as O

        res = vk.extract_features(vk.Volume(a), PipelineConfig(num_octaves=3))
        want = O.extract(a, num_octaves=3)
        assert [len(o.levels) for o in res.pyramid.octaves] == [len(o) for o in want["pyramid"]["octaves"]]
        for o, oc in enumerate(res.pyramid.octaves):
            for i, lv in enumerate(oc.levels):
                assert np.array_equal(lv.data, want["pyramid"]["octaves"][o][i])
        assert len(res.keypoints) == len(want["keypoints"])
    # constant volume: no keypoints, no frames
    res = vk.extract_features(vk.Volume(np.full((20, 20, 20), 3.0, np.float32)))
    assert res.stats["keypoints"] == 0 and res.records == []
    # errors mirror the reference
    with pytest.raises(vk.ParameterError):
        vk.scalespace.subsample_half(vk.Volume(np.zeros((1, 4, 4), np.float32)))
    with pytest.raises(vk.ParameterError):
        vk.build_gaussian_pyramid(vk.Volume(np.zeros((8, 8, 8), np.float32)), levels_per_octave=3)
    with pytest.raises(vk.ParameterError):
        vk.nearest_neighbor_matches(np.zeros((3, 8)), np.zeros((1, 8)))


@pytest.mark.parametrize("kind", ["siftrank", "brief"])
def test_fast_path_adversarial(kind):
    """Quantised / plateau volumes (exact ties, zero gradients, axis-aligned
    gradients): the bounded fast path must equal forced reference order, and
    both must equal the oracle."""
    from oracle import volkey_oracle as O

    rng = np.random.default_rng(11)
    smooth = synthetic.random_blob_phantom((36, 38, 34), rng, n_blobs=14, margin=4)
    vols = [np.round(smooth * 256.0).astype(np.float32) / 256.0,                   # plateaus + ties
            rng.integers(0, 9, size=(30, 32, 28)).astype(np.float32),              # integer noise
            np.where(smooth > 0.05, 1.0, 0.0).astype(np.float32) + smooth * 1e-3]  # near-binary
    cfg = PipelineConfig(descriptor=kind, num_octaves=2)
    n_desc = []
    for vol in vols:
        outs = []
        for exact in (False, True):
            ex = vk.Extractor(vol.shape, cfg, batch=1, exact_only=exact)
            ex.input[0].copy_(vk.volume.to_device(vol))
            ex.enqueue()
            outs.append(ex.results())
        a, b = outs
        assert np.array_equal(a["frame_prim"], b["frame_prim"]) and np.array_equal(a["frame_sec"], b["frame_sec"])
        assert np.array_equal(a["desc"], b["desc"])
        want = O.extract(vol, descriptor=kind, num_octaves=2)
        assert a["n_keypoints"] == len(want["keypoints"])
        assert len(a["desc"]) == len(want["records"])
        if len(want["records"]):
            assert np.array_equal(a["desc"].astype(np.int64), O.desc_array(want["records"], kind).astype(np.int64))
        n_desc.append(len(want["records"]))
    assert sum(n_desc) > 20


def test_database_matching_single_rank():
    """configs[4] composition on one rank: match_database == per-subject
    nearest_neighbor_matches(desc_i, concat_{j != i} desc_j) of the oracle."""
    import torch.distributed as dist

    from oracle import volkey_oracle as O
    from paper_2112_10258_b200.distributed import match_database

    rng = np.random.default_rng(5)
    subjects = {i: np.stack([rng.permutation(64) for _ in range(int(rng.integers(20, 60)))]) for i in range(5)}
    if not dist.is_initialized():
        import os
        import socket

        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=0, world_size=1)
    bits = {i: rng.integers(0, 256, size=(int(rng.integers(20, 60)), 8)).astype(np.uint8) for i in range(5)}
    try:
        got = match_database(subjects, 0.9, "euclidean")   # one tensor-core launch, per-row exclusions
        got_h = match_database(bits, 0.9, "hamming")         # popcount kernel, per subject
    finally:
        dist.destroy_process_group()
    for subj, res, metric in ((subjects, got, "euclidean"), (bits, got_h, "hamming")):
        for i, a in subj.items():
            others = np.concatenate([subj[j] for j in sorted(subj) if j != i])
            ref = O.nn_match(a, others, 0.9, metric)
            best, d1, d2, keep = res[i]
            mine = [(q, int(best[q]), float(d1[q]), float(d2[q])) for q in np.flatnonzero(keep)]
            assert mine == ref, f"{metric} subject {i}"


def test_point_samplers_match_oracle():
    """gradients_at (volume.py:244-264) and sample_trilinear_array
    (volume.py:203-236) on the GPU == the oracle, bit for bit, including
    border voxels, clamped out-of-range points and degenerate (1-voxel) axes."""
    from oracle import volkey_oracle as O
    from paper_2112_10258_b200.volume import (VoxelIndex, central_gradient, gradients_at, sample_trilinear_array,
                                              trilinear_sample)

    rng = np.random.default_rng(11)
    for dims in ((17, 23, 9), (1, 5, 4), (6, 1, 1)):
        data = rng.standard_normal(dims).astype(np.float32)
        idx = np.stack([rng.integers(0, d, 500) for d in dims], axis=1)
        idx[:8] = [[0, 0, 0], [dims[0] - 1, dims[1] - 1, dims[2] - 1]] * 4
        assert np.array_equal(gradients_at(data, idx), O.grads_at(data, idx))
        pts = rng.uniform(-2.0, np.array(dims) + 1.0, size=(700, 3))
        pts[:4] = [[0, 0, 0], np.array(dims) - 1.0, [0.5, 0.5, 0.5], np.array(dims) - 1.5]
        assert np.array_equal(sample_trilinear_array(data, pts), O.trilinear(data, pts))
        one = sample_trilinear_array(data, pts[5])
        assert np.ndim(one) == 0 and one == O.trilinear(data, pts[5:6])[0]
        v = vk.Volume(data)
        assert trilinear_sample(v, pts[6]) == float(O.trilinear(data, pts[6:7])[0])
        assert np.array_equal(central_gradient(v, VoxelIndex(*idx[9])), O.grads_at(data, idx[9:10])[0])
    assert gradients_at(data, np.zeros((0, 3), dtype=np.int64)).shape == (0, 3)
    with pytest.raises(IndexError):
        gradients_at(data, [[dims[0], 0, 0]])


def test_patch_building_blocks_match_oracle():
    """extract_patch / preblur_patch / brief_descriptor / rrief_descriptor
    (descriptor.py:96-111,196-224) one stage at a time on the GPU == the
    oracle, and composed == the fused describe_all records."""
    from oracle import volkey_oracle as O
    from paper_2112_10258_b200 import descriptor as D

    g, vol, cfg = case_inputs("small0.npz")
    res = vk.extract_features(vk.Volume(vol), cfg.model_copy(update={"descriptor": "brief"}))
    pairs = D.sample_point_pairs(cfg.method, cfg.pairs, 1.0, cfg.seed)
    opairs = (pairs.p1, pairs.p2)
    recs_r, _ = D.describe_all(res.pyramid, res.oriented, "rrief", pairs, cfg.patch_side, cfg.blur_sigma)
    assert len(res.records) >= 8
    for i in range(0, len(res.records), max(1, len(res.records) // 8)):
        rec = res.records[i]
        kp, fr = rec.keypoint, rec.frame
        okp = O.OKp(tuple(kp.position), kp.sigma, kp.octave, kp.level, kp.dog_value, kp.sign)
        want = O.patch({"source": vol}, okp, np.asarray(fr.rotation), cfg.patch_side)
        p = D.extract_patch(res.pyramid, kp, fr, cfg.patch_side)
        assert isinstance(p, D.Patch) and p.side == cfg.patch_side and np.array_equal(p.data, want)
        pb = D.preblur_patch(p, cfg.blur_sigma)
        want_b = O.preblur(want, cfg.blur_sigma)
        assert np.array_equal(pb.data, want_b)
        diffs = O.pair_diffs(want_b, opairs)
        bits = D.brief_descriptor(pb, pairs).bits
        assert np.array_equal(bits, (diffs > 0).astype(np.uint8))
        assert np.array_equal(bits, rec.descriptor.bits)
        ranks = D.rrief_descriptor(pb, pairs).ranks
        assert np.array_equal(ranks, O.ranks(diffs)) and np.array_equal(ranks, recs_r[i].descriptor.ranks)
    assert D.preblur_patch(p, 0.0) is p
    with pytest.raises(vk.ParameterError):
        D.extract_patch(res.pyramid, kp, fr, 14)


def test_dump_pyramid_round_trip(tmp_path):
    """dump_pyramid (scalespace.py:226-235): one .f32 per level, named by
    octave / level / sigma, reloading to the level's voxels."""
    from paper_2112_10258_b200.scalespace import build_gaussian_pyramid, dump_pyramid

    vol = synthetic.random_blob_phantom((20, 18, 16), np.random.default_rng(2), n_blobs=4, margin=3, noise=0.02)
    g = build_gaussian_pyramid(vk.Volume(vol), num_octaves=2)
    paths = dump_pyramid(g, tmp_path / "dump")
    assert len(paths) == sum(len(o.levels) for o in g.octaves)
    assert paths[0].endswith("oct0_lvl0_sigma%.4g.f32" % g.octaves[0].sigmas[0])
    back = vk.load_volume(paths[-1])
    assert np.array_equal(back.data, g.octaves[-1].levels[-1].data)


def test_uncertain_bin_repair_on_brain_batch():
    """configs[0]-style volumes hit near-tied SIFT-Rank bins (a few frames per
    volume) and near-tied orientation decisions (rarer): the uncertain-bin
    repairs (sr_exact_subset, ori_exact_subset) must give the same frames and
    ranks as the full reference-order accumulation of every keypoint."""
    dims = (145, 174, 145)
    host = synthetic.batch_from(synthetic.brain_volume(), 4, seed=3)
    outs, fallbacks = [], {}
    for exact in (False, True):
        ex = vk.Extractor(dims, PipelineConfig(), batch=4, exact_only=exact)
        for i, v in enumerate(host):
            ex.input[i].copy_(vk.volume.to_device(v))
        ex.enqueue()
        outs.append(ex.results())
        if not exact:
            fallbacks = ex.counts()
    a, b = outs
    assert fallbacks["siftrank_fallbacks"] > 0 and fallbacks["orient_fallbacks"] > 0, fallbacks
    assert np.array_equal(a["frame_prim"], b["frame_prim"]) and np.array_equal(a["frame_sec"], b["frame_sec"])
    assert len(a["desc"]) == len(b["desc"]) > 10000
    assert np.array_equal(a["desc"], b["desc"])


def test_orientation_field_walk_equals_gradient_walk():
    """The orientation field (vk_orient_field: per-voxel fast |g| + exact
    nearest direction, walked by every keypoint) gives the same frames and
    descriptors as recomputing gradients in each ball walk."""
    dims = (145, 174, 145)
    host = synthetic.batch_from(synthetic.brain_volume(), 2, seed=9)
    outs = []
    for field in (True, False):  # field walk (opt-in) vs the default fused walk
        ex = vk.Extractor(dims, PipelineConfig(), batch=2, orient_field=field)
        for i, v in enumerate(host):
            ex.input[i].copy_(vk.volume.to_device(v))
        ex.enqueue()
        outs.append(ex.results())
    a, b = outs
    assert np.array_equal(a["frame_prim"], b["frame_prim"]) and np.array_equal(a["frame_sec"], b["frame_sec"])
    assert np.array_equal(a["desc"], b["desc"]) and len(a["desc"]) > 5000


@pytest.mark.parametrize("radius_factor", [2.5, 3.0])
def test_fused_orientation_siftrank_equals_separate_and_exact(radius_factor):
    """The fused kernel (vk_orient_siftrank: stencil spheres staged in shared
    memory, clamped at the volume boundary, frames decided in the CTA) gives
    the same frames and rank vectors as the separate fast kernels and as the
    reference-order accumulation (exact_only, pinned to the reference's
    goldens elsewhere).  Radius factors whose balls fit the staging buffer;
    octaves 1-2 put many balls across the volume boundary."""
    dims = (145, 174, 145)
    base = synthetic.soup_volume(dims, np.random.default_rng(20240817), noise=0.01)
    host = synthetic.batch_from(base, 2, seed=13)
    cfg = PipelineConfig(radius_factor=radius_factor)
    outs = {}
    for mode in ("fused", "separate", "exact"):
        ex = vk.Extractor(dims, cfg, batch=2, exact_only=mode == "exact", fused=mode == "fused")
        assert ex.fused == (mode == "fused")
        for i, v in enumerate(host):
            ex.input[i].copy_(vk.volume.to_device(v))
        ex.enqueue()
        outs[mode] = ex.results()
    a = outs["fused"]
    assert a["n_frames"] > 2000
    for other in ("separate", "exact"):
        b = outs[other]
        assert a["n_frames"] == b["n_frames"] and a["dropped_orientation"] == b["dropped_orientation"]
        assert np.array_equal(a["frame_kp"], b["frame_kp"])
        assert np.array_equal(a["frame_prim"], b["frame_prim"]) and np.array_equal(a["frame_sec"], b["frame_sec"])
        assert np.array_equal(a["rot"], b["rot"])
        assert np.array_equal(a["desc"], b["desc"]), f"fused descriptors differ from {other}"


def test_full_distance_matrices_match_oracle():
    """match.py:64-78 full-matrix helpers on the GPU: popcount distances of
    packed bits and fp64 euclidean distances of integer rows (ranks, int8
    values: every product and sum is an exact fp64 integer, so the result is
    the reference's bit for bit; non-integer float rows follow cuBLAS's
    summation order instead of OpenBLAS's)."""
    from oracle import volkey_oracle as O

    rng = np.random.default_rng(8)
    a = rng.integers(0, 256, size=(57, 16)).astype(np.uint8)
    b = rng.integers(0, 256, size=(91, 16)).astype(np.uint8)
    got = vk.match.hamming_distances(a, b)
    assert np.array_equal(got, O.hamming(a, b))
    for lo, hi, dim in ((0, 64, 64), (-128, 128, 96)):
        a = rng.integers(lo, hi, size=(63, dim)).astype(np.int64)
        b = rng.integers(lo, hi, size=(77, dim)).astype(np.int64)
        b[5] = a[3]  # an exact zero distance
        got = vk.match.euclidean_distances(a, b)
        assert np.array_equal(got, O.euclid(a, b))


def test_batch_of_70_volumes_offsets():
    """More volumes than a warp (batch_offsets_kernel scans 32 at a time): the
    volume-major SoA of a 70-volume batch equals one-volume extractions."""
    base = small_volume(load_golden("small0.npz"))[:40, :44, :36]
    rng = np.random.default_rng(70)
    vols = [np.ascontiguousarray(np.roll(base, int(rng.integers(0, 9)), axis=int(rng.integers(0, 3))) +
                                 rng.normal(0, 0.01, base.shape).astype(np.float32)) for _ in range(70)]
    res = vk.extract_batch(np.stack(vols), PipelineConfig())
    off = list(res["vol_offset"]) + [res["n_keypoints"]]
    assert len(res["vol_offset"]) == 70
    for b in (0, 31, 32, 33, 63, 64, 69):
        single = vk.extract_features(vk.Volume(vols[b]))
        assert off[b + 1] - off[b] == len(single.keypoints), b
        assert np.array_equal(res["pos"][off[b]:off[b + 1]], np.array([k.position for k in single.keypoints]).reshape(-1, 3))
