"""GPU parity on the volumes the benchmark extracts, the SURVEY §8(d) C3
volumes, zero-background / tiny-gradient volumes, and configs[4]-style
database matching -- all against outputs of the REAL reference
(tests/golden/make_bench_golden.py) or the oracle composition of
match.py:81-121.

The benchmark volumes run exactly as bench.py runs them: resident inputs, an
ExtractorGroup of parallel-stream sub-batches, captured as one CUDA graph and
replayed, fast (certified) accumulation path."""

import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, sha

pytestmark = pytest.mark.gpu

vk = pytest.importorskip("paper_2112_10258_b200")
from paper_2112_10258_b200 import synthetic  # noqa: E402
from paper_2112_10258_b200.config import PipelineConfig  # noqa: E402

sys.path.insert(0, GOLDEN)
from digest import digest_results  # noqa: E402

DIMS = (145, 174, 145)


def _bench_inputs(g):
    base = synthetic.brain_volume()
    vols = [("bench", i, v) for i, v in enumerate(synthetic.batch_from(base, 4, seed=1000))]
    vols += [("c3", s, synthetic.brain_volume(seed=s)) for s in (0, 1, 2, 3)]
    for tag, i, v in vols:
        assert sha(v) == str(g[f"{tag}{i}_input_sha"]), f"{tag}{i}: input generator diverged"
    return vols


def test_bench_and_c3_volumes_through_graphed_group():
    """8 full-size volumes (bench.py rank-0 inputs + C3 seeds 0..3) as 4
    parallel-stream sub-batches of 2 in one replayed CUDA graph: every
    volume's keypoints, frames and SIFT-Rank descriptors hash-equal the
    reference's (tests/golden/bench.npz)."""
    import torch

    from paper_2112_10258_b200.engine import Extractor, ExtractorGroup

    g = load_golden("bench.npz")
    vols = _bench_inputs(g)
    dev = torch.stack([vk.volume.to_device(v) for _, _, v in vols])
    cfg = PipelineConfig()
    members = [Extractor(DIMS, cfg, batch=2, input=dev[2 * m: 2 * m + 2]) for m in range(4)]
    grp = ExtractorGroup(members)
    grp.capture()
    for _ in range(2):  # replay twice: the second replay must not see state of the first
        grp.run()
    torch.cuda.synchronize()
    for m, ex in enumerate(members):
        r = ex.results()
        for j in range(2):
            tag, i, _ = vols[2 * m + j]
            d = digest_results(r, j)
            for k in ("n_kp", "n_fr", "kp", "fr", "desc"):
                assert d[k] == (int(g[f"{tag}{i}_{k}"]) if k.startswith("n_") else str(g[f"{tag}{i}_{k}"])), \
                    f"{tag}{i}: {k} differs from the reference"


def _zeroback(j, g):
    dims = tuple(int(d) for d in g[f"z{j}_dims"])
    return synthetic.zero_background_volume(dims, int(g[f"z{j}_seed"]), scale=float(g[f"z{j}_scale"]))


@pytest.mark.parametrize("j", [0, 1, 2])
def test_zero_background_volumes(j):
    """Zero outside a sphere (skull-stripped-MRI-like) and, for j = 2, a
    1e-22 scale where every fp32 sum of squared gradient components
    underflows: frames and all three descriptor kinds equal the reference's
    (fast fp32 |g| votes must be rescaled, never 0 for a nonzero fp64
    gradient -- vk_common.cuh norm3_f32 / nz_vote)."""
    from test_gpu_parity import check_extraction

    g = load_golden("zeroback.npz")
    vol = _zeroback(j, g)
    assert sha(vol) == str(g[f"z{j}_input_sha"])
    check_extraction(g, vol, PipelineConfig(), prefix=f"z{j}_")


@pytest.mark.parametrize("j", [0, 2])
def test_zero_background_histograms(j):
    g = load_golden("zeroback.npz")
    vol = _zeroback(j, g)
    pyr = vk.build_gaussian_pyramid(vk.Volume(vol))
    p = f"z{j}_"
    for i in range(len(g[p + "kp_sigma"])):
        kp = vk.Keypoint(tuple(g[p + "kp_pos"][i]), float(g[p + "kp_sigma"][i]), int(g[p + "kp_octave"][i]),
                         int(g[p + "kp_level"][i]), float(g[p + "kp_dog"][i]),
                         "peak" if g[p + "kp_sign"][i] > 0 else "valley")
        h = vk.orient.gradient_histogram(pyr, kp, 4.0)
        assert np.array_equal(h.weights, g[p + "hist"][i]), f"keypoint {i}"


# ------------------------------------------------------------ database matching
def _init_single_rank():
    import socket

    import torch.distributed as dist

    if dist.is_initialized():
        return False
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    return True


def _check_against_oracle(subjects, res, metric):
    from oracle import volkey_oracle as O

    for i, a in subjects.items():
        others = np.concatenate([subjects[j] for j in sorted(subjects) if j != i])
        ref = O.nn_match(a, others, 0.9, metric)
        best, d1, d2, keep = res[i]
        mine = [(q, int(best[q]), float(d1[q]), float(d2[q])) for q in np.flatnonzero(keep)]
        assert mine == ref, f"{metric} subject {i}"


def test_database_matching_20_subjects_real_descriptors():
    """configs[4] composition on 20 subjects whose SIFT-Rank and RRIEF
    descriptors come from the GPU extractor on distinct C3-style volumes
    (reduced 64^3 size): match_database == per-subject oracle
    nearest_neighbor_matches(desc_i, concat_{j != i} desc_j), plus one subject
    with no descriptors."""
    import torch.distributed as dist

    from paper_2112_10258_b200.distributed import match_database

    subj = {}
    for kind in ("siftrank", "rrief"):
        cfg = PipelineConfig(descriptor=kind)
        vols = np.stack([synthetic.brain_volume(seed=s, dims=(64, 60, 56)) for s in range(20)])
        r = vk.extract_batch(vols, cfg)
        off = list(r["vol_offset"]) + [r["n_keypoints"]]
        d = {}
        for s in range(20):
            sel = (r["frame_kp"] >= off[s]) & (r["frame_kp"] < off[s + 1])
            d[s] = r["desc"][sel].astype(np.int64)
        d[20] = np.zeros((0, d[0].shape[1]), np.int64)  # a subject whose every keypoint was dropped
        subj[kind] = d
    own = _init_single_rank()
    try:
        got = {k: match_database(v, 0.9, "euclidean") for k, v in subj.items()}
    finally:
        if own:
            dist.destroy_process_group()
    for kind in subj:
        assert sum(len(v) for v in subj[kind].values()) > 1000
        assert len(got[kind][20][0]) == 0
        _check_against_oracle(subj[kind], got[kind], "euclidean")


def test_database_matching_wide_ranks_use_fp64():
    """RRIEF with pairs > 128 gives ranks up to pairs - 1, outside int8: the
    database path must not wrap them (fp64 kernel instead), == oracle."""
    import torch.distributed as dist

    from paper_2112_10258_b200.distributed import match_database

    rng = np.random.default_rng(11)
    subjects = {i: np.stack([rng.permutation(200) for _ in range(int(rng.integers(10, 30)))]) for i in range(6)}
    own = _init_single_rank()
    try:
        got = match_database(subjects, 0.9, "euclidean")
    finally:
        if own:
            dist.destroy_process_group()
    _check_against_oracle(subjects, got, "euclidean")
