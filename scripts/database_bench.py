"""configs[4] end to end: S synthetic subjects -> GPU extraction (SIFT-Rank)
-> descriptor database all-gathered over NCCL -> per-subject nearest
neighbours against every other subject on the tcgen05 matcher.

    python scripts/database_bench.py [--subjects 1000]                      # 1 GPU
    torchrun --nproc-per-node 8 scripts/database_bench.py --subjects 1000   # 8 GPUs

Subjects are the configs[0] phantom with per-subject flips / cyclic shifts and
fresh N(0, 0.01) noise generated on the device (seeded).  Prints one JSON line
(rank 0) with the stage times (max over ranks, CUDA events).
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import paper_2112_10258_b200 as vk
from paper_2112_10258_b200 import _lib, synthetic
from paper_2112_10258_b200.distributed import match_database, shard_range
from paper_2112_10258_b200.engine import Extractor

ap = argparse.ArgumentParser()
ap.add_argument("--subjects", type=int, default=1000)
ap.add_argument("--batch", type=int, default=24)
a = ap.parse_args()
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29512")
dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
dims = (145, 174, 145)
base = synthetic.brain_volume()
tmp = torch.from_numpy(base[None]).cuda()
base_x = torch.empty((1,) + dims[::-1], device="cuda")
_lib.call("vk_transpose_zfast_to_xfast", tmp.data_ptr(), base_x.data_ptr(), 1, *dims, _lib.stream_ptr())
base_x = base_x[0]
lo, hi = shard_range(a.subjects, rank, world)
B = a.batch
ex = Extractor(dims, vk.PipelineConfig(), batch=B, kp_cap=B * 3000, frame_cap=B * 5200)
gen = torch.Generator(device="cuda")


def fill(first, n):
    for i in range(n):
        s = first + i
        gen.manual_seed(1000003 * (s + 1))
        r = np.random.default_rng(s)
        v = base_x
        flips = [ax for ax in (0, 1, 2) if r.random() < 0.5]
        if flips:
            v = torch.flip(v, flips)
        v = torch.roll(v, tuple(int(t) for t in r.integers(0, 16, size=3)), dims=(0, 1, 2))
        ex.input[i].copy_(v + 0.01 * torch.randn(v.shape, device="cuda", generator=gen))


torch.cuda.synchronize()
dist.barrier()
st = torch.cuda.current_stream()
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
t0 = time.time()
e0.record(st)
descs = {}
for first in range(lo, hi, B):
    n = min(B, hi - first)
    fill(first, n)
    ex.enqueue()
    r = ex.results()
    vol_of_frame = r["kp"]["vol"][r["frame_kp"]]
    for i in range(n):
        descs[first + i] = r["desc"][vol_of_frame == i]
e1.record(st)
res = match_database(descs, 0.9, "euclidean")
e2.record(st)
torch.cuda.synchronize()
wall = time.time() - t0
t = torch.tensor([e0.elapsed_time(e1), e1.elapsed_time(e2), wall * 1e3], device="cuda")
dist.all_reduce(t, op=dist.ReduceOp.MAX)
nd = torch.tensor([sum(len(d) for d in descs.values())], device="cuda")
dist.all_reduce(nd)
kept = torch.tensor([sum(int(v[3].sum()) for v in res.values())], device="cuda")
dist.all_reduce(kept)
spot = None
if world == 1 and len(descs) >= 3:
    # spot-check 3 subjects against the reference composition (match.py:81-121 applied to the
    # subject's rows vs the concatenation of every other subject, in id order), evaluated with the
    # independent dp4a kernel (vk_set_match_path(1)): best index, d1, d2 and ratio decision
    ids = sorted(descs)
    picks = [ids[0], ids[len(ids) // 2], ids[-1]]
    spot = {"subjects": picks, "equal": True, "kernel": "dp4a (vk_set_match_path 1)"}
    _lib.call("vk_set_match_path", 1)
    try:
        for i in picks:
            a8 = np.ascontiguousarray(descs[i].astype(np.int8))
            b8 = np.ascontiguousarray(np.concatenate([descs[j] for j in ids if j != i]).astype(np.int8))
            A, Bm = torch.from_numpy(a8).cuda(), torch.from_numpy(b8).cuda()
            n = len(a8)
            out = [torch.empty(n, dtype=dt, device="cuda") for dt in (torch.int32, torch.float64, torch.float64, torch.uint8)]
            _lib.call("vk_match", 1, A.data_ptr(), n, Bm.data_ptr(), len(b8), 64, 0.9, *[o.data_ptr() for o in out],
                      _lib.stream_ptr())
            got = [o.cpu().numpy() for o in out]
            spot["equal"] = spot["equal"] and all(np.array_equal(np.asarray(x), np.asarray(y)) for x, y in zip(got, res[i]))
    finally:
        _lib.call("vk_set_match_path", 0)
if rank == 0:
    total = int(nd.item())
    print(json.dumps({"workload": "configs[4]: database matching, SIFT-Rank", "subjects": a.subjects, "n_gpus": world,
                      "descriptors": total, "extract_ms": round(float(t[0]), 1), "gather_match_ms": round(float(t[1]), 1),
                      "wall_ms": round(float(t[2]), 1), "ratio_test_kept": int(kept.item()),
                      "pairs": total * total, "pairs_per_s_match": round(total * total / (float(t[1]) / 1e3)),
                      "spot_check": spot}))
dist.destroy_process_group()
