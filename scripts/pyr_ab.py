"""A/B of the pyramid kernels on one 8-volume sub-batch (CUDA events, median
of 7) plus a bit-equality check of every level / DoG between the variants.
    python scripts/pyr_ab.py [--batch 8]"""
import argparse
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2112_10258_b200 as vk  # noqa: E402
from paper_2112_10258_b200 import _lib, synthetic  # noqa: E402
from paper_2112_10258_b200.engine import Extractor  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--dims", default="145,174,145")
ap.add_argument("--octaves", type=int, default=6)
ap.add_argument("--variants", default="0:1,0:0")  # xy kernel : z kernel
ap.add_argument("--reps", type=int, default=7)
a = ap.parse_args()
dims = tuple(int(x) for x in a.dims.split(","))
cfg = vk.PipelineConfig(num_octaves=a.octaves)
host = synthetic.batch_from(synthetic.soup_volume(dims, np.random.default_rng(1), noise=0.01), a.batch, seed=5)
ex = Extractor(dims, cfg, batch=a.batch)
for i, v in enumerate(host):
    ex.input[i].copy_(vk.volume.to_device(v))
st = torch.cuda.current_stream()
lib = _lib.load()


def run(variant):
    xy, z = (int(v) for v in variant.split(":"))
    lib.vk_set_xy_kernel(xy)
    lib.vk_set_z_kernel(z)
    ex.enqueue_pyramid(st.cuda_stream)
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        ex.enqueue_pyramid(st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    snap = [t.clone() for lv in ex.levels for t in lv] + [t.clone() for dg in ex.dogs for t in dg]
    return statistics.median(ts), snap


sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import pyramid_bytes  # noqa: E402
import json  # noqa: E402

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
res = {}
for v in a.variants.split(','):
    ms, snap = run(v)
    res[v] = snap
    gbs = pyramid_bytes(ex.plan) * a.batch / (ms / 1e3) / 1e9
    print(f"xy:z kernels {v}: pyramid {ms:.4f} ms / {a.batch} volumes = {1e3 * ms / a.batch:.1f} us/volume, "
          f"{gbs:.0f} GB/s = {gbs / peak:.3f} of peak", flush=True)
keys = list(res)
for k in keys[1:]:
    same = all(torch.equal(x, y) for x, y in zip(res[keys[0]], res[k]))
    print(f"levels + DoG bit-identical {keys[0]} vs {k}:", same)
lib.vk_set_xy_kernel(0)
lib.vk_set_z_kernel(0)
