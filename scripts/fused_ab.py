"""A/B of the fused orientation + SIFT-Rank kernel (vk_orient_siftrank) against
the separate orient_kernel + siftrank_kernel on bench-style volumes: outputs
must be identical; prints device times (CUDA events, min of reps)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2112_10258_b200 as vk
from paper_2112_10258_b200 import _lib, synthetic
from paper_2112_10258_b200.engine import Extractor

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--dims", default="145,174,145")
ap.add_argument("--radius-factor", type=float, default=4.0, help="staged mode: balls must fit the staging buffer")
ap.add_argument("--mode", default="global", choices=("stage", "global"))
a = ap.parse_args()
dims = tuple(int(v) for v in a.dims.split(","))
base = synthetic.soup_volume(dims, np.random.default_rng(20240817), noise=0.01)
host = synthetic.batch_from(base, a.batch, seed=3)
dev = torch.stack([vk.volume.to_device(v) for v in host])
ex = Extractor(dims, vk.PipelineConfig(radius_factor=a.radius_factor), batch=a.batch, input=dev,
               fused=True if a.mode == "stage" else "global")
assert ex.fused, "fused path not selected"
st = torch.cuda.current_stream()
s = st.cuda_stream
ex.enqueue_pyramid(s)
ex.enqueue_detect(s)
torch.cuda.synchronize()


def timed(fn):
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), sorted(ts)[len(ts) // 2]


t_sep = timed(lambda: (ex.enqueue_orient(s), ex.enqueue_describe(s)))
sep = {k: v.copy() for k, v in ex.results().items() if isinstance(v, np.ndarray)}
c_sep = ex.counts()
t_fus = timed(lambda: ex.enqueue_orient_describe(s))
fus = {k: v.copy() for k, v in ex.results().items() if isinstance(v, np.ndarray)}
c_fus = ex.counts()
same = {k: bool(np.array_equal(sep[k], fus[k])) for k in sep}
print("separate ms (min, median):", t_sep, "fused ms:", t_fus)
print("keypoints", c_fus["keypoints"], "frames", c_fus["frames"], "sep fallbacks", c_sep["orient_fallbacks"],
      c_sep["siftrank_fallbacks"], "fused fallbacks", c_fus["orient_fallbacks"], c_fus["siftrank_fallbacks"])
print("identical:", all(same.values()), {k: v for k, v in same.items() if not v})
