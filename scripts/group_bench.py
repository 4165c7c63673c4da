"""Throughput of B volumes as G parallel-stream sub-batches (one CUDA graph)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2112_10258_b200 as vk
from paper_2112_10258_b200 import _lib, synthetic
from paper_2112_10258_b200.engine import Extractor, ExtractorGroup

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="16x1,8x2,4x4,12x2,10x2,20x1")
ap.add_argument("--steps", type=int, default=8)
a = ap.parse_args()
dims = (145, 174, 145)
host = synthetic.batch_from(synthetic.brain_volume(), 40, seed=1)
dev = torch.empty((40,) + dims[::-1], dtype=torch.float32, device="cuda")
tmp = torch.from_numpy(host).cuda()
_lib.call("vk_transpose_zfast_to_xfast", tmp.data_ptr(), dev.data_ptr(), 40, *dims, _lib.stream_ptr())
del tmp
cfg = vk.PipelineConfig()
for spec in a.configs.split(","):
    b, g = (int(v) for v in spec.split("x"))
    exs = [Extractor(dims, cfg, batch=b, input=dev[i * b:(i + 1) * b]) for i in range(g)]
    grp = ExtractorGroup(exs)
    grp.enqueue()
    torch.cuda.synchronize()
    grp.capture()
    for _ in range(2):
        grp.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        grp.run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    print(f"B={b}x{g} ms/step={ms:.3f} vol/s={b * g / ms * 1e3:.1f} kps={[e.counts()['keypoints'] for e in exs]}", flush=True)
    del grp, exs
    torch.cuda.empty_cache()
