"""Run N eager pipeline steps on a batch of B brain-size volumes (for ncu)."""
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
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--descriptor", default="siftrank")
a = ap.parse_args()
dims = (145, 174, 145)
host = synthetic.batch_from(synthetic.brain_volume(), a.batch, seed=1)
dev = torch.empty((a.batch,) + dims[::-1], dtype=torch.float32, device="cuda")
tmp = torch.from_numpy(host).cuda()
_lib.call("vk_transpose_zfast_to_xfast", tmp.data_ptr(), dev.data_ptr(), a.batch, *dims, _lib.stream_ptr())
ex = Extractor(dims, vk.PipelineConfig(descriptor=a.descriptor), batch=a.batch, input=dev)
for _ in range(a.steps):
    ex.enqueue()
torch.cuda.synchronize()
print(f"batch={a.batch} steps={a.steps}")
print(ex.counts())
