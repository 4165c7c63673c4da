"""Device time of the separate orientation + SIFT-Rank kernels (enqueue_orient +
enqueue_describe) on bench-style volumes for the library in VK_LIB_PATH (A/B of
compile-time variants); prints ms and a digest of the outputs."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2112_10258_b200 as vk
from paper_2112_10258_b200 import synthetic
from paper_2112_10258_b200.engine import Extractor

B = int(os.environ.get("AB_BATCH", "8"))
dims = (145, 174, 145)
base = synthetic.soup_volume(dims, np.random.default_rng(20240817), noise=0.01)
dev = torch.stack([vk.volume.to_device(v) for v in synthetic.batch_from(base, B, seed=3)])
ex = Extractor(dims, vk.PipelineConfig(), batch=B, input=dev)
st = torch.cuda.current_stream()
s = st.cuda_stream
ex.enqueue_pyramid(s)
ex.enqueue_detect(s)
torch.cuda.synchronize()
out = {}
for name, fn in (("orient", lambda: ex.enqueue_orient(s)), ("describe", lambda: ex.enqueue_describe(s))):
    ts = []
    for _ in range(5):
        if name == "orient":
            pass
        else:
            ex.enqueue_orient(s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    out[name] = round(min(ts), 3)
r = ex.results()
dg = hashlib.sha256(r["desc"].tobytes() + r["rot"].tobytes()).hexdigest()[:16]
print(os.environ.get("VK_LIB_PATH", "default"), out, "sum", round(sum(out.values()), 3), "digest", dg, "frames", r["n_frames"])
