"""Per-stage device times + fast-path fallback counts for a batch (diagnostics)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2112_10258_b200 as vk
from paper_2112_10258_b200 import _lib, synthetic
from paper_2112_10258_b200.engine import Extractor

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--descriptor", default="siftrank")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
dims = (145, 174, 145)
host = synthetic.batch_from(synthetic.brain_volume(), a.batch, seed=1)
dev = torch.empty((a.batch,) + dims[::-1], dtype=torch.float32, device="cuda")
tmp = torch.from_numpy(host).cuda()
_lib.call("vk_transpose_zfast_to_xfast", tmp.data_ptr(), dev.data_ptr(), a.batch, *dims, _lib.stream_ptr())
for exact in (False, True):
    ex = Extractor(dims, vk.PipelineConfig(descriptor=a.descriptor), batch=a.batch, input=dev, exact_only=exact)
    st = torch.cuda.current_stream()
    s = st.cuda_stream
    times = {k: [] for k in ("pyramid", "detect", "gradients", "orient", "describe")}
    for _ in range(a.reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record(st); ex.enqueue_pyramid(s); ev[1].record(st); ex.enqueue_detect(s); ev[2].record(st)
        ex.enqueue_gradients(s); ev[3].record(st)
        ex.enqueue_orient(s); ev[4].record(st); ex.enqueue_describe(s); ev[5].record(st)
        torch.cuda.synchronize()
        for k, e0, e1 in zip(times, ev[:-1], ev[1:]):
            times[k].append(e0.elapsed_time(e1))
    c = ex.counts()
    print(f"exact_only={exact} batch={a.batch} ms:", {k: round(min(v), 3) for k, v in times.items()},
          "kp", c["keypoints"], "frames", c["frames"], "orient_fb", c["orient_fallbacks"], "sr_fb", c["siftrank_fallbacks"])
