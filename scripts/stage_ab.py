"""Per-stage device times of one Extractor step (pyramid+detect, orient incl.
orientation fields, describe) for a 12-volume batch, best of 4; the
orientation field on and off."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2112_10258_b200 as vk
from paper_2112_10258_b200 import _lib, synthetic
from paper_2112_10258_b200.engine import Extractor

dims = (145, 174, 145)
B = 12
host = synthetic.batch_from(synthetic.brain_volume(), B, seed=1)
dev = torch.empty((B,) + dims[::-1], dtype=torch.float32, device="cuda")
tmp = torch.from_numpy(host).cuda()
_lib.call("vk_transpose_zfast_to_xfast", tmp.data_ptr(), dev.data_ptr(), B, *dims, _lib.stream_ptr())
for field in (True, False):
    ex = Extractor(dims, vk.PipelineConfig(), batch=B, input=dev, orient_field=field)
    st = torch.cuda.current_stream()
    s = st.cuda_stream
    best = None
    for _ in range(4):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(st); ex.enqueue_pyramid(s); ex.enqueue_detect(s); ev[1].record(st)
        ex.enqueue_orient(s); ev[2].record(st); ex.enqueue_describe(s); ev[3].record(st)
        torch.cuda.synchronize()
        t = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
        best = t if best is None or sum(t) < sum(best) else best
    c = ex.counts()
    print(f"orient_field={field}: pyr+det {best[0]:.3f} orient {best[1]:.3f} describe {best[2]:.3f} ms "
          f"total {sum(best):.3f}  kp {c['keypoints']} frames {c['frames']} fallbacks {c['orient_fallbacks']}/{c['siftrank_fallbacks']}")
