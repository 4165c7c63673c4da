"""Throughput of the int8 rank-descriptor matcher: tensor-core path vs dp4a path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2112_10258_b200 import _lib

rng = np.random.default_rng(0)
for na, nb in ((3333, 3290), (32768, 262144), (131072, 1048576)):
    a = torch.from_numpy(np.argsort(rng.random((na, 64)), axis=1).astype(np.int8)).cuda()
    b = torch.from_numpy(np.argsort(rng.random((nb, 64)), axis=1).astype(np.int8)).cuda()
    out = [torch.empty(na, dtype=t, device="cuda") for t in (torch.int32, torch.float64, torch.float64, torch.uint8)]
    res = {}
    for path in (0, 2, 1):  # 0: warp-specialised tcgen05, 2: barrier tcgen05 (tc kernel 1), 1: dp4a
        if path == 1 and na * nb > 2e10:
            continue
        _lib.call("vk_set_match_path", 1 if path == 1 else 0)
        _lib.call("vk_set_match_tc_kernel", 1 if path == 2 else 0)
        st = _lib.stream_ptr()
        call = lambda: _lib.call("vk_match", 1, a.data_ptr(), na, b.data_ptr(), nb, 64, 0.9, *[o.data_ptr() for o in out], st)
        call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps):
            call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[path] = [o.cpu().numpy() for o in out]
        tops = 2.0 * na * nb * 64 / (ms * 1e-3) / 1e12
        print(f"na={na} nb={nb} path={['tcgen05-ws', 'dp4a', 'tcgen05-barrier'][path]}: {ms:.3f} ms  "
              f"{na * nb / (ms * 1e-3) / 1e12:.2f} Tpairs/s  {tops:.1f} TOPS (int8 MAC=2 ops)", flush=True)
    for other in (1, 2):
        if other in res:
            print(f"  path 0 == path {other}:", all(np.array_equal(x, y) for x, y in zip(res[0], res[other])))
_lib.call("vk_set_match_path", 0)
_lib.call("vk_set_match_tc_kernel", 0)
