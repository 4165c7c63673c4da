"""Where do the tensor-core and dp4a int8 matchers disagree? (debug aid)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2112_10258_b200 import _lib

rng = np.random.default_rng(0)
na, nb = int(sys.argv[1]), int(sys.argv[2])
a_np = np.argsort(rng.random((na, 64)), axis=1).astype(np.int8)
b_np = np.argsort(rng.random((nb, 64)), axis=1).astype(np.int8)
a, b = torch.from_numpy(a_np).cuda(), torch.from_numpy(b_np).cuda()
res = []
for path in (0, 1):
    out = [torch.empty(na, dtype=t, device="cuda") for t in (torch.int32, torch.float64, torch.float64, torch.uint8)]
    _lib.call("vk_set_match_path", path)
    _lib.call("vk_match", 1, a.data_ptr(), na, b.data_ptr(), nb, 64, 0.9, *[o.data_ptr() for o in out], _lib.stream_ptr())
    torch.cuda.synchronize()
    res.append([o.cpu().numpy() for o in out])
bad = np.nonzero((res[0][0] != res[1][0]) | (res[0][1] != res[1][1]) | (res[0][2] != res[1][2]))[0]
print("mismatching rows:", len(bad), bad[:10])
A = a.float()
for q in bad[:5]:
    d = (A[q] * A[q]).sum() + (b.float() ** 2).sum(1) - 2 * (b.float() @ A[q])
    d = d.cpu().numpy().astype(np.int64)
    j = int(np.argmin(d))
    s = np.sort(d)
    print(f"q={q} tc=({res[0][0][q]}, {res[0][1][q]**2:.0f}, {res[0][2][q]**2:.0f}) dp4a=({res[1][0][q]}, {res[1][1][q]**2:.0f}, {res[1][2][q]**2:.0f})"
          f" true=({j}, {s[0]}, {s[1]})")
