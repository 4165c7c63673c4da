import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2112_10258_b200 import _lib
rng = np.random.default_rng(0)
na, nb = 32768, 262144
a = torch.from_numpy(np.argsort(rng.random((na, 64)), axis=1).astype(np.int8)).cuda()
b = torch.from_numpy(np.argsort(rng.random((nb, 64)), axis=1).astype(np.int8)).cuda()
out = [torch.empty(na, dtype=t, device="cuda") for t in (torch.int32, torch.float64, torch.float64, torch.uint8)]
_lib.call("vk_match", 1, a.data_ptr(), na, b.data_ptr(), nb, 64, 0.9, *[o.data_ptr() for o in out], _lib.stream_ptr())
torch.cuda.synchronize()
