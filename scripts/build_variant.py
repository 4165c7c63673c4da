"""Build an A/B variant of the library with extra nvcc defines:
    python scripts/build_variant.py NAME -DVK_VOTE_COPIES=16 ...
-> variants/libvolkey_NAME.so; load it with VK_LIB_PATH=variants/libvolkey_NAME.so."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_10258_b200 import build as B  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
out_dir = os.path.join(B.REPO, "variants")
os.makedirs(out_dir, exist_ok=True)
out = os.path.join(out_dir, f"libvolkey_{name}.so")
cmd = [B.NVCC, *B.ARCH, *B.FLAGS_C, "-shared", "-cudart", "shared", *defs, "-I", os.path.join(B.REPO, "include"), *B.sources(), "-o", out]
subprocess.run(cmd, check=True)
print(out)
