"""Build ``libvolkey_b200.so`` in-tree with nvcc for sm_100a.

    python -m paper_2112_10258_b200.build [--verbose]

The library is a plain C ABI (``include/volkey_b200.h``); the Python host
binds it with ctypes (``paper_2112_10258_b200/_lib.py``).  Rebuilds only when
a source is newer than the library.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libvolkey_b200.so")
HEADER = os.path.join(REPO, "include", "volkey_b200.h")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS_C = ["-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-Xcompiler", "-fPIC,-O2",
           "--expt-relaxed-constexpr"]


CXX = os.environ.get("CXX", "g++")
# host C++ (vk_consensus.cpp): IEEE double arithmetic step for step as CPython / numpy
# do it -- no FMA contraction, no fast-math; -mfma only so that the explicit fma()
# calls (OpenBLAS kernel restatements) become single instructions
FLAGS_CXX = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-mfma", "-Wall"]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [HEADER]
    return any(os.path.getmtime(p) > t for p in deps)


def _compile(src: str, objdir: str, verbose: bool) -> str:
    base, ext = os.path.splitext(os.path.basename(src))
    obj = os.path.join(objdir, base + (".o" if ext == ".cu" else "_cpp.o"))
    if ext == ".cpp":
        cmd = [CXX, *FLAGS_CXX, "-I", os.path.join(REPO, "include"), "-c", src, "-o", obj]
    else:
        cmd = [NVCC, *ARCH, *FLAGS_C, "-I", os.path.join(REPO, "include"), "-c", src, "-o", obj]
    if verbose and ext == ".cu":
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {os.path.basename(src)} with exit code {res.returncode}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every csrc/*.cu in parallel (one nvcc per translation unit),
    then link the shared library."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(PKG, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    srcs = sources()
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + [HEADER]
    t_hdr = max(os.path.getmtime(p) for p in hdrs)

    def one(src):  # incremental: reuse an object newer than its source and every header
        base, ext = os.path.splitext(os.path.basename(src))
        obj = os.path.join(objdir, base + (".o" if ext == ".cu" else "_cpp.o"))
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(os.path.getmtime(src), t_hdr):
            return obj
        return _compile(src, objdir, verbose)

    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(one, srcs))
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "shared", *objs, "-ldl", "-o", LIB + ".tmp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed with exit code {res.returncode}")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
