"""CPU: the C-ABI library loads and exports every symbol include/*.h
declares; the ctypes layouts match the header; no GPU compute is called."""

import ctypes
import glob
import os
import re

import numpy as np
import pytest

from conftest import REPO

from paper_2112_10258_b200 import _lib


def declared_functions():
    names = []
    for h in glob.glob(os.path.join(REPO, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?[a-z_ ]+\**\s*\**(vk_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # every declared entry point has a ctypes signature in the binding
    assert set(names) <= set(_lib.SIGNATURES), set(names) - set(_lib.SIGNATURES)
    assert lib.vk_abi_version() == 2


def test_record_layouts_match_header():
    src = open(os.path.join(REPO, "include", "volkey_b200.h")).read()
    assert _lib.LEVEL_DTYPE.itemsize == 32 and _lib.KP_DTYPE.itemsize == 32
    assert _lib.BALL_DTYPE.itemsize == 32 and _lib.FRAME_DTYPE.itemsize == 16
    for struct, dt in (("vk_kp", _lib.KP_DTYPE), ("vk_ball", _lib.BALL_DTYPE), ("vk_frame", _lib.FRAME_DTYPE)):
        body = re.search(r"typedef struct %s \{(.*?)\}" % struct, src, re.S).group(1)
        fields = re.findall(r"int\s+([\w, ]+);", body)
        flat = [f.strip() for grp in fields for f in grp.split(",")]
        assert len(flat) == len(dt.names), struct


def test_parameter_errors_need_no_gpu():
    """Argument validation runs before any CUDA call and maps to ParameterError."""
    lib = _lib.load()
    rc = lib.vk_blur3d(None, None, None, None, 1, 4, 4, 4, None, 3, None)
    assert rc == 5 and "vk_blur3d" in _lib.last_error()
    with pytest.raises(Exception) as ei:
        _lib.check(rc, "vk_blur3d")
    assert type(ei.value).__name__ == "ParameterError"
    assert lib.vk_match(0, None, 1, None, 1, 8, 0.9, None, None, None, None, None) == 5


def test_compute_entry_points_fail_loudly_without_gpu():
    from conftest import has_gpu

    if has_gpu():
        pytest.skip("GPU present")
    import paper_2112_10258_b200 as vk

    with pytest.raises(vk.DeviceError):
        vk.extract_features(vk.Volume(np.zeros((8, 8, 8), np.float32)))


def test_sm100a_code_in_library():
    """The library carries sm_100a SASS (cuobjdump), not just PTX."""
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump missing")
    out = subprocess.run([tool, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
