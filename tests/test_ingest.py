"""Volume ingest (volume.py:73-200) against golden arrays produced by the real
reference loaders (tests/golden/make_ingest_golden.py)."""

import os

import numpy as np
import pytest

from conftest import load_golden
from paper_2112_10258_b200 import ingest
from paper_2112_10258_b200.errors import FormatError, InputOutputError

NAMES = {"f32": ".f32", "u8": ".nii", "i16": ".nii", "f32be": ".nii", "i16gz": ".nii.gz"}


def _write(tmp_path, name, g):
    p = os.path.join(tmp_path, name + NAMES[name])
    with open(p, "wb") as fh:
        fh.write(g[f"{name}_bytes"].tobytes())
    return p


def test_header_and_format_errors_need_no_gpu(tmp_path):
    g = load_golden("ingest.npz")
    with open(tmp_path / "v.hdr.txt", "w") as fh:
        fh.write("dims: 10 9 8\nspacing: 0.5 1 2\n")
    assert ingest.read_raw_header(tmp_path / "v.hdr.txt") == ((10, 9, 8), (0.5, 1.0, 2.0))
    with open(tmp_path / "bad.hdr.txt", "w") as fh:
        fh.write("dims: 10 9\nspacing: 1 1 1\n")
    with pytest.raises(FormatError):
        ingest.read_raw_header(tmp_path / "bad.hdr.txt")
    with pytest.raises(InputOutputError):
        ingest.read_raw_header(tmp_path / "missing.hdr.txt")
    p = _write(str(tmp_path), "f32", g)
    with pytest.raises(FormatError):
        ingest.load_raw(p, (10, 9, 9))                      # size mismatch, before any device work
    with pytest.raises(FormatError):
        ingest.load_volume(str(tmp_path / "v.vol"))
    short = tmp_path / "short.nii"
    short.write_bytes(b"\0" * 100)
    with pytest.raises(FormatError):
        ingest.load_nifti_subset(short)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(NAMES))
def test_loaders_match_reference(tmp_path, name):
    g = load_golden("ingest.npz")
    p = _write(str(tmp_path), name, g)
    v = ingest.load_raw(p, tuple(g["dims"])) if name == "f32" else ingest.load_volume(p)
    assert np.array_equal(v.data, g[f"{name}_data"]), name
    assert tuple(v.spacing) == tuple(g[f"{name}_spacing"])


@pytest.mark.gpu
def test_save_raw_roundtrip_and_batch_reader(tmp_path):
    import torch

    from paper_2112_10258_b200 import Volume
    from paper_2112_10258_b200.errors import DataError

    rng = np.random.default_rng(3)
    vols = [rng.standard_normal((12, 11, 10)).astype(np.float32) for _ in range(3)]
    paths = []
    for i, a in enumerate(vols):
        dp, hp = ingest.save_raw(Volume(a, (1.0, 2.0, 3.0)), tmp_path / f"s{i}")
        paths.append(dp)
        v = ingest.load_volume(dp)
        assert np.array_equal(v.data, a) and v.spacing == (1.0, 2.0, 3.0)
        assert np.array_equal(ingest.load_raw(ingest.save_raw(v, tmp_path / f"t{i}.f32")[0], (12, 11, 10)).data, a)
    reader = ingest.RawBatchReader((12, 11, 10), batch=4)
    dst = torch.zeros((4, 10, 11, 12), device="cuda")
    reader.submit(paths)
    torch.cuda.current_stream().wait_event(reader.to_device(dst))
    got = dst[:3].cpu().numpy()
    for i, a in enumerate(vols):
        assert np.array_equal(got[i], a.transpose(2, 1, 0))
    bad = vols[0].copy()
    bad[1, 2, 3] = np.nan
    bp = ingest.save_raw(Volume(bad), tmp_path / "bad")[0]
    reader.submit([paths[0], bp])
    with pytest.raises(DataError):
        reader.to_device(dst)
