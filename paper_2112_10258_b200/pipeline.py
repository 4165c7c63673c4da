"""End-to-end extraction on the GPU -- drop-in for volkey pipeline.py.

``extract_features`` (pipeline.py:70-102) runs the whole batch-of-one pipeline
through ``engine.Extractor``: one stream, no host round trip until the counts
are read at the end.  The returned ``ExtractionResult`` has the reference's
fields; pyramid and DoG levels stay in HBM (``DeviceVolume``) and the Python
objects (keypoints, frames, records) are built on first access.
"""

from __future__ import annotations

from functools import lru_cache

import numpy as np

from . import _lib
from . import tables as T
from .config import PipelineConfig
from .descriptor import records_from
from .detect import Keypoint
from .engine import Extractor
from .errors import DataError
from .orient import OrientationFrame
from .scalespace import DoGOctave, DoGPyramid, GaussianPyramid, PyramidOctave, _stage
from .volume import DeviceVolume, Volume, device_of


class ExtractionResult:
    """pipeline.py:20-38 (pyramid, dog, keypoints, oriented, records, drop counts)."""

    def __init__(self, pyramid, dog, keypoints=None, oriented=None, records=None, dropped_orientation=0,
                 dropped_descriptor=0, _soa=None, _kind="siftrank", _npairs=64):
        self.pyramid = pyramid
        self.dog = dog
        self._keypoints, self._oriented, self._records = keypoints, oriented, records
        self.dropped_orientation = dropped_orientation
        self.dropped_descriptor = dropped_descriptor
        self._soa, self._kind, self._npairs = _soa, _kind, _npairs

    @property
    def refined(self) -> np.ndarray | None:
        """(n_keypoints, 6) float64 sub-voxel / sub-level refinement -- x, y, z,
        sigma, dog_value, status (0 converged, 1 offset > 0.5, 2 singular) --
        when extract_features(..., refine=True); None otherwise."""
        return None if self._soa is None else self._soa.get("refined")

    @property
    def soa(self) -> dict | None:
        """Structure-of-arrays results straight from the device (no objects)."""
        return self._soa

    @property
    def keypoints(self) -> list:
        if self._keypoints is None:
            s = self._soa
            P, S, D, G = s["pos"].tolist(), s["sigma"].tolist(), s["dog"].astype(np.float64).tolist(), s["sign"].tolist()
            o, lv = s["kp"]["octave"].tolist(), s["kp"]["level"].tolist()
            self._keypoints = [Keypoint(tuple(P[i]), S[i], o[i], lv[i], D[i], "peak" if G[i] > 0 else "valley")
                               for i in range(len(S))]
        return self._keypoints

    @property
    def oriented(self) -> list:
        if self._oriented is None:
            kps = self.keypoints
            _, rot = T.default_frame_tables()
            out = []
            for k, p, q in zip(self._soa["frame_kp"].tolist(), self._soa["frame_prim"].tolist(),
                               self._soa["frame_sec"].tolist()):
                r = rot[p, q].copy()
                r.setflags(write=False)
                out.append((kps[k], OrientationFrame(r)))
            self._oriented = out
        return self._oriented

    @property
    def records(self) -> list:
        if self._records is None:
            self._records = records_from(self.oriented, self._soa["desc"], self._kind, self._npairs)
        return self._records

    @property
    def stats(self) -> dict:
        n_kp = len(self._keypoints) if self._keypoints is not None else self._soa["n_keypoints"]
        n_fr = len(self._oriented) if self._oriented is not None else self._soa["n_frames"]
        n_de = len(self._records) if self._records is not None else self._soa["n_frames"]
        return {"octaves": self.pyramid.num_octaves, "keypoints": n_kp, "frames": n_fr, "descriptors": n_de,
                "dropped": self.dropped_orientation + self.dropped_descriptor}


def assign_orientations(pyr: GaussianPyramid, keypoints: list, config: PipelineConfig, recorder=None):
    """pipeline.py:41-67: frames per keypoint (input order), zero-frame keypoints dropped."""
    from .stages import run_orientation

    rec = _stage(recorder)
    with rec("orient", -1, -1):
        out = run_orientation(pyr, keypoints, config.radius_factor, config.secondary_ratio, config.max_frames)
    _, rot = T.default_frame_tables()
    flat, dropped = [], 0
    for i, kp in enumerate(keypoints):
        nf = int(out["nframes"][i])
        if nf == 0:
            dropped += 1
            continue
        for f in range(nf):
            r = rot[out["prim"][i, f], out["sec"][i, f]].copy()
            r.setflags(write=False)
            flat.append((kp, OrientationFrame(r)))
    return flat, dropped


def _wrap_pyramids(ex: Extractor, volume: Volume):
    P, L = ex.plan, ex.cfg.levels_per_octave
    octs, dogs = [], []
    spacing = tuple(volume.spacing)
    for o in range(P.n_octaves):
        octs.append(PyramidOctave([DeviceVolume(ex.levels[o][i][0], spacing) for i in range(L)], P.sigmas[o]))
        dogs.append(DoGOctave([DeviceVolume(ex.dogs[o][i][0], spacing) for i in range(L - 1)], P.sigmas[o][:-1]))
        spacing = tuple(2.0 * s for s in spacing)
    pyr = GaussianPyramid(octs, ex.cfg.base_sigma, P.kappa, L, source=volume)
    return pyr, DoGPyramid(dogs, P.kappa, L)


class _ExtractorPool:
    """Extractors cached per (dims, config) for the drop-in API: building one
    (plan, host tables, every device buffer) costs far more than running it on
    one volume.  A returned ExtractionResult keeps views of its Extractor's
    pyramid levels, so an Extractor is reused only once the result of its
    previous call is gone (weak reference); a loop that keeps the previous
    result alive alternates between two.  At most ``cap`` per key."""

    def __init__(self, cap: int = 3):
        self.cap = cap
        self.entries: dict = {}

    def get(self, key, make):
        import weakref

        lst = self.entries.setdefault(key, [])
        for e in lst:
            if e[1] is None or e[1]() is None:
                return e
        e = [make(), None]
        if len(lst) < self.cap:
            lst.append(e)
        return e

    def clear(self):
        self.entries.clear()


_POOL = _ExtractorPool()


def clear_extractor_cache() -> None:
    """Drop the cached drop-in Extractors (frees their device memory)."""
    _POOL.clear()


def extract_features(volume: Volume, config: PipelineConfig | None = None, recorder=None, *,
                     refine: bool = False) -> ExtractionResult:
    """pipeline.py:70-102 on the GPU (Extractor cached per (dims, config)).

    refine=True (an extension, off by default: the reference reports lattice
    positions) adds ``result.refined``: per keypoint the sub-voxel / sub-level
    quadratic refinement (x, y, z, sigma, dog_value, status) of
    vk_refine_keypoints; the reference fields are unchanged."""
    import weakref

    cfg = config or PipelineConfig()
    if cfg.descriptor != "siftrank":
        from .descriptor import sample_point_pairs

        sample_point_pairs(cfg.method, cfg.pairs, 1.0, cfg.seed)  # validation order of pipeline.py:86-88
    key = (tuple(volume.dims), cfg.model_dump_json(), bool(refine))
    entry = _POOL.get(key, lambda: Extractor(volume.dims, cfg, batch=1, refine=refine))
    ex = entry[0]
    while True:
        ex.input[0].copy_(device_of(volume))
        if recorder is None and ex.graph is not None:
            ex.graph.replay()  # the cached Extractor's pipeline as one CUDA graph (~60 launches)
        else:
            ex.enqueue(rec=_stage(recorder) if recorder is not None else None)
        c = ex.check_capacity()
        if not c["overflow"]:
            break
        kp_cap = max(ex.kp_cap, c["keypoints"] + 1)
        frame_cap = max(ex.frame_cap, c["frames"] + 1)
        cand_cap = None
        if c["cand_overflow"]:
            cand_cap = int(c["cand"].max()) + 1
            kp_cap = max(kp_cap, cand_cap)
            frame_cap = max(frame_cap, kp_cap * cfg.max_frames)
        ex = Extractor(volume.dims, cfg, batch=1, kp_cap=kp_cap, frame_cap=frame_cap,
                       cand_cap=max(ex.cand_cap, cand_cap or 0), refine=refine)
        entry[0] = ex  # the grown Extractor replaces the cached one
    soa = ex.results()
    if recorder is None and ex.graph is None:
        # second call on this Extractor: capture its pipeline for the following calls
        # (Extractor.capture runs one more eager pass first; the results above are kept)
        if getattr(ex, "_dropin_calls", 0) >= 1:
            ex.capture()
        ex._dropin_calls = getattr(ex, "_dropin_calls", 0) + 1
    pyr, dog = _wrap_pyramids(ex, volume)
    res = ExtractionResult(pyr, dog, dropped_orientation=soa["dropped_orientation"], _soa=soa, _kind=cfg.descriptor,
                           _npairs=cfg.pairs)
    entry[1] = weakref.ref(res)
    return res


def extract_batch(volumes, config: PipelineConfig | None = None, extractor: Extractor | None = None):
    """Throughput API: (B, nx, ny, nz) numpy (reference layout) or a (B, nz, ny, nx)
    x-fastest CUDA tensor -> SoA results for the whole batch (volume-major)."""
    t = _lib.torch()
    cfg = config or PipelineConfig()
    if isinstance(volumes, np.ndarray):
        B, nx, ny, nz = volumes.shape
        host = t.from_numpy(np.ascontiguousarray(volumes, dtype=np.float32)).cuda()
        dev = t.empty((B, nz, ny, nx), dtype=t.float32, device="cuda")
        _lib.call("vk_transpose_zfast_to_xfast", host.data_ptr(), dev.data_ptr(), B, nx, ny, nz, _lib.stream_ptr())
    else:
        dev = volumes
        B, nz, ny, nx = dev.shape
    ex = extractor or Extractor((nx, ny, nz), cfg, batch=B)
    ex.run(dev)
    return ex.results()
