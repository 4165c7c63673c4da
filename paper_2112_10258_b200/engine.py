"""Batched GPU extraction engine: plan, device buffers, launch sequence.

``Plan`` is the host schedule of ``build_gaussian_pyramid`` /
``detect_keypoints`` / ``assign_orientations`` / ``describe_all`` for one
volume shape and one ``PipelineConfig`` (octave dims, blur taps, detection
segments, neighbourhood balls, frame tables, point pairs).  ``Extractor``
owns the device buffers for a batch of B volumes of that shape and enqueues
the whole pipeline on one CUDA stream with no host synchronisation, so a
step can be captured in a CUDA graph.  Counts (keypoints, frames) stay on the
device; ``Extractor.results()`` reads them back.

Device layout (HBM): every pyramid / DoG level is one tensor
``(B, nz, ny, nx)`` float32, x fastest; keypoints and frames are
structure-of-arrays records (include/volkey_b200.h).
"""

from __future__ import annotations

import math
from contextlib import nullcontext
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import tables as T
from .config import PipelineConfig
from .errors import DataError, ParameterError

SCALE_CALIBRATION = math.sqrt(1.5)  # detect.py:26


def _no_stage(*_a):
    return nullcontext()


def _memset(tensor, stream: int) -> None:
    """Zero a device tensor on the pipeline stream (graph-capturable)."""
    _lib.call("vk_memset_async", tensor.data_ptr(), tensor.numel() * tensor.element_size(), stream)
KIND_CODE = {"brief": 1, "rrief": 2}


def level_records(tensors, dims_list) -> np.ndarray:
    """vk_level records for batched level tensors (None -> null entry)."""
    rec = np.zeros(len(tensors), dtype=_lib.LEVEL_DTYPE)
    for i, (t, d) in enumerate(zip(tensors, dims_list)):
        if t is None:
            continue
        nx, ny, nz = d
        rec[i] = (t.data_ptr(), nx * ny * nz, nx, ny, nz, 0)
    return rec


@dataclass
class Plan:
    dims: tuple
    cfg: PipelineConfig
    kappa: float = 0.0
    local: list = field(default_factory=list)
    octave_dims: list = field(default_factory=list)
    sigmas: list = field(default_factory=list)        # absolute sigma per (octave, level)
    taps: list = field(default_factory=list)          # per level i: GaussianKernel1D (level 0 = base blur)
    seg_info: np.ndarray | None = None                 # (nseg, 4) int32
    seg_sigma: np.ndarray | None = None                # (nseg,) fp64
    balls: T.BallTable = field(default_factory=T.BallTable)

    @classmethod
    def build(cls, dims, cfg: PipelineConfig, segments: bool = True) -> "Plan":
        if cfg.base_sigma <= 0:
            raise ParameterError(f"base_sigma must be > 0, got {cfg.base_sigma}")
        if cfg.levels_per_octave < 4:
            raise ParameterError(f"levels_per_octave must be >= 4, got {cfg.levels_per_octave}")
        if cfg.num_octaves < 1:
            raise ParameterError(f"num_octaves must be >= 1, got {cfg.num_octaves}")
        p = cls(tuple(int(d) for d in dims), cfg)
        L = cfg.levels_per_octave
        p.kappa, p.local = T.octave_sigmas(cfg.base_sigma, L)
        p.taps = [T.gaussian_kernel(p.local[0])] + [
            T.gaussian_kernel(T.incremental_sigma(p.local[i - 1], p.local[i])) for i in range(1, L)]
        cur = p.dims
        p.octave_dims = [cur]
        # octave truncation rule of scalespace.py:199-203
        for o in range(cfg.num_octaves):
            if o + 1 == cfg.num_octaves:
                break
            nxt = tuple(d // 2 for d in cur)
            if min(nxt) < cfg.min_octave_dim or min(cur) < 2:
                break
            p.octave_dims.append(nxt)
            cur = nxt
        p.sigmas = [[s * 2.0 ** o for s in p.local] for o in range(len(p.octave_dims))]
        if not segments:
            return p
        nseg = len(p.octave_dims) * L
        if nseg > 128:
            raise ParameterError("num_octaves * levels_per_octave above 128 is not supported")
        p.seg_info = np.full((nseg, 4), -1, dtype=np.int32)
        p.seg_sigma = np.zeros(nseg, dtype=np.float64)
        for o in range(len(p.octave_dims)):
            scale = 2.0 ** o
            for i in range(1, L - 2):
                # level_sigma_local (detect.py:143-146); keypoint sigma (detect.py:110)
                finer = p.sigmas[o][i] / (2.0 ** o)
                sl = finer * math.sqrt(p.kappa) * SCALE_CALIBRATION
                sigma = sl * scale
                radius = cfg.radius_factor * (sigma / scale)  # orient.py:83-104
                s = o * L + i
                p.seg_info[s] = (o, i, o * L + i, p.balls.index(radius))
                p.seg_sigma[s] = sigma
        return p

    @property
    def n_octaves(self) -> int:
        return len(self.octave_dims)


class DeviceTables:
    """Per-plan constant tables resident on the device."""

    def __init__(self, plan: Plan):
        t = _lib.torch()
        cfg = plan.cfg
        self.K = 42
        dirs = T.icosphere_directions()
        ok, rot = T.default_frame_tables()
        self.dirs = t.from_numpy(np.ascontiguousarray(dirs).copy()).cuda()
        self.pair_ok = t.from_numpy(ok.copy()).cuda()
        self.rot_table = t.from_numpy(rot.reshape(-1).copy()).cuda()
        self.ico = np.ascontiguousarray(T.icosphere_structure())
        self.ico_lut = t.from_numpy(T.icosphere_lut().copy()).cuda()
        balls, off, win, planes = plan.balls.arrays()
        self.balls = _lib.to_device_records(balls)
        self.ball_offsets = t.from_numpy(off.copy()).cuda()
        self.windows = t.from_numpy(win.copy()).cuda()
        self.plane_starts = t.from_numpy(planes.copy()).cuda()
        self.windows32 = t.from_numpy(win.astype(np.float32)).cuda()
        # stencil spheres of the balls (fused orientation + SIFT-Rank, vk_orsr.cu)
        srec, srows, sent, biggest = T.sphere_tables(plan.balls.radii)
        self.sph_ball = t.from_numpy(srec.reshape(-1).copy()).cuda()
        self.sph_rows = t.from_numpy(srows.reshape(-1).copy()).cuda()
        self.sph_ent = t.from_numpy(sent.reshape(-1).copy()).cuda()
        # staging buffer: the largest stencil (fused kernel only up to 14000 floats = 56 KB:
        # with the 58 KB CTA state two CTAs fit an SM; larger balls use the separate kernels)
        self.box_cap = int(biggest)
        self.box_fits = self.box_cap <= 14000
        self.pairs = None
        self.pts = None
        if cfg.descriptor != "siftrank":
            from .descriptor import sample_point_pairs

            self.pairs = sample_point_pairs(cfg.method, cfg.pairs, 1.0, cfg.seed)
            pts = T.pair_points(self.pairs.p1, self.pairs.p2, cfg.patch_side, self.pairs.sigma_unit)
            self.pts = t.from_numpy(np.ascontiguousarray(pts).reshape(-1).copy()).cuda()
        self.grid = np.ascontiguousarray(T.patch_axis(cfg.patch_side), dtype=np.float64)
        if cfg.blur_sigma > 0:
            k = T.gaussian_kernel(cfg.blur_sigma)
            self.pre_taps, self.pre_radius = np.ascontiguousarray(k.weights), k.radius
        else:
            self.pre_taps, self.pre_radius = np.zeros(1, np.float32), 0


class Extractor:
    """Device buffers + launch sequence for B volumes of one shape and config."""

    def __init__(self, dims, cfg: PipelineConfig | None = None, batch: int = 1, kp_cap: int | None = None,
                 frame_cap: int | None = None, exact_only: bool = False, input=None, gradient_volumes: bool = False,
                 orient_field: bool = False, cand_cap: int | None = None, fused: bool | str | None = None,
                 refine: bool = False):
        t = _lib.torch()
        self.cfg = cfg or PipelineConfig()
        self.plan = Plan.build(dims, self.cfg)
        self.tables = DeviceTables(self.plan)
        self.B = int(batch)
        self.exact_only = int(bool(exact_only))
        nx, ny, nz = self.plan.dims
        vox = nx * ny * nz
        self.cand_cap = int(cand_cap or max(4096, vox // 128))
        self.kp_cap = int(kp_cap or self.B * max(2048, vox // 512))
        self.frame_cap = int(frame_cap or 2 * self.kp_cap)
        self.maxf = int(self.cfg.max_frames)
        if self.maxf > 8:
            raise ParameterError("max_frames above 8 is not supported by the device path")
        L = self.cfg.levels_per_octave
        B = self.B
        f32 = t.float32
        if input is not None:
            if tuple(input.shape) != (B, nz, ny, nx) or input.dtype != f32 or not input.is_contiguous():
                raise ParameterError(f"input must be a contiguous float32 tensor of shape {(B, nz, ny, nx)}")
            self.input = input
        else:
            self.input = t.empty((B, nz, ny, nx), dtype=f32, device="cuda")
        # (x, y)-blurred intermediate of the split blur (vk_blur3d_ws), one octave-0 level
        # with rows pitched to a multiple of 4 floats (16-byte aligned rows for the z pass)
        self.blur_work = t.empty(B * ((nx + 3) // 4 * 4) * ny * nz + 4, dtype=f32, device="cuda")  # + work counters
        self.levels, self.dogs = [], []
        for (ox, oy, oz) in self.plan.octave_dims:
            self.levels.append([t.empty((B, oz, oy, ox), dtype=f32, device="cuda") for _ in range(L)])
            self.dogs.append([t.empty((B, oz, oy, ox), dtype=f32, device="cuda") for _ in range(L - 1)])
        nseg = self.plan.n_octaves * L
        lvl_t, dog_t, dims_l = [None] * nseg, [None] * nseg, [None] * nseg
        for o, d in enumerate(self.plan.octave_dims):
            for i in range(L):
                lvl_t[o * L + i] = self.levels[o][i]
                dims_l[o * L + i] = d
                if i < L - 1:
                    dog_t[o * L + i] = self.dogs[o][i]
        self.level_table = _lib.to_device_records(level_records(lvl_t, dims_l))
        self.accum = _lib.accum_work()  # orientation / SIFT-Rank vote histograms
        # octaves from here on are small enough for the fused shared-memory kernel
        self.small_from = self.plan.n_octaves
        for o, d in enumerate(self.plan.octave_dims):
            if o > 0 and int(np.prod(d)) <= 16384 and max(k.radius for k in self.plan.taps[1:]) <= 32:
                self.small_from = o
                break
        # dense gradient volumes of the keypoint levels (orientation / SIFT-Rank fast paths)
        self.grad_levels = []  # (octave, level, g4 tensor, bin tensor)
        grec = np.zeros(nseg, dtype=_lib.GRADLEVEL_DTYPE)
        if gradient_volumes:
            for o, (ox, oy, oz) in enumerate(self.plan.octave_dims):
                for i in range(1, L - 2):
                    g4 = t.empty((B, oz, oy, ox, 4), dtype=f32, device="cuda")
                    bn = t.empty((B, oz, oy, ox), dtype=t.uint8, device="cuda")
                    self.grad_levels.append((o, i, g4, bn))
                    grec[o * L + i] = (g4.data_ptr(), bn.data_ptr(), ox * oy * oz, ox, oy, oz, 0)
        # orientation fields of the keypoint levels (vk_orient_field): per voxel the
        # fast path's |g| and exact nearest direction, shared by every keypoint's walk.
        # Off by default: measured on B200 the field walk executes 4x fewer
        # instructions but is DRAM-latency bound (2.5x over-read of the field), and
        # field + walk (~2.5 ms / 12 volumes) does not beat the fused walk (2.65 ms)
        self.field_levels = []  # (octave, level, mag tensor, bin tensor)
        if orient_field and not gradient_volumes:
            for o, (ox, oy, oz) in enumerate(self.plan.octave_dims):
                for i in range(1, L - 2):
                    mg = t.empty((B, oz, oy, ox), dtype=f32, device="cuda")
                    bn = t.empty((B, oz, oy, ox), dtype=t.uint8, device="cuda")
                    self.field_levels.append((o, i, mg, bn))
                    grec[o * L + i] = (mg.data_ptr(), bn.data_ptr(), ox * oy * oz, ox, oy, oz, 1)
        self.grad_table = _lib.to_device_records(grec)
        self.dog_table = _lib.to_device_records(level_records(dog_t, dims_l))
        self.source_table = _lib.to_device_records(level_records([self.input], [self.plan.dims]))
        i32 = t.int32
        self.cand_keys = t.empty(B * self.cand_cap, dtype=t.int64, device="cuda")
        self.cand_count = t.zeros(B, dtype=i32, device="cuda")
        self.kps = t.empty(self.kp_cap * 32, dtype=t.uint8, device="cuda")
        self.pos = t.empty(self.kp_cap * 3, dtype=t.float64, device="cuda")
        self.sigma = t.empty(self.kp_cap, dtype=t.float64, device="cuda")
        self.dogv = t.empty(self.kp_cap, dtype=f32, device="cuda")
        self.sign = t.empty(self.kp_cap, dtype=t.int8, device="cuda")
        self.vol_offset = t.zeros(B, dtype=i32, device="cuda")
        self.total = t.zeros(2, dtype=i32, device="cuda")
        self.nframes = t.zeros(self.kp_cap, dtype=i32, device="cuda")
        self.frame_first = t.zeros(self.kp_cap, dtype=i32, device="cuda")
        self.prim = t.zeros(self.kp_cap * self.maxf, dtype=i32, device="cuda")
        self.sec = t.zeros(self.kp_cap * self.maxf, dtype=i32, device="cuda")
        self.status = t.zeros(4, dtype=i32, device="cuda")  # [0] DataError bit, [1] orient fallbacks, [2] sr fallbacks
        self.frames = t.empty(self.frame_cap * 16, dtype=t.uint8, device="cuda")
        self.rot = t.empty(self.frame_cap * 9, dtype=t.float64, device="cuda")
        self.n_frames = t.zeros(1, dtype=i32, device="cuda")
        self.dropped = t.zeros(1, dtype=i32, device="cuda")
        # optional sub-voxel / sub-level refinement (vk_refine_keypoints; not a reference output)
        self.refine = bool(refine)
        self.refined = t.empty(self.kp_cap * 6, dtype=t.float64, device="cuda") if self.refine else None
        kind = self.cfg.descriptor
        if kind == "siftrank":
            self.desc = t.empty((self.frame_cap, 64), dtype=t.uint8, device="cuda")
        elif kind == "brief":
            self.desc = t.empty((self.frame_cap, (self.cfg.pairs + 7) // 8), dtype=t.uint8, device="cuda")
        else:
            self.desc = t.empty((self.frame_cap, self.cfg.pairs), dtype=t.int16, device="cuda")
        # fused orientation + SIFT-Rank (vk_orient_siftrank, stencil spheres staged in shared
        # memory): fast path, SIFT-Rank, no dense gradient / field volumes, every ball's sphere
        # within the staging cap.  Off by default (fused=None -> VK_FUSED, default 0): on B200
        # its 2 CTAs/SM (shared-memory bound) measured slower than the separate latency-bound
        # kernels at 3-4 CTAs/SM
        # fused="global" (or VK_FUSED=2): the fused kernel without the staged spheres (both walks
        # gather from global memory, the SIFT-Rank walk on L1 / L2-warm data)
        want = fused if fused is not None else {"1": True, "2": "global"}.get(os.environ.get("VK_FUSED", "0"), False)
        self.fused_stage = want is True
        self.fused = bool(want and not self.exact_only and kind == "siftrank" and not self.grad_levels
                          and not self.field_levels and (self.tables.box_fits or not self.fused_stage))
        self.desc_kp = (t.empty((self.kp_cap * self.maxf, 64), dtype=t.uint8, device="cuda") if self.fused else None)
        # volumes per pyramid chunk (enqueue_pyramid); env override for A/B runs
        self.pyr_chunk = int(os.environ.get("VK_PYR_CHUNK", "0")) or self.B
        # DoG of level pair (i-2, i-1) inside level i's (x, y) kernel (1) or in each level's z pass (0)
        self.dog_in_xy = os.environ.get("VK_DOG_IN_XY", "1") == "1"
        self.graph = None

    # ------------------------------------------------------------ pipeline
    def enqueue_pyramid(self, s: int, with_dog: bool = True, rec=None) -> None:
        """Gaussian levels with fused DoG + handoff subsample (scalespace.py:158-223)."""
        L, B, P = self.cfg.levels_per_octave, self.B, self.plan
        rec = rec or _no_stage
        handoff = L - 3
        small = self.small_from if with_dog else P.n_octaves
        # Volume chunks: every level of a chunk is produced before the next chunk starts, so
        # the level just written (the next blur's source, the DoG minuend) and the (x, y)
        # intermediate are still L2-resident when they are read again.
        ch = max(1, min(B, self.pyr_chunk))
        for c0 in range(0, B, ch):
            nb = min(ch, B - c0)
            for o, (nx, ny, nz) in enumerate(P.octave_dims):
                if o >= small:
                    break
                off = c0 * nx * ny * nz * 4
                lv, dg = self.levels[o], self.dogs[o]
                if o == 0:
                    k = P.taps[0]
                    with rec("convolution", o, 0):
                        _lib.call("vk_blur3d_ws", self.input.data_ptr() + off, lv[0].data_ptr() + off, None, None,
                                  nb, nx, ny, nz, k.weights.ctypes.data, k.radius, self.blur_work.data_ptr(),
                                  self.blur_work.numel(), s)
                for i in range(1, L):
                    k = P.taps[i]
                    half = None
                    if i == handoff and o + 1 < P.n_octaves:
                        hx, hy, hz = P.octave_dims[o + 1]
                        half = self.levels[o + 1][0].data_ptr() + c0 * hx * hy * hz * 4
                    # DoG_{i-2} = L_{i-2} - L_{i-1} is written by this level's (x, y) kernel from its staged
                    # source; only the last pair's DoG (L_{L-2} - L_{L-1}) comes from the z pass
                    fuse = self.dog_in_xy
                    dog_out = dg[i - 1].data_ptr() + off if (with_dog and (i == L - 1 or not fuse)) else None
                    prev = lv[i - 2].data_ptr() + off if (with_dog and fuse and i >= 2) else None
                    prev_dog = dg[i - 2].data_ptr() + off if (with_dog and fuse and i >= 2) else None
                    with rec("convolution", o, i):
                        _lib.call("vk_blur3d_ws2", lv[i - 1].data_ptr() + off, lv[i].data_ptr() + off, dog_out, half,
                                  prev, prev_dog, nb, nx, ny, nz, k.weights.ctypes.data, k.radius,
                                  self.blur_work.data_ptr(), self.blur_work.numel(), s)
                    # DoG and the handoff subsample are epilogues of the blur launches: their stage
                    # rows (bench.py STAGES) carry only what is left outside them, i.e. ~0
                    if with_dog:
                        with rec("dog", o, i - 1):
                            pass
                    if half is not None:
                        with rec("subsample", o, i):
                            pass
        if small < P.n_octaves:
            import ctypes as C

            n = P.n_octaves - small
            dims = np.array(P.octave_dims[small:], dtype=np.int32).reshape(-1)
            lp = (C.c_void_p * (n * L))(*[self.levels[o][i].data_ptr() for o in range(small, P.n_octaves)
                                          for i in range(L)])
            dp = (C.c_void_p * (n * L))(*[(self.dogs[o][i].data_ptr() if i < L - 1 else 0)
                                          for o in range(small, P.n_octaves) for i in range(L)])
            rad = np.array([0] + [k.radius for k in P.taps[1:]], dtype=np.int32)
            taps = np.zeros((L, 65), dtype=np.float32)
            for i in range(1, L):
                taps[i, : 2 * P.taps[i].radius + 1] = P.taps[i].weights
            with rec("convolution", small, -1):
                _lib.call("vk_small_octaves", n, L, handoff, dims.ctypes.data, C.cast(lp, C.c_void_p),
                          C.cast(dp, C.c_void_p), rad.ctypes.data, taps.ctypes.data, B, s)
            with rec("dog", small, -1):  # fused into vk_small_octaves
                pass
            if n > 1:
                with rec("subsample", small, handoff):
                    pass

    def enqueue_detect(self, s: int, rec=None) -> None:
        """detect_keypoints (detect.py:149-182) for the whole batch."""
        import ctypes as C

        L, P, cfg = self.cfg.levels_per_octave, self.plan, self.cfg
        rec = rec or _no_stage
        _memset(self.cand_count, s)
        cmin = float(np.float32(cfg.contrast_min))
        for o, (nx, ny, nz) in enumerate(P.octave_dims):
            ptrs = (C.c_void_p * (L - 1))(*[d.data_ptr() for d in self.dogs[o]])
            with rec("peak_detect", o, -1):
                _lib.call("vk_detect_octave", C.cast(ptrs, C.c_void_p), L - 1, self.B, nx, ny, nz, o * L,
                          cfg.threshold_band, cmin, self.cand_keys.data_ptr(), self.cand_count.data_ptr(),
                          self.cand_cap, s)
        seg = np.ascontiguousarray(P.seg_info)
        sig = np.ascontiguousarray(P.seg_sigma)
        _lib.call("vk_order_keypoints", self.cand_keys.data_ptr(), self.cand_count.data_ptr(), self.B,
                  self.cand_cap, seg.ctypes.data, sig.ctypes.data, len(sig), self.dog_table.data_ptr(),
                  self.kps.data_ptr(), self.pos.data_ptr(), self.sigma.data_ptr(), self.dogv.data_ptr(),
                  self.sign.data_ptr(), self.vol_offset.data_ptr(), self.total.data_ptr(), self.kp_cap, s)
        if self.refine:
            _lib.call("vk_refine_keypoints", self.kps.data_ptr(), self.total.data_ptr(), self.kp_cap,
                      self.dog_table.data_ptr(), cfg.levels_per_octave, float(P.kappa), self.sigma.data_ptr(),
                      self.refined.data_ptr(), s)

    def enqueue_gradients(self, s: int) -> None:
        """Dense gradient / nearest-direction volumes of the keypoint levels."""
        tb = self.tables
        for o, i, g4, bn in self.grad_levels:
            nx, ny, nz = self.plan.octave_dims[o]
            _lib.call("vk_gradient_volume", self.levels[o][i].data_ptr(), g4.data_ptr(), bn.data_ptr(), self.B, nx, ny,
                      nz, tb.dirs.data_ptr(), tb.ico.ctypes.data, s)

    def _grads_ptr(self):
        """The gradient / field level table, or NULL when no level has one (the walk kernels
        then take their default fast path, split into interior and border launches)."""
        return self.grad_table.data_ptr() if (self.grad_levels or self.field_levels) else None

    def enqueue_orient(self, s: int) -> None:
        """assign_orientations (pipeline.py:41-67)."""
        tb, cfg = self.tables, self.cfg
        _memset(self.status, s)
        if not self.exact_only:
            for o, i, mg, bn in self.field_levels:
                nx, ny, nz = self.plan.octave_dims[o]
                _lib.call("vk_orient_field", self.levels[o][i].data_ptr(), mg.data_ptr(), bn.data_ptr(), self.B, nx,
                          ny, nz, tb.dirs.data_ptr(), tb.ico.ctypes.data, tb.ico_lut.data_ptr(), s)
        _lib.call("vk_orient", self.kps.data_ptr(), self.total.data_ptr(), self.kp_cap, self.level_table.data_ptr(),
                  tb.balls.data_ptr(), tb.ball_offsets.data_ptr(), tb.windows.data_ptr(), tb.windows32.data_ptr(),
                  tb.dirs.data_ptr(), tb.K,
                  tb.pair_ok.data_ptr(), float(cfg.secondary_ratio), self.maxf, None, self.nframes.data_ptr(),
                  self.prim.data_ptr(), self.sec.data_ptr(), self.status.data_ptr(), self.exact_only,
                  tb.ico.ctypes.data, tb.ico_lut.data_ptr(), self._grads_ptr(), self.accum.data_ptr(), s)
        _lib.call("vk_expand_frames", self.nframes.data_ptr(), self.prim.data_ptr(), self.sec.data_ptr(),
                  self.total.data_ptr(), self.kp_cap, self.maxf, tb.rot_table.data_ptr(), tb.K,
                  self.frames.data_ptr(), self.rot.data_ptr(), self.n_frames.data_ptr(), self.dropped.data_ptr(),
                  self.frame_cap, self.frame_first.data_ptr(), s)

    def enqueue_orient_describe(self, s: int) -> None:
        """assign_orientations + describe_all for SIFT-Rank in one kernel
        (pipeline.py:41-67, descriptor.py:227-306): frames per keypoint and
        their rank vectors, then the frame expansion and the row scatter into
        frame order."""
        tb, cfg = self.tables, self.cfg
        _memset(self.status, s)
        _lib.call("vk_orient_siftrank", self.kps.data_ptr(), self.total.data_ptr(), self.kp_cap,
                  self.level_table.data_ptr(), tb.balls.data_ptr(), tb.ball_offsets.data_ptr(), tb.windows.data_ptr(),
                  tb.windows32.data_ptr(), tb.dirs.data_ptr(), tb.K, tb.pair_ok.data_ptr(), float(cfg.secondary_ratio),
                  self.maxf, tb.rot_table.data_ptr(), self.nframes.data_ptr(), self.prim.data_ptr(),
                  self.sec.data_ptr(), self.desc_kp.data_ptr(), self.status.data_ptr(), tb.ico.ctypes.data,
                  tb.ico_lut.data_ptr(), tb.sph_ball.data_ptr(), tb.sph_rows.data_ptr(), tb.sph_ent.data_ptr(),
                  tb.box_cap if self.fused_stage else 0, self.accum.data_ptr(), s)
        _lib.call("vk_expand_frames", self.nframes.data_ptr(), self.prim.data_ptr(), self.sec.data_ptr(),
                  self.total.data_ptr(), self.kp_cap, self.maxf, tb.rot_table.data_ptr(), tb.K,
                  self.frames.data_ptr(), self.rot.data_ptr(), self.n_frames.data_ptr(), self.dropped.data_ptr(),
                  self.frame_cap, self.frame_first.data_ptr(), s)
        _lib.call("vk_scatter_frame_rows", self.frames.data_ptr(), self.frame_first.data_ptr(),
                  self.n_frames.data_ptr(), self.frame_cap, self.maxf, self.desc_kp.data_ptr(), self.desc.data_ptr(), s)

    def enqueue_describe(self, s: int) -> None:
        """describe_all (descriptor.py:266-306)."""
        tb, cfg = self.tables, self.cfg
        if cfg.descriptor == "siftrank":
            # one work item per keypoint: its frames are contiguous from frame_first[i]
            _lib.call("vk_describe_siftrank", self.frames.data_ptr(), self.rot.data_ptr(), self.frame_first.data_ptr(),
                      self.nframes.data_ptr(), self.total.data_ptr(), self.kp_cap, self.maxf, self.kps.data_ptr(),
                      self.level_table.data_ptr(), tb.balls.data_ptr(), tb.ball_offsets.data_ptr(),
                      self.desc.data_ptr(), self.exact_only, self.status.data_ptr() + 8,
                      self._grads_ptr(), self.accum.data_ptr(), s)
        else:
            code = KIND_CODE[cfg.descriptor]
            _lib.call("vk_describe_patch", code, self.frames.data_ptr(), self.rot.data_ptr(),
                      self.n_frames.data_ptr(), self.frame_cap, self.kps.data_ptr(), self.pos.data_ptr(),
                      self.sigma.data_ptr(), self.source_table.data_ptr(), cfg.patch_side, tb.grid.ctypes.data,
                      tb.pre_taps.ctypes.data, tb.pre_radius, tb.pts.data_ptr(), cfg.pairs,
                      self.desc.data_ptr() if code == 1 else None, self.desc.data_ptr() if code == 2 else None, s)

    def enqueue(self, stream=None, rec=None) -> None:
        s = _lib.stream_ptr(stream)
        rec = rec or _no_stage
        self.enqueue_pyramid(s, rec=rec)
        self.enqueue_detect(s, rec=rec)
        if self.grad_levels:  # optional dense gradient volumes (not a reference stage)
            with rec("gradients", -1, -1):
                self.enqueue_gradients(s)
        if self.fused:
            with rec("orient", -1, -1):  # one kernel: its time is the orient row
                self.enqueue_orient_describe(s)
            with rec("descriptor", -1, -1):
                pass
            return
        with rec("orient", -1, -1):
            self.enqueue_orient(s)
        with rec("descriptor", -1, -1):
            self.enqueue_describe(s)

    def run(self, volumes=None, stream=None) -> None:
        """Copy ``volumes`` (B, nz, ny, nx) into the input buffer (if given) and
        enqueue one full extraction; replays the CUDA graph if captured."""
        if volumes is not None:
            self.input.copy_(volumes, non_blocking=True)
        if self.graph is not None:
            self.graph.replay()
        else:
            self.enqueue(stream)

    def capture(self) -> None:
        """Capture one extraction step into a CUDA graph (after a warm-up run)."""
        t = _lib.torch()
        s = t.cuda.Stream()
        s.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(s):
            self.enqueue(s)
        t.cuda.current_stream().wait_stream(s)
        t.cuda.synchronize()
        g = t.cuda.CUDAGraph()
        with t.cuda.graph(g, stream=s):
            self.enqueue(s)
        t.cuda.synchronize()
        self.graph = g

    # ------------------------------------------------------------- results
    def counts(self) -> dict:
        tot = self.total.cpu().numpy()
        nf = int(self.n_frames.cpu().item())
        stv = self.status.cpu().numpy()
        st = int(stv[0])
        return dict(keypoints=int(tot[0]), cand_overflow=bool(tot[1]), frames=nf, status=st,
                    orient_fallbacks=int(stv[1]), siftrank_fallbacks=int(stv[2]),
                    dropped=int(self.dropped.cpu().item()), cand=self.cand_count.cpu().numpy())

    def check_capacity(self) -> dict:
        c = self.counts()
        if c["status"] & 1:
            raise DataError("orientation neighborhood lies entirely outside the volume")
        c["overflow"] = c["cand_overflow"] or c["keypoints"] > self.kp_cap or c["frames"] > self.frame_cap
        return c

    def results(self) -> dict:
        """Host copies of the keypoint / frame / descriptor SoA (volume-major)."""
        c = self.check_capacity()
        if c["overflow"]:
            raise ParameterError("device capacity exceeded; rebuild the Extractor with larger caps")
        n, m = c["keypoints"], c["frames"]
        kps = self.kps[: n * 32].cpu().numpy().view(_lib.KP_DTYPE)
        fr = self.frames[: m * 16].cpu().numpy().view(_lib.FRAME_DTYPE)
        return dict(
            n_keypoints=n, n_frames=m, dropped_orientation=c["dropped"],
            kp=kps, pos=self.pos[: 3 * n].cpu().numpy().reshape(n, 3), sigma=self.sigma[:n].cpu().numpy(),
            dog=self.dogv[:n].cpu().numpy(), sign=self.sign[:n].cpu().numpy(),
            vol_offset=self.vol_offset.cpu().numpy(), frame_kp=fr["kp"].copy(), frame_prim=fr["prim"].copy(),
            frame_sec=fr["sec"].copy(), rot=self.rot[: 9 * m].cpu().numpy().reshape(m, 3, 3),
            desc=self.desc[:m].cpu().numpy(),
            refined=self.refined[: 6 * n].cpu().numpy().reshape(n, 6) if self.refine else None,
        )


class ExtractorGroup:
    """Several Extractors (sub-batches) whose pipelines run on parallel streams
    inside one CUDA graph: the tails and the latency-bound small-octave /
    bookkeeping launches of one sub-batch overlap the bulk work of the others."""

    def __init__(self, extractors: list):
        if not extractors:
            raise ParameterError("ExtractorGroup needs at least one Extractor")
        self.members = list(extractors)
        self.graph = None

    @property
    def B(self) -> int:
        return sum(e.B for e in self.members)

    def enqueue(self, stream=None) -> None:
        t = _lib.torch()
        main = stream if stream is not None else t.cuda.current_stream()
        subs = [t.cuda.Stream() for _ in self.members]
        for sub, ex in zip(subs, self.members):
            sub.wait_stream(main)
            with t.cuda.stream(sub):
                ex.enqueue(sub)
        for sub in subs:
            main.wait_stream(sub)

    def run(self) -> None:
        if self.graph is not None:
            self.graph.replay()
        else:
            self.enqueue()

    def capture(self) -> None:
        t = _lib.torch()
        s = t.cuda.Stream()
        s.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(s):
            self.enqueue(s)
        t.cuda.current_stream().wait_stream(s)
        t.cuda.synchronize()
        g = t.cuda.CUDAGraph()
        with t.cuda.graph(g, stream=s):
            self.enqueue(s)
        t.cuda.synchronize()
        self.graph = g
