#!/usr/bin/env python
"""Benchmark: volumes/s for 145x174x145 detect + describe (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B] [--impl ours|reference]

One step = one batch of B synthetic 145x174x145 volumes per GPU through the
whole hot path (Gaussian pyramid + DoG + 80-neighbour detection + orientation
+ SIFT-Rank descriptors), replayed as one CUDA graph.  Inputs are resident in
HBM before the timed region; consecutive steps read different input slots
(S*B*14.6 MB > L2), so no step starts with its input in L2.  Multi-GPU: one
process per GPU (torchrun), each rank its own volumes, no collective in the
data path (weak scaling); timing is CUDA events on the pipeline stream, max
over ranks.  Rank 0 prints one JSON line.

``--impl reference`` times the reference on the host cores instead: the
unmodified volkey package staged into oracle/_ref by oracle/make_ref.py (it
travels to the GPU box with the snapshot), one full volume per
single-threaded process, all cores concurrently.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

DIMS = (145, 174, 145)
with open(os.path.join(REPO, "BASELINE.json")) as _fh:
    METRIC = json.load(_fh)["metric"]
UNIT = "volumes/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=64, help="volumes per GPU per step")
    ap.add_argument("--streams", type=int, default=8, help="parallel sub-batches (streams) per GPU")
    ap.add_argument("--slots", type=int, default=2, help="distinct input batches cycled over steps")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--backend", default="nccl", choices=("nccl", "gloo"),
                    help="process-group backend for N > 1 (gloo: several ranks sharing one GPU, tests only)")
    ap.add_argument("--descriptor", default="siftrank", choices=("siftrank", "brief", "rrief"))
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-matching", action="store_true", help="skip the descriptor-matching side measurement")
    ap.add_argument("--no-extras", action="store_true", help="skip the drop-in API latency and configs[3] lines")
    ap.add_argument("--ref-steps", type=int, default=2, help="cap on timed reference steps (each ~30 s)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc, self.thread = gpu, [], None, None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = set()
        for r in self.rows:
            if len(r) < 9:
                continue
            for n, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------ algorithmic bytes
def pyramid_bytes(plan) -> int:
    """Compulsory HBM bytes of the fused pyramid per volume: every Gaussian
    level read once + written once, every DoG level written once, the handoff
    subsample written once (SURVEY.md §8(d) minus the detection read)."""
    L = plan.cfg.levels_per_octave
    total = 0
    for o, d in enumerate(plan.octave_dims):
        n = int(np.prod(d))
        if o == 0:
            total += 8 * n                      # input -> level 0
        total += (L - 1) * 12 * n               # read prev, write level, write DoG
        if o + 1 < plan.n_octaves:
            total += 4 * int(np.prod(plan.octave_dims[o + 1]))
    return total


def ncu_pyramid_traffic(batch: int):
    """DRAM bytes (read + write) of all blur3d launches of one step, from the
    committed ncu capture (profiles/*/pyramid_dram.csv, batch noted in its
    companion log), scaled to `batch` volumes; (bytes, source) or (None, None)."""
    import csv
    import glob

    paths = sorted(glob.glob(os.path.join(REPO, "profiles", "r*", "pyramid_dram.csv")))
    if not paths:
        return None, None
    path = paths[-1]
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r]
    if not hi:
        return None, None
    h = rows[hi[0]]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = 0.0
    for r in rows[hi[0] + 1:]:
        if len(r) > vi and "blur" in r[ki] and r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            tot += float(r[vi].replace(",", ""))
    # the capture's batch: scripts/profile_step.py prints "batch=N" (older logs: the
    # per-volume candidate-count array of its counts() line has one entry per volume)
    log = path[:-4] + ".log"
    captured_batch = None
    if os.path.exists(log):
        import re

        txt = open(log).read()
        m = re.search(r"batch=(\d+)", txt)
        if m:
            captured_batch = int(m.group(1))
        else:
            m = re.search(r"'cand': array\(\[([^\]]*)\]", txt)
            if m:
                captured_batch = len([v for v in m.group(1).replace("\n", " ").split(",") if v.strip()])
    if not captured_batch:
        return None, None
    return tot * batch / captured_batch, os.path.relpath(path, REPO)


def ncu_blur_kernel_dram(peak_gbs):
    """Per blur-kernel class, from the same committed capture: DRAM bytes moved
    per second of kernel time (serialised launches, cold cache) -- how close the
    kernels run to the HBM peak on the traffic they actually move, beside the
    stage roofline on compulsory bytes.  {class: {gbs, frac}} or None."""
    import csv
    import glob

    paths = sorted(glob.glob(os.path.join(REPO, "profiles", "r*", "pyramid_dram.csv")))
    if not paths:
        return None
    rows = list(csv.reader(open(paths[-1])))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r]
    if not hi:
        return None
    h = rows[hi[0]]
    ii, ki, mi, vi = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    per = {}
    for r in rows[hi[0] + 1:]:
        if len(r) > vi and "blur" in r[ki]:
            cls = r[ki].split("(")[0].split("<")[0].replace("void ", "").strip()
            d = per.setdefault((r[ii], cls), {})
            d[r[mi]] = float(r[vi].replace(",", ""))
    agg = {}
    for (_, cls), d in per.items():
        a = agg.setdefault(cls, [0.0, 0.0])
        a[0] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        a[1] += d.get("gpu__time_duration.sum", 0.0)  # ns
    out = {}
    for cls, (b, t) in agg.items():
        if t > 0:
            gbs = b / t  # bytes per ns == GB/s
            out[cls] = {"dram_gbs": round(gbs, 1), "frac": round(gbs / peak_gbs, 3) if peak_gbs else None}
    return out or None


def _concurrent_pyramid(plan, volumes, ms, peak_gbs):
    """Pyramid stage of all sub-batches of one step on parallel streams (as in the step)."""
    gbs = pyramid_bytes(plan) * volumes / (ms / 1e3) / 1e9
    return {"volumes": volumes, "ms": round(ms, 4), "achieved": round(gbs, 1),
            "frac": round(gbs / peak_gbs, 4) if peak_gbs else None,
            "note": "the per-step pyramid of every sub-batch on its own stream (eager, CUDA events)"}


def detect_bytes(plan) -> int:
    """Detection reads each of the L-1 DoG levels once per octave."""
    L = plan.cfg.levels_per_octave
    return sum((L - 1) * 4 * int(np.prod(d)) for d in plan.octave_dims)


# ------------------------------------------------------------ CPU reference
REF_DIR = os.path.join(REPO, "oracle", "_ref")  # staged by oracle/make_ref.py (unmodified reference copy)


def ref_available() -> bool:
    return os.path.isfile(os.path.join(REF_DIR, "volkey", "pipeline.py"))


def _cpu_worker(args):
    """One full volume through the CPU path in this (spawned) process:
    impl "reference" = the unmodified volkey.extract_features (pipeline.py:70-102)
    from oracle/_ref with PipelineConfig(workers=1); impl "port" = the numpy
    restatement oracle/volkey_oracle.py."""
    seed, kind, barrier, impl = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    import threadpoolctl

    from paper_2112_10258_b200 import synthetic

    with threadpoolctl.threadpool_limits(1):
        base = synthetic.brain_volume()
        vol = synthetic.batch_from(base, 1, seed=seed)[0] if seed else base
        warm = np.ones((24, 24, 24), np.float32) * np.arange(24, dtype=np.float32)
        if impl == "reference":
            sys.path.insert(0, REF_DIR)
            import volkey

            cfg = volkey.PipelineConfig(descriptor=kind, workers=1)
            run = lambda v: volkey.extract_features(volkey.Volume(v), cfg)  # noqa: E731
            count = lambda r: (len(r.keypoints), len(r.records))  # noqa: E731
        else:
            from oracle import volkey_oracle as O

            run = lambda v: O.extract(v, descriptor=kind)  # noqa: E731
            count = lambda r: (len(r["keypoints"]), len(r["records"]))  # noqa: E731
        run(warm)
        if barrier is not None:
            barrier.wait()
        t0 = time.time()
        res = run(vol)
        t1 = time.time()
    nk, nr = count(res)
    return t0, t1, nk, nr


def cpu_volumes_per_s(kind: str, procs: int, steps: int, impl: str):
    """CPU path on the host cores: `procs` concurrent single-threaded
    processes, one full volume each per step.  Returns (volumes/s, details)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    times, kps = [], []
    for s in range(steps):
        if procs == 1:
            r = [_cpu_worker((s, kind, None, impl))]
        else:
            with ctx.Manager() as mgr:
                bar = mgr.Barrier(procs)
                with ctx.Pool(procs) as pool:
                    r = pool.map(_cpu_worker, [(s * procs + i, kind, bar, impl) for i in range(procs)])
        start, end = min(x[0] for x in r), max(x[1] for x in r)
        times.append(end - start)
        kps += [x[2] for x in r]
    return procs * steps / sum(times), dict(step_s=times, keypoints=kps)


# ---------------------------------------------------------------- ours
def run_ours(a):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    dev_index = local % max(1, torch.cuda.device_count())  # gloo tests run several ranks on one GPU
    torch.cuda.set_device(dev_index)
    if world > 1:
        if a.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group("gloo")

    def max_over_ranks(v: float) -> float:
        # the driver's contract: time on the device per rank, report the max over ranks
        t = torch.tensor([v], device="cuda" if a.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    import paper_2112_10258_b200 as vk
    from paper_2112_10258_b200 import _lib, synthetic
    from paper_2112_10258_b200.engine import Extractor

    cfg = vk.PipelineConfig(descriptor=a.descriptor)
    B, S = a.batch, max(1, a.slots)
    # ---- inputs: distinct volumes per rank and slot, resident in HBM (x fastest)
    base = synthetic.brain_volume()
    host = synthetic.batch_from(base, B * S, seed=1000 + rank)            # (B*S, nx, ny, nz)
    dev_in = torch.empty((B * S,) + DIMS[::-1], dtype=torch.float32, device="cuda")
    tmp = torch.from_numpy(host).cuda()
    _lib.call("vk_transpose_zfast_to_xfast", tmp.data_ptr(), dev_in.data_ptr(), B * S, *DIMS, _lib.stream_ptr())
    del tmp
    pinned = torch.from_numpy(np.ascontiguousarray(host.transpose(0, 3, 2, 1))).pin_memory()  # x-fastest host copy
    del host
    # ---- one extractor group per slot: G parallel-stream sub-batches reading the resident slot
    from paper_2112_10258_b200.engine import ExtractorGroup

    G = max(1, min(a.streams, B))
    subs = [B * g // G for g in range(G + 1)]
    groups = []
    for s_ in range(S):
        members = []
        for g in range(G):
            lo, hi = s_ * B + subs[g], s_ * B + subs[g + 1]
            members.append(Extractor(DIMS, cfg, batch=hi - lo, input=dev_in[lo:hi]))
        groups.append(ExtractorGroup(members))
    # capacity check on a first eager run, grow buffers if needed
    for grp in groups:
        for i, ex in enumerate(grp.members):
            ex.enqueue()
            c = ex.check_capacity()
            if c["overflow"]:
                ex2 = Extractor(DIMS, cfg, batch=ex.B, kp_cap=2 * c["keypoints"] + 1024,
                                frame_cap=2 * c["frames"] + 1024, input=ex.input)
                grp.members[i] = ex2
                ex2.enqueue()
    torch.cuda.synchronize()
    exs = [grp.members[0] for grp in groups]
    counts = {k: sum(m.counts()[k] for m in groups[0].members) for k in ("keypoints", "frames")}
    # ---- cross-rank parity: every rank extracts the same two
    # volumes -- the first two of tests/golden/bench.npz, made by the unmodified
    # reference -- and the per-volume digests (tests/golden/digest.py) are
    # all-gathered: every GPU's outputs must equal each other AND the reference's
    chk = Extractor(DIMS, cfg, batch=2)
    chk.input.copy_(torch.from_numpy(np.ascontiguousarray(
        synthetic.batch_from(base, 2, seed=1000).transpose(0, 3, 2, 1))).cuda())
    chk.enqueue()
    rc = chk.results()
    sys.path.insert(0, os.path.join(REPO, "tests", "golden"))
    from digest import digest_results

    vd = [digest_results(rc, v) for v in range(2)]
    digest = hashlib.sha256(json.dumps(vd, sort_keys=True).encode()).hexdigest()
    digests = [digest]
    if world > 1:
        digests = [None] * world
        dist.all_gather_object(digests, digest)
    rank_parity = {"checked_volumes": 2, "keypoints": int(rc["n_keypoints"]), "digest": digest[:16],
                   "ranks": world, "all_ranks_equal": len(set(digests)) == 1}
    gpath = os.path.join(REPO, "tests", "golden", "bench.npz")
    if cfg.descriptor == "siftrank" and os.path.exists(gpath):
        g = np.load(gpath)
        rank_parity["matches_reference"] = all(
            d[k] == (int(g[f"bench{v}_{k}"]) if k.startswith("n_") else str(g[f"bench{v}_{k}"]))
            for v, d in enumerate(vd) for k in ("n_kp", "n_fr", "kp", "fr", "desc"))
        rank_parity["reference"] = "tests/golden/bench.npz (unmodified volkey, make_bench_golden.py)"
    del chk, rc
    launches0 = _lib.load().vk_launch_count()
    groups[0].enqueue()
    torch.cuda.synchronize()
    launches_per_step = _lib.load().vk_launch_count() - launches0
    # ---- per-stage device times of one sub-batch: each stage captured in its own CUDA graph and
    # replayed in pipeline order (as the step runs it: no host launch gaps), CUDA events between the
    # replays; the eager per-launch figures are reported beside them
    st = torch.cuda.current_stream()
    names = ("pyramid", "detect", "gradients", "orient", "describe")
    ex = exs[0]
    fns = (ex.enqueue_pyramid, ex.enqueue_detect, ex.enqueue_gradients, ex.enqueue_orient, ex.enqueue_describe)
    stage_graphs = []
    cap = torch.cuda.Stream()
    cap.wait_stream(st)
    for k, fn in zip(names, fns):
        if k == "gradients" and not ex.grad_levels:
            stage_graphs.append(None)  # no launches
            continue
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            fn(cap.cuda_stream)
        stage_graphs.append(g)
    st.wait_stream(cap)
    torch.cuda.synchronize()

    def time_stages(run_stage):
        ms = {k: [] for k in names}
        for _ in range(5):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
            ev[0].record(st)
            for i in range(len(names)):
                run_stage(i)
                ev[i + 1].record(st)
            torch.cuda.synchronize()
            for k, (e0, e1) in zip(names, zip(ev[:-1], ev[1:])):
                ms[k].append(e0.elapsed_time(e1))
        return {k: statistics.median(v) for k, v in ms.items()}

    def graph_stage(i):
        if stage_graphs[i] is not None:
            stage_graphs[i].replay()

    stage_ms_eager = time_stages(lambda i: fns[i](st.cuda_stream))
    stage_ms = time_stages(graph_stage)
    del stage_graphs
    # the pyramid stage of a whole step as the step runs it: the G sub-batch pyramids on G
    # parallel streams (eager, CUDA events on the joining stream), compulsory bytes of all B volumes
    conc_ms = []
    for _ in range(3):
        subs_s = [torch.cuda.Stream() for _ in groups[0].members]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for ss, ex in zip(subs_s, groups[0].members):
            ss.wait_stream(st)
            ex.enqueue_pyramid(ss.cuda_stream)
        for ss in subs_s:
            st.wait_stream(ss)
        e1.record(st)
        torch.cuda.synchronize()
        conc_ms.append(e0.elapsed_time(e1))
    pyramid_concurrent_ms = statistics.median(conc_ms)
    # ball-voxel visits of the timed sub-batch (orientation / SIFT-Rank work units)
    r0 = exs[0].results()
    bcount = exs[0].tables.balls.cpu().numpy().view(_lib.BALL_DTYPE)["count"].astype(np.int64)
    kp_visits = bcount[r0["kp"]["ball"]]
    frames_per_kp = np.bincount(r0["frame_kp"], minlength=len(kp_visits))
    walk = {"orient_visits": int(kp_visits.sum()), "siftrank_visit_frames": int((kp_visits * frames_per_kp).sum()),
            "note": "ball voxels per keypoint (incl. the few outside the volume) on the timed sub-batch"}
    walk["orient_visits_per_s"] = round(walk["orient_visits"] / (stage_ms["orient"] / 1e3))
    walk["siftrank_visit_frames_per_s"] = round(walk["siftrank_visit_frames"] / (stage_ms["describe"] / 1e3))
    # ---- graphs
    use_graph = not a.no_graph
    if use_graph:
        for grp in groups:
            grp.capture()
    # ---- warmup + timed region
    for w in range(a.warmup):
        groups[w % S].run()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(dev_index)
    clocks.start()
    time.sleep(0.3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for k in range(a.steps):
        groups[k % S].run()
    e1.record(st)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        dist.barrier()
        ms = max_over_ranks(ms)
    value = world * B * a.steps / (ms / 1e3)

    # ---- end to end through the public API: pinned host -> HBM -> results -> host.
    # Every step copies its own volumes in (H2D on a copy stream, into the
    # input slot the previous step is not using, so it overlaps that step's
    # compute) and reads its keypoint / frame / descriptor SoA back (D2H).
    e2e = None
    if not a.no_e2e:
        h2d = B * int(np.prod(DIMS)) * 4
        d2h_tot = 0
        copy = torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in range(S)]
        ev_done = [torch.cuda.Event() for _ in range(S)]

        diag = os.environ.get("VK_E2E_DIAG", "")  # diagnostics only: "no_h2d" / "no_rb" (not a bench value)

        def stage(slot):  # step data of `slot` -> that group's input buffers
            if diag == "no_h2d":
                ev_in[slot].record(copy)
                return
            with torch.cuda.stream(copy):
                copy.wait_event(ev_done[slot])
                for g, m in enumerate(groups[slot].members):
                    m.input.copy_(pinned[slot * B + subs[g]: slot * B + subs[g + 1]], non_blocking=True)
                ev_in[slot].record(copy)

        rb = torch.cuda.Stream()

        def read_back(slot):
            # D2H on its own stream, ordered after that step only (not after the
            # step now running on the compute stream)
            nonlocal d2h_tot
            if diag == "no_rb":
                return
            with torch.cuda.stream(rb):
                rb.wait_event(ev_done[slot])
                for m in groups[slot].members:   # counts, then exactly the produced SoA to host
                    r = m.results()
                    d2h_tot += 16 + sum(v.nbytes for v in r.values() if isinstance(v, np.ndarray))

        def run_steps(n):
            # step k's results are read back while step k+1 computes (S >= 2 slots)
            stage(0)
            for k in range(n):
                slot = k % S
                st.wait_event(ev_in[slot])
                groups[slot].run()
                ev_done[slot].record(st)
                if k + 1 < n:
                    stage((k + 1) % S)
                if k > 0:
                    read_back((k - 1) % S)
            read_back((n - 1) % S)

        run_steps(max(1, a.warmup))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        d2h_tot = 0
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(st)
        run_steps(a.steps)
        f1.record(st)
        torch.cuda.synchronize()
        ems = f0.elapsed_time(f1)
        if world > 1:
            ems = max_over_ranks(ems)
        e2e = {"value": world * B * a.steps / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int(d2h_tot / a.steps), "ms_per_step": ems / a.steps,
               "path": "ExtractorGroup.run() per step on volumes copied in from pinned host memory (H2D on a copy "
                       "stream, double-buffered input slots) + Extractor.results() of every step (SoA to host, read "
                       "while the next step computes)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    plan = exs[0].plan
    Bs = exs[0].B  # stage timings / roofline are measured on one sub-batch
    with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
        peaks = json.load(fh)
    pbytes = pyramid_bytes(plan) * Bs
    achieved = pbytes / (stage_ms["pyramid"] / 1e3) / 1e9
    traffic, tsrc = ncu_pyramid_traffic(Bs)
    roofline = {"bound": "hbm", "kernel": "blur_xy_plane_kernel + blur_zt_kernel (split separable blur, fused DoG + "
                                          "subsample), all pyramid launches",
                "achieved": round(achieved, 1), "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                "frac": round(achieved / peaks["hbm_gbs"], 4) if peaks.get("hbm_gbs") else None,
                "traffic": round(traffic) if traffic else None, "traffic_source": tsrc,
                "kernel_dram": ncu_blur_kernel_dram(peaks.get("hbm_gbs")),
                "concurrent": _concurrent_pyramid(plan, B, pyramid_concurrent_ms, peaks.get("hbm_gbs")),
                "algorithmic_bytes": pbytes,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, burst)"}
    det_gbs = detect_bytes(plan) * Bs / (stage_ms["detect"] / 1e3) / 1e9
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 (pyramid, detection) + f64 (orientation, descriptors)",
        "data": "synthetic (reference kernel-soup phantom, seed 20240817, flipped/shifted + fresh noise per volume)",
        "config": {"workload": f"configs[2]-style batch: {B} x 145x174x145 volumes per GPU per step, detect + "
                               f"describe ({a.descriptor}), defaults of PipelineConfig",
                   "volume": list(DIMS), "batch_per_gpu": B, "descriptor": a.descriptor,
                   "l2_policy": f"inputs larger than L2: {S} resident input slots x {B} volumes x 14.6 MB cycled",
                   "streams_per_gpu": G, "stage_timing_subbatch": Bs,
                   "cuda_graph": use_graph, "parallelism": f"dp{world} (independent volumes, no collective)",
                   **({"backend": a.backend} if world > 1 else {})},
        "roofline": roofline,
        "stages_ms_per_step": {k: round(v, 4) for k, v in stage_ms.items()},
        "stages_ms_eager": {k: round(v, 4) for k, v in stage_ms_eager.items()},
        "detect_gbs": round(det_gbs, 1),
        "walks": walk,
        "rank_parity": rank_parity,
        "keypoints_per_volume": counts["keypoints"] / B, "frames_per_volume": counts["frames"] / B,
        "roofline_note": "pyramid stage of one sub-batch of stage_timing_subbatch volumes, its launches replayed from a "
                         "CUDA graph as the step runs them (eager per-launch timing: stages_ms_eager)",
        "gpu_launches": int(launches_per_step * a.steps),
        "clocks": clk,
    }
    if e2e:
        out["e2e"] = e2e
    if not a.no_matching:
        out["matching"] = bench_matching()
    if not a.no_extras:
        out["dropin"] = bench_dropin()
        out["configs3"] = bench_configs3()
    if world == 1 and not a.no_cpu_baseline:
        impl = "reference" if ref_available() else "port"
        vps, det = cpu_volumes_per_s(a.descriptor, 1, 1, impl)
        src = ("the unmodified reference volkey.extract_features (oracle/_ref, staged by oracle/make_ref.py), "
               "PipelineConfig(workers=1)" if impl == "reference" else
               "oracle/volkey_oracle.py (numpy restatement; oracle/_ref not staged)")
        out["cpu_baseline"] = {"value": round(vps, 5), "unit": UNIT, "cores": 1, "kind": impl,
                               "sample": f"1 full 145x174x145 volume through {src}, 1 thread, OPENBLAS_NUM_THREADS=1",
                               "seconds": det["step_s"]}
        if impl == "reference" and os.environ.get("VK_BENCH_PORT", "1") != "0":
            pv, pd = cpu_volumes_per_s(a.descriptor, 1, 1, "port")
            out["cpu_baseline"]["port_note"] = {"value": round(pv, 5), "seconds": pd["step_s"],
                                                "what": "the oracle restatement on the same volume (not the baseline)"}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def bench_dropin(reps: int = 5) -> dict:
    """Per-call latency of the reference-facing drop-in API on a host numpy
    volume: extract_features(Volume(ndarray)) (cached Extractor, H2D of the
    volume, the whole pipeline, SoA read-back) plus materialising the
    reference's Python objects (keypoints, oriented frames, descriptor
    records), wall clock, median of `reps` calls after 2 warm-up calls."""
    import paper_2112_10258_b200 as vk
    from paper_2112_10258_b200 import synthetic

    vol = vk.Volume(synthetic.brain_volume())
    cfg = vk.PipelineConfig()

    def call(materialise):
        t0 = time.perf_counter()
        r = vk.extract_features(vol, cfg)
        t1 = time.perf_counter()
        if materialise:
            _ = (r.keypoints, r.oriented, r.records)
        return t1 - t0, time.perf_counter() - t0, len(r.soa["desc"])

    for _ in range(2):
        call(True)
    soa_only = [call(False)[0] for _ in range(reps)]
    full = [call(True) for _ in range(reps)]
    med_full = statistics.median(f[1] for f in full)
    return {"api": "extract_features(Volume(numpy 145x174x145), PipelineConfig()) + .keypoints/.oriented/.records",
            "ms_per_call": round(1e3 * med_full, 2), "volumes_per_s": round(1.0 / med_full, 2),
            "ms_per_call_soa_only": round(1e3 * statistics.median(soa_only), 2),
            "descriptors": full[0][2], "reps": reps, "timing": "host wall clock (perf_counter), median"}


def bench_configs3(steps: int = 5) -> dict:
    """configs[3]: 256^3 synthetic volumes, num_octaves=4,
    detect + describe, as 4 parallel-stream sub-batches of 2 volumes in one
    CUDA graph; device time with CUDA events; pyramid roofline on one
    sub-batch."""
    import torch

    import paper_2112_10258_b200 as vk
    from paper_2112_10258_b200 import _lib, synthetic
    from paper_2112_10258_b200.engine import Extractor, ExtractorGroup

    dims = (256, 256, 256)
    cfg = vk.PipelineConfig(num_octaves=4)
    base = synthetic.soup_volume(dims, np.random.default_rng(20240817), noise=0.01)
    host = synthetic.batch_from(base, 8, seed=31)
    dev = torch.stack([vk.volume.to_device(v) for v in host])
    members = [Extractor(dims, cfg, batch=2, input=dev[2 * m: 2 * m + 2]) for m in range(4)]
    for ex in members:
        ex.enqueue()
    torch.cuda.synchronize()
    grp = ExtractorGroup(members)
    grp.capture()
    for _ in range(2):
        grp.run()
    st = torch.cuda.current_stream()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        grp.run()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    ex = members[0]
    pt = []
    for _ in range(3):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        ex.enqueue_pyramid(st.cuda_stream)
        a1.record(st)
        torch.cuda.synchronize()
        pt.append(a0.elapsed_time(a1))
    with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
        peak = json.load(fh).get("hbm_gbs")
    pb = pyramid_bytes(ex.plan) * ex.B
    ach = pb / (statistics.median(pt) / 1e3) / 1e9
    c = {k: sum(m.counts()[k] for m in members) for k in ("keypoints", "frames")}
    return {"workload": "configs[3]: 8 x 256^3 volumes per step, num_octaves=4, detect + describe (siftrank)",
            "volumes_per_s": round(8 / (ms / 1e3), 2), "ms_per_step": round(ms, 3),
            "keypoints_per_volume": c["keypoints"] / 8, "frames_per_volume": c["frames"] / 8,
            "pyramid_ms_per_subbatch_of_2": round(statistics.median(pt), 4),
            "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(ach / peak, 4) if peak else None, "algorithmic_bytes": pb}}


def bench_matching() -> dict:
    """Side measurement of the matching hot path (configs[1] / configs[4]):
    SIFT-Rank rows (int8 rank permutations) matched on the tcgen05 kind::i8
    kernel.  Device time with CUDA events, inputs resident.  Reported apart
    from the volumes/s headline."""
    import torch

    from paper_2112_10258_b200 import _lib

    rng = np.random.default_rng(7)

    def ranks(n):
        return torch.from_numpy(np.argsort(rng.random((n, 64)), axis=1).astype(np.int8)).cuda()

    def timed(na, nb, reps):
        a, b = ranks(na), ranks(nb)
        out = [torch.empty(na, dtype=t, device="cuda") for t in (torch.int32, torch.float64, torch.float64, torch.uint8)]
        st = torch.cuda.current_stream()
        call = lambda: _lib.call("vk_match", 1, a.data_ptr(), na, b.data_ptr(), nb, 64, 0.9,
                                 *[o.data_ptr() for o in out], st.cuda_stream)
        call()
        call()
        torch.cuda.synchronize()
        trials = []
        for _ in range(5):  # median of 5 trials: single short trials vary by up to 1.5x on a shared box
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                call()
            e1.record(st)
            torch.cuda.synchronize()
            trials.append(e0.elapsed_time(e1) / reps)
        return float(np.median(trials))

    pair_ms = timed(3400, 3300, 20)
    na, nb = 65536, 1 << 20
    db_ms = timed(na, nb, 2)
    pairs_s = na * nb / (db_ms / 1e3)
    tops = 2.0 * 64 * pairs_s / 1e12
    subj, per = 1000, 3400
    return {
        "kernel": "match_i8_ws_kernel (warp-specialised: TMA tiles, tcgen05.mma kind::i8 M=2x128 N=128, s32 TMEM accumulators, top-2 epilogue warps)",
        "image_pair_ms": round(pair_ms, 4), "image_pair_shape": [3400, 3300],
        "database_sample": {"queries": na, "database_rows": nb, "ms": round(db_ms, 3),
                            "pairs_per_s": round(pairs_s), "unit": "descriptor pairs/s"},
        "configs4_projection_s_per_gpu": {str(g): round(subj * per / g * subj * per / pairs_s, 3) for g in (1, 2, 4, 8)},
        "roofline": {"bound": "tensor", "achieved": round(tops, 1), "peak": 4500.0, "unit": "TOPS",
                     "frac": round(tops / 4500.0, 4),
                     "peak_source": "nominal dense int8/fp8 B200 (B200_PROFILING.md table); epilogue-bound"},
    }


def run_reference(a):
    """The reference arm: the unmodified volkey (oracle/_ref) on every host
    core, one single-threaded process per core, one full volume each per step
    (falls back to the oracle port, kind "port", if oracle/_ref is not staged)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    procs = os.cpu_count() or 1
    steps = max(1, min(a.steps, a.ref_steps))
    impl = "reference" if ref_available() else "port"
    vps, det = cpu_volumes_per_s(a.descriptor, procs, steps, impl)
    what = ("the unmodified reference volkey.extract_features(Volume, PipelineConfig(workers=1)) from oracle/_ref"
            if impl == "reference" else "oracle/volkey_oracle.py (oracle/_ref not staged)")
    out = {
        "impl": "reference", "metric": METRIC, "value": round(vps, 5), "unit": UNIT, "n_gpus": world,
        "steps": steps, "steps_requested": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * statistics.mean(det["step_s"]),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 + f64 (numpy)",
        "data": "synthetic (same phantom family as the GPU arm)",
        "config": {"workload": f"1 x 145x174x145 volume per process per step, {procs} processes, detect + describe "
                               f"({a.descriptor})", "volume": list(DIMS), "descriptor": a.descriptor},
        "cpu_baseline": {"value": round(vps, 5), "unit": UNIT, "cores": procs, "kind": impl,
                         "sample": f"{procs} concurrent single-threaded processes (OPENBLAS_NUM_THREADS=1) x {steps} "
                                   f"step(s), one full volume each, {what}"},
        "e2e": {"value": round(vps, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_seconds": det["step_s"],
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
