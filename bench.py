#!/usr/bin/env python
"""bench.py -- tet-mesh ray traversal throughput on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

Workload (BASELINE.json configs[1], the metric's single-GPU config):
config 2 = the reference's blob generator at GRID=55 (1,109,444 tets,
byte-identical to gen_model_mesh -> parse_tetgen -> encode, pinned by
tests/test_host_mirror.py), TetMesh-20, Hilbert-sorted, 1920x1080 primary
rays from the blob camera, all starting in the located camera tet.
A "step" traces one frame per GPU.  Weak scaling: at N GPUs the job is N
frames (camera jittered per frame), 16x16 tiles dealt round-robin to ranks,
hit buffers gathered to rank 0 with one NCCL collective inside the timed
region.

value  = rays / device time of the trace kernel (CUDA events on the launch
         stream, inputs resident in HBM, L2 flushed between steps).
e2e    = the same rays through the C ABI with pinned HOST buffers
         (tb_cast_rays_host: H2D, kernel, D2H, sync) per step.
roofline = SURVEY.md s8(d) algorithmic bytes / kernel time vs measured HBM.
cpu_baseline = the reference's compiled kernels (oracle/_ref) + its batch
         epilogue on all host cores (rank 0, N=1, bounded sample).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    1: dict(grid=12, width=256, height=256, layout="tet80", walk="sctp", scheme="none",
            desc="cfg1: blob GRID=12 (11,029 tets), 256x256 primary rays, TetMesh-80 + ScTP walk"),
    2: dict(grid=55, width=1920, height=1080, layout="tet20", scheme="hilbert",
            desc="cfg2: blob GRID=55 (1,109,444 tets), 1920x1080 primary rays, TetMesh-20 Hilbert-sorted"),
    3: dict(grid=55, width=3840, height=2160, layout="tet16", scheme="hilbert",
            desc="cfg3: blob GRID=55 (1,109,444 tets), 3840x2160 primary rays, TetMesh-16 Hilbert-sorted"),
    4: dict(grid=55, width=4096, height=4096, layout="tet16", scheme="hilbert", secondaries=True,
            desc="cfg4: blob GRID=55, 16.7M diffuse secondaries from 4096x4096 primary hits, TetMesh-16"),
    # config 5 names no layout (BASELINE.json configs[4]); with 180 GB of HBM the
    # 1 GB TetMesh-20 beats the 0.8 GB TetMesh-16 (r01 A/B: 825 vs 707 Mrays/s)
    5: dict(kuhn=203, width=7680, height=4320, layout="tet20", scheme="none",
            desc="cfg5: Kuhn box n=203 (50,192,562 tets) stretched 4x in z with thin strip occluders "
                 "(long thin triangles), 7680x4320 primary rays, TetMesh-20"),
}
L2_FLUSH_BYTES = 256 << 20
FALLBACK_HBM_GBS = 6650.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def build_scene(cfg):
    from paper_2103_02309_b200.scenes import blob_scene, kuhn_strip_scene

    t0 = time.perf_counter()
    if "kuhn" in cfg:
        sc = kuhn_strip_scene(cfg["kuhn"], layout=cfg["layout"], scheme=cfg["scheme"])
    else:
        host_layout = "tet32" if cfg["layout"] == "tet80" else cfg["layout"]
        sc = blob_scene(cfg["grid"], layout=host_layout, scheme=cfg["scheme"], check=False)
    log(f"[bench] scene {sc.name}: {sc.mesh.n_tets} tets, {sc.mesh.n_points} points, "
        f"{sc.mesh.n_constrained} constrained faces, built in {time.perf_counter() - t0:.1f}s")
    return sc


def frame_rays(cfg, frame: int):
    from paper_2103_02309_b200.scenes import BLOB_CAMERA, camera_rays, kuhn_camera

    cam = kuhn_camera(cfg["kuhn"]) if "kuhn" in cfg else BLOB_CAMERA
    pos = np.asarray(cam["position"], dtype=np.float64) + np.array([0.0, 0.02, 0.0]) * frame
    o, d = camera_rays(tuple(pos), cam["look_at"], cam["up"], cam["fov"], cfg["width"], cfg["height"])
    return o, d, pos


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))

    def mark(self, name: str):
        setattr(self, name, time.perf_counter())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0=None, t1=None):
        """Median SM clock and throttle reasons over samples read in [t0, t1]."""
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ts, line in self.lines:
            if (t0 is not None and ts < t0) or (t1 is not None and ts > t1):
                continue
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference_trace(mesh, o, d, st, threads: int):
    """The reference's CPU path for one batch: compiled kernels (oracle/_ref,
    _kernels.pyx:271-370, GIL released) + the batch epilogue (batch.py:57-71),
    chunked over a thread pool like the reference renderer's tile pool."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import pyoracle

    K = pyoracle.ref_kernels()
    kind = "reference"
    if K is None:
        K, kind = pyoracle, "port"
    n = len(st)
    chunks = max(1, min(threads * 16, n // 4096))  # >= 4096 rays per chunk: pool overhead stays small
    bounds = np.linspace(0, n, chunks + 1).astype(np.int64)

    def work(i):
        a, b = bounds[i], bounds[i + 1]
        if a == b:
            return 0
        status, cf, tet, visited = K.cast_rays(mesh, o[a:b], d[a:b], st[a:b])
        pyoracle.batch_epilogue(mesh, o[a:b], d[a:b], status, cf, tet)
        return int(visited.sum())

    with ThreadPoolExecutor(max_workers=threads) as pool:
        total_vis = sum(pool.map(work, range(chunks)))
    return kind, total_vis


def cpu_single_thread(mesh, o, d, st, reps: int = 2) -> dict:
    """the reference's CPU path on ONE thread, its compiled
    kernels and the host batch epilogue timed separately (best of reps)."""
    from oracle import pyoracle

    K = pyoracle.ref_kernels() or pyoracle
    best_k = best_e = None
    for _ in range(reps):
        t0 = time.perf_counter()
        status, cf, tet, _ = K.cast_rays(mesh, o, d, st)
        t1 = time.perf_counter()
        pyoracle.batch_epilogue(mesh, o, d, status, cf, tet)
        t2 = time.perf_counter()
        best_k = t1 - t0 if best_k is None else min(best_k, t1 - t0)
        best_e = t2 - t1 if best_e is None else min(best_e, t2 - t1)
    n = len(st)
    return {"value": n / (best_k + best_e) / 1e6, "unit": "Mrays/s", "cores": 1, "rays": n,
            "kernel_only": n / best_k / 1e6, "epilogue_share": best_e / (best_k + best_e)}


def run_reference_arm(args, cfg):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    sc = build_scene(cfg)
    mesh = sc.mesh
    from oracle import pyoracle

    o, d, pos = frame_rays(cfg, 0)
    K = pyoracle.ref_kernels() or pyoracle
    cam, _ = K.locate_points(mesh, pos[None], np.array([mesh.source_tet], np.int32))
    st = np.full(len(o), int(cam[0]), dtype=np.int32)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        kind, _ = cpu_reference_trace(mesh, o, d, st, threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        kind, vis = cpu_reference_trace(mesh, o, d, st, threads)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = len(o) * args.steps / total / 1e6
    line = {
        "impl": "reference", "metric": "Mrays/s", "value": value, "unit": "Mrays/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["desc"], "rays_per_step": len(o), "layout": mesh.layout,
                   "scheme": cfg["scheme"],
                   **({"note": "the reference has no TetMesh-80 layout and no ScTP walk: its 2-D walk on "
                               "the Tet32 mesh of the same scene and rays"} if cfg["layout"] == "tet80" else {})},
        "tets_visited_per_ray": {"mean": vis / len(o)},
        "cpu_baseline": {"value": value, "unit": "Mrays/s", "cores": threads, "kind": kind,
                         "sample": f"full frame ({len(o)} rays) per step: compiled _kernels.cast_rays + "
                                   "batch epilogue, ThreadPoolExecutor over min(16 per thread, n / 4096) chunks"},
        "e2e": {"value": value, "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def digest(*arrays) -> str:
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def algorithmic_bytes(visited: np.ndarray, layout: str) -> int:
    """sum_rays [(visited-1)(L+12) + 68] + 53 N."""
    L = {"tet32": 32, "tet20": 20, "tet16": 16, "tet80": 80}[layout]
    point = 0 if layout == "tet80" else 12
    v = visited.astype(np.int64)
    return int(((v - 1) * (L + point)).sum() + 68 * len(v) + 53 * len(v))


def l2_gather_roof(dm, stream, flush, layout: str, walk_steps: float, achieved_gbs: float) -> dict:
    """for meshes that fit in L2, the walk's algorithmic bytes
    against a measured random-gather roof of the same mesh -- tb_probe_gather
    issues one step's loads (record + axis-permuted point) at independent
    pseudo-random indices, 8 per thread in flight, L2 flushed before each
    rep like the timed steps."""
    import torch

    from paper_2103_02309_b200._lib import check, lib

    L = {"tet32": 32, "tet20": 20, "tet16": 16}[layout]
    n_pairs = int(min(max(32 << 20, walk_steps), 256 << 20))
    sink = torch.zeros(1, dtype=torch.int32, device=flush.device)

    def probe():
        check(lib.tb_probe_gather(dm.handle, n_pairs, 12345, sink.data_ptr(), stream.cuda_stream), "tb_probe_gather")

    for _ in range(2):
        probe()
    ms = []
    for _ in range(5):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        probe()
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    t = float(np.median(ms)) / 1e3
    peak = n_pairs * (L + 12) / t / 1e9
    l2 = torch.cuda.get_device_properties(flush.device).L2_cache_size
    resident = dm.hot_bytes <= l2
    return {"bound": "l2_gather", "achieved": achieved_gbs, "peak": peak, "unit": "GB/s",
            "frac": achieved_gbs / peak,
            "probe": {"kernel": f"gather_probe_kernel<{L}>", "pairs": n_pairs, "bytes_per_pair": L + 12,
                      "ms": t * 1e3, "working_set_bytes": int(dm.hot_bytes), "l2_bytes": int(l2)},
            "note": ("peak = random (record, point) gathers over this mesh's hot arrays "
                     + ("(L2 resident)" if resident else "(larger than L2: an HBM random-gather roof)")
                     + "; the walk exceeds it when coherent rays share L1/L2 lines (frac > 1) -- its binding "
                       "roof is roofline_issue")}


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2103_02309_b200 import multigpu
    from paper_2103_02309_b200._lib import addr, check, lib
    from paper_2103_02309_b200.device import device_mesh
    from paper_2103_02309_b200.trace import empty_result, locate, trace

    world, rank, local = dist_env()
    # one rank per GPU; TETB200_DIST_BACKEND=gloo lets several ranks share one
    # GPU to exercise the N>1 code path on a single device (test only)
    backend = os.environ.get("TETB200_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    sc = build_scene(cfg)
    mesh = sc.mesh
    # tet80 has no host record dtype: the host mesh stays tet32 and the device
    # builds the 80-byte records from the side tables
    dm = device_mesh(mesh, device=local, layout=cfg["layout"] if cfg["layout"] == "tet80" else None)
    sctp = cfg.get("walk") == "sctp"
    W, H = cfg["width"], cfg["height"]
    per_frame = W * H

    # this rank's share of the N-frame job (16x16 tiles round-robin)
    idx = multigpu.shard_pixels(W, H, rank, world, 16, frames=world)
    frames = idx // per_frame
    o = np.empty((len(idx), 3), np.float32)
    d = np.empty((len(idx), 3), np.float32)
    st = np.empty(len(idx), np.int32)
    for f in np.unique(frames):
        of, df, pos = frame_rays(cfg, int(f))
        sel = frames == f
        o[sel] = of[idx[sel] % per_frame]
        d[sel] = df[idx[sel] % per_frame]
        q = torch.tensor(pos[None], dtype=torch.float64, device=dev)
        cam, _ = locate(dm, q, torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
        st[sel] = int(cam.item())
    if cfg.get("secondaries"):
        # config 4: the timed rays are the diffuse secondaries spawned from this
        # shard's primary hits (traced here, untimed), in shard order
        from paper_2103_02309_b200.scenes import diffuse_secondaries

        prim = trace(dm, *(torch.from_numpy(a).to(dev) for a in (o, d, st)))
        torch.cuda.synchronize()
        hit = prim.triangle.cpu().numpy() >= 0
        o, d, st = diffuse_secondaries(o, d, prim.t.cpu().numpy(), prim.triangle.cpu().numpy(),
                                       prim.tet.cpu().numpy(), mesh.triangle_coords(), seed=4 + rank)
        idx = idx[hit]
        del prim
    n = len(st)
    go, gd, gs = (torch.from_numpy(a).to(dev) for a in (o, d, st))
    res = empty_result(n, dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    gidx = torch.from_numpy(idx).to(dev)

    # ray schedule: one ray per lane for primaries; incoherent secondaries
    # (config 4) are binned by direction cell first (96 cube-map cells) and
    # walked in binned order (r01: 3.36 vs 2.37 Grays/s one ray per lane,
    # 2.30 block compaction; profiles/r01_experiments.md) -- what a
    # renderer's bounce pass selects with trace(schedule="binned").  --schedule or
    # TETB200_SCHED (sweeps, via the process-wide "auto" setting) override.
    schedule = args.schedule or ("auto" if os.environ.get("TETB200_SCHED") else
                                 ("binned" if cfg.get("secondaries") else "lane"))

    def step():
        trace(dm, go, gd, gs, out=res, stream=stream, sctp=sctp, schedule=schedule)

    fg = None
    pg = None
    gather_mode = None
    if world > 1 and args.gather == "p2p":
        # every step assembles its frame set on rank 0 inside the trace: each
        # rank's kernel stores every finished ray into rank 0's full-frame
        # arrays (CUDA IPC, P2P over NVLink) -- no collective moves the hits
        try:
            root_rays = True  # lean assembly: ranks store 13 B per ray, rank 0 derives the epilogue
            if rank == 0:
                if cfg.get("secondaries"):
                    root_rays = None  # secondaries are spawned per rank: the root lacks their rays
                else:  # the job's rays in global order (frame-major), resident on rank 0 (untimed setup)
                    frames_rays = [frame_rays(cfg, f)[:2] for f in range(world)]
                    root_rays = tuple(torch.from_numpy(np.ascontiguousarray(np.concatenate([fr[i] for fr in
                                                                                             frames_rays])))
                                      .to(dev) for i in (0, 1))
            lean_flags = [None] * world
            dist.all_gather_object(lean_flags, root_rays is not None)
            if not all(lean_flags):
                root_rays = None
            pg = multigpu.PeerFrameGather(W, H, world, rank, world, dev, root_rays=root_rays)
            gather_mode = "p2p"

            def step():  # noqa: F811  (the N > 1 step: fused trace + frame assembly)
                return pg.step(dm, go, gd, gs, stream)
        except Exception as exc:  # no peer access / IPC: fall back to the NCCL gather
            log(f"[bench] p2p frame assembly unavailable ({exc!r}); using the NCCL gather")
            pg = None
    if world > 1 and pg is None:
        # every step gathers its frame set to rank 0: the shard is traced in
        # chunks and each chunk's 20 B records go out with an async NCCL
        # gather while the next chunk traces (multigpu.FrameGather)
        from paper_2103_02309_b200.trace import TraceResult

        gather_mode = "nccl"
        fg = multigpu.FrameGather(W, H, world, rank, world, args.gather_chunks, dev, mesh.cf_triangle, mesh.cf_tets)
        views = [TraceResult(*(getattr(res, f)[a:b] for f in ("status", "cf", "triangle", "t", "tet", "tet_back",
                                                                 "visited"))) for (a, b) in fg.my_pieces()]
        pieces = fg.my_pieces()

        def step():  # noqa: F811  (the N > 1 step: trace + per-frame gather)
            for k, ((a, b), v) in enumerate(zip(pieces, views)):
                if b > a:
                    trace(dm, go[a:b], gd[a:b], gs[a:b], out=v, stream=stream, sctp=sctp, schedule=schedule)
                fg.send(k, v.status, v.cf, v.tet, v.visited, v.t)
            return fg.finish()

    # warm-up
    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    if pg is not None:
        # p2p: the hits live in rank 0's frame; rank 0 checks its own rays'
        # slice below, and the visited statistics come from the whole frame
        from paper_2103_02309_b200.trace import TraceResult as _TR

        if rank == 0:
            res = _TR(*(pg.frame[k][gidx] for k in ("status", "cf", "triangle", "t", "tet", "tet_back", "visited")))

    # parity at full size: the reference's own digest of this frame (rank 0, N=1)
    parity = None
    dig_path = os.path.join(ROOT, "tests", "golden", "golden_digests.json")
    key = f"blob{cfg.get('grid')}/{cfg['scheme']}/cast"
    if world == 1 and os.path.exists(dig_path) and cfg.get("layout") in ("tet20", "tet16", "tet32") \
            and not cfg.get("secondaries") and "grid" in cfg:
        digs = json.load(open(dig_path))
        if key in digs and (W, H) == {12: (256, 256), 55: (1920, 1080)}.get(cfg["grid"]):
            inv = np.empty_like(idx)
            inv[idx] = np.arange(len(idx))  # shard position of each row-major pixel

            def rm(x):
                return x.cpu().numpy()[inv]

            got = digest(rm(res.status), rm(res.cf), rm(res.tet), rm(res.visited))
            ep = digest(rm(res.triangle), rm(res.t), rm(res.tet_back))
            parity = {"vs": "reference digest " + key,
                      "traversal_bit_exact": got == digs[key],
                      "epilogue_bit_exact": ep == digs[key.replace("/cast", "/epilogue")]}
    if parity is None and rank == 0 and not args.no_parity:
        # no reference digest for this workload: check a strided sample of
        # rays against the CPU oracle (the checker, never the measured path)
        from oracle import pyoracle

        stride = max(1, n // args.parity_sample)
        sl = slice(0, n, stride)
        exp = pyoracle.cast_rays_full(mesh, o[sl], d[sl], st[sl], layout=dm.layout, sctp=sctp)
        got = [x.cpu().numpy()[sl] for x in (res.status, res.cf, res.tet, res.visited, res.triangle, res.t,
                                              res.tet_back)]
        mism = int(sum(np.count_nonzero(a != b) for a, b in zip(got, exp)))
        parity = {"vs": f"C oracle (oracle/tetoracle.c) on every {stride}th ray", "rays_checked": int(len(exp[0])),
                  "mismatched_values": mism, "bit_exact": mism == 0}
    if pg is None:
        visited = res.visited.cpu().numpy()
    else:  # the whole job's visited counts on rank 0, none elsewhere
        visited = pg.frame["visited"].cpu().numpy() if rank == 0 else np.zeros(0, np.int32)

    # timed region: K steps between barrier + sync; per-step kernel events.
    # nvidia-smi samples clocks from a short untimed ramp (so the sampler is
    # up and the clocks have left idle) through the end of the timed region.
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    gather_check = None
    gather_error = None
    with ClockSampler(local) as clocks:
        time.sleep(0.3)  # nvidia-smi start-up
        clocks.mark("t_ramp")
        r0 = time.perf_counter()
        if world > 1:  # collectives in the step: every rank runs the same count
            for _ in range(16):
                flush.zero_()
                step()
            torch.cuda.synchronize()
        while world == 1 and time.perf_counter() - r0 < args.ramp_s:
            for _ in range(8):
                flush.zero_()
                step()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        clocks.mark("t_end")
        if world > 1:
            dist.barrier()
        time.sleep(0.05)
    kernel_ms = np.array([a.elapsed_time(b) for a, b in evs])
    if world > 1:
        # N > 1: the gathered frame set of the last step, checked on rank 0
        try:
            full = step()
            torch.cuda.synchronize()
            if full is not None:
                gather_check = int((full["visited"] > 0).sum().item())
                dig_path = os.path.join(ROOT, "tests", "golden", "golden_digests.json")
                key = f"blob{cfg.get('grid')}/{cfg['scheme']}/cast"
                if os.path.exists(dig_path) and "grid" in cfg and (W, H) == (1920, 1080) \
                        and not cfg.get("secondaries") and cfg["layout"] != "tet80":
                    digs = json.load(open(dig_path))
                    if key in digs:  # frame 0 is the reference camera: compare with its digest
                        f0 = [full[k][:per_frame].cpu().numpy() for k in ("status", "cf", "tet", "visited")]
                        e0 = [full[k][:per_frame].cpu().numpy() for k in ("triangle", "t", "tet_back")]
                        gather_check = {"rays": gather_check, "frame0_vs_reference_digest": digest(*f0) == digs[key],
                                        "frame0_epilogue_vs_reference_digest":
                                            digest(*e0) == digs[key.replace("/cast", "/epilogue")]}
        except Exception as exc:  # report, do not lose the line
            gather_error = repr(exc)
    my_ms = float(kernel_ms.sum())
    if world > 1:
        t = torch.tensor([my_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        max_ms = float(t.item())
        vt = torch.tensor([int(visited.sum()), int(visited.max(initial=0)), len(visited)], dtype=torch.int64,
                          device=dev)
        vmax = vt.clone()
        dist.all_reduce(vt, op=dist.ReduceOp.SUM)
        dist.all_reduce(vmax, op=dist.ReduceOp.MAX)
        vis_sum, vis_max, total_rays = int(vt[0]), int(vmax[1]), int(vt[2])
    else:
        max_ms = my_ms
        vis_sum, vis_max, total_rays = int(visited.sum()), int(visited.max()), n

    value = total_rays * args.steps / (max_ms / 1e3) / 1e6
    ms_per_step = max_ms / args.steps

    # end to end through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        ho = torch.from_numpy(o).pin_memory()
        hd = torch.from_numpy(d).pin_memory()
        hs = torch.from_numpy(st).pin_memory()
        outs = [torch.empty(n, dtype=dt).pin_memory() for dt in
                (torch.uint8, torch.int32, torch.int32, torch.int32, torch.int32, torch.float64, torch.int32)]

        host_fn = lib.tb_sctp_cast_rays_host if sctp else lib.tb_cast_rays_host

        def host_call():
            check(host_fn(dm.handle, n, addr(ho), addr(hd), addr(hs), *[addr(x) for x in outs]),
                  "tb_sctp_cast_rays_host" if sctp else "tb_cast_rays_host")

        for _ in range(max(1, args.warmup)):
            host_call()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            host_call()
        e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_s = float(t.item())
        e2e = {"value": total_rays * args.steps / e_s / 1e6, "unit": "Mrays/s",
               "h2d_bytes_per_step": int(n * (12 + 12 + 4)), "d2h_bytes_per_step": int(n * (1 + 4 * 5 + 8)),
               "ms_per_step": e_s / args.steps * 1e3,
               "gpu_launches_per_step": 1 if os.environ.get("TETB200_E2E", "0") == "0" else -(-n // (1 << 18)),
               "path": f"{'tb_sctp_cast_rays_host' if sctp else 'tb_cast_rays_host'} (C ABI) on pinned host "
                       "buffers: zero-copy trace over PCIe (TETB200_E2E=1: 3-stream chunked H2D/trace/D2H)"}

    # incoherent secondaries of this frame (BASELINE's metric names primary
    # AND incoherent secondary rays): diffuse bounces from this rank's
    # primary hits (render.py:353-359 semantics, seed 4), traced on the
    # device under each schedule, same timing protocol; checked on
    # a strided sample against the oracle.
    secondary = None
    if not args.no_secondary and not cfg.get("secondaries") and not sctp and world == 1:
        from paper_2103_02309_b200.scenes import diffuse_secondaries
        from paper_2103_02309_b200.trace import TraceResult as _TR

        so, sd, sst = diffuse_secondaries(o, d, res.t.cpu().numpy(), res.triangle.cpu().numpy(),
                                          res.tet.cpu().numpy(), mesh.triangle_coords(), seed=4)
        ns = len(sst)
        if ns:
            g2 = [torch.from_numpy(a).to(dev) for a in (so, sd, sst)]
            r2 = empty_result(ns, dev)
            sec = {}
            for sched2 in ("compact", "lane", "binned"):
                for _ in range(args.warmup):
                    flush.zero_()
                    trace(dm, *g2, out=r2, stream=stream, schedule=sched2)
                ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(args.steps)]
                torch.cuda.synchronize()
                for a, b in ev2:
                    flush.zero_()
                    a.record(stream)
                    trace(dm, *g2, out=r2, stream=stream, schedule=sched2)
                    b.record(stream)
                torch.cuda.synchronize()
                sec[sched2] = float(np.mean([a.elapsed_time(b) for a, b in ev2]))
            v2 = r2.visited.cpu().numpy()
            par2 = None
            if not args.no_parity:
                from oracle import pyoracle

                stride = max(1, ns // args.parity_sample)
                sl2 = slice(0, ns, stride)
                exp2 = pyoracle.cast_rays_full(mesh, so[sl2], sd[sl2], sst[sl2], layout=dm.layout)
                got2 = [x.cpu().numpy()[sl2] for x in (r2.status, r2.cf, r2.tet, r2.visited, r2.triangle, r2.t,
                                                        r2.tet_back)]
                mism2 = int(sum(np.count_nonzero(a != b) for a, b in zip(got2, exp2)))
                par2 = {"vs": f"C oracle on every {stride}th ray", "rays_checked": int(len(exp2[0])),
                        "bit_exact": mism2 == 0}
            secondary = {"value": ns / sec["binned"] / 1e3, "unit": "Mrays/s", "rays": ns,
                         "kernel_ms": sec["binned"], "schedule": "binned",
                         "note": "direction-cell counting sort (96 cube-map cells) + the walk in binned order, "
                                 "both inside the events",
                         "one_ray_per_lane": {"value": ns / sec["lane"] / 1e3, "kernel_ms": sec["lane"]},
                         "block_compaction": {"value": ns / sec["compact"] / 1e3, "kernel_ms": sec["compact"]},
                         "tets_visited_per_ray": {"mean": float(v2.mean()), "max": int(v2.max())},
                         "rays_from": "diffuse hemisphere bounces of this frame's primary hits (seed 4)",
                         "parity": par2}

    # render-style end to end: camera rays generated in HBM (no ray upload),
    # trace, all 7 hit arrays copied back to pinned host memory, per step
    e2e_render = None
    if not args.no_e2e and world == 1 and not cfg.get("secondaries"):
        from paper_2103_02309_b200.scenes import BLOB_CAMERA, kuhn_camera
        from paper_2103_02309_b200.trace import trace_camera

        from paper_2103_02309_b200.trace import TraceResult

        cam = kuhn_camera(cfg["kuhn"]) if "kuhn" in cfg else BLOB_CAMERA
        # hits land in pinned host memory, written by the trace kernel itself
        hres = TraceResult(*[torch.empty(W * H, dtype=dt).pin_memory() for dt in
                             (torch.uint8, torch.int32, torch.int32, torch.float64, torch.int32, torch.int32,
                              torch.int32)])
        _, cam_tet = trace_camera(dm, cam, W, H, out=hres, stream=stream, sctp=sctp)  # camera located once

        def render_call():
            trace_camera(dm, cam, W, H, out=hres, stream=stream, cam_tet=cam_tet, sctp=sctp)
            torch.cuda.synchronize()

        for _ in range(max(1, args.warmup)):
            render_call()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            render_call()
        r_s = time.perf_counter() - t0
        e2e_render = {"value": W * H * args.steps / r_s / 1e6, "unit": "Mrays/s", "h2d_bytes_per_step": 14 * 8,
                      "d2h_bytes_per_step": int(W * H * 29), "ms_per_step": r_s / args.steps * 1e3,
                      "path": "trace_camera: rays generated in HBM, trace writes all 7 hit arrays straight to "
                              "pinned host memory (camera tet located once)"}

    if rank != 0:
        if pg is not None:
            pg.close()
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = measured_peak()
    alg = algorithmic_bytes(visited, cfg["layout"])
    kern_s = float(kernel_ms.mean()) / 1e3
    achieved = alg / kern_s / 1e9
    # Issue roofline of the walk (the kernel is instruction-issue / ALU-pipe
    # bound, ncu r01): peak ray-steps/s if every scheduler issued one
    # full-warp step instruction per cycle = SMs x 4 x clock x 32 lanes /
    # SASS instructions per step (tools/sass_steps.py, committed per build).
    roofline_issue = None
    sp = os.path.join(ROOT, "profiles", "sass_step_counts.json")
    clk_mhz = clocks.summary(clocks.t_ramp, clocks.t_end).get("sm_mhz")
    if os.path.exists(sp) and clk_mhz and not sctp:
        counts = json.load(open(sp))
        kname = ("cast_compact_kernel" if schedule in ("compact", "compact512") else "cast_kernel")
        entry = counts.get(f"{kname}<{cfg['layout'][3:]}, validated>") or counts.get(f"{kname}<{cfg['layout'][3:]}, clamp>")
        if entry:
            per_step = (entry.get("unrolled_x4_per_step") or entry["single_step"])["total"]
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            peak_steps = sms * 4 * clk_mhz * 1e6 * 32 / per_step
            steps = (vis_sum - total_rays) / world  # walk steps of one rank's launch
            ach_steps = steps / kern_s
            roofline_issue = {"bound": "issue", "achieved": ach_steps / 1e9, "peak": peak_steps / 1e9,
                              "unit": "G ray-steps/s", "frac": ach_steps / peak_steps,
                              "sass_per_step": per_step, "sms": sms, "sm_mhz": clk_mhz,
                              "note": "peak = SMs x 4 schedulers x clock x 32 lanes / SASS per walk step; "
                                      "the gap is init/epilogue, SIMT divergence, latency and the tail"}
    roofline_l2 = None
    if not sctp and cfg["layout"] != "tet80" and not args.no_l2_probe:
        roofline_l2 = l2_gather_roof(dm, stream, flush, cfg["layout"], (vis_sum - total_rays) / world, achieved)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"cfg{args.config}/{cfg['layout']}")
    line = {
        "metric": "Mrays/s", "value": value, "unit": "Mrays/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["desc"], "rays_per_gpu": n, "layout": cfg["layout"], "scheme": cfg["scheme"],
                   "parallelism": f"tile-shard x{world}, mesh replicated", "l2": "flushed between steps (256 MiB)",
                   "schedule": schedule,
                   "frames": world},
        "tets_visited_per_ray": {"mean": vis_sum / total_rays, "max": vis_max},
        "kernel_ms": {"mean": float(kernel_ms.mean()), "min": float(kernel_ms.min()), "max": float(kernel_ms.max())},
        "gather_ms": None,
        "gather": None if world == 1 else (
            {"rays_gathered_to_rank0": gather_check, "rays_expected": per_frame * world, "error": gather_error,
             "mode": "p2p",
             "per_step": "every step assembles its frame set on rank 0 inside the timed region: each rank's trace "
                         "epilogue stores every finished ray into rank 0's full-frame arrays (CUDA IPC, P2P over "
                         "NVLink), then stream sync + barrier",
             "bytes_to_rank0_per_step": int((13 if pg.lean else 29) * per_frame * (world - 1)),
             "lean": bool(pg.lean), "collective": "none (barrier only)"}
            if gather_mode == "p2p" else
            {"rays_gathered_to_rank0": gather_check, "rays_expected": per_frame * world, "error": gather_error,
             "mode": "nccl",
             "per_step": "every step gathers its frame set to rank 0 inside the timed region (chunked, overlapped "
                         "with the trace)",
             "bytes_to_rank0_per_step": int(20 * per_frame * (world - 1)), "chunks": args.gather_chunks,
             "collective": "torch.distributed.gather (NCCL, async), 20 B records"}),
        "wall_ms_per_step": wall / args.steps * 1e3,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": alg,
                     "kernel": (f"sctp_kernel<{cfg['layout'][3:]}>" if sctp else
                                f"{'cast_compact_kernel' if schedule in ('compact', 'compact512') else 'cast_kernel'}"
                                f"<{cfg['layout'][3:]}>"
                                + (" after bin_count/bin_seg_scan/bin_scatter (direction binning, inside the events)"
                                   if schedule == "binned" else "")),
                     "note": "algorithmic gather bytes (SURVEY s8d) over the HBM copy peak; the walk's "
                             "gathers are served by L1/L2 (ncu: DRAM traffic is a few % of them), so frac "
                             "can exceed 1 -- the binding roofline is roofline_issue"},
        "roofline_issue": roofline_issue,
        "roofline_l2": roofline_l2,
        "clocks": dict(clocks.summary(clocks.t_ramp, clocks.t_end), window=f"{args.ramp_s:.1f}s untimed ramp + timed region"),
        "gpu_launches": args.steps * ((1 if fg is None else sum(1 for a, b in fg.my_pieces() if b > a))
                                      * (4 if schedule == "binned" else 1)  # binned: count, scan, scatter, walk
                                      + (1 if pg is not None and pg.lean else 0)),  # lean p2p: root epilogue
        "parity": parity,
        "e2e": e2e,
        "e2e_render": e2e_render,
        "secondary": secondary,
    }
    if not args.no_cpu_baseline and world == 1:
        from concurrent.futures import ThreadPoolExecutor  # noqa: F401

        threads = os.cpu_count() or 1
        m = min(n, args.cpu_sample)
        t0 = time.perf_counter()
        reps = 0
        best = None
        while reps < 3 and (time.perf_counter() - t0) < 20.0:
            s0 = time.perf_counter()
            kind, _ = cpu_reference_trace(mesh, o[:m], d[:m], st[:m], threads)
            dt = time.perf_counter() - s0
            best = dt if best is None else min(best, dt)
            reps += 1
        m1 = min(m, 131072)
        line["cpu_baseline"] = {"value": m / best / 1e6, "unit": "Mrays/s", "cores": threads, "kind": kind,
                                "sample": f"first {m} rays of the frame, best of {reps}: compiled reference "
                                          "kernels + batch epilogue on a thread pool",
                                "single_thread": cpu_single_thread(mesh, o[:m1], d[:m1], st[:m1])}
    print(json.dumps(line), flush=True)
    if pg is not None:
        pg.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--layout", default=None)
    ap.add_argument("--scheme", default=None)
    ap.add_argument("--no-secondary", action="store_true", help="skip the secondary-ray measurement")
    ap.add_argument("--gather", choices=("p2p", "nccl"), default="p2p",
                    help="N > 1 frame assembly: fused P2P stores (default) or the chunked NCCL gather")
    ap.add_argument("--gather-chunks", type=int, default=4, help="N > 1: trace/gather pipeline depth per step")
    ap.add_argument("--schedule", default=None, choices=("auto", "lane", "refill", "compact", "compact512", "binned"),
                    help="ray-to-lane schedule of the timed trace (default: compact for secondaries, else lane)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-l2-probe", action="store_true", help="skip the L2 gather-roof probe (roofline_l2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=2_073_600)
    ap.add_argument("--ramp-s", type=float, default=0.5, help="untimed load before the timed region (clock ramp)")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--parity-sample", type=int, default=262_144, help="rays checked against the oracle")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    cfg = dict(CONFIGS[args.config])
    if args.layout:
        cfg["layout"] = args.layout
    if args.scheme:
        cfg["scheme"] = args.scheme
    if args.impl == "reference":
        run_reference_arm(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
