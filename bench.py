#!/usr/bin/env python
"""bench.py -- tet-mesh ray traversal throughput on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

``--gpus N`` without a torchrun environment relaunches itself under
``torch.distributed.run`` with N ranks (fails loudly when N exceeds the
visible GPUs).

Workload (BASELINE.json configs[1], the metric's single-GPU config):
config 2 = the reference's blob generator at GRID=55 (1,109,444 tets,
byte-identical to gen_model_mesh -> parse_tetgen -> encode, pinned by
tests/test_host_mirror.py), TetMesh-20, Hilbert-sorted, 1920x1080 primary
rays from the blob camera, all starting in the located camera tet.
A "step" traces one frame per GPU.  Weak scaling: at N GPUs the job is N
frames (camera moved per frame), 16x16 tiles dealt round-robin to ranks,
every ray's results stored into rank 0's frame arrays inside the trace
(P2P over NVLink) -- the frame set is assembled on rank 0 every step.

value    = rays / device time of the trace (CUDA events on the launch stream,
           inputs resident in HBM, 256 MiB written between steps to flush L2).
e2e      = the same metric through the C ABI with pinned HOST buffers
           (N=1: tb_cast_rays_host, rays read / hits written over PCIe; N>1:
           H2D of each rank's rays + fused trace/assembly + D2H of rank 0's
           assembled frame), per step.
roofline = the binding roof of the walk: instruction issue (SASS per step
           from tools/sass_steps.py x walk steps vs SMs x 4 schedulers x
           clock x 32 lanes).  The SURVEY s8(d) algorithmic bytes over HBM
           and over a measured L2 gather roof ride along as roofline_hbm /
           roofline_l2, ncu DRAM bytes per launch as roofline.traffic.
secondary_cfg4 = BASELINE config 4 (16.7 M diffuse secondaries from
           4096x4096 primary hits, Tet16) measured in the same run.
cpu_baseline / --impl reference = the reference's own public API
           (tetray.batch.cast_rays on its compiled kernels, installed under
           oracle/_ref/site) on all host threads.  The reference arm loads
           its scene with tetray.cli.load_compact from a file the reference's
           own pipeline wrote (oracle/make_ref_scene.py) and never maps this
           repo's CUDA library.
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
    # 1.6 GB TetMesh-32 (46.5 SASS per step) beats the 1 GB TetMesh-20 (53.75)
    # and the 0.8 GB TetMesh-16 (r02 A/B, profiles/r02_layouts.jsonl: 855 / 827 /
    # 720 Mrays/s)
    5: dict(kuhn=203, width=7680, height=4320, layout="tet32", scheme="none", sample_stride=64,
            desc="cfg5: Kuhn box n=203 (50,192,562 tets) stretched 4x in z with thin strip occluders "
                 "(long thin triangles), 7680x4320 primary rays, TetMesh-32"),
}
L2_FLUSH_BYTES = 256 << 20
FALLBACK_HBM_GBS = 6650.0
LAYOUT_BYTES = {"tet32": 32, "tet20": 20, "tet16": 16, "tet80": 80}
# layouts built on the device from the side tables (the host mesh stays Tet32)
DEVICE_BUILT = ("tet80",)


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


def config_dict(cfg, world: int) -> dict:
    """The workload description -- identical in both arms (the driver compares them)."""
    return {"workload": cfg["desc"], "rays_per_gpu": cfg["width"] * cfg["height"], "frames": world,
            "layout": cfg["layout"], "scheme": cfg["scheme"],
            "parallelism": f"tile-shard x{world}, mesh replicated" if world > 1 else "single GPU",
            "l2": "GPU arm writes 256 MiB between timed steps (L2 flush); CPU arm n/a"}


def camera_of(cfg, frame: int = 0):
    from paper_2103_02309_b200.workload import BLOB_CAMERA, kuhn_camera

    cam = dict(kuhn_camera(cfg["kuhn"]) if "kuhn" in cfg else BLOB_CAMERA)
    cam["position"] = tuple(np.asarray(cam["position"], dtype=np.float64) + np.array([0.0, 0.02, 0.0]) * frame)
    return cam


def frame_rays(cfg, frame: int):
    from paper_2103_02309_b200.workload import camera_rays

    cam = camera_of(cfg, frame)
    o, d = camera_rays(cam["position"], cam["look_at"], cam["up"], cam["fov"], cfg["width"], cfg["height"])
    return o, d, np.asarray(cam["position"], dtype=np.float64)


def sample_pixels(cfg) -> np.ndarray | None:
    """Config 5's reference sample: every 64th pixel."""
    s = cfg.get("sample_stride")
    return None if not s else np.arange(0, cfg["width"] * cfg["height"], s, dtype=np.int64)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list = []

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


# ---------------------------------------------------------------------------
# The reference's CPU path (oracle/_ref/site: the unmodified tetray package)

def ref_package():
    """The installed reference (oracle/_ref/site, built by oracle/build_ref.sh)."""
    site = os.path.join(ROOT, "oracle", "_ref", "site")
    if not os.path.isdir(os.path.join(site, "tetray")):
        raise RuntimeError(f"{site}/tetray missing: run oracle/build_ref.sh (or __graft_entry__.build())")
    if site not in sys.path:
        sys.path.insert(0, site)
    import tetray
    from tetray import backend

    if backend.active_backend() != "compiled":
        raise RuntimeError("the reference's compiled kernels did not import")
    return tetray


def ref_trace(mesh, o, d, st, threads: int, *, outputs: bool = False):
    """The reference's CPU path for one batch, through its public API:
    tetray.batch.cast_rays (compiled _kernels.cast_rays, GIL released, +
    the batch epilogue, batch.py:39-80) over a thread pool of >= 4096-ray
    chunks, the way its renderer's tile pool calls it (render.py:538-541).
    Returns the summed visited count (and the 7 arrays when ``outputs``)."""
    from concurrent.futures import ThreadPoolExecutor

    from tetray import batch

    n = len(st)
    chunks = max(1, min(threads * 16, n // 4096))
    bounds = np.linspace(0, n, chunks + 1).astype(np.int64)
    res = [None] * chunks

    def work(i):
        a, b = bounds[i], bounds[i + 1]
        if a == b:
            return 0
        h = batch.cast_rays(mesh, o[a:b], d[a:b], st[a:b])
        if outputs:
            res[i] = (h.status, h.cf, h.tet_front, h.visited, h.triangle, h.t, h.tet_back)
        return int(h.visited.sum())

    with ThreadPoolExecutor(max_workers=threads) as pool:
        total_vis = sum(pool.map(work, range(chunks)))
    if outputs:
        parts = [r for r in res if r is not None]
        return total_vis, [np.concatenate([p[k] for p in parts]) for k in range(7)]
    return total_vis


def ref_cast_full(mesh, o, d, st, threads: int):
    """The 7 result arrays of the reference (parity checker, never measured)."""
    return ref_trace(mesh, o, d, st, threads, outputs=True)[1]


def ref_scene(cfg):
    """The config's scene as a reference CompactMesh, never touching this
    repo's CUDA library: blob scenes from the file the reference's own
    pipeline wrote (oracle/make_ref_scene.py; built here if missing),
    re-encoded with the reference's relayout; the Kuhn box (too large for the
    reference's Python builder) from raw arrays dumped by a child process of
    the native builder, wrapped in the reference's CompactMesh."""
    ref_package()
    from tetray.cli import load_compact
    from tetray.tetmesh import LAYOUT_DTYPES, CompactMesh, SceneTriangleSoup, relayout

    layout = "tet32" if cfg["layout"] in DEVICE_BUILT else cfg["layout"]
    if "grid" in cfg:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import make_ref_scene

        path = make_ref_scene.scene_path(cfg["grid"], "tet20", cfg["scheme"])
        if not path.exists():
            log(f"[bench/ref] building {path.name} with the reference pipeline (minutes)")
            make_ref_scene.build(cfg["grid"], "tet20", cfg["scheme"])
        return relayout(load_compact(path), layout), "reference pipeline (oracle/make_ref_scene.py) + load_compact"
    out = os.path.join("/tmp", f"tetb200_kuhn{cfg['kuhn']}_{layout}_{cfg['scheme']}")
    if not os.path.exists(os.path.join(out, "done")):
        subprocess.run([sys.executable, os.path.abspath(__file__), "--dump-scene", str(cfg["kuhn"]), "--layout",
                        layout, "--scheme", cfg["scheme"], "--out", out], check=True)
    z = {k: np.load(os.path.join(out, k + ".npy")) for k in
         ("points", "records", "side_verts", "side_neighbors", "cf_triangle", "cf_tets", "cf_verts", "soup_vertices",
          "soup_triangles", "soup_materials", "source_tet")}
    mesh = CompactMesh(layout=layout, points=z["points"], records=z["records"].view(LAYOUT_DTYPES[layout]).reshape(-1),
                       side_verts=z["side_verts"], side_neighbors=z["side_neighbors"], cf_triangle=z["cf_triangle"],
                       cf_tets=z["cf_tets"], cf_verts=z["cf_verts"], source_tet=int(z["source_tet"]),
                       soup=SceneTriangleSoup(vertices=z["soup_vertices"], triangles=z["soup_triangles"],
                                              material_ids=z["soup_materials"]))
    return mesh, "native builder arrays (child process) wrapped in the reference's CompactMesh"


def dump_scene(n: int, layout: str, scheme: str, out: str):
    """--dump-scene: the config-5 Kuhn mesh as raw .npy arrays for the reference arm."""
    from paper_2103_02309_b200.scenes import kuhn_strip_scene

    m = kuhn_strip_scene(n, layout=layout, scheme=scheme).mesh
    os.makedirs(out, exist_ok=True)
    for k, v in (("points", m.points), ("records", m.records_u32()), ("side_verts", m.side_verts),
                 ("side_neighbors", m.side_neighbors), ("cf_triangle", m.cf_triangle), ("cf_tets", m.cf_tets),
                 ("cf_verts", m.cf_verts), ("soup_vertices", m.soup.vertices), ("soup_triangles", m.soup.triangles),
                 ("soup_materials", m.soup.material_ids), ("source_tet", np.array(m.source_tet))):
        np.save(os.path.join(out, k + ".npy"), np.ascontiguousarray(v))
    open(os.path.join(out, "done"), "w").close()


def ref_rays(cfg, mesh, frame: int = 0, pixels=None):
    """Rays of the config through the reference's own camera
    (render.camera_rays, render.py:169-185) and its locate_points."""
    from tetray import batch
    from tetray.render import RenderConfig, camera_rays

    cam = camera_of(cfg, frame)
    W, H = cfg["width"], cfg["height"]
    rc = RenderConfig(camera_position=cam["position"], camera_look_at=cam["look_at"], camera_up=cam["up"],
                      fov=cam["fov"], width=W, height=H)
    pix = np.arange(W * H, dtype=np.int64) if pixels is None else pixels
    o, d = camera_rays(rc, (pix % W).astype(np.float64), (pix // W).astype(np.float64))
    cam_tet, _ = batch.locate_points(mesh, np.asarray(cam["position"], dtype=np.float64)[None])
    return np.ascontiguousarray(o), np.ascontiguousarray(d), np.full(len(o), int(cam_tet[0]), np.int32)


def native_libs_loaded() -> list:
    """In-tree shared objects mapped into this process (reference-arm hygiene)."""
    libs = set()
    try:
        for line in open("/proc/self/maps"):
            p = line.split()[-1] if line.strip() else ""
            if p.endswith(".so") or ".so." in p:
                if p.startswith(ROOT):
                    libs.add(os.path.relpath(p, ROOT))
    except OSError:
        pass
    return sorted(libs)


def run_reference_arm(args, cfg):
    world, rank, _ = dist_env()
    world = max(world, args.gpus)
    if rank != 0:
        return
    t0 = time.perf_counter()
    tetray = ref_package()
    mesh, scene_src = ref_scene(cfg)
    log(f"[bench/ref] scene {mesh.n_tets} tets ({scene_src}) in {time.perf_counter() - t0:.1f}s")
    threads = os.cpu_count() or 1
    pix = sample_pixels(cfg)
    o, d, st = ref_rays(cfg, mesh, 0, pix)
    sample = f"frame 0, {len(o)} rays" + (" (every 64th pixel)" if pix is not None else " (full frame)")
    if cfg.get("secondaries"):
        from paper_2103_02309_b200.workload import diffuse_secondaries

        _, prim = ref_trace(mesh, o, d, st, threads, outputs=True)  # untimed: the primaries
        o, d, st = diffuse_secondaries(o, d, prim[5], prim[4], prim[2], mesh.triangle_coords(), seed=4)
        m = min(len(st), args.ref_sample)
        o, d, st = o[:m], d[:m], st[:m]
        sample = f"first {m} of the frame's diffuse secondaries (seed 4)"
    for _ in range(args.warmup):
        ref_trace(mesh, o, d, st, threads)
    times = []
    vis = 0
    for _ in range(args.steps):
        s0 = time.perf_counter()
        vis = ref_trace(mesh, o, d, st, threads)
        times.append(time.perf_counter() - s0)
    total = sum(times)
    value = len(st) * args.steps / total / 1e6
    line = {
        "impl": "reference", "metric": "Mrays/s", "value": value, "unit": "Mrays/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(cfg, world),
        "tets_visited_per_ray": {"mean": vis / len(st)},
        "cpu_baseline": {"value": value, "unit": "Mrays/s", "cores": threads, "kind": "reference",
                         "sample": sample + ": tetray.batch.cast_rays (compiled kernels + batch epilogue), "
                                            "ThreadPoolExecutor over min(16 per thread, n / 4096) chunks"},
        "e2e": {"value": value, "unit": "Mrays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference": {"package": os.path.relpath(os.path.dirname(tetray.__file__), ROOT), "scene": scene_src,
                      "layout_note": ("the reference has no TetMesh-80 and no ScTP walk: its 2-D walk on the "
                                      "Tet32 mesh of the same scene and rays") if cfg["layout"] == "tet80" else None},
        "native_so_loaded": native_libs_loaded(),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Our arm

def build_scene(cfg):
    from paper_2103_02309_b200.scenes import blob_scene, kuhn_strip_scene

    t0 = time.perf_counter()
    if "kuhn" in cfg:
        sc = kuhn_strip_scene(cfg["kuhn"], layout=cfg["layout"], scheme=cfg["scheme"])
    else:
        host_layout = "tet32" if cfg["layout"] in DEVICE_BUILT else cfg["layout"]
        sc = blob_scene(cfg["grid"], layout=host_layout, scheme=cfg["scheme"], check=False)
    log(f"[bench] scene {sc.name}: {sc.mesh.n_tets} tets, {sc.mesh.n_points} points, "
        f"{sc.mesh.n_constrained} constrained faces, built in {time.perf_counter() - t0:.1f}s")
    return sc


def digest(*arrays) -> str:
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def algorithmic_bytes(visited: np.ndarray, layout: str) -> int:
    """sum_rays [(visited-1)(L+12) + 68] + 53 N."""
    L = LAYOUT_BYTES[layout]
    point = 0 if layout == "tet80" else 12
    v = visited.astype(np.int64)
    return int(((v - 1) * (L + point)).sum() + 68 * len(v) + 53 * len(v))


def timed(fn, steps: int, warmup: int, stream, flush):
    """Device time per call (ms): CUDA events on the launch stream, L2 flushed before each."""
    import torch

    for _ in range(warmup):
        flush.zero_()
        fn()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for a, b in evs:
        flush.zero_()
        a.record(stream)
        fn()
        b.record(stream)
    torch.cuda.synchronize()
    return np.array([a.elapsed_time(b) for a, b in evs])


# sm_100 pipe rates (B300_MICROARCH.md "Pipe rates": IADD3/LOP3/SHF/PRMT/SEL/
# compares on the ALU pipe at one warp instruction per 2 cycles per SMSP; ncu
# sm__inst_executed_pipe_alu of the config-2 walk = 62.6 % of that peak)
ALU_CYCLES_PER_INST = 2


def issue_roof(layout: str, schedule: str, walk_steps: float, kern_s: float, clk_mhz, sms: int):
    """The walk's binding roof from its SASS (tools/sass_steps.py, committed
    per build): a warp-step needs max(SASS per step, 2 x ALU-pipe SASS per
    step) scheduler cycles -- whichever of instruction issue and the ALU pipe
    binds (the ALU pipe for every layout: tet20 2 x 27.5 > 53.75)."""
    sp = os.path.join(ROOT, "profiles", "sass_step_counts.json")
    if not (os.path.exists(sp) and clk_mhz):
        return None
    counts = json.load(open(sp))
    kname = "cast_compact_kernel" if schedule in ("compact", "compact512") else "cast_kernel"
    entry = counts.get(f"{kname}<{layout[3:]}, validated>") or counts.get(f"{kname}<{layout[3:]}, clamp>")
    if not entry:
        return None
    mix = next((v for k, v in entry.items() if k.startswith("unrolled_x")), None) or entry["single_step"]
    per_step, alu = mix["total"], mix["alu"]
    cycles = max(per_step, ALU_CYCLES_PER_INST * alu)
    peak_steps = sms * 4 * clk_mhz * 1e6 * 32 / cycles
    issue_peak = sms * 4 * clk_mhz * 1e6 * 32 / per_step
    ach = walk_steps / kern_s
    return {"bound": "alu_pipe" if cycles > per_step else "issue", "achieved": ach / 1e9, "peak": peak_steps / 1e9,
            "unit": "G ray-steps/s", "frac": ach / peak_steps, "sass_per_step": per_step, "alu_per_step": alu,
            "cycles_per_warp_step": cycles, "issue_frac": ach / issue_peak, "sms": sms, "sm_mhz": clk_mhz,
            "note": "peak = SMs x 4 schedulers x SM clock x 32 lanes / max(SASS, 2 x ALU-pipe SASS) per walk step; "
                    "the gap is init/epilogue, SIMT divergence, latency stalls and the tail"}


def l1_pipe_roof(key: str, kern_s: float, clk_mhz, sms: int):
    """The L1 data pipe as a roof (the incoherent walk's binding unit, ncu
    r02): the walk's LSU wavefronts per launch, counted once by ncu for this
    workload (profiles/pipe_util.json, tools/evidence_from_ncu.py), over the
    live kernel time, against SMs x wavefronts per SM cycle x the live SM
    clock.  None when no capture counted them."""
    p = pipes_of(key) or {}
    wf, per_cycle = p.get("l1tex_lsu_wavefronts_per_launch"), p.get("l1tex_lsu_wavefronts_peak_per_sm_cycle")
    if not (wf and per_cycle and clk_mhz):
        return None
    peak = sms * per_cycle * clk_mhz * 1e6
    return {"bound": "l1_data_pipe", "achieved": wf / kern_s / 1e9, "peak": peak / 1e9, "unit": "G wavefronts/s",
            "frac": wf / kern_s / peak, "wavefronts_per_launch": wf, "sms": sms, "sm_mhz": clk_mhz,
            "note": "L1TEX data-pipe (LSU) wavefronts of the walk per launch from one ncu capture of this workload, "
                    "over the live kernel time; peak = SMs x wavefronts per SM cycle (ncu) x live SM clock"}


def binding_roof(alu, l1):
    """The roof that binds: the larger utilisation of the ALU-pipe issue roof
    and the L1 data-pipe roof; the other rides along."""
    if l1 is None:
        return alu
    if alu is None or l1["frac"] > alu["frac"]:
        return dict(l1, roofline_alu_pipe=alu)
    return dict(alu, roofline_l1_data_pipe=l1)


def pipes_of(key: str):
    """ncu pipe / L1 utilisation of the walk (profiles/pipe_util.json)."""
    pp = os.path.join(ROOT, "profiles", "pipe_util.json")
    if os.path.exists(pp):
        return json.load(open(pp)).get(key)
    return None


def traffic_of(key: str):
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        return json.load(open(tp)).get(key)
    return None


def l2_gather_roof(dm, stream, flush, layout: str, walk_steps: float, achieved_gbs: float) -> dict:
    """for meshes that fit in L2, the walk's algorithmic bytes
    against a measured random-gather roof of the same mesh -- tb_probe_gather
    issues one step's loads (record + axis-permuted point) at independent
    pseudo-random indices, 8 per thread in flight, L2 flushed before each
    rep like the timed steps."""
    import torch

    from paper_2103_02309_b200._lib import check, lib

    L = LAYOUT_BYTES[layout]
    n_pairs = int(min(max(32 << 20, walk_steps), 256 << 20))
    sink = torch.zeros(1, dtype=torch.int32, device=flush.device)

    def probe():
        check(lib.tb_probe_gather(dm.handle, n_pairs, 12345, sink.data_ptr(), stream.cuda_stream), "tb_probe_gather")

    t = float(np.median(timed(probe, 5, 2, stream, flush))) / 1e3
    peak = n_pairs * (L + 12) / t / 1e9
    l2 = torch.cuda.get_device_properties(flush.device).L2_cache_size
    return {"bound": "l2_gather", "achieved": achieved_gbs, "peak": peak, "unit": "GB/s", "frac": achieved_gbs / peak,
            "probe": {"kernel": f"gather_probe_kernel<{L}>", "pairs": n_pairs, "bytes_per_pair": L + 12,
                      "ms": t * 1e3, "working_set_bytes": int(dm.hot_bytes), "l2_bytes": int(l2)},
            "note": "peak = random (record, point) gathers over this mesh's hot arrays; the walk exceeds it when "
                    "coherent rays share L1/L2 lines (frac > 1) -- its binding roof is `roofline` (issue)"}


def parity_vs_reference(mesh, o, d, st, got, stride: int, threads: int, layout: str) -> dict:
    """A strided sample of rays against the reference itself (oracle/_ref/
    site: tetray.batch.cast_rays on its compiled kernels) -- the checker."""
    sl = slice(0, len(st), stride)
    exp = ref_cast_full(mesh_for_ref(mesh, {"layout": layout}), o[sl], d[sl], st[sl], threads)
    names = ("status", "cf", "tet", "visited", "triangle", "t", "tet_back")
    mism = {k: int(np.count_nonzero(g[sl] != e)) for k, g, e in zip(names, got, exp)}
    tg, te = got[5][sl], exp[5]
    fin = np.isfinite(tg) & np.isfinite(te)
    t_rel = float((np.abs(tg[fin] - te[fin]) / np.maximum(np.abs(te[fin]), 1e-30)).max(initial=0.0))
    return {"vs": f"reference tetray.batch.cast_rays (oracle/_ref) on every {stride}th ray",
            "rays_checked": int(len(exp[0])), "mismatched_values": mism, "bit_exact": not any(mism.values()),
            # the contract's float tolerance for t (the live reference epilogue
            # runs on this box's numpy; the kernel pins numpy 2.3's einsum order)
            "t_max_rel_err": t_rel, "numpy": np.__version__,
            "within_contract": not any(v for k, v in mism.items() if k != "t") and t_rel <= 1e-5}


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
    ndev = torch.cuda.device_count()
    if world > ndev and backend == "nccl":
        raise SystemExit(f"--gpus {world} but only {ndev} visible GPU(s)")
    local = local % ndev
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
    dm = device_mesh(mesh, device=local, layout=cfg["layout"] if cfg["layout"] in DEVICE_BUILT else None)
    sctp = cfg.get("walk") == "sctp"
    W, H = cfg["width"], cfg["height"]
    per_frame = W * H
    threads = os.cpu_count() or 1

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
        from paper_2103_02309_b200.workload import diffuse_secondaries

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

    # ray schedule: incoherent secondaries (config 4) are binned by direction
    # cell first (96 cube-map cells) and walked in binned order (r01: 3.36 vs
    # 2.37 Grays/s one ray per lane); primaries take "auto": the sampled
    # longest-first block order, split so its pre-pass hides under the head of
    # the launch, for launches of 6-48 waves (configs 2 and 3), one ray per
    # lane otherwise (tb_auto_schedule)
    schedule = args.schedule or ("binned" if cfg.get("secondaries") else "auto")
    if schedule == "auto" and world == 1 and not sctp:
        from paper_2103_02309_b200._lib import SCHEDULES

        resolved = int(lib.tb_auto_schedule(local, n))
        schedule = next(k for k, v in SCHEDULES.items() if v == resolved)
    split = schedule == "sampled" and world == 1 and int(lib.tb_sampled_head_blocks(local, n)) > 0

    def step():
        trace(dm, go, gd, gs, out=res, stream=stream, sctp=sctp, schedule=schedule)

    fg = pg = None
    gather_mode = None
    if world > 1 and args.gather == "p2p":
        # every step assembles its frame set on rank 0 inside the trace: each
        # rank's kernel stores every finished ray into rank 0's full-frame
        # arrays (CUDA IPC, P2P over NVLink) -- no collective moves the hits
        try:
            lean = not cfg.get("secondaries")  # secondaries are spawned per rank: the root lacks their rays
            root_rays = None
            if lean:
                root_rays = True
                if rank == 0:  # the job's rays in global order (frame-major), resident on rank 0 (untimed setup)
                    frs = [frame_rays(cfg, f)[:2] for f in range(world)]
                    root_rays = tuple(torch.from_numpy(np.ascontiguousarray(np.concatenate([fr[i] for fr in frs])))
                                      .to(dev) for i in (0, 1))
            # pipelined: rank 0's whole-job epilogue of step k overlaps step k+1's trace
            pg = multigpu.PeerFrameGather(W, H, world, rank, world, dev, root_rays=root_rays, index=idx,
                                          pipelined=lean)
            gather_mode = "p2p"

            def step():  # noqa: F811  (the N > 1 step: fused trace + frame assembly)
                return pg.step(dm, go, gd, gs, stream, schedule=schedule, sctp=sctp)
        except Exception as exc:  # no peer access / IPC: fall back to the NCCL gather
            log(f"[bench] p2p frame assembly unavailable ({exc!r}); using the NCCL gather")
            pg = None
    if world > 1 and pg is None:
        # every step gathers its frame set to rank 0: the shard is traced in
        # chunks and each chunk's 20 B records go out with an async NCCL
        # gather while the next chunk traces (multigpu.FrameGather)
        from paper_2103_02309_b200.trace import TraceResult

        gather_mode = "nccl"
        fg = multigpu.FrameGather(W, H, world, rank, world, args.gather_chunks, dev, mesh.cf_triangle, mesh.cf_tets,
                                  index=idx)
        pieces = fg.my_pieces()
        views = [TraceResult(*(getattr(res, f)[a:b] for f in ("status", "cf", "triangle", "t", "tet", "tet_back",
                                                                 "visited"))) for (a, b) in pieces]

        def step():  # noqa: F811  (the N > 1 step: trace + per-frame gather)
            for k, ((a, b), v) in enumerate(zip(pieces, views)):
                if b > a:
                    trace(dm, go[a:b], gd[a:b], gs[a:b], out=v, stream=stream, sctp=sctp, schedule=schedule)
                fg.send(k, v.status, v.cf, v.tet, v.visited, v.t)
            return fg.finish()

    for _ in range(args.warmup):
        flush.zero_()
        step()
    if pg is not None:
        pg.finish()
    torch.cuda.synchronize()
    if pg is not None and rank == 0:
        # p2p: this rank's hits live in the root's frame
        from paper_2103_02309_b200.trace import TraceResult as _TR

        gidx = torch.from_numpy(idx).to(dev)
        res = _TR(*(pg.frame[k][gidx] for k in ("status", "cf", "triangle", "t", "tet", "tet_back", "visited")))

    # parity at full size: the reference's own digest of this frame (N=1,
    # config 2 / config 1 sizes); otherwise a strided sample vs the reference
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

            parity = {"vs": "reference digest " + key,
                      "traversal_bit_exact": digest(rm(res.status), rm(res.cf), rm(res.tet), rm(res.visited))
                      == digs[key],
                      "epilogue_bit_exact": digest(rm(res.triangle), rm(res.t), rm(res.tet_back))
                      == digs[key.replace("/cast", "/epilogue")]}
    got_all = None
    if parity is None and rank == 0 and not args.no_parity:
        got_all = [x.cpu().numpy() for x in (res.status, res.cf, res.tet, res.visited, res.triangle, res.t,
                                             res.tet_back)]
        parity = parity_vs_reference(mesh, o, d, st, got_all, max(1, n // args.parity_sample), threads,
                                     cfg["layout"])
        if sctp:
            # the ScTP walk has no reference implementation: bit-exact vs its C
            # restatement; vs the reference's 2-D walk only ties may differ
            from oracle import pyoracle

            sl = slice(0, n, max(1, n // args.parity_sample))
            exp = pyoracle.cast_rays_full(mesh, o[sl], d[sl], st[sl], layout=dm.layout, sctp=True)
            parity["sctp_vs_c_restatement_bit_exact"] = all(np.array_equal(g[sl], e) for g, e in zip(got_all, exp))
            parity["note"] = "ScTP vs the reference's 2-D walk: mismatches are exact ties (SURVEY s8 a-14)"

    # visited statistics over the rays actually traced (every rank's own)
    visited_mine = res.visited.cpu().numpy() if (pg is None or rank == 0) else None
    if pg is not None and rank != 0:
        visited_mine = None  # lives in rank 0's frame; rank 0 reports the whole job's below

    # timed region: K steps between barrier + sync; per-step kernel events.
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
        if pg is not None and pg.pipelined:
            # the last step's pipelined root epilogue belongs to the timed work
            evs.append((torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)))
            evs[-1][0].record(stream)
            pg.finish()
            evs[-1][1].record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        clocks.mark("t_end")
        if world > 1:
            dist.barrier()
        time.sleep(0.05)
    kernel_ms = np.array([a.elapsed_time(b) for a, b in evs])
    if world > 1:
        # N > 1: the assembled frame set of the last step, checked on rank 0
        try:
            full = step()
            if pg is not None:
                full = pg.finish()
            torch.cuda.synchronize()
            if full is not None:
                gather_check = {"rays_in_frame": int((full["visited"] > 0).sum().item())}
                if os.path.exists(dig_path) and "grid" in cfg and (W, H) == (1920, 1080) \
                        and not cfg.get("secondaries") and cfg["layout"] != "tet80":
                    digs = json.load(open(dig_path))
                    if key in digs:  # frame 0 is the reference camera: compare with its digest
                        f0 = [full[k][:per_frame].cpu().numpy() for k in ("status", "cf", "tet", "visited")]
                        e0 = [full[k][:per_frame].cpu().numpy() for k in ("triangle", "t", "tet_back")]
                        gather_check["frame0_vs_reference_digest"] = digest(*f0) == digs[key]
                        gather_check["frame0_epilogue_vs_reference_digest"] = \
                            digest(*e0) == digs[key.replace("/cast", "/epilogue")]
        except Exception as exc:  # report, do not lose the line
            gather_error = repr(exc)
    my_ms = float(kernel_ms.sum())
    if world > 1:
        t = torch.tensor([my_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        max_ms = float(t.item())
        if pg is not None:  # every traced ray's visited count is in rank 0's frame
            fv = pg.frame["visited"].cpu().numpy() if rank == 0 else np.zeros(0, np.int32)
            vt = torch.tensor([int(fv.sum()), int(fv.max(initial=0)), n], dtype=torch.int64, device=dev)
        else:
            vt = torch.tensor([int(visited_mine.sum()), int(visited_mine.max(initial=0)), n], dtype=torch.int64,
                              device=dev)
        vsum = vt.clone()
        dist.all_reduce(vsum, op=dist.ReduceOp.SUM)
        dist.all_reduce(vt, op=dist.ReduceOp.MAX)
        vis_sum, vis_max, total_rays = int(vsum[0]), int(vt[1]), int(vsum[2])
    else:
        max_ms = my_ms
        vis_sum, vis_max, total_rays = int(visited_mine.sum()), int(visited_mine.max()), n

    value = total_rays * args.steps / (max_ms / 1e3) / 1e6
    ms_per_step = max_ms / args.steps

    # end to end with pinned HOST buffers, per step
    e2e = None
    if not args.no_e2e:
        ho = torch.from_numpy(o).pin_memory()
        hd = torch.from_numpy(d).pin_memory()
        hs = torch.from_numpy(st).pin_memory()
        if world == 1:
            outs = [torch.empty(n, dtype=dt).pin_memory() for dt in
                    (torch.uint8, torch.int32, torch.int32, torch.int32, torch.int32, torch.float64, torch.int32)]
            host_fn = lib.tb_sctp_cast_rays_host if sctp else lib.tb_cast_rays_host

            def e2e_call():
                check(host_fn(dm.handle, n, addr(ho), addr(hd), addr(hs), *[addr(x) for x in outs]),
                      "tb_sctp_cast_rays_host" if sctp else "tb_cast_rays_host")
            h2d, d2h = n * (12 + 12 + 4), n * (1 + 4 * 5 + 8)
            path = (f"{'tb_sctp_cast_rays_host' if sctp else 'tb_cast_rays_host'} (C ABI) on pinned host buffers: "
                    "zero-copy trace over PCIe")
        else:
            # each rank: its rays host -> HBM, the fused trace + frame assembly
            # into rank 0, and rank 0 copies the assembled job back to the host
            full0 = step()  # every rank (the step may hold collectives); rank 0 gets the frame set
            if pg is not None:
                full0 = pg.finish()
            fr_host = None
            if rank == 0:
                fr_host = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in full0.items()}

            def e2e_call():
                go.copy_(ho, non_blocking=True)
                gd.copy_(hd, non_blocking=True)
                gs.copy_(hs, non_blocking=True)
                full = step()
                if pg is not None:
                    full = pg.finish()  # this step's frame set, complete
                if rank == 0:
                    for k2, v2 in full.items():
                        fr_host[k2].copy_(v2, non_blocking=True)
                torch.cuda.synchronize()
            h2d = n * (12 + 12 + 4)
            d2h = (total_rays * 29) if rank == 0 else 0
            path = ("H2D of each rank's rays (pinned), fused trace + P2P frame assembly on rank 0, D2H of the "
                    "assembled frame set (29 B/ray) from rank 0, synchronised; max over ranks")
        for _ in range(max(1, args.warmup)):
            e2e_call()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_call()
        e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_s = float(t.item())
        e2e = {"value": total_rays * args.steps / e_s / 1e6, "unit": "Mrays/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_s / args.steps * 1e3, "path": path}

    extra = {}
    if world == 1 and not cfg.get("secondaries") and not sctp:
        if not args.no_secondary:
            extra["secondary"] = frame_secondaries(args, cfg, mesh, dm, o, d, res, stream, flush, threads)
        if not args.no_cfg4 and args.config == 2:
            extra["secondary_cfg4"] = config4_secondaries(args, mesh, stream, flush, threads, clocks)
        if not args.no_e2e:
            extra["e2e_render"] = render_e2e(args, cfg, dm, stream, sctp)
        if not args.no_small_batch:
            extra["small_batch"] = small_batch(args, mesh, o, d, st, threads)

    if rank != 0:
        if pg is not None:
            pg.close()
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = measured_peak()
    alg = algorithmic_bytes(visited_mine, cfg["layout"])  # this rank's launch
    kern_s = float(kernel_ms.mean()) / 1e3
    clk = clocks.summary(clocks.t_ramp, clocks.t_end)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    walk_steps = (vis_sum - total_rays) / world  # one rank's launch
    roof = issue_roof(cfg["layout"], schedule, walk_steps, kern_s, clk.get("sm_mhz"), sms) if not sctp else None
    if not sctp:
        roof = binding_roof(roof, l1_pipe_roof(f"cfg{args.config}/{cfg['layout']}", kern_s, clk.get("sm_mhz"), sms))
    traffic = traffic_of(f"cfg{args.config}/{cfg['layout']}")
    kname = (f"sctp_kernel<{cfg['layout'][3:]}>" if sctp else
             f"{'cast_compact_kernel' if schedule in ('compact', 'compact512') else 'cast_kernel'}"
             f"<{cfg['layout'][3:]}>" + (" after bin_count/bin_seg_scan/bin_scatter (direction binning, inside "
                                          "the events; in two pieces of whole sorting segments when "
                                          "tb_binned_pieces says so: the second binned on a high-priority side "
                                          "stream beside the first one's walk)" if schedule == "binned" else
                                          (" with its tail's blocks launched longest first: the head walks in "
                                           "launch order while block_probe/block_scatter (a capped one-ray-per-block "
                                           "pre-pass) order the tail on a high-priority side stream, all inside the "
                                           "events" if split else
                                           " with its blocks launched longest first, after block_probe/"
                                           "block_scatter (a capped one-ray-per-block pre-pass, inside the events)")
                                          if schedule == "sampled" else ""))
    hbm = {"bound": "hbm", "achieved": alg / kern_s / 1e9, "peak": peak, "unit": "GB/s", "peak_source": peak_src,
           "algorithmic_bytes_per_launch": alg,
           "frac": alg / kern_s / 1e9 / peak,
           "dram_bytes_per_launch": traffic,
           "dram_frac": (traffic / kern_s / 1e9 / peak) if traffic else None,
           "note": "SURVEY s8(d) algorithmic gather bytes over the HBM copy peak: the walk's gathers are served "
                   "by L1/L2 (DRAM sees a few % of them, dram_bytes_per_launch from ncu), so this can exceed 1 "
                   "and is not the binding roof"}
    if roof is None:
        roof = dict(hbm)
    roof = dict(roof, traffic=traffic, kernel=kname, ncu_pipes=pipes_of(f"cfg{args.config}/{cfg['layout']}"))
    line = {
        "metric": "Mrays/s", "value": value, "unit": "Mrays/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(cfg, world),
        "schedule": schedule, "rays_per_step": total_rays,
        "tets_visited_per_ray": {"mean": vis_sum / total_rays, "max": vis_max},
        "kernel_ms": {"mean": float(kernel_ms.mean()), "min": float(kernel_ms.min()), "max": float(kernel_ms.max())},
        "gather": None if world == 1 else {
            "mode": gather_mode, "check": gather_check, "error": gather_error,
            "per_step": ("every step assembles its frame set on rank 0 inside the timed region: each rank's trace "
                         "epilogue stores every finished ray into rank 0's full-frame arrays (CUDA IPC, P2P over "
                         "NVLink), then stream sync + barrier" if gather_mode == "p2p" else
                         "every step gathers its frame set to rank 0 inside the timed region (chunked NCCL "
                         "gather, overlapped with the trace)"),
            "bytes_to_rank0_per_step": int((13 if (pg is not None and pg.lean) else (29 if pg is not None else 20))
                                           * (total_rays - n)),
            "lean": bool(pg is not None and pg.lean)},
        "wall_ms_per_step": wall / args.steps * 1e3,
        "roofline": roof,
        "roofline_hbm": hbm,
        "roofline_l2": (l2_gather_roof(dm, stream, flush, cfg["layout"], walk_steps, alg / kern_s / 1e9)
                        if (not sctp and cfg["layout"] != "tet80" and not args.no_l2_probe) else None),
        "clocks": dict(clk, window=f"{args.ramp_s:.1f}s untimed ramp + timed region"),
        "gpu_launches": args.steps * ((1 if fg is None else sum(1 for a, b in fg.my_pieces() if b > a))
                                      * (4 * (int(lib.tb_binned_pieces(n)) if pg is None else 1)
                                         if schedule == "binned" else
                                         ((4 if split else 3) if schedule == "sampled" else 1))
                                      # binned: count, scan, scatter, walk (per piece); sampled: probe,
                                      # scatter, walk
                                      # (+ the head's walk when split)
                                      + (1 if (pg is not None and schedule == "binned") else 0)  # compose
                                      + (1 if pg is not None and pg.lean else 0)),  # lean p2p: root epilogue
        "parity": parity,
        "e2e": e2e,
        "mesh_bytes": {"hbm_total": int(dm.hbm_bytes), "hot": int(dm.hot_bytes),
                       "reference_accelerator_bytes": int(mesh.records_u32().nbytes + mesh.points.nbytes)},
        **extra,
    }
    if not args.no_cpu_baseline and world == 1:
        m = min(n, args.cpu_sample)
        t0 = time.perf_counter()
        reps, best = 0, None
        while reps < 3 and (time.perf_counter() - t0) < 20.0:
            s0 = time.perf_counter()
            ref_trace(mesh_for_ref(mesh, cfg), o[:m], d[:m], st[:m], threads)
            dt = time.perf_counter() - s0
            best = dt if best is None else min(best, dt)
            reps += 1
        line["cpu_baseline"] = {"value": m / best / 1e6, "unit": "Mrays/s", "cores": threads, "kind": "reference",
                                "sample": f"first {m} rays of the frame, best of {reps}: the reference's "
                                          "tetray.batch.cast_rays (compiled kernels + batch epilogue, oracle/_ref) "
                                          "on a thread pool"
                                          + (" on the Tet32 mesh, 2-D walk (no TetMesh-80 / ScTP in the reference)"
                                             if cfg["layout"] == "tet80" else "")}
    print(json.dumps(line), flush=True)
    if pg is not None:
        pg.close()
    if world > 1:
        dist.destroy_process_group()


def mesh_for_ref(mesh, cfg):
    ref_package()
    if cfg["layout"] in DEVICE_BUILT:
        from paper_2103_02309_b200.tetmesh import relayout

        return relayout(mesh, "tet32")
    return mesh


def frame_secondaries(args, cfg, mesh, dm, o, d, res, stream, flush, threads):
    """The frame's own diffuse bounces (render.py:353-359 semantics, seed 4),
    binned and one ray per lane, parity-sampled against the reference."""
    import torch

    from paper_2103_02309_b200.trace import empty_result, trace
    from paper_2103_02309_b200.workload import diffuse_secondaries

    dev = flush.device
    so, sd, sst = diffuse_secondaries(o, d, res.t.cpu().numpy(), res.triangle.cpu().numpy(), res.tet.cpu().numpy(),
                                      mesh.triangle_coords(), seed=4)
    ns = len(sst)
    if not ns:
        return None
    g2 = [torch.from_numpy(a).to(dev) for a in (so, sd, sst)]
    r2 = empty_result(ns, dev)
    ms = {}
    for sched in ("lane", "binned"):
        ms[sched] = float(timed(lambda: trace(dm, *g2, out=r2, stream=stream, schedule=sched), args.steps,
                                args.warmup, stream, flush).mean())
    v2 = r2.visited.cpu().numpy()
    par = None
    if not args.no_parity:
        got = [x.cpu().numpy() for x in (r2.status, r2.cf, r2.tet, r2.visited, r2.triangle, r2.t, r2.tet_back)]
        par = parity_vs_reference(mesh, so, sd, sst, got, max(1, ns // args.parity_sample), threads, cfg["layout"])
    return {"value": ns / ms["binned"] / 1e3, "unit": "Mrays/s", "rays": ns, "kernel_ms": ms["binned"],
            "schedule": "binned", "one_ray_per_lane": {"value": ns / ms["lane"] / 1e3, "kernel_ms": ms["lane"]},
            "tets_visited_per_ray": {"mean": float(v2.mean()), "max": int(v2.max())},
            "rays_from": "diffuse hemisphere bounces of this frame's primary hits (seed 4)", "parity": par}


def config4_secondaries(args, mesh20, stream, flush, threads, clocks):
    """BASELINE config 4 inside the default run: 4096x4096 primaries on the
    Tet16 encoding of the same scene (untimed), their 16.7 M diffuse
    secondaries (render.py:353-359 semantics, seed 4) traced binned and one
    ray per lane (timed), parity on a strided sample vs the reference."""
    import torch

    from paper_2103_02309_b200.device import DeviceMesh
    from paper_2103_02309_b200.tetmesh import relayout
    from paper_2103_02309_b200.trace import empty_result, locate, trace
    from paper_2103_02309_b200.workload import diffuse_secondaries

    from paper_2103_02309_b200.multigpu import shard_pixels

    cfg = CONFIGS[4]
    dev = flush.device
    mesh = relayout(mesh20, cfg["layout"])
    dm = DeviceMesh(mesh, dev.index)
    o, d, pos = frame_rays(cfg, 0)
    # the reference renderer traces (and spawns secondaries) per 16x16 tile
    # (render.py:496-514, 538-541): rays in tile order, as bench.py --config 4
    tiles = shard_pixels(cfg["width"], cfg["height"], 0, 1, 16)
    o, d = o[tiles], d[tiles]
    cam, _ = locate(dm, torch.tensor(pos[None], dtype=torch.float64, device=dev),
                    torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
    st = np.full(len(o), int(cam.item()), np.int32)
    prim = trace(dm, torch.from_numpy(o).to(dev), torch.from_numpy(d).to(dev), torch.from_numpy(st).to(dev))
    so, sd, sst = diffuse_secondaries(o, d, prim.t.cpu().numpy(), prim.triangle.cpu().numpy(), prim.tet.cpu().numpy(),
                                      mesh.triangle_coords(), seed=4)
    del prim
    ns = len(sst)
    g2 = [torch.from_numpy(a).to(dev) for a in (so, sd, sst)]
    r2 = empty_result(ns, dev)
    ms = {}
    for sched in ("lane", "binned"):
        ms[sched] = timed(lambda: trace(dm, *g2, out=r2, stream=stream, schedule=sched), args.steps, args.warmup,
                          stream, flush)
    v2 = r2.visited.cpu().numpy()
    par = None
    if not args.no_parity:
        got = [x.cpu().numpy() for x in (r2.status, r2.cf, r2.tet, r2.visited, r2.triangle, r2.t, r2.tet_back)]
        par = parity_vs_reference(mesh, so, sd, sst, got, max(1, ns // args.parity_sample), threads, "tet16")
    kb = float(ms["binned"].mean())
    clk = clocks.summary(clocks.t_ramp, clocks.t_end).get("sm_mhz")
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    roof = binding_roof(issue_roof("tet16", "binned", float(v2.astype(np.int64).sum() - ns), kb / 1e3, clk, sms),
                        l1_pipe_roof("cfg4/tet16", kb / 1e3, clk, sms))
    out = {"value": ns / kb / 1e3, "unit": "Mrays/s", "rays": ns, "kernel_ms": kb, "schedule": "binned",
           "one_ray_per_lane": {"value": ns / float(ms["lane"].mean()) / 1e3, "kernel_ms": float(ms["lane"].mean())},
           "tets_visited_per_ray": {"mean": float(v2.mean()), "max": int(v2.max())},
           "roofline": roof, "traffic": traffic_of("cfg4/tet16"), "ncu_pipes": pipes_of("cfg4/tet16"),
           "algorithmic_bytes_per_launch": algorithmic_bytes(v2, "tet16"),
           "rays_from": "diffuse hemisphere bounces of the 4096x4096 blob-camera frame's primary hits (seed 4), "
                        "16x16-tile order (the reference renderer's), Tet16 Hilbert mesh of the same scene",
           "parity": par}
    dm.close()
    return out


def render_e2e(args, cfg, dm, stream, sctp):
    """Render-style end to end: camera rays generated in HBM, hits written by
    the trace straight to pinned host memory, per step."""
    import torch

    from paper_2103_02309_b200.trace import TraceResult, trace_camera

    W, H = cfg["width"], cfg["height"]
    cam = camera_of(cfg, 0)
    hres = TraceResult(*[torch.empty(W * H, dtype=dt).pin_memory() for dt in
                         (torch.uint8, torch.int32, torch.int32, torch.float64, torch.int32, torch.int32, torch.int32)])
    _, cam_tet = trace_camera(dm, cam, W, H, out=hres, stream=stream, sctp=sctp)  # camera located once

    def call():
        trace_camera(dm, cam, W, H, out=hres, stream=stream, cam_tet=cam_tet, sctp=sctp)
        torch.cuda.synchronize()

    for _ in range(max(1, args.warmup)):
        call()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        call()
    r_s = time.perf_counter() - t0
    return {"value": W * H * args.steps / r_s / 1e6, "unit": "Mrays/s", "h2d_bytes_per_step": 14 * 8,
            "d2h_bytes_per_step": int(W * H * 29), "ms_per_step": r_s / args.steps * 1e3,
            "path": "trace_camera (tb_trace_camera): one launch forms each pixel's ray in registers, walks it and "
                    "writes all 7 hit arrays straight to pinned host memory (camera tet located once)"}


def small_batch(args, mesh, o, d, st, threads):
    """Renderer granularity (render.py:192-207,300-331,538-541: one
    batch.cast_rays per 16x16 tile from a thread pool): the reference's
    batch.cast_rays with kernels= the CUDA module vs its own compiled
    kernels, at 256 / 4096 / 65536 rays per call from all host threads over
    the frame's first 2^20 rays."""
    from concurrent.futures import ThreadPoolExecutor

    import paper_2103_02309_b200.kernels as cuda

    ref_package()
    from tetray import backend, batch

    K = backend.get_kernels("compiled")
    total = min(len(st), 1 << 20)
    out = {}
    for size in (256, 4096, 65536):
        starts = list(range(0, total, size))

        def run(kern):
            def one(a):
                batch.cast_rays(mesh, o[a:a + size], d[a:a + size], st[a:a + size], kernels=kern)
            with ThreadPoolExecutor(max_workers=threads) as pool:
                list(pool.map(one, starts))

        row = {}
        for name, kern in (("cuda", cuda), ("reference", K)):
            run(kern)  # warm (uploads, thread contexts)
            t0 = time.perf_counter()
            reps = 0
            while reps < 2 or time.perf_counter() - t0 < 0.5:
                run(kern)
                reps += 1
            row[name] = total * reps / (time.perf_counter() - t0) / 1e6
        row["speedup"] = row["cuda"] / row["reference"]
        out[str(size)] = row
    cross = next((int(s) for s, r in out.items() if r["speedup"] >= 1.0), None)
    return {"unit": "Mrays/s", "threads": threads, "rays": total, "per_call": out,
            "crossover_rays_per_call": cross,
            "path": "tetray.batch.cast_rays(kernels=paper_2103_02309_b200.kernels) vs kernels=its compiled "
                    "_kernels, host numpy buffers, one call per chunk from a thread pool"}


def relaunch(args):
    """--gpus N outside torchrun: one rank per GPU via torch.distributed.run."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    log(f"[bench] --gpus {args.gpus}: relaunching under torch.distributed.run")
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--layout", default=None)
    ap.add_argument("--scheme", default=None)
    ap.add_argument("--no-secondary", action="store_true", help="skip the frame's own secondary rays")
    ap.add_argument("--no-cfg4", action="store_true", help="skip the config-4 secondaries in the default run")
    ap.add_argument("--no-small-batch", action="store_true", help="skip the renderer-granularity measurement")
    ap.add_argument("--gather", choices=("p2p", "nccl"), default="p2p",
                    help="N > 1 frame assembly: fused P2P stores (default) or the chunked NCCL gather")
    ap.add_argument("--gather-chunks", type=int, default=4, help="N > 1 NCCL gather: trace/gather pipeline depth")
    ap.add_argument("--schedule", default=None, choices=("auto", "lane", "refill", "compact", "compact512", "dynamic", "binned",
                                                          "sampled"),
                    help="ray-to-lane schedule of the timed trace (default: binned for secondaries, else auto)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-l2-probe", action="store_true", help="skip the L2 gather-roof probe (roofline_l2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=2_073_600)
    ap.add_argument("--ref-sample", type=int, default=2_097_152, help="reference arm: rays per step (config 4)")
    ap.add_argument("--ramp-s", type=float, default=0.5, help="untimed load before the timed region (clock ramp)")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--parity-sample", type=int, default=65_536, help="rays checked against the reference")
    ap.add_argument("--dump-scene", type=int, default=None, help=argparse.SUPPRESS)
    ap.add_argument("--out", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.dump_scene is not None:
        dump_scene(args.dump_scene, args.layout, args.scheme, args.out)
        return
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    cfg = dict(CONFIGS[args.config])
    if args.layout:
        cfg["layout"] = args.layout
    if args.scheme:
        cfg["scheme"] = args.scheme
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return
    if world == 0 and args.gpus > 1:
        relaunch(args)
    if world and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    run_ours(args, cfg)


if __name__ == "__main__":
    main()
