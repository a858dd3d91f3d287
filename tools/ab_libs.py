#!/usr/bin/env python
"""Same-process A/B of several builds of libtetb200.so (kernel experiments).

    python tools/ab_libs.py base.so variant1.so ... [--configs 2,3,4] [--reps 10] [--rounds 3]

Builds the bench scenes once, uploads each mesh through every library's own
C ABI, and times the trace launch with CUDA events (L2 flushed between
launches), interleaving the libraries round by round so clock drift hits all
of them alike.  Every variant's outputs must equal the first library's bit
for bit (status, cf, tet, visited, triangle, t, tet_back).  Prints one JSON
line per (config, library) with the median kernel time and Mrays/s.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
from ctypes import POINTER, c_int, c_int64, c_void_p

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS, build_scene, frame_rays  # noqa: E402
from paper_2103_02309_b200.trace import empty_result, locate, trace  # noqa: E402
from paper_2103_02309_b200.device import device_mesh  # noqa: E402

P = c_void_p
LAYOUTS = {"tet32": 32, "tet20": 20, "tet16": 16, "tet80": 80}


def load(path):
    lib = ctypes.CDLL(os.path.abspath(path))
    lib.tb_mesh_create.restype = c_int
    lib.tb_mesh_create.argtypes = [c_int, c_int, c_int64, P, c_int64, P, P, P, c_int64, P, P, c_int64, P,
                                   POINTER(c_void_p)]
    lib.tb_mesh_destroy.argtypes = [c_void_p]
    lib.tb_cast_rays_sched.restype = c_int
    lib.tb_cast_rays_sched.argtypes = [c_void_p, c_int64, P, P, P, P, P, P, P, P, P, P, c_int, c_void_p]
    lib.tb_last_error.restype = ctypes.c_char_p
    return lib


def upload(lib, mesh, layout):
    code = LAYOUTS[layout]
    pts = np.ascontiguousarray(mesh.points, dtype=np.float32)
    sv = np.ascontiguousarray(mesh.side_verts, dtype=np.int32)
    sn = np.ascontiguousarray(mesh.side_neighbors, dtype=np.uint32)
    recs = None if code == 80 else np.ascontiguousarray(mesh.records_u32(), dtype=np.uint32)
    cft = np.ascontiguousarray(mesh.cf_triangle, dtype=np.int32)
    cfk = np.ascontiguousarray(np.asarray(mesh.cf_tets, dtype=np.int32).reshape(-1, 2))
    tri = np.ascontiguousarray(mesh.triangle_coords(), dtype=np.float64).reshape(-1, 9)
    h = c_void_p()
    a = lambda x: None if x is None else x.ctypes.data  # noqa: E731
    rc = lib.tb_mesh_create(torch.cuda.current_device(), code, len(pts), a(pts), len(sv), a(recs), a(sv), a(sn),
                            len(cft), a(cft), a(cfk), len(tri), a(tri), ctypes.byref(h))
    if rc:
        raise RuntimeError(lib.tb_last_error())
    return h


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--configs", default="2,3,4")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--rounds", type=int, default=3)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    libs = [load(p) for p in args.libs]
    flush = torch.empty(256 << 18, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    for c in [int(x) for x in args.configs.split(",")]:
        cfg = CONFIGS[c]
        if os.environ.get("AB_LAYOUT"):  # this config's scene and rays on another record layout
            cfg = dict(cfg, layout=os.environ["AB_LAYOUT"])
        sc = build_scene(cfg)
        mesh = sc.mesh
        o, d, pos = frame_rays(cfg, 0)
        if os.environ.get("AB_TILES"):  # the reference renderer's 16x16-tile ray order
            from paper_2103_02309_b200.multigpu import shard_pixels

            tiles = shard_pixels(cfg["width"], cfg["height"], 0, 1, 16)
            o, d = o[tiles], d[tiles]
        if os.environ.get("AB_RAYS"):  # only the first N rays of the frame (small launches)
            o, d = o[: int(os.environ["AB_RAYS"])], d[: int(os.environ["AB_RAYS"])]
        if os.environ.get("AB_FLIP"):  # the frame's rays in reverse order (bottom-right tile first)
            o, d = np.ascontiguousarray(o[::-1]), np.ascontiguousarray(d[::-1])
        dm = device_mesh(mesh)
        cam, _ = locate(dm, torch.tensor(pos[None], dtype=torch.float64, device=dev),
                        torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
        st = np.full(len(o), int(cam.item()), np.int32)
        sched = int(os.environ.get("AB_PRIMARY_SCHED", "1"))
        if cfg.get("secondaries") or os.environ.get("AB_SECONDARIES"):
            from paper_2103_02309_b200.scenes import diffuse_secondaries

            prim = trace(dm, *(torch.from_numpy(x).to(dev) for x in (o, d, st)))
            torch.cuda.synchronize()
            o, d, st = diffuse_secondaries(o, d, prim.t.cpu().numpy(), prim.triangle.cpu().numpy(),
                                           prim.tet.cpu().numpy(), mesh.triangle_coords(), seed=4)
            sched = int(os.environ.get("AB_SCHED", "3"))
        go, gd, gs = (torch.from_numpy(x).to(dev) for x in (o, d, st))
        n = len(st)
        handles = [upload(lib, mesh, cfg["layout"]) for lib in libs]
        outs = [empty_result(n, dev) for _ in libs]
        times = [[] for _ in libs]

        def launch(i):
            r = outs[i]
            rc = libs[i].tb_cast_rays_sched(handles[i], n, go.data_ptr(), gd.data_ptr(), gs.data_ptr(),
                                            r.status.data_ptr(), r.cf.data_ptr(), r.tet.data_ptr(),
                                            r.visited.data_ptr(), r.triangle.data_ptr(), r.t.data_ptr(),
                                            r.tet_back.data_ptr(), sched, stream.cuda_stream)
            if rc:
                raise RuntimeError(libs[i].tb_last_error())

        for i in range(len(libs)):
            for _ in range(3):
                launch(i)
        for _ in range(args.rounds):
            for i in range(len(libs)):
                for _ in range(args.reps):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    launch(i)
                    b.record()
                    times[i].append((a, b))
        torch.cuda.synchronize()
        base = outs[0]
        for i, p in enumerate(args.libs):
            same = all(torch.equal(getattr(outs[i], k), getattr(base, k)) for k in
                       ("status", "cf", "tet", "visited", "triangle", "t", "tet_back"))
            ms = float(np.median([a.elapsed_time(b) for a, b in times[i]]))
            print(json.dumps({"cfg": c, "lib": os.path.basename(p), "sched": sched, "kernel_ms": round(ms, 4),
                              "Mrays_s": round(n / ms / 1e3, 1), "equal_to_first": same}), flush=True)
        for lib, h in zip(libs, handles):
            lib.tb_mesh_destroy(h)


if __name__ == "__main__":
    main()
