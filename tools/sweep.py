#!/usr/bin/env python
"""Variant sweep on one GPU: layouts x reorder schemes x walk kernel, plus a
PCIe probe.  Device-timed (CUDA events, L2 flushed between launches).
Writes one JSON object per line to stdout; used for profiles/ tables.

    python tools/sweep.py [--grid 55] [--width 1920 --height 1080] [--reps 20]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2103_02309_b200.device import DeviceMesh  # noqa: E402
from paper_2103_02309_b200.scenes import BLOB_CAMERA, blob_scene, camera_rays, diffuse_secondaries  # noqa: E402
from paper_2103_02309_b200.tetmesh import relayout, reorder  # noqa: E402
from paper_2103_02309_b200.trace import empty_result, locate, trace  # noqa: E402


def timed(fn, reps, flush):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for _ in range(3):
        flush.zero_()
        fn()
    for a, b in evs:
        flush.zero_()
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in evs]))


def pcie_probe(dev, nbytes=64 << 20, reps=10):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    g = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    g2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name, f in (("h2d", lambda: g.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(g, non_blocking=True))):
        f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            f()
        torch.cuda.synchronize()
        out[name + "_GBps"] = nbytes * reps / (time.perf_counter() - t0) / 1e9
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s1):
            g.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(g2, non_blocking=True)
    torch.cuda.synchronize()
    out["bidir_GBps_each"] = nbytes * reps / (time.perf_counter() - t0) / 1e9
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=55)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--layouts", default="tet20,tet16,tet32,tet80")
    ap.add_argument("--schemes", default="hilbert,none,shuffle")
    ap.add_argument("--sctp", action="store_true")
    ap.add_argument("--secondaries", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
    print(json.dumps({"probe": "pcie", **pcie_probe(dev)}), flush=True)
    base = blob_scene(args.grid, layout="tet20", scheme="none", check=False).mesh
    c = BLOB_CAMERA
    o, d = camera_rays(c["position"], c["look_at"], c["up"], c["fov"], args.width, args.height)
    go, gd = torch.from_numpy(o).to(dev), torch.from_numpy(d).to(dev)
    n = len(o)
    for scheme in args.schemes.split(","):
        ms = reorder(base, scheme)
        dm20 = DeviceMesh(ms, 0)
        cam, _ = locate(dm20, torch.tensor([c["position"]], dtype=torch.float64, device=dev),
                        torch.tensor([ms.source_tet], dtype=torch.int32, device=dev))
        gs = torch.full((n,), int(cam.item()), dtype=torch.int32, device=dev)
        for layout in args.layouts.split(","):
            dm = dm20 if layout == "tet20" else DeviceMesh(ms if layout == "tet80" else relayout(ms, layout), 0,
                                                          layout=layout)
            res = empty_result(n, dev)
            kinds = [("2d", False)] + ([("sctp", True)] if args.sctp else [])
            for kind, sctp in kinds:
                ms_t = timed(lambda: trace(dm, go, gd, gs, out=res, sctp=sctp), args.reps, flush)
                vis = res.visited.double()
                print(json.dumps({"scheme": scheme, "layout": layout, "walk": kind, "rays": n, "kernel_ms": ms_t,
                                  "Mrays_s": n / ms_t / 1e3, "visited_mean": float(vis.mean()),
                                  "visited_max": int(vis.max()), "hot_bytes": dm.hot_bytes}), flush=True)
            if args.secondaries and scheme == "hilbert" and layout in ("tet16", "tet20"):
                torch.cuda.synchronize()
                so, sd, sst = diffuse_secondaries(o, d, res.t.cpu().numpy(), res.triangle.cpu().numpy(),
                                                  res.tet.cpu().numpy(), ms.triangle_coords(), seed=4)
                g2o, g2d, g2s = (torch.from_numpy(a).to(dev) for a in (so, sd, sst))
                res2 = empty_result(len(so), dev)
                ms_t = timed(lambda: trace(dm, g2o, g2d, g2s, out=res2), args.reps, flush)
                vis = res2.visited.double()
                print(json.dumps({"scheme": scheme, "layout": layout, "walk": "2d-secondaries", "rays": len(so),
                                  "kernel_ms": ms_t, "Mrays_s": len(so) / ms_t / 1e3,
                                  "visited_mean": float(vis.mean()), "visited_max": int(vis.max())}), flush=True)


if __name__ == "__main__":
    main()
