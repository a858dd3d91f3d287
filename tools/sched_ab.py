#!/usr/bin/env python
"""Same-process A/B of ray schedules (trace(schedule=...)) on the bench workloads.

    python tools/sched_ab.py [--configs 2,3,5] [--schedules lane,dynamic] [--reps 20] [--rounds 3]
                             [--secondaries] [--layouts tet20,tet32] [--tiles]

Builds each bench scene once, times the trace with CUDA events (256 MiB
written between launches to flush L2), schedules interleaved round by round,
and checks every schedule's seven outputs equal the first's bit for bit.
--secondaries: time the frame's diffuse bounces (config 4 semantics, seed 4)
instead of the primaries.  --layouts: device layouts to compare (default:
the config's own; tet80 is built on the device from the same host mesh).
--tiles: rays in 16x16-tile order (the reference renderer's) instead of row
major.  One JSON line per (config, layout, schedule).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS, build_scene, frame_rays, timed  # noqa: E402
from paper_2103_02309_b200.device import DeviceMesh  # noqa: E402
from paper_2103_02309_b200.trace import empty_result, locate, trace  # noqa: E402
from paper_2103_02309_b200.workload import diffuse_secondaries  # noqa: E402

FIELDS = ("status", "cf", "tet", "visited", "triangle", "t", "tet_back")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3")
    ap.add_argument("--schedules", default="lane,dynamic")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--secondaries", action="store_true")
    ap.add_argument("--layout", default=None)
    ap.add_argument("--layouts", default=None)
    ap.add_argument("--tiles", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
    for c in (int(x) for x in a.configs.split(",")):
        cfg = dict(CONFIGS[c])
        if a.layout:
            cfg["layout"] = a.layout
        layouts = a.layouts.split(",") if a.layouts else [cfg["layout"]]
        if cfg["layout"] == "tet80":
            cfg["layout"] = "tet32"
        mesh = build_scene(cfg).mesh
        dm = DeviceMesh(mesh, 0, layout=layouts[0])
        o, d, pos = frame_rays(cfg, 0)
        if a.tiles:
            from paper_2103_02309_b200.multigpu import shard_pixels

            tiles = shard_pixels(cfg["width"], cfg["height"], 0, 1, 16)
            o, d = o[tiles], d[tiles]
        cam, _ = locate(dm, torch.tensor(pos[None], dtype=torch.float64, device=dev),
                        torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
        st = np.full(len(o), int(cam.item()), np.int32)
        if a.secondaries or cfg.get("secondaries"):
            prim = trace(dm, *(torch.from_numpy(x).to(dev) for x in (o, d, st)))
            o, d, st = diffuse_secondaries(o, d, prim.t.cpu().numpy(), prim.triangle.cpu().numpy(),
                                           prim.tet.cpu().numpy(), mesh.triangle_coords(), seed=4)
            del prim
        g = [torch.from_numpy(x).to(dev) for x in (o, d, st)]
        dms = {layouts[0]: dm}
        for lay in layouts[1:]:
            dms[lay] = DeviceMesh(mesh, 0, layout=lay)
        runs = [(lay, s) for lay in layouts for s in a.schedules.split(",")]
        outs = {k: empty_result(len(st), dev) for k in runs}
        ms = {k: [] for k in runs}
        for _ in range(a.rounds):
            for k in runs:
                ms[k].extend(timed(lambda: trace(dms[k[0]], *g, out=outs[k], stream=stream, schedule=k[1]), a.reps, 3,
                                   stream, flush).tolist())
        ref = outs[runs[0]]
        vis = ref.visited.cpu().numpy()
        for k in runs:
            same = all(torch.equal(getattr(outs[k], f), getattr(ref, f)) for f in FIELDS)
            med = float(np.median(ms[k]))
            print(json.dumps({"config": c, "layout": k[0], "secondaries": bool(a.secondaries or
                                                                              cfg.get("secondaries")),
                              "order": "tiles16" if a.tiles else "row-major",
                              "schedule": k[1], "rays": len(st), "kernel_ms_median": med,
                              "kernel_ms_min": float(np.min(ms[k])), "mrays_s": len(st) / med / 1e3,
                              "tets_per_ray": float(vis.mean()), "equal_to_first": same}), flush=True)
        for x in dms.values():
            x.close()


if __name__ == "__main__":
    main()
