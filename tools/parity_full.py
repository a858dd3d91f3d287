#!/usr/bin/env python
"""Full-size parity: every ray of a bench workload, GPU vs the C oracle.

The bench checks config 2 against the reference's own digest and configs 3-5
on a strided sample; this runs the C restatement (oracle/tetoracle.c, all
host threads) over EVERY ray of the workload -- the primary frame, and for
config 4 the 16.7 M diffuse secondaries under both the one-ray-per-lane and
the binned schedule -- and compares all seven output arrays bit for bit.
Test infrastructure only (the oracle is the checker here, never measured).

    python tools/parity_full.py [--configs 3,4,5]
    python tools/parity_full.py --layouts      # config 2 in every layout, 2-D and ScTP walks
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

from bench import CONFIGS, build_scene, frame_rays  # noqa: E402
from oracle import pyoracle  # noqa: E402
from paper_2103_02309_b200.device import device_mesh  # noqa: E402
from paper_2103_02309_b200.trace import locate, trace  # noqa: E402

NAMES = ("status", "cf", "tet", "visited", "triangle", "t", "tet_back")


def compare(res, exp):
    bad = {}
    for k, e in zip(NAMES, exp):
        g = getattr(res, k).cpu().numpy()
        m = int(np.count_nonzero(g != e))
        if m:
            bad[k] = m
    return bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3,4,5")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    for c in (int(x) for x in args.configs.split(",")):
        cfg = CONFIGS[c]
        mesh = build_scene(cfg).mesh
        dm = device_mesh(mesh)
        o, d, pos = frame_rays(cfg, 0)
        cam, _ = locate(dm, torch.tensor(pos[None], dtype=torch.float64, device=dev),
                        torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
        st = np.full(len(o), int(cam.item()), np.int32)
        runs = [("primaries", o, d, st, "lane")]
        if cfg.get("secondaries"):
            from paper_2103_02309_b200.scenes import diffuse_secondaries

            prim = trace(dm, *(torch.from_numpy(a).to(dev) for a in (o, d, st)))
            torch.cuda.synchronize()
            so, sd, sst = diffuse_secondaries(o, d, prim.t.cpu().numpy(), prim.triangle.cpu().numpy(),
                                              prim.tet.cpu().numpy(), mesh.triangle_coords(), seed=4)
            runs = [("secondaries", so, sd, sst, "lane"), ("secondaries", so, sd, sst, "binned")]
        exp_cache = {}
        for name, ro, rd, rs, sched in runs:
            res = trace(dm, *(torch.from_numpy(a).to(dev) for a in (ro, rd, rs)), schedule=sched)
            torch.cuda.synchronize()
            if name not in exp_cache:
                t0 = time.perf_counter()
                exp_cache[name] = pyoracle.cast_rays_full(mesh, ro, rd, rs, layout=dm.layout)
                oracle_s = time.perf_counter() - t0
            bad = compare(res, exp_cache[name])
            print(json.dumps({"config": c, "rays": name, "n": len(rs), "schedule": sched, "layout": dm.layout,
                              "mismatched": bad, "bit_exact": not bad, "oracle_s": round(oracle_s, 1),
                              "oracle_threads": os.cpu_count()}), flush=True)


def layouts_cfg2():
    """Config 2's full frame in every layout, 2-D and ScTP walks, vs the oracle
    (TetMesh-80 against the oracle's own TetMesh-80 restatement)."""
    from paper_2103_02309_b200.tetmesh import relayout

    dev = torch.device("cuda", 0)
    cfg = CONFIGS[2]
    base = build_scene(cfg).mesh
    o, d, pos = frame_rays(cfg, 0)
    for layout in ("tet32", "tet20", "tet16", "tet80"):
        mesh = base if layout in (base.layout, "tet80") else relayout(base, layout)
        dm = device_mesh(mesh, layout=layout if layout == "tet80" else None)
        cam, _ = locate(dm, torch.tensor(pos[None], dtype=torch.float64, device=dev),
                        torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
        st = np.full(len(o), int(cam.item()), np.int32)
        for sctp in (False, True):
            if sctp and layout not in ("tet20", "tet80"):
                continue
            res = trace(dm, *(torch.from_numpy(a).to(dev) for a in (o, d, st)), sctp=sctp)
            torch.cuda.synchronize()
            exp = pyoracle.cast_rays_full(mesh, o, d, st, layout=dm.layout, sctp=sctp)
            bad = compare(res, exp)
            print(json.dumps({"config": 2, "rays": "primaries", "n": len(st), "layout": layout,
                              "walk": "sctp" if sctp else "2d", "mismatched": bad, "bit_exact": not bad}),
                  flush=True)


if __name__ == "__main__":
    if "--layouts" in sys.argv:
        layouts_cfg2()
    else:
        main()
