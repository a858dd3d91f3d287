#!/usr/bin/env python
"""Schedules for incoherent secondaries: one ray per lane vs direction
binning vs block compaction (256 / 512 threads, several round lengths), per layout and
primary-frame size, on the blob GRID=55 scene.  Device time per launch
(CUDA events, L2 flushed), median of --reps; outputs compared across
schedules bit for bit.

    python tools/secondary_probe.py [--sizes 1920x1080,4096x4096] [--layouts tet20,tet16]
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

from paper_2103_02309_b200 import _lib  # noqa: E402
from paper_2103_02309_b200.device import device_mesh  # noqa: E402
from paper_2103_02309_b200.scenes import BLOB_CAMERA, blob_scene, camera_rays, diffuse_secondaries  # noqa: E402
from paper_2103_02309_b200.tetmesh import relayout  # noqa: E402
from paper_2103_02309_b200.trace import empty_result, locate, trace  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1920x1080,4096x4096")
    ap.add_argument("--layouts", default="tet20,tet16")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
    base = blob_scene(55, layout="tet20", scheme="hilbert", check=False).mesh
    for layout in args.layouts.split(","):
        mesh = relayout(base, layout)
        dm = device_mesh(mesh)
        cam = BLOB_CAMERA
        c, _ = locate(dm, torch.tensor([cam["position"]], dtype=torch.float64, device=dev),
                      torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
        for size in args.sizes.split(","):
            W, H = (int(x) for x in size.split("x"))
            o, d = camera_rays(cam["position"], cam["look_at"], cam["up"], cam["fov"], W, H)
            st = np.full(len(o), int(c.item()), np.int32)
            prim = trace(dm, *(torch.from_numpy(a).to(dev) for a in (o, d, st)))
            torch.cuda.synchronize()
            so, sd, sst = diffuse_secondaries(o, d, prim.t.cpu().numpy(), prim.triangle.cpu().numpy(),
                                              prim.tet.cpu().numpy(), mesh.triangle_coords(), seed=4)
            g = [torch.from_numpy(a).to(dev) for a in (so, sd, sst)]
            n = len(sst)
            ref = None
            for sched, rounds in (("lane", 32), ("binned", 32), ("compact", 16), ("compact", 32), ("compact", 64),
                                  ("compact512", 32)):
                _lib.set_schedule(None, rounds)
                out = empty_result(n, dev)
                for _ in range(3):
                    trace(dm, *g, out=out, schedule=sched)
                evs = []
                for _ in range(args.reps):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    trace(dm, *g, out=out, schedule=sched)
                    b.record()
                    evs.append((a, b))
                torch.cuda.synchronize()
                ms = float(np.median([a.elapsed_time(b) for a, b in evs]))
                cur = [out.status, out.cf, out.tet, out.visited, out.t]
                if ref is None:
                    ref = [x.clone() for x in cur]
                same = all(torch.equal(a, b) for a, b in zip(cur, ref))
                print(json.dumps({"layout": layout, "frame": size, "rays": n, "schedule": sched, "rounds": rounds,
                                  "ms": round(ms, 4), "Mrays_s": round(n / ms / 1e3, 1),
                                  "visited_mean": round(float(out.visited.double().mean()), 2),
                                  "equal": same}), flush=True)


if __name__ == "__main__":
    main()
