#!/usr/bin/env python
"""Pixel order of a camera frame vs trace throughput (coherence per warp).

The same rays, cast in four orders: row-major (one warp = 32 pixels of one
row), 16x16 render tiles (render.py:496-514 tile geometry; one warp = 16x2),
8x4 warp tiles inside 16x16 tiles, and Morton (Z) order.  Device time per
launch (CUDA events, L2 flushed), median of --reps; every order's outputs,
permuted back to row-major, must equal the row-major run bit for bit.

    python tools/ray_order_probe.py [--sizes 1920x1080,3840x2160] [--layouts tet20,tet16]
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

from paper_2103_02309_b200.device import device_mesh  # noqa: E402
from paper_2103_02309_b200.scenes import BLOB_CAMERA, blob_scene, camera_rays  # noqa: E402
from paper_2103_02309_b200.tetmesh import relayout  # noqa: E402
from paper_2103_02309_b200.trace import empty_result, locate, trace  # noqa: E402


def _tile_key(x, y, tw, th, W):
    tiles_x = (W + tw - 1) // tw
    return ((y // th) * tiles_x + x // tw) * (tw * th) + (y % th) * tw + (x % tw)


def pixel_orders(W, H):
    y, x = np.divmod(np.arange(W * H, dtype=np.int64), W)
    morton = np.zeros_like(x)
    for b in range(13):
        morton |= ((x >> b) & 1) << (2 * b) | ((y >> b) & 1) << (2 * b + 1)
    t16 = _tile_key(x, y, 16, 16, W)
    w84 = t16 // 256 * 256 + _tile_key(x % 16, y % 16, 8, 4, 16)
    return {"row": np.arange(W * H), "tile16": np.argsort(t16, kind="stable"),
            "tile16_warp8x4": np.argsort(w84, kind="stable"), "morton": np.argsort(morton, kind="stable")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1920x1080,3840x2160")
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
            n = len(st)
            ref = None
            for name, perm in pixel_orders(W, H).items():
                g = [torch.from_numpy(np.ascontiguousarray(a[perm])).to(dev) for a in (o, d, st)]
                out = empty_result(n, dev)
                for _ in range(3):
                    trace(dm, *g, out=out)
                evs = []
                for _ in range(args.reps):
                    flush.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    trace(dm, *g, out=out)
                    b.record()
                    evs.append((a, b))
                torch.cuda.synchronize()
                ms = float(np.median([a.elapsed_time(b) for a, b in evs]))
                inv = torch.from_numpy(np.argsort(perm)).to(dev)
                cur = [x[inv] for x in (out.status, out.cf, out.tet, out.visited, out.t)]
                if ref is None:
                    ref = cur
                same = all(torch.equal(a, b) for a, b in zip(cur, ref))
                print(json.dumps({"layout": layout, "frame": size, "order": name, "ms": round(ms, 4),
                                  "Mrays_s": round(n / ms / 1e3, 1), "equal": same}), flush=True)


if __name__ == "__main__":
    main()
