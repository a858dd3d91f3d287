#!/usr/bin/env python
"""Binning incoherent secondaries before the walk: trace time by ray order.

Config 4's 16.7 M diffuse secondaries (from 4096x4096 primary hits, tet16,
blob GRID=55) traced in several orders; the sort itself is NOT timed here
(torch, outside the events) -- this bounds what a native binning pass could
gain.  Keys: direction octant; start tet (Hilbert-ordered ids, so id
proximity is spatial proximity) at several granularities; both combined.
Outputs are scattered back (tb_cast_rays_scatter) and must equal the
unsorted run bit for bit.

    python tools/bin_probe.py [--size 4096] [--layout tet16]
    BIN_KEYS="cube4;cube4,start>>8" python tools/bin_probe.py   # only these keys (+ the unsorted run)

Keys also include cube-map direction cells (dominant axis and sign x a k x k grid, k = 1, 2,
4, 8) alone and combined with start-tet buckets.
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

from paper_2103_02309_b200._lib import addr, check, lib  # noqa: E402,F401
from paper_2103_02309_b200.device import device_mesh  # noqa: E402
from paper_2103_02309_b200.scenes import BLOB_CAMERA, blob_scene, camera_rays, diffuse_secondaries  # noqa: E402
from paper_2103_02309_b200.tetmesh import relayout  # noqa: E402
from paper_2103_02309_b200.trace import empty_result, locate, trace  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--layout", default="tet16")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
    mesh = relayout(blob_scene(55, layout="tet20", scheme="hilbert", check=False).mesh, args.layout)
    dm = device_mesh(mesh)
    cam = BLOB_CAMERA
    c, _ = locate(dm, torch.tensor([cam["position"]], dtype=torch.float64, device=dev),
                  torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
    W = H = args.size
    o, d = camera_rays(cam["position"], cam["look_at"], cam["up"], cam["fov"], W, H)
    if os.environ.get("BIN_TILES"):  # the reference renderer's 16x16-tile ray order (bench.py config 4)
        from paper_2103_02309_b200.multigpu import shard_pixels

        tiles = shard_pixels(W, H, 0, 1, 16)
        o, d = o[tiles], d[tiles]
    st = np.full(len(o), int(c.item()), np.int32)
    prim = trace(dm, *(torch.from_numpy(a).to(dev) for a in (o, d, st)))
    torch.cuda.synchronize()
    so, sd, sst = diffuse_secondaries(o, d, prim.t.cpu().numpy(), prim.triangle.cpu().numpy(),
                                      prim.tet.cpu().numpy(), mesh.triangle_coords(), seed=4)
    g = [torch.from_numpy(a).to(dev) for a in (so, sd, sst)]
    n = len(sst)
    octant = ((g[1][:, 0] < 0).int() | ((g[1][:, 1] < 0).int() << 1) | ((g[1][:, 2] < 0).int() << 2)).long()
    start = g[2].long()
    keys = {"none": None, "octant": octant}
    for shift in (4, 8, 12):
        keys[f"start>>{shift}"] = start >> shift
        keys[f"octant,start>>{shift}"] = (octant << 40) | (start >> shift)
    # cube-map direction bins: dominant axis and its sign (6 faces) x a k x k
    # grid over the face's two other coordinates (divided by the dominant one)
    dd = g[1].double()
    ax = dd.abs().argmax(dim=1)
    sgn = (dd.gather(1, ax[:, None])[:, 0] < 0).long()
    face = ax * 2 + sgn
    other = torch.tensor([[1, 2], [0, 2], [0, 1]], device=dev)[ax]
    uv = dd.gather(1, other) / dd.gather(1, ax[:, None]).abs()
    for k in (1, 2, 4, 8):
        cell = ((uv + 1) * 0.5 * k).long().clamp(0, k - 1)
        keys[f"cube{k}"] = (face * k + cell[:, 0]) * k + cell[:, 1]
        if k in (2, 4):
            for shift in (8, 12, 16):
                keys[f"cube{k},start>>{shift}"] = (keys[f"cube{k}"] << 40) | (start >> shift)
    # the production order (schedule "binned"): stable by (256 K-ray segment, cube4 cell),
    # and the same with a spatial sub-key inside each cell: the start tet's Hilbert id
    seg = torch.arange(n, device=dev, dtype=torch.long) >> 18
    keys["seg,cube4"] = (seg << 50) | (keys["cube4"] << 40)
    for shift in (6, 8, 10, 12, 14):
        keys[f"seg,cube4,start>>{shift}"] = (seg << 50) | (keys["cube4"] << 40) | (start >> shift)
    ref = None
    only = os.environ.get("BIN_KEYS")
    for name, key in keys.items():
        if only and name not in only.split(";") and name != "none":
            continue
        if key is None:
            perm = torch.arange(n, device=dev)
        else:
            perm = torch.sort(key, stable=True).indices
        go, gd, gs = (x[perm].contiguous() for x in g)
        oidx = perm.to(torch.int64).contiguous()
        out = empty_result(n, dev)

        def call():
            check(lib.tb_cast_rays_scatter(dm.handle, n, go.data_ptr(), gd.data_ptr(), gs.data_ptr(),
                                           oidx.data_ptr(), out.status.data_ptr(), out.cf.data_ptr(),
                                           out.tet.data_ptr(), out.visited.data_ptr(), out.triangle.data_ptr(),
                                           out.t.data_ptr(), out.tet_back.data_ptr(),
                                           torch.cuda.current_stream(dev).cuda_stream), "tb_cast_rays_scatter")

        for _ in range(3):
            call()
        evs = []
        for _ in range(args.reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call()
            b.record()
            evs.append((a, b))
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in evs]))
        cur = [out.status, out.cf, out.tet, out.visited, out.t, out.triangle, out.tet_back]
        if ref is None:
            ref = [x.clone() for x in cur]
        same = all(torch.equal(a, b) for a, b in zip(cur, ref))
        print(json.dumps({"key": name, "rays": n, "ms": round(ms, 4), "Mrays_s": round(n / ms / 1e3, 1),
                          "equal": same}), flush=True)


if __name__ == "__main__":
    main()
