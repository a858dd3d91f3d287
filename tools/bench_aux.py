#!/usr/bin/env python
"""Device throughput of the §8(f) kernels around the hot path, on the config-2
scene (blob GRID=55, 1.1 M tets, tet20 Hilbert):

  * locate_points (f1): the primary hit points re-located from their front
    tet (short walks) and random interior points from the source tet (long
    walks);
  * shadow_rays (f2): hit point -> point light, p_tet = front tet;
  * visit recording (f4): the CSR second pass for the whole frame;
  * camera rays on the device (f4).

CUDA events around each launch (median of --reps, L2 flushed in between).
One JSON line per measurement.  Parity of these kernels is pinned by
tests/test_cuda_parity.py; this tool only times them.

    python tools/bench_aux.py [--reps 10]
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

from bench import CONFIGS, build_scene, frame_rays  # noqa: E402
from paper_2103_02309_b200._lib import addr, check, lib  # noqa: E402
from paper_2103_02309_b200.device import device_mesh  # noqa: E402
from paper_2103_02309_b200.scenes import BLOB_CAMERA, interior_rays  # noqa: E402
from paper_2103_02309_b200.trace import camera_rays_device, locate, trace  # noqa: E402


def timed(fn, reps, flush):
    evs = []
    for _ in range(2):
        fn()
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a, b in evs]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
    cfg = CONFIGS[2]
    mesh = build_scene(cfg).mesh
    dm = device_mesh(mesh)
    o, d, pos = frame_rays(cfg, 0)
    cam, _ = locate(dm, torch.tensor(pos[None], dtype=torch.float64, device=dev),
                    torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
    n = len(o)
    go, gd = torch.from_numpy(o).to(dev), torch.from_numpy(d).to(dev)
    gs = torch.full((n,), int(cam.item()), dtype=torch.int32, device=dev)
    res = trace(dm, go, gd, gs)
    torch.cuda.synchronize()
    hit = res.status == 1
    # hit points in fp64 (render.py:353 form), their front tets
    p = (go.double() + res.t.unsqueeze(1) * gd.double())[hit].contiguous()
    ptet = res.tet[hit].contiguous()
    m = p.shape[0]

    def out(name, ms, count, unit, extra=None):
        print(json.dumps({"kernel": name, "count": count, "ms": round(ms, 4), unit: round(count / ms / 1e3, 1),
                          **(extra or {})}), flush=True)

    # f1: locate, short walks (hint = the point's own front tet)
    tet = torch.empty(m, dtype=torch.int32, device=dev)
    vis = torch.empty(m, dtype=torch.int32, device=dev)
    s = torch.cuda.current_stream(dev).cuda_stream

    def loc(q, h, t_, v_, k):
        check(lib.tb_locate_points(dm.handle, k, addr(q), addr(h), addr(t_), addr(v_), s), "tb_locate_points")

    ms = timed(lambda: loc(p, ptet, tet, vis, m), args.reps, flush)
    out("locate_kernel<20> (hit points, hint = front tet)", ms, m, "Mpoints_s",
        {"visited_mean": float(vis.double().mean())})
    # f1: locate, long walks (random interior points from the source tet)
    ro, _, rst = interior_rays(mesh, 262144, 5)
    q = torch.from_numpy(ro.astype(np.float64)).to(dev)
    h = torch.full((len(ro),), mesh.source_tet, dtype=torch.int32, device=dev)
    t2 = torch.empty(len(ro), dtype=torch.int32, device=dev)
    v2 = torch.empty(len(ro), dtype=torch.int32, device=dev)
    ms = timed(lambda: loc(q, h, t2, v2, len(ro)), args.reps, flush)
    out("locate_kernel<20> (random points, hint = source tet)", ms, len(ro), "Mpoints_s",
        {"visited_mean": float(v2.double().mean())})

    # f2: shadow rays to a point light inside the scene
    light = torch.tensor([[5.0, 9.0, 5.0]], dtype=torch.float64, device=dev)
    lt, _ = locate(dm, light, torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
    occ = torch.empty(m, dtype=torch.uint8, device=dev)
    sv = torch.empty(m, dtype=torch.int32, device=dev)

    def shadow():
        check(lib.tb_shadow_rays(dm.handle, m, addr(p), addr(light), 0, addr(ptet), addr(lt), 0, 1e-4, addr(occ),
                                 addr(sv), s), "tb_shadow_rays")

    ms = timed(shadow, args.reps, flush)
    out("shadow_kernel<20> (hit point -> point light)", ms, m, "Mrays_s",
        {"visited_mean": float(sv.double().mean()), "occluded_frac": float(occ.double().mean())})

    # f2 probe: the same shadow rays sorted by direction cell of (light - p)
    # (torch sort outside the timed region) -- what binning could buy here
    dd = light - p
    ax = dd.abs().argmax(dim=1)
    face = ax * 2 + (dd.gather(1, ax[:, None])[:, 0] < 0).long()
    other = torch.tensor([[1, 2], [0, 2], [0, 1]], device=dev)[ax]
    uv = dd.gather(1, other) / dd.gather(1, ax[:, None]).abs()
    cell = ((uv + 1) * 2).long().clamp(0, 3)
    perm = torch.sort((face * 4 + cell[:, 0]) * 4 + cell[:, 1], stable=True).indices
    ps, pts_ = p[perm].contiguous(), ptet[perm].contiguous()
    occ2 = torch.empty(m, dtype=torch.uint8, device=dev)
    sv2 = torch.empty(m, dtype=torch.int32, device=dev)

    def shadow_sorted():
        check(lib.tb_shadow_rays(dm.handle, m, addr(ps), addr(light), 0, addr(pts_), addr(lt), 0, 1e-4, addr(occ2),
                                 addr(sv2), s), "tb_shadow_rays")

    ms = timed(shadow_sorted, args.reps, flush)
    same = bool(torch.equal(occ2, occ[perm]) and torch.equal(sv2, sv[perm]))
    out("shadow_kernel<20> (same rays sorted by direction cell, sort untimed)", ms, m, "Mrays_s",
        {"equal_after_unpermute": same})

    # f4: visit recording (CSR second pass over the frame)
    offs = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    offs[1:] = torch.cumsum(res.visited.long(), 0)
    seq = torch.empty(int(offs[-1].item()), dtype=torch.int32, device=dev)

    def visits():
        check(lib.tb_cast_rays_visits(dm.handle, n, addr(go), addr(gd), addr(gs), addr(offs), addr(seq), s),
              "tb_cast_rays_visits")

    ms = timed(visits, args.reps, flush)
    out("visits_kernel<20> (CSR visit sequences, full frame)", ms, n, "Mrays_s",
        {"visits": int(seq.numel()), "GB_s_written": round(seq.numel() * 4 / ms / 1e6, 1)})

    # f4: device camera rays
    ms = timed(lambda: camera_rays_device(BLOB_CAMERA, 1920, 1080, dev), args.reps, flush)
    out("camera_rays_kernel (1920x1080, fp64)", ms, n, "Mrays_s", {"GB_s_written": round(n * 24 / ms / 1e6, 1)})


if __name__ == "__main__":
    main()
