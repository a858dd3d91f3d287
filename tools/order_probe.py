#!/usr/bin/env python
"""Block launch order against the SM-idle tail of a primary frame.

The config-2 frame (16x16-tile ray order) is traced once per candidate order
of its 128-ray blocks: as given, longest block first by the frame's own walk
lengths (the upper bound -- those costs exist only after the walk), and
longest first by the walk lengths of a *neighbouring* frame (camera moved by
--move scene units: what a renderer tracing frame after frame has).  Rays are
permuted per block on the device (copies, untimed) and traced with
tb_cast_rays_scatter, whose stores go back to each ray's own slot; every
order's outputs must equal the unpermuted trace bit for bit.

    python tools/order_probe.py [--move 0.05] [--reps 20]
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

from bench import CONFIGS, build_scene, camera_of  # noqa: E402
from paper_2103_02309_b200._lib import check, lib  # noqa: E402
from paper_2103_02309_b200.device import device_mesh  # noqa: E402
from paper_2103_02309_b200.multigpu import shard_pixels  # noqa: E402
from paper_2103_02309_b200.trace import empty_result, locate, trace  # noqa: E402
from paper_2103_02309_b200.workload import camera_rays  # noqa: E402

BLOCK = 128


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--move", type=float, default=0.05)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--animation", action="store_true", help="frame sequence with longest_first of the previous frame")
    ap.add_argument("--frames", type=int, default=12)
    args = ap.parse_args()
    if args.animation:
        return animation(args)
    dev = torch.device("cuda", 0)
    cfg = CONFIGS[args.config]
    mesh = build_scene(cfg).mesh
    dm = device_mesh(mesh)
    W, H = cfg["width"], cfg["height"]
    tiles = shard_pixels(W, H, 0, 1, 16)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)

    def frame(shift):
        cam = dict(camera_of(cfg, 0))
        pos = np.asarray(cam["position"], np.float64) + np.array([shift, 0.0, 0.0])
        o, d = camera_rays(pos, cam["look_at"], cam["up"], cam["fov"], W, H)
        c, _ = locate(dm, torch.tensor(pos[None], dtype=torch.float64, device=dev),
                      torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
        st = np.full(len(o), int(c.item()), np.int32)
        return [torch.from_numpy(np.ascontiguousarray(a[tiles])).to(dev) for a in (o, d, st)]

    g = frame(0.0)
    n = g[2].numel()
    nb = (n + BLOCK - 1) // BLOCK

    def costs(rays):
        r = trace(dm, *rays)
        torch.cuda.synchronize()
        v = torch.zeros(nb * BLOCK, dtype=torch.int32, device=dev)
        v[:n] = r.visited
        return v.view(nb, BLOCK).max(dim=1).values, r

    own, ref = costs(g)
    v_own = torch.zeros(nb * BLOCK, dtype=torch.int32, device=dev)
    v_own[:n] = ref.visited
    one_ray = v_own.view(nb, BLOCK)[:, BLOCK // 2]      # one sampled ray per block
    stride8 = v_own.view(nb, BLOCK)[:, ::16].max(dim=1).values  # 8 sampled rays per block
    moved, _ = costs(frame(args.move))
    ar = torch.arange(nb, device=dev)
    orders = {"as given": ar,
              "reversed": torch.flip(ar, [0]),
              "interleaved (b x 7919 mod B)": torch.argsort((ar * 7919) % nb),
              "interleaved by 148 (SM-strided)": torch.argsort((ar % 148) * nb + ar),
              "random": torch.randperm(nb, device=dev, generator=torch.Generator(device=dev).manual_seed(1)),
              "longest first, own costs (bound)": torch.argsort(own, descending=True, stable=True),
              "longest first, one sampled ray per block": torch.argsort(one_ray, descending=True, stable=True),
              "longest first, 8 sampled rays per block": torch.argsort(stride8, descending=True, stable=True),
              **{f"longest first, one sampled ray capped at {k} steps":
                 torch.argsort(one_ray.clamp(max=k), descending=True, stable=True) for k in (16, 24, 32, 48, 96)},
              **{f"longest first, one sampled ray capped at {k} steps, ties shuffled":
                 torch.argsort(one_ray.clamp(max=k).to(torch.float64) * 4 + torch.rand(nb, device=dev,
                               generator=torch.Generator(device=dev).manual_seed(3), dtype=torch.float64),
                               descending=True) for k in (24, 32)},
              f"longest first, costs of the frame moved by {args.move}": torch.argsort(moved, descending=True,
                                                                                       stable=True)}
    for name, bo in orders.items():
        perm = (bo[:, None] * BLOCK + torch.arange(BLOCK, device=dev)[None, :]).reshape(-1)
        perm = perm[perm < n].contiguous()
        go, gd, gs = (x[perm].contiguous() for x in g)
        out = empty_result(n, dev)

        def call():
            check(lib.tb_cast_rays_scatter(dm.handle, n, go.data_ptr(), gd.data_ptr(), gs.data_ptr(),
                                           perm.data_ptr(), out.status.data_ptr(), out.cf.data_ptr(),
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
        same = all(torch.equal(getattr(out, k), getattr(ref, k)) for k in
                   ("status", "cf", "tet", "visited", "triangle", "t", "tet_back"))
        print(json.dumps({"order": name, "rays": n, "ms": round(ms, 4), "Mrays_s": round(n / ms / 1e3, 1),
                          "equal": same}), flush=True)




def animation(args):
    """Frames f = 0..F of an animation (camera moved 0.02 per frame, bench.py's
    frame sequence), each traced (a) as given, (b) in the order longest_first
    builds from the previous frame's visited counts -- computed on the device
    inside the timed frame -- and checked bit for bit against (a)."""
    from paper_2103_02309_b200.trace import longest_first

    dev = torch.device("cuda", 0)
    cfg = CONFIGS[args.config]
    mesh = build_scene(cfg).mesh
    dm = device_mesh(mesh)
    W, H = cfg["width"], cfg["height"]
    tiles = torch.from_numpy(shard_pixels(W, H, 0, 1, 16)).to(dev)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
    frames = []
    for f in range(args.frames):
        cam = camera_of(cfg, f)
        o, d = camera_rays(cam["position"], cam["look_at"], cam["up"], cam["fov"], W, H)
        c, _ = locate(dm, torch.tensor([cam["position"]], dtype=torch.float64, device=dev),
                      torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
        go, gd = (torch.from_numpy(a).to(dev)[tiles].contiguous() for a in (o, d))
        frames.append((go, gd, torch.full((go.shape[0],), int(c.item()), dtype=torch.int32, device=dev)))
    n = frames[0][2].numel()
    outs = [empty_result(n, dev) for _ in range(2)]
    rows = {}
    # the orders each frame would get from its predecessor, built ahead (untimed)
    pre = [None] + [longest_first(trace(dm, *frames[f - 1]).visited) for f in range(1, args.frames)]
    modes = ("as given", "longest first by the previous frame", "longest first by frame f-2, built beside frame f-1",
             "precomputed order of the previous frame")
    side = torch.cuda.Stream(dev)
    outs.append(empty_result(n, dev))
    names = ("status", "cf", "tet", "visited", "triangle", "t", "tet_back")
    refs = [trace(dm, *fr) for fr in frames]
    torch.cuda.synchronize()

    def run(mode, check):
        """All frames enqueued back to back (the host runs ahead, as a renderer's
        does); one event pair around the lot.  Returns GPU ms for the frames."""
        prev = trace(dm, *frames[0], out=outs[0])
        pending = None
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        results = []
        for f in range(1, args.frames):
            flush.zero_()
            bo = None
            if mode.startswith("longest first by the previous"):
                bo = longest_first(prev.visited)
            elif mode.startswith("precomputed"):
                bo = pre[f]
            elif mode.startswith("longest first by frame f-2"):
                if pending is not None:
                    torch.cuda.current_stream(dev).wait_event(pending[0])
                    bo = pending[1]
                ev = torch.cuda.Event()
                ev.record()
                side.wait_event(ev)
                with torch.cuda.stream(side):
                    nxt = longest_first(prev.visited, stream=side)
                    done = torch.cuda.Event()
                    done.record(side)
                pending = (done, nxt)
            cur = trace(dm, *frames[f], out=outs[f % 3], block_order=bo)
            if check:
                results.append([getattr(cur, k).clone() for k in names])
            prev = cur
        b.record()
        torch.cuda.synchronize()
        if check:
            for f, got in zip(range(1, args.frames), results):
                assert all(torch.equal(g, getattr(refs[f], k)) for g, k in zip(got, names)), (mode, f)
        return a.elapsed_time(b)

    # the flushes alone, to subtract
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for f in range(1, args.frames):
        flush.zero_()
    b.record()
    torch.cuda.synchronize()
    flush_ms = a.elapsed_time(b)
    modes = ("as given", "longest first by the previous frame", "longest first by frame f-2, built beside frame f-1",
             "precomputed order of the previous frame")
    for mode in modes:
        run(mode, check=True)
    for mode in modes + modes:
        ms = (run(mode, check=False) - flush_ms) / (args.frames - 1)
        rows.setdefault(mode, []).append(ms)
    for mode, v in rows.items():
        ms = min(v)
        print(json.dumps({"animation": mode, "frames": args.frames - 1, "rays": n, "ms_per_frame": round(ms, 4),
                          "Mrays_s": round(n / ms / 1e3, 1), "bit_exact_vs_unordered": True}), flush=True)


if __name__ == "__main__":
    main()
