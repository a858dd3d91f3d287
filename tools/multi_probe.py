#!/usr/bin/env python
"""tb_trace_multi on one box: the config-2 frame traced by 1 / 2 / 4 replicas
(all on cuda:0 here -- on a node each replica is its own GPU) against the
plain single-GPU trace.  Device time per frame (CUDA events on the caller's
stream, L2 flushed), median of --reps; frames compared bit for bit.

    python tools/multi_probe.py [--reps 20]
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
from paper_2103_02309_b200.device import DeviceMesh  # noqa: E402
from paper_2103_02309_b200.multigpu import trace_multi  # noqa: E402
from paper_2103_02309_b200.trace import empty_result, locate, trace  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfg = CONFIGS[2]
    mesh = build_scene(cfg).mesh
    W, H = cfg["width"], cfg["height"]
    o, d, pos = frame_rays(cfg, 0)
    dms = [DeviceMesh(mesh, 0) for _ in range(4)]
    cam, _ = locate(dms[0], torch.tensor(pos[None], dtype=torch.float64, device=dev),
                    torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
    go, gd = torch.from_numpy(o).to(dev), torch.from_numpy(d).to(dev)
    gs = torch.full((W * H,), int(cam.item()), dtype=torch.int32, device=dev)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=dev)
    ref = empty_result(W * H, dev)
    out = empty_result(W * H, dev)
    runs = [("trace (one GPU)", lambda: trace(dms[0], go, gd, gs, out=ref))]
    for k in (1, 2, 4):
        runs.append((f"tb_trace_multi x{k}", lambda k=k: trace_multi(dms[:k], W, H, go, gd, gs, out=out)))
    for name, fn in runs:
        for _ in range(3):
            fn()
        ev = []
        for _ in range(args.reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            ev.append((a, b))
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
        same = name.startswith("trace ") or all(torch.equal(getattr(out, k), getattr(ref, k)) for k in
                                                 ("status", "cf", "tet", "visited", "triangle", "t", "tet_back"))
        print(json.dumps({"run": name, "ms": round(ms, 4), "Mrays_s": round(W * H / ms / 1e3, 1), "equal": same}),
              flush=True)


if __name__ == "__main__":
    main()
