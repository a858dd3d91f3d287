#!/usr/bin/env python
"""End-to-end transport variants of tb_cast_rays_host on one box (config 2):

  TETB200_E2E=0  zero copy: the kernel reads rays and writes hits over PCIe
  TETB200_E2E=1  staged: chunked H2D copy / trace / D2H copy on 3 streams
  TETB200_E2E=2  copy-engine H2D, hits written by the kernel to host memory

with TETB200_CHUNK rays per chunk for the chunked modes.  Pinned host
buffers, wall clock per call (the C call synchronises), median of --reps.
Results of every variant are compared with mode 0 bit for bit.

    python tools/e2e_probe.py [--reps 20]
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
from paper_2103_02309_b200._lib import addr, check, lib  # noqa: E402
from paper_2103_02309_b200.device import device_mesh  # noqa: E402
from paper_2103_02309_b200.trace import locate  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--config", type=int, default=2)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    cfg = CONFIGS[args.config]
    mesh = build_scene(cfg).mesh
    dm = device_mesh(mesh)
    o, d, pos = frame_rays(cfg, 0)
    cam, _ = locate(dm, torch.tensor(pos[None], dtype=torch.float64, device=dev),
                    torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
    n = len(o)
    st = np.full(n, int(cam.item()), np.int32)
    ins = [torch.from_numpy(x).pin_memory() for x in (o, d, st)]
    dts = (torch.uint8, torch.int32, torch.int32, torch.int32, torch.int32, torch.float64, torch.int32)
    ref = None
    for mode, chunk in ((0, 0), (1, 1 << 18), (1, 1 << 17), (2, 1 << 18)):
        os.environ["TETB200_E2E"] = str(mode)
        os.environ["TETB200_CHUNK"] = str(chunk or (1 << 18))
        outs = [torch.empty(n, dtype=dt).pin_memory() for dt in dts]

        def call():
            check(lib.tb_cast_rays_host(dm.handle, n, *(addr(x) for x in ins), *(addr(x) for x in outs)),
                  "tb_cast_rays_host")

        for _ in range(3):
            call()
        ts = []
        for _ in range(args.reps):
            t0 = time.perf_counter()
            call()
            ts.append(time.perf_counter() - t0)
        ms = float(np.median(ts)) * 1e3
        if ref is None:
            ref = [x.clone() for x in outs]
        same = all(torch.equal(a, b) for a, b in zip(outs, ref))
        print(json.dumps({"mode": mode, "chunk": chunk, "ms": round(ms, 3), "Mrays_s": round(n / ms / 1e3, 1),
                          "equal_to_mode0": same}), flush=True)


if __name__ == "__main__":
    main()
