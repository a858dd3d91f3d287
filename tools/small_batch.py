#!/usr/bin/env python
"""Renderer-granularity calls (bench.small_batch) on the config-2 scene:
tetray.batch.cast_rays with kernels= the CUDA module vs the reference's own
compiled kernels, 256 / 4096 / 65536 rays per call from all host threads.

    python tools/small_batch.py [--config 2]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    mesh = bench.build_scene(cfg).mesh
    from paper_2103_02309_b200 import kernels as K

    o, d, pos = bench.frame_rays(cfg, 0)
    cam, _ = K.locate_points(mesh, pos[None], np.array([mesh.source_tet], np.int32))
    st = np.full(len(o), cam[0], np.int32)
    print(json.dumps(bench.small_batch(argparse.Namespace(), mesh, o, d, st, os.cpu_count() or 1)), flush=True)


if __name__ == "__main__":
    main()
