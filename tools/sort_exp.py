#!/usr/bin/env python
"""Experiment: does sorting incoherent rays before the walk pay on B200?
Config-4 style secondaries; keys: start tet, start tet + direction octant,
origin Hilbert cell + octant.  Times sort + gather + trace + scatter."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_02309_b200.device import DeviceMesh  # noqa: E402
from paper_2103_02309_b200.scenes import BLOB_CAMERA, blob_scene, camera_rays, diffuse_secondaries  # noqa: E402
from paper_2103_02309_b200.trace import empty_result, locate, trace  # noqa: E402


def t_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = []
    for _ in range(reps):
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b))
    return float(np.median(out))


def main():
    W = H = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    dev = torch.device("cuda", 0)
    sc = blob_scene(55, layout="tet16", scheme="hilbert", check=False)
    m = sc.mesh
    dm = DeviceMesh(m, 0)
    c = BLOB_CAMERA
    o, d = camera_rays(c["position"], c["look_at"], c["up"], c["fov"], W, H)
    cam, _ = locate(dm, torch.tensor([c["position"]], dtype=torch.float64, device=dev),
                    torch.tensor([m.source_tet], dtype=torch.int32, device=dev))
    go, gd = torch.from_numpy(o).to(dev), torch.from_numpy(d).to(dev)
    gs = torch.full((len(o),), int(cam.item()), dtype=torch.int32, device=dev)
    prim = trace(dm, go, gd, gs)
    torch.cuda.synchronize()
    so, sd, sst = diffuse_secondaries(o, d, prim.t.cpu().numpy(), prim.triangle.cpu().numpy(),
                                      prim.tet.cpu().numpy(), m.triangle_coords(), seed=4)
    n = len(so)
    O, D, S = (torch.from_numpy(a).to(dev) for a in (so, sd, sst))
    res = empty_result(n, dev)
    base = t_ms(lambda: trace(dm, O, D, S, out=res))
    ref_vis = res.visited.clone()
    print(f"n={n} unsorted trace {base:.3f} ms  {n / base / 1e3:.0f} Mrays/s", flush=True)
    octant = ((D[:, 0] > 0).long() << 2) | ((D[:, 1] > 0).long() << 1) | (D[:, 2] > 0).long()
    keys = {
        "tet": S.long(),
        "tet+oct": (S.long() << 3) | octant,
        "oct+tet": (octant << 32) | S.long(),
    }
    for name, key in keys.items():
        def run():
            perm = torch.argsort(key)
            r2 = trace(dm, O[perm].contiguous(), D[perm].contiguous(), S[perm].contiguous())
            out = empty_result(n, dev)
            for src, dst in zip((r2.status, r2.cf, r2.tet, r2.visited, r2.triangle, r2.t, r2.tet_back),
                                (out.status, out.cf, out.tet, out.visited, out.triangle, out.t, out.tet_back)):
                dst[perm] = src
            return out
        tot = t_ms(run)
        perm = torch.argsort(key)
        Os, Ds, Ss = O[perm].contiguous(), D[perm].contiguous(), S[perm].contiguous()
        only = t_ms(lambda: trace(dm, Os, Ds, Ss, out=res))
        chk = run()
        ok = bool(torch.equal(chk.visited, ref_vis))
        print(f"{name:8s} total {tot:.3f} ms ({n / tot / 1e3:.0f} Mrays/s), trace only {only:.3f} ms, equal={ok}",
              flush=True)


if __name__ == "__main__":
    main()
