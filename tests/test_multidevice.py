"""Multi-GPU paths on DISTINCT devices (skipped on a one-GPU box).

Everything the one-GPU tests exercise with ranks / replicas sharing cuda:0,
here across real device boundaries: peer access and cross-device copies
(tb_mesh_replicate), cross-device event joins and P2P loads / stores
(tb_trace_multi), CUDA IPC handles opened on another GPU (PeerFrameGather),
and bench.py --gpus 2 end to end (frame 0 of the assembled job equals the
reference's digest).  SURVEY s8(e): per-ray outputs must equal the
single-GPU run and the oracle.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def _ndev() -> int:
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


pytestmark = [pytest.mark.gpu, pytest.mark.skipif(_ndev() < 2, reason="needs >= 2 GPUs")]


def _scene():
    from paper_2103_02309_b200.scenes import BLOB_CAMERA, blob_scene, camera_rays

    mesh = blob_scene(12, layout="tet20").mesh
    W, H = 203, 117
    o, d = camera_rays(BLOB_CAMERA["position"], BLOB_CAMERA["look_at"], BLOB_CAMERA["up"], BLOB_CAMERA["fov"], W, H)
    return mesh, W, H, o, d


def test_replicate_and_trace_multi_across_devices():
    import torch

    from paper_2103_02309_b200.device import DeviceMesh
    from paper_2103_02309_b200.multigpu import trace_multi
    from paper_2103_02309_b200.scenes import BLOB_CAMERA
    from paper_2103_02309_b200.trace import locate, trace

    mesh, W, H, o, d = _scene()
    n = min(_ndev(), 4)
    dms = [DeviceMesh(mesh, 0)]
    dms += [dms[0].replicate(k) for k in range(1, n)]  # peer-to-peer HBM copies
    dev0 = torch.device("cuda", 0)
    cam, _ = locate(dms[0], torch.tensor([BLOB_CAMERA["position"]], dtype=torch.float64, device=dev0),
                    torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev0))
    go, gd = torch.from_numpy(o).to(dev0), torch.from_numpy(d).to(dev0)
    gs = torch.full((W * H,), int(cam.item()), dtype=torch.int32, device=dev0)
    ref = trace(dms[0], go, gd, gs)
    for k in range(1, n):  # each replica alone, on its own device
        dk = torch.device("cuda", k)
        rk = trace(dms[k], go.to(dk), gd.to(dk), gs.to(dk))
        for f in ("status", "cf", "tet", "visited", "triangle", "t", "tet_back"):
            assert torch.equal(getattr(rk, f).to(dev0), getattr(ref, f)), (k, f)
    got = trace_multi(dms, W, H, go, gd, gs)  # P2P loads / stores + cross-device joins
    torch.cuda.synchronize()
    for f in ("status", "cf", "tet", "visited", "triangle", "t", "tet_back"):
        assert torch.equal(getattr(got, f), getattr(ref, f)), f


def _worker(rank, world, port, path):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        from oracle import pyoracle
        from paper_2103_02309_b200 import multigpu
        from paper_2103_02309_b200.device import device_mesh

        mesh, W, H, o, d = _scene()
        cam, _ = pyoracle.locate_points(mesh, np.array([[0.9, 5.0, 5.05]]), np.array([mesh.source_tet], np.int32))
        o_all = np.concatenate([o] * world)
        d_all = np.concatenate([d] * world)
        st_all = np.full(len(o_all), cam[0], np.int32)
        rr = tuple(torch.from_numpy(a).to(dev) for a in (o_all, d_all)) if rank == 0 else True
        pg = multigpu.PeerFrameGather(W, H, world, rank, world, dev, root_rays=rr)  # IPC opened on another GPU
        idx = pg.idx.cpu().numpy()
        dm = device_mesh(mesh, device=rank)
        g = [torch.from_numpy(np.ascontiguousarray(a[idx])).to(dev) for a in (o_all, d_all, st_all)]
        for sched in ("lane", "binned"):
            frame = pg.step(dm, *g, schedule=sched)
        if rank == 0:
            exp = pyoracle.cast_rays_full(mesh, o_all, d_all, st_all)
            ok = all(np.array_equal(frame[k].cpu().numpy(), e) for k, e in
                     zip(("status", "cf", "tet", "visited", "triangle", "t", "tet_back"), exp))
            open(path, "w").write("ok" if ok else "mismatch")
        pg.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_peer_frame_assembly_across_devices(tmp_path):
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    path = str(tmp_path / "r.txt")
    mp.start_processes(_worker, args=(2, port, path), nprocs=2, start_method="spawn", join=True)
    assert open(path).read() == "ok"


@pytest.mark.timeout(1200)
def test_bench_two_gpus():
    env = dict(os.environ, NCCL_DEBUG="INFO")
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "5", "--warmup", "3", "--no-e2e",
                          "--no-l2-probe"], cwd=ROOT, capture_output=True, text=True, timeout=1200, env=env)
    assert out.returncode == 0, out.stderr[-4000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    chk = line["gather"]["check"]
    assert chk["frame0_vs_reference_digest"] and chk["frame0_epilogue_vs_reference_digest"], chk
    if (ROOT / "gpurun_out").is_dir():
        (ROOT / "gpurun_out" / "bench_2gpu_nccl_debug.log").write_text(out.stderr[-200000:])
