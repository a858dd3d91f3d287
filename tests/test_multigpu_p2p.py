"""The fused multi-GPU frame assembly (PeerFrameGather): two ranks -- here
two processes sharing cuda:0, the same CUDA IPC mapping that spans GPUs over
NVLink on a multi-GPU node -- trace their tiles and store every ray's results
straight into the root's full-frame arrays; the frame must equal a
single-process trace of the whole job (the C oracle)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_path, mode="full"):
    """mode: "full" (29 B per ray stored), "lean" (13 B, root epilogue),
    "pipelined" (lean, the root epilogue of step k run beside step k+1;
    each step returns the previous job's frame, finish() the last one),
    "binned" (the binned walk's permutation composed with the scatter
    index), "sctp" (the ScTP walk scattering), "partial" (each rank traces
    a data-dependent subset -- like diffuse secondaries of primary hits --
    under the binned schedule; untraced slots keep the "no ray" values).
    Every mode runs two steps with different rays (camera moved between
    them): the returned frame must be the second job's, exactly."""
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle
        from paper_2103_02309_b200 import multigpu
        from paper_2103_02309_b200.device import device_mesh
        from paper_2103_02309_b200.ingestion import build_box_fixture
        from paper_2103_02309_b200.scenes import camera_rays
        from paper_2103_02309_b200.tetmesh import encode

        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        raw, soup = build_box_fixture(6, occluders=[(0, 3, (1, 1), (5, 5))])
        mesh = encode(raw, "tet20", soup)
        W, H, frames = 80, 60, world

        def job(shift):
            o_all, d_all, st_all = [], [], []
            for f in range(frames):
                pos = (0.6 + 0.05 * f + shift, 2.9, 3.1)
                o, d = camera_rays(pos, (5.5, 3.2, 2.8), (0, 1, 0), 60.0, W, H)
                cam, _ = pyoracle.locate_points(mesh, np.array([pos]), np.array([0], np.int32))
                o_all.append(o)
                d_all.append(d)
                st_all.append(np.full(len(o), cam[0], np.int32))
            return [np.concatenate(a) for a in (o_all, d_all, st_all)]

        jobs = [job(0.0), job(0.13)] + ([job(0.21)] if mode == "pipelined" else [])
        lean = mode in ("lean", "pipelined")
        index = None
        if mode == "partial":  # drop every third ray of this rank's shard
            shard = multigpu.shard_pixels(W, H, rank, world, 16, frames)
            index = shard[np.arange(len(shard)) % 3 != 1]
        root_rays = None
        if lean:
            root_rays = tuple(torch.from_numpy(a).to(dev) for a in jobs[0][:2]) if rank == 0 else True
        pg = multigpu.PeerFrameGather(W, H, world, rank, frames, dev, root_rays=root_rays, index=index,
                                      pipelined=mode == "pipelined")
        idx = pg.idx.cpu().numpy()
        dm = device_mesh(mesh, device=0)
        schedule = "binned" if mode in ("binned", "partial") else "lane"
        names = ("status", "cf", "tet", "visited", "triangle", "t", "tet_back")
        lagged_ok = True
        for k, (o_all, d_all, st_all) in enumerate(jobs):  # reusable frame after frame, rays changing
            g = [torch.from_numpy(np.ascontiguousarray(a[idx])).to(dev) for a in (o_all, d_all, st_all)]
            rr = tuple(torch.from_numpy(a).to(dev) for a in (o_all, d_all)) if (lean and rank == 0) else None
            frame = pg.step(dm, *g, schedule=schedule, sctp=mode == "sctp", root_rays=rr)
            if mode == "pipelined" and rank == 0 and k >= 1:  # step k returns job k-1, complete
                prev = pyoracle.cast_rays_full(mesh, *jobs[k - 1], n_threads=1)
                bad = [nm for nm, e in zip(names, prev) if not np.array_equal(frame[nm].cpu().numpy(), e)]
                if bad:
                    lagged_ok = False
                    print(f"pipelined step {k}: lagged frame differs in {bad}", flush=True)
        if mode == "pipelined":
            frame = pg.finish()
        with pytest.raises(ValueError):  # the ray count must match the rank's index
            pg.step(dm, g[0][:-1], g[1][:-1], g[2][:-1])
        if rank == 0:
            o_all, d_all, st_all = jobs[-1]
            exp = list(pyoracle.cast_rays_full(mesh, o_all, d_all, st_all, n_threads=1, sctp=mode == "sctp"))
            if mode == "partial":  # slots no rank traced
                traced = np.zeros(len(st_all), bool)
                for r in range(world):
                    sh = multigpu.shard_pixels(W, H, r, world, 16, frames)
                    traced[sh[np.arange(len(sh)) % 3 != 1]] = True
                for e, fill in zip(exp, (0, -1, -1, 0, -1, np.inf, -1)):
                    e[~traced] = fill
            bad = [k for k, e in zip(names, exp) if not np.array_equal(frame[k].cpu().numpy(), e)]
            if bad:
                print(f"{mode}: final frame differs in {bad}", flush=True)
            ok = lagged_ok and not bad
            with open(result_path, "w") as fh:
                fh.write("ok" if ok else "mismatch")
        pg.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("mode", ("full", "lean", "pipelined", "binned", "sctp", "partial"))
def test_p2p_frame_assembly_two_ranks(tmp_path, mode):
    """Two ranks (sharing cuda:0 here) assemble the frame set on rank 0 by P2P
    stores, in every mode (see _worker); the frame equals the oracle."""
    import torch.multiprocessing as mp

    path = str(tmp_path / "result.txt")
    mp.start_processes(_worker, args=(2, _free_port(), path, mode), nprocs=2, start_method="spawn", join=True)
    assert open(path).read() == "ok"


@pytest.mark.gpu
@pytest.mark.parametrize("replicas,layout", [(1, "tet20"), (2, "tet20"), (3, "tet16")])
def test_trace_multi_equals_single_trace(replicas, layout):
    """tb_trace_multi with replicas sharing cuda:0 (the single-GPU box; on a
    node each replica sits on its own GPU): the tile split, the gathered ray
    reads and the scattered stores give exactly the single-GPU frame."""
    import numpy as np
    import torch

    from paper_2103_02309_b200.device import DeviceMesh
    from paper_2103_02309_b200.multigpu import trace_multi
    from paper_2103_02309_b200.scenes import BLOB_CAMERA, blob_scene, camera_rays
    from paper_2103_02309_b200.tetmesh import relayout
    from paper_2103_02309_b200.trace import locate, trace

    mesh = relayout(blob_scene(8, layout="tet20").mesh, layout)
    W, H = 101, 67  # ragged edge tiles
    o, d = camera_rays(BLOB_CAMERA["position"], BLOB_CAMERA["look_at"], BLOB_CAMERA["up"], BLOB_CAMERA["fov"], W, H)
    dev = torch.device("cuda", 0)
    dms = [DeviceMesh(mesh, 0)]
    dms += [dms[0].replicate(0) for _ in range(replicas - 1)]  # peer copies (same device on this box)
    cam, _ = locate(dms[0], torch.tensor([BLOB_CAMERA["position"]], dtype=torch.float64, device=dev),
                    torch.tensor([mesh.source_tet], dtype=torch.int32, device=dev))
    go, gd = torch.from_numpy(o).to(dev), torch.from_numpy(d).to(dev)
    gs = torch.full((W * H,), int(cam.item()), dtype=torch.int32, device=dev)
    ref = trace(dms[0], go, gd, gs)
    got = trace_multi(dms, W, H, go, gd, gs)
    torch.cuda.synchronize()
    for k in ("status", "cf", "tet", "visited", "triangle", "t", "tet_back"):
        assert torch.equal(getattr(got, k), getattr(ref, k)), k
    assert int(got.visited.min()) >= 1


@pytest.mark.gpu
def test_trace_multi_rejects_non_replicas():
    import torch

    from paper_2103_02309_b200._lib import TetB200Error
    from paper_2103_02309_b200.device import DeviceMesh
    from paper_2103_02309_b200.multigpu import trace_multi
    from paper_2103_02309_b200.scenes import blob_scene
    from paper_2103_02309_b200.tetmesh import relayout

    mesh = blob_scene(6, layout="tet20").mesh
    a, b = DeviceMesh(mesh, 0), DeviceMesh(relayout(mesh, "tet16"), 0)
    z3 = torch.zeros((16 * 16, 3), dtype=torch.float32, device="cuda")
    st = torch.zeros(16 * 16, dtype=torch.int32, device="cuda")
    with pytest.raises(TetB200Error, match="replica"):
        trace_multi([a, b], 16, 16, z3, z3, st)
