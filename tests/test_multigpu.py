"""Multi-GPU host logic on CPU: tile sharding + the single hit-buffer gather,
world_size 2 over gloo (the NCCL path runs the same code on GPUs)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_02309_b200 import multigpu


def test_shards_partition_the_job():
    W, H = 70, 37
    for world in (1, 2, 3, 8):
        for frames in (1, world):
            parts = [multigpu.shard_pixels(W, H, r, world, 16, frames) for r in range(world)]
            allp = np.concatenate(parts)
            assert np.array_equal(np.sort(allp), np.arange(W * H * frames))
            # interleaved tiles: tile counts per rank differ by at most one
            n_tiles = len(multigpu.tile_origins(W, H, 16)) * frames
            counts = [len(range(r, n_tiles, world)) for r in range(world)]
            assert max(counts) - min(counts) <= 1


def test_tile_order_matches_renderer():
    tiles = multigpu.tile_origins(40, 20, 16)
    assert tiles[:3] == [(0, 0, 16, 16), (16, 0, 32, 16), (32, 0, 40, 16)]
    assert tiles[3] == (0, 16, 16, 20)


def test_pack_roundtrip():
    n = 50
    g = torch.Generator().manual_seed(0)
    idx = torch.randperm(n, generator=g)
    vals = dict(status=torch.randint(0, 3, (n,), dtype=torch.uint8), cf=torch.randint(-1, 99, (n,), dtype=torch.int32),
                tet=torch.randint(0, 999, (n,), dtype=torch.int32), visited=torch.randint(1, 50, (n,), dtype=torch.int32),
                triangle=torch.randint(-1, 99, (n,), dtype=torch.int32), t=torch.rand(n, dtype=torch.float64),
                tet_back=torch.randint(-1, 999, (n,), dtype=torch.int32))
    buf = multigpu.pack_hits(idx, vals["status"], vals["cf"], vals["tet"], vals["visited"], vals["triangle"],
                             vals["t"], vals["tet_back"])
    out = multigpu.unpack_hits(buf)
    assert torch.equal(out["idx"], idx)
    for k, v in vals.items():
        assert torch.equal(out[k], v), k


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle
        from paper_2103_02309_b200.ingestion import build_box_fixture
        from paper_2103_02309_b200.scenes import camera_rays
        from paper_2103_02309_b200.tetmesh import encode

        raw, soup = build_box_fixture(6, occluders=[(0, 3, (1, 1), (5, 5))])
        mesh = encode(raw, "tet16", soup)
        W, H, frames = 48, 40, world
        idx = multigpu.shard_pixels(W, H, rank, world, 16, frames)
        o_all, d_all, st_all = [], [], []
        for f in range(frames):
            o, d = camera_rays((0.6 + 0.05 * f, 2.9, 3.1), (5.5, 3.2, 2.8), (0, 1, 0), 60.0, W, H)
            cam, _ = pyoracle.locate_points(mesh, np.array([[0.6 + 0.05 * f, 2.9, 3.1]]), np.array([0], np.int32))
            o_all.append(o)
            d_all.append(d)
            st_all.append(np.full(len(o), cam[0], np.int32))
        o_all, d_all, st_all = (np.concatenate(a) for a in (o_all, d_all, st_all))
        # per-rank trace of the shard (the CPU oracle stands in for the GPU kernel here)
        s, cf, tet, vis, tri, t, back = pyoracle.cast_rays_full(mesh, o_all[idx], d_all[idx], st_all[idx], n_threads=1)
        T = torch.from_numpy
        packed = multigpu.pack_hits(T(idx), T(s), T(cf), T(tet), T(vis), T(tri), T(t), T(back))
        full = multigpu.gather_hits(packed, W * H * frames)
        if rank == 0:
            exp = pyoracle.cast_rays_full(mesh, o_all, d_all, st_all, n_threads=1)
            ok = all(np.array_equal(full[k].numpy(), e) for k, e in
                     zip(("status", "cf", "tet", "visited", "triangle", "t", "tet_back"), exp))
            with open(result_path, "w") as fh:
                fh.write("ok" if ok else "mismatch")
        else:
            assert full is None
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_gather_equals_single_process(tmp_path):
    path = str(tmp_path / "result.txt")
    mp.start_processes(_worker, args=(2, _free_port(), path), nprocs=2, start_method="spawn", join=True)
    assert open(path).read() == "ok"


def _frame_worker(rank, world, port, result_path, chunks):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import pyoracle
        from paper_2103_02309_b200.ingestion import build_box_fixture
        from paper_2103_02309_b200.scenes import camera_rays
        from paper_2103_02309_b200.tetmesh import encode

        raw, soup = build_box_fixture(6, occluders=[(0, 3, (1, 1), (5, 5))])
        mesh = encode(raw, "tet20", soup)
        W, H, frames = 50, 36, world
        o_all, d_all, st_all = [], [], []
        for f in range(frames):
            o, d = camera_rays((0.6 + 0.05 * f, 2.9, 3.1), (5.5, 3.2, 2.8), (0, 1, 0), 60.0, W, H)
            cam, _ = pyoracle.locate_points(mesh, np.array([[0.6 + 0.05 * f, 2.9, 3.1]]), np.array([0], np.int32))
            o_all.append(o)
            d_all.append(d)
            st_all.append(np.full(len(o), cam[0], np.int32))
        o_all, d_all, st_all = (np.concatenate(a) for a in (o_all, d_all, st_all))
        fg = multigpu.FrameGather(W, H, world, rank, frames, chunks, "cpu", mesh.cf_triangle, mesh.cf_tets)
        idx = multigpu.shard_pixels(W, H, rank, world, 16, frames)
        T = torch.from_numpy
        for step in range(2):  # the gatherer is reusable frame after frame
            for k, (a, b) in enumerate(fg.my_pieces()):
                sel = idx[a:b]
                s, cf, tet, vis, tri, t, back = pyoracle.cast_rays_full(mesh, o_all[sel], d_all[sel], st_all[sel],
                                                                        n_threads=1)
                fg.send(k, T(s), T(cf), T(tet), T(vis), T(t))
            full = fg.finish()
        if rank == 0:
            exp = pyoracle.cast_rays_full(mesh, o_all, d_all, st_all, n_threads=1)
            ok = all(np.array_equal(full[k].numpy(), e) for k, e in
                     zip(("status", "cf", "tet", "visited", "triangle", "t", "tet_back"), exp))
            with open(result_path, "w") as fh:
                fh.write("ok" if ok else "mismatch")
        else:
            assert full is None
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("chunks", (1, 3))
def test_gloo_world2_frame_gather_overlapped(tmp_path, chunks):
    """The per-frame chunked gather (20 B records, root rebuilds triangle /
    tet_back / ray index) equals a single-process trace of the whole job."""
    path = str(tmp_path / "result.txt")
    mp.start_processes(_frame_worker, args=(2, _free_port(), path, chunks), nprocs=2, start_method="spawn",
                       join=True)
    assert open(path).read() == "ok"


def test_split_chunks():
    assert multigpu.split_chunks(10, 3) == [(0, 3), (3, 6), (6, 10)]
    assert multigpu.split_chunks(2, 4) == [(0, 0), (0, 1), (1, 1), (1, 2)]
    assert multigpu.split_chunks(0, 2) == [(0, 0), (0, 0)]


def _peer_fail_worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # no GPU here: the root's device allocation fails; every rank must
        # raise together (the bench then falls back to FrameGather) instead of
        # the others waiting forever for an IPC handle
        try:
            multigpu.PeerFrameGather(32, 16, world, rank, world, "cpu:0")
            outcome = "constructed"
        except RuntimeError as exc:
            outcome = "raised" if "peer frame assembly unavailable" in str(exc) else f"other: {exc}"
        flags = [None] * world
        dist.all_gather_object(flags, outcome)
        if rank == 0:
            with open(result_path, "w") as fh:
                fh.write(",".join(flags))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_peer_gather_failure_is_collective(tmp_path):
    path = str(tmp_path / "result.txt")
    mp.start_processes(_peer_fail_worker, args=(2, _free_port(), path), nprocs=2, start_method="spawn", join=True)
    assert open(path).read() == "raised,raised"


def test_trace_multi_checks_shapes_before_any_device_work():
    """multigpu.trace_multi validates the frame's ray arrays on the host side."""
    with pytest.raises(ValueError, match="frame"):
        multigpu.trace_multi([], 4, 4, torch.zeros((15, 3)), torch.zeros((16, 3)), torch.zeros(16, dtype=torch.int32))
    with pytest.raises(ValueError, match="contiguous"):
        multigpu.trace_multi([], 4, 4, torch.zeros((16, 3), dtype=torch.float64), torch.zeros((16, 3)),
                             torch.zeros(16, dtype=torch.int32))
