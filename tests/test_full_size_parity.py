"""Every BASELINE config at full size against the REFERENCE ITSELF.

The checker is the reference's own public batch API on its compiled kernels
(oracle/_ref/site: tetray.batch.cast_rays = _kernels.cast_rays +
the fp64 batch epilogue, /root/reference/pkg/src/tetray/_kernels.pyx:271-370,
batch.py:39-80), run on the GPU box's host cores over a thread pool.  All
seven per-ray arrays must be bit-identical:

* config 3 -- the config-2 scene in TetMesh-16, 3840x2160 primaries (8.3 M rays);
* config 4 -- 4096x4096 primaries on that mesh, then their 16.7 M diffuse
  secondaries (render.py:353-359 semantics, seed 4) spawned from the
  REFERENCE's primary hits, traced one ray per lane and direction-binned;
* config 5 -- the 50 M-tet Kuhn box (TetMesh-20, strip occluders), every
  64th pixel of 7680x4320 (518,400 rays), checked inside a full
  33 M-ray trace of the frame.
"""

from __future__ import annotations

import numpy as np
import pytest

from refpkg import have_ref, hits_mismatch, ref_cast_full

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_ref(), reason="oracle/_ref/site missing")]

NAMES = ("status", "cf", "tet", "visited", "triangle", "t", "tet_back")


def _trace_all(mesh, o, d, st, schedule="lane", chunk=1 << 24):
    import torch

    from paper_2103_02309_b200.device import device_mesh
    from paper_2103_02309_b200.trace import trace

    dev = torch.device("cuda", 0)
    dm = device_mesh(mesh, device=0)
    out = [[] for _ in NAMES]
    for a in range(0, len(st), chunk):
        b = min(len(st), a + chunk)
        r = trace(dm, *(torch.from_numpy(np.ascontiguousarray(x[a:b])).to(dev) for x in (o, d, st)),
                  schedule=schedule)
        for k, name in enumerate(NAMES):
            out[k].append(getattr(r, name).cpu().numpy())
    return [np.concatenate(x) for x in out]


def _assert_equal(got, exp, what):
    bad = hits_mismatch(got, exp)
    assert not any(bad.values()), f"{what}: mismatched values per array {bad}"


@pytest.fixture(scope="module")
def blob55_tet16():
    from paper_2103_02309_b200.scenes import blob_scene
    from paper_2103_02309_b200.tetmesh import relayout

    return relayout(blob_scene(55, layout="tet20", scheme="hilbert", check=False).mesh, "tet16")


def _camera_job(mesh, cam, W, H):
    from paper_2103_02309_b200 import kernels as K
    from paper_2103_02309_b200.workload import camera_rays

    o, d = camera_rays(cam["position"], cam["look_at"], cam["up"], cam["fov"], W, H)
    t, _ = K.locate_points(mesh, np.array([cam["position"]]), np.array([mesh.source_tet], np.int32))
    assert t[0] >= 0
    return o, d, np.full(len(o), t[0], np.int32)


@pytest.mark.timeout(1800)
def test_config3_full_frame_vs_reference(blob55_tet16):
    from paper_2103_02309_b200.workload import BLOB_CAMERA

    o, d, st = _camera_job(blob55_tet16, BLOB_CAMERA, 3840, 2160)
    got = _trace_all(blob55_tet16, o, d, st)
    exp = ref_cast_full(blob55_tet16, o, d, st)
    _assert_equal(got, exp, "config 3 (8,294,400 rays, tet16)")
    assert (exp[0] == 1).all()


@pytest.mark.timeout(2400)
def test_config4_secondaries_vs_reference(blob55_tet16):
    from paper_2103_02309_b200.workload import BLOB_CAMERA, diffuse_secondaries

    mesh = blob55_tet16
    o, d, st = _camera_job(mesh, BLOB_CAMERA, 4096, 4096)
    prim = ref_cast_full(mesh, o, d, st)
    _assert_equal(_trace_all(mesh, o, d, st), prim, "config 4 primaries (16,777,216 rays)")
    so, sd, sst = diffuse_secondaries(o, d, prim[5], prim[4], prim[2], mesh.triangle_coords(), seed=4)
    assert len(sst) == 16_777_216  # every primary hits
    exp = ref_cast_full(mesh, so, sd, sst)
    for schedule in ("lane", "binned"):
        _assert_equal(_trace_all(mesh, so, sd, sst, schedule=schedule), exp, f"config 4 secondaries ({schedule})")
    assert 60 < exp[3].mean() < 70  # 65.03 tets/ray


@pytest.mark.timeout(2400)
def test_config5_sampled_vs_reference():
    import torch

    from paper_2103_02309_b200.device import DeviceMesh
    from paper_2103_02309_b200.scenes import kuhn_strip_scene
    from paper_2103_02309_b200.trace import trace
    from paper_2103_02309_b200.workload import kuhn_camera

    mesh = kuhn_strip_scene(203, layout="tet20").mesh
    assert mesh.n_tets == 50_192_562
    W, H = 7680, 4320
    o, d, st = _camera_job(mesh, kuhn_camera(203), W, H)
    dev = torch.device("cuda", 0)
    dm = DeviceMesh(mesh, 0)
    res = trace(dm, *(torch.from_numpy(x).to(dev) for x in (o, d, st)))
    sl = slice(0, W * H, 64)
    got = [getattr(res, n)[sl].cpu().numpy() for n in NAMES]
    dm.close()
    exp = ref_cast_full(mesh, o[sl], d[sl], st[sl], chunk=1 << 12)
    _assert_equal(got, exp, "config 5 (every 64th pixel, 518,400 rays)")
    assert exp[3].mean() > 100
