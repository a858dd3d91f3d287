"""GPU parity: the sm_100a kernels vs the reference's outputs (golden) and
the CPU oracle, bit for bit.  Modelled on the reference's backend-parity
suite (tests/test_kernels.py:26-103) and acceptance criteria 2/3/9
(tests/test_acceptance.py:67-119,325-342).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import FIXTURES, RAY_SEEDS, digest, golden_mesh

pytestmark = pytest.mark.gpu

LAYOUTS4 = ("tet32", "tet20", "tet16", "tet80")
NAMES7 = ("status", "cf", "tet", "visited", "triangle", "t", "tet_back")


@pytest.fixture(scope="module")
def K():
    from paper_2103_02309_b200 import kernels

    return kernels


@pytest.fixture(scope="module")
def O():
    from oracle import pyoracle

    return pyoracle


def _rays(mesh, name, n=10000):
    from paper_2103_02309_b200.scenes import interior_rays

    return interior_rays(mesh, n, RAY_SEEDS[name])


@pytest.mark.parametrize("name", FIXTURES)
@pytest.mark.parametrize("layout", LAYOUTS4)
def test_cast_matches_reference_golden(golden, digests, K, name, layout):
    """All 7 per-ray outputs (incl. fused epilogue) equal the reference's."""
    base = golden_mesh(golden, name, "tet20" if layout == "tet80" else layout)
    o, d, st = _rays(base, name)
    assert digest(o, d, st) == digests[f"{name}/rays"]
    out = K.cast_rays_full(base, o, d, st, layout=layout)
    ref_layout = "tet32" if layout == "tet80" else layout
    assert digest(*out[:4]) == digests[f"{name}/{ref_layout}/cast10k"]
    assert digest(*out[4:]) == digests[f"{name}/{ref_layout}/cast10k_epilogue"]
    for k, a in zip(NAMES7, out):
        assert np.array_equal(a[:2000], golden[f"{name}/cast/{k}"]), k


@pytest.mark.parametrize("name", ("pane4", "model"))
def test_cast_protocol_and_oracle(golden, K, O, name):
    """The 4-tuple protocol call equals the C oracle on 50k rays."""
    from paper_2103_02309_b200.scenes import interior_rays

    m = golden_mesh(golden, name)
    o, d, st = interior_rays(m, 50000, 7)
    got = K.cast_rays(m, o, d, st)
    exp = O.cast_rays(m, o, d, st)
    for a, b in zip(got, exp):
        assert a.dtype == b.dtype and np.array_equal(a, b)


@pytest.mark.parametrize("layout", LAYOUTS4)
def test_visit_sequences(golden, K, layout):
    """Visit sequences equal the reference's for every layout (acceptance 3)."""
    from paper_2103_02309_b200.scenes import interior_rays

    m = golden_mesh(golden, "region4")
    o, d, st = interior_rays(m, 500, 41)
    *_, seq, off = K.cast_rays_csr(m, o, d, st, layout=layout)
    assert np.array_equal(off, golden["region4/visits/offsets"])
    assert np.array_equal(seq, golden["region4/visits/seq"])


def test_visits_sink_protocol(golden, K):
    """visits_sink wavefronts reassemble like the reference batch layer does."""
    from paper_2103_02309_b200.scenes import interior_rays

    m = golden_mesh(golden, "region4")
    o, d, st = interior_rays(m, 500, 41)
    sink: list = []
    _, _, _, visited = K.cast_rays(m, o, d, st, visits_sink=sink)
    offsets = np.zeros(len(o) + 1, dtype=np.int64)
    np.cumsum(visited, out=offsets[1:])
    visits = np.empty(int(offsets[-1]), dtype=np.int32)
    pos = offsets[:-1].copy()
    for rays, tets in sink:  # batch.py:103-114 scatter path
        visits[pos[rays]] = tets
        pos[rays] += 1
    assert np.array_equal(visits, golden["region4/visits/seq"])


def test_locate(golden, K):
    m = golden_mesh(golden, "region4")
    tet, vis = K.locate_points(m, golden["region4/locate/q"], np.full(3000, m.source_tet, np.int32))
    assert np.array_equal(tet, golden["region4/locate/tet"])
    assert np.array_equal(vis, golden["region4/locate/visited"])
    assert (tet == -1).any() and (tet >= 0).any()


@pytest.mark.parametrize("layout", ("tet32", "tet20", "tet16"))
def test_shadow(golden, K, layout):
    from paper_2103_02309_b200.tetmesh import relayout

    m = relayout(golden_mesh(golden, "pane4"), layout)
    occ, vis = K.shadow_rays(m, golden["pane4/shadow/p"], golden["pane4/shadow/light"], golden["pane4/shadow/p_tet"],
                             int(golden["pane4/shadow/light_tet"][0]))
    assert occ.dtype == bool
    assert np.array_equal(occ, golden["pane4/shadow/occ"])
    assert np.array_equal(vis, golden["pane4/shadow/visited"])
    assert 0.0 < occ.mean() < 1.0


@pytest.mark.parametrize("name", ("pane4", "region4", "model"))
@pytest.mark.parametrize("layout", LAYOUTS4)
def test_sctp_kernel_matches_oracle(golden, K, O, name, layout):
    """The fp64 ScTP fallback walk: bit-exact vs the C restatement, and equal
    to the 2-D walk except counted tie rays (walk unpinned)."""
    base = golden_mesh(golden, name, "tet20" if layout == "tet80" else layout)
    o, d, st = _rays(base, name)
    got = K.cast_rays_full(base, o, d, st, layout=layout, sctp=True)
    exp = O.cast_rays_full(base, o, d, st, layout=layout, sctp=True)
    for k, a, b in zip(NAMES7, got, exp):
        assert np.array_equal(a, b), k
    two_d = K.cast_rays_full(base, o, d, st, layout=layout)
    mism = int(np.sum((got[4] != two_d[4]) | (got[2] != two_d[2])))
    assert mism <= len(o) // 1000  # grazing/tie rays only


def test_cycle_guard_lattice_camera(digests, K, O):
    """The reference's own cycle-guard rays: status 2 and
    visited = n_tets + 1 on exactly the same 4 rays, all else identical."""
    from paper_2103_02309_b200.ingestion import build_box_fixture
    from paper_2103_02309_b200.scenes import camera_rays
    from paper_2103_02309_b200.tetmesh import encode

    raw, soup = build_box_fixture(8, occluders=[(0, 4, (2, 2), (6, 6))])
    m = encode(raw, "tet20", soup)
    o, d = camera_rays((4.0, 4.0, 0.5), (4.0, 4.0, 8.0), (0.0, 1.0, 0.0), 68.0, 1024, 1024)
    assert digest(o, d) == digests["lattice8/rays"]
    cam, _ = K.locate_points(m, np.array([[4.0, 4.0, 0.5]]), np.array([m.source_tet], np.int32))
    assert int(cam[0]) == digests["lattice8/cam_tet"]
    st = np.full(len(o), cam[0], np.int32)
    out = K.cast_rays(m, o, d, st)
    assert digest(*out) == digests["lattice8/cast"]
    err = np.nonzero(out[0] == 2)[0]
    assert err.tolist() == digests["lattice8/errors"]["rays"]
    assert out[3][err].tolist() == [m.n_tets + 1] * len(err)


@pytest.mark.parametrize("layout", ("tet16", "tet20", "tet32"))
def test_cycle_guard_fast_forward_exact(K, O, layout):
    """n_tets (24,576) above the device's cycle-check threshold: the guard
    rays go through the Brent fast-forward (long_walk) and must still give
    the reference's status / terminating tet / visited = n_tets + 1."""
    from paper_2103_02309_b200.ingestion import build_kuhn_box
    from paper_2103_02309_b200.scenes import camera_rays
    from paper_2103_02309_b200.tetmesh import encode

    raw, soup = build_kuhn_box(16, [(0, 8, (4, 4), (12, 12))])
    m = encode(raw, layout, soup)
    o, d = camera_rays((8.0, 8.0, 0.5), (8.0, 8.0, 16.0), (0.0, 1.0, 0.0), 68.0, 512, 512)
    cam, _ = O.locate_points(m, np.array([[8.0, 8.0, 0.5]]), np.array([0], np.int32))
    st = np.full(len(o), cam[0], np.int32)
    got = K.cast_rays_full(m, o, d, st)
    exp = O.cast_rays_full(m, o, d, st)
    for k, a, b in zip(NAMES7, got, exp):
        assert np.array_equal(a, b), k
    err = np.nonzero(got[0] == 2)[0]
    assert len(err) == 3 and (got[3][err] == m.n_tets + 1).all()


def test_config5_builder_small_scale_parity(K, O):
    """The config-5 scene family (stretched Kuhn box + thin strip occluders)
    at a small size: GPU == oracle on every ray of a camera frame."""
    from paper_2103_02309_b200.scenes import camera_rays, kuhn_camera, kuhn_strip_scene

    sc = kuhn_strip_scene(24, layout="tet16")
    cam = kuhn_camera(24)
    o, d = camera_rays(cam["position"], cam["look_at"], cam["up"], cam["fov"], 320, 240)
    c, _ = K.locate_points(sc.mesh, np.array([cam["position"]]), np.array([sc.mesh.source_tet], np.int32))
    assert c[0] >= 0
    st = np.full(len(o), c[0], np.int32)
    got = K.cast_rays_full(sc.mesh, o, d, st)
    exp = O.cast_rays_full(sc.mesh, o, d, st)
    for k, a, b in zip(NAMES7, got, exp):
        assert np.array_equal(a, b), k
    assert (got[0] == 1).all()


@pytest.mark.parametrize("scheme", ("none", "hilbert"))
def test_config1_blob12_camera(digests, K, scheme):
    """BASELINE config 1 (blob GRID=12, 256x256 primaries) equals the
    reference end to end: scene build, camera tet, hits, fp64 t."""
    from paper_2103_02309_b200.scenes import BLOB_CAMERA, blob_scene, camera_rays
    from conftest import mesh_digest

    sc = blob_scene(12, layout="tet20", scheme=scheme)
    assert mesh_digest(sc.mesh) == digests[f"blob12/{scheme}/mesh"]
    o, d = camera_rays(BLOB_CAMERA["position"], BLOB_CAMERA["look_at"], BLOB_CAMERA["up"], BLOB_CAMERA["fov"], 256, 256)
    assert digest(o, d) == digests["blob12/rays"]
    cam, _ = K.locate_points(sc.mesh, np.array([BLOB_CAMERA["position"]]), np.array([sc.mesh.source_tet], np.int32))
    assert int(cam[0]) == digests[f"blob12/{scheme}/cam_tet"]
    out = K.cast_rays_full(sc.mesh, o, d, np.full(len(o), cam[0], np.int32))
    assert digest(*out[:4]) == digests[f"blob12/{scheme}/cast"]
    assert digest(*out[4:]) == digests[f"blob12/{scheme}/epilogue"]


@pytest.mark.parametrize("name", ("box4", "pane4", "open_box4"))
def test_cast_rays_auto_vs_reference(golden, K, name):
    """Batched cast_ray_auto (locate or hull-clip, then walk) against the
    reference's scalar traversal.cast_ray_auto on origins in and out of the
    box: hit/miss, constrained face, triangle, front/back tets and visited
    exact; t to 1e-12 relative (the scalar engine sums dot products in a
    different order than the batch epilogue)."""
    from paper_2103_02309_b200 import batch

    m = golden_mesh(golden, name)
    o, d = golden[f"{name}/auto/o"], golden[f"{name}/auto/d"]
    ref = golden[f"{name}/auto/result"]
    h = batch.cast_rays_auto(m, o, d)
    hit = ref[:, 0] == 1
    assert np.array_equal(h.status == 1, hit)
    assert np.array_equal(h.cf[hit], ref[hit, 1].astype(np.int32))
    assert np.array_equal(h.triangle[hit], ref[hit, 2].astype(np.int32))
    assert np.allclose(h.t[hit], ref[hit, 3], rtol=1e-12, atol=0)
    assert np.array_equal(h.tet_front[hit], ref[hit, 4].astype(np.int32))
    assert np.array_equal(h.tet_back[hit], ref[hit, 5].astype(np.int32))
    assert np.array_equal(h.visited, ref[:, 6].astype(np.int32))


@pytest.mark.parametrize("name", ("region4", "model"))
@pytest.mark.parametrize("scheme", ("none", "hilbert", "shuffle"))
def test_visit_locality_metric(golden, digests, name, scheme):
    """render.visit_locality_metric (render.py:565-591) from GPU visit
    sequences equals the reference's value for every reorder scheme."""
    from paper_2103_02309_b200.io import visit_locality_metric
    from paper_2103_02309_b200.tetmesh import reorder

    m = reorder(golden_mesh(golden, name), scheme)
    assert visit_locality_metric(m) == digests[f"{name}/locality/{scheme}"]


def test_device_camera_rays_and_trace_camera(digests):
    """On-device primary rays are bit-identical to render.camera_rays, and the
    all-device render pass reproduces the reference's config-1 digests."""
    import torch

    from paper_2103_02309_b200.scenes import BLOB_CAMERA, blob_scene, camera_rays
    from paper_2103_02309_b200.trace import camera_rays_device, trace_camera

    o_h, d_h = camera_rays(BLOB_CAMERA["position"], BLOB_CAMERA["look_at"], BLOB_CAMERA["up"], BLOB_CAMERA["fov"],
                           256, 256)
    o, d = camera_rays_device(BLOB_CAMERA, 256, 256, "cuda:0")
    assert np.array_equal(o.cpu().numpy(), o_h) and np.array_equal(d.cpu().numpy(), d_h)
    assert digest(o.cpu().numpy(), d.cpu().numpy()) == digests["blob12/rays"]
    pix = torch.tensor([5, 70000 % 65536, 65535], dtype=torch.int64, device="cuda:0")
    o2, d2 = camera_rays_device(BLOB_CAMERA, 256, 256, "cuda:0", pixels=pix)
    assert np.array_equal(d2.cpu().numpy(), d_h[pix.cpu().numpy()])
    sc = blob_scene(12, scheme="hilbert")
    res, cam = trace_camera(sc.mesh, BLOB_CAMERA, 256, 256)
    torch.cuda.synchronize()
    assert cam == digests["blob12/hilbert/cam_tet"]
    got = [x.cpu().numpy() for x in (res.status, res.cf, res.tet, res.visited, res.triangle, res.t, res.tet_back)]
    assert digest(*got[:4]) == digests["blob12/hilbert/cast"]
    assert digest(*got[4:]) == digests["blob12/hilbert/epilogue"]
    # hits written straight into pinned host memory (zero-copy outputs)
    from paper_2103_02309_b200.trace import TraceResult

    host = TraceResult(*[torch.empty(256 * 256, dtype=x.dtype).pin_memory() for x in
                         (res.status, res.cf, res.triangle, res.t, res.tet, res.tet_back, res.visited)])
    trace_camera(sc.mesh, BLOB_CAMERA, 256, 256, out=host, cam_tet=cam)
    torch.cuda.synchronize()
    h = [x.numpy() for x in (host.status, host.cf, host.tet, host.visited, host.triangle, host.t, host.tet_back)]
    assert digest(*h[:4]) == digests["blob12/hilbert/cast"] and digest(*h[4:]) == digests["blob12/hilbert/epilogue"]


@pytest.mark.parametrize("layout", ("tet16", "tet20", "tet32", "tet80"))
def test_fused_camera_pass_equals_two_launch_path(layout):
    """tb_trace_camera (the pixel's ray formed in registers, one launch) is
    bit-identical to tb_camera_rays + the cast, for every layout, a ragged
    frame (partial last block), device and pinned-host outputs; bad
    arguments fail loudly."""
    import torch

    from paper_2103_02309_b200._lib import lib
    from paper_2103_02309_b200.device import device_mesh
    from paper_2103_02309_b200.scenes import BLOB_CAMERA, blob_scene
    from paper_2103_02309_b200.trace import TraceResult, trace_camera

    sc = blob_scene(12, scheme="hilbert")
    for W, H in ((256, 256), (333, 217)):
        a, cam = trace_camera(sc.mesh, BLOB_CAMERA, W, H, layout=layout, fused=False)
        b, cam_b = trace_camera(sc.mesh, BLOB_CAMERA, W, H, layout=layout, cam_tet=cam)
        host = TraceResult(*[torch.empty(W * H, dtype=x.dtype).pin_memory() for x in
                             (a.status, a.cf, a.triangle, a.t, a.tet, a.tet_back, a.visited)])
        trace_camera(sc.mesh, BLOB_CAMERA, W, H, layout=layout, cam_tet=cam, out=host)
        torch.cuda.synchronize()
        assert cam_b == cam
        for k in NAMES7:
            assert torch.equal(getattr(a, k), getattr(b, k)), (layout, W, H, k)
            assert torch.equal(getattr(a, k).cpu(), getattr(host, k)), (layout, W, H, k)
    dm = device_mesh(sc.mesh, device=0, layout=layout)
    fr = np.zeros(14)
    r = a
    args = (fr.ctypes.data, 0, r.status.data_ptr(), r.cf.data_ptr(), r.tet.data_ptr(), r.visited.data_ptr(), None,
            None, None, None)
    assert lib.tb_trace_camera(dm.handle, 0, 4, *args) != 0
    assert lib.tb_trace_camera(dm.handle, 4, 4, fr.ctypes.data, -1, *args[2:]) != 0
    assert lib.tb_trace_camera(dm.handle, 4, 4, fr.ctypes.data, 1 << 30, *args[2:]) != 0
    assert lib.tb_trace_camera(dm.handle, 4, 4, None, 0, *args[2:]) != 0
    with pytest.raises(ValueError):
        trace_camera(sc.mesh, BLOB_CAMERA, 8, 8, layout=layout, cam_tet=cam, out=a)  # wrong-size out


def test_batch_layer_mirror(golden, K):
    """The mirrored batch API (batch.py:39-80 semantics) over the CUDA module."""
    from paper_2103_02309_b200 import batch
    from paper_2103_02309_b200.scenes import interior_rays

    m = golden_mesh(golden, "pane4")
    o, d, st = interior_rays(m, 4000, 40)
    h = batch.cast_rays(m, o, d, st)
    assert (h.visited >= 1).all() and len(h) == 4000
    hit = h.triangle >= 0
    assert np.all(np.isfinite(h.t[hit])) and np.all(np.isinf(h.t[~hit]))
    tets, vis = batch.locate_points(m, o[:100].astype(np.float64))
    assert (tets >= 0).all()


def test_empty_and_errors(golden, K):
    m = golden_mesh(golden, "box4")
    z3 = np.zeros((0, 3), np.float32)
    out = K.cast_rays(m, z3, z3, np.zeros(0, np.int32))
    assert all(len(a) == 0 for a in out)
    with pytest.raises(IndexError):
        K.cast_rays(m, np.zeros((1, 3), np.float32), np.ones((1, 3), np.float32), np.array([m.n_tets], np.int32))
    with pytest.raises(ValueError):
        K.cast_rays(m, np.zeros((2, 3), np.float32), np.ones((1, 3), np.float32), np.array([0, 0], np.int32))
    from paper_2103_02309_b200 import batch

    bad = golden_mesh(golden, "box4")
    with pytest.raises(RuntimeError):  # batch layer raises on cycle-guard rays (batch.py:53-55)
        from paper_2103_02309_b200.ingestion import build_box_fixture
        from paper_2103_02309_b200.scenes import camera_rays
        from paper_2103_02309_b200.tetmesh import encode

        raw, soup = build_box_fixture(8, occluders=[(0, 4, (2, 2), (6, 6))])
        bad = encode(raw, "tet20", soup)
        o, d = camera_rays((4.0, 4.0, 0.5), (4.0, 4.0, 8.0), (0.0, 1.0, 0.0), 68.0, 1024, 1024)
        cam, _ = K.locate_points(bad, np.array([[4.0, 4.0, 0.5]]), np.array([0], np.int32))
        batch.cast_rays(bad, o, d, np.full(len(o), cam[0], np.int32))


def test_trace_torch_api(golden):
    import torch

    from paper_2103_02309_b200.scenes import interior_rays
    from paper_2103_02309_b200.trace import trace
    from oracle import pyoracle

    m = golden_mesh(golden, "model", "tet16")
    o, d, st = interior_rays(m, 20000, 11)
    dev = torch.device("cuda", 0)
    res = trace(m, torch.from_numpy(o).to(dev), torch.from_numpy(d).to(dev), torch.from_numpy(st).to(dev))
    torch.cuda.synchronize()
    exp = pyoracle.cast_rays_full(m, o, d, st)
    got = (res.status, res.cf, res.tet, res.visited, res.triangle, res.t, res.tet_back)
    for k, a, b in zip(NAMES7, got, exp):
        assert np.array_equal(a.cpu().numpy(), b), k


@pytest.fixture
def schedule():
    from paper_2103_02309_b200 import _lib

    saved = _lib.get_schedule()
    yield _lib.set_schedule
    _lib.set_schedule(*saved)


@pytest.mark.parametrize("mode,rounds", [("lane", 16), ("refill", 16), ("compact", 1), ("compact", 7),
                                          ("compact", 16), ("compact512", 32), ("binned", 16)])
@pytest.mark.parametrize("layout", LAYOUTS4)
def test_schedules_identical_results(golden, digests, K, O, schedule, mode, rounds, layout):
    """Every ray-to-lane schedule (one ray per lane, per-lane refill, block
    compaction at several round lengths) gives the reference's results bit
    for bit: golden fixtures, incoherent random rays, and a ragged batch."""
    schedule(mode, rounds)
    for name in ("pane4", "model"):
        base = golden_mesh(golden, name, "tet20" if layout == "tet80" else layout)
        o, d, st = _rays(base, name)
        out = K.cast_rays_full(base, o, d, st, layout=layout)
        ref_layout = "tet32" if layout == "tet80" else layout
        assert digest(*out[:4]) == digests[f"{name}/{ref_layout}/cast10k"]
        assert digest(*out[4:]) == digests[f"{name}/{ref_layout}/cast10k_epilogue"]
        # ragged: not a multiple of 32 / of the block, fewer rays than one block
        for n in (1, 33, 257, 4099):
            got = K.cast_rays_full(base, o[:n], d[:n], st[:n], layout=layout)
            for k, a, b in zip(NAMES7, got, out):
                assert np.array_equal(a, b[:n]), (k, n)


@pytest.mark.parametrize("mode", ("compact", "compact512", "refill", "binned"))
def test_schedules_cycle_guard(digests, K, O, schedule, mode):
    """Guard rays (status 2, visited = n_tets + 1) through the compacting
    scheduler, on the lattice camera and on the Brent fast-forward mesh."""
    from paper_2103_02309_b200.ingestion import build_box_fixture, build_kuhn_box
    from paper_2103_02309_b200.scenes import camera_rays
    from paper_2103_02309_b200.tetmesh import encode

    schedule(mode, 5)
    raw, soup = build_box_fixture(8, occluders=[(0, 4, (2, 2), (6, 6))])
    m = encode(raw, "tet20", soup)
    o, d = camera_rays((4.0, 4.0, 0.5), (4.0, 4.0, 8.0), (0.0, 1.0, 0.0), 68.0, 1024, 1024)
    st = np.full(len(o), digests["lattice8/cam_tet"], np.int32)
    out = K.cast_rays(m, o, d, st)
    assert digest(*out) == digests["lattice8/cast"]
    raw, soup = build_kuhn_box(16, [(0, 8, (4, 4), (12, 12))])
    m = encode(raw, "tet16", soup)
    o, d = camera_rays((8.0, 8.0, 0.5), (8.0, 8.0, 16.0), (0.0, 1.0, 0.0), 68.0, 512, 512)
    cam, _ = O.locate_points(m, np.array([[8.0, 8.0, 0.5]]), np.array([0], np.int32))
    st = np.full(len(o), cam[0], np.int32)
    got = K.cast_rays_full(m, o, d, st)
    exp = O.cast_rays_full(m, o, d, st)
    for k, a, b in zip(NAMES7, got, exp):
        assert np.array_equal(a, b), k


@pytest.mark.parametrize("schedule", ("lane", "refill", "compact", "compact512", "binned", "sampled"))
def test_trace_schedule_argument(golden, K, O, schedule):
    """trace(schedule=...) on device tensors (tb_cast_rays_sched) equals the
    oracle for an incoherent batch larger than one wave of blocks."""
    import torch

    from paper_2103_02309_b200.scenes import interior_rays
    from paper_2103_02309_b200.trace import trace

    m = golden_mesh(golden, "model", "tet16")
    o, d, st = interior_rays(m, 300_000, 11)
    dev = torch.device("cuda", 0)
    res = trace(m, *(torch.from_numpy(a).to(dev) for a in (o, d, st)), schedule=schedule)
    exp = O.cast_rays_full(m, o, d, st)
    got = (res.status, res.cf, res.tet, res.visited, res.triangle, res.t, res.tet_back)
    for k, a, b in zip(NAMES7, got, exp):
        assert np.array_equal(a.cpu().numpy(), b), k


@pytest.mark.parametrize("mode", ("auto", "compact", "binned"))
def test_host_path_coherent_and_incoherent(golden, K, O, schedule, mode):
    """tb_cast_rays_host on a camera batch (one start tet) and an incoherent
    batch: both equal the oracle, with pinned (zero-copy) and pageable
    buffers, under the default, the compacting and the binned schedule
    (the staged path bins each chunk)."""
    from paper_2103_02309_b200.scenes import camera_rays, interior_rays

    schedule(mode, 32)
    m = golden_mesh(golden, "model", "tet20")
    o, d, st = interior_rays(m, 100_000, 12)
    cam = np.asarray(o[0], np.float64)
    oc, dc = camera_rays(tuple(cam), (0.5, 0.5, 0.5), (0.0, 1.0, 0.0), 60.0, 320, 200)
    stc = np.full(len(oc), st[0], np.int32)
    import torch

    from paper_2103_02309_b200._lib import addr, check, lib
    from paper_2103_02309_b200.device import device_mesh

    dm = device_mesh(m)
    for oo, dd, ss in ((o, d, st), (oc, dc, stc)):
        exp = O.cast_rays_full(m, oo, dd, ss)
        got = K.cast_rays_full(m, oo, dd, ss)  # pageable: staged copies
        for k, a, b in zip(NAMES7, got, exp):
            assert np.array_equal(a, b), k
        # pinned: the zero-copy path (kernel reads rays / writes hits over PCIe)
        n = len(ss)
        pin = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in (oo, dd, ss)]
        outs = [torch.empty(n, dtype=dt).pin_memory() for dt in (torch.uint8, torch.int32, torch.int32, torch.int32,
                                                                  torch.int32, torch.float64, torch.int32)]
        check(lib.tb_cast_rays_host(dm.handle, n, *(addr(x) for x in pin), *(addr(x) for x in outs)),
              "tb_cast_rays_host")
        for k, a, b in zip(NAMES7, outs, exp):
            assert np.array_equal(a.numpy(), b), (k, "pinned")


@pytest.mark.parametrize("layout", ("tet20", "tet80"))
def test_sctp_host_zero_copy(golden, K, O, layout):
    """tb_sctp_cast_rays_host with mapped pinned buffers (the kernel reads
    rays / writes hits over PCIe) equals the C oracle's ScTP walk."""
    import torch

    from paper_2103_02309_b200._lib import addr, check, lib
    from paper_2103_02309_b200.device import device_mesh

    base = golden_mesh(golden, "model", "tet20")
    o, d, st = _rays(base, "model")
    exp = O.cast_rays_full(base, o, d, st, layout=layout, sctp=True)
    dm = device_mesh(base, layout=layout)
    n = len(st)
    pin = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in (o, d, st)]
    outs = [torch.empty(n, dtype=dt).pin_memory() for dt in (torch.uint8, torch.int32, torch.int32, torch.int32,
                                                              torch.int32, torch.float64, torch.int32)]
    check(lib.tb_sctp_cast_rays_host(dm.handle, n, *(addr(x) for x in pin), *(addr(x) for x in outs)),
          "tb_sctp_cast_rays_host")
    for k, a, b in zip(NAMES7, outs, exp):
        assert np.array_equal(a.numpy(), b), k


def test_upload_validation_and_corrupt_records(golden, K, O):
    """Every consistent mesh validates (no per-step clamp); a record mutated
    in place fails validation, keeps the clamp and still walks in bounds
    (no CUDA fault; the reference reads out of bounds there)."""
    import torch

    from paper_2103_02309_b200.device import DeviceMesh

    for layout in ("tet32", "tet20", "tet16"):
        m = golden_mesh(golden, "model", layout)
        assert DeviceMesh(m).validated
        assert not DeviceMesh(m, layout="tet80").validated  # inline points: nothing to validate
    m = golden_mesh(golden, "model", "tet20")
    o, d, st = _rays(m, "model")
    exp = O.cast_rays_full(m, o, d, st)
    bad = m.records.copy()
    words = bad.view("<u4").reshape(len(bad), -1)
    words[:, 0] ^= 0x00FFFFFF  # every vx word now points far outside the point array
    from dataclasses import replace

    mb = replace(m, records=bad)
    dmb = DeviceMesh(mb)
    assert not dmb.validated
    got = K.cast_rays_full(dmb, o, d, st)
    torch.cuda.synchronize()
    assert got[0].shape == exp[0].shape  # completed without a fault
    dmg = DeviceMesh(m)  # the good mesh still gives the oracle's results afterwards
    for k, a, b in zip(NAMES7, K.cast_rays_full(dmg, o, d, st), exp):
        assert np.array_equal(a, b), k


def test_concurrent_calls_from_host_threads(golden, K, O):
    """The reference renderer calls cast_rays concurrently on one mesh from
    its tile pool (render.py:538-541): 8 host threads x 6 calls each through
    the host entry points (pageable buffers -> per-thread staging streams)
    must give the oracle's results."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2103_02309_b200.device import device_mesh
    from paper_2103_02309_b200.scenes import interior_rays

    m = golden_mesh(golden, "model", "tet16")
    device_mesh(m)  # upload once up front, as render() does on first use
    batches = [interior_rays(m, 3000 + 257 * i, 40 + i) for i in range(48)]
    exp = [O.cast_rays_full(m, *b) for b in batches]

    def run(i):
        o, d, st = batches[i]
        got = K.cast_rays_full(m, o, d, st)
        return all(np.array_equal(a, b) for a, b in zip(got, exp[i]))

    with ThreadPoolExecutor(8) as ex:
        ok = list(ex.map(run, range(len(batches))))
    assert all(ok)


def test_host_path_staging_released_at_thread_exit(golden, K):
    """Each host thread's staging for the chunked host path (~44 MB of HBM)
    is released when the thread exits -- a renderer's churning tile pool must
    not leak device memory."""
    import threading

    import torch

    from paper_2103_02309_b200.device import device_mesh
    from paper_2103_02309_b200.scenes import interior_rays

    m = golden_mesh(golden, "model", "tet20")
    device_mesh(m)
    o, d, st = interior_rays(m, 5000, 9)
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(3):
        ts = [threading.Thread(target=K.cast_rays_full, args=(m, o, d, st)) for _ in range(8)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    # a joined thread's C++ thread_local destructors run as the OS thread
    # exits, which can trail join() slightly: allow them a moment
    import time

    for _ in range(50):
        torch.cuda.synchronize()
        free1, _ = torch.cuda.mem_get_info()
        if free0 - free1 < 64 << 20:
            break
        time.sleep(0.05)
    assert free0 - free1 < 64 << 20, (free0 - free1) / 2**20  # 24 threads x 44 MB would be ~1 GB


@pytest.mark.parametrize("scheme", ("none", "hilbert"))
def test_config2_full_frame_vs_reference(digests, K, scheme):
    """BASELINE config 2 at full size (blob GRID=55, 1.1 M tets, the whole
    1920x1080 frame) equals the reference's own digests: scene bytes, camera
    tet, all 2,073,600 rays' status/cf/tet/visited and the fp64 epilogue --
    for every layout (the layout-equivalence invariant), through
    both the host path and the device API."""
    import torch

    from conftest import mesh_digest
    from paper_2103_02309_b200.scenes import BLOB_CAMERA, blob_scene, camera_rays
    from paper_2103_02309_b200.tetmesh import relayout
    from paper_2103_02309_b200.trace import trace

    sc = blob_scene(55, layout="tet20", scheme=scheme, check=False)
    assert mesh_digest(sc.mesh) == digests[f"blob55/{scheme}/mesh"]
    o, d = camera_rays(BLOB_CAMERA["position"], BLOB_CAMERA["look_at"], BLOB_CAMERA["up"], BLOB_CAMERA["fov"],
                       1920, 1080)
    assert digest(o, d) == digests["blob55/rays"]
    cam, _ = K.locate_points(sc.mesh, np.array([BLOB_CAMERA["position"]]), np.array([sc.mesh.source_tet], np.int32))
    assert int(cam[0]) == digests[f"blob55/{scheme}/cam_tet"]
    st = np.full(len(o), cam[0], np.int32)
    for layout in ("tet20", "tet16", "tet32"):
        m = relayout(sc.mesh, layout)
        out = K.cast_rays_full(m, o, d, st)
        assert digest(*out[:4]) == digests[f"blob55/{scheme}/cast"], layout
        assert digest(*out[4:]) == digests[f"blob55/{scheme}/epilogue"], layout
    dev = torch.device("cuda", 0)
    res = trace(sc.mesh, *(torch.from_numpy(a).to(dev) for a in (o, d, st)))
    got = [x.cpu().numpy() for x in (res.status, res.cf, res.tet, res.visited)]
    assert digest(*got) == digests[f"blob55/{scheme}/cast"]


def test_binned_many_segments_matches_lane(golden):
    """A batch of ~9 binning segments (262144 rays each) with a ragged last
    segment and tile: the binned results must equal one ray per lane
    (itself pinned to the oracle above) for every ray."""
    import torch

    from paper_2103_02309_b200.scenes import interior_rays
    from paper_2103_02309_b200.trace import trace

    m = golden_mesh(golden, "model", "tet16")
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    n = l2 // 57 + 70_001
    o, d, st = interior_rays(m, n, 23)
    dev = torch.device("cuda", 0)
    g = [torch.from_numpy(a).to(dev) for a in (o, d, st)]
    a = trace(m, *g, schedule="lane")
    b = trace(m, *g, schedule="binned")
    torch.cuda.synchronize()
    for k in NAMES7:
        assert torch.equal(getattr(a, k), getattr(b, k)), k


@pytest.mark.parametrize("schedule", ("lane", "binned", "compact", "sampled"))
def test_schedules_without_epilogue(golden, O, schedule):
    """trace(epilogue=False): triangle / t / tet_back are not computed (NULL in
    the C call) under every schedule; status / cf / tet / visited still equal
    the oracle."""
    import torch

    from paper_2103_02309_b200.scenes import interior_rays
    from paper_2103_02309_b200.trace import trace

    m = golden_mesh(golden, "model", "tet20")
    o, d, st = interior_rays(m, 50_000, 31)
    dev = torch.device("cuda", 0)
    res = trace(m, *(torch.from_numpy(a).to(dev) for a in (o, d, st)), epilogue=False, schedule=schedule)
    exp = O.cast_rays_full(m, o, d, st)
    for k, a, b in zip(NAMES7[:4], (res.status, res.cf, res.tet, res.visited), exp[:4]):
        assert np.array_equal(a.cpu().numpy(), b), k


def test_cast_epilogue_equals_fused_epilogue(golden):
    """tb_cast_epilogue (the lean multi-GPU assembly's root pass) derives
    triangle / t / tet_back from stored cf / tet bit for bit like the fused
    epilogue, for hits and misses, in every host-visible layout."""
    import torch

    from paper_2103_02309_b200._lib import addr, check, lib
    from paper_2103_02309_b200.device import device_mesh
    from paper_2103_02309_b200.scenes import interior_rays
    from paper_2103_02309_b200.trace import empty_result, trace

    dev = torch.device("cuda", 0)
    for layout in ("tet32", "tet20", "tet16"):
        m = golden_mesh(golden, "model", layout)
        o, d, st = interior_rays(m, 30_000, 44)
        g = [torch.from_numpy(a).to(dev) for a in (o, d, st)]
        full = trace(m, *g)
        lean = trace(m, *g, epilogue=False)
        out = empty_result(len(st), dev)
        check(lib.tb_cast_epilogue(device_mesh(m).handle, len(st), addr(g[0]), addr(g[1]), addr(lean.cf),
                                   addr(lean.tet), addr(out.triangle), addr(out.t), addr(out.tet_back),
                                   torch.cuda.current_stream(dev).cuda_stream), "tb_cast_epilogue")
        torch.cuda.synchronize()
        assert int((full.status == 1).sum()) > 0 and int((full.status == 0).sum()) >= 0
        for k in ("triangle", "t", "tet_back"):
            assert torch.equal(getattr(out, k), getattr(full, k)), (layout, k)


@pytest.mark.parametrize("name", FIXTURES)
def test_fastcall_equals_ctypes_path(golden, digests, K, name):
    """kernels.cast_rays' C fast path (csrc/fastcall.c, the per-tile call the
    reference renderer makes) and the general ctypes path return identical
    arrays, equal to the reference's digest; tile-sized calls too."""
    assert K._fastcall is not None
    m = golden_mesh(golden, name, "tet20")
    o, d, st = _rays(m, name)
    fast = K.cast_rays(m, o, d, st)
    plain = K._cast_plain(m, o, d, st)[:4]
    assert digest(*fast) == digests[f"{name}/tet20/cast10k"]
    for a, b in zip(fast, plain):
        assert a.dtype == b.dtype and np.array_equal(a, b)
    for a0 in range(0, 2048, 256):
        tile = K.cast_rays(m, o[a0:a0 + 256], d[a0:a0 + 256], st[a0:a0 + 256])
        for a, b in zip(tile, plain):
            assert np.array_equal(a, b[a0:a0 + 256])


def test_block_order_launch_equals_plain_trace(golden, K):
    """trace(block_order=...) launches whole blocks in a caller-chosen order
    (tb_cast_rays_ordered); results stay in place and equal the plain launch
    bit for bit -- for longest_first of the batch's own walk lengths, a random
    permutation and a ragged last block.  Bad orders fail loudly."""
    import torch

    from paper_2103_02309_b200._lib import TetB200Error
    from paper_2103_02309_b200.trace import block_size, longest_first, trace

    dev = torch.device("cuda", 0)
    m = golden_mesh(golden, "model", "tet20")
    o, d, st = _rays(m, "model", n=10000 + 37)
    g = [torch.from_numpy(a).to(dev) for a in (o, d, st)]
    ref = trace(m, *g)
    nb = (len(st) + block_size() - 1) // block_size()
    lf = longest_first(ref.visited)  # tb_block_order: a permutation, block maxima non-increasing
    assert sorted(lf.cpu().tolist()) == list(range(nb))
    v = torch.zeros(nb * block_size(), dtype=torch.int32, device=dev)
    v[:len(st)] = ref.visited
    keys = v.view(nb, -1).max(dim=1).values[lf.long()].cpu().numpy()

    def bucket(x):  # tb_block_order's classes: exact below 16, then 4 per power of two
        if x < 16:
            return int(x)
        e = int(x).bit_length() - 1
        return min(16 + (e - 4) * 4 + ((int(x) >> (e - 2)) & 3), 63)

    classes = [bucket(k) for k in keys]
    assert all(a >= b for a, b in zip(classes, classes[1:]))  # longest class first
    gen = torch.Generator(device="cpu").manual_seed(5)
    for order in (longest_first(ref.visited), torch.randperm(nb, generator=gen).to(torch.int32).to(dev)):
        got = trace(m, *g, block_order=order)
        for k in NAMES7:
            assert torch.equal(getattr(got, k), getattr(ref, k)), k
    with pytest.raises(TetB200Error, match="block_order"):
        trace(m, *g, block_order=torch.arange(nb - 1, dtype=torch.int32, device=dev))
    with pytest.raises(ValueError):
        trace(m, *g, block_order=torch.arange(nb, dtype=torch.int64, device=dev))
    with pytest.raises(ValueError):
        trace(m, *g, block_order=torch.arange(nb, dtype=torch.int32, device=dev), sctp=True)


@pytest.mark.parametrize("layout", LAYOUTS4)
def test_sampled_schedule_matches_lane(golden, digests, K, layout):
    """schedule="sampled" (a capped one-ray-per-block pre-pass orders the
    blocks longest first, then the full walk in that order) equals one ray per
    lane for every ray: golden fixtures at full digest, ragged sizes (1 ray,
    less than a block, a ragged last block), every layout, and the lattice
    camera whose rays trip the cycle guard."""
    import torch

    from paper_2103_02309_b200.scenes import camera_rays
    from paper_2103_02309_b200.tetmesh import encode
    from paper_2103_02309_b200.trace import trace

    dev = torch.device("cuda", 0)
    for name in ("pane4", "model"):
        base = golden_mesh(golden, name, "tet20" if layout == "tet80" else layout)
        o, d, st = _rays(base, name)
        g = [torch.from_numpy(a).to(dev) for a in (o, d, st)]
        got = trace(base, *g, schedule="sampled", layout=layout)
        ref_layout = "tet32" if layout == "tet80" else layout
        assert digest(*(getattr(got, k).cpu().numpy() for k in ("status", "cf", "tet", "visited"))) == \
            digests[f"{name}/{ref_layout}/cast10k"]
        for n in (1, 33, 129, 4099):
            a = trace(base, *(x[:n] for x in g), schedule="sampled", layout=layout)
            b = trace(base, *(x[:n] for x in g), schedule="lane", layout=layout)
            for k in NAMES7:
                assert torch.equal(getattr(a, k), getattr(b, k)), (name, n, k)
    if layout == "tet20":  # the lattice camera: exact ties, cycle-guard rays (status 2)
        from paper_2103_02309_b200.ingestion import build_box_fixture

        raw, soup = build_box_fixture(8, occluders=[(0, 4, (2, 2), (6, 6))])
        m = encode(raw, "tet20", soup)
        o, d = camera_rays((4.0, 4.0, 0.5), (4.0, 4.0, 8.0), (0.0, 1.0, 0.0), 68.0, 1024, 1024)
        st = np.full(len(o), digests["lattice8/cam_tet"], np.int32)
        g = [torch.from_numpy(a).to(dev) for a in (o, d, st)]
        from paper_2103_02309_b200._lib import lib

        # 1 M rays = 8192 blocks: a split launch (head in launch order, the
        # probed tail longest first on the side stream), also with a ragged tail
        assert lib.tb_sampled_head_blocks(0, len(o)) > 0
        a = trace(m, *g, schedule="sampled")
        assert digest(*(getattr(a, k).cpu().numpy() for k in ("status", "cf", "tet", "visited"))) == \
            digests["lattice8/cast"]
        n = len(o) - 77
        a = trace(m, *(x[:n] for x in g), schedule="sampled")
        b = trace(m, *(x[:n] for x in g), schedule="lane")
        for k in NAMES7:
            assert torch.equal(getattr(a, k), getattr(b, k)), k


def test_sampled_split_rule():
    """tb_sampled_head_blocks / tb_auto_schedule: no split below 3 waves of
    blocks, a head of >= 3 waves and a tail of <= 16 waves beyond; auto picks
    the sampled schedule for 6-48 waves only."""
    import torch

    from paper_2103_02309_b200._lib import lib

    wave = torch.cuda.get_device_properties(0).multi_processor_count * 10
    blk = lib.tb_cast_block_size()
    for waves in (0.5, 2, 3, 5.5, 11, 44, 146):
        n = int(waves * wave * blk)
        nb = -(-n // blk)
        head = lib.tb_sampled_head_blocks(0, n)
        if nb <= 3 * wave:
            assert head == 0, waves
        else:
            assert head >= 3 * wave and nb - head <= 16 * wave and nb - head >= 1, (waves, head)
        assert lib.tb_auto_schedule(0, n) == (7 if 6 * wave <= nb <= 48 * wave else 1), waves
