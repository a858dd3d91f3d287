"""GPU vs the reference's own compiled kernels (oracle/_ref, built from
_kernels.pyx) on tie-heavy and random inputs: lattice-aligned origins and
axis/diagonal directions on Kuhn boxes (exact zeros in the basis, exact
ties in Algorithm 1 and the init face pick), random occluder boxes, every
layout.  Falls back to the C oracle when oracle/_ref is absent."""

from __future__ import annotations

import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def REF():
    from oracle import pyoracle

    return pyoracle.ref_kernels() or pyoracle


def _lattice_rays(n_box, rng, count):
    """Origins on lattice points / edge midpoints / face centres strictly
    inside the box, directions along axes, face and space diagonals."""
    dirs = [np.array(v, dtype=np.float32) for v in itertools.product((-1, 0, 1), repeat=3) if any(v)]
    dirs += [np.array(v, dtype=np.float32) for v in ((1, 2, 0), (2, -1, 1), (0, 1, 3), (-1, -1, 2))]
    o, d = [], []
    for _ in range(count):
        base = rng.integers(1, n_box, 3).astype(np.float32)
        off = rng.choice([0.0, 0.5], size=3).astype(np.float32)
        o.append(np.minimum(base + off - 0.5 * (base + off >= n_box), n_box - 0.5))
        d.append(dirs[rng.integers(len(dirs))])
    return np.array(o, np.float32), np.array(d, np.float32)


@pytest.mark.parametrize("layout", ("tet32", "tet20", "tet16"))
def test_lattice_ties_vs_reference(REF, layout):
    from paper_2103_02309_b200 import kernels as K
    from paper_2103_02309_b200.ingestion import build_kuhn_box
    from paper_2103_02309_b200.tetmesh import encode

    rng = np.random.default_rng(7)
    raw, soup = build_kuhn_box(6, [(0, 3, (1, 1), (5, 5)), (2, 2, (0, 2), (6, 4))])
    m = encode(raw, layout, soup)
    o, d = _lattice_rays(6, rng, 6000)
    st, _ = K.locate_points(m, o.astype(np.float64), np.full(len(o), m.source_tet, np.int32))
    keep = st >= 0
    o, d, st = o[keep], d[keep], st[keep]
    got = K.cast_rays(m, o, d, st)
    exp = REF.cast_rays(m, o, d, st)
    for a, b in zip(got, exp):
        assert np.array_equal(a, b)
    # the lattice makes ties: make sure the set actually exercises them
    assert len(o) > 3000


@pytest.mark.parametrize("seed", range(6))
def test_random_occluder_boxes_vs_reference(REF, seed):
    from paper_2103_02309_b200 import kernels as K
    from paper_2103_02309_b200.ingestion import build_kuhn_box
    from paper_2103_02309_b200.scenes import interior_rays
    from paper_2103_02309_b200.tetmesh import encode, reorder

    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(3, 9))
    occ = []
    for _ in range(int(rng.integers(0, 4))):
        axis = int(rng.integers(0, 3))
        k = int(rng.integers(1, n))
        u0, v0 = (int(x) for x in rng.integers(0, n - 1, 2))
        u1, v1 = int(rng.integers(u0 + 1, n + 1)), int(rng.integers(v0 + 1, n + 1))
        if all((a != axis or kk != k) for a, kk, *_ in occ):  # no overlapping occluders
            occ.append((axis, k, (u0, v0), (u1, v1)))
    walls = "open" if seed % 3 == 2 else "constrained"
    raw, soup = build_kuhn_box(n, occ, walls=walls, scale=(1.0, 1.0 + 0.37 * seed, 1.0))
    layout = ("tet32", "tet20", "tet16")[seed % 3]
    m = reorder(encode(raw, layout, soup), ("none", "hilbert", "shuffle")[seed % 3])
    o, d, st = interior_rays(m, 8000, seed)
    got = K.cast_rays_full(m, o, d, st)
    exp = REF.cast_rays(m, o, d, st)
    for a, b in zip(got[:4], exp):
        assert np.array_equal(a, b)


def test_degenerate_directions_vs_c_oracle():
    """Zero and non-finite directions: the reference reads SLOT_A[-1] (UB);
    both the device and the C restatement pin slot 0 and must agree."""
    from oracle import pyoracle
    from paper_2103_02309_b200 import kernels as K
    from paper_2103_02309_b200.ingestion import build_box_fixture
    from paper_2103_02309_b200.tetmesh import encode

    raw, soup = build_box_fixture(4, occluders=[(0, 2, (1, 1), (3, 3))])
    m = encode(raw, "tet20", soup)
    o = np.full((6, 3), 1.3, np.float32)
    d = np.array([[0, 0, 0], [np.nan, 1, 0], [np.inf, 0, 0], [0, 0, 1e-30], [1e30, 1, 1], [0, -0.0, 1]],
                 np.float32)
    st = np.full(6, int(K.locate_points(m, o[:1].astype(np.float64), np.array([0], np.int32))[0][0]), np.int32)
    got = K.cast_rays(m, o, d, st)
    exp = pyoracle.cast_rays(m, o, d, st)
    for a, b in zip(got, exp):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("schedule", ("lane", "binned"))
def test_degenerate_directions_device_schedules(schedule):
    """The same degenerate rays, mixed into a batch spanning several binning
    tiles, through trace(schedule=...): the binned schedule's direction cell
    of a zero / NaN / inf direction is arbitrary but its results must still
    equal the C restatement ray for ray."""
    import torch

    from oracle import pyoracle
    from paper_2103_02309_b200 import kernels as K
    from paper_2103_02309_b200.ingestion import build_box_fixture
    from paper_2103_02309_b200.scenes import interior_rays
    from paper_2103_02309_b200.tetmesh import encode
    from paper_2103_02309_b200.trace import trace

    raw, soup = build_box_fixture(4, occluders=[(0, 2, (1, 1), (3, 3))])
    m = encode(raw, "tet16", soup)
    o, d, st = interior_rays(m, 9000, 5)
    bad = np.array([[0, 0, 0], [np.nan, 1, 0], [np.inf, 0, 0], [0, 0, 1e-30], [1e30, 1, 1], [0, -0.0, 1],
                    [-np.inf, np.nan, 2]], np.float32)
    d[::1301][: len(bad)] = bad[: len(d[::1301])]
    dev = torch.device("cuda", 0)
    res = trace(m, *(torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (o, d, st)), schedule=schedule)
    exp = pyoracle.cast_rays_full(m, o, d, st)
    got = (res.status, res.cf, res.tet, res.visited, res.triangle, res.t, res.tet_back)
    for a, b in zip(got, exp):
        assert np.array_equal(a.cpu().numpy(), b, equal_nan=True)


def test_large_batch_ragged_sizes(REF):
    """Sizes that are not multiples of the block / warp / chunk sizes."""
    from paper_2103_02309_b200 import kernels as K
    from paper_2103_02309_b200.scenes import blob_scene, interior_rays

    m = blob_scene(8, layout="tet16").mesh
    for n in (1, 31, 33, 127, 129, 262_145):
        o, d, st = interior_rays(m, n, n)
        got = K.cast_rays(m, o, d, st)
        exp = REF.cast_rays(m, o, d, st)
        for a, b in zip(got, exp):
            assert np.array_equal(a, b), n


@pytest.mark.parametrize("layout", ("tet20", "tet80"))
def test_sctp_degenerate_and_extreme_rays_vs_c_oracle(layout):
    """The edge-cached ScTP step decides faces from min / max of cached
    values and must fall back to the exact per-face order whenever a value
    is NaN: zero / NaN / inf / tiny / huge directions and far origins give
    the C oracle's ScTP results bit for bit."""
    from oracle import pyoracle
    from paper_2103_02309_b200 import kernels as K
    from paper_2103_02309_b200.ingestion import build_box_fixture
    from paper_2103_02309_b200.scenes import interior_rays
    from paper_2103_02309_b200.tetmesh import encode

    raw, soup = build_box_fixture(4, occluders=[(0, 2, (1, 1), (3, 3))])
    m = encode(raw, "tet20", soup)
    o = np.full((8, 3), 1.3, np.float32)
    d = np.array([[0, 0, 0], [np.nan, 1, 0], [np.inf, 0, 0], [0, 0, 1e-30], [1e30, 1, 1], [0, -0.0, 1],
                  [1e-38, 1e-38, 1e-38], [-np.inf, np.inf, 1]], np.float32)
    st = np.full(len(o), int(K.locate_points(m, o[:1].astype(np.float64), np.array([0], np.int32))[0][0]), np.int32)
    ro, rd, rst = interior_rays(m, 4000, 77)
    rd[::7] *= np.float32(1e-20)  # tiny directions: products underflow toward zero / subnormals
    oo, dd, ss = (np.concatenate(a) for a in ((o, ro), (d, rd), (st, rst)))
    got = K.cast_rays_full(m, oo, dd, ss, layout=layout, sctp=True)
    exp = pyoracle.cast_rays_full(m, oo, dd, ss, layout=layout, sctp=True)
    for k, a, b in zip(("status", "cf", "tet", "visited", "triangle", "t", "tet_back"), got, exp):
        assert np.array_equal(a, b, equal_nan=(k == "t")), k


def test_cached_mesh_arrays_are_frozen_until_invalidate():
    """The device cache cannot go stale silently: while a mesh is cached, its
    mirrored arrays are read-only (the reference re-reads them every call,
    _kernels.pyx:276-282); invalidate() thaws them and the next call uploads
    the mutated mesh."""
    from paper_2103_02309_b200 import device, kernels as K
    from paper_2103_02309_b200.ingestion import build_box_fixture
    from paper_2103_02309_b200.scenes import interior_rays
    from paper_2103_02309_b200.tetmesh import encode
    from oracle import pyoracle

    raw, soup = build_box_fixture(4, occluders=[(0, 2, (1, 1), (3, 3))])
    mesh = encode(raw, "tet20", soup)
    o, d, st = interior_rays(mesh, 2000, 5)
    first = K.cast_rays(mesh, o, d, st)
    assert not mesh.points.flags.writeable and not mesh.side_neighbors.flags.writeable
    with pytest.raises(ValueError):
        mesh.points[0, 0] = 0.5
    device.invalidate(mesh)
    assert mesh.points.flags.writeable and mesh.records.flags.writeable
    mesh.points[:] = mesh.points * np.float32(2.0)  # scale the scene in place
    o2 = o * np.float32(2.0)
    got = K.cast_rays(mesh, o2, d, st)
    exp = pyoracle.cast_rays(mesh, o2, d, st)
    for a, b in zip(got, exp):
        assert np.array_equal(a, b)
    assert first[3].shape == got[3].shape
    # replacing an array (not in place) re-uploads without invalidate and thaws the old one
    old = mesh.points
    mesh.points = mesh.points.copy()
    K.cast_rays(mesh, o2, d, st)
    assert old.flags.writeable and not mesh.points.flags.writeable
    device.invalidate(mesh)


def test_small_batch_protocol_calls_from_threads(REF):
    """Renderer granularity: 256-ray calls of the protocol module from 16
    host threads (render.py:538-541) give the reference's results."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2103_02309_b200 import kernels as K
    from paper_2103_02309_b200.ingestion import build_box_fixture
    from paper_2103_02309_b200.scenes import interior_rays
    from paper_2103_02309_b200.tetmesh import encode

    raw, soup = build_box_fixture(6, occluders=[(0, 3, (1, 1), (5, 5))])
    mesh = encode(raw, "tet16", soup)
    o, d, st = interior_rays(mesh, 256 * 64, 9)
    exp = REF.cast_rays(mesh, o, d, st)

    def one(i):
        sl = slice(256 * i, 256 * (i + 1))
        return K.cast_rays(mesh, o[sl], d[sl], st[sl])

    with ThreadPoolExecutor(max_workers=16) as pool:
        parts = list(pool.map(one, range(64)))
    for k in range(4):
        assert np.array_equal(np.concatenate([p[k] for p in parts]), exp[k])
    from paper_2103_02309_b200 import device

    device.invalidate(mesh)
