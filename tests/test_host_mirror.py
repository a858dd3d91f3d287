"""Host-side mesh mirror vs the reference: builders, encoding, layouts,
Hilbert reordering and validation produce byte-identical arrays
(digests from tests/golden/make_golden.py).  Modelled on the reference's
test_tetmesh.py / test_hilbert.py / test_reorder.py / test_ingestion.py.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import FIXTURES, GOLDEN as ROOT_GOLDEN, PANE_OCC, REGION_OCC, digest, golden_mesh, mesh_digest

from paper_2103_02309_b200 import hilbert, scenes
from paper_2103_02309_b200.ingestion import build_box_fixture
from paper_2103_02309_b200.tetmesh import (
    LAYOUT_BYTES,
    LAYOUTS,
    BOUNDARY_REF,
    CONSTRAINED_BIT,
    compute_xor_sum,
    decode_ref,
    encode,
    face_ref,
    recover_fourth_vertex,
    relayout,
    reorder,
    validate,
)

BOX_ARGS = {
    "box1": dict(n=1),
    "box4": dict(n=4),
    "pane4": dict(n=4, occluders=PANE_OCC),
    "region4": dict(n=4, occluders=REGION_OCC),
    "open_box4": dict(n=4, walls="open"),
}


def _build(name):
    if name == "model":
        return scenes.blob_scene(8, layout="tet20").mesh
    kw = dict(BOX_ARGS[name])
    raw, soup = build_box_fixture(kw.pop("n"), **kw)
    return encode(raw, "tet20", soup)


@pytest.mark.parametrize("name", FIXTURES)
def test_builders_match_reference(digests, name):
    m = _build(name)
    for layout in LAYOUTS:
        assert mesh_digest(relayout(m, layout)) == digests[f"{name}/{layout}/mesh"], layout


@pytest.mark.parametrize("name", FIXTURES)
@pytest.mark.parametrize("scheme", ("hilbert", "hilbert_regions", "shuffle"))
def test_reorder_matches_reference(digests, name, scheme):
    m = _build(name)
    r = reorder(m, scheme)
    assert mesh_digest(r) == digests[f"{name}/reorder/{scheme}"]
    assert validate(r) == []


def test_golden_meshes_validate(meshes):
    for name, m in meshes.items():
        assert validate(m) == [], name


def test_record_sizes(meshes):
    for layout in LAYOUTS:
        m = relayout(meshes["model"], layout)
        assert m.records.dtype.itemsize == LAYOUT_BYTES[layout] == {"tet32": 32, "tet20": 20, "tet16": 16}[layout]
        assert m.records_u32().shape == (m.n_tets, LAYOUT_BYTES[layout] // 4)


def test_ref_helpers():
    assert face_ref(5) == CONSTRAINED_BIT | 5
    assert decode_ref(BOUNDARY_REF) == -1 and decode_ref(face_ref(3)) == -1 and decode_ref(17) == 17
    assert compute_xor_sum(1, 2, 4, 8) == 15
    assert recover_fourth_vertex(1, 2, 4, 15) == 8


@pytest.mark.parametrize("bad", ("vx", "link", "order"))
def test_validate_detects_faults(meshes, bad):
    m = relayout(meshes["region4"], "tet16" if bad == "link" else "tet20")
    rec = m.records.copy()
    if bad == "vx":
        rec["vx"][7] ^= 1
    elif bad == "link":
        rec["nx1"][3] ^= 4
    else:
        rec["n0"][5], rec["n1"][5] = rec["n1"][5], rec["n0"][5]
    from dataclasses import replace

    probs = validate(replace(m, records=rec))
    assert probs, bad


def test_hilbert_bijection_and_adjacency():
    order = 3
    g = np.stack(np.meshgrid(*[np.arange(8)] * 3, indexing="ij"), -1).reshape(-1, 3)
    k = hilbert.hilbert_keys(g, order)
    assert np.array_equal(np.sort(k), np.arange(512, dtype=np.uint64))
    cells = g[np.argsort(k)]
    assert np.all(np.abs(np.diff(cells, axis=0)).sum(axis=1) == 1)
    assert hilbert.hilbert_index((0, 0, 0), 4) == 0


def test_camera_rays_match_reference(digests):
    c = scenes.BLOB_CAMERA
    o, d = scenes.camera_rays(c["position"], c["look_at"], c["up"], c["fov"], 256, 256)
    assert digest(o, d) == digests["blob12/rays"]


@pytest.mark.parametrize("scheme", ("none", "hilbert"))
def test_blob12_scene_matches_reference(digests, scheme):
    sc = scenes.blob_scene(12, scheme=scheme)
    assert mesh_digest(sc.mesh) == digests[f"blob12/{scheme}/mesh"]


@pytest.mark.slow
def test_blob55_config2_scene_matches_reference(digests):
    """The BASELINE config-2 scene (GRID=55, 1.1 M tets) is byte-identical to
    the reference's gen_model_mesh -> parse_tetgen -> encode -> reorder."""
    if "blob55/sizes" not in digests:
        pytest.skip("golden digests generated without --big")
    sc = scenes.blob_scene(55, scheme="none", check=False)
    assert mesh_digest(sc.mesh) == digests["blob55/none/mesh"]
    assert mesh_digest(reorder(sc.mesh, "hilbert")) == digests["blob55/hilbert/mesh"]
    assert sc.mesh.n_tets == digests["blob55/sizes"]["tets"]


def test_interior_rays_match_reference(meshes, digests):
    from conftest import RAY_SEEDS

    for name, m in meshes.items():
        o, d, st = scenes.interior_rays(m, 10000, RAY_SEEDS[name])
        assert digest(o, d, st) == digests[f"{name}/rays"]


def test_golden_mesh_roundtrip(golden):
    m = golden_mesh(golden, "pane4", "tet16")
    assert m.records_u32().shape == (m.n_tets, 4)


def test_npz_interop_with_reference_cli(tmp_path, golden):
    """load_compact reads a file written by the reference's cli.save_compact
    (cli.py:249-265), and save/load round-trips byte-identically."""
    from paper_2103_02309_b200.io import load_compact, save_compact

    ref = load_compact(ROOT_GOLDEN / "pane4_tet16_ref.npz")
    assert ref.layout == "tet16"
    assert mesh_digest(ref) == mesh_digest(relayout(golden_mesh(golden, "pane4"), "tet16"))
    p = tmp_path / "m.npz"
    save_compact(ref, p)
    assert mesh_digest(load_compact(p)) == mesh_digest(ref)


def test_hull_faces_order(meshes):
    from paper_2103_02309_b200.tetmesh import hull_faces

    h = hull_faces(meshes["box4"])
    assert len(h) == 6 * 2 * 16  # every wall face of the n=4 box
    assert np.all(np.diff(h[:, 0] * 4 + h[:, 1]) > 0)  # tet-major, slot-minor
    assert len(hull_faces(meshes["open_box4"])) == len(h)


def _consume_sink(sink, visited):
    """The reference's sink consumer, restated (batch.py:98-114)."""
    offsets = np.zeros(len(visited) + 1, dtype=np.int64)
    np.cumsum(visited, out=offsets[1:])
    visits = np.empty(int(offsets[-1]), dtype=np.int32)
    pos = offsets[:-1].copy()
    for rays, tets in sink:
        if len(rays) and rays[0] == rays[-1] and (rays == rays[0]).all():
            i = int(rays[0])
            visits[pos[i]:pos[i] + len(tets)] = tets
            pos[i] += len(tets)
        else:
            visits[pos[rays]] = tets
            pos[rays] += 1
    return visits, offsets


def test_visits_sink_emission_is_linear_and_consumable():
    """kernels.emit_visits: short rays as step wavefronts, long
    and cycle-guard rays as one chunk each -- the reference consumer rebuilds
    the exact CSR, and the chunk count stays O(32 + long rays) even with a
    ray of a million visits."""
    from paper_2103_02309_b200.kernels import emit_visits

    rng = np.random.default_rng(7)
    visited = rng.integers(1, 60, 5000).astype(np.int32)
    visited[17] = 1_000_001  # a cycle-guard ray on a 1 M-tet mesh
    visited[4000] = 1
    offsets = np.zeros(len(visited) + 1, np.int64)
    np.cumsum(visited, out=offsets[1:])
    seq = rng.integers(0, 1 << 30, int(offsets[-1])).astype(np.int32)
    sink: list = []
    emit_visits(sink, visited, seq, offsets)
    assert len(sink) <= 32 + int((visited > 32).sum())
    got, off = _consume_sink(sink, visited)
    assert np.array_equal(off, offsets) and np.array_equal(got, seq)
