"""Generate the golden fixtures in tests/golden/ from the reference itself.

Run in the build container (needs /root/reference; the GPU box never does):

    python tests/golden/make_golden.py          # small fixtures (seconds)
    python tests/golden/make_golden.py --big    # + config-2 blob GRID=55 digests (minutes)

Everything here is produced by the UNMODIFIED reference package imported
from /root/reference/pkg/src -- its builders (ingestion, tetmesh), its batch
layer and epilogue (batch.cast_rays), its camera (render.camera_rays), its
ScTP predicate (traversal.sctp_exit_face) and its compiled kernels
(_kernels.pyx, built by oracle/build_ref.sh into oracle/_ref/).  Outputs:
  golden_small.npz  fixture meshes + reference outputs (arrays)
  golden_digests.json  sha256 digests + sums for the larger cases
"""

from __future__ import annotations

import argparse
import hashlib
import importlib.util
import json
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
REF = Path(os.environ.get("TETRAY_REF", "/root/reference/pkg"))
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REPO))

from tetray import batch, traversal  # noqa: E402
from tetray.geometry import Ray, Vec3  # noqa: E402
from tetray.ingestion import associate_constrained_faces, build_box_fixture, load_obj, parse_tetgen  # noqa: E402
from tetray.render import RenderConfig, camera_rays  # noqa: E402
from tetray.tetmesh import encode, relayout, reorder  # noqa: E402

from oracle.pyoracle import ref_kernels  # noqa: E402

OUT = Path(__file__).resolve().parent
PANE_OCC = [(0, 2, (1, 1), (3, 3))]
REGION_OCC = [(axis, k, (1, 1), (3, 3)) for axis in range(3) for k in (1, 3)]


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]


def interior_rays(mesh, n, seed):  # tests/conftest.py:61-73 of the reference
    rng = np.random.default_rng(seed)
    ti = rng.integers(0, mesh.n_tets, n).astype(np.int32)
    bary = rng.dirichlet(np.ones(4) * 4.0, n)
    pts = mesh.points.astype(np.float64)
    o = np.einsum("ij,ijk->ik", bary, pts[mesh.side_verts[ti]])
    d = rng.normal(size=(n, 3))
    return o.astype(np.float32), d.astype(np.float32), ti


def model_mesh():
    data = REF / "data" / "model"
    raw = parse_tetgen(data / "blob.1")
    soup = load_obj(data / "blob.obj")
    faces = np.array([cf.vertex_ids for cf in raw.constrained_faces], dtype=np.int64)
    tri_ids = associate_constrained_faces(raw.points, faces, soup, tolerance=1e-9)
    for cf, tid in zip(raw.constrained_faces, tri_ids):
        cf.triangle_id = int(tid)
    return encode(raw, "tet20", soup)


def mesh_arrays(prefix, m, out):
    out[f"{prefix}/points"] = m.points
    out[f"{prefix}/side_verts"] = m.side_verts
    out[f"{prefix}/side_neighbors"] = m.side_neighbors
    out[f"{prefix}/cf_triangle"] = m.cf_triangle
    out[f"{prefix}/cf_tets"] = m.cf_tets
    out[f"{prefix}/cf_verts"] = m.cf_verts
    out[f"{prefix}/soup_vertices"] = m.soup.vertices
    out[f"{prefix}/soup_triangles"] = m.soup.triangles
    out[f"{prefix}/soup_material_ids"] = m.soup.material_ids
    out[f"{prefix}/source_tet"] = np.array(m.source_tet)


def mesh_digest(m) -> str:
    return digest(m.points, m.side_verts, m.side_neighbors, m.cf_triangle, m.cf_tets, m.cf_verts, m.records_u32(),
                  m.soup.vertices, m.soup.triangles, np.array([m.source_tet]))


def hits_arrays(h):
    return [h.status, h.cf, h.tet_front, h.visited, h.triangle, h.t, h.tet_back]


def load_gen_model_mesh():
    spec = importlib.util.spec_from_file_location("gen_model_mesh", REF / "tools" / "gen_model_mesh.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def reference_blob(grid: int):
    """The reference pipeline for a blob scene: gen_model_mesh at GRID ->
    TetGen/OBJ files -> parse_tetgen / load_obj / associate -> encode."""
    gen = load_gen_model_mesh()
    gen.GRID = grid
    with tempfile.TemporaryDirectory() as tmp:
        gen.ROOT = Path(tmp)
        import contextlib
        import io

        with contextlib.redirect_stdout(io.StringIO()):
            gen.main()
        data = Path(tmp) / "data" / "model"
        raw = parse_tetgen(data / "blob.1")
        soup = load_obj(data / "blob.obj")
    faces = np.array([cf.vertex_ids for cf in raw.constrained_faces], dtype=np.int64)
    tri_ids = associate_constrained_faces(raw.points, faces, soup, tolerance=1e-9)
    for cf, tid in zip(raw.constrained_faces, tri_ids):
        cf.triangle_id = int(tid)
    return raw, soup


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also the GRID=55 config-2 scene (minutes)")
    args = ap.parse_args()
    K = ref_kernels()
    if K is None:
        raise SystemExit("oracle/_ref missing: run oracle/build_ref.sh first")
    arrays: dict = {}
    dig: dict = {}
    digest_path = OUT / "golden_digests.json"
    if digest_path.exists():
        dig = json.loads(digest_path.read_text())

    fixtures = {
        "box1": _fx(1),
        "box4": _fx(4),
        "pane4": _fx(4, occluders=PANE_OCC),
        "region4": _fx(4, occluders=REGION_OCC),
        "open_box4": _fx(4, walls="open"),
        "model": model_mesh(),
    }
    seeds = {"box4": 100, "pane4": 101, "region4": 102, "model": 103, "open_box4": 104, "box1": 105}
    for name, m in fixtures.items():
        mesh_arrays(name, m, arrays)
        o, d, st = interior_rays(m, 10000, seeds[name])
        dig[f"{name}/rays"] = digest(o, d, st)
        for layout in ("tet32", "tet20", "tet16"):
            ml = relayout(m, layout)
            dig[f"{name}/{layout}/mesh"] = mesh_digest(ml)
            h = batch.cast_rays(ml, o, d, st, kernels=K)
            outs = hits_arrays(h)
            dig[f"{name}/{layout}/cast10k"] = digest(*outs[:4])
            dig[f"{name}/{layout}/cast10k_epilogue"] = digest(*outs[4:])
            if layout == "tet20":
                for k, a in zip(("status", "cf", "tet", "visited", "triangle", "t", "tet_back"), outs):
                    arrays[f"{name}/cast/{k}"] = a[:2000]
                dig[f"{name}/sums"] = {
                    "hits": int((h.status == 1).sum()), "miss": int((h.status == 0).sum()),
                    "err": int((h.status == 2).sum()), "visited": int(h.visited.sum()),
                    "visited_max": int(h.visited.max()), "cf": int(h.cf[h.status == 1].sum()),
                    "tet": int(h.tet_front.sum()), "triangle": int(h.triangle[h.triangle >= 0].sum()),
                    "t": float(h.t[np.isfinite(h.t)].sum()),
                }
        for scheme in ("hilbert", "hilbert_regions", "shuffle"):
            r = reorder(m, scheme)
            dig[f"{name}/reorder/{scheme}"] = mesh_digest(r)
            if name in ("region4", "model"):
                h = batch.cast_rays(r, o[:2000], d[:2000], _remap_start(m, r, st[:2000]), kernels=K)
                dig[f"{name}/reorder/{scheme}/cast2k"] = digest(h.status, h.triangle, h.visited)

    # locality metric (render.py:565-591) and the reference's .npz format (cli.py:249-290)
    from tetray.cli import save_compact
    from tetray.render import visit_locality_metric

    for name in ("region4", "model"):
        for scheme in ("none", "hilbert", "shuffle"):
            dig[f"{name}/locality/{scheme}"] = visit_locality_metric(reorder(fixtures[name], scheme), kernels=K)
    save_compact(relayout(fixtures["pane4"], "tet16"), OUT / "pane4_tet16_ref.npz")

    # cast_ray_auto: origins inside and outside the hull (traversal.py:545-589)
    for name in ("box4", "pane4", "open_box4"):
        m = fixtures[name]
        rng = np.random.default_rng(50)
        o = rng.uniform(-2.0, 6.0, size=(400, 3)).astype(np.float32)
        d = rng.normal(size=(400, 3)).astype(np.float32)
        rows = []
        for i in range(len(o)):
            res = traversal.cast_ray_auto(Ray(Vec3(*o[i]), Vec3(*d[i])), m)
            if isinstance(res, traversal.HitRecord):
                rows.append((1, res.cf_index, res.triangle_id, res.t, res.tet_front, res.tet_back, res.visited))
            else:
                rows.append((0, -1, -1, np.inf, -1, -1, res.visited))
        a = np.array(rows, dtype=np.float64)
        arrays[f"{name}/auto/o"] = o
        arrays[f"{name}/auto/d"] = d
        arrays[f"{name}/auto/result"] = a  # kind, cf, triangle, t, front, back, visited

    # visit sequences (test_kernels.py:44-51)
    m = fixtures["region4"]
    o, d, st = interior_rays(m, 500, 41)
    _, visits, offsets = batch.cast_rays_visits(m, o, d, st, kernels=K)
    arrays["region4/visits/seq"] = visits
    arrays["region4/visits/offsets"] = offsets

    # point location (test_kernels.py:71-79)
    rng = np.random.default_rng(43)
    q = rng.uniform(-0.5, 4.5, size=(3000, 3))
    tq, vq = batch.locate_points(m, q, kernels=K)
    arrays["region4/locate/q"] = q
    arrays["region4/locate/tet"] = tq
    arrays["region4/locate/visited"] = vq

    # shadow rays (test_kernels.py:82-93)
    m = fixtures["pane4"]
    rng = np.random.default_rng(44)
    light = np.array([1.23, 2.91, 3.05])
    lt, _ = batch.locate_points(m, light[None], kernels=K)
    p = rng.uniform(0.05, 3.95, size=(3000, 3))
    pt, _ = batch.locate_points(m, p, kernels=K)
    occ, vs = batch.shadow_rays(m, p, light, pt, int(lt[0]), kernels=K)
    arrays["pane4/shadow/p"] = p
    arrays["pane4/shadow/p_tet"] = pt
    arrays["pane4/shadow/light"] = light
    arrays["pane4/shadow/light_tet"] = lt
    arrays["pane4/shadow/occ"] = occ
    arrays["pane4/shadow/visited"] = vs

    # ScTP predicate on random tets (test_traversal.py:349-368)
    rng = np.random.default_rng(35)
    cases, sctp, proj = [], [], []
    for _ in range(3000):
        tet = rng.normal(size=(4, 3))
        vol = np.dot(tet[1] - tet[0], np.cross(tet[2] - tet[0], tet[3] - tet[0]))
        if abs(vol) < 1e-3:
            continue
        bary = rng.dirichlet(np.ones(4) * 2.0)
        o3 = bary @ tet
        d3 = rng.normal(size=3)
        ray = Ray(Vec3(*o3), Vec3(*d3))
        cases.append(np.concatenate([tet.ravel(), o3, d3]))
        sctp.append(traversal.sctp_exit_face(ray, tet))
        proj.append(traversal.first_exit_face(ray, tet))
    arrays["sctp/cases"] = np.asarray(cases)
    arrays["sctp/exit"] = np.asarray(sctp, dtype=np.int8)
    arrays["sctp/first_exit_2d"] = np.asarray(proj, dtype=np.int8)

    # lattice camera: cycle-guard rays of the reference itself
    raw, soup = build_box_fixture(8, occluders=[(0, 4, (2, 2), (6, 6))])
    m = encode(raw, "tet20", soup)
    cfg = RenderConfig(camera_position=(4.0, 4.0, 0.5), camera_look_at=(4.0, 4.0, 8.0), width=1024, height=1024)
    ys, xs = np.mgrid[0:1024, 0:1024]
    o, d = camera_rays(cfg, xs.ravel().astype(np.float64), ys.ravel().astype(np.float64))
    cam, _ = batch.locate_points(m, np.array([cfg.camera_position]), kernels=K)
    st = np.full(len(o), cam[0], dtype=np.int32)
    status, cf, tet, visited = K.cast_rays(m, o, d, st)
    dig["lattice8/rays"] = digest(o, d)
    dig["lattice8/cam_tet"] = int(cam[0])
    dig["lattice8/cast"] = digest(status, cf, tet, visited)
    err = np.nonzero(status == 2)[0]
    dig["lattice8/errors"] = {"rays": err.tolist(), "tet": tet[err].tolist(), "visited": visited[err].tolist()}

    # config 1: blob GRID=12, 256x256 primaries from the blob camera
    for grid, w, h, key in ([(12, 256, 256, "blob12")] + ([(55, 1920, 1080, "blob55")] if args.big else [])):
        raw, soup = reference_blob(grid)
        base = encode(raw, "tet20", soup)
        cfg = RenderConfig(camera_position=(0.9, 5.0, 5.05), camera_look_at=(8.2, 5.1, 4.9), width=w, height=h)
        ys, xs = np.mgrid[0:h, 0:w]
        o, d = camera_rays(cfg, xs.ravel().astype(np.float64), ys.ravel().astype(np.float64))
        dig[f"{key}/rays"] = digest(o, d)
        for scheme in ("none", "hilbert"):
            mm = reorder(base, scheme)
            dig[f"{key}/{scheme}/mesh"] = mesh_digest(mm)
            cam, _ = batch.locate_points(mm, np.array([cfg.camera_position]), kernels=K)
            st = np.full(len(o), cam[0], dtype=np.int32)
            hh = batch.cast_rays(mm, o, d, st, kernels=K)
            dig[f"{key}/{scheme}/cam_tet"] = int(cam[0])
            dig[f"{key}/{scheme}/cast"] = digest(*hits_arrays(hh)[:4])
            dig[f"{key}/{scheme}/epilogue"] = digest(*hits_arrays(hh)[4:])
            dig[f"{key}/{scheme}/visited"] = {"sum": int(hh.visited.sum()), "max": int(hh.visited.max()),
                                             "hits": int((hh.status == 1).sum())}
        dig[f"{key}/sizes"] = {"points": int(base.n_points), "tets": int(base.n_tets), "cf": int(base.n_constrained)}

    np.savez_compressed(OUT / "golden_small.npz", **arrays)
    digest_path.write_text(json.dumps(dig, indent=1, sort_keys=True) + "\n")
    print(f"wrote {OUT / 'golden_small.npz'} ({(OUT / 'golden_small.npz').stat().st_size} B) and {digest_path}")


def _remap_start(m, r, st):
    """Start tets of the same rays in a reordered mesh: the tet whose sorted
    quadruple maps onto the original one (reorder keeps tets, renumbers)."""
    pts_new = {tuple(p): i for i, p in enumerate(r.points.tolist())}
    old2new_pt = np.array([pts_new[tuple(p)] for p in m.points.tolist()])
    quads = {tuple(q): i for i, q in enumerate(np.sort(r.side_verts, axis=1).tolist())}
    return np.array([quads[tuple(sorted(old2new_pt[m.side_verts[t]].tolist()))] for t in st], dtype=np.int32)


def _fx(n, **kw):
    raw, soup = build_box_fixture(n, **kw)
    return encode(raw, "tet20", soup)


if __name__ == "__main__":
    main()
