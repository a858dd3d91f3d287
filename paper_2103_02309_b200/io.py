"""Compact-mesh persistence and traversal statistics.

* ``save_compact`` / ``load_compact`` -- the reference's ``.npz`` format
  (cli.py:249-290, same keys), so meshes converted by the reference CLI load
  here and vice versa; ``load_device`` goes straight from a file to an
  HBM-resident ``DeviceMesh``.
* ``visit_locality_metric`` -- mean |index distance| between consecutively
  visited tets (render.py:565-591), the reorder-quality measure of the
  reference, computed from GPU visit sequences.
"""

from __future__ import annotations

import numpy as np

from .tetmesh import LAYOUT_DTYPES, CompactMesh, SceneTriangleSoup


def save_compact(mesh: CompactMesh, path) -> None:
    np.savez_compressed(
        path,
        layout=np.array(mesh.layout),
        points=mesh.points,
        records=mesh.records_u32(),
        side_verts=mesh.side_verts,
        side_neighbors=mesh.side_neighbors,
        cf_triangle=mesh.cf_triangle,
        cf_tets=mesh.cf_tets,
        cf_verts=mesh.cf_verts,
        source_tet=np.array(mesh.source_tet),
        soup_vertices=mesh.soup.vertices,
        soup_triangles=mesh.soup.triangles,
        soup_materials=mesh.soup.material_ids,
    )


def load_compact(path) -> CompactMesh:
    data = np.load(path)
    layout = str(data["layout"])
    recs = np.ascontiguousarray(data["records"]).view(LAYOUT_DTYPES[layout]).reshape(-1)
    soup = SceneTriangleSoup(
        vertices=data["soup_vertices"], triangles=data["soup_triangles"], material_ids=data["soup_materials"]
    )
    return CompactMesh(
        layout=layout,
        points=np.ascontiguousarray(data["points"]),
        records=recs,
        side_verts=np.ascontiguousarray(data["side_verts"]),
        side_neighbors=np.ascontiguousarray(data["side_neighbors"]),
        cf_triangle=np.ascontiguousarray(data["cf_triangle"]),
        cf_tets=np.ascontiguousarray(data["cf_tets"]),
        cf_verts=np.ascontiguousarray(data["cf_verts"]),
        source_tet=int(data["source_tet"]),
        soup=soup,
    )


def load_device(path, device: int | None = None, layout: str | None = None):
    """``.npz`` -> (CompactMesh, DeviceMesh resident in HBM)."""
    from .device import DeviceMesh

    mesh = load_compact(path)
    return mesh, DeviceMesh(mesh, device, layout)


def visit_locality_metric(mesh: CompactMesh, n_rays: int = 1024, seed: int = 5, kernels=None) -> float:
    """render.visit_locality_metric (render.py:565-591) on the GPU kernels:
    random interior origins located from the source tet, random directions,
    mean |tet index delta| along the visit sequences."""
    from . import batch

    rng = np.random.default_rng(seed)
    pts = mesh.points.astype(np.float64)
    lo, hi = pts.min(axis=0), pts.max(axis=0)
    span = hi - lo
    o = rng.uniform(lo + 0.02 * span, hi - 0.02 * span, size=(n_rays, 3))
    d = rng.normal(size=(n_rays, 3))
    starts, _ = batch.locate_points(mesh, o, kernels=kernels)
    ok = starts >= 0
    _, visits, offsets = batch.cast_rays_visits(mesh, o[ok], d[ok], starts[ok], kernels=kernels)
    seq = visits.astype(np.int64)
    if len(seq) < 2:
        return 0.0
    delta = np.abs(np.diff(seq))
    # drop the jumps between consecutive rays' sequences
    same = np.ones(len(delta), dtype=bool)
    ends = offsets[1:-1] - 1
    same[ends[(ends >= 0) & (ends < len(delta))]] = False
    delta = delta[same]
    return float(delta.mean()) if len(delta) else 0.0
