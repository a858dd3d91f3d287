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


# The reference's .npz member names (cli.py:249-290) and where each lives on a
# CompactMesh: a file written by either side loads on the other.
_NPZ_ARRAYS = (
    ("points", lambda m: m.points),
    ("records", lambda m: m.records_u32()),
    ("side_verts", lambda m: m.side_verts),
    ("side_neighbors", lambda m: m.side_neighbors),
    ("cf_triangle", lambda m: m.cf_triangle),
    ("cf_tets", lambda m: m.cf_tets),
    ("cf_verts", lambda m: m.cf_verts),
    ("soup_vertices", lambda m: m.soup.vertices),
    ("soup_triangles", lambda m: m.soup.triangles),
    ("soup_materials", lambda m: m.soup.material_ids),
)


def save_compact(mesh: CompactMesh, path) -> None:
    """Write ``mesh`` in the reference's compressed .npz layout."""
    members = {name: get(mesh) for name, get in _NPZ_ARRAYS}
    members["layout"] = np.array(mesh.layout)
    members["source_tet"] = np.array(mesh.source_tet)
    np.savez_compressed(path, **members)


def load_compact(path) -> CompactMesh:
    """Read a .npz written by ``save_compact`` or the reference CLI."""
    with np.load(path) as z:
        arr = {name: np.ascontiguousarray(z[name]) for name, _ in _NPZ_ARRAYS}
        layout = str(z["layout"])
        source = int(z["source_tet"])
    soup = SceneTriangleSoup(arr.pop("soup_vertices"), arr.pop("soup_triangles"), arr.pop("soup_materials"))
    records = arr.pop("records").view(LAYOUT_DTYPES[layout]).reshape(-1)
    return CompactMesh(layout=layout, records=records, source_tet=source, soup=soup, **arr)


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
