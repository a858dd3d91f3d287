"""Synthetic scenes and ray sources for the benchmark configurations.

* ``blob_scene`` -- the reference's model-mesh generator
  (/root/reference/pkg/tools/gen_model_mesh.py:25-127: jittered grid,
  Delaunay, sliver filter, spherical blob surface + convex hull as the
  constrained faces) followed by what ``parse_tetgen`` / ``load_obj`` /
  ``associate_constrained_faces`` make of its files (ingestion.py:87-288,
  470-529) -- built straight into arrays, no files, so GRID=55 (1.1 M tets,
  BASELINE config 2) builds in seconds instead of minutes.
* ``camera_rays`` -- fp64 pinhole rays cast to f32 (render.py:169-185).
* ``diffuse_secondaries`` -- config 4's incoherent rays: hit point in fp64,
  start at the front tet (render.py:353,404-407), cosine-free uniform
  hemisphere about the face normal flipped toward the incoming side.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .tetmesh import (
    BOUNDARY_REF,
    CompactMesh,
    RawTetMesh,
    SceneTriangleSoup,
    encode,
    face_incidence_arrays,
    reorder,
    unpack_keys,
)
from .ingestion import mark_constrained

EXTENT = 10.0
JITTER = 0.32
BLOB_RADIUS = 3.15
BLOB_CENTER = np.array([5.0, 5.0, 5.0])

# BASELINE config cameras: the blob camera of
# test_render.py:174-178 / render.py:51 defaults.
from .workload import BLOB_CAMERA  # noqa: E402,F401  (test_render.py:174-178 / render.py:51)


def blob_points(grid: int, seed: int) -> np.ndarray:
    """Jittered grid rounded to f32-representable values (gen_model_mesh.py:32-40)."""
    rng = np.random.default_rng(seed)
    axes = np.linspace(0.0, EXTENT, grid)
    pts = np.stack(np.meshgrid(axes, axes, axes, indexing="ij"), axis=-1).reshape(-1, 3)
    spacing = EXTENT / (grid - 1)
    pts = pts + rng.uniform(-JITTER, JITTER, size=pts.shape) * spacing
    return pts.astype(np.float32).astype(np.float64)


def _volumes(points, tets):
    p = points[tets]
    return np.einsum("ij,ij->i", p[:, 1] - p[:, 0], np.cross(p[:, 2] - p[:, 0], p[:, 3] - p[:, 0]))


def blob_tetrahedralization(grid: int, seed: int):
    """Delaunay + orientation fix + sliver filter (gen_model_mesh.py:52-63);
    None when the seed fails the filter."""
    from scipy.spatial import Delaunay

    points = blob_points(grid, seed)
    tets = Delaunay(points).simplices.astype(np.int64)
    vols = _volumes(points, tets)
    neg = vols < 0
    tets[neg] = tets[neg][:, [0, 2, 1, 3]]
    vols = _volumes(points, tets)
    v32 = _volumes(points.astype(np.float32).astype(np.float64), tets)
    if vols.min() < 1e-7 * np.median(vols) or v32.min() <= 0:
        return None
    return points, tets


@dataclass
class Scene:
    mesh: CompactMesh
    raw: RawTetMesh
    soup: SceneTriangleSoup
    seed: int
    name: str


def blob_raw(grid: int = 8, seed: int | None = None):
    """RawTetMesh + soup exactly as parse_tetgen/load_obj/associate would
    produce them from gen_model_mesh's output for this GRID."""
    seeds = range(100) if seed is None else [seed]
    got = None
    for s in seeds:
        got = blob_tetrahedralization(grid, s)
        if got is not None:
            seed = s
            break
    if got is None:
        raise RuntimeError("no sliver-free tetrahedralization found")
    points, tets = got
    n_points = len(points)
    keys, first, second = face_incidence_arrays(tets, n_points)
    centroids = points[tets].mean(axis=1)
    inside = np.linalg.norm(centroids - BLOB_CENTER, axis=1) < BLOB_RADIUS
    pair = second >= 0
    nbr = np.full((len(tets), 4), -1, dtype=np.int64)
    t0, j0, t1, j1 = first[pair] // 4, first[pair] % 4, second[pair] // 4, second[pair] % 4
    nbr[t0, j0] = t1
    nbr[t1, j1] = t0
    surface = np.where(pair, inside[first // 4] != inside[np.where(pair, second, first) // 4], True)
    face_keys = unpack_keys(keys[surface], n_points)  # ascending key order = file order
    refs = np.where(nbr < 0, np.int64(BOUNDARY_REF), nbr).astype(np.uint32)
    raw = RawTetMesh(points=points, tets=tets.astype(np.int32), neighbors=refs)
    mark_constrained(raw, face_keys)
    # load_obj of the matching OBJ: used vertices in ascending id order, one
    # triangle per constrained face in file order (gen_model_mesh.py:112-123);
    # association is then the identity (each face is its own triangle).
    used = np.unique(face_keys)
    remap = np.full(n_points, -1, dtype=np.int64)
    remap[used] = np.arange(len(used))
    soup = SceneTriangleSoup(
        vertices=points[used].copy(),
        triangles=remap[face_keys].astype(np.int32),
        material_ids=np.zeros(len(face_keys), dtype=np.int32),
    )
    raw.cf_triangle = np.arange(len(face_keys), dtype=np.int32)
    return raw, soup, seed


def blob_scene(grid: int = 8, seed: int | None = None, layout: str = "tet20", scheme: str = "none",
               check: bool = True) -> Scene:
    raw, soup, seed = blob_raw(grid, seed)
    mesh = encode(raw, layout, soup, check=check)
    mesh = reorder(mesh, scheme)
    return Scene(mesh=mesh, raw=raw, soup=soup, seed=seed, name=f"blob-grid{grid}")


# ---------------------------------------------------------------------------
# Config 5: large Kuhn box with long thin triangles.  The reference's builder
# cannot produce 50 M tets; build_kuhn_box is the
# analytic restatement of its box fixture (identical arrays, tested), here
# stretched along z so tets, wall triangles and the strip occluders are long
# and thin, with strip occluders (1 x 4-cell-high bands across y) on x planes.

KUHN5_N = 203
KUHN5_SCALE = (1.0, 1.0, 4.0)


def kuhn_strips(n: int):
    """Thin strip occluders on x planes: y in [0.1n, 0.9n), 4 cells of z."""
    ks = sorted({max(1, min(n - 1, int(round(f * n)))) for f in (0.2, 0.4, 0.6, 0.8, 0.98)})
    y0, y1 = int(0.1 * n), max(int(0.1 * n) + 1, int(0.9 * n))
    z0 = int(0.47 * n)
    return [(0, k, (y0, z0), (y1, min(n, z0 + 4))) for k in ks]


from .workload import kuhn_camera  # noqa: E402,F401


def kuhn_strip_scene(n: int = KUHN5_N, layout: str = "tet16", scheme: str = "none", scale=KUHN5_SCALE) -> Scene:
    from .ingestion import build_kuhn_box

    raw, soup = build_kuhn_box(n, kuhn_strips(n), walls="constrained", scale=tuple(float(s) for s in scale))
    mesh = reorder(encode(raw, layout, soup, check=False), scheme)
    return Scene(mesh=mesh, raw=raw, soup=soup, seed=0, name=f"kuhn{n}-strips")


# ---------------------------------------------------------------------------
# Rays


# The ray sources live in workload.py (numpy only: the bench's reference arm
# generates the same rays without loading this package's CUDA library).
from .workload import camera_frame, camera_rays, diffuse_secondaries, interior_rays  # noqa: E402,F401
