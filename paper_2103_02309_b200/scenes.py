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
BLOB_CAMERA = dict(position=(0.9, 5.0, 5.05), look_at=(8.2, 5.1, 4.9), up=(0.0, 1.0, 0.0), fov=68.0)


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


def kuhn_camera(n: int, scale=KUHN5_SCALE):
    """Off-lattice camera looking down +x (the Kuhn-box camera of SURVEY
    8(d), nudged off the lattice so no ray ties exactly on a diagonal)."""
    pos = (0.11 * n + 0.0137, 0.53 * n + 0.0173, (0.52 * n + 0.0111) * scale[2])
    look = (0.97 * n, 0.46 * n, 0.48 * n * scale[2])
    return dict(position=pos, look_at=look, up=(0.0, 1.0, 0.0), fov=68.0)


def kuhn_strip_scene(n: int = KUHN5_N, layout: str = "tet16", scheme: str = "none", scale=KUHN5_SCALE) -> Scene:
    from .ingestion import build_kuhn_box

    raw, soup = build_kuhn_box(n, kuhn_strips(n), walls="constrained", scale=tuple(float(s) for s in scale))
    mesh = reorder(encode(raw, layout, soup, check=False), scheme)
    return Scene(mesh=mesh, raw=raw, soup=soup, seed=0, name=f"kuhn{n}-strips")


# ---------------------------------------------------------------------------
# Rays


def camera_frame(position, look_at, up, fov, width, height) -> np.ndarray:
    """The per-frame camera constants of render.camera_rays (render.py:169-185):
    float64 [fwd(3), right(3), up2(3), pos(3), half_w, half_h] -- what the
    device ray generator (tb_camera_rays) needs."""
    pos = np.asarray(position, dtype=np.float64)
    look = np.asarray(look_at, dtype=np.float64)
    upv = np.asarray(up, dtype=np.float64)
    fwd = look - pos
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, upv)
    right = right / np.linalg.norm(right)
    up2 = np.cross(right, fwd)
    half_h = np.tan(np.radians(fov) * 0.5)
    half_w = half_h * width / height
    return np.concatenate([fwd, right, up2, pos, [half_w, half_h]]).astype(np.float64)


def camera_rays(position, look_at, up, fov, width, height, xs=None, ys=None):
    """f32 (origins, dirs) through pixel centres, row-major over the frame
    unless explicit pixel coordinates are given (render.py:169-185)."""
    if xs is None:
        yy, xx = np.mgrid[0:height, 0:width]
        xs = xx.ravel().astype(np.float64)
        ys = yy.ravel().astype(np.float64)
    fr = camera_frame(position, look_at, up, fov, width, height)
    fwd, right, up2, pos = fr[0:3], fr[3:6], fr[6:9], fr[9:12]
    half_w, half_h = fr[12], fr[13]
    sx = ((xs + 0.5) / width * 2.0 - 1.0) * half_w
    sy = (1.0 - (ys + 0.5) / height * 2.0) * half_h
    d = fwd[None] + sx[:, None] * right[None] + sy[:, None] * up2[None]
    o = np.broadcast_to(pos, d.shape)
    return np.ascontiguousarray(o, dtype=np.float32), np.ascontiguousarray(d, dtype=np.float32)


def diffuse_secondaries(origins, dirs, t, triangle, tet_front, tri_coords, seed: int = 4):
    """Incoherent secondary rays from primary hits (BASELINE config 4).

    origin = f32(o + t d) in fp64, start = front tet, direction uniform on
    the hemisphere around the face normal that faces the incoming ray.
    Returns (o32, d32, start) for the hit rays only, in ray order.
    """
    hit = triangle >= 0
    o64 = origins[hit].astype(np.float64)
    d64 = dirs[hit].astype(np.float64)
    hp = o64 + t[hit][:, None] * d64
    tc = tri_coords[triangle[hit]]
    n = np.cross(tc[:, 1] - tc[:, 0], tc[:, 2] - tc[:, 0])
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    d_unit = d64 / np.linalg.norm(d64, axis=1, keepdims=True)
    flip = np.sum(n * d_unit, axis=1) > 0
    n[flip] = -n[flip]
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(len(hp), 3))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    back = np.sum(v * n, axis=1) < 0
    v[back] = -v[back]
    return hp.astype(np.float32), v.astype(np.float32), tet_front[hit].astype(np.int32)


def interior_rays(mesh, n: int, seed: int):
    """Random rays from interior points of random tets (the reference's
    parity ray source, tests/conftest.py:61-73)."""
    rng = np.random.default_rng(seed)
    ti = rng.integers(0, mesh.n_tets, n).astype(np.int32)
    bary = rng.dirichlet(np.ones(4) * 4.0, n)
    pts = mesh.points.astype(np.float64)
    o = np.einsum("ij,ijk->ik", bary, pts[mesh.side_verts[ti]])
    d = rng.normal(size=(n, 3))
    return o.astype(np.float32), d.astype(np.float32), ti
