"""Synthetic workloads of the benchmark configurations -- numpy only.

Kept free of the CUDA library so the bench's reference arm (bench.py
--impl reference) can generate exactly the same rays in a process that
never maps libtetb200.so.

* ``camera_rays`` -- fp64 pinhole rays cast to f32 (render.py:169-185).
* ``diffuse_secondaries`` -- config 4's incoherent rays: hit point in fp64,
  start at the front tet (render.py:353,404-407), uniform hemisphere about
  the face normal flipped toward the incoming side (render.py:355-359).
* ``interior_rays`` -- the reference's parity ray source (tests/conftest.py:61-73).
"""

from __future__ import annotations

import numpy as np

# BASELINE config cameras: the blob camera of
# test_render.py:174-178 / render.py:51 defaults.
BLOB_CAMERA = dict(position=(0.9, 5.0, 5.05), look_at=(8.2, 5.1, 4.9), up=(0.0, 1.0, 0.0), fov=68.0)
KUHN5_SCALE = (1.0, 1.0, 4.0)


def kuhn_camera(n: int, scale=KUHN5_SCALE):
    """Off-lattice camera looking down +x (the Kuhn-box camera of SURVEY
    8(d), nudged off the lattice so no ray ties exactly on a diagonal)."""
    pos = (0.11 * n + 0.0137, 0.53 * n + 0.0173, (0.52 * n + 0.0111) * scale[2])
    look = (0.97 * n, 0.46 * n, 0.48 * n * scale[2])
    return dict(position=pos, look_at=look, up=(0.0, 1.0, 0.0), fov=68.0)


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
