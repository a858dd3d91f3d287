"""Batch ray operations (mirror of the reference batch layer, batch.py:1-159).

Same entry points, arguments and ``BatchHits`` fields as
/root/reference/pkg/src/tetray/batch.py.  The difference is where the
epilogue runs: the reference computes triangle ids, fp64 ``t`` and the back
tet in host numpy after the kernel (batch.py:57-71, 0.25-0.4 us/ray); here
the kernel module's ``cast_rays_full`` returns them fused from the GPU.
``kernels`` defaults to this package's CUDA module; a kernels object must
provide ``cast_rays_full`` (there is no host epilogue to fall back to).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

STATUS_ERROR = 2


@dataclass
class BatchHits:
    status: np.ndarray  # (n,) uint8
    cf: np.ndarray  # (n,) int32
    triangle: np.ndarray  # (n,) int32, -1 on miss
    t: np.ndarray  # (n,) float64, +inf on miss
    tet_front: np.ndarray  # (n,) int32
    tet_back: np.ndarray  # (n,) int32, -1 on hull / miss
    visited: np.ndarray  # (n,) int32

    def __len__(self) -> int:
        return len(self.status)


def _kernels(k):
    if k is None:
        from . import kernels as k
    if not hasattr(k, "cast_rays_full"):
        raise TypeError(f"kernels module {getattr(k, 'BACKEND_NAME', k)!r} has no fused cast_rays_full")
    return k


def _raise_on_error(status) -> None:
    if np.any(status == STATUS_ERROR):
        bad = int(np.nonzero(status == STATUS_ERROR)[0][0])
        raise RuntimeError(f"traversal cycle guard tripped for ray {bad}")


def cast_rays(mesh, origins, dirs, start_tets, *, kernels=None) -> BatchHits:
    """Cast rays from known start tets (batch.py:39-80)."""
    k = _kernels(kernels)
    status, cf, tet, visited, triangle, t, back = k.cast_rays_full(mesh, origins, dirs, start_tets)
    _raise_on_error(status)
    return BatchHits(status=status, cf=cf, triangle=triangle, t=t, tet_front=tet, tet_back=back, visited=visited)


def cast_rays_auto(mesh, origins, dirs, *, kernels=None) -> BatchHits:
    """Cast from arbitrary origins (no start tets): batched
    traversal.cast_ray_auto (traversal.py:545-589) -- locate, or clip to the
    hull.  Rays entering through a constrained hull face hit it immediately
    (tet_front -1, tet_back = hull tet, visited 0)."""
    k = _kernels(kernels)
    status, cf, tet, visited, triangle, t, back = k.cast_rays_auto(mesh, origins, dirs)
    _raise_on_error(status)
    return BatchHits(status=status, cf=cf, triangle=triangle, t=t, tet_front=tet, tet_back=back, visited=visited)


def cast_rays_visits(mesh, origins, dirs, start_tets, *, kernels=None):
    """Cast and also return visit sequences (batch.py:83-137):
    (hits, visits, offsets), ray i visited visits[offsets[i]:offsets[i+1]]."""
    k = _kernels(kernels)
    hits = cast_rays(mesh, origins, dirs, start_tets, kernels=k)
    _, _, _, visited, seq, offsets = k.cast_rays_csr(mesh, origins, dirs, start_tets)
    if not np.array_equal(visited, hits.visited):
        raise RuntimeError("visit recording disagrees with the traversal")
    return hits, seq.astype(np.int32), offsets.astype(np.int64)


def locate_points(mesh, points, hints=None, *, kernels=None):
    """Point location -> (tets, visited), -1 outside (batch.py:140-148)."""
    k = _kernels(kernels)
    q = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    if hints is None:
        hints = np.full(len(q), mesh.source_tet, dtype=np.int32)
    else:
        hints = np.broadcast_to(np.asarray(hints, dtype=np.int32), (len(q),)).copy()
    return k.locate_points(mesh, q, hints)


def shadow_rays(mesh, points, light, point_tets, light_tet, *, eps=1e-4, kernels=None):
    """Occlusion tests -> (occluded, visited) (batch.py:151-159)."""
    k = _kernels(kernels)
    p = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    light = np.broadcast_to(np.asarray(light, dtype=np.float64).reshape(-1, 3), p.shape)
    pt = np.asarray(point_tets, dtype=np.int32)
    return k.shadow_rays(mesh, p, np.ascontiguousarray(light), pt, light_tet, eps)
