"""CUDA kernel module: the reference's backend protocol on sm_100a.

Drop-in for ``tetray._kernels`` (/root/reference/pkg/src/tetray/
_kernels.pyx:15-19,271,416,527): same module-level names, argument meaning,
output dtypes and per-ray status semantics, so it can be handed to the
reference's own batch layer as ``batch.cast_rays(mesh, o, d, st,
kernels=paper_2103_02309_b200.kernels)``.  Every call runs on the GPU
through the C ABI (include/tetb200.h); the mesh is uploaded to HBM once and
cached (device.py).  ``cast_rays_full`` additionally returns the fused
epilogue (triangle, fp64 t, back tet) that the reference computes on the
host (batch.py:57-71).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from ._lib import TetB200Error, addr, check, lib
from .device import device_mesh

# Per-tile fast path (csrc/fastcall.c): the same tb_cast_rays_host call with
# the argument handling in C and the GIL released -- the reference renderer
# calls cast_rays per 16x16 tile from a thread pool, where the backend's
# GIL-held time is what limits it.  Built with the library (make); without
# it every call takes the ctypes path below (same kernel, same results).
try:
    from . import _fastcall

    if os.environ.get("TETB200_NO_FASTCALL"):  # A/B knob: the ctypes path only
        raise ImportError
except ImportError:  # pragma: no cover - the Makefile builds it with the library
    _fastcall = None
else:
    _fastcall.bind(ctypes.cast(lib.tb_cast_rays_host, ctypes.c_void_p).value,
                   ctypes.cast(lib.tb_last_error, ctypes.c_void_p).value, TetB200Error)

BACKEND_NAME = "cuda"

STATUS_MISS = 0
STATUS_HIT = 1
STATUS_ERROR = 2


def _f32x3(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(-1, 3))


def _f64x3(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1, 3))


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))


def _check_tets(tets: np.ndarray, n_tets: int, what: str) -> None:
    if tets.size and (tets.min() < 0 or tets.max() >= n_tets):
        bad = int(np.nonzero((tets < 0) | (tets >= n_tets))[0][0])
        raise IndexError(f"{what}[{bad}] = {int(tets[bad])} is not a tet index (n_tets={n_tets})")


def _prep_cast(mesh, o32, d32, start):
    o = _f32x3(o32)
    d = _f32x3(d32)
    st = _i32(start)
    if not (len(o) == len(d) == len(st)):
        raise ValueError(f"length mismatch: {len(o)} origins, {len(d)} dirs, {len(st)} starts")
    _check_tets(st, mesh.n_tets, "start")
    return o, d, st


def cast_rays_full(mesh, o32, d32, start, *, layout: str | None = None, sctp: bool = False):
    """Traversal + fused epilogue: (status, cf, tet, visited, triangle, t, tet_back)."""
    o, d, st = _prep_cast(mesh, o32, d32, start)
    n = len(st)
    status = np.zeros(n, dtype=np.uint8)
    cf = np.full(n, -1, dtype=np.int32)
    tet = np.full(n, -1, dtype=np.int32)
    visited = np.ones(n, dtype=np.int32)
    triangle = np.full(n, -1, dtype=np.int32)
    t = np.full(n, np.inf, dtype=np.float64)
    back = np.full(n, -1, dtype=np.int32)
    if n:
        dm = device_mesh(mesh, layout=layout)
        fn = lib.tb_sctp_cast_rays_host if sctp else lib.tb_cast_rays_host
        check(
            fn(dm.handle, n, addr(o), addr(d), addr(st), addr(status), addr(cf), addr(tet), addr(visited),
               addr(triangle), addr(t), addr(back)),
            "tb_sctp_cast_rays_host" if sctp else "tb_cast_rays_host",
        )
        _check_cf(dm, mesh, status, cf)
    return status, cf, tet, visited, triangle, t, back


def _check_cf(dm, mesh, status, cf) -> None:
    """An unvalidated (corrupt) mesh can hit a constrained ref past the cf
    table; the kernel then skips the epilogue gathers and this raises, as the
    reference's batch epilogue does on mesh.cf_triangle[cf] (batch.py:63)."""
    if not dm.validated:
        n_cf = dm.n_cf  # ``mesh`` may itself be the DeviceMesh
        bad = np.nonzero((status == STATUS_HIT) & ((cf < 0) | (cf >= n_cf)))[0]
        if len(bad):
            raise IndexError(f"ray {int(bad[0])} hit constrained face {int(cf[bad[0]])}, outside the mesh's "
                             f"{n_cf} constrained faces")


def cast_rays(mesh, o32, d32, start, visits_sink=None):
    """Batch traversal -> (status u8, cf i32, tet i32, visited i32) (_kernels.pyx:271-370).

    With ``visits_sink`` (a list) the visited-tet sequences are appended as
    per-step (ray indices, tets) wavefronts, the format the reference's
    ``batch.cast_rays_visits`` consumes (batch.py:101-114).
    """
    if visits_sink is None:
        if _fastcall is not None:
            dm = device_mesh(mesh)
            r = _fastcall.cast4(dm.handle.value or 0, mesh.n_tets, o32, d32, start)
            if r is not None:
                _check_cf(dm, mesh, r[0], r[1])
                return r
        status, cf, tet, visited, *_ = _cast_plain(mesh, o32, d32, start)
        return status, cf, tet, visited
    status, cf, tet, visited, seq, offsets = cast_rays_csr(mesh, o32, d32, start)
    emit_visits(visits_sink, visited, seq, offsets)
    return status, cf, tet, visited


# Rays longer than this go to the sink as one chunk each (the compiled
# reference's format); shorter ones as step wavefronts.
_WAVEFRONT_STEPS = 32


def emit_visits(sink: list, visited: np.ndarray, seq: np.ndarray, offsets: np.ndarray) -> None:
    """CSR visit sequences -> the sink chunks batch.cast_rays_visits consumes
    (batch.py:101-114): ``(rays, tets)`` with distinct rays, appended in step
    order per ray.  Rays of at most 32 visits go out as step wavefronts (one
    chunk per step k: every short ray with more than k visits), longer rays
    -- and cycle-guard rays, n_tets + 1 visits -- as one chunk per ray, like
    the compiled reference (_kernels.pyx:307-341).  Cost O(total visits)."""
    n = len(visited)
    if n == 0:
        return
    short = np.nonzero(visited <= _WAVEFRONT_STEPS)[0]
    vs = visited[short]
    for k in range(int(vs.max(initial=0))):
        rays = short[vs > k]
        sink.append((rays.astype(np.int64), seq[offsets[rays] + k]))
    for r in np.nonzero(visited > _WAVEFRONT_STEPS)[0]:
        sink.append((np.full(int(visited[r]), r, dtype=np.int64), seq[offsets[r]:offsets[r + 1]].copy()))


def _cast_plain(mesh, o32, d32, start):
    o, d, st = _prep_cast(mesh, o32, d32, start)
    n = len(st)
    # every output element is written by the kernel
    status = np.empty(n, dtype=np.uint8)
    cf = np.empty(n, dtype=np.int32)
    tet = np.empty(n, dtype=np.int32)
    visited = np.empty(n, dtype=np.int32)
    if n:
        dm = device_mesh(mesh)
        check(
            lib.tb_cast_rays_host(dm.handle, n, addr(o), addr(d), addr(st), addr(status), addr(cf), addr(tet),
                                  addr(visited), None, None, None),
            "tb_cast_rays_host",
        )
    return status, cf, tet, visited


def cast_rays_csr(mesh, o32, d32, start, *, layout: str | None = None):
    """Traversal plus visit sequences as CSR: (status, cf, tet, visited, seq, offsets)."""
    import torch

    o, d, st = _prep_cast(mesh, o32, d32, start)
    n = len(st)
    if n == 0:
        z = np.zeros(0, dtype=np.int32)
        return np.zeros(0, np.uint8), z, z.copy(), z.copy(), z.copy(), np.zeros(1, np.int64)
    dm = device_mesh(mesh, layout=layout)
    dev = torch.device("cuda", dm.device)
    go, gd, gs = (torch.from_numpy(a).to(dev) for a in (o, d, st))
    status = torch.empty(n, dtype=torch.uint8, device=dev)
    cf, tet, visited = (torch.empty(n, dtype=torch.int32, device=dev) for _ in range(3))
    stream = torch.cuda.current_stream(dev).cuda_stream
    check(lib.tb_cast_rays(dm.handle, n, addr(go), addr(gd), addr(gs), addr(status), addr(cf), addr(tet),
                           addr(visited), None, None, None, stream), "tb_cast_rays")
    offsets = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(visited, 0, out=offsets[1:])
    total = int(offsets[-1].item())
    seq = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    check(lib.tb_cast_rays_visits(dm.handle, n, addr(go), addr(gd), addr(gs), addr(offsets), addr(seq), stream),
          "tb_cast_rays_visits")
    return (status.cpu().numpy(), cf.cpu().numpy(), tet.cpu().numpy(), visited.cpu().numpy(),
            seq[:total].cpu().numpy(), offsets.cpu().numpy())


def hull_clip(mesh, o32, d32):
    """Nearest boundary face hit by each ray (GPU brute force, fp64):
    returns (hull (k, 2) (tet, slot), face index per ray (-1 none), t)."""
    import torch

    from .tetmesh import hull_faces

    o = _f32x3(o32)
    d = _f32x3(d32)
    n = len(o)
    hull = hull_faces(mesh)
    face = np.full(n, -1, dtype=np.int32)
    tt = np.zeros(n, dtype=np.float64)
    if n == 0 or len(hull) == 0:
        return hull, face, tt
    others = np.array([[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]])
    vids = mesh.side_verts[hull[:, 0][:, None], others[hull[:, 1]]]
    table = np.ascontiguousarray(np.concatenate([hull[:, :1], vids], axis=1).astype(np.int32))
    dm = device_mesh(mesh)
    dev = torch.device("cuda", dm.device)
    go, gd, gt = (torch.from_numpy(a).to(dev) for a in (o, d, table))
    gf = torch.empty(n, dtype=torch.int32, device=dev)
    gtt = torch.empty(n, dtype=torch.float64, device=dev)
    check(lib.tb_hull_clip(dm.handle, n, addr(go), addr(gd), None, len(table), addr(gt), addr(gf), addr(gtt),
                           torch.cuda.current_stream(dev).cuda_stream), "tb_hull_clip")
    return hull, gf.cpu().numpy(), gtt.cpu().numpy()


def _scalar_t(o, d, tri):
    """traversal._ray_triangle_t (traversal.py:301-331): sequential-order fp64
    t for the few rays that enter through a constrained hull face."""
    e1 = tri[:, 1] - tri[:, 0]
    e2 = tri[:, 2] - tri[:, 0]
    p = np.stack([d[:, 1] * e2[:, 2] - d[:, 2] * e2[:, 1], d[:, 2] * e2[:, 0] - d[:, 0] * e2[:, 2],
                  d[:, 0] * e2[:, 1] - d[:, 1] * e2[:, 0]], axis=1)
    det = (e1[:, 0] * p[:, 0] + e1[:, 1] * p[:, 1]) + e1[:, 2] * p[:, 2]
    tv = o - tri[:, 0]
    q = np.stack([tv[:, 1] * e1[:, 2] - tv[:, 2] * e1[:, 1], tv[:, 2] * e1[:, 0] - tv[:, 0] * e1[:, 2],
                  tv[:, 0] * e1[:, 1] - tv[:, 1] * e1[:, 0]], axis=1)
    with np.errstate(divide="ignore", invalid="ignore"):
        t = ((e2[:, 0] * q[:, 0] + e2[:, 1] * q[:, 1]) + e2[:, 2] * q[:, 2]) * (1.0 / det)
        nrm = np.cross(e1, e2)
        den = (nrm[:, 0] * d[:, 0] + nrm[:, 1] * d[:, 1]) + nrm[:, 2] * d[:, 2]
        rel = tri[:, 0] - o
        tp = np.where(den != 0.0, ((nrm[:, 0] * rel[:, 0] + nrm[:, 1] * rel[:, 1]) + nrm[:, 2] * rel[:, 2]) / den, 0.0)
    return np.where(det != 0.0, t, tp)


def cast_rays_auto(mesh, o32, d32):
    """Cast without start tets (traversal.cast_ray_auto, traversal.py:545-589),
    batched on the GPU: locate each origin; origins outside the mesh are
    clipped to the nearest hull face -- entering through a constrained hull
    face is an immediate hit (front -1, back = the hull tet, visited 0),
    through an open boundary face the walk starts in that tet; no hull hit is
    a miss with visited 0.  Returns the 7 arrays of cast_rays_full."""
    o = _f32x3(o32)
    d = _f32x3(d32)
    n = len(o)
    start, _ = locate_points(mesh, o.astype(np.float64), np.full(n, mesh.source_tet, np.int32))
    status = np.zeros(n, np.uint8)
    cf = np.full(n, -1, np.int32)
    tet = np.full(n, -1, np.int32)
    visited = np.zeros(n, np.int32)
    triangle = np.full(n, -1, np.int32)
    t = np.full(n, np.inf)
    back = np.full(n, -1, np.int32)
    out = np.nonzero(start < 0)[0]
    if len(out):
        hull, face, _ = hull_clip(mesh, o[out], d[out])
        got = face >= 0
        ht, hj = hull[face[got], 0], hull[face[got], 1]
        refs = mesh.side_neighbors[ht, hj].astype(np.int64)
        con = (refs & (1 << 31)) != 0
        rays = out[got]
        start[rays[~con]] = ht[~con]
        hit = rays[con]
        cfi = (refs[con] & 0x7FFFFFFF).astype(np.int32)
        status[hit] = STATUS_HIT
        cf[hit] = cfi
        triangle[hit] = mesh.cf_triangle[cfi]
        back[hit] = ht[con]
        t[hit] = _scalar_t(o[hit].astype(np.float64), d[hit].astype(np.float64),
                           mesh.triangle_coords()[mesh.cf_triangle[cfi]])
    go = np.nonzero(start >= 0)[0]
    if len(go):
        res = cast_rays_full(mesh, o[go], d[go], start[go])
        for dst, src in zip((status, cf, tet, visited, triangle, t, back), res):
            dst[go] = src
    return status, cf, tet, visited, triangle, t, back


def locate_points(mesh, q, hints):
    """Batch point location -> (tet i32 (-1 outside), visited i32) (_kernels.pyx:416-492)."""
    qq = _f64x3(q)
    h = _i32(hints)
    n = len(qq)
    if len(h) != n:
        raise ValueError("hints length mismatch")
    out = np.full(n, -1, dtype=np.int32)
    visited = np.ones(n, dtype=np.int32)
    if n == 0:
        return out, visited
    _check_tets(h, mesh.n_tets, "hints")
    dm = device_mesh(mesh)
    check(lib.tb_locate_points_host(dm.handle, n, addr(qq), addr(h), addr(out), addr(visited)), "tb_locate_points_host")
    return out, visited


def shadow_rays(mesh, p, light, p_tet, light_tet, eps=1e-4):
    """Batch occlusion -> (occluded bool, visited i32) (_kernels.pyx:527-614).

    ``light`` is one (3,) point or (n, 3); ``light_tet`` an int or (n,).
    """
    pp = _f64x3(p)
    n = len(pp)
    ll = _f64x3(light)
    lt = np.ascontiguousarray(np.asarray(light_tet, dtype=np.int32).reshape(-1))
    pt = _i32(p_tet)
    if len(pt) != n:
        raise ValueError("p_tet length mismatch")
    if len(ll) not in (1, n) or len(lt) not in (1, n):
        raise ValueError("light / light_tet must be one value or one per ray")
    occ = np.zeros(n, dtype=bool)
    visited = np.ones(n, dtype=np.int32)
    if n == 0:
        return occ, visited
    _check_tets(pt, mesh.n_tets, "p_tet")
    lstride = 3 if (len(ll) == n and n > 1) else 0
    ltstride = 1 if (len(lt) == n and n > 1) else 0
    dm = device_mesh(mesh)
    check(
        lib.tb_shadow_rays_host(dm.handle, n, addr(pp), addr(ll), lstride, addr(pt), addr(lt), ltstride, float(eps),
                                addr(occ.view(np.uint8)), addr(visited)),
        "tb_shadow_rays_host",
    )
    return occ, visited
