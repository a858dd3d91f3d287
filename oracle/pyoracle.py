"""Python face of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Binds oracle/libtetoracle.so (the C restatement in tetoracle.c) with the
same kernel-module protocol as the reference (_kernels.pyx:15-19,271,416,
527) plus ``cast_rays_full`` / ``cast_rays_csr`` / ``sctp_cast_rays``, so
tests can compare it call-for-call with the CUDA module.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline leg may import this.

``ref_kernels()`` returns the reference's own compiled kernels built by
oracle/build_ref.sh into oracle/_ref/ (None when absent).
"""

from __future__ import annotations

import ctypes
import os
import sys
from ctypes import POINTER, c_double, c_int, c_int64, c_void_p

import numpy as np

BACKEND_NAME = "oracle-c"
STATUS_MISS, STATUS_HIT, STATUS_ERROR = 0, 1, 2

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libtetoracle.so")
_lib = None

LAYOUT_CODES = {"tet32": 32, "tet20": 20, "tet16": 16, "tet80": 80}


class _Mesh(ctypes.Structure):
    _fields_ = [
        ("layout", c_int),
        ("n_points", c_int64),
        ("n_tets", c_int64),
        ("pts", c_void_p),
        ("recs", c_void_p),
        ("sv", c_void_p),
        ("sn", c_void_p),
        ("cf_tri", c_void_p),
        ("cf_tets", c_void_p),
        ("tri", c_void_p),
    ]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} missing: run `make oracle/libtetoracle.so`")
        L = ctypes.CDLL(_LIB_PATH)
        P = c_void_p
        L.to_cast_rays.argtypes = [POINTER(_Mesh), c_int64, P, P, P, P, P, P, P, P, P, P, c_int]
        L.to_sctp_cast_rays.argtypes = [POINTER(_Mesh), c_int64, P, P, P, P, P, P, P, P, P, P, c_int]
        L.to_cast_rays_visits.argtypes = [POINTER(_Mesh), c_int64, P, P, P, P, P]
        L.to_locate_points.argtypes = [POINTER(_Mesh), c_int64, P, P, P, P, c_int]
        L.to_shadow_rays.argtypes = [POINTER(_Mesh), c_int64, P, P, c_int, P, P, c_int, c_double, P, P, c_int]
        L.to_sctp_exit_face.argtypes = [P, P, P, c_int]
        L.to_sctp_exit_face.restype = c_int
        L.to_build_tet80.argtypes = [P, P, P, c_int64, P]
        L.to_mt_t.argtypes = [P, P, P]
        L.to_mt_t.restype = c_double
        _lib = L
    return _lib


def _a(x):
    return None if x is None else x.ctypes.data


class OracleMesh:
    """Keeps the contiguous arrays alive for the C struct."""

    def __init__(self, mesh, layout: str | None = None):
        self.layout = layout or mesh.layout
        self.pts = np.ascontiguousarray(mesh.points, dtype=np.float32)
        self.sv = np.ascontiguousarray(mesh.side_verts, dtype=np.int32)
        self.sn = np.ascontiguousarray(mesh.side_neighbors, dtype=np.uint32)
        if self.layout == "tet80":
            self.recs = np.empty((len(self.sv), 20), dtype=np.uint32)
            lib().to_build_tet80(_a(self.sv), _a(self.sn), _a(self.pts), len(self.sv), _a(self.recs))
        elif self.layout == mesh.layout:
            self.recs = np.ascontiguousarray(mesh.records_u32(), dtype=np.uint32)
        else:
            from paper_2103_02309_b200.tetmesh import _records_from_tables

            self.recs = np.ascontiguousarray(
                _records_from_tables(self.layout, self.sv, self.sn).view("<u4").reshape(len(self.sv), -1))
        self.cf_tri = np.ascontiguousarray(mesh.cf_triangle, dtype=np.int32)
        self.cf_tets = np.ascontiguousarray(np.asarray(mesh.cf_tets, dtype=np.int32).reshape(-1, 2))
        self.tri = np.ascontiguousarray(mesh.triangle_coords(), dtype=np.float64).reshape(-1, 9)
        self.n_tets = len(self.sv)
        self.c = _Mesh(LAYOUT_CODES[self.layout], len(self.pts), len(self.sv), _a(self.pts), _a(self.recs),
                       _a(self.sv), _a(self.sn), _a(self.cf_tri), _a(self.cf_tets), _a(self.tri))


def _threads(n_threads):
    return int(n_threads) if n_threads else (os.cpu_count() or 1)


def _prep(o32, d32, start):
    o = np.ascontiguousarray(np.asarray(o32, dtype=np.float32).reshape(-1, 3))
    d = np.ascontiguousarray(np.asarray(d32, dtype=np.float32).reshape(-1, 3))
    st = np.ascontiguousarray(np.asarray(start, dtype=np.int32).reshape(-1))
    return o, d, st


def cast_rays_full(mesh, o32, d32, start, *, layout=None, n_threads=None, sctp=False):
    om = OracleMesh(mesh, layout)
    o, d, st = _prep(o32, d32, start)
    n = len(st)
    out = (np.zeros(n, np.uint8), np.full(n, -1, np.int32), np.full(n, -1, np.int32), np.ones(n, np.int32),
           np.full(n, -1, np.int32), np.full(n, np.inf), np.full(n, -1, np.int32))
    if n:
        fn = lib().to_sctp_cast_rays if sctp else lib().to_cast_rays
        fn(ctypes.byref(om.c), n, _a(o), _a(d), _a(st), *[_a(x) for x in out], _threads(n_threads))
    return out


def cast_rays(mesh, o32, d32, start, visits_sink=None):
    status, cf, tet, visited, *_ = cast_rays_full(mesh, o32, d32, start)
    if visits_sink is not None:
        _, _, _, _, seq, offsets = cast_rays_csr(mesh, o32, d32, start)
        for r in range(len(status)):
            visits_sink.append((np.full(visited[r], r, dtype=np.int64), seq[offsets[r]:offsets[r + 1]].copy()))
    return status, cf, tet, visited


def cast_rays_csr(mesh, o32, d32, start, *, layout=None):
    status, cf, tet, visited, *_ = cast_rays_full(mesh, o32, d32, start, layout=layout)
    offsets = np.zeros(len(visited) + 1, dtype=np.int64)
    np.cumsum(visited, out=offsets[1:])
    seq = np.empty(int(offsets[-1]), dtype=np.int32)
    om = OracleMesh(mesh, layout)
    o, d, st = _prep(o32, d32, start)
    if len(st):
        lib().to_cast_rays_visits(ctypes.byref(om.c), len(st), _a(o), _a(d), _a(st), _a(offsets), _a(seq))
    return status, cf, tet, visited, seq, offsets


def locate_points(mesh, q, hints, *, n_threads=None):
    om = OracleMesh(mesh)
    qq = np.ascontiguousarray(np.asarray(q, dtype=np.float64).reshape(-1, 3))
    h = np.ascontiguousarray(np.asarray(hints, dtype=np.int32).reshape(-1))
    out = np.full(len(qq), -1, np.int32)
    vis = np.ones(len(qq), np.int32)
    if len(qq):
        lib().to_locate_points(ctypes.byref(om.c), len(qq), _a(qq), _a(h), _a(out), _a(vis), _threads(n_threads))
    return out, vis


def shadow_rays(mesh, p, light, p_tet, light_tet, eps=1e-4, *, n_threads=None):
    om = OracleMesh(mesh)
    pp = np.ascontiguousarray(np.asarray(p, dtype=np.float64).reshape(-1, 3))
    n = len(pp)
    ll = np.ascontiguousarray(np.asarray(light, dtype=np.float64).reshape(-1, 3))
    lt = np.ascontiguousarray(np.asarray(light_tet, dtype=np.int32).reshape(-1))
    pt = np.ascontiguousarray(np.asarray(p_tet, dtype=np.int32).reshape(-1))
    occ = np.zeros(n, np.uint8)
    vis = np.ones(n, np.int32)
    if n:
        lib().to_shadow_rays(ctypes.byref(om.c), n, _a(pp), _a(ll), 3 if len(ll) == n and n > 1 else 0, _a(pt),
                             _a(lt), 1 if len(lt) == n and n > 1 else 0, float(eps), _a(occ), _a(vis),
                             _threads(n_threads))
    return occ.astype(bool), vis


def sctp_exit_face(verts, o, d, entry=None) -> int:
    v = np.ascontiguousarray(np.asarray(verts, dtype=np.float64).reshape(4, 3))
    oo = np.ascontiguousarray(np.asarray(o, dtype=np.float64).reshape(3))
    dd = np.ascontiguousarray(np.asarray(d, dtype=np.float64).reshape(3))
    return int(lib().to_sctp_exit_face(_a(v), _a(oo), _a(dd), -1 if entry is None else int(entry)))


def ref_kernels():
    """The reference's own compiled kernels (oracle/_ref), or None."""
    ref_dir = os.path.join(_HERE, "_ref")
    if not os.path.isdir(ref_dir):
        return None
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    try:
        import _kernels  # type: ignore

        return _kernels
    except ImportError:
        return None


def batch_epilogue(mesh, o32, d32, status, cf, tet):
    """numpy restatement of the reference batch layer's host epilogue
    (batch.py:57-71 + _kernels_py._mt_t, _kernels_py.py:435-454): the part of
    batch.cast_rays that runs after the compiled kernel.  Used to time the
    reference's CPU path end to end (bench.py --impl reference)."""
    n = len(status)
    triangle = np.full(n, -1, dtype=np.int32)
    t = np.full(n, np.inf, dtype=np.float64)
    back = np.full(n, -1, dtype=np.int32)
    hit = status == STATUS_HIT
    if hit.any():
        cfs = cf[hit]
        triangle[hit] = mesh.cf_triangle[cfs]
        tri = mesh.triangle_coords()[mesh.cf_triangle[cfs]]
        o = np.asarray(o32)[hit].astype(np.float64)
        d = np.asarray(d32)[hit].astype(np.float64)
        e1 = tri[:, 1] - tri[:, 0]
        e2 = tri[:, 2] - tri[:, 0]
        pv = np.cross(d, e2)
        det = np.einsum("ij,ij->i", e1, pv)
        tv = o - tri[:, 0]
        with np.errstate(divide="ignore", invalid="ignore"):
            inv = np.where(det != 0.0, 1.0 / det, 0.0)
            tt = np.einsum("ij,ij->i", e2, np.cross(tv, e1)) * inv
        par = det == 0.0
        if par.any():
            nrm = np.cross(e1[par], e2[par])
            den = np.einsum("ij,ij->i", nrm, d[par])
            num = np.einsum("ij,ij->i", nrm, tri[par, 0] - o[par])
            with np.errstate(divide="ignore", invalid="ignore"):
                tt[par] = np.where(den != 0.0, num / den, 0.0)
        t[hit] = tt
        a = mesh.cf_tets[cfs, 0]
        b = mesh.cf_tets[cfs, 1]
        back[hit] = np.where(a == tet[hit], b, a)
    return triangle, t, back
