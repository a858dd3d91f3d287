"""HBM-resident meshes: upload once, cache per (mesh, layout, device).

The reference kernels read the mesh arrays on every call
(_kernels.pyx:276-282); here a ``CompactMesh`` is uploaded to HBM on first
use and the handle is cached.  The cache key is the mesh object plus the
identity and shape of every array the device copy is built from (the entry
holds those arrays, so identities cannot be recycled while it lives):
replacing an array (``relayout``, ``reorder``, ``dataclasses.replace``,
``mesh.points = ...``) triggers a fresh upload.  In-place mutation cannot go
stale silently: while a device copy is cached, the arrays it mirrors are
marked read-only, so writing into them raises numpy's "assignment
destination is read-only" -- call ``invalidate(mesh)`` first (it restores
writability; the next call uploads again).  The per-call check is a tuple
of ids and shapes (~1 us), not a hash of the data: renderers call
``cast_rays`` once per 16x16 tile (render.py:538-541).
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np

from . import _lib
from ._lib import addr, check, lib

LAYOUT_CODES = {"tet32": 32, "tet20": 20, "tet16": 16, "tet80": 80}


def default_device() -> int:
    env = os.environ.get("TETB200_DEVICE")
    if env is not None:
        return int(env)
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:  # torch is plumbing only; the library does not need it
        pass
    return 0


class DeviceMesh:
    """A mesh resident in one GPU's HBM (wraps a ``tb_mesh*``).

    ``layout`` defaults to the mesh's own; ``"tet80"`` builds TetMesh-80
    records (ids + refs + inline coordinates) on the device.
    """

    def __init__(self, mesh, device: int | None = None, layout: str | None = None):
        self.device = default_device() if device is None else int(device)
        self.layout = layout or mesh.layout
        if self.layout not in LAYOUT_CODES:
            raise ValueError(f"unknown layout {self.layout!r}")
        code = LAYOUT_CODES[self.layout]
        pts = np.ascontiguousarray(mesh.points, dtype=np.float32)
        sv = np.ascontiguousarray(mesh.side_verts, dtype=np.int32)
        sn = np.ascontiguousarray(mesh.side_neighbors, dtype=np.uint32)
        if code == 80:
            recs = None
        else:
            if self.layout != mesh.layout:
                from .tetmesh import _records_from_tables

                recs = _records_from_tables(self.layout, sv, sn).view("<u4").reshape(len(sv), -1)
            else:
                recs = np.ascontiguousarray(mesh.records_u32(), dtype=np.uint32)
            if recs.shape != (len(sv), code // 4):
                raise ValueError(f"records shape {recs.shape} does not match layout {self.layout}")
        cft = np.ascontiguousarray(mesh.cf_triangle, dtype=np.int32)
        cfk = np.ascontiguousarray(np.asarray(mesh.cf_tets, dtype=np.int32).reshape(-1, 2))
        tri = np.ascontiguousarray(mesh.triangle_coords(), dtype=np.float64).reshape(-1, 9)
        if pts.ndim != 2 or pts.shape[1] != 3 or sv.shape != (len(sv), 4) or sn.shape != sv.shape:
            raise ValueError("mesh arrays have unexpected shapes")
        h = ctypes.c_void_p()
        check(
            lib.tb_mesh_create(
                self.device, code, len(pts), addr(pts), len(sv), addr(recs), addr(sv), addr(sn),
                len(cft), addr(cft), addr(cfk), len(tri), addr(tri), ctypes.byref(h),
            ),
            "tb_mesh_create",
        )
        self.handle = h
        self.source_tet = int(mesh.source_tet)
        self.n_tets = len(sv)
        self.n_points = len(pts)
        self.n_cf = len(cft)
        hbm, hot = ctypes.c_int64(), ctypes.c_int64()
        check(lib.tb_mesh_info(h, None, None, None, None, None, ctypes.byref(hbm), ctypes.byref(hot)), "tb_mesh_info")
        self.hbm_bytes = hbm.value
        self.hot_bytes = hot.value
        ok = ctypes.c_int()
        check(lib.tb_mesh_validated(h, ctypes.byref(ok)), "tb_mesh_validated")
        self.validated = bool(ok.value)
        self._finalizer = weakref.finalize(self, lib.tb_mesh_destroy, h)

    def replicate(self, device: int) -> "DeviceMesh":
        """A copy of this device mesh on ``device``, made peer to peer from HBM
        (``tb_mesh_replicate``; no host upload, no rebuild)."""
        h = ctypes.c_void_p()
        check(lib.tb_mesh_replicate(self.handle, int(device), ctypes.byref(h)), "tb_mesh_replicate")
        rep = object.__new__(DeviceMesh)
        rep.__dict__.update({k: v for k, v in self.__dict__.items() if k not in ("handle", "_finalizer")})
        rep.device = int(device)
        rep.handle = h
        rep._finalizer = weakref.finalize(rep, lib.tb_mesh_destroy, h)
        return rep

    @property
    def layout_code(self) -> int:
        return LAYOUT_CODES[self.layout]

    def close(self) -> None:
        """Free the device copy now; later calls through this object fail
        loudly (NULL handle) instead of touching freed memory."""
        self._finalizer()
        self.handle = ctypes.c_void_p()


def _mirrored(mesh) -> tuple:
    """The host arrays a device copy is built from."""
    return (mesh.points, mesh.records, mesh.side_verts, mesh.side_neighbors, mesh.cf_triangle, mesh.cf_tets,
            mesh.soup.vertices, mesh.soup.triangles)


def _fingerprint(arrs, layout) -> tuple:
    return tuple((id(a), a.shape) for a in arrs) + (layout,)


class _Entry:
    """A cached upload: the device mesh, its fingerprint, the mirrored arrays
    (kept alive) and their writeable flags before the cache froze them."""

    __slots__ = ("dm", "fp", "arrs", "was_writeable")

    def __init__(self, dm, fp, arrs):
        self.dm, self.fp, self.arrs = dm, fp, arrs
        self.was_writeable = []
        for a in arrs:
            w = bool(a.flags.writeable)
            self.was_writeable.append(w)
            if w:
                a.flags.writeable = False

    def thaw(self) -> None:
        """Restore writability (unless another cached copy still mirrors the array)."""
        frozen = {id(a) for e in _cache.values() if e is not self for a in e.arrs}
        for a, w in zip(self.arrs, self.was_writeable):
            if w and id(a) not in frozen:
                try:
                    a.flags.writeable = True
                except ValueError:  # a view whose base became read-only meanwhile
                    pass


_lock = threading.Lock()
_cache: dict = {}


def device_mesh(mesh, device: int | None = None, layout: str | None = None) -> DeviceMesh:
    """Cached upload of ``mesh`` (a CompactMesh or a DeviceMesh, returned as is)."""
    if isinstance(mesh, DeviceMesh):
        return mesh
    dev = default_device() if device is None else int(device)
    key = (id(mesh), layout or mesh.layout, dev)
    arrs = _mirrored(mesh)
    fp = _fingerprint(arrs, mesh.layout)
    with _lock:
        hit = _cache.get(key)
        if hit is not None and hit.fp == fp:
            return hit.dm
        if hit is not None:  # an array was replaced: the old entry's arrays are no longer the mesh's
            _cache.pop(key)
            hit.thaw()
        dm = DeviceMesh(mesh, dev, layout)
        _cache[key] = _Entry(dm, fp, arrs)
        try:
            weakref.finalize(mesh, _evict, key)
        except TypeError:
            pass
        return dm


def _evict(key) -> None:
    # the host mesh died: forget the cache entry.  The device copy itself is
    # freed by DeviceMesh's own finalizer once no caller holds it any more
    # (a caller may keep using a DeviceMesh after its host mesh is gone).
    with _lock:
        e = _cache.pop(key, None)
        if e is not None:
            e.thaw()


def invalidate(mesh) -> None:
    """Drop every cached device copy of ``mesh`` and make its arrays writeable
    again (call before mutating them in place): the next ``device_mesh(mesh)``
    uploads again.  DeviceMesh objects already handed out stay valid until
    released."""
    with _lock:
        for k in [k for k in _cache if k[0] == id(mesh)]:
            _cache.pop(k).thaw()


__all__ = ["DeviceMesh", "device_mesh", "invalidate", "default_device", "LAYOUT_CODES", "_lib"]
