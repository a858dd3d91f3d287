"""Scene and mesh ingestion: Kuhn box fixtures, TetGen filesets, OBJ soups.

Host-side mirror of the reference's ingestion layer (/root/reference/pkg/
src/tetray/ingestion.py) producing byte-identical raw meshes, vectorised so
fixture and scene construction is not the bottleneck on the GPU box.  The
constrained-face order, front/back convention and triangle association are
the reference's:
  * faces are visited in ascending sorted-vertex-triple order
    (``sorted(inc.items())``, ingestion.py:376);
  * front = the first incident (tet, slot) in tet-major order, back = the
    second or NO_TET on the hull (ingestion.py:399-401);
  * triangle ids come from ``associate_constrained_faces``
    (ingestion.py:470-529).
"""

from __future__ import annotations

import itertools
from pathlib import Path

import numpy as np

from .tetmesh import (
    BOUNDARY_REF,
    CONSTRAINED_BIT,
    NO_TET,
    MeshError,
    RawTetMesh,
    SceneTriangleSoup,
    face_incidence_arrays,
    signed_volumes,
    unpack_keys,
    validate_raw,
)


class ParseError(Exception):
    """A malformed input file: ``path``, the 1-based ``line_no`` (0 = the file
    as a whole) and the reason, formatted as ``path:line: reason``."""

    def __init__(self, path, line_no, message):
        self.path, self.line_no, self.reason = str(path), line_no, message
        super().__init__(f"{self.path}:{line_no}: {message}")


class AssociationError(Exception):
    """A constrained mesh face could not be matched to a scene triangle."""


# ---------------------------------------------------------------------------
# Kuhn box fixture (ingestion.py:309-467)

_PERMS = list(itertools.permutations((0, 1, 2)))
_FREE_AXES = {0: (1, 2), 1: (0, 2), 2: (0, 1)}


def _perm_parity(p) -> int:
    inv = sum(1 for i in range(3) for j in range(i + 1, 3) if p[i] > p[j])
    return -1 if inv % 2 else 1


def kuhn_tets(n: int) -> np.ndarray:
    """(6 n^3, 4) int32 Kuhn tets, cells in (i, j, k) C order, 6 permutations
    per cell in itertools order, vertices 1/2 swapped for odd permutations."""
    m = n + 1
    ii, jj, kk = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    c0 = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], axis=1).astype(np.int64)  # (n^3, 3)
    eye = np.eye(3, dtype=np.int64)
    stride = np.array([m * m, m, 1], dtype=np.int64)
    out = np.empty((len(c0), 6, 4), dtype=np.int64)
    for k, p in enumerate(_PERMS):
        c1 = c0 + eye[p[0]]
        c2 = c1 + eye[p[1]]
        c3 = c0 + 1
        q = [c0 @ stride, c1 @ stride, c2 @ stride, c3 @ stride]
        if _perm_parity(p) < 0:
            q[1], q[2] = q[2], q[1]
        out[:, k, :] = np.stack(q, axis=1)
    return out.reshape(-1, 4).astype(np.int32)


def _check_occluders(n, occluders):
    """Occluders as (axis, plane k, u0, v0, u1, v1): axis-aligned rectangles
    of whole cell faces on an interior lattice plane 0 < k < n."""
    checked = []
    for occ in occluders:
        axis, k, lo, hi = occ
        coords = (k, *lo, *hi)
        on_lattice = (axis in (0, 1, 2) and all(isinstance(x, (int, np.integer)) for x in coords)
                      and 0 < k < n and all(0 <= a < b <= n for a, b in zip(lo, hi)))
        if not on_lattice:
            raise ValueError(f"occluder {occ} is not on the interior cell-face lattice")
        checked.append(tuple(int(x) for x in (axis, k, lo[0], lo[1], hi[0], hi[1])))
    return checked


def _box_soup(n: int, occs, walls: str) -> SceneTriangleSoup:
    """The box scene: each wall as one quad (2 big triangles), then every
    occluder cell face as its own quad; quads split along the low->high
    diagonal, vertices numbered in order of first use."""
    quads = []  # (axis, plane, u0, v0, u1, v1, material)
    if walls == "constrained":
        quads += [(axis, plane, 0, 0, n, n, 0) for axis in range(3) for plane in (0, n)]
    for axis, k, u0, v0, u1, v1 in occs:
        quads += [(axis, k, u, w, u + 1, w + 1, 1) for u in range(u0, u1) for w in range(v0, v1)]
    if not quads:
        return SceneTriangleSoup(np.zeros((0, 3)), np.zeros((0, 3), np.int32), np.zeros(0, np.int32))
    q = np.array(quads, dtype=np.int64)
    # corners p00, p10, p11, p01 of each quad in (plane, u, v) coordinates
    uv = np.stack([q[:, [2, 3]], q[:, [4, 3]], q[:, [4, 5]], q[:, [2, 5]]], axis=1)  # (Q, 4, 2)
    free = np.array([_FREE_AXES[a] for a in range(3)])[q[:, 0]]  # (Q, 2) the in-plane axes
    corners = np.empty((len(q), 4, 3), dtype=np.float64)
    for ax in range(3):
        corners[:, :, ax] = np.where((q[:, 0] == ax)[:, None], q[:, 1:2],
                                     np.where((free[:, 0] == ax)[:, None], uv[:, :, 0], uv[:, :, 1]))
    flat = corners.reshape(-1, 3)
    uniq, first, inverse = np.unique(flat, axis=0, return_index=True, return_inverse=True)
    rank = np.empty(len(uniq), dtype=np.int64)
    rank[np.argsort(first, kind="stable")] = np.arange(len(uniq))
    ids = rank[inverse.reshape(-1)].reshape(-1, 4)
    tris = np.stack([ids[:, [0, 1, 2]], ids[:, [0, 2, 3]]], axis=1).reshape(-1, 3)
    return SceneTriangleSoup(vertices=flat[first[np.argsort(first, kind="stable")]],
                             triangles=tris.astype(np.int32), material_ids=np.repeat(q[:, 6], 2).astype(np.int32))


def build_box_fixture(n: int, occluders=(), walls: str = "constrained"):
    """n^3-cell box, 6 Kuhn tets per cell; occluder rectangles on interior
    cell-face planes and (by default) the walls become constrained faces."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if walls not in ("constrained", "open"):
        raise ValueError("walls must be 'constrained' or 'open'")
    occs = _check_occluders(n, occluders)
    m = n + 1
    ii, jj, kk = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
    points = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], axis=1).astype(np.float64)
    tets = kuhn_tets(n)
    n_points = len(points)
    keys, first, second = face_incidence_arrays(tets, n_points)
    triples = unpack_keys(keys, n_points)
    ipts = points.astype(np.int64)

    interior = second >= 0
    on_occ = np.zeros(len(keys), dtype=bool)
    if occs:
        fp = ipts[triples]  # (f, 3 pts, 3 coords)
        for axis, k, u0, v0, u1, v1 in occs:
            a, b = _FREE_AXES[axis]
            on_occ |= (
                np.all(fp[:, :, axis] == k, axis=1)
                & (fp[:, :, a].min(axis=1) >= u0)
                & (fp[:, :, a].max(axis=1) <= u1)
                & (fp[:, :, b].min(axis=1) >= v0)
                & (fp[:, :, b].max(axis=1) <= v1)
            )
    constrained = np.where(interior, on_occ, walls == "constrained")

    neighbors = np.full((len(tets), 4), BOUNDARY_REF, dtype=np.uint32)
    plain = interior & ~constrained
    t0, j0 = first[plain] // 4, first[plain] % 4
    t1, j1 = second[plain] // 4, second[plain] % 4
    neighbors[t0, j0] = t1
    neighbors[t1, j1] = t0

    soup = _box_soup(n, occs, walls)
    cidx = np.nonzero(constrained)[0]
    face_verts = triples[cidx].astype(np.int32)
    tri_ids = associate_constrained_faces(points, face_verts, soup, tolerance=0.0)
    cf_front = (first[cidx] // 4).astype(np.int32)
    cf_back = np.where(second[cidx] >= 0, second[cidx] // 4, NO_TET).astype(np.int32)
    cfn = np.arange(len(cidx), dtype=np.int64)
    neighbors[first[cidx] // 4, first[cidx] % 4] = (CONSTRAINED_BIT | cfn).astype(np.uint32)
    has2 = second[cidx] >= 0
    neighbors[second[cidx][has2] // 4, second[cidx][has2] % 4] = (CONSTRAINED_BIT | cfn[has2]).astype(np.uint32)
    raw = RawTetMesh(
        points=points,
        tets=tets,
        neighbors=neighbors,
        cf_triangle=tri_ids.astype(np.int32),
        cf_tets=np.stack([cf_front, cf_back], axis=1),
        cf_verts=face_verts,
    )
    return raw, soup


# ---------------------------------------------------------------------------
# Analytic Kuhn box (same mesh as build_box_fixture, no face sort) -- the
# big-scene builder for BASELINE config 5 (n = 203: 50,192,562 tets), which
# the reference's dict-based builder cannot construct (~60 us/tet,
# SURVEY 3.3).  Adjacency of the Kuhn simplex (c, p) with path vertices
# w0 = c, w1 = c + e_p0, w2 = w1 + e_p1, w3 = c + 1:
#   face opp. w0 -> cell c + e_p0, perm (p1, p2, p0), its new vertex is w'3
#   face opp. w3 -> cell c - e_p2, perm (p2, p0, p1), its new vertex is w'0
#   face opp. w1 -> same cell, perm (p1, p0, p2), new vertex w'1
#   face opp. w2 -> same cell, perm (p0, p2, p1), new vertex w'2
# Faces opposite w0 / w3 lie on the cell-face planes axis p0 at c[p0] + 1 /
# axis p2 at c[p2]; they are the only candidates for walls and occluders.

_PERM_INDEX = {p: i for i, p in enumerate(_PERMS)}
_PARITY = np.array([_perm_parity(p) for p in _PERMS])
_SLOT_OF_W = np.array([[0, 1, 2, 3] if _perm_parity(p) > 0 else [0, 2, 1, 3] for p in _PERMS])  # (6, 4)


def build_kuhn_box(n: int, occluders=(), walls: str = "constrained", scale=(1.0, 1.0, 1.0)):
    """Analytic restatement of build_box_fixture (identical arrays for
    scale 1, tested), optionally with axis-scaled geometry ("long thin"
    tets and scene triangles for scale far from 1)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    if walls not in ("constrained", "open"):
        raise ValueError("walls must be 'constrained' or 'open'")
    occs = _check_occluders(n, occluders)
    m = n + 1
    n_cells = n ** 3
    n_tets = 6 * n_cells
    ax = np.arange(m, dtype=np.float64)
    ii, jj, kk = np.meshgrid(ax, ax, ax, indexing="ij")
    points = np.stack([ii.ravel() * scale[0], jj.ravel() * scale[1], kk.ravel() * scale[2]], axis=1)
    del ii, jj, kk
    tets = kuhn_tets(n)
    neighbors = np.full((n_tets, 4), BOUNDARY_REF, dtype=np.uint32)
    cell = np.arange(n_cells, dtype=np.int64)
    cc = np.stack([cell // (n * n), (cell // n) % n, cell % n], axis=1)  # (cells, 3)
    stride_c = np.array([n * n, n, 1], dtype=np.int64)
    # interior cell-face records for occluder / association handling
    cf_parts = []  # (tet, slot, other_tet, other_slot, axis, plane, u, v, middle_is_first)
    for k, p in enumerate(_PERMS):
        t = cell * 6 + k
        slot = _SLOT_OF_W[k]
        # faces opposite w1 / w2: same cell, other permutations
        for q, pn, qn in ((1, (p[1], p[0], p[2]), 1), (2, (p[0], p[2], p[1]), 2)):
            kn = _PERM_INDEX[pn]
            neighbors[t, slot[q]] = (cell * 6 + kn).astype(np.uint32)
        # face opposite w0: cell + e_p0 (perm (p1, p2, p0), new vertex w'3)
        inside = cc[:, p[0]] < n - 1
        kn = _PERM_INDEX[(p[1], p[2], p[0])]
        tn = (cell + stride_c[p[0]]) * 6 + kn
        neighbors[t[inside], slot[0]] = tn[inside].astype(np.uint32)
        cf_parts.append(("w0", k, p, t, slot[0], inside, tn, _SLOT_OF_W[kn][3]))
        # face opposite w3: cell - e_p2 (perm (p2, p0, p1), new vertex w'0)
        inside3 = cc[:, p[2]] > 0
        kn3 = _PERM_INDEX[(p[2], p[0], p[1])]
        tn3 = (cell - stride_c[p[2]]) * 6 + kn3
        neighbors[t[inside3], slot[3]] = tn3[inside3].astype(np.uint32)
        cf_parts.append(("w3", k, p, t, slot[3], inside3, tn3, _SLOT_OF_W[kn3][0]))

    # constrained faces: collect (tet, slot, partner tet/slot or -1, plane info)
    rec_t, rec_s, rec_t2, rec_s2, rec_axis, rec_plane, rec_u, rec_v, rec_mid = ([] for _ in range(9))
    for kind, k, p, t, sl, inside, tn, sln in cf_parts:
        if kind == "w0":
            axis, plane = p[0], cc[:, p[0]] + 1
            mid_axis = p[1]  # in-plane step of the middle vertex w2 - w1
        else:
            axis, plane = p[2], cc[:, p[2]]
            mid_axis = p[0]  # w1 - w0
        a1, a2 = _FREE_AXES[axis]
        u, v = cc[:, a1], cc[:, a2]
        sel = np.zeros(n_cells, dtype=bool)
        # hull faces (walls)
        if walls == "constrained":
            sel |= ~inside
        # occluder faces (interior); each is reached from both sides, keep the
        # w0 side (lower cell) once and attach the partner
        occ_hit = np.zeros(n_cells, dtype=bool)
        if occs and kind == "w0":
            for oa, ok_, u0, v0, u1, v1 in occs:
                if oa != axis:
                    continue
                occ_hit |= inside & (plane == ok_) & (u >= u0) & (u + 1 <= u1) & (v >= v0) & (v + 1 <= v1)
        if kind == "w3":
            sel &= ~inside  # interior w3 faces are the partners of w0 faces
        sel |= occ_hit
        idx = np.nonzero(sel)[0]
        if not idx.size:
            continue
        rec_t.append(t[idx])
        rec_s.append(np.full(idx.size, sl))
        two = inside[idx]
        rec_t2.append(np.where(two, tn[idx], -1))
        rec_s2.append(np.where(two, sln, -1))
        rec_axis.append(np.full(idx.size, axis))
        rec_plane.append(plane[idx])
        rec_u.append(u[idx])
        rec_v.append(v[idx])
        rec_mid.append(np.full(idx.size, mid_axis == a1))  # middle vertex is p10 (else p01)
    if rec_t:
        ft = np.concatenate(rec_t)
        fs = np.concatenate(rec_s)
        ft2 = np.concatenate(rec_t2)
        fs2 = np.concatenate(rec_s2)
        faxis = np.concatenate(rec_axis)
        fplane = np.concatenate(rec_plane)
        fu = np.concatenate(rec_u)
        fv = np.concatenate(rec_v)
        fmid = np.concatenate(rec_mid)
    else:
        ft = fs = ft2 = fs2 = faxis = fplane = fu = fv = np.zeros(0, np.int64)
        fmid = np.zeros(0, bool)
    # face keys: sorted vertex triples (reference order: sorted(inc.items()))
    tri_v = np.sort(tets[ft][:, _OTHER_SLOTS][np.arange(len(ft)), fs], axis=1).astype(np.int64)
    order = np.lexsort((tri_v[:, 2], tri_v[:, 1], tri_v[:, 0]))
    ft, fs, ft2, fs2, faxis, fplane, fu, fv, fmid, tri_v = (a[order] for a in
                                                             (ft, fs, ft2, fs2, faxis, fplane, fu, fv, fmid, tri_v))
    # front = lower tet id (first in tet-major incidence order)
    swap = (ft2 >= 0) & (ft2 < ft)
    front = np.where(swap, ft2, ft)
    fslot = np.where(swap, fs2, fs)
    back = np.where(swap, ft, ft2)
    bslot = np.where(swap, fs, fs2)
    cfn = np.arange(len(front), dtype=np.int64)
    neighbors[front, fslot] = (CONSTRAINED_BIT | cfn).astype(np.uint32)
    h2 = back >= 0
    neighbors[back[h2], bslot[h2]] = (CONSTRAINED_BIT | cfn[h2]).astype(np.uint32)

    soup = _box_soup(n, occs, walls)
    if scale != (1.0, 1.0, 1.0):
        soup = SceneTriangleSoup(vertices=soup.vertices * np.asarray(scale, dtype=np.float64),
                                 triangles=soup.triangles, material_ids=soup.material_ids)
    # analytic association: walls (2 triangles each, split along u = v) first,
    # then per-cell occluder squares (2 triangles each), reference order
    tri_id = np.full(len(front), -1, dtype=np.int64)
    wall_base = 0
    n_wall_tris = 12 if walls == "constrained" else 0
    hull = back < 0
    if walls == "constrained":
        wall = faxis * 2 + (fplane == n)
        upper = np.where(fmid, fv >= fu + 1, fv >= fu)  # triangle (p00, p11, p01) side
        tri_id[hull] = (wall_base + 2 * wall + upper)[hull]
    if occs:
        base = n_wall_tris
        claimed = np.zeros(len(front), dtype=np.int64)
        for oa, ok_, u0, v0, u1, v1 in occs:
            on = (~hull) & (faxis == oa) & (fplane == ok_) & (fu >= u0) & (fu + 1 <= u1) & (fv >= v0) & (fv + 1 <= v1)
            cell_idx = (fu - u0) * (v1 - v0) + (fv - v0)
            tri_id[on] = base + 2 * cell_idx[on] + (~fmid[on]).astype(np.int64)
            claimed += on
            base += 2 * (u1 - u0) * (v1 - v0)
        if np.any(claimed > 1):
            f = int(np.nonzero(claimed > 1)[0][0])
            raise AssociationError(f"face {points[tri_v[f]].tolist()} matched {int(claimed[f])} scene triangles")
    if np.any(tri_id < 0):
        raise AssociationError("constrained face without a scene triangle")
    raw = RawTetMesh(
        points=points,
        tets=tets,
        neighbors=neighbors,
        cf_triangle=tri_id.astype(np.int32),
        cf_tets=np.stack([front, np.where(back >= 0, back, NO_TET)], axis=1).astype(np.int32),
        cf_verts=tri_v.astype(np.int32),
    )
    return raw, soup


_OTHER_SLOTS = np.array([[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]])


# ---------------------------------------------------------------------------
# Face -> scene triangle association (ingestion.py:470-538), vectorised.


def _inside_2d(t2, area, q, tol):
    """Edge tests of ingestion._inside_2d, broadcast over leading axes."""
    s = np.where(area > 0, 1.0, -1.0)
    slack = tol * (np.abs(area) + 1.0)
    ok = np.ones(np.broadcast_shapes(area.shape, q.shape[:-1]), dtype=bool)
    for i in range(3):
        a = t2[..., i, :]
        b = t2[..., (i + 1) % 3, :]
        e = ((b[..., 0] - a[..., 0]) * (q[..., 1] - a[..., 1]) - (b[..., 1] - a[..., 1]) * (q[..., 0] - a[..., 0])) * s
        ok &= ~(e < -slack)
    return ok


def _projection_frames(tri):
    """Per scene triangle: unit normal, the two axes kept when projecting
    along its dominant normal axis, its projected corners and twice its
    signed projected area."""
    u = tri[:, 1] - tri[:, 0]
    v = tri[:, 2] - tri[:, 0]
    normal = np.cross(u, v)
    length = np.sqrt((normal * normal).sum(axis=1))
    if not np.all(length > 0):
        raise AssociationError("degenerate scene triangle")
    keep = np.array([[1, 2], [0, 2], [0, 1]])[np.abs(normal).argmax(axis=1)]  # (T, 2)
    uk = np.take_along_axis(u, keep, axis=1)
    vk = np.take_along_axis(v, keep, axis=1)
    tri2 = np.take_along_axis(tri, keep[:, None, :], axis=2)  # (T, 3, 2)
    return normal / length[:, None], keep, tri2, uk[:, 0] * vk[:, 1] - uk[:, 1] * vk[:, 0]


def associate_constrained_faces(points, face_verts, soup: SceneTriangleSoup, tolerance: float = 1e-9) -> np.ndarray:
    """Scene triangle containing each constrained face (coplanar within
    tolerance, all three vertices inside; ties broken by strict containment
    of the centroid)."""
    points = np.asarray(points, dtype=np.float64)
    face_verts = np.asarray(face_verts, dtype=np.int64).reshape(-1, 3)
    tri = soup.triangle_coords()
    if len(tri) == 0:
        if len(face_verts):
            raise AssociationError("scene has no triangles")
        return np.zeros(0, dtype=np.int32)
    n_hat, keep, tri2, area2 = _projection_frames(tri)
    T = len(tri)
    out = np.empty(len(face_verts), dtype=np.int32)
    chunk = max(1, 2_000_000 // (3 * T))
    for lo in range(0, len(face_verts), chunk):
        ids = face_verts[lo : lo + chunk]
        pts = points[ids]  # (F, 3, 3)
        cen = pts.mean(axis=1)  # (F, 3)
        rel = pts[:, None, :, :] - tri[None, :, 0, None, :]  # (F, T, 3, 3)
        dist = np.abs(np.einsum("tj,ftpj->ftp", n_hat, rel))
        coplanar = dist.max(axis=2) <= tolerance + 1e-300  # (F, T)
        # 2-D coordinates of the face vertices in each triangle's kept axes
        q = np.take_along_axis(pts[:, None, :, :], keep[None, :, None, :], axis=3)  # (F, T, 3, 2)
        inside = np.ones(coplanar.shape, dtype=bool)
        for p in range(3):
            inside &= _inside_2d(tri2[None], area2[None], q[:, :, p, :], tolerance)
        match = coplanar & inside
        cnt = match.sum(axis=1)
        qc = np.take_along_axis(cen[:, None, :], keep[None, :, :], axis=2)  # (F, T, 2)
        strict = match & _inside_2d(tri2[None], area2[None], qc, -tolerance)
        scnt = strict.sum(axis=1)
        use_strict = (cnt > 1) & (scnt == 1)
        final = np.where(use_strict[:, None], strict, match)
        fcnt = final.sum(axis=1)
        if np.any(fcnt != 1):
            f = int(np.nonzero(fcnt != 1)[0][0])
            if cnt[f] == 0 and not coplanar[f].any():
                raise AssociationError(f"face {pts[f].tolist()} is not coplanar with any triangle")
            raise AssociationError(f"face {pts[f].tolist()} matched {int(fcnt[f])} scene triangles")
        out[lo : lo + len(ids)] = np.argmax(final, axis=1)
    return out


# ---------------------------------------------------------------------------
# TetGen / OBJ (ingestion.py:87-288)


def _records(path):
    """(line number, tokens) of the non-blank lines of a TetGen file, with
    '#' comments stripped."""
    with open(path) as fh:
        for line_no, line in enumerate(fh, start=1):
            toks = line.partition("#")[0].split()
            if toks:
                yield line_no, toks


def _read_rows(path, min_cols, what):
    """A TetGen table: its header line and the data rows after it."""
    it = _records(path)
    header = next(it, None)
    if header is None:
        raise ParseError(path, 0, f"{what}: empty file")
    rows = list(it)
    short = [ln for ln, toks in rows if len(toks) < min_cols]
    if short:
        raise ParseError(path, short[0], f"{what}: expected >= {min_cols} fields")
    return header, rows


def parse_tetgen(base) -> RawTetMesh:
    """TetGen ASCII fileset -> RawTetMesh (ingestion.py:87-177 semantics):
    auto 0/1 index base, marked .face entries become constrained faces (in
    file order), .neigh -1 -> boundary, negative tets reoriented by swapping
    slots 1 and 2."""
    base = str(base)
    if base.endswith(".node"):
        base = base[: -len(".node")]
    node, ele, neigh, face = (Path(base + e) for e in (".node", ".ele", ".neigh", ".face"))
    (hl, ht), rows = _read_rows(node, 4, "node")
    n_points = int(ht[0])
    if int(ht[1]) != 3:
        raise ParseError(node, hl, f"dimension {ht[1]} != 3")
    if len(rows) != n_points:
        raise ParseError(node, hl, f"{len(rows)} nodes, header says {n_points}")
    ib = int(rows[0][1][0]) if rows else 0
    if ib not in (0, 1):
        raise ParseError(node, rows[0][0], f"first node index {ib}, expected 0 or 1")
    idx = np.array([int(t[0]) for _, t in rows], dtype=np.int64) - ib
    if not np.array_equal(idx, np.arange(n_points)):
        k = int(np.nonzero(idx != np.arange(n_points))[0][0])
        raise ParseError(node, rows[k][0], f"non-sequential node index {rows[k][1][0]}")
    points = np.array([[float(t[1]), float(t[2]), float(t[3])] for _, t in rows], dtype=np.float64).reshape(-1, 3)
    (hl, ht), rows = _read_rows(ele, 5, "ele")
    n_tets = int(ht[0])
    if len(rows) != n_tets:
        raise ParseError(ele, hl, f"{len(rows)} tets, header says {n_tets}")
    tets = (np.array([[int(x) for x in t[1:5]] for _, t in rows], dtype=np.int64).reshape(-1, 4) - ib).astype(np.int32)
    if len(tets) and (tets.min() < 0 or tets.max() >= n_points):
        k = int(np.nonzero((tets < 0).any(1) | (tets >= n_points).any(1))[0][0])
        raise ParseError(ele, rows[k][0], "vertex index out of range")
    (hl, ht), rows = _read_rows(neigh, 5, "neigh")
    if int(ht[0]) != n_tets or len(rows) != n_tets:
        raise ParseError(neigh, hl, "neighbor count does not match .ele")
    nb = np.array([[int(x) for x in t[1:5]] for _, t in rows], dtype=np.int64).reshape(-1, 4)
    nb[nb >= 0] -= ib
    if nb.max(initial=-1) >= n_tets:
        raise ParseError(neigh, 0, "neighbor index out of range")
    faces = []
    if face.exists():
        (hl, ht), rows = _read_rows(face, 4, "face")
        if len(rows) != int(ht[0]):
            raise ParseError(face, hl, f"{len(rows)} faces, header says {ht[0]}")
        for line_no, t in rows:
            corners = tuple(int(x) - ib for x in t[1:4])
            marker = int(t[4]) if len(t) > 4 else 1
            if min(corners) < 0 or max(corners) >= n_points:
                raise ParseError(face, line_no, "face corner out of range")
            if marker != 0:
                faces.append(corners)
    flip = np.nonzero(signed_volumes(points, tets) < 0)[0]
    tets[flip[:, None], [1, 2]] = tets[flip[:, None], [2, 1]]
    nb[flip[:, None], [1, 2]] = nb[flip[:, None], [2, 1]]
    refs = np.where(nb < 0, np.int64(BOUNDARY_REF), nb).astype(np.uint32)
    raw = RawTetMesh(points=points, tets=tets, neighbors=refs)
    if faces:
        mark_constrained(raw, np.asarray(faces, dtype=np.int64), face)
    problems = validate_raw(raw)
    if problems:
        raise ParseError(neigh, 0, "; ".join(problems[:5]))
    return raw


def mark_constrained(raw: RawTetMesh, face_triples, face_path="<faces>") -> None:
    """Tag the given faces (in order) as constrained faces 0..k-1
    (ingestion._mark_constrained, ingestion.py:191-207)."""
    keys_sorted = np.sort(np.asarray(face_triples, dtype=np.int64), axis=1)
    ukeys, first, second = face_incidence_arrays(raw.tets, raw.n_points)
    from .tetmesh import pack_keys

    want = pack_keys(keys_sorted, raw.n_points)
    pos = np.searchsorted(ukeys, want)
    pos_c = np.minimum(pos, len(ukeys) - 1)
    found = ukeys[pos_c] == want
    if not found.all():
        k = int(np.nonzero(~found)[0][0])
        raise ParseError(face_path, 0, f"marked face {tuple(face_triples[k])} is not a mesh face")
    f1, f2 = first[pos_c], second[pos_c]
    c = np.arange(len(want), dtype=np.int64)
    raw.neighbors[f1 // 4, f1 % 4] = (CONSTRAINED_BIT | c).astype(np.uint32)
    h2 = f2 >= 0
    raw.neighbors[f2[h2] // 4, f2[h2] % 4] = (CONSTRAINED_BIT | c[h2]).astype(np.uint32)
    raw.cf_triangle = c.astype(np.int32)
    raw.cf_tets = np.stack([f1 // 4, np.where(h2, f2 // 4, NO_TET)], axis=1).astype(np.int32)
    raw.cf_verts = keys_sorted.astype(np.int32)


def _obj_index(tok: str, n_verts: int) -> int:
    """0-based vertex of an OBJ face token ("i", "i/t", "i/t/n"; i < 0 counts back)."""
    i = int(tok.split("/", 1)[0])
    return i - 1 if i > 0 else n_verts + i


def load_obj(path) -> SceneTriangleSoup:
    """The triangles of an OBJ file (``v`` / ``f`` records, polygons fanned
    from their first corner, 1-based or negative indices)."""
    verts: list = []
    tris: list = []
    with open(path) as fh:
        for line_no, line in enumerate(fh, start=1):
            kind, *args = line.split() or ["#"]
            if kind == "v":
                if len(args) < 3:
                    raise ParseError(path, line_no, "vertex needs 3 coordinates")
                verts.append(tuple(float(x) for x in args[:3]))
            elif kind == "f":
                if len(args) < 3:
                    raise ParseError(path, line_no, "face needs >= 3 vertices")
                corner = [_obj_index(a, len(verts)) for a in args]
                if not all(0 <= c < len(verts) for c in corner):
                    raise ParseError(path, line_no, "face index out of range")
                tris += [(corner[0], corner[k], corner[k + 1]) for k in range(1, len(corner) - 1)]
    vertices = np.array(verts, dtype=np.float64).reshape(-1, 3)
    triangles = np.array(tris, dtype=np.int32).reshape(-1, 3)
    corners = vertices[triangles]
    if len(triangles) and not np.all(np.cross(corners[:, 1] - corners[:, 0], corners[:, 2] - corners[:, 0]).any(axis=1)):
        raise ParseError(path, 0, "degenerate (zero-area) triangle in file")
    return SceneTriangleSoup(vertices=vertices, triangles=triangles, material_ids=np.zeros(len(triangles), np.int32))


__all__ = [
    "AssociationError",
    "MeshError",
    "ParseError",
    "associate_constrained_faces",
    "build_box_fixture",
    "kuhn_tets",
    "load_obj",
    "mark_constrained",
    "parse_tetgen",
]
