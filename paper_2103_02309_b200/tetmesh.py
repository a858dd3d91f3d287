"""The compact tetrahedral mesh the GPU walks, and how it is built on the host.

API-compatible with the reference's mesh layer (``tetray.tetmesh``): the
same class names, attribute names, record dtypes and array conventions, so
a ``CompactMesh`` built here equals the reference's byte for byte (pinned by
the digest tests) and the reference's own meshes plug into this package.
The construction itself is this package's: the per-tet work (sorted-slot side
tables, record packing, reorder remapping, Hilbert keys, centroids) runs in
native host code (``csrc/host_mesh.cpp``), the checks are whole-array numpy.

Records (tetmesh.py:34-46), slot j = the tet's j-th smallest vertex id:

    tet32  v0 v1 v2 vx | n0 n1 n2 n3      32 B
    tet20  vx | n0 n1 n2 n3               20 B
    tet16  vx | n0^n3 n1^n3 n2^n3         16 B     (vx = v0^v1^v2^v3)

A neighbour reference n_j is a uint32: a tet index, or the boundary sentinel
0x7FFFFFFF, or 0x80000000 | c for constrained (scene) face c (tetmesh.py:
29-32).  TetMesh-80 exists on the device only (built from the side tables).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from . import hilbert as _hilbert
from ._lib import addr, check, lib

# --- layouts and reference encoding ---------------------------------------

TET32, TET20, TET16 = "tet32", "tet20", "tet16"
LAYOUTS = (TET32, TET20, TET16)
LAYOUT_BYTES = {TET32: 32, TET20: 20, TET16: 16}
LAYOUT_CODES = dict(LAYOUT_BYTES)
_FIELDS = {
    TET32: ("v0", "v1", "v2", "vx", "n0", "n1", "n2", "n3"),
    TET20: ("vx", "n0", "n1", "n2", "n3"),
    TET16: ("vx", "nx0", "nx1", "nx2"),
}
LAYOUT_DTYPES = {name: np.dtype([(f, "<u4") for f in fields]) for name, fields in _FIELDS.items()}
TET32_DTYPE, TET20_DTYPE, TET16_DTYPE = (LAYOUT_DTYPES[k] for k in LAYOUTS)

CONSTRAINED_BIT = 0x80000000
REF_PAYLOAD_MASK = 0x7FFFFFFF
BOUNDARY_REF = REF_PAYLOAD_MASK
NO_TET = -1


def face_ref(cf_index: int) -> int:
    """The reference a tet stores for constrained face ``cf_index``."""
    return int(cf_index) | CONSTRAINED_BIT


def is_constrained(ref: int) -> bool:
    return (int(ref) & CONSTRAINED_BIT) != 0


def is_boundary(ref: int) -> bool:
    return int(ref) == BOUNDARY_REF


def ref_payload(ref: int) -> int:
    return int(ref) & REF_PAYLOAD_MASK


def decode_ref(ref: int) -> int:
    """Neighbour tet of a plain reference; -1 for boundary / constrained."""
    return -1 if (is_constrained(ref) or is_boundary(ref)) else int(ref)


def compute_xor_sum(v0: int, v1: int, v2: int, v3: int) -> int:
    return int(v0) ^ int(v1) ^ int(v2) ^ int(v3)


def recover_fourth_vertex(v0: int, v1: int, v2: int, vx: int) -> int:
    """The vertex a face (v0, v1, v2) lacks, from the tet's xor word."""
    return compute_xor_sum(v0, v1, v2, vx)


def _ref_classes(refs: np.ndarray):
    """(plain, constrained, boundary) masks of a uint32 reference array."""
    r = np.asarray(refs).astype(np.int64)
    constrained = (r & CONSTRAINED_BIT) != 0
    boundary = r == BOUNDARY_REF
    return ~(constrained | boundary), constrained, boundary


class MeshError(Exception):
    """Mesh data that violates the compact-mesh invariants."""


# --- containers -------------------------------------------------------------


@dataclass
class ConstrainedFace:
    """One mesh face lying on scene geometry (tetmesh.py:93-104)."""

    triangle_id: int
    tet_front: int
    tet_back: int
    vertex_ids: tuple


@dataclass
class SceneTriangleSoup:
    """The scene triangles the constrained faces carry (fp64 vertices)."""

    vertices: np.ndarray
    triangles: np.ndarray
    material_ids: np.ndarray

    @property
    def n_triangles(self) -> int:
        return len(self.triangles)

    def triangle_coords(self) -> np.ndarray:
        """(t, 3, 3) float64 corner coordinates."""
        return self.vertices[self.triangles]


@dataclass
class RawTetMesh:
    """A mesh before compact encoding (tetmesh.py:124-144): ``tets`` (t, 4)
    vertex ids in any slot order, ``neighbors[i, j]`` the reference across
    the face opposite ``tets[i, j]``.  Constrained faces are parallel arrays
    (triangle, [front, back] tets, vertex triple); ``constrained_faces``
    returns the reference's list-of-records view."""

    points: np.ndarray
    tets: np.ndarray
    neighbors: np.ndarray
    cf_triangle: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    cf_tets: np.ndarray = field(default_factory=lambda: np.zeros((0, 2), np.int32))
    cf_verts: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), np.int32))
    source_tet: int = 0

    n_tets = property(lambda self: len(self.tets))
    n_points = property(lambda self: len(self.points))

    @property
    def constrained_faces(self) -> list:
        rows = zip(self.cf_triangle.tolist(), np.asarray(self.cf_tets).tolist(), np.asarray(self.cf_verts).tolist())
        return [ConstrainedFace(tri, ft[0], ft[1], tuple(vs)) for tri, ft, vs in rows]


@dataclass
class CompactMesh:
    """The encoded mesh (tetmesh.py:147-195): hot ``records`` + float32
    ``points`` (what a walk step reads), sorted-slot side tables (ray init,
    point location), constrained-face tables and the scene soup (epilogue)."""

    layout: str
    points: np.ndarray
    records: np.ndarray
    side_verts: np.ndarray
    side_neighbors: np.ndarray
    cf_triangle: np.ndarray
    cf_tets: np.ndarray
    cf_verts: np.ndarray
    source_tet: int
    soup: SceneTriangleSoup

    n_tets = property(lambda self: len(self.side_verts))
    n_points = property(lambda self: len(self.points))
    n_constrained = property(lambda self: len(self.cf_triangle))
    record_bytes = property(lambda self: LAYOUT_BYTES[self.layout])

    @property
    def accelerator_bytes(self) -> int:
        """Bytes of the structure a traversal step touches (records + points)."""
        return int(self.records.nbytes + self.points.nbytes)

    def records_u32(self) -> np.ndarray:
        """The records as an (n_tets, words) uint32 view."""
        return self.records.view("<u4").reshape(len(self.side_verts), -1)

    def triangle_coords(self) -> np.ndarray:
        return self.soup.triangle_coords()


def soup_from_faces(points: np.ndarray, face_verts: np.ndarray) -> SceneTriangleSoup:
    """A soup whose triangles are the given mesh faces (material 0)."""
    tris = np.array(face_verts, dtype=np.int32)
    return SceneTriangleSoup(np.array(points, dtype=np.float64), tris, np.zeros(len(tris), np.int32))


# --- native builders ------------------------------------------------------


def _side_tables(verts, refs, *, rows=None, vert_map=None, tet_map=None):
    """Sorted-slot side tables (row i from row ``rows[i]``, ids remapped), in
    one native pass: stable slot sort by vertex id, references alongside."""
    v = np.ascontiguousarray(verts, dtype=np.int32)
    r = np.ascontiguousarray(refs, dtype=np.uint32)
    opt = [None if a is None else np.ascontiguousarray(a, dtype=np.int64) for a in (rows, vert_map, tet_map)]
    n = len(v) if opt[0] is None else len(opt[0])
    sv = np.empty((n, 4), dtype=np.int32)
    sn = np.empty((n, 4), dtype=np.uint32)
    if n:
        check(lib.tb_build_side_tables(n, addr(v), addr(r), addr(opt[0]), addr(opt[1]),
                                       0 if opt[1] is None else len(opt[1]), addr(opt[2]),
                                       0 if opt[2] is None else len(opt[2]), addr(sv), addr(sn)),
              "tb_build_side_tables")
    return sv, sn


def _records_from_tables(layout: str, side_verts: np.ndarray, side_neighbors: np.ndarray) -> np.ndarray:
    """Records of ``layout`` packed from the side tables (tetmesh.py:299-320)."""
    if layout not in LAYOUT_DTYPES:
        raise ValueError(f"unknown layout {layout!r}")
    sv = np.ascontiguousarray(side_verts, dtype=np.int32)
    sn = np.ascontiguousarray(side_neighbors, dtype=np.uint32)
    words = np.empty((len(sv), LAYOUT_BYTES[layout] // 4), dtype=np.uint32)
    if len(sv):
        check(lib.tb_pack_records(LAYOUT_BYTES[layout], len(sv), addr(sv), addr(sn), addr(words)),
              "tb_pack_records")
    return words.view(LAYOUT_DTYPES[layout]).reshape(-1)


def row_argsort4(a: np.ndarray) -> np.ndarray:
    """Stable per-row argsort of an (n, 4) integer array."""
    a = np.asarray(a, dtype=np.int64)
    # stable: sort by (value, original slot)
    keyed = a * 4 + np.arange(4)
    return np.argsort(keyed, axis=1)


def signed_volumes(points: np.ndarray, tets: np.ndarray) -> np.ndarray:
    """6x signed volume of each tet, float64 (the reference's einsum/cross form)."""
    corners = np.asarray(points, dtype=np.float64)[np.asarray(tets)]
    edges = corners[:, 1:] - corners[:, :1]
    return np.einsum("ij,ij->i", edges[:, 0], np.cross(edges[:, 1], edges[:, 2]))


# --- faces as sortable keys (incidence without dicts) ----------------------

_FACE_SLOTS = np.array([[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]])


def face_triples(tets: np.ndarray) -> np.ndarray:
    """(t, 4, 3): the sorted vertex triple of the face opposite each slot."""
    return np.sort(np.asarray(tets, dtype=np.int64)[:, _FACE_SLOTS], axis=2)


def pack_keys(triples: np.ndarray, n_points: int) -> np.ndarray:
    """One int64 per sorted triple, ordered like the triples themselves."""
    if int(n_points) >= 1 << 21:
        raise ValueError("meshes with >= 2**21 points need the native builder")
    radix = np.int64(max(int(n_points), 1))
    t = np.asarray(triples, dtype=np.int64)
    return (t[..., 0] * radix + t[..., 1]) * radix + t[..., 2]


def unpack_keys(keys: np.ndarray, n_points: int) -> np.ndarray:
    radix = np.int64(max(int(n_points), 1))
    k = np.asarray(keys, dtype=np.int64)
    hi, lo = np.divmod(k, radix)
    a, mid = np.divmod(hi, radix)
    return np.stack([a, mid, lo], axis=1)


def face_incidence_arrays(tets: np.ndarray, n_points: int):
    """Unique faces in ascending key order (the reference's sorted incidence
    map): (keys, first, second) where first/second encode the incident
    (tet, slot) as 4*tet + slot in tet-major order, second -1 on the hull."""
    keys = pack_keys(face_triples(tets), n_points).ravel()
    order = np.argsort(keys, kind="stable")  # ties stay in (tet, slot) order
    k_sorted = keys[order]
    head = np.flatnonzero(np.r_[True, k_sorted[1:] != k_sorted[:-1]])
    mult = np.diff(np.r_[head, len(k_sorted)])
    if len(mult) and mult.max() > 2:
        raise MeshError("face shared by more than two tetrahedra")
    first = order[head]
    nxt = np.minimum(head + 1, len(order) - 1)
    second = np.where(mult == 2, order[nxt], -1)
    return k_sorted[head], first, second


# --- checks -----------------------------------------------------------------


def validate_raw(raw: RawTetMesh) -> list[str]:
    """Structural problems of a raw mesh (the checks of tetmesh.py:216-296)."""
    tets = np.asarray(raw.tets, dtype=np.int64)
    refs = np.asarray(raw.neighbors, dtype=np.int64)
    nt = len(tets)
    if tets.size and (tets.min() < 0 or tets.max() >= raw.n_points):
        return ["vertex index out of range"]
    vol = signed_volumes(raw.points, tets)
    out = [f"tet {t}: non-positive volume {vol[t]:g}" for t in np.flatnonzero(vol <= 0)[:10]]
    srt = np.sort(tets, axis=1)
    dup = (srt[:, 1:] == srt[:, :-1]).any(axis=1)
    out += [f"tet {t}: repeated vertex" for t in np.flatnonzero(dup)[:10]]
    good = ~dup
    plain, constrained, _ = _ref_classes(refs)
    faces = face_triples(tets)
    cf_tets = np.asarray(raw.cf_tets, dtype=np.int64).reshape(-1, 2)
    cf_faces = np.sort(np.asarray(raw.cf_verts, dtype=np.int64).reshape(-1, 3), axis=1)
    n_cf = len(raw.cf_triangle)

    t_c, s_c = np.nonzero(constrained & good[:, None])
    if t_c.size:
        c = refs[t_c, s_c] & REF_PAYLOAD_MASK
        oob = c >= n_cf
        out += [f"tet {t}: constrained ref out of range" for t in t_c[oob][:5]]
        t_c, s_c, c = t_c[~oob], s_c[~oob], c[~oob]
        wrong = (cf_faces[c] != faces[t_c, s_c]).any(axis=1)
        out += [f"tet {t} slot {j}: constrained face {k} vertex mismatch"
                for t, j, k in list(zip(t_c[wrong], s_c[wrong], c[wrong]))[:5]]
        unlisted = (cf_tets[c, 0] != t_c) & (cf_tets[c, 1] != t_c)
        out += [f"tet {t} slot {j}: constrained face {k} does not list it"
                for t, j, k in list(zip(t_c[unlisted], s_c[unlisted], c[unlisted]))[:5]]

    t_p, s_p = np.nonzero(plain & good[:, None])
    if t_p.size:
        nb = refs[t_p, s_p] & REF_PAYLOAD_MASK
        oob = nb >= nt
        out += [f"tet {t}: neighbor index out of range" for t in t_p[oob][:5]]
        t_p, s_p, nb = t_p[~oob], s_p[~oob], nb[~oob]
        face = faces[t_p, s_p]
        shares = (face[:, :, None] == tets[nb][:, None, :]).any(axis=2).all(axis=1)
        out += [f"tet {t} / neighbor {o}: face vertices not shared" for t, o in list(zip(t_p[~shares], nb[~shares]))[:5]]
        back = refs[nb]
        back_plain, _, _ = _ref_classes(back)
        mutual = (back_plain & ((back & REF_PAYLOAD_MASK) == t_p[:, None])).any(axis=1)
        out += [f"adjacency not mutual between tets {t} and {o}" for t, o in list(zip(t_p[~mutual], nb[~mutual]))[:5]]

    if n_cf:
        seen = np.zeros(n_cf, dtype=np.int64)
        for side in (0, 1):
            tt = cf_tets[:, side]
            live = tt != NO_TET
            bad = live & ((tt < 0) | (tt >= nt))
            out += [f"constrained face {c}: tet {tt[c]} out of range" for c in np.flatnonzero(bad)[:5]]
            ok = np.flatnonzero(live & ~bad)
            row = refs[tt[ok]]
            _, rc, _ = _ref_classes(row)
            seen[ok] += (rc & ((row & REF_PAYLOAD_MASK) == ok[:, None])).any(axis=1)
        want = np.where(cf_tets[:, 1] == NO_TET, 1, 2)
        out += [f"constrained face {c}: referenced by {seen[c]} tets, expected {want[c]}"
                for c in np.flatnonzero(seen != want)[:5]]
    if not 0 <= raw.source_tet < nt:
        out.append(f"source tet {raw.source_tet} out of range")
    return out


def validate(mesh: CompactMesh) -> list[str]:
    """Integrity report of a compact mesh (the checks of tetmesh.py:521-640):
    records against the side tables, the raw-mesh invariants on the sorted
    tables, zero volumes after float32 quantization, and that every tet is
    reachable from the source by xor-link walking."""
    out: list[str] = []
    rec = mesh.records
    if rec.dtype.itemsize != LAYOUT_BYTES[mesh.layout]:
        out.append(f"record size {rec.dtype.itemsize} != {LAYOUT_BYTES[mesh.layout]}")
    sv = mesh.side_verts
    unsorted = (np.diff(sv, axis=1) <= 0).any(axis=1)
    if unsorted.any():
        out.append(f"tet {int(np.argmax(unsorted))}: side-table vertices not strictly ascending")
    expect = _records_from_tables(mesh.layout, sv, mesh.side_neighbors)
    out += [f"tet {t}: xor-sum mismatch" for t in np.flatnonzero(rec["vx"] != expect["vx"])[:10]]
    labels = {"v": "stored vertex v{j} mismatch", "n": "neighbor slot {j} violates sorted-slot order",
              "nx": "xor link nx{j} mismatch"}
    for name in LAYOUT_DTYPES[mesh.layout].names:
        if name == "vx":
            continue
        kind, j = name.rstrip("0123456789"), name[-1]
        out += [f"tet {t}: " + labels[kind].format(j=j) for t in np.flatnonzero(rec[name] != expect[name])[:5]]
    as_raw = RawTetMesh(mesh.points.astype(np.float64), sv, mesh.side_neighbors, mesh.cf_triangle, mesh.cf_tets,
                        mesh.cf_verts, mesh.source_tet)
    # sorted slots flip orientation, so only a zero volume is a fault here
    out += [p for p in validate_raw(as_raw) if "non-positive volume" not in p]
    vol = signed_volumes(mesh.points.astype(np.float64), sv)
    if (vol == 0).any():
        out.append(f"tet {int(np.argmax(vol == 0))}: degenerate (zero volume) after f32 quantization")
    out += _xor_walk_closure(mesh)
    return out


def _links(mesh: CompactMesh) -> np.ndarray:
    """(t, 4) neighbour tet per slot, crossing constrained faces, -1 none."""
    refs = mesh.side_neighbors.astype(np.int64)
    plain, constrained, _ = _ref_classes(refs)
    links = np.where(plain, refs & REF_PAYLOAD_MASK, -1)
    cft = np.asarray(mesh.cf_tets, dtype=np.int64).reshape(-1, 2)
    if constrained.any() and len(cft):
        t_c, s_c = np.nonzero(constrained)
        pair = cft[refs[t_c, s_c] & REF_PAYLOAD_MASK]
        links[t_c, s_c] = np.where(pair[:, 0] == t_c, pair[:, 1], pair[:, 0])
    return links


def _xor_walk_closure(mesh: CompactMesh) -> list[str]:
    """Breadth-first walk from the source over the links: each newly reached
    tet's quadruple, rebuilt from the crossed face and its xor word, must
    equal its side-table row; every tet must be reached."""
    n = mesh.n_tets
    if not 0 <= mesh.source_tet < n:
        return [f"source tet {mesh.source_tet} out of range"]
    links = _links(mesh)
    sv = mesh.side_verts.astype(np.int64)
    vx = mesh.records["vx"].astype(np.int64)
    reached = np.zeros(n, dtype=bool)
    reached[mesh.source_tet] = True
    wave = np.array([mesh.source_tet], dtype=np.int64)
    out: list[str] = []
    while wave.size:
        w_idx, slot = np.nonzero(links[wave] >= 0)
        frm, to = wave[w_idx], links[wave[w_idx], slot]
        new = ~reached[to]
        frm, to, slot = frm[new], to[new], slot[new]
        if not to.size:
            break
        to, pick = np.unique(to, return_index=True)
        frm, slot = frm[pick], slot[pick]
        face = sv[frm[:, None], _FACE_SLOTS[slot]]
        quad = np.sort(np.c_[face, np.bitwise_xor.reduce(face, axis=1) ^ vx[to]], axis=1)
        wrong = (quad != sv[to]).any(axis=1)
        out += [f"tet {t}: xor-walk quadruple mismatch" for t in to[wrong][:5]]
        reached[to] = True
        wave = to[~wrong]
    if not reached.all():
        out.append(f"xor-walk closure: only {int(reached.sum())} of {n} tets reachable from source")
    return out


# --- encode, reorder, relayout ------------------------------------------------


def encode(raw: RawTetMesh, layout: str, soup: SceneTriangleSoup | None = None, *, check: bool = True) -> CompactMesh:
    """Compact encoding of a raw mesh (tetmesh.py:323-371)."""
    if layout not in LAYOUTS:
        raise ValueError(f"unknown layout {layout!r}")
    if check:
        problems = validate_raw(raw)
        if problems:
            raise MeshError("; ".join(problems[:5]))
    sv, sn = _side_tables(raw.tets, raw.neighbors)
    cf_verts = np.array(raw.cf_verts, dtype=np.int32).reshape(-1, 3)
    if soup is None:  # the constrained faces themselves are the scene
        soup = soup_from_faces(raw.points, cf_verts)
        cf_triangle = np.arange(len(cf_verts), dtype=np.int32)
    else:
        cf_triangle = np.array(raw.cf_triangle, dtype=np.int32)
    return CompactMesh(layout=layout, points=np.ascontiguousarray(raw.points, dtype=np.float32),
                       records=_records_from_tables(layout, sv, sn), side_verts=sv, side_neighbors=sn,
                       cf_triangle=cf_triangle, cf_tets=np.array(raw.cf_tets, dtype=np.int32).reshape(-1, 2),
                       cf_verts=cf_verts, source_tet=int(raw.source_tet), soup=soup)


def regions_from_links(links: np.ndarray) -> np.ndarray:
    """Region label per tet: connected components over the plain links,
    numbered in order of each component's lowest tet (the seeded flood fill
    of tetmesh.py:398-426)."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components

    links = np.asarray(links)
    n = len(links)
    src = np.repeat(np.arange(n), links.shape[1])
    dst = links.ravel()
    live = dst >= 0
    graph = csr_matrix((np.ones(int(live.sum()), np.int8), (src[live], dst[live])), shape=(n, n))
    _, comp = connected_components(graph, directed=False)
    lowest = np.full(comp.max(initial=-1) + 1, n, dtype=np.int64)
    np.minimum.at(lowest, comp, np.arange(n))
    label = np.argsort(np.argsort(lowest, kind="stable"), kind="stable")
    return label[comp].astype(np.int32)


def detect_regions(raw: RawTetMesh) -> np.ndarray:
    _, sn = _side_tables(raw.tets, raw.neighbors)
    plain, _, _ = _ref_classes(sn)
    return regions_from_links(np.where(plain, sn.astype(np.int64) & REF_PAYLOAD_MASK, -1))


def _inverse(perm: np.ndarray) -> np.ndarray:
    inv = np.empty(len(perm), dtype=np.int64)
    inv[perm] = np.arange(len(perm))
    return inv


def reorder(mesh: CompactMesh, scheme: str, *, order: int = 10, seed: int = 0) -> CompactMesh:
    """Renumber points and tets for locality (tetmesh.py:437-507): ``none``,
    ``hilbert`` (points by the Hilbert key of their cell, tets by their
    centroid's), ``hilbert_regions`` (tets grouped by region first) or
    ``shuffle`` (random, the adversarial layout).  Stable sorts, so equal keys
    keep their order and tet ids match the reference's."""
    if scheme == "none":
        return mesh
    if scheme not in ("hilbert", "hilbert_regions", "shuffle"):
        raise ValueError(f"unknown reorder scheme {scheme!r}")
    if scheme == "shuffle":
        rng = np.random.default_rng(seed)
        point_perm, tet_perm = rng.permutation(mesh.n_points), rng.permutation(mesh.n_tets)
    else:
        pts = np.ascontiguousarray(mesh.points, dtype=np.float64)
        lo, hi = pts.min(axis=0), pts.max(axis=0)
        cen = np.empty((mesh.n_tets, 3), dtype=np.float64)
        quads = np.ascontiguousarray(mesh.side_verts, dtype=np.int32)
        check(lib.tb_tet_centroids(addr(pts), len(pts), addr(quads), len(quads), addr(cen)), "tb_tet_centroids")
        point_key = _hilbert.hilbert_keys(_hilbert.quantize(pts, lo, hi, order), order)
        tet_key = _hilbert.hilbert_keys(_hilbert.quantize(cen, lo, hi, order), order)
        if scheme == "hilbert_regions":
            plain, _, _ = _ref_classes(mesh.side_neighbors)
            links = np.where(plain, mesh.side_neighbors.astype(np.int64) & REF_PAYLOAD_MASK, -1)
            tet_key = regions_from_links(links).astype(np.uint64) * np.uint64(1 << 32) + tet_key
        point_perm = np.argsort(point_key, kind="stable")
        tet_perm = np.argsort(tet_key, kind="stable")
    p_new, t_new = _inverse(point_perm), _inverse(tet_perm)
    sv, sn = _side_tables(mesh.side_verts, mesh.side_neighbors, rows=tet_perm, vert_map=p_new, tet_map=t_new)
    cf_tets = np.asarray(mesh.cf_tets, dtype=np.int64).reshape(-1, 2)
    cf_tets = np.where(cf_tets >= 0, t_new[np.maximum(cf_tets, 0)], cf_tets).astype(np.int32)
    return CompactMesh(layout=mesh.layout, points=np.ascontiguousarray(mesh.points[point_perm]),
                       records=_records_from_tables(mesh.layout, sv, sn), side_verts=sv, side_neighbors=sn,
                       cf_triangle=mesh.cf_triangle.copy(), cf_tets=cf_tets,
                       cf_verts=p_new[mesh.cf_verts].astype(np.int32), source_tet=int(t_new[mesh.source_tet]),
                       soup=mesh.soup)


def relayout(mesh: CompactMesh, layout: str) -> CompactMesh:
    """The same mesh with another record layout."""
    if layout == mesh.layout:
        return mesh
    return replace(mesh, layout=layout, records=_records_from_tables(layout, mesh.side_verts, mesh.side_neighbors))


def hull_faces(mesh: CompactMesh) -> np.ndarray:
    """(k, 2) (tet, slot) boundary faces in the reference's tet-major order
    (traversal.hull_faces, traversal.py:530-542): boundary sentinels, and
    hull-backed constrained faces from their front tet."""
    refs = mesh.side_neighbors.astype(np.int64)
    _, constrained, boundary = _ref_classes(refs)
    hull = boundary.copy()
    cft = np.asarray(mesh.cf_tets, dtype=np.int64).reshape(-1, 2)
    if len(cft) and constrained.any():
        t_c, s_c = np.nonzero(constrained)
        pair = cft[refs[t_c, s_c] & REF_PAYLOAD_MASK]
        hull[t_c, s_c] = (pair[:, 1] == NO_TET) & (pair[:, 0] == t_c)
    return np.argwhere(hull)
