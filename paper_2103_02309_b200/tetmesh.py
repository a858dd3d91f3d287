"""Compact xor-linked tetrahedral mesh: record layouts, encoding, reordering.

Host-side mirror of the reference's mesh layer (``tetray.tetmesh``,
/root/reference/pkg/src/tetray/tetmesh.py) with the same names, dtypes and
array conventions, so meshes built here and there are byte-identical.  All
invariant checks are vectorised (the reference walks Python dicts per tet,
tetmesh.py:216-296, ~60 us/tet) so million-tet scenes encode in seconds.

Layouts (tetmesh.py:34-46):
  tet32 [v0, v1, v2, vx, n0..n3]   32 B   (v sorted, v3 implicit via xor)
  tet20 [vx, n0..n3]               20 B
  tet16 [vx, n0^n3, n1^n3, n2^n3]  16 B
Slot j <-> the j-th smallest vertex id ("sorted-slot convention").
A neighbour reference is a u32: bit 31 = constrained face, low 31 bits =
tet or constrained-face index, 0x7FFFFFFF = mesh boundary (tetmesh.py:29-32).

The device side additionally supports TetMesh-80 (ids, refs and inline
vertex coordinates, built on the device from the side tables); it has no
host record dtype here because the reference has no such layout.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

from . import hilbert as _hilbert

TET32 = "tet32"
TET20 = "tet20"
TET16 = "tet16"
LAYOUTS = (TET32, TET20, TET16)

CONSTRAINED_BIT = 1 << 31
REF_PAYLOAD_MASK = CONSTRAINED_BIT - 1
BOUNDARY_REF = REF_PAYLOAD_MASK
NO_TET = -1

TET32_DTYPE = np.dtype([(f, "<u4") for f in ("v0", "v1", "v2", "vx", "n0", "n1", "n2", "n3")])
TET20_DTYPE = np.dtype([(f, "<u4") for f in ("vx", "n0", "n1", "n2", "n3")])
TET16_DTYPE = np.dtype([(f, "<u4") for f in ("vx", "nx0", "nx1", "nx2")])
LAYOUT_DTYPES = {TET32: TET32_DTYPE, TET20: TET20_DTYPE, TET16: TET16_DTYPE}
LAYOUT_BYTES = {TET32: 32, TET20: 20, TET16: 16}
LAYOUT_CODES = {TET32: 32, TET20: 20, TET16: 16}


def face_ref(cf_index: int) -> int:
    """Reference tagging constrained face ``cf_index`` (tetmesh.py:49-51)."""
    return CONSTRAINED_BIT | int(cf_index)


def is_constrained(ref: int) -> bool:
    return bool(int(ref) & CONSTRAINED_BIT)


def is_boundary(ref: int) -> bool:
    return int(ref) == BOUNDARY_REF


def ref_payload(ref: int) -> int:
    return int(ref) & REF_PAYLOAD_MASK


def decode_ref(ref: int) -> int:
    """Tet index of a plain reference, -1 for boundary/constrained (tetmesh.py:67-76)."""
    r = int(ref)
    if r & CONSTRAINED_BIT or r == BOUNDARY_REF:
        return -1
    return r


def compute_xor_sum(v0: int, v1: int, v2: int, v3: int) -> int:
    return v0 ^ v1 ^ v2 ^ v3


def recover_fourth_vertex(v0: int, v1: int, v2: int, vx: int) -> int:
    return v0 ^ v1 ^ v2 ^ vx


class MeshError(Exception):
    """A structural problem in mesh data."""


@dataclass
class ConstrainedFace:
    """A mesh face lying on scene geometry (tetmesh.py:93-104)."""

    triangle_id: int
    tet_front: int
    tet_back: int
    vertex_ids: tuple


@dataclass
class SceneTriangleSoup:
    vertices: np.ndarray  # (p, 3) float64
    triangles: np.ndarray  # (t, 3) int32
    material_ids: np.ndarray  # (t,) int32

    @property
    def n_triangles(self) -> int:
        return len(self.triangles)

    def triangle_coords(self) -> np.ndarray:
        return self.vertices[self.triangles]


@dataclass
class RawTetMesh:
    """Mesh as built/loaded, before compact encoding (tetmesh.py:124-144).

    ``neighbors[i, j]`` is the reference across the face opposite
    ``tets[i, j]``.  Constrained faces are held as parallel arrays (the
    reference keeps a list of ``ConstrainedFace``; ``constrained_faces``
    gives that view) so million-tet scenes stay vectorised.
    """

    points: np.ndarray  # (p, 3) float64
    tets: np.ndarray  # (t, 4) int32
    neighbors: np.ndarray  # (t, 4) uint32
    cf_triangle: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    cf_tets: np.ndarray = field(default_factory=lambda: np.zeros((0, 2), np.int32))
    cf_verts: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), np.int32))
    source_tet: int = 0

    @property
    def n_tets(self) -> int:
        return len(self.tets)

    @property
    def n_points(self) -> int:
        return len(self.points)

    @property
    def constrained_faces(self) -> list:
        return [
            ConstrainedFace(int(t), int(f), int(b), tuple(int(v) for v in vs))
            for t, (f, b), vs in zip(self.cf_triangle, self.cf_tets, self.cf_verts)
        ]


@dataclass
class CompactMesh:
    """Encoded mesh: hot records + points, plus cold side tables (tetmesh.py:147-195)."""

    layout: str
    points: np.ndarray  # (p, 3) float32
    records: np.ndarray  # structured per layout
    side_verts: np.ndarray  # (t, 4) int32 ascending
    side_neighbors: np.ndarray  # (t, 4) uint32 sorted-slot refs
    cf_triangle: np.ndarray  # (c,) int32
    cf_tets: np.ndarray  # (c, 2) int32
    cf_verts: np.ndarray  # (c, 3) int32
    source_tet: int
    soup: SceneTriangleSoup

    @property
    def n_tets(self) -> int:
        return len(self.side_verts)

    @property
    def n_points(self) -> int:
        return len(self.points)

    @property
    def n_constrained(self) -> int:
        return len(self.cf_triangle)

    @property
    def record_bytes(self) -> int:
        return LAYOUT_BYTES[self.layout]

    @property
    def accelerator_bytes(self) -> int:
        return self.records.nbytes + self.points.nbytes

    def records_u32(self) -> np.ndarray:
        k = LAYOUT_BYTES[self.layout] // 4
        return self.records.view("<u4").reshape(self.n_tets, k)

    def triangle_coords(self) -> np.ndarray:
        return self.soup.triangle_coords()


def soup_from_faces(points: np.ndarray, face_verts: np.ndarray) -> SceneTriangleSoup:
    return SceneTriangleSoup(
        vertices=np.asarray(points, dtype=np.float64).copy(),
        triangles=np.asarray(face_verts, dtype=np.int32).copy(),
        material_ids=np.zeros(len(face_verts), dtype=np.int32),
    )


def row_argsort4(a: np.ndarray) -> np.ndarray:
    """np.argsort(a, axis=1, kind="stable") for (n, 4) integer rows, as a
    16-comparison rank network (argsort along a length-4 axis is ~20x slower
    on 50 M rows)."""
    a = np.asarray(a)
    n = len(a)
    rank = np.zeros((n, 4), dtype=np.int8)
    for j in range(4):
        for k in range(4):
            if k == j:
                continue
            # stable: equal keys keep their original order
            rank[:, j] += (a[:, k] < a[:, j]) if k > j else (a[:, k] <= a[:, j])
    order = np.empty((n, 4), dtype=np.int64)
    np.put_along_axis(order, rank.astype(np.int64), np.broadcast_to(np.arange(4), (n, 4)), axis=1)
    return order


def signed_volumes(points: np.ndarray, tets: np.ndarray) -> np.ndarray:
    """6x signed volume per tet, float64, in the reference's einsum/cross order."""
    p = np.asarray(points, dtype=np.float64)[np.asarray(tets)]
    a = p[:, 1] - p[:, 0]
    b = p[:, 2] - p[:, 0]
    c = p[:, 3] - p[:, 0]
    return np.einsum("ij,ij->i", a, np.cross(b, c))


# ---------------------------------------------------------------------------
# Face keys: every (tet, slot) face as a sorted vertex triple packed into one
# integer, so incidence is a sort instead of a dict (ingestion.py:180-188).

_OTHER = np.array([[1, 2, 3], [0, 2, 3], [0, 1, 3], [0, 1, 2]])


def face_triples(tets: np.ndarray) -> np.ndarray:
    """(t, 4, 3) sorted vertex triples of the face opposite each slot."""
    tets = np.asarray(tets, dtype=np.int64)
    tri = tets[:, _OTHER]  # (t, 4, 3)
    return np.sort(tri, axis=2)


def pack_keys(triples: np.ndarray, n_points: int) -> np.ndarray:
    """Pack sorted triples into sortable scalars (lexicographic order kept)."""
    base = np.int64(max(int(n_points), 1))
    t = np.asarray(triples, dtype=np.int64)
    if int(n_points) < (1 << 21):
        return (t[..., 0] * base + t[..., 1]) * base + t[..., 2]
    raise ValueError("meshes with >= 2**21 points need the native builder")


def face_incidence_arrays(tets: np.ndarray, n_points: int):
    """Face incidence as arrays.

    Returns (keys, first, second) over unique faces in ascending key order
    (= the reference's ``sorted(inc.items())``): ``first``/``second`` are
    (tet, slot) pairs encoded as 4*tet+slot in the reference's append order
    (tet-major, slot-minor); ``second`` is -1 for hull faces.
    """
    tri = face_triples(tets)
    keys = pack_keys(tri, n_points).reshape(-1)
    code = np.arange(keys.size, dtype=np.int64)  # 4*tet + slot, append order
    order = np.lexsort((code, keys))
    ks = keys[order]
    cs = code[order]
    start = np.ones(ks.size, dtype=bool)
    start[1:] = ks[1:] != ks[:-1]
    idx = np.nonzero(start)[0]
    counts = np.diff(np.append(idx, ks.size))
    if counts.max(initial=1) > 2:
        raise MeshError("face shared by more than two tetrahedra")
    first = cs[idx]
    second = np.where(counts == 2, cs[np.minimum(idx + 1, ks.size - 1)], -1)
    return ks[idx], first, second


def unpack_keys(keys: np.ndarray, n_points: int) -> np.ndarray:
    base = np.int64(max(int(n_points), 1))
    k = np.asarray(keys, dtype=np.int64)
    c = k % base
    k = k // base
    b = k % base
    a = k // base
    return np.stack([a, b, c], axis=1)


# ---------------------------------------------------------------------------
# Validation (vectorised restatement of validate_raw, tetmesh.py:216-296).


def validate_raw(raw: RawTetMesh) -> list[str]:
    problems: list[str] = []
    tets = np.asarray(raw.tets, dtype=np.int64)
    nbrs = np.asarray(raw.neighbors, dtype=np.int64)
    n_tets = raw.n_tets
    if tets.min(initial=0) < 0 or tets.max(initial=-1) >= raw.n_points:
        problems.append("vertex index out of range")
        return problems
    vols = signed_volumes(raw.points, tets)
    for t in np.nonzero(vols <= 0)[0][:10]:
        problems.append(f"tet {t}: non-positive volume {vols[t]:g}")
    st = np.sort(tets, axis=1)
    rep = np.any(st[:, 1:] == st[:, :-1], axis=1)
    for t in np.nonzero(rep)[0][:10]:
        problems.append(f"tet {t}: repeated vertex")

    ok_rows = ~rep
    tri = face_triples(tets)  # (t, 4, 3) sorted
    boundary = nbrs == BOUNDARY_REF
    constrained = (nbrs & CONSTRAINED_BIT) != 0
    plain = ~boundary & ~constrained & ok_rows[:, None]
    n_cf = len(raw.cf_triangle)
    cf_tets = np.asarray(raw.cf_tets, dtype=np.int64).reshape(-1, 2)
    cf_verts = np.sort(np.asarray(raw.cf_verts, dtype=np.int64).reshape(-1, 3), axis=1)

    # constrained references
    ci, cj = np.nonzero(constrained & ok_rows[:, None])
    if ci.size:
        cfi = nbrs[ci, cj] & REF_PAYLOAD_MASK
        bad = cfi >= n_cf
        for t in ci[bad][:5]:
            problems.append(f"tet {t}: constrained ref out of range")
        good = ~bad
        ci, cj, cfi = ci[good], cj[good], cfi[good]
        mism = np.any(cf_verts[cfi] != tri[ci, cj], axis=1)
        for t, j, c in zip(ci[mism][:5], cj[mism][:5], cfi[mism][:5]):
            problems.append(f"tet {t} slot {j}: constrained face {c} vertex mismatch")
        notlisted = (cf_tets[cfi, 0] != ci) & (cf_tets[cfi, 1] != ci)
        for t, j, c in zip(ci[notlisted][:5], cj[notlisted][:5], cfi[notlisted][:5]):
            problems.append(f"tet {t} slot {j}: constrained face {c} does not list it")

    # plain references: shared face + mutual adjacency
    pi, pj = np.nonzero(plain)
    if pi.size:
        other = nbrs[pi, pj] & REF_PAYLOAD_MASK
        oor = other >= n_tets
        for t in pi[oor][:5]:
            problems.append(f"tet {t}: neighbor index out of range")
        pi, pj, other = pi[~oor], pj[~oor], other[~oor]
        ov = tets[other]  # (k, 4)
        shared = tri[pi, pj]  # (k, 3)
        has = (shared[:, :, None] == ov[:, None, :]).any(axis=2).all(axis=1)
        for t, o in zip(pi[~has][:5], other[~has][:5]):
            problems.append(f"tet {t} / neighbor {o}: face vertices not shared")
        back_ref = nbrs[other]  # (k, 4)
        back_plain = (back_ref != BOUNDARY_REF) & ((back_ref & CONSTRAINED_BIT) == 0)
        mutual = (back_plain & ((back_ref & REF_PAYLOAD_MASK) == pi[:, None])).any(axis=1)
        for t, o in zip(pi[~mutual][:5], other[~mutual][:5]):
            problems.append(f"adjacency not mutual between tets {t} and {o}")

    # every constrained face referenced by 1 (hull) or 2 tets
    if n_cf:
        cref = np.zeros(n_cf, dtype=np.int64)
        for side in range(2):
            t = cf_tets[:, side]
            live = t != NO_TET
            oob = live & ((t < 0) | (t >= n_tets))
            for c in np.nonzero(oob)[0][:5]:
                problems.append(f"constrained face {c}: tet {t[c]} out of range")
            ok = live & ~oob
            rows = nbrs[t[ok]]
            hit = (((rows & CONSTRAINED_BIT) != 0) & ((rows & REF_PAYLOAD_MASK) == np.nonzero(ok)[0][:, None])).any(axis=1)
            cref[np.nonzero(ok)[0]] += hit
        expect = np.where(cf_tets[:, 1] == NO_TET, 1, 2)
        for c in np.nonzero(cref != expect)[0][:5]:
            problems.append(f"constrained face {c}: referenced by {cref[c]} tets, expected {expect[c]}")
    if not (0 <= raw.source_tet < n_tets):
        problems.append(f"source tet {raw.source_tet} out of range")
    return problems


def _records_from_tables(layout: str, side_verts: np.ndarray, side_neighbors: np.ndarray) -> np.ndarray:
    """Pack the hot records from the side tables (tetmesh.py:299-320)."""
    if layout not in LAYOUT_DTYPES:
        raise ValueError(f"unknown layout {layout!r}")
    sv = np.asarray(side_verts).astype(np.uint32)
    sn = np.asarray(side_neighbors, dtype=np.uint32)
    n = len(sv)
    words = np.empty((n, LAYOUT_BYTES[layout] // 4), dtype=np.uint32)
    vx = sv[:, 0] ^ sv[:, 1] ^ sv[:, 2] ^ sv[:, 3]
    if layout == TET32:
        words[:, 0:3] = sv[:, 0:3]
        words[:, 3] = vx
        words[:, 4:8] = sn
    elif layout == TET20:
        words[:, 0] = vx
        words[:, 1:5] = sn
    else:
        words[:, 0] = vx
        words[:, 1:4] = sn[:, 0:3] ^ sn[:, 3:4]
    return words.view(LAYOUT_DTYPES[layout]).reshape(n)


def encode(raw: RawTetMesh, layout: str, soup: SceneTriangleSoup | None = None, *, check: bool = True) -> CompactMesh:
    """Encode a raw mesh into a compact layout (tetmesh.py:323-371)."""
    if layout not in LAYOUTS:
        raise ValueError(f"unknown layout {layout!r}")
    if check:
        problems = validate_raw(raw)
        if problems:
            raise MeshError("; ".join(problems[:5]))
    order = row_argsort4(raw.tets)
    side_verts = np.take_along_axis(raw.tets, order, axis=1).astype(np.int32)
    side_neighbors = np.take_along_axis(raw.neighbors, order, axis=1).astype(np.uint32)
    cf_verts = np.asarray(raw.cf_verts, dtype=np.int32).reshape(-1, 3)
    if soup is None:
        soup = soup_from_faces(raw.points, cf_verts)
        cf_triangle = np.arange(len(cf_verts), dtype=np.int32)
    else:
        cf_triangle = np.asarray(raw.cf_triangle, dtype=np.int32).copy()
    return CompactMesh(
        layout=layout,
        points=np.ascontiguousarray(raw.points, dtype=np.float32),
        records=_records_from_tables(layout, side_verts, side_neighbors),
        side_verts=side_verts,
        side_neighbors=side_neighbors,
        cf_triangle=cf_triangle,
        cf_tets=np.asarray(raw.cf_tets, dtype=np.int32).reshape(-1, 2).copy(),
        cf_verts=cf_verts.copy(),
        source_tet=int(raw.source_tet),
        soup=soup,
    )


def _plain_neighbor_matrix(side_neighbors: np.ndarray) -> np.ndarray:
    refs = side_neighbors.astype(np.int64)
    plain = ((refs & CONSTRAINED_BIT) == 0) & (refs != BOUNDARY_REF)
    return np.where(plain, refs & REF_PAYLOAD_MASK, -1)


def regions_from_links(links: np.ndarray) -> np.ndarray:
    """Connected components over plain links, labelled in order of each
    component's lowest tet index -- the labels of the reference's seeded
    flood fill (tetmesh.py:398-426)."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components

    n = len(links)
    rows = np.repeat(np.arange(n, dtype=np.int64), links.shape[1])
    cols = np.asarray(links).reshape(-1)
    keep = cols >= 0
    g = coo_matrix((np.ones(int(keep.sum()), dtype=np.int8), (rows[keep], cols[keep])), shape=(n, n))
    _, comp = connected_components(g, directed=False)
    first = np.full(comp.max(initial=-1) + 1, n, dtype=np.int64)
    np.minimum.at(first, comp, np.arange(n, dtype=np.int64))
    rank = np.empty_like(first)
    rank[np.argsort(first, kind="stable")] = np.arange(first.size)
    return rank[comp].astype(np.int32)


def detect_regions(raw: RawTetMesh) -> np.ndarray:
    order = np.argsort(raw.tets, axis=1, kind="stable")
    side_neighbors = np.take_along_axis(raw.neighbors, order, axis=1).astype(np.uint32)
    return regions_from_links(_plain_neighbor_matrix(side_neighbors))


def _remap_refs(side_neighbors: np.ndarray, tet_old2new: np.ndarray) -> np.ndarray:
    refs = side_neighbors.astype(np.int64)
    plain = ((refs & CONSTRAINED_BIT) == 0) & (refs != BOUNDARY_REF)
    out = refs.copy()
    out[plain] = tet_old2new[refs[plain]]
    return out.astype(np.uint32)


def reorder(mesh: CompactMesh, scheme: str, *, order: int = 10, seed: int = 0) -> CompactMesh:
    """Reorder points and tets for locality (tetmesh.py:437-507).

    Schemes: none, hilbert (points by position key, tets by centroid key),
    hilbert_regions (tets grouped by enclosed region first), shuffle.
    """
    if scheme == "none":
        return mesh
    if scheme not in ("hilbert", "hilbert_regions", "shuffle"):
        raise ValueError(f"unknown reorder scheme {scheme!r}")
    pts = mesh.points.astype(np.float64)
    lo, hi = pts.min(axis=0), pts.max(axis=0)
    if scheme == "shuffle":
        rng = np.random.default_rng(seed)
        point_perm = rng.permutation(mesh.n_points)
        tet_perm = rng.permutation(mesh.n_tets)
    else:
        centroids = pts[mesh.side_verts].mean(axis=1)
        pkeys = _hilbert.hilbert_keys(_hilbert.quantize(pts, lo, hi, order), order)
        point_perm = np.argsort(pkeys, kind="stable")
        tkeys = _hilbert.hilbert_keys(_hilbert.quantize(centroids, lo, hi, order), order)
        if scheme == "hilbert_regions":
            regions = regions_from_links(_plain_neighbor_matrix(mesh.side_neighbors)).astype(np.uint64)
            tkeys = regions * np.uint64(1 << 32) + tkeys
        tet_perm = np.argsort(tkeys, kind="stable")
    point_old2new = np.empty(mesh.n_points, dtype=np.int64)
    point_old2new[point_perm] = np.arange(mesh.n_points)
    tet_old2new = np.empty(mesh.n_tets, dtype=np.int64)
    tet_old2new[tet_perm] = np.arange(mesh.n_tets)

    verts = point_old2new[mesh.side_verts[tet_perm]]
    nbrs = _remap_refs(mesh.side_neighbors[tet_perm], tet_old2new)
    row_order = row_argsort4(verts)
    side_verts = np.take_along_axis(verts, row_order, axis=1).astype(np.int32)
    side_neighbors = np.take_along_axis(nbrs, row_order, axis=1)
    cf_tets = mesh.cf_tets.copy()
    live = cf_tets >= 0
    cf_tets[live] = tet_old2new[cf_tets[live]].astype(np.int32)
    return CompactMesh(
        layout=mesh.layout,
        points=np.ascontiguousarray(mesh.points[point_perm]),
        records=_records_from_tables(mesh.layout, side_verts, side_neighbors),
        side_verts=side_verts,
        side_neighbors=side_neighbors,
        cf_triangle=mesh.cf_triangle.copy(),
        cf_tets=cf_tets,
        cf_verts=point_old2new[mesh.cf_verts].astype(np.int32),
        source_tet=int(tet_old2new[mesh.source_tet]),
        soup=mesh.soup,
    )


def relayout(mesh: CompactMesh, layout: str) -> CompactMesh:
    """Same mesh, other record layout (tetmesh.py:510-518)."""
    if layout == mesh.layout:
        return mesh
    return replace(mesh, layout=layout, records=_records_from_tables(layout, mesh.side_verts, mesh.side_neighbors))


def validate(mesh: CompactMesh) -> list[str]:
    """Integrity report for a compact mesh (tetmesh.py:521-608), vectorised.

    Covers record size, xor sums/links vs the side tables, sorted slots,
    mutual adjacency, constrained-face cross references, f32 degeneracy and
    reachability of every tet from the source through xor links
    (the closure of tetmesh.py:611-640, done as a BFS over link arrays).
    """
    problems: list[str] = []
    rec = mesh.records
    if rec.dtype.itemsize != LAYOUT_BYTES[mesh.layout]:
        problems.append(f"record size {rec.dtype.itemsize} != {LAYOUT_BYTES[mesh.layout]}")
    sv = mesh.side_verts
    asc = np.any(np.diff(sv, axis=1) <= 0, axis=1)
    if asc.any():
        problems.append(f"tet {int(np.nonzero(asc)[0][0])}: side-table vertices not strictly ascending")
    svu = sv.astype(np.uint32)
    vx_expect = svu[:, 0] ^ svu[:, 1] ^ svu[:, 2] ^ svu[:, 3]
    for t in np.nonzero(rec["vx"] != vx_expect)[0][:10]:
        problems.append(f"tet {t}: xor-sum mismatch")
    if mesh.layout == TET32:
        for j in range(3):
            for t in np.nonzero(rec[f"v{j}"] != svu[:, j])[0][:5]:
                problems.append(f"tet {t}: stored vertex v{j} mismatch")
    if mesh.layout in (TET32, TET20):
        for j in range(4):
            for t in np.nonzero(rec[f"n{j}"] != mesh.side_neighbors[:, j])[0][:5]:
                problems.append(f"tet {t}: neighbor slot {j} violates sorted-slot order")
    if mesh.layout == TET16:
        for j in range(3):
            expect = mesh.side_neighbors[:, j] ^ mesh.side_neighbors[:, 3]
            for t in np.nonzero(rec[f"nx{j}"] != expect)[0][:5]:
                problems.append(f"tet {t}: xor link nx{j} mismatch")
    raw = RawTetMesh(
        points=mesh.points.astype(np.float64),
        tets=sv,
        neighbors=mesh.side_neighbors,
        cf_triangle=mesh.cf_triangle,
        cf_tets=mesh.cf_tets,
        cf_verts=mesh.cf_verts,
        source_tet=mesh.source_tet,
    )
    for p in validate_raw(raw):
        if "non-positive volume" in p:
            continue  # sorted slots flip orientation; only zero volume is a fault here
        problems.append(p)
    vols = signed_volumes(mesh.points.astype(np.float64), sv)
    if np.any(vols == 0):
        problems.append(f"tet {int(np.nonzero(vols == 0)[0][0])}: degenerate (zero volume) after f32 quantization")
    problems.extend(_xor_walk_closure(mesh))
    return problems


def hull_faces(mesh: CompactMesh) -> np.ndarray:
    """(k, 2) int64 (tet, slot) of the mesh boundary faces in the reference's
    order (traversal.hull_faces, traversal.py:530-542): unconstrained boundary
    sentinels plus hull-backed constrained faces seen from their front tet."""
    refs = mesh.side_neighbors.astype(np.int64)
    boundary = refs == BOUNDARY_REF
    constrained = (refs & CONSTRAINED_BIT) != 0
    cf = np.where(constrained, refs & REF_PAYLOAD_MASK, 0)
    rows = np.broadcast_to(np.arange(mesh.n_tets)[:, None], refs.shape)
    cft = np.asarray(mesh.cf_tets).reshape(-1, 2)
    hull_cf = constrained & (cft[cf, 1] == NO_TET) & (cft[cf, 0] == rows) if len(cft) else np.zeros_like(constrained)
    t, j = np.nonzero(boundary | hull_cf)
    return np.stack([t, j], axis=1)


def _cross_links(side_neighbors: np.ndarray, cf_tets: np.ndarray) -> np.ndarray:
    refs = side_neighbors.astype(np.int64)
    out = _plain_neighbor_matrix(side_neighbors)
    tagged = (refs & CONSTRAINED_BIT) != 0
    if tagged.any() and len(cf_tets):
        rows = np.broadcast_to(np.arange(len(refs))[:, None], refs.shape)
        cfs = (refs & REF_PAYLOAD_MASK)[tagged]
        here = rows[tagged]
        front = cf_tets[cfs, 0]
        back = cf_tets[cfs, 1]
        out[tagged] = np.where(front == here, back, front)
    return out


def _xor_walk_closure(mesh: CompactMesh) -> list[str]:
    """BFS from the source over xor links: each neighbour's quadruple is
    reconstructed from the shared face and its xor sum and compared with the
    side table."""
    n = mesh.n_tets
    if not (0 <= mesh.source_tet < n):
        return [f"source tet {mesh.source_tet} out of range"]
    vx = mesh.records["vx"].astype(np.int64)
    links = _cross_links(mesh.side_neighbors, mesh.cf_tets)
    sv = mesh.side_verts.astype(np.int64)
    seen = np.zeros(n, dtype=bool)
    seen[mesh.source_tet] = True
    frontier = np.array([mesh.source_tet], dtype=np.int64)
    problems: list[str] = []
    while frontier.size:
        nb = links[frontier]  # (f, 4)
        f_idx, j = np.nonzero(nb >= 0)
        src = frontier[f_idx]
        dst = nb[f_idx, j]
        fresh = ~seen[dst]
        src, dst, j = src[fresh], dst[fresh], j[fresh]
        if not dst.size:
            break
        dst, first = np.unique(dst, return_index=True)
        src, j = src[first], j[first]
        face = sv[src][:, _OTHER][np.arange(len(src)), j]  # (k, 3)
        fourth = face[:, 0] ^ face[:, 1] ^ face[:, 2] ^ vx[dst]
        quad = np.sort(np.concatenate([face, fourth[:, None]], axis=1), axis=1)
        bad = np.any(quad != sv[dst], axis=1)
        for t in dst[bad][:5]:
            problems.append(f"tet {t}: xor-walk quadruple mismatch")
        seen[dst] = True
        frontier = dst[~bad]
    reach = int(seen.sum())
    if reach < n:
        problems.append(f"xor-walk closure: only {reach} of {n} tets reachable from source")
    return problems
