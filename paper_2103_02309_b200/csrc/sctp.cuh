// sctp.cuh -- ScTP (scalar triple product) exit-face test and walk step.
//
// Predicate: traversal.sctp_exit_face (/root/reference/pkg/src/tetray/
// traversal.py:484-511): fp64, for each face j != entry of the sorted-slot
// quad (outward winding by the orientation rho), s_k = d . (A x B) on
// origin-relative vertices; first face with min >= 0 and max > 0, else the
// least violated.  The reference has the predicate only; the walk around it
// (entry face = the face opposite the recovered vertex i3, exit vertex ->
// next reference by the layout's own rule) is this repo's, restated in
// oracle/tetoracle.c so both agree bit for bit.  Dot products accumulate
// left to right: (x0*y0 + x1*y1) + x2*y2.
#pragma once

#include "traverse.cuh"

namespace tb {

struct D3 {
  double x, y, z;
};

__device__ __forceinline__ D3 dsub3(const D3& a, const D3& b) {
  return {__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z)};
}
__device__ __forceinline__ D3 dcross3(const D3& a, const D3& b) {
  return {__dsub_rn(__dmul_rn(a.y, b.z), __dmul_rn(a.z, b.y)),
          __dsub_rn(__dmul_rn(a.z, b.x), __dmul_rn(a.x, b.z)),
          __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))};
}
__device__ __forceinline__ double ddot3(const D3& a, const D3& b) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}
__device__ __forceinline__ D3 dsel(bool c, const D3& a, const D3& b) { return c ? a : b; }

// Exit slot of the sorted quad (P, ids ascending); entry < 0 = none.
// rho_pos: sign of the quad's fp64 orientation (p1-p0).((p2-p0)x(p3-p0)) --
// the same expression as orientation() in traverse.cuh, so it comes from
// the per-tet table MeshView.orient instead of 30 fp64 ops per step.
__device__ __forceinline__ int sctp_exit(const float4 (&P)[4], const uint32_t (&)[4], const double (&O)[3],
                                         const double (&Dd)[3], int entry, bool rho_pos) {
  const D3 o = {O[0], O[1], O[2]};
  const D3 d = {Dd[0], Dd[1], Dd[2]};
  D3 p[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) p[i] = {(double)P[i].x, (double)P[i].y, (double)P[i].z};
  int best_j = -1;
  double best_m = -INFINITY;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (j == entry) continue;
    const int a = (j == 0) ? 1 : 0;
    const int b0 = (j <= 1) ? 2 : 1;
    const int c0 = (j == 3) ? 2 : 3;
    const bool swap = ((j & 1) == 0) != rho_pos;
    const D3 A = dsub3(p[a], o);
    const D3 Bv = dsub3(p[b0], o);
    const D3 Cv = dsub3(p[c0], o);
    const D3 B = dsel(swap, Cv, Bv);
    const D3 C = dsel(swap, Bv, Cv);
    const double s0 = ddot3(d, dcross3(A, B));
    const double s1 = ddot3(d, dcross3(B, C));
    const double s2 = ddot3(d, dcross3(C, A));
    double mn = s0, mx = s0;
    if (s1 < mn) mn = s1;
    if (s2 < mn) mn = s2;
    if (s1 > mx) mx = s1;
    if (s2 > mx) mx = s2;
    if (mn >= 0.0 && mx > 0.0) return j;
    if (mn > best_m) {
      best_m = mn;
      best_j = j;
    }
  }
  // All-NaN (degenerate ray): the first admissible slot.
  if (best_j < 0) best_j = (entry == 0) ? 1 : 0;
  return best_j;
}

// The entry-face window of the ScTP walk: three ascending vertex ids and
// their coordinates (kept in registers, so each step fetches one point).
struct SctpWindow {
  uint32_t id[3];
  float4 P[3];
  // Keep the three slots of the sorted quad other than j (SLOT_A/B/C order,
  // _kernels.pyx:105-111), which stays ascending.
  __device__ __forceinline__ void drop(const float4 (&Q)[4], const uint32_t (&ids)[4], int j) {
    const int a = (j == 0) ? 1 : 0;
    const int b = (j <= 1) ? 2 : 1;
    const int c = (j == 3) ? 2 : 3;
    id[0] = (a == 0) ? ids[0] : ids[1];
    P[0] = (a == 0) ? Q[0] : Q[1];
    id[1] = (b == 1) ? ids[1] : ids[2];
    P[1] = (b == 1) ? Q[1] : Q[2];
    id[2] = (c == 2) ? ids[2] : ids[3];
    P[2] = (c == 2) ? Q[2] : Q[3];
  }
};

template <int L>
__device__ __forceinline__ uint32_t sctp_advance(const MeshView& m, SctpWindow& w, const double (&O)[3],
                                                 const double (&D)[3], uint32_t nxt, uint32_t prev) {
  Record<L> rec;
  rec.load(m, nxt);
  uint32_t i3 = w.id[0] ^ w.id[1] ^ w.id[2] ^ rec.vxw();
  if (L != 80) i3 = min(i3, (uint32_t)m.n_points - 1u);
  const float4 q = fetch_vertex<L>(m, rec, i3);
  const int pos = (w.id[0] < i3) + (w.id[1] < i3) + (w.id[2] < i3);  // entry slot
  uint32_t ids[4];
  float4 P[4];
  ids[0] = (pos == 0) ? i3 : w.id[0];
  P[0] = (pos == 0) ? q : w.P[0];
  ids[1] = (pos < 1) ? w.id[0] : ((pos == 1) ? i3 : w.id[1]);
  P[1] = (pos < 1) ? w.P[0] : ((pos == 1) ? q : w.P[1]);
  ids[2] = (pos < 2) ? w.id[1] : ((pos == 2) ? i3 : w.id[2]);
  P[2] = (pos < 2) ? w.P[1] : ((pos == 2) ? q : w.P[2]);
  ids[3] = (pos < 3) ? w.id[2] : i3;
  P[3] = (pos < 3) ? w.P[2] : q;
  const int j = sctp_exit(P, ids, O, D, pos, __ldg(&m.orient[nxt]) != 0);
  const uint32_t idxf = (j == 0) ? ids[0] : ((j == 1) ? ids[1] : ((j == 2) ? ids[2] : ids[3]));
  const uint32_t nref = rec.next_ref(w.id, i3, idxf, prev);
  w.drop(P, ids, j);
  return nref;
}

// ----------------------------------------------------------------------------
// Edge-cached ScTP step.  The predicate's face values are scalar triple
// products s = d . (A x B) of origin-relative vertices, one per directed
// edge of the face.  For the quad's slots x < y let E[x][y] = d.(R_x x R_y);
// then d.(R_y x R_x) = -E[x][y] *exactly* (fp64 cross and dot are
// antisymmetric bit for bit in round-to-nearest), so every s the reference
// computes is +-E of one of the tet's six edges.  Three of them belong to the
// entry face and were computed in the previous tet (carried in `SctpEdges`);
// only the three edges to the new vertex V are new: 3 triple products per
// step instead of up to 9 (plus 9-27 fp64 subtractions) in sctp_exit.
//
// Face k (opposite window vertex w_k, k = 0..2, i.e. slots j = 0..3 minus the
// entry slot, visited in the reference's order) has vertices {w_p, w_q, V},
// p < q.  With X = e_pq, tp = d.(R_p x R_V), tq = d.(R_q x R_V), its ordered
// values (s0, s1, s2) are one of (-tp, X, tq), (-tq, -X, tp), (tp, -tq, -X),
// (X, tq, -tp) -- as multisets all +-{-tp, X, tq}, the sign being + exactly
// when swap == (V lies between w_p and w_q in id order).  The reference's
// decision uses the values only through min, max and comparisons with 0, so
// it is evaluated on the multiset; signed zeros and the order of equal values
// cannot change any comparison.  NaNs would make the order matter: any NaN
// among the step's values takes the exact per-face path (sctp_exit) instead.
struct SctpEdges {
  double e01, e02, e12;  // entry face, window order (ascending ids)
};

__device__ __forceinline__ double triple(const D3& d, const D3& a, const D3& b) { return ddot3(d, dcross3(a, b)); }

__device__ __forceinline__ D3 rel(const float4& P, const D3& o) {
  return {__dsub_rn((double)P.x, o.x), __dsub_rn((double)P.y, o.y), __dsub_rn((double)P.z, o.z)};
}

// Edges of a fresh window (init, NaN fallback).
__device__ __forceinline__ void window_edges(const SctpWindow& w, const D3& o, const D3& d, SctpEdges& e) {
  const D3 R0 = rel(w.P[0], o), R1 = rel(w.P[1], o), R2 = rel(w.P[2], o);
  e.e01 = triple(d, R0, R1);
  e.e02 = triple(d, R0, R2);
  e.e12 = triple(d, R1, R2);
}

template <int L>
__device__ __forceinline__ uint32_t sctp_advance_cached(const MeshView& m, SctpWindow& w, SctpEdges& e,
                                                        const double (&O)[3], const double (&Dd)[3], uint32_t nxt,
                                                        uint32_t prev) {
  Record<L> rec;
  rec.load(m, nxt);
  uint32_t i3 = w.id[0] ^ w.id[1] ^ w.id[2] ^ rec.vxw();
  if (L != 80) i3 = min(i3, (uint32_t)m.n_points - 1u);
  const float4 q = fetch_vertex<L>(m, rec, i3);
  const bool rho = __ldg(&m.orient[nxt]) != 0;
  // a_k: window vertex k precedes V in id order (pos = a0 + a1 + a2)
  const bool a0 = w.id[0] < i3, a1 = w.id[1] < i3, a2 = w.id[2] < i3;
  const D3 o = {O[0], O[1], O[2]}, d = {Dd[0], Dd[1], Dd[2]};
  const D3 RV = rel(q, o);
  const double t0 = triple(d, rel(w.P[0], o), RV);
  const double t1 = triple(d, rel(w.P[1], o), RV);
  const double t2 = triple(d, rel(w.P[2], o), RV);
  if (isnan(t0) || isnan(t1) || isnan(t2) || isnan(e.e01) || isnan(e.e02) || isnan(e.e12)) {
    // exact per-face path (the order of the values matters with NaNs)
    const uint32_t nref = sctp_advance<L>(m, w, O, Dd, nxt, prev);
    window_edges(w, o, d, e);
    return nref;
  }
  int exit_k = -1, best_k = -1;
  double best_m = -INFINITY;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    // face opposite w_k: p < q the other window vertices
    const bool ap = (k == 0) ? a1 : a0;
    const bool aq = (k == 2) ? a1 : a2;
    const bool ak = (k == 0) ? a0 : ((k == 1) ? a1 : a2);
    const double X = (k == 0) ? e.e12 : ((k == 1) ? e.e02 : e.e01);
    const double tp = (k == 0) ? t1 : t0;
    const double tq = (k == 2) ? t1 : t2;
    const int j = ak ? k : k + 1;  // the face's slot in the sorted quad
    const bool swap = ((j & 1) == 0) != rho;
    const bool middle = ap && !aq;
    const bool pos_sign = swap == middle;
    const double v0 = -tp;
    const double lo = fmin(fmin(v0, X), tq), hi = fmax(fmax(v0, X), tq);
    const double mn = pos_sign ? lo : -hi;
    const bool accept = pos_sign ? (lo >= 0.0 && hi > 0.0) : (hi <= 0.0 && lo < 0.0);
    if (exit_k < 0) {
      if (accept) {
        exit_k = k;
      } else if (mn > best_m) {
        best_m = mn;
        best_k = k;
      }
    }
  }
  if (exit_k < 0) exit_k = best_k >= 0 ? best_k : 0;  // all-NaN cannot happen here; slot rule of sctp_exit
  const int k = exit_k;
  const uint32_t idxf = (k == 0) ? w.id[0] : ((k == 1) ? w.id[1] : w.id[2]);
  const uint32_t nref = rec.next_ref(w.id, i3, idxf, prev);
  // new window {w_p, w_q, V} in id order, with its edges
  const bool ap = (k == 0) ? a1 : a0;
  const bool aq = (k == 2) ? a1 : a2;
  const uint32_t idp = (k == 0) ? w.id[1] : w.id[0], idq = (k == 2) ? w.id[1] : w.id[2];
  const float4 Pp = (k == 0) ? w.P[1] : w.P[0], Pq = (k == 2) ? w.P[1] : w.P[2];
  const double X = (k == 0) ? e.e12 : ((k == 1) ? e.e02 : e.e01);
  const double tp = (k == 0) ? t1 : t0;
  const double tq = (k == 2) ? t1 : t2;
  if (!ap) {  // V first
    w.id[0] = i3; w.P[0] = q; w.id[1] = idp; w.P[1] = Pp; w.id[2] = idq; w.P[2] = Pq;
    e.e01 = -tp; e.e02 = -tq; e.e12 = X;
  } else if (!aq) {  // V between
    w.id[0] = idp; w.P[0] = Pp; w.id[1] = i3; w.P[1] = q; w.id[2] = idq; w.P[2] = Pq;
    e.e01 = tp; e.e02 = X; e.e12 = -tq;
  } else {  // V last
    w.id[0] = idp; w.P[0] = Pp; w.id[1] = idq; w.P[1] = Pq; w.id[2] = i3; w.P[2] = q;
    e.e01 = X; e.e02 = tp; e.e12 = tq;
  }
  return nref;
}

}  // namespace tb
