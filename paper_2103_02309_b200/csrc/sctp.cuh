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

}  // namespace tb
