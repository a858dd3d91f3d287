// traverse.cuh -- device-side traversal arithmetic for sm_100a.
//
// Every floating-point operation here is written with explicit round-to-
// nearest intrinsics (__fmul_rn/__fadd_rn/__fsub_rn/__fdiv_rn and the __d*
// fp64 forms) in the exact expression order of the reference's compiled
// kernels (/root/reference/pkg/src/tetray/_kernels.pyx, built with
// -ffp-contract=off, pkg/setup.py:17-20).  The intrinsics are never
// contracted into FFMA/DFMA, so results are bit-identical to the reference
// for the same fp32 inputs; the library is additionally compiled with
// -fmad=false -ftz=false -prec-div=true as a second line of defence.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tb {

constexpr uint32_t kConstrained = 0x80000000u;  // tetmesh.py:29
constexpr uint32_t kPayload = 0x7FFFFFFFu;      // tetmesh.py:30
constexpr uint32_t kBoundary = 0x7FFFFFFFu;     // tetmesh.py:31

constexpr uint8_t kMiss = 0, kHit = 1, kError = 2;  // _kernels.pyx:17-19

// ----------------------------------------------------------------------------
// Device view of an uploaded mesh.  Layout-specific record arrays:
//   tet16: rec4[t]            = {vx, nx0, nx1, nx2}            (16 B)
//   tet20: vx[t] (4 B) + rec4[t] = {n0, n1, n2, n3}           (4 + 16 B, SoA)
//   tet32: rec4[2t], rec4[2t+1] = {v0, v1, v2, vx}, {n0..n3}  (32 B, one sector)
//   tet80: rec4[5t .. 5t+4]   = {v0..v3}, {n0..n3}, 12 floats (80 B, inline xyz)
struct MeshView {
  const float4* __restrict__ pts;     // 6 x (p,): copy k = (q[mx],q[ot],q[mn],0); copy 0 = x,y,z,0
  const uint4* __restrict__ rec4;     // layout records (see above)
  const uint32_t* __restrict__ vx;    // tet20 only
  const int4* __restrict__ sv;        // side_verts (t,) ascending
  const uint4* __restrict__ sn;       // side_neighbors (t,) sorted-slot refs
  const int32_t* __restrict__ cf_tri; // (c,)
  const int2* __restrict__ cf_tets;   // (c,) front, back
  const double* __restrict__ tri;     // (n_tri, 9)
  const uint8_t* __restrict__ orient; // (t,) rho(sorted quad) > 0, see orientation()
  int64_t n_points;
  int64_t n_tets;
  int64_t n_cf;   // constrained faces (rows of cf_tri / cf_tets)
  int64_t n_tri;  // scene triangles (rows of tri)
};

// Index of the axis-permuted point copy holding (q[mx], q[ot], q[mn]).
__device__ __forceinline__ int perm_index(int mx, int ot) { return mx * 2 + (ot > mx ? ot - 1 : ot); }

__device__ __forceinline__ float pick3(float x, float y, float z, int a) {
  return a == 0 ? x : (a == 1 ? y : z);
}
// Component k (0..3) of a uint4 as a 2-level select on the bits of k
// (keeps ptxas from emitting a branch island per pick).
__device__ __forceinline__ uint32_t pick4u(uint4 v, int k) {
  const uint32_t lo = (k & 1) ? v.y : v.x;
  const uint32_t hi = (k & 1) ? v.w : v.z;
  return (k & 2) ? hi : lo;
}

__device__ __forceinline__ float4 ldg_f4(const float4* p) { return __ldg(p); }
// 16 B read-only load of base[i] with the address formed by one mad.wide
// (base is a per-ray pointer; keeps the 64-bit index math off the hot
// chain).  An opaque runtime stride (IMAD.WIDE instead of LEA) measured
// slower (r01 A/B: cfg2 -2 %, cfg3 -2 %).
__device__ __forceinline__ float4 ldg_f4_at(const float4* base, uint32_t i) {
  float4 r;
  asm("{\n\t.reg .u64 a;\n\tmad.wide.u32 a, %4, 16, %5;\n\t"
      "ld.global.nc.v4.f32 {%0, %1, %2, %3}, [a];\n\t}"
      : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
      : "r"(i), "l"(base));
  return r;
}
__device__ __forceinline__ uint4 ldg_u4(const uint4* p) { return __ldg(p); }

// ----------------------------------------------------------------------------
// Scaled basis, _kernels.pyx:42-86 (spec geometry.py:120-221, Eqs. 1-3).
struct Basis {
  int mn, mx, ot;
  float umax, vmax, voth, sgn, pox, poy;
};

__device__ __forceinline__ void build_basis(float o0, float o1, float o2, float d0, float d1,
                                            float d2, Basis& b) {
  // Written with per-axis predicates and value selects (no axis indices):
  // the index-then-pick form compiled to ~25 branch islands (BSSY/BRA/BSYNC)
  // in every ray's init.  Same IEEE operations in the same order.
  const float a0 = fabsf(d0), a1 = fabsf(d1), a2 = fabsf(d2);
  // min axis: argmin |d|, lowest index on ties (_kernels.pyx:43-52)
  const bool c10 = a1 < a0, c21 = a2 < a1, c20 = a2 < a0;
  const bool mn2 = c10 ? c21 : c20;
  const bool mn1 = c10 && !c21;
  const bool mn0 = !mn1 && !mn2;
  // the other two axes in index order r0 < r1; max among them, '>=' keeps r0
  const float ar0 = mn0 ? a1 : a0;
  const float ar1 = mn2 ? a1 : a2;
  const bool x0 = ar0 >= ar1;  // mx = r0 (else r1); ot = the other
  const int r0 = mn0 ? 1 : 0, r1 = mn2 ? 1 : 2;
  b.mn = mn0 ? 0 : (mn1 ? 1 : 2);
  b.mx = x0 ? r0 : r1;
  b.ot = x0 ? r1 : r0;
  const float dr0 = mn0 ? d1 : d0, dr1 = mn2 ? d1 : d2;
  const float dmx = x0 ? dr0 : dr1, dot = x0 ? dr1 : dr0;
  const float umax = -__fdiv_rn(dot, dmx);
  b.umax = umax;
  // u = e_ot + umax e_mx in xyz (u[mn] = 0), t = d x u (_kernels.pyx:64-75)
  const bool ot0 = b.ot == 0, ot1 = b.ot == 1, mx0 = b.mx == 0, mx1 = b.mx == 1;
  const float u0 = ot0 ? 1.0f : (mx0 ? umax : 0.0f);
  const float u1 = ot1 ? 1.0f : (mx1 ? umax : 0.0f);
  const float u2 = (!ot0 && !ot1) ? 1.0f : ((!mx0 && !mx1) ? umax : 0.0f);
  const float t0 = __fsub_rn(__fmul_rn(d1, u2), __fmul_rn(d2, u1));
  const float t1 = __fsub_rn(__fmul_rn(d2, u0), __fmul_rn(d0, u2));
  const float t2 = __fsub_rn(__fmul_rn(d0, u1), __fmul_rn(d1, u0));
  const float tmn = mn0 ? t0 : (mn1 ? t1 : t2);
  const float tr0 = mn0 ? t1 : t0, tr1 = mn2 ? t1 : t2;
  const float tmx = x0 ? tr0 : tr1, tot = x0 ? tr1 : tr0;
  const float sgn = (tmn > 0.0f) ? 1.0f : -1.0f;
  const float tabs = (tmn > 0.0f) ? tmn : -tmn;
  b.sgn = sgn;
  b.vmax = __fdiv_rn(tmx, tabs);
  b.voth = __fdiv_rn(tot, tabs);
  const float or0 = mn0 ? o1 : o0, or1 = mn2 ? o1 : o2;
  const float omx = x0 ? or0 : or1, oot = x0 ? or1 : or0, omn = mn0 ? o0 : (mn1 ? o1 : o2);
  b.pox = __fadd_rn(__fmul_rn(umax, omx), oot);
  b.poy = __fadd_rn(__fadd_rn(__fmul_rn(b.vmax, omx), __fmul_rn(b.voth, oot)), __fmul_rn(sgn, omn));
}

// project, _kernels.pyx:89-91.
__device__ __forceinline__ void project(const Basis& b, float qx, float qy, float qz, float& x,
                                        float& y) {
  const float qmx = pick3(qx, qy, qz, b.mx);
  const float qot = pick3(qx, qy, qz, b.ot);
  const float qmn = pick3(qx, qy, qz, b.mn);
  x = __fsub_rn(__fadd_rn(__fmul_rn(b.umax, qmx), qot), b.pox);
  y = __fsub_rn(
      __fadd_rn(__fadd_rn(__fmul_rn(b.vmax, qmx), __fmul_rn(b.voth, qot)), __fmul_rn(b.sgn, qmn)),
      b.poy);
}

// project() on a point already in (mx, ot, mn) order: same operations, same order.
//
// sm_100 issues two fp32 multiplies (or adds) per instruction (FMUL2 / FADD2,
// PTX mul/sub.rn.f32x2 on register pairs).  The walk step is issue bound, so
// the projection pairs (vmax*q.x, voth*q.y) -- the point copy's first two
// words are already a register pair -- and the final (x1 - pox, y2 - poy):
// and (y1 + sgn*q.z) is one FFMA: sgn is +-1, so its product is exact and
// the fused add rounds once, exactly like the separate multiply and add.
// 6 FMA-pipe instructions instead of 9; every other product and sum is
// rounded exactly as before.  Caution: ptxas contracts a single-use f32x2
// product into a following f32x2 add (FFMA2) even under -fmad=false; here
// every f32x2 product feeds scalar adds or compares only, and
// tools/sass_steps.py fails the build check if a walk loop holds an FFMA2 or
// more FFMA than these sign-fused adds.
#ifndef TB_NO_F32X2
#define TB_F32X2 1
#endif
__device__ __forceinline__ void project_perm(const Basis& b, const float4& q, float& x, float& y) {
#ifdef TB_F32X2
  asm("{\n\t"
      ".reg .b64 s, c, m;\n\t"
      ".reg .f32 m0, m1, ux, x1, y1, y2;\n\t"
      "mov.b64 s, {%2, %3};\n\t"
      "mov.b64 c, {%6, %7};\n\t"
      "mul.rn.f32x2 m, s, c;\n\t"   // (vmax*q.x, voth*q.y)
      "mov.b64 {m0, m1}, m;\n\t"
      "mul.rn.f32 ux, %5, %2;\n\t"  // umax*q.x
      "add.rn.f32 x1, ux, %3;\n\t"  // + q.y
      "add.rn.f32 y1, m0, m1;\n\t"
      "fma.rn.f32 y2, %8, %4, y1;\n\t"  // y1 + sgn*q.z: sgn = +-1, the product is exact
      "mov.b64 s, {x1, y2};\n\t"
      "mov.b64 c, {%9, %10};\n\t"
      "sub.rn.f32x2 m, s, c;\n\t"   // (x1 - pox, y2 - poy)
      "mov.b64 {%0, %1}, m;\n\t"
      "}"
      : "=f"(x), "=f"(y)
      : "f"(q.x), "f"(q.y), "f"(q.z), "f"(b.umax), "f"(b.vmax), "f"(b.voth), "f"(b.sgn), "f"(b.pox), "f"(b.poy));
#else
  x = __fsub_rn(__fadd_rn(__fmul_rn(b.umax, q.x), q.y), b.pox);
  y = __fsub_rn(__fadd_rn(__fadd_rn(__fmul_rn(b.vmax, q.x), __fmul_rn(b.voth, q.y)), __fmul_rn(b.sgn, q.z)),
                b.poy);
#endif
}

// Algorithm 1, _kernels.pyx:94-102: index of the window point replaced by p3.
__device__ __forceinline__ int exit_face(float px, float py, const float (&p)[6]) {
  const float a0 = __fmul_rn(px, p[1]), b0 = __fmul_rn(py, p[0]);
  const float a2 = __fmul_rn(px, p[5]), b2 = __fmul_rn(py, p[4]);
  const float a1 = __fmul_rn(px, p[3]), b1 = __fmul_rn(py, p[2]);
  if (a0 < b0) return (a2 >= b2) ? 1 : 0;
  return (a1 < b1) ? 2 : 0;
}

// fp64 orientation of four points as init_ray computes it for the start
// quad (_kernels.pyx:133-147): e_k = P_k - P_0 in double, then
// e1x (e2y e3z - e2z e3y) + e1y (e2z e3x - e2x e3z) + e1z (e2x e3y - e2y e3x).
__device__ __forceinline__ double orientation(const float4& P0, const float4& P1, const float4& P2,
                                              const float4& P3) {
  const double e1x = __dsub_rn((double)P1.x, (double)P0.x);
  const double e1y = __dsub_rn((double)P1.y, (double)P0.y);
  const double e1z = __dsub_rn((double)P1.z, (double)P0.z);
  const double e2x = __dsub_rn((double)P2.x, (double)P0.x);
  const double e2y = __dsub_rn((double)P2.y, (double)P0.y);
  const double e2z = __dsub_rn((double)P2.z, (double)P0.z);
  const double e3x = __dsub_rn((double)P3.x, (double)P0.x);
  const double e3y = __dsub_rn((double)P3.y, (double)P0.y);
  const double e3z = __dsub_rn((double)P3.z, (double)P0.z);
  return __dadd_rn(__dadd_rn(__dmul_rn(e1x, __dsub_rn(__dmul_rn(e2y, e3z), __dmul_rn(e2z, e3y))),
                             __dmul_rn(e1y, __dsub_rn(__dmul_rn(e2z, e3x), __dmul_rn(e2x, e3z)))),
                   __dmul_rn(e1z, __dsub_rn(__dmul_rn(e2x, e3y), __dmul_rn(e2y, e3x))));
}

// ----------------------------------------------------------------------------
// Ray initialisation, _kernels.pyx:114-192.  Returns the selected slot.
__device__ __forceinline__ int init_ray(const MeshView& m, float o0, float o1, float o2, float d0,
                                        float d1, float d2, int start, Basis& b, uint32_t (&idx)[3],
                                        float (&p)[6]) {
  build_basis(o0, o1, o2, d0, d1, d2, b);
  const int4 qd = __ldg(&m.sv[start]);
  const int quad[4] = {qd.x, qd.y, qd.z, qd.w};
  // the four start points from the ray's axis-permuted copy: already in
  // projection order, no per-component selects
  const float4* __restrict__ Pp = m.pts + (size_t)perm_index(b.mx, b.ot) * (size_t)m.n_points;
  float q2[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    // 32-bit index (ids are < n_points < 2^31): one LEA pair per address
    // instead of a sign-extended 64-bit add + LEA pair
    const float4 Q = ldg_f4_at(Pp, (uint32_t)quad[i]);
    project_perm(b, Q, q2[2 * i], q2[2 * i + 1]);
  }
  // sign of the fp64 orientation rho of the sorted quad (_kernels.pyx:133-147),
  // precomputed per tet at upload (orient_kernel, identical arithmetic)
  const bool rho_pos = __ldg(&m.orient[start]) != 0;

#ifndef TB_INIT_LEGACY
  // Start-face selection (_kernels.pyx:153-186), branch-free over the tet's
  // six edges.  Face j's edge functions are 2-D cross products of its
  // corners: unswapped (a, b, c) = (i < k < l) gives (d0, d1, d2) =
  // (E_ik, E_kl, -E_il) with E_ik = q_i x q_k, and the swapped winding
  // (i, l, k) gives (-d2, -d1, -d0) of that.  fl(u - v) = -fl(v - u) and
  // products commute, so q_k x q_i is exactly -E_ik: six cross products
  // instead of twelve, the same IEEE values (a zero may change sign, which
  // no comparison below can see).  min(d0, d1, d2) keeps the reference's
  // sequential "if d < m" NaN behaviour: NaN iff d0 is NaN.
  float E[6];  // (0,1) (0,2) (0,3) (1,2) (1,3) (2,3)
  {
    const int ei[6] = {0, 0, 0, 1, 1, 2}, ek[6] = {1, 2, 3, 2, 3, 3};
#pragma unroll
    for (int e = 0; e < 6; ++e)
      E[e] = __fsub_rn(__fmul_rn(q2[2 * ei[e]], q2[2 * ek[e] + 1]), __fmul_rn(q2[2 * ei[e] + 1], q2[2 * ek[e]]));
  }
  int sel = -1, best_j = -1;
  float best_m = -3.4e38f;
#pragma unroll
  for (int j = 3; j >= 0; --j) {  // reversed: the first accepting face wins
    // corners i < k < l of face j (SLOT_A/B/C, _kernels.pyx:105-111)
    const int eik = (j == 0) ? 3 : ((j == 1) ? 1 : 0);  // (1,2) / (0,2) / (0,1) / (0,1)
    const int ekl = (j == 0) ? 5 : ((j == 1) ? 5 : ((j == 2) ? 4 : 3));  // (2,3) (2,3) (1,3) (1,2)
    const int eil = (j == 0) ? 4 : ((j == 1) ? 2 : ((j == 2) ? 2 : 1));  // (1,3) (0,3) (0,3) (0,2)
    const bool sw = ((j & 1) == 0) != rho_pos;
    const float A = E[eik], B = E[ekl], C = E[eil];
    const float dd0 = sw ? C : A;
    const float dd1 = sw ? -B : B;
    const float dd2 = sw ? -A : -C;
    const float mm = (dd0 != dd0) ? dd0 : fminf(fminf(dd0, dd1), dd2);
    const bool acc = mm >= 0.0f && fmaxf(fmaxf(dd0, dd1), dd2) > 0.0f;
    if (acc) sel = j;
  }
  // no accepting face: the first face of largest min (strictly greater)
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int eik = (j == 0) ? 3 : ((j == 1) ? 1 : 0);
    const int ekl = (j == 0) ? 5 : ((j == 1) ? 5 : ((j == 2) ? 4 : 3));
    const int eil = (j == 0) ? 4 : ((j == 1) ? 2 : ((j == 2) ? 2 : 1));
    const bool sw = ((j & 1) == 0) != rho_pos;
    const float A = E[eik], B = E[ekl], C = E[eil];
    const float dd0 = sw ? C : A;
    const float dd1 = sw ? -B : B;
    const float dd2 = sw ? -A : -C;
    const float mm = (dd0 != dd0) ? dd0 : fminf(fminf(dd0, dd1), dd2);
    if (mm > best_m) { best_m = mm; best_j = j; }
  }
#else
  int sel = -1, best_j = -1;
  float best_m = -3.4e38f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    // SLOT_A/B/C, _kernels.pyx:105-111: the face opposite slot j.
    const int ia = (j == 0) ? 1 : 0;
    const int ib = (j <= 1) ? 2 : 1;
    const int ic = (j == 3) ? 2 : 3;
    // outward winding swaps b <-> c; selects keep q2[] in registers
    const bool sw = ((j & 1) == 0) != rho_pos;
    const float ax = q2[2 * ia], ay = q2[2 * ia + 1];
    const float bx = sw ? q2[2 * ic] : q2[2 * ib], by = sw ? q2[2 * ic + 1] : q2[2 * ib + 1];
    const float cx = sw ? q2[2 * ib] : q2[2 * ic], cy = sw ? q2[2 * ib + 1] : q2[2 * ic + 1];
    const float dd0 = __fsub_rn(__fmul_rn(ax, by), __fmul_rn(ay, bx));
    const float dd1 = __fsub_rn(__fmul_rn(bx, cy), __fmul_rn(by, cx));
    const float dd2 = __fsub_rn(__fmul_rn(cx, ay), __fmul_rn(cy, ax));
    float mm = dd0;
    if (dd1 < mm) mm = dd1;
    if (dd2 < mm) mm = dd2;
    if (sel < 0) {
      if (mm >= 0.0f && (dd0 > 0.0f || dd1 > 0.0f || dd2 > 0.0f)) {
        sel = j;
      } else if (mm > best_m) {
        best_m = mm;
        best_j = j;
      }
    }
  }
#endif
  if (sel < 0) sel = best_j;
  // All-NaN windows (degenerate rays) leave best_j = -1; the reference reads
  // SLOT_A[-1] there (undefined behaviour).  Pin it to slot 0, the choice of
  // the reference's pure twin (np.argmax over NaNs, _kernels_py.py:134).
  if (sel < 0) sel = 0;
  const int ia = (sel == 0) ? 1 : 0;
  int ib = (sel <= 1) ? 2 : 1;
  int ic = (sel == 3) ? 2 : 3;
  if (((sel & 1) == 0) != rho_pos) { const int tmp = ib; ib = ic; ic = tmp; }
  // Dynamic selects over the 4 projected points (registers, no local memory).
  auto qsel = [&](int k, float& x, float& y, int& id) {
    x = k == 0 ? q2[0] : (k == 1 ? q2[2] : (k == 2 ? q2[4] : q2[6]));
    y = k == 0 ? q2[1] : (k == 1 ? q2[3] : (k == 2 ? q2[5] : q2[7]));
    id = k == 0 ? quad[0] : (k == 1 ? quad[1] : (k == 2 ? quad[2] : quad[3]));
  };
  int i0, i1, i2;
  qsel(ia, p[0], p[1], i0);
  qsel(ib, p[2], p[3], i1);
  qsel(ic, p[4], p[5], i2);
  idx[0] = (uint32_t)i0; idx[1] = (uint32_t)i1; idx[2] = (uint32_t)i2;
  return sel;
}

// ----------------------------------------------------------------------------
// Layout-specific record access.  A step needs: the xor word vx (to recover
// the fourth vertex i3) and, after the exit decision, the exit reference.
template <int L>
struct Record;

// (r01: ranks as IMAD/IMAD.HI sign products measured slower -- a longer
// dependent chain; the sign-bit sums of decide<L> compile to IMAD.IADD +
// LEA.HI pairs instead and are faster, see profiles/r01_experiments.md.)

// next_ref: the exit reference given the exited vertex idxf (Alg. 3/5/7).
// The 2-D walk computes it inside decide<L> (PTX, below) together with
// Algorithm 1 and the window update; these C++ forms serve the ScTP walk,
// which picks idxf with the fp64 predicate instead.
template <>
struct Record<16> {
  uint4 r;  // {vx, n0^n3, n1^n3, n2^n3}
  __device__ __forceinline__ void load(const MeshView& m, uint32_t t) { r = ldg_u4(&m.rec4[t]); }
  __device__ __forceinline__ uint32_t vxw() const { return r.x; }
  // Alg. 7, _kernels.pyx:222-235:
  //   rank = #{idx0, idx1, idx2, i3 < idxf}, order_a = #{idx0, idx1, idx2 < i3},
  //   nref = prev ^ nx[order_a] (if != 3) ^ nx[rank] (if != 3).
  __device__ __forceinline__ uint32_t next_ref(const uint32_t (&idx)[3], uint32_t i3, uint32_t idxf,
                                               uint32_t prev) const {
    const uint4 nx = make_uint4(r.y, r.z, r.w, 0u);  // nx[3] := 0 makes the "!= 3" xors unconditional
    const int rank = (idx[0] < idxf) + (idx[1] < idxf) + (idx[2] < idxf) + (i3 < idxf);
    const int order_a = (idx[0] < i3) + (idx[1] < i3) + (idx[2] < i3);
    return prev ^ pick4u(nx, order_a) ^ pick4u(nx, rank);
  }
};

template <>
struct Record<20> {
  uint32_t v;  // vx
  uint4 n;     // n0..n3
  __device__ __forceinline__ void load(const MeshView& m, uint32_t t) {
    v = __ldg(&m.vx[t]);
    n = ldg_u4(&m.rec4[t]);
  }
  __device__ __forceinline__ uint32_t vxw() const { return v; }
  // Alg. 5, _kernels.pyx:207-221: nref = n[#{idx0, idx1, idx2, i3 < idxf}].
  __device__ __forceinline__ uint32_t next_ref(const uint32_t (&idx)[3], uint32_t i3, uint32_t idxf,
                                               uint32_t) const {
    return pick4u(n, (idx[0] < idxf) + (idx[1] < idxf) + (idx[2] < idxf) + (i3 < idxf));
  }
};

template <>
struct Record<32> {
  uint4 a, n;  // {v0, v1, v2, vx}, {n0..n3}
  __device__ __forceinline__ void load(const MeshView& m, uint32_t t) {
    a = ldg_u4(&m.rec4[2 * (size_t)t]);
    n = ldg_u4(&m.rec4[2 * (size_t)t + 1]);
  }
  __device__ __forceinline__ uint32_t vxw() const { return a.w; }
  // Alg. 3, _kernels.pyx:204-209.
  __device__ __forceinline__ uint32_t next_ref(const uint32_t (&)[3], uint32_t, uint32_t idxf,
                                               uint32_t) const {
    uint32_t nref = n.w;
    if (a.x == idxf) nref = n.x;
    if (a.y == idxf) nref = n.y;
    if (a.z == idxf) nref = n.z;
    return nref;
  }
};

// TetMesh-80: sorted ids, sorted-slot refs and the four vertices inline.
template <>
struct Record<80> {
  uint4 v, n;
  const uint4* base;
  __device__ __forceinline__ void load(const MeshView& m, uint32_t t) {
    base = m.rec4 + 5 * (size_t)t;
    v = ldg_u4(base);
    n = ldg_u4(base + 1);
  }
  __device__ __forceinline__ uint32_t vxw() const { return v.x ^ v.y ^ v.z ^ v.w; }
  __device__ __forceinline__ int slot_of(uint32_t id) const {
    return (v.x == id) ? 0 : ((v.y == id) ? 1 : ((v.z == id) ? 2 : 3));
  }
  // Vertex coordinates of slot k from the inline block (floats 8..19).
  __device__ __forceinline__ float4 vertex(int k) const {
    const float* f = reinterpret_cast<const float*>(base + 2);
    return make_float4(__ldg(f + 3 * k), __ldg(f + 3 * k + 1), __ldg(f + 3 * k + 2), 0.0f);
  }
  __device__ __forceinline__ uint32_t next_ref(const uint32_t (&)[3], uint32_t, uint32_t idxf,
                                               uint32_t) const {
    return pick4u(n, slot_of(idxf));
  }
};

template <int L>
__device__ __forceinline__ float4 fetch_vertex(const MeshView& m, const Record<L>&, uint32_t i3) {
  return ldg_f4(&m.pts[i3]);
}
template <>
__device__ __forceinline__ float4 fetch_vertex<80>(const MeshView&, const Record<80>& r,
                                                   uint32_t i3) {
  return r.vertex(r.slot_of(i3));
}

// ----------------------------------------------------------------------------
// Axis-permuted point copies.  The projection reads q[mx], q[ot], q[mn] in
// that order (_kernels.pyx:89-91); selecting them per step costs six SELs
// plus predicate traffic in an issue-bound loop.  The device keeps six
// copies of the points, copy k holding (q[mx], q[ot], q[mn], 0) for the
// k-th (mx, ot) pair, so one 16 B load delivers the components already in
// projection order.  Copy 0 is (x, y, z): MeshView.pts[i] stays the plain
// point for every other user.
__device__ __forceinline__ const float4* ray_points(const MeshView& m, const Basis& b) {
  return m.pts + (size_t)perm_index(b.mx, b.ot) * (size_t)m.n_points;
}


// ----------------------------------------------------------------------------
// The decision half of a step in PTX: Algorithm 1 (_kernels.pyx:94-102), the
// exit reference (Alg. 3/5/7, _kernels.pyx:195-235) and the window update,
// with the exit face kept in predicates.  Written in C++ the compiler
// materialises "f == 0" as an integer (4 ALU ops) because every predicate
// register is live at that point, recomputes one compare, and extracts the
// rank bits with three more ops; here f0 is one PLOP3, the rank bits one R2P,
// and the ranks are sums of sign bits ((a - b) >> 31 == [a < b] for ids
// < 2^31) whose subtractions run on the FMA pipe as IMAD.IADD.  The walk is
// ALU-pipe bound (ncu, r01), so this is where its time goes: tet20
// 71 -> 59 SASS per step, 41 -> 30 ALU-pipe ops (tools/sass_steps.py).
// Same IEEE operations in the same order as before (mul.rn, ordered
// setp.lt / setp.ge), so results are bit-identical.
//
// Operands: %0 nref; %1-%3 idx (in/out); %4-%9 p (in/out); %10 qx; %11 qy;
// %12 i3; %13.. layout words.
// The six products of Algorithm 1 as three FMUL2: (qx, qy) * (p[2k+1], p[2k])
// = (a_k, e_k); the window pair (y_k, x_k) stays one aligned register pair.
#ifdef TB_F32X2
#define TB_STEP_PRODUCTS                               \
  ".reg .b64 Q2, W2, A2;\n\t"                          \
  "mov.b64 Q2, {%10, %11};\n\t"                        \
  "mov.b64 W2, {%5, %4};\n\t"                          \
  "mul.rn.f32x2 A2, Q2, W2;\n\t"                       \
  "mov.b64 {a0, e0}, A2;\n\t"                          \
  "mov.b64 W2, {%9, %8};\n\t"                          \
  "mul.rn.f32x2 A2, Q2, W2;\n\t"                       \
  "mov.b64 {a2, e2}, A2;\n\t"                          \
  "mov.b64 W2, {%7, %6};\n\t"                          \
  "mul.rn.f32x2 A2, Q2, W2;\n\t"                       \
  "mov.b64 {a1, e1}, A2;\n\t"
#else
#define TB_STEP_PRODUCTS                               \
  "mul.rn.f32 a0, %10, %5;\n\t"                        \
  "mul.rn.f32 e0, %11, %4;\n\t"                        \
  "mul.rn.f32 a2, %10, %9;\n\t"                        \
  "mul.rn.f32 e2, %11, %8;\n\t"                        \
  "mul.rn.f32 a1, %10, %7;\n\t"                        \
  "mul.rn.f32 e1, %11, %6;\n\t"
#endif
#define TB_STEP_HEAD                                   \
  "{\n\t"                                              \
  ".reg .pred c0, c1, c2, f1, f2, g, q0, q1;\n\t"      \
  ".reg .f32 a0, a1, a2, e0, e1, e2;\n\t"              \
  ".reg .b32 fi, rk, t, lo, hi;\n\t"                   \
  TB_STEP_PRODUCTS                                     \
  "setp.lt.f32 c0, a0, e0;\n\t"                        \
  "setp.ge.f32 c2, a2, e2;\n\t"                        \
  "setp.lt.f32 c1, a1, e1;\n\t"                        \
  "and.pred f1, c0, c2;\n\t"                           \
  "not.pred c0, c0;\n\t"                               \
  "and.pred f2, c0, c1;\n\t"                           \
  "or.pred g, f1, f2;\n\t"                             \
  "selp.b32 fi, %2, %1, f1;\n\t"                       \
  "@f2 mov.b32 fi, %3;\n\t"
// rk = #{idx0, idx1, idx2, i3 < fi}
#define TB_STEP_RANK                                   \
  "sub.u32 t, %1, fi;\n\t"                             \
  "shr.u32 rk, t, 31;\n\t"                             \
  "sub.u32 t, %2, fi;\n\t"                             \
  "shr.u32 t, t, 31;\n\t"                              \
  "add.u32 rk, rk, t;\n\t"                             \
  "sub.u32 t, %3, fi;\n\t"                             \
  "shr.u32 t, t, 31;\n\t"                              \
  "add.u32 rk, rk, t;\n\t"                             \
  "sub.u32 t, %12, fi;\n\t"                            \
  "shr.u32 t, t, 31;\n\t"                              \
  "add.u32 rk, rk, t;\n\t"                             \
  "and.b32 t, rk, 1;\n\t"                              \
  "setp.ne.u32 q0, t, 0;\n\t"                          \
  "and.b32 t, rk, 2;\n\t"                              \
  "setp.ne.u32 q1, t, 0;\n\t"
#define TB_STEP_TAIL                                   \
  "@!g mov.b32 %1, %12;\n\t"                           \
  "@!g mov.f32 %4, %10;\n\t"                           \
  "@!g mov.f32 %5, %11;\n\t"                           \
  "@f1 mov.b32 %2, %12;\n\t"                           \
  "@f1 mov.f32 %6, %10;\n\t"                           \
  "@f1 mov.f32 %7, %11;\n\t"                           \
  "@f2 mov.b32 %3, %12;\n\t"                           \
  "@f2 mov.f32 %8, %10;\n\t"                           \
  "@f2 mov.f32 %9, %11;\n\t"                           \
  "}"
#define TB_STEP_OUTS                                                                                        \
  "=r"(nref), "+r"(idx[0]), "+r"(idx[1]), "+r"(idx[2]), "+f"(p[0]), "+f"(p[1]), "+f"(p[2]), "+f"(p[3]), \
      "+f"(p[4]), "+f"(p[5])

template <int L>
__device__ __forceinline__ uint32_t decide(const Record<L>& rec, uint32_t (&idx)[3], float (&p)[6], float qx,
                                           float qy, uint32_t i3, uint32_t prev);

// Alg. 5 (Tet20): nref = n[rank].  %13-%16 = n0..n3.
template <>
__device__ __forceinline__ uint32_t decide<20>(const Record<20>& rec, uint32_t (&idx)[3], float (&p)[6], float qx,
                                               float qy, uint32_t i3, uint32_t) {
  uint32_t nref;
  asm(TB_STEP_HEAD TB_STEP_RANK
      "selp.b32 lo, %14, %13, q0;\n\t"
      "selp.b32 hi, %16, %15, q0;\n\t"
      "selp.b32 %0, hi, lo, q1;\n\t" TB_STEP_TAIL
      : TB_STEP_OUTS
      : "f"(qx), "f"(qy), "r"(i3), "r"(rec.n.x), "r"(rec.n.y), "r"(rec.n.z), "r"(rec.n.w));
  return nref;
}

// Alg. 7 (Tet16): nref = prev ^ nx[order_a] ^ nx[rank], nx[3] = 0,
// order_a = #{idx0, idx1, idx2 < i3}.  %13-%15 = nx0..nx2, %16 = prev.
template <>
__device__ __forceinline__ uint32_t decide<16>(const Record<16>& rec, uint32_t (&idx)[3], float (&p)[6], float qx,
                                               float qy, uint32_t i3, uint32_t prev) {
  uint32_t nref;
  asm(TB_STEP_HEAD TB_STEP_RANK
      "selp.b32 lo, %14, %13, q0;\n\t"
      "selp.b32 hi, 0, %15, q0;\n\t"
      "selp.b32 rk, hi, lo, q1;\n\t"
      "sub.u32 t, %1, %12;\n\t"
      "shr.u32 fi, t, 31;\n\t"
      "sub.u32 t, %2, %12;\n\t"
      "shr.u32 t, t, 31;\n\t"
      "add.u32 fi, fi, t;\n\t"
      "sub.u32 t, %3, %12;\n\t"
      "shr.u32 t, t, 31;\n\t"
      "add.u32 fi, fi, t;\n\t"
      "and.b32 t, fi, 1;\n\t"
      "setp.ne.u32 q0, t, 0;\n\t"
      "and.b32 t, fi, 2;\n\t"
      "setp.ne.u32 q1, t, 0;\n\t"
      "selp.b32 lo, %14, %13, q0;\n\t"
      "selp.b32 hi, 0, %15, q0;\n\t"
      "selp.b32 lo, hi, lo, q1;\n\t"
      "lop3.b32 %0, %16, rk, lo, 0x96;\n\t" TB_STEP_TAIL  // prev ^ nx[rank] ^ nx[order_a], one LOP3
      : TB_STEP_OUTS
      : "f"(qx), "f"(qy), "r"(i3), "r"(rec.r.y), "r"(rec.r.z), "r"(rec.r.w), "r"(prev));
  return nref;
}

// Alg. 3 (Tet32; also TetMesh-80, whose sorted ids and sorted-slot refs are
// the same words): nref = n_i where v_i == idxf (i = 0..2), else n3.
// %13-%15 = v0..v2, %16-%19 = n0..n3.
__device__ __forceinline__ uint32_t decide_alg3(uint32_t (&idx)[3], float (&p)[6], float qx, float qy, uint32_t i3,
                                                const uint4& v, const uint4& n) {
  uint32_t nref;
  asm(TB_STEP_HEAD
      "mov.b32 %0, %19;\n\t"
      "setp.eq.u32 q0, %13, fi;\n\t"
      "@q0 mov.b32 %0, %16;\n\t"
      "setp.eq.u32 q0, %14, fi;\n\t"
      "@q0 mov.b32 %0, %17;\n\t"
      "setp.eq.u32 q0, %15, fi;\n\t"
      "@q0 mov.b32 %0, %18;\n\t" TB_STEP_TAIL
      : TB_STEP_OUTS
      : "f"(qx), "f"(qy), "r"(i3), "r"(v.x), "r"(v.y), "r"(v.z), "r"(n.x), "r"(n.y), "r"(n.z), "r"(n.w));
  return nref;
}

template <>
__device__ __forceinline__ uint32_t decide<32>(const Record<32>& rec, uint32_t (&idx)[3], float (&p)[6], float qx,
                                               float qy, uint32_t i3, uint32_t) {
  return decide_alg3(idx, p, qx, qy, i3, rec.a, rec.n);
}

template <>
__device__ __forceinline__ uint32_t decide<80>(const Record<80>& rec, uint32_t (&idx)[3], float (&p)[6], float qx,
                                               float qy, uint32_t i3, uint32_t) {
  return decide_alg3(idx, p, qx, qy, i3, rec.v, rec.n);
}

// One traversal step into tet `nxt`, _kernels.pyx:238-259.  Updates the
// window (idx, p) and returns the exit reference of `nxt`.  `P` is the ray's
// axis-permuted point copy (ignored for TetMesh-80, whose points are inline).
// kClamp keeps the point index in bounds for meshes whose records were not
// validated at upload (a corrupt record could send i3 anywhere); a mesh that
// passed validate_kernel cannot produce an out-of-range i3 (see there).
template <int L, bool kClamp = true>
__device__ __forceinline__ uint32_t advance(const MeshView& m, const float4* __restrict__ P, const Basis& b,
                                            uint32_t (&idx)[3], float (&p)[6], uint32_t nxt, uint32_t prev) {
  Record<L> rec;
  rec.load(m, nxt);
#ifndef TB_NO_XOR_EARLY
  // idx0 ^ idx1 ^ idx2 formed before the record arrives (opaque to ptxas,
  // which otherwise folds vx in first): one LOP3 between the vx load and the
  // point address instead of two (r02 A/B +0.4 ... +1.5 %)
  uint32_t wx;
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(wx) : "r"(idx[0]), "r"(idx[1]), "r"(idx[2]));
  uint32_t i3 = wx ^ rec.vxw();
#else
  uint32_t i3 = idx[0] ^ idx[1] ^ idx[2] ^ rec.vxw();
#endif
  float qx, qy;
  if constexpr (L != 80) {
    if (kClamp) i3 = min(i3, (uint32_t)m.n_points - 1u);  // corrupt record: stay in bounds
    const float4 q = ldg_f4_at(P, i3);
    project_perm(b, q, qx, qy);
    return decide<L>(rec, idx, p, qx, qy, i3, prev);
  } else {
    // TetMesh-80: the new vertex's slot in the sorted ids, then its inline
    // coordinates loaded straight in projection order (q[mx], q[ot], q[mn])
    // -- no per-step axis selects; the decision is Tet32's (same words).
    // A corrupt record cannot leave the 80-byte record (k is 0..3).
    const int k = (rec.v.x == i3) ? 0 : ((rec.v.y == i3) ? 1 : ((rec.v.z == i3) ? 2 : 3));
    const float* f = reinterpret_cast<const float*>(rec.base + 2) + 3 * k;
    const float4 q = make_float4(__ldg(f + b.mx), __ldg(f + b.ot), __ldg(f + b.mn), 0.0f);
    project_perm(b, q, qx, qy);
    return decide<80>(rec, idx, p, qx, qy, i3, prev);
  }
}

// ----------------------------------------------------------------------------
// fp64 epilogue: t of the ray/triangle pair, _kernels_py._mt_t
// (_kernels_py.py:435-454) -- reciprocal-multiply form, numpy's np.cross
// operation order, plane-distance fallback for det == 0.  The dot products
// are numpy's einsum("ij,ij->i") over 3 terms, which numpy 2.3 reduces as
// SIMD lanes [p0, p1, p2, 0] summed pairwise: (p0 + p2) + p1 (measured
// against the reference's outputs, tests/test_oracle.py).
__device__ __forceinline__ double einsum3(double x0, double y0, double x1, double y1, double x2, double y2) {
  return __dadd_rn(__dadd_rn(__dmul_rn(x0, y0), __dmul_rn(x2, y2)), __dmul_rn(x1, y1));
}

__device__ __forceinline__ double mt_t(double ox, double oy, double oz, double dx, double dy,
                                       double dz, const double* __restrict__ T) {
  const double ax = __ldg(T + 0), ay = __ldg(T + 1), az = __ldg(T + 2);
  const double bx = __ldg(T + 3), by = __ldg(T + 4), bz = __ldg(T + 5);
  const double cx = __ldg(T + 6), cy = __ldg(T + 7), cz = __ldg(T + 8);
  const double e1x = __dsub_rn(bx, ax), e1y = __dsub_rn(by, ay), e1z = __dsub_rn(bz, az);
  const double e2x = __dsub_rn(cx, ax), e2y = __dsub_rn(cy, ay), e2z = __dsub_rn(cz, az);
  // pv = cross(d, e2)
  const double pvx = __dsub_rn(__dmul_rn(dy, e2z), __dmul_rn(dz, e2y));
  const double pvy = __dsub_rn(__dmul_rn(dz, e2x), __dmul_rn(dx, e2z));
  const double pvz = __dsub_rn(__dmul_rn(dx, e2y), __dmul_rn(dy, e2x));
  const double det = einsum3(e1x, pvx, e1y, pvy, e1z, pvz);
  const double tvx = __dsub_rn(ox, ax), tvy = __dsub_rn(oy, ay), tvz = __dsub_rn(oz, az);
  if (det != 0.0) {
    const double inv = __ddiv_rn(1.0, det);
    // cross(tv, e1)
    const double qx = __dsub_rn(__dmul_rn(tvy, e1z), __dmul_rn(tvz, e1y));
    const double qy = __dsub_rn(__dmul_rn(tvz, e1x), __dmul_rn(tvx, e1z));
    const double qz = __dsub_rn(__dmul_rn(tvx, e1y), __dmul_rn(tvy, e1x));
    return __dmul_rn(einsum3(e2x, qx, e2y, qy, e2z, qz), inv);
  }
  // parallel: plane distance
  const double nx = __dsub_rn(__dmul_rn(e1y, e2z), __dmul_rn(e1z, e2y));
  const double ny = __dsub_rn(__dmul_rn(e1z, e2x), __dmul_rn(e1x, e2z));
  const double nz = __dsub_rn(__dmul_rn(e1x, e2y), __dmul_rn(e1y, e2x));
  const double denom = einsum3(nx, dx, ny, dy, nz, dz);
  if (denom == 0.0) return 0.0;
  const double num = einsum3(nx, __dsub_rn(ax, ox), ny, __dsub_rn(ay, oy), nz, __dsub_rn(az, oz));
  return __ddiv_rn(num, denom);
}

// Segment/triangle parameter of the compiled shadow walk, _kernels.pyx:495-524
// (division form, not the reciprocal of mt_t).
__device__ __forceinline__ double seg_tri_t(const double (&o)[3], const double (&d)[3],
                                            const double* __restrict__ T) {
  const double ax = __ldg(T + 0), ay = __ldg(T + 1), az = __ldg(T + 2);
  const double e1x = __dsub_rn(__ldg(T + 3), ax), e1y = __dsub_rn(__ldg(T + 4), ay),
               e1z = __dsub_rn(__ldg(T + 5), az);
  const double e2x = __dsub_rn(__ldg(T + 6), ax), e2y = __dsub_rn(__ldg(T + 7), ay),
               e2z = __dsub_rn(__ldg(T + 8), az);
  const double pvx = __dsub_rn(__dmul_rn(d[1], e2z), __dmul_rn(d[2], e2y));
  const double pvy = __dsub_rn(__dmul_rn(d[2], e2x), __dmul_rn(d[0], e2z));
  const double pvz = __dsub_rn(__dmul_rn(d[0], e2y), __dmul_rn(d[1], e2x));
  const double det = __dadd_rn(__dadd_rn(__dmul_rn(e1x, pvx), __dmul_rn(e1y, pvy)), __dmul_rn(e1z, pvz));
  const double tvx = __dsub_rn(o[0], ax), tvy = __dsub_rn(o[1], ay), tvz = __dsub_rn(o[2], az);
  if (det != 0.0) {
    const double qx = __dsub_rn(__dmul_rn(tvy, e1z), __dmul_rn(tvz, e1y));
    const double qy = __dsub_rn(__dmul_rn(tvz, e1x), __dmul_rn(tvx, e1z));
    const double qz = __dsub_rn(__dmul_rn(tvx, e1y), __dmul_rn(tvy, e1x));
    return __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(e2x, qx), __dmul_rn(e2y, qy)), __dmul_rn(e2z, qz)), det);
  }
  const double nx = __dsub_rn(__dmul_rn(e1y, e2z), __dmul_rn(e1z, e2y));
  const double ny = __dsub_rn(__dmul_rn(e1z, e2x), __dmul_rn(e1x, e2z));
  const double nz = __dsub_rn(__dmul_rn(e1x, e2y), __dmul_rn(e1y, e2x));
  const double denom = __dadd_rn(__dadd_rn(__dmul_rn(nx, d[0]), __dmul_rn(ny, d[1])), __dmul_rn(nz, d[2]));
  if (denom == 0.0) return 0.0;
  const double num = __dadd_rn(__dadd_rn(__dmul_rn(nx, __dsub_rn(ax, o[0])), __dmul_rn(ny, __dsub_rn(ay, o[1]))),
                               __dmul_rn(nz, __dsub_rn(az, o[2])));
  return __ddiv_rn(num, denom);
}

// _det3, _kernels.pyx:408-413.
__device__ __forceinline__ double det3(double ax, double ay, double az, double bx, double by,
                                       double bz, double cx, double cy, double cz) {
  return __dadd_rn(__dadd_rn(__dmul_rn(ax, __dsub_rn(__dmul_rn(by, cz), __dmul_rn(bz, cy))),
                             __dmul_rn(ay, __dsub_rn(__dmul_rn(bz, cx), __dmul_rn(bx, cz)))),
                   __dmul_rn(az, __dsub_rn(__dmul_rn(bx, cy), __dmul_rn(by, cx))));
}

// fp64 point-in-tet with relative epsilon, _kernels.pyx:373-405.
__device__ __forceinline__ bool contains(const MeshView& m, uint32_t t, const double (&q)[3]) {
  const int4 v = __ldg(&m.sv[t]);
  const int vid[4] = {v.x, v.y, v.z, v.w};
  double P[4][3];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 f = ldg_f4(&m.pts[vid[i]]);
    P[i][0] = f.x; P[i][1] = f.y; P[i][2] = f.z;
  }
  const double vol = det3(__dsub_rn(P[1][0], P[0][0]), __dsub_rn(P[1][1], P[0][1]), __dsub_rn(P[1][2], P[0][2]),
                          __dsub_rn(P[2][0], P[0][0]), __dsub_rn(P[2][1], P[0][1]), __dsub_rn(P[2][2], P[0][2]),
                          __dsub_rn(P[3][0], P[0][0]), __dsub_rn(P[3][1], P[0][1]), __dsub_rn(P[3][2], P[0][2]));
  const double s = vol > 0.0 ? 1.0 : -1.0;
  const double eps = __dadd_rn(__dmul_rn(1e-10, fabs(vol)), 1e-300);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double S[4][3];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
      for (int k = 0; k < 3; ++k) S[i][k] = (i == j) ? q[k] : P[i][k];
    }
    const double dd = det3(__dsub_rn(S[1][0], S[0][0]), __dsub_rn(S[1][1], S[0][1]), __dsub_rn(S[1][2], S[0][2]),
                           __dsub_rn(S[2][0], S[0][0]), __dsub_rn(S[2][1], S[0][1]), __dsub_rn(S[2][2], S[0][2]),
                           __dsub_rn(S[3][0], S[0][0]), __dsub_rn(S[3][1], S[0][1]), __dsub_rn(S[3][2], S[0][2]));
    if (__dmul_rn(s, dd) < -eps) return false;
  }
  return true;
}

}  // namespace tb
