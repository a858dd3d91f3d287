// tetb200.cu -- sm_100a kernels and the C ABI declared in include/tetb200.h.
//
// Hot path: batch.cast_rays -> _kernels.cast_rays
// (/root/reference/pkg/src/tetray/batch.py:39-80, _kernels.pyx:271-370).
// One lane per ray walks the compact xor-linked records of an HBM-resident
// mesh; the host epilogue of batch.cast_rays (triangle id, fp64 t, back tet;
// batch.py:57-71) is fused into the termination path.  See DESIGN.md.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>
#include <string>

#include "../../include/tetb200.h"
#include "sctp.cuh"
#include "traverse.cuh"

using namespace tb;

// ----------------------------------------------------------------------------
// Error plumbing
static thread_local std::string g_last_error;

static int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

#define TB_CUDA(call)                                                                  \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      return set_error(e_ == cudaErrorMemoryAllocation ? TB_E_OOM : TB_E_CUDA,         \
                       "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, \
                       __LINE__);                                                      \
    }                                                                                  \
  } while (0)

struct tb_mesh {
  int device = 0;
  int layout = 0;
  int64_t n_points = 0, n_tets = 0, n_cf = 0, n_tri = 0;
  float4* pts = nullptr;
  uint4* rec4 = nullptr;
  uint32_t* vx = nullptr;
  int4* sv = nullptr;
  uint4* sn = nullptr;
  int32_t* cf_tri = nullptr;
  int2* cf_tets = nullptr;
  double* tri = nullptr;
  uint8_t* orient = nullptr;
  bool safe = false;  // records validated at upload (validate_kernel): no per-step index clamp
  int64_t hbm_bytes = 0;
  int64_t hot_bytes = 0;

  MeshView view() const {
    MeshView v;
    v.pts = pts; v.rec4 = rec4; v.vx = vx; v.sv = sv; v.sn = sn;
    v.cf_tri = cf_tri; v.cf_tets = cf_tets; v.tri = tri; v.orient = orient;
    v.n_points = n_points; v.n_tets = n_tets; v.n_cf = n_cf; v.n_tri = n_tri;
    return v;
  }
};

namespace {

constexpr int kBlock = 128;
// cast_kernel block size (r01 A/B: 32 / 64 / 256 threads were 1-7 % slower)
#ifndef TB_CAST_BLOCK
#define TB_CAST_BLOCK 128
#endif
constexpr int kCastBlock = TB_CAST_BLOCK;
#ifndef TB_CAST_MIN_BLOCKS
#define TB_CAST_MIN_BLOCKS (1280 / TB_CAST_BLOCK)  // cast_kernel residency target: 48 registers (r01 A/B)
#endif
// Residency per walk (r02 A/B, tools/gpu_r02k.sh): coherent Tet16 / Tet20 walks
// issue best at 10 blocks per SM (48 registers: 12 blocks spill into the step
// and lose 2 %); walks bound by gather latency -- Tet32's 32 B records on the
// 50 M-tet mesh, and every direction-binned (kGather) secondary batch -- gain
// from 12 blocks (40 registers, the epilogue's ray reloaded after the walk):
// config 5 +5 %, config 4 +2.6 %.
#ifndef TB_CAST_MIN_BLOCKS_LATENCY
#define TB_CAST_MIN_BLOCKS_LATENCY (1536 / TB_CAST_BLOCK)
#endif
// ... except the binned Tet20 walk, whose 20 B records (two loads) do not fit
// 40 registers without spilling into the step: 10 blocks, r02 A/B config-2
// frame secondaries 2237 -> 2487 Mrays/s, config-4 rays on Tet20 3200 -> 3385.
#ifndef TB_GATHER20_MIN_BLOCKS
#define TB_GATHER20_MIN_BLOCKS TB_CAST_MIN_BLOCKS
#endif
template <int L, bool kGather>
constexpr int cast_min_blocks() {
  return (L == 20 && kGather) ? TB_GATHER20_MIN_BLOCKS
                              : ((L == 32 || kGather) ? TB_CAST_MIN_BLOCKS_LATENCY : TB_CAST_MIN_BLOCKS);
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

inline unsigned grid_for(int64_t n, int block) { return (unsigned)((n + block - 1) / block); }

// ----------------------------------------------------------------------------
// Mesh build kernels (run once per upload).
// Six axis-permuted float4 copies of the points (traverse.cuh, perm_index):
// copy k = mx * 2 + (ot > mx ? ot - 1 : ot) holds (q[mx], q[ot], q[mn], 0).
__global__ void pad_points_kernel(const float* __restrict__ xyz, float4* __restrict__ out, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float q[3] = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
#pragma unroll
  for (int mx = 0; mx < 3; ++mx) {
#pragma unroll
    for (int ot = 0; ot < 3; ++ot) {
      if (ot == mx) continue;
      const int mn = 3 - mx - ot;
      out[(size_t)perm_index(mx, ot) * (size_t)n + i] = make_float4(q[mx], q[ot], q[mn], 0.0f);
    }
  }
}

// Per-tet sign of the start-quad orientation used by init_ray and the ScTP
// predicate (_kernels.pyx:133-147, traversal.py:499): computed once here with
// the same fp64 expression instead of once per ray (or per ScTP step).
__global__ void orient_kernel(const int4* __restrict__ sv, const float4* __restrict__ pts,
                              uint8_t* __restrict__ out, int64_t n, int64_t n_points) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int4 v = sv[i];
  // indices clamped only to keep a corrupt table in bounds (validate_kernel flags it)
  const int64_t hi = n_points - 1;
  auto c = [&](int k) { return k < 0 ? 0 : (k > hi ? hi : (int64_t)k); };
  out[i] = orientation(pts[c(v.x)], pts[c(v.y)], pts[c(v.z)], pts[c(v.w)]) > 0.0 ? 1 : 0;
}

// Upload-time record validation.  A walk computes the next vertex as
// i3 = idx0 ^ idx1 ^ idx2 ^ vx[nxt]; it lies in [0, n_points) whenever the
// window is a face of nxt, which holds by induction when (1) every
// side_verts row is strictly ascending and in range, (2) the layout records
// equal the ones the side tables define (_records_from_tables,
// tetmesh.py:299-320), and (3) every plain neighbour reference is symmetric
// and shares the face (u = sn[t][j] holds t's face opposite slot j, and
// sn[u][k] == t for u's vertex k off that face).  A mesh passing all three
// runs the kernels without the per-step index clamp; any violation (e.g. a
// record mutated by a test) keeps the clamp, so a corrupt mesh still cannot
// read out of bounds.  (4) extends the proof across constrained faces, which
// the locate / shadow walks cross through cf_tets and the epilogue gathers
// through cf_tri.  Sets *bad on any violation.
__global__ void validate_kernel(int layout, const int4* __restrict__ sv, const uint4* __restrict__ sn,
                                const uint4* __restrict__ rec4, const uint32_t* __restrict__ vx, int64_t n_tets,
                                int64_t n_points, const int32_t* __restrict__ cf_tri, const int2* __restrict__ cf_tets,
                                int64_t n_cf, int64_t n_tri, unsigned int* __restrict__ bad) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_tets) return;
  const int4 v = sv[t];
  bool ok = v.x >= 0 && v.x < v.y && v.y < v.z && v.z < v.w && (int64_t)v.w < n_points;
  const uint4 nb = sn[t];
  const uint32_t x = (uint32_t)(v.x ^ v.y ^ v.z ^ v.w);
  if (layout == 16) {
    const uint4 r = rec4[t];
    ok = ok && r.x == x && r.y == (nb.x ^ nb.w) && r.z == (nb.y ^ nb.w) && r.w == (nb.z ^ nb.w);
  } else if (layout == 20) {
    const uint4 r = rec4[t];
    ok = ok && vx[t] == x && r.x == nb.x && r.y == nb.y && r.z == nb.z && r.w == nb.w;
  } else if (layout == 32) {
    const uint4 a = rec4[2 * t], r = rec4[2 * t + 1];
    ok = ok && a.x == (uint32_t)v.x && a.y == (uint32_t)v.y && a.z == (uint32_t)v.z && a.w == x && r.x == nb.x &&
         r.y == nb.y && r.z == nb.z && r.w == nb.w;
  }
  const int vv[4] = {v.x, v.y, v.z, v.w};
  const uint32_t nn[4] = {nb.x, nb.y, nb.z, nb.w};
  for (int j = 0; j < 4 && ok; ++j) {
    uint32_t u = nn[j];
    if ((u & kConstrained) != 0u) {
      // (4) a constrained ref names a row of the cf tables that lists t as one
      // side, a scene triangle in range, and, on the other side, -1 (hull) or
      // a tet sharing the face whose slot holds the same tagged ref -- the
      // epilogue, locate and shadow walks gather through exactly these
      const uint32_t cfi = u & kPayload;
      if (cfi >= (uint64_t)n_cf) { ok = false; break; }
      const int2 ct = cf_tets[cfi];
      const int32_t tri = cf_tri[cfi];
      if ((ct.x != (int32_t)t && ct.y != (int32_t)t) || tri < 0 || (int64_t)tri >= n_tri) { ok = false; break; }
      const int32_t other = (ct.x == (int32_t)t) ? ct.y : ct.x;
      if (other < 0) continue;  // hull
      if ((int64_t)other >= n_tets || (int64_t)other == t) { ok = false; break; }
      u = (uint32_t)other;  // then the face-sharing check below, expecting the tagged ref back
    } else if (u >= (uint64_t)n_tets) {
      // the boundary sentinel: the walk stops there.  Any other plain ref past
      // the table is corrupt and keeps the clamped walk, so on a validated
      // mesh "ref < n_tets" and "ref < kBoundary" agree (walk_ray's loop test)
      if (u != kBoundary) { ok = false; break; }
      continue;
    }
    if ((int64_t)u == t) { ok = false; break; }
    const uint32_t back = (nn[j] & kConstrained) ? nn[j] : (uint32_t)t;
    const int4 w = sv[u];
    const int ww[4] = {w.x, w.y, w.z, w.w};
    const uint4 un = sn[u];
    const uint32_t unn[4] = {un.x, un.y, un.z, un.w};
    int shared = 0, off = -1;
    for (int k = 0; k < 4; ++k) {
      bool in_face = false;
      for (int i = 0; i < 4; ++i) in_face = in_face || (i != j && vv[i] == ww[k]);
      if (in_face) ++shared; else off = k;
    }
    ok = shared == 3 && off >= 0 && unn[off] == back;
  }
  if (!ok) atomicOr(bad, 1u);
}

__global__ void split_tet20_kernel(const uint32_t* __restrict__ rec, uint32_t* __restrict__ vx,
                                   uint4* __restrict__ nb, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const uint32_t* r = rec + 5 * i;
    vx[i] = r[0];
    nb[i] = make_uint4(r[1], r[2], r[3], r[4]);
  }
}

__global__ void build_tet80_kernel(const int4* __restrict__ sv, const uint4* __restrict__ sn,
                                   const float4* __restrict__ pts, uint4* __restrict__ out, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int4 v = sv[i];
  const float4 a = pts[v.x], b = pts[v.y], c = pts[v.z], d = pts[v.w];
  uint4* o = out + 5 * i;
  o[0] = make_uint4((uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w);
  o[1] = sn[i];
  o[2] = make_uint4(__float_as_uint(a.x), __float_as_uint(a.y), __float_as_uint(a.z), __float_as_uint(b.x));
  o[3] = make_uint4(__float_as_uint(b.y), __float_as_uint(b.z), __float_as_uint(c.x), __float_as_uint(c.y));
  o[4] = make_uint4(__float_as_uint(c.z), __float_as_uint(d.x), __float_as_uint(d.y), __float_as_uint(d.z));
}

// ----------------------------------------------------------------------------
// Warp-cooperative load of one (n, 3) float32 row per lane: the warp reads
// its 96 consecutive floats as three fully coalesced 128 B rows and
// redistributes them with shuffles, so every input byte is requested once
// (this matters most when the rays live in mapped host memory and each
// request crosses PCIe).  Must be called by all 32 lanes of the warp.
__device__ __forceinline__ void load_xyz_warp(const float* __restrict__ a, int64_t r, int64_t n, float& x,
                                              float& y, float& z) {
  const int lane = threadIdx.x & 31;
  const int64_t base = 3 * (r - lane);  // first float of the warp's window (16 B aligned: 96 floats per warp)
  const int64_t lim = 3 * n;
  // lanes 0..23 fetch one 16 B vector each (384 B per warp, one request per
  // 128 B line); the ragged tail falls back to scalar loads
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  const int64_t e0 = base + 4 * lane;
  if (lane < 24) {
    if (e0 + 3 < lim && ((reinterpret_cast<uintptr_t>(a) & 15u) == 0)) {
      v = __ldg(reinterpret_cast<const float4*>(a + e0));
    } else {
      if (e0 < lim) v.x = __ldg(a + e0);
      if (e0 + 1 < lim) v.y = __ldg(a + e0 + 1);
      if (e0 + 2 < lim) v.z = __ldg(a + e0 + 2);
      if (e0 + 3 < lim) v.w = __ldg(a + e0 + 3);
    }
  }
  float out[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const int e = 3 * lane + c;  // element of the warp's 96-float window
    const float s0 = __shfl_sync(0xffffffffu, v.x, e >> 2);
    const float s1 = __shfl_sync(0xffffffffu, v.y, e >> 2);
    const float s2 = __shfl_sync(0xffffffffu, v.z, e >> 2);
    const float s3 = __shfl_sync(0xffffffffu, v.w, e >> 2);
    const int k = e & 3;
    out[c] = (k == 0) ? s0 : ((k == 1) ? s1 : ((k == 2) ? s2 : s3));
  }
  x = out[0];
  y = out[1];
  z = out[2];
}

// ----------------------------------------------------------------------------
// Shared termination + fused epilogue (batch.py:57-71).
//
// Ray origin / direction for the epilogue's fp64 t.  Kept live through the
// walk they cost six registers (plus the 64-bit ray index) across the whole
// loop; device-resident rays are instead re-read -- only for hits -- after the
// walk, which frees the registers for the loop (r02 A/B: +0.9 ... +1.5 %;
// -DTB_NO_RELOAD_RAY restores the register copy).  The
// loads are volatile so the front end cannot merge them with the init loads
// and keep the values live after all.
struct RayRef {
  const float* o;
  const float* d;
  int64_t q;
  __device__ __forceinline__ static float ld(const float* a) {
    float v;
    asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(a));
    return v;
  }
  __device__ __forceinline__ double mt(const MeshView& m, int32_t tri) const {
    const float* po = o + 3 * q;
    const float* pd = d + 3 * q;
    return mt_t((double)ld(po), (double)ld(po + 1), (double)ld(po + 2), (double)ld(pd), (double)ld(pd + 1),
                (double)ld(pd + 2), m.tri + 9 * (int64_t)tri);
  }
};
// The ray's values kept in registers (host-mapped rays, the other walks).
struct RayVal {
  float o0, o1, o2, d0, d1, d2;
  __device__ __forceinline__ double mt(const MeshView& m, int32_t tri) const {
    return mt_t((double)o0, (double)o1, (double)o2, (double)d0, (double)d1, (double)d2, m.tri + 9 * (int64_t)tri);
  }
};

// Ray I/O cache hints: the walk's result stores, and the ray loads of walks
// that read their rays in place, are issued evict-first (st/ld.global.cs), so
// the streamed ray and hit arrays give way to the mesh in L2.  Same-process
// A/B (profiles/r02_ab_stream_hints.jsonl, bit-identical): config 2 +1.0 %
// in the A/B harness (neutral through bench.py), binned config 4 +0.3 %,
// frame secondaries +0.6 %, configs 3 / 5 within 0.2 %.  Gathered (binned) walks keep cached loads: evict-first ray loads
// through the permutation cost config 4 0.5 %.  TB_STREAM_HINTS=0 turns the
// hints off (1: stores only, 2: every ray load too, 3: the default).
#ifndef TB_STREAM_HINTS
#define TB_STREAM_HINTS 3
#endif
#if TB_STREAM_HINTS >= 3
#define TB_LDR(p) (kGather ? __ldg(p) : __ldcs(p))
#elif TB_STREAM_HINTS >= 2
#define TB_LDR(p) __ldcs(p)
#else
#define TB_LDR(p) __ldg(p)
#endif
#if TB_STREAM_HINTS >= 1
#define TB_STR(p, v) __stcs((p), (v))
#else
#define TB_STR(p, v) (*(p) = (v))
#endif

template <class Ray>
__device__ __forceinline__ void write_result_ray(const MeshView& m, int64_t r, uint8_t st, uint32_t ref,
                                                 uint32_t cur, int vis, const Ray& ray, uint8_t* status,
                                                 int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle,
                                                 double* t, int32_t* tet_back) {
  if (status != nullptr) TB_STR(reinterpret_cast<signed char*>(status) + r, (signed char)st);
  const int32_t cfi = (st == kHit) ? (int32_t)(ref & kPayload) : -1;
  TB_STR(cf + r, cfi);
  TB_STR(tet + r, (int32_t)cur);
  TB_STR(visited + r, vis);
  if (triangle != nullptr || t != nullptr || tet_back != nullptr) {
    int32_t tri = -1, back = -1;
    double tt = INFINITY;
    // A corrupt (unvalidated) mesh can carry a constrained ref past the cf
    // table: no gather then -- the host wrappers raise IndexError on cf >=
    // n_cf, as the reference's batch epilogue does (batch.py:63).
    if (cfi >= 0 && cfi < m.n_cf) {
      tri = __ldg(&m.cf_tri[cfi]);
      if (t != nullptr && (uint32_t)tri < (uint64_t)m.n_tri) tt = ray.mt(m, tri);
      const int2 ct = __ldg(&m.cf_tets[cfi]);
      back = (ct.x == (int32_t)cur) ? ct.y : ct.x;
    }
    if (triangle != nullptr) TB_STR(triangle + r, tri);
    if (t != nullptr) TB_STR(t + r, tt);
    if (tet_back != nullptr) TB_STR(tet_back + r, back);
  }
}

__device__ __forceinline__ void write_result(const MeshView& m, int64_t r, uint8_t st, uint32_t ref,
                                             uint32_t cur, int vis, float o0, float o1, float o2,
                                             float d0, float d1, float d2, uint8_t* status, int32_t* cf,
                                             int32_t* tet, int32_t* visited, int32_t* triangle,
                                             double* t, int32_t* tet_back) {
  write_result_ray(m, r, st, ref, cur, vis, RayVal{o0, o1, o2, d0, d1, d2}, status, cf, tet, visited, triangle,
                   t, tet_back);
}

// Batch epilogue alone (batch.py:57-71) from stored cf / tet: the multi-GPU
// frame assembly ships only status / cf / tet / visited to the root, which
// derives triangle, t and tet_back here from its own copy of the rays.
__global__ void __launch_bounds__(256) epilogue_kernel(MeshView m, int64_t n, const float* __restrict__ o,
                                                       const float* __restrict__ d, const int32_t* __restrict__ cf,
                                                       const int32_t* __restrict__ tet, int32_t* __restrict__ triangle,
                                                       double* __restrict__ t, int32_t* __restrict__ tet_back) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int32_t cfi = __ldg(cf + r);
  int32_t tri = -1, back = -1;
  double tt = INFINITY;
  if (cfi >= 0 && cfi < m.n_cf) {
    tri = __ldg(&m.cf_tri[cfi]);
    if (t != nullptr && (uint32_t)tri < (uint64_t)m.n_tri)
      tt = mt_t((double)__ldg(o + 3 * r), (double)__ldg(o + 3 * r + 1), (double)__ldg(o + 3 * r + 2),
                (double)__ldg(d + 3 * r), (double)__ldg(d + 3 * r + 1), (double)__ldg(d + 3 * r + 2),
                m.tri + 9 * (int64_t)tri);
    const int2 ct = __ldg(&m.cf_tets[cfi]);
    const int32_t cur = __ldg(tet + r);
    back = (ct.x == cur) ? ct.y : ct.x;
  }
  if (triangle != nullptr) triangle[r] = tri;
  if (t != nullptr) t[r] = tt;
  if (tet_back != nullptr) tet_back[r] = back;
}

// ----------------------------------------------------------------------------
// Cycle guard without the O(n_tets) walk.  The reference stops a ray once it
// has visited more than n_tets tets (_kernels.pyx:365-368); rays that tie
// exactly on lattice-aligned meshes loop forever and pay n_tets steps (50 M
// on config 5).  The step is a pure function of (ref, idx[3], cur) -- the
// projected window p[] is a function of idx for a fixed ray -- so once a
// state repeats the walk is periodic.  Brent's algorithm finds the period
// lam; the walk then jumps a whole number of periods (state unchanged) and
// finishes the last < lam steps, giving exactly the reference's terminating
// tet and visited = n_tets + 1.  Only walks longer than kCycleCheckAfter
// steps enter here, so the hot loop is untouched.  Returns true on guard.
constexpr uint32_t kCycleCheckAfter = 1u << 14;

template <int L, bool kClamp = true>
__device__ __forceinline__ bool long_walk(const MeshView& m, const float4* __restrict__ P, const Basis& b,
                                       uint32_t (&idx)[3], float (&p)[6], uint32_t& ref, uint32_t& cur, int& vis) {
  const uint32_t n_tets = (uint32_t)m.n_tets;
  uint32_t s_ref = ref, s_i0 = idx[0], s_i1 = idx[1], s_i2 = idx[2], s_cur = cur;
  uint32_t power = 1, lam = 0;
  bool jumped = false;
  while (ref < n_tets) {
    const uint32_t nxt = ref;
    ref = advance<L, kClamp>(m, P, b, idx, p, nxt, cur);
    cur = nxt;
    if ((uint32_t)++vis > n_tets) return true;
    ++lam;
    if (!jumped && ref == s_ref && idx[0] == s_i0 && idx[1] == s_i1 && idx[2] == s_i2 && cur == s_cur) {
      const uint64_t remaining = (uint64_t)n_tets + 1 - (uint64_t)vis;  // steps until the guard
      vis += (int)((remaining / lam) * lam);
      jumped = true;
      if ((uint32_t)vis > n_tets) return true;
      continue;
    }
    if (lam == power) {  // Brent: move the tortoise, double the window
      s_ref = ref; s_i0 = idx[0]; s_i1 = idx[1]; s_i2 = idx[2]; s_cur = cur;
      power <<= 1;
      lam = 0;
    }
  }
  return false;
}

// The walk of one ray, _kernels.pyx:343-369: init (basis, start window,
// first exit), the 4x-unrolled xor walk, the exact single-step tail with the
// cycle guard.  On return `cur` is the terminating tet, `ref` the exit
// reference, `vis` the visited count and `st` the status.  Shared by the
// launch-per-128-rays kernel and the dynamically scheduled one.
#ifndef TB_UNROLL
#define TB_UNROLL 8  // r02 A/B: 8 vs 4 -- loop bookkeeping per step 1.25 -> 0.6 SASS (+0.5 ... +2 %)
#endif
constexpr int kUnroll = TB_UNROLL;
static_assert(kUnroll == 4 || kUnroll == 8, "the unrolled walk body is written out for 4 or 8 steps");

template <int L, bool kClamp>
__device__ __forceinline__ void walk_ray(const MeshView& m, float o0, float o1, float o2, float d0, float d1,
                                         float d2, uint32_t& cur, uint32_t& ref, int& vis, uint8_t& st) {
  Basis b;
  uint32_t idx[3];
  float p[6];
  const int j = init_ray(m, o0, o1, o2, d0, d1, d2, (int)cur, b, idx, p);
  ref = pick4u(__ldg(&m.sn[cur]), j);
  const float4* __restrict__ P = ray_points(m, b);
  vis = 1;
  st = 255;
  const uint32_t n_tets = (uint32_t)m.n_tets;
  // Every plain tet reference is < n_tets; the boundary sentinel
  // (0x7FFFFFFF) and constrained refs (bit 31) are >= n_tets, so one
  // unsigned compare per step decides "keep walking" (corrupt refs also land
  // outside and are classified below).  On a validated mesh every plain ref
  // is < n_tets and every terminal one is >= kBoundary (validate_kernel), so
  // the test is against the immediate kBoundary: no register and no per-step
  // copy of n_tets (ptxas re-read it from a uniform register every step).
  const uint32_t live = kClamp ? n_tets : kBoundary;
  const uint32_t fast_limit = n_tets < kCycleCheckAfter ? n_tets : kCycleCheckAfter;
  // Unrolled fast loop: the visited count and its threshold test once per
  // kUnroll steps (saves ~2.5 ALU-pipe ops per step, r01 A/B +1.5-3 %).  It
  // only runs while all kUnroll steps fit under fast_limit; the exact
  // single-step loop below finishes the walk.
  // (The early exits add their own step count, so no per-step counter.)
  while (ref < live && vis + kUnroll <= (int)fast_limit) {
    uint32_t nxt;
#define TB_WALK_STEP(k)                                   \
    nxt = ref;                                            \
    ref = advance<L, kClamp>(m, P, b, idx, p, nxt, cur);  \
    cur = nxt;                                            \
    if (ref >= live) { vis += (k); break; }
    TB_WALK_STEP(1) TB_WALK_STEP(2) TB_WALK_STEP(3)
#if TB_UNROLL == 8
    TB_WALK_STEP(4) TB_WALK_STEP(5) TB_WALK_STEP(6) TB_WALK_STEP(7)
#endif
#undef TB_WALK_STEP
    nxt = ref;
    ref = advance<L, kClamp>(m, P, b, idx, p, nxt, cur);
    cur = nxt;
    vis += kUnroll;
  }
  while (ref < live) {
    const uint32_t nxt = ref;
    ref = advance<L, kClamp>(m, P, b, idx, p, nxt, cur);
    cur = nxt;
    if ((uint32_t)++vis > fast_limit) {
      // Long walk: finish it in the cycle-detecting slow path (exact).
      if ((uint32_t)vis > n_tets || long_walk<L, kClamp>(m, P, b, idx, p, ref, cur, vis)) st = kError;
      break;
    }
  }
  if (st != kError) st = (ref == kBoundary) ? kMiss : ((ref & kConstrained) ? kHit : kError);
}

// ----------------------------------------------------------------------------
// Primary traversal kernel: one lane per ray, _kernels.pyx:343-369.

// kHostRays: the ray arrays are mapped pinned host memory (zero-copy e2e
// path) -- load them with the warp-cooperative 16 B row loads so every input
// byte crosses PCIe once.  Device-resident rays use three plain coalesced
// loads per array instead (fewer instructions: no shuffles; r01 A/B +3 %),
// issued together with the start-tet load.  (An L2 prefetch of the next
// wave's rays measured neutral-to-negative and was dropped.)  The
// __launch_bounds__ minimum of 10 blocks keeps the walk at 48 registers
// (10 blocks / 40 warps per SM) -- without it the branch-free basis grew the
// kernel to 53 registers and 9 blocks (r01 A/B: config 5 -2.7 %).
// kScatter: ray r's hits go to slot oidx[r] of the output arrays instead of
// r -- the multi-GPU frame assembly, where the outputs are the root GPU's
// full-frame arrays mapped into this process (CUDA IPC over NVLink) and each
// ray's result is stored there by the epilogue the moment its walk ends.
// kGather: ray r is read from index ridx[r] -- the direction-binned schedule
// walks the rays in binned order straight from the caller's arrays, so the
// binning pass writes only the 4-byte permutation; with kScatter its results
// go back to oidx[r], or to ridx[r] (the ray's own slot) when oidx is null.
template <int L, bool kClamp, bool kHostRays, bool kScatter, bool kGather = false, bool kBlockMap = false>
__global__ void __launch_bounds__(kCastBlock, (cast_min_blocks<L, kGather>())) cast_kernel(MeshView m, int64_t n, const float* __restrict__ o,
                                                      const float* __restrict__ d,
                                                      const int32_t* __restrict__ start,
                                                      uint8_t* __restrict__ status, int32_t* __restrict__ cf,
                                                      int32_t* __restrict__ tet, int32_t* __restrict__ visited,
                                                      int32_t* __restrict__ triangle, double* __restrict__ t,
                                                      int32_t* __restrict__ tet_back,
                                                      const int64_t* __restrict__ oidx,
                                                      const int32_t* __restrict__ ridx,
                                                      const int32_t* __restrict__ bmap) {
  // kBlockMap: block b walks the rays of block bmap[b] (a caller-chosen launch
  // order of whole 128-ray blocks, e.g. longest first by a previous frame's
  // walk lengths -- tb_cast_rays_ordered); rays and results stay in place
  const int64_t blk = kBlockMap ? (int64_t)__ldg(bmap + blockIdx.x) : (int64_t)blockIdx.x;
  const int64_t r = blk * (int64_t)blockDim.x + threadIdx.x;
  float o0, o1, o2, d0, d1, d2;
  uint32_t cur;
  if constexpr (kHostRays) {
    load_xyz_warp(o, r, n, o0, o1, o2);  // whole warp participates (shuffles)
    load_xyz_warp(d, r, n, d0, d1, d2);
    if (r >= n) return;
    cur = (uint32_t)__ldg(start + r);
  } else {
    if (r >= n) return;
    const int64_t q = kGather ? (int64_t)__ldg(ridx + r) : r;
    cur = (uint32_t)TB_LDR(start + q);
    o0 = TB_LDR(o + 3 * q); o1 = TB_LDR(o + 3 * q + 1); o2 = TB_LDR(o + 3 * q + 2);
    d0 = TB_LDR(d + 3 * q); d1 = TB_LDR(d + 3 * q + 1); d2 = TB_LDR(d + 3 * q + 2);
  }
  uint32_t ref;
  int vis;
  uint8_t st;
  walk_ray<L, kClamp>(m, o0, o1, o2, d0, d1, d2, cur, ref, vis, st);
  // kGather alone reads through ridx and stores in place; the binned walk
  // stores back through its permutation (oidx null: the index already
  // loaded) or through a composed one (multi-GPU scatter of a binned batch)
  int64_t w = r;
  if constexpr (kScatter) w = (kGather && oidx == nullptr) ? (int64_t)__ldg(ridx + r) : __ldg(oidx + r);
  if constexpr (kHostRays) {
    // Zero-copy outputs cross PCIe as the warps' stores: every array gets
    // >= 128 B per warp store except the 1-byte status (32 B per warp).  A
    // full block stages its 128 status bytes in shared memory and writes them
    // as one 128 B store (r01: e2e +2.6 %; staging every array instead gained
    // nothing more).  No thread of a full block exited early, so the barrier
    // is safe; the ragged last block writes status directly.
    if ((int64_t)(blockIdx.x + 1) * kCastBlock <= n && (reinterpret_cast<uintptr_t>(status) & 3u) == 0) {
      __shared__ uint32_t s_status[kCastBlock / 4];
      reinterpret_cast<uint8_t*>(s_status)[threadIdx.x] = st;
      write_result(m, w, st, ref, cur, vis, o0, o1, o2, d0, d1, d2, nullptr, cf, tet, visited, triangle, t,
                   tet_back);
      __syncthreads();
      if (threadIdx.x < kCastBlock / 4)
        reinterpret_cast<uint32_t*>(status + (int64_t)blockIdx.x * kCastBlock)[threadIdx.x] = s_status[threadIdx.x];
      return;
    }
  }
#ifndef TB_NO_RELOAD_RAY
  if constexpr (!kHostRays) {
    const int64_t q = kGather ? (int64_t)__ldg(ridx + r) : r;
    write_result_ray(m, w, st, ref, cur, vis, RayRef{o, d, q}, status, cf, tet, visited, triangle, t, tet_back);
    return;
  }
#endif
  write_result(m, w, st, ref, cur, vis, o0, o1, o2, d0, d1, d2, status, cf, tet, visited, triangle, t,
               tet_back);
}

// ----------------------------------------------------------------------------
// Dynamically scheduled walk (schedule 5, "dynamic"): one wave of resident
// blocks; each warp takes the next 32 consecutive rays from a global counter
// (one atomicAdd per chunk, issued a chunk ahead so its latency hides under
// the walk) until the batch is exhausted.  Chunks go out in batch order, so
// the frame-order wavefront of the block launch is kept, but a warp whose
// rays end early takes new work at once instead of holding its block's slot
// until the block's slowest warp ends, and no SM idles through a tail of
// late-launched blocks (ncu r01, config 2: achieved occupancy 54 % of a 62.5 %
// limit, SMs active 89 %).  Same init / walk / epilogue code (walk_ray), so
// results are identical.  *next must be 0 at launch.
template <int L, bool kClamp>
__global__ void __launch_bounds__(kCastBlock, TB_CAST_MIN_BLOCKS) cast_dyn_kernel(
    MeshView m, int64_t n, const float* __restrict__ o, const float* __restrict__ d,
    const int32_t* __restrict__ start, uint8_t* __restrict__ status, int32_t* __restrict__ cf,
    int32_t* __restrict__ tet, int32_t* __restrict__ visited, int32_t* __restrict__ triangle, double* __restrict__ t,
    int32_t* __restrict__ tet_back, unsigned long long* __restrict__ next) {
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(next, 32ull);
  base = __shfl_sync(0xffffffffu, base, 0);
  while (base < (unsigned long long)n) {
    unsigned long long ahead = 0;
    if (lane == 0) ahead = atomicAdd(next, 32ull);  // the next chunk, fetched while this one walks
    const int64_t r = (int64_t)base + lane;
    if (r < n) {
      uint32_t cur = (uint32_t)__ldg(start + r);
      const float o0 = __ldg(o + 3 * r), o1 = __ldg(o + 3 * r + 1), o2 = __ldg(o + 3 * r + 2);
      const float d0 = __ldg(d + 3 * r), d1 = __ldg(d + 3 * r + 1), d2 = __ldg(d + 3 * r + 2);
      uint32_t ref;
      int vis;
      uint8_t st;
      walk_ray<L, kClamp>(m, o0, o1, o2, d0, d1, d2, cur, ref, vis, st);
      write_result(m, r, st, ref, cur, vis, o0, o1, o2, d0, d1, d2, status, cf, tet, visited, triangle, t,
                   tet_back);
    }
    base = __shfl_sync(0xffffffffu, ahead, 0);
  }
}

// ----------------------------------------------------------------------------
// Persistent variant with warp-level ray refill, for divergent (incoherent)
// batches.  One lane per ray, but a lane whose ray terminates takes the next
// ray of its warp's stream instead of idling until the warp's longest ray
// ends (incoherent secondaries run at ~50 % SIMT efficiency otherwise, ncu
// r01 cfg4).  Each warp owns the interleaved 32-ray chunks
// c = warp, warp + n_warps, ... (static, balanced, no atomics); a refill
// round hands consecutive stream positions to the idle lanes (ballot + popc)
// whenever at most kRefillBelow lanes are still walking, then every lane
// walks up to kStepsPerRound steps.  Results per ray are identical to
// cast_kernel (same init, step, guard and epilogue code).
constexpr int kRefillBelow = 20;
constexpr int kStepsPerRound = 16;

template <int L>
__global__ void __launch_bounds__(kBlock) cast_persist_kernel(
    MeshView m, int64_t n, const float* __restrict__ o, const float* __restrict__ d,
    const int32_t* __restrict__ start, uint8_t* __restrict__ status, int32_t* __restrict__ cf,
    int32_t* __restrict__ tet, int32_t* __restrict__ visited, int32_t* __restrict__ triangle,
    double* __restrict__ t, int32_t* __restrict__ tet_back) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t n_chunks = (n + 31) >> 5;
  const int64_t stream_len = (n_chunks > warp) ? ((n_chunks - warp + n_warps - 1) / n_warps) * 32 : 0;
  const uint32_t n_tets = (uint32_t)m.n_tets;
  const uint32_t fast_limit = n_tets < kCycleCheckAfter ? n_tets : kCycleCheckAfter;
  int64_t pos = 0;  // warp-uniform position in this warp's ray stream
  bool has = false;
  int64_t r = 0;
  float o0 = 0.f, o1 = 0.f, o2 = 0.f, d0 = 0.f, d1 = 0.f, d2 = 0.f;
  Basis b;
  uint32_t idx[3] = {0, 0, 0};
  float p[6] = {0, 0, 0, 0, 0, 0};
  uint32_t ref = 0, cur = 0;
  int vis = 0;
  const float4* __restrict__ P = m.pts;
  while (true) {
    const unsigned act = __ballot_sync(0xffffffffu, has);
    if (__popc(act) <= kRefillBelow) {
      if (pos >= stream_len && act == 0u) break;
      const unsigned need = ~act;
      const int64_t q = pos + __popc(need & ((1u << lane) - 1u));
      if (!has && q < stream_len) {
        r = (warp + (q >> 5) * n_warps) * 32 + (q & 31);
        if (r < n) {
          o0 = __ldg(o + 3 * r); o1 = __ldg(o + 3 * r + 1); o2 = __ldg(o + 3 * r + 2);
          d0 = __ldg(d + 3 * r); d1 = __ldg(d + 3 * r + 1); d2 = __ldg(d + 3 * r + 2);
          cur = (uint32_t)__ldg(start + r);
          const int j = init_ray(m, o0, o1, o2, d0, d1, d2, (int)cur, b, idx, p);
          ref = pick4u(__ldg(&m.sn[cur]), j);
          P = ray_points(m, b);
          vis = 1;
          has = true;
        }
      }
      pos += __popc(need);
    }
    if (!has) continue;
    uint8_t st = 255;
#pragma unroll 1
    for (int s = 0; s < kStepsPerRound; ++s) {
      if (ref >= n_tets) { st = 0; break; }
      const uint32_t nxt = ref;
      ref = advance<L>(m, P, b, idx, p, nxt, cur);
      cur = nxt;
      if ((uint32_t)++vis > fast_limit) {
        st = ((uint32_t)vis > n_tets || long_walk<L>(m, P, b, idx, p, ref, cur, vis)) ? kError : 0;
        break;
      }
    }
    if (st != 255) {  // terminated this round
      if (st != kError) st = (ref == kBoundary) ? kMiss : ((ref & kConstrained) ? kHit : kError);
      write_result(m, r, st, ref, cur, vis, o0, o1, o2, d0, d1, d2, status, cf, tet, visited, triangle, t,
                   tet_back);
      has = false;
    }
  }
}

// ----------------------------------------------------------------------------
// Block-compacting persistent variant, for divergent (incoherent) batches.
//
// The per-lane refill above loses because every refill runs init_ray with
// only the idle lanes of a warp active, so init is paid at a fraction of
// SIMT width over and over.  Here the unit of scheduling is the block:
// every round each walking lane takes up to `rounds` steps, then the block
// compacts its surviving rays into the lowest thread slots through shared
// memory (20 words of walk state per ray, SoA so the exchange is
// bank-conflict free) and refills the free tail slots -- whole warps plus
// at most one partial warp -- with fresh rays, which therefore initialise at
// (nearly) full SIMT width.  Walking warps stay dense until the block's ray
// stream runs dry; then survivors concentrate in the fewest warps and the
// emptied warps only wait at the barriers.  Per-ray results are identical to
// cast_kernel: same init_ray / advance / long_walk / write_result code, and
// a ray's step sequence does not depend on which lane walks it.
//
// Rays are dealt to blocks in 32-ray chunks round-robin (chunk c -> block
// c mod gridDim), so every block sees the whole image/batch and the tail is
// balanced without atomics or per-call scratch.
constexpr int kCompactWords = 20;

template <int L, int BT, bool kClamp>
__global__ void __launch_bounds__(BT) cast_compact_kernel(
    MeshView m, int64_t n, const float* __restrict__ o, const float* __restrict__ d,
    const int32_t* __restrict__ start, uint8_t* __restrict__ status, int32_t* __restrict__ cf,
    int32_t* __restrict__ tet, int32_t* __restrict__ visited, int32_t* __restrict__ triangle,
    double* __restrict__ t, int32_t* __restrict__ tet_back, int steps_per_round) {
  constexpr int NW = BT / 32;
  __shared__ uint32_t sw[kCompactWords][BT];
  __shared__ int warp_cnt[NW];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t G = gridDim.x;
  const int64_t n_chunks = (n + 31) >> 5;
  const int64_t my_chunks = n_chunks > (int64_t)blockIdx.x ? (n_chunks - 1 - blockIdx.x) / G + 1 : 0;
  const int64_t stream_len = my_chunks * 32;
  const uint32_t n_tets = (uint32_t)m.n_tets;
  const uint32_t fast_limit = n_tets < kCycleCheckAfter ? n_tets : kCycleCheckAfter;

  int64_t qpos = 0;  // block-uniform position in this block's ray stream
  int A = 0;         // block-uniform: threads [0, A) hold a walking ray
  bool has = false;
  uint32_t r = 0;
  Basis b;
  b.mn = b.mx = b.ot = 0;
  b.umax = b.vmax = b.voth = b.sgn = b.pox = b.poy = 0.f;
  int perm = 0;
  uint32_t idx[3] = {0, 0, 0};
  float p[6] = {0, 0, 0, 0, 0, 0};
  uint32_t ref = 0, cur = 0;
  int vis = 0;
  while (true) {
    // refill: free slots [A, BT) take the next rays of the block's stream
    if (tid >= A) {
      const int64_t q = qpos + (tid - A);
      if (q < stream_len) {
        const int64_t rr = (blockIdx.x + (q >> 5) * G) * 32 + (q & 31);
        if (rr < n) {
          r = (uint32_t)rr;
          const float o0 = __ldg(o + 3 * rr), o1 = __ldg(o + 3 * rr + 1), o2 = __ldg(o + 3 * rr + 2);
          const float d0 = __ldg(d + 3 * rr), d1 = __ldg(d + 3 * rr + 1), d2 = __ldg(d + 3 * rr + 2);
          cur = (uint32_t)__ldg(start + rr);
          const int j = init_ray(m, o0, o1, o2, d0, d1, d2, (int)cur, b, idx, p);
          ref = pick4u(__ldg(&m.sn[cur]), j);
          perm = perm_index(b.mx, b.ot);
          vis = 1;
          has = true;
        }
      }
    }
    qpos += BT - A;
    // walk: up to steps_per_round steps per lane
    if (has) {
      const float4* __restrict__ P = m.pts + (size_t)perm * (size_t)m.n_points;
      bool done = false, guard = false;
      int budget = steps_per_round;
      // 4x unrolled part, as in cast_kernel (exits add their own count)
      while (budget >= 4 && ref < n_tets && vis + 4 <= (int)fast_limit) {
        uint32_t nxt = ref;
        ref = advance<L, kClamp>(m, P, b, idx, p, nxt, cur);
        cur = nxt;
        if (ref >= n_tets) { vis += 1; break; }
        nxt = ref;
        ref = advance<L, kClamp>(m, P, b, idx, p, nxt, cur);
        cur = nxt;
        if (ref >= n_tets) { vis += 2; break; }
        nxt = ref;
        ref = advance<L, kClamp>(m, P, b, idx, p, nxt, cur);
        cur = nxt;
        if (ref >= n_tets) { vis += 3; break; }
        nxt = ref;
        ref = advance<L, kClamp>(m, P, b, idx, p, nxt, cur);
        cur = nxt;
        vis += 4;
        budget -= 4;
      }
#pragma unroll 1
      for (; budget > 0 && ref < n_tets; --budget) {
        const uint32_t nxt = ref;
        ref = advance<L, kClamp>(m, P, b, idx, p, nxt, cur);
        cur = nxt;
        if ((uint32_t)++vis > fast_limit) {
          guard = (uint32_t)vis > n_tets || long_walk<L, kClamp>(m, P, b, idx, p, ref, cur, vis);
          done = true;
          break;
        }
      }
      if (!done && ref >= n_tets) done = true;
      if (done) {
        const uint8_t st = guard ? kError : ((ref == kBoundary) ? kMiss : ((ref & kConstrained) ? kHit : kError));
        const float o0 = __ldg(o + 3 * (int64_t)r), o1 = __ldg(o + 3 * (int64_t)r + 1),
                    o2 = __ldg(o + 3 * (int64_t)r + 2);
        const float d0 = __ldg(d + 3 * (int64_t)r), d1 = __ldg(d + 3 * (int64_t)r + 1),
                    d2 = __ldg(d + 3 * (int64_t)r + 2);
        write_result(m, r, st, ref, cur, vis, o0, o1, o2, d0, d1, d2, status, cf, tet, visited, triangle, t,
                     tet_back);
        has = false;
      }
    }
    // compaction: survivors move to slots [0, total)
    const unsigned bal = __ballot_sync(0xffffffffu, has);
    if (lane == 0) warp_cnt[wid] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int c = warp_cnt[w];
      before += (w < wid) ? c : 0;
      total += c;
    }
    if (total == 0 && qpos >= stream_len) break;
    const int slot = before + __popc(bal & ((1u << lane) - 1u));
    const bool move_out = has && slot != tid;
    if (move_out) {
      sw[0][slot] = r;
      sw[1][slot] = __float_as_uint(b.umax);
      sw[2][slot] = __float_as_uint(b.vmax);
      sw[3][slot] = __float_as_uint(b.voth);
      sw[4][slot] = __float_as_uint(b.sgn);
      sw[5][slot] = __float_as_uint(b.pox);
      sw[6][slot] = __float_as_uint(b.poy);
      sw[7][slot] = (uint32_t)perm;
      sw[8][slot] = idx[0];
      sw[9][slot] = idx[1];
      sw[10][slot] = idx[2];
#pragma unroll
      for (int k = 0; k < 6; ++k) sw[11 + k][slot] = __float_as_uint(p[k]);
      sw[17][slot] = ref;
      sw[18][slot] = cur;
      sw[19][slot] = (uint32_t)vis;
    }
    __syncthreads();
    // a slot keeps its registers when its own ray stayed in place
    const bool stay = has && slot == tid;
    if (tid < total && !stay) {
      r = sw[0][tid];
      b.umax = __uint_as_float(sw[1][tid]);
      b.vmax = __uint_as_float(sw[2][tid]);
      b.voth = __uint_as_float(sw[3][tid]);
      b.sgn = __uint_as_float(sw[4][tid]);
      b.pox = __uint_as_float(sw[5][tid]);
      b.poy = __uint_as_float(sw[6][tid]);
      perm = (int)sw[7][tid];
      // the axes, for project() (TetMesh-80 reads inline xyz): invert perm_index
      b.mx = perm >> 1;
      b.ot = ((perm & 1) >= b.mx) ? (perm & 1) + 1 : (perm & 1);
      b.mn = 3 - b.mx - b.ot;
      idx[0] = sw[8][tid];
      idx[1] = sw[9][tid];
      idx[2] = sw[10][tid];
#pragma unroll
      for (int k = 0; k < 6; ++k) p[k] = __uint_as_float(sw[11 + k][tid]);
      ref = sw[17][tid];
      cur = sw[18][tid];
      vis = (int)sw[19][tid];
    }
    has = tid < total;
    A = total;
  }
}

// Visit-sequence recorder (second pass; offsets from a prior cast), _kernels.pyx:307-341.
template <int L>
__global__ void __launch_bounds__(kBlock) visits_kernel(MeshView m, int64_t n, const float* __restrict__ o,
                                                        const float* __restrict__ d,
                                                        const int32_t* __restrict__ start,
                                                        const int64_t* __restrict__ offsets,
                                                        int32_t* __restrict__ seq) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const float o0 = o[3 * r], o1 = o[3 * r + 1], o2 = o[3 * r + 2];
  const float d0 = d[3 * r], d1 = d[3 * r + 1], d2 = d[3 * r + 2];
  uint32_t cur = (uint32_t)start[r];
  int64_t pos = offsets[r];
  const int64_t end = offsets[r + 1];
  Basis b;
  uint32_t idx[3];
  float p[6];
  const int j = init_ray(m, o0, o1, o2, d0, d1, d2, (int)cur, b, idx, p);
  uint32_t ref = pick4u(__ldg(&m.sn[cur]), j);
  const float4* __restrict__ P = ray_points(m, b);
  if (pos < end) seq[pos++] = (int32_t)cur;
  int vis = 1;
  const uint32_t n_tets = (uint32_t)m.n_tets;
  while (pos < end && ref < n_tets) {
    const uint32_t nxt = ref;
    ref = advance<L>(m, P, b, idx, p, nxt, cur);
    cur = nxt;
    ++vis;
    seq[pos++] = (int32_t)cur;
    if ((uint32_t)vis > n_tets) break;
  }
}

// Point location, _kernels.pyx:416-492.
template <int L>
__global__ void __launch_bounds__(kBlock) locate_kernel(MeshView m, int64_t n, const double* __restrict__ q,
                                                        const int32_t* __restrict__ hints,
                                                        int32_t* __restrict__ out, int32_t* __restrict__ visited) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const double qq[3] = {q[3 * r], q[3 * r + 1], q[3 * r + 2]};
  uint32_t cur = (uint32_t)hints[r];
  int32_t res = -1;
  int vis = 1;
  const uint32_t n_tets = (uint32_t)m.n_tets;
  if (contains(m, cur, qq)) {
    out[r] = (int32_t)cur;
    visited[r] = 1;
    return;
  }
  const int4 sv = __ldg(&m.sv[cur]);
  const int vid[4] = {sv.x, sv.y, sv.z, sv.w};
  double c[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 P = ldg_f4(&m.pts[vid[i]]);
    c[0] = __dadd_rn(c[0], (double)P.x);
    c[1] = __dadd_rn(c[1], (double)P.y);
    c[2] = __dadd_rn(c[2], (double)P.z);
  }
  c[0] = __ddiv_rn(c[0], 4.0); c[1] = __ddiv_rn(c[1], 4.0); c[2] = __ddiv_rn(c[2], 4.0);
  const float d0 = __double2float_rn(__dsub_rn(qq[0], c[0]));
  const float d1 = __double2float_rn(__dsub_rn(qq[1], c[1]));
  const float d2 = __double2float_rn(__dsub_rn(qq[2], c[2]));
  if (d0 == 0.0f && d1 == 0.0f && d2 == 0.0f) {
    out[r] = -1;
    visited[r] = 1;
    return;
  }
  const float o0 = __double2float_rn(c[0]), o1 = __double2float_rn(c[1]), o2 = __double2float_rn(c[2]);
  Basis b;
  uint32_t idx[3];
  float p[6];
  const int j = init_ray(m, o0, o1, o2, d0, d1, d2, (int)cur, b, idx, p);
  uint32_t ref = pick4u(__ldg(&m.sn[cur]), j);
  while (true) {
    uint32_t nxt, entry;
    if (ref == kBoundary) break;
    if (ref & kConstrained) {
      if ((ref & kPayload) >= (uint64_t)m.n_cf) break;  // corrupt mesh: no out-of-bounds gather
      const int2 ct = __ldg(&m.cf_tets[ref & kPayload]);
      const int32_t other = (ct.x == (int32_t)cur) ? ct.y : ct.x;
      if (other < 0) break;
      nxt = (uint32_t)other;
      entry = ref;  // Tet16 xor partner is the tagged face ref
    } else {
      nxt = ref & kPayload;
      entry = cur;
    }
    if (nxt >= n_tets) break;
    ref = advance<L>(m, ray_points(m, b), b, idx, p, nxt, entry);
    cur = nxt;
    ++vis;
    if (contains(m, nxt, qq)) { res = (int32_t)nxt; break; }
    if ((uint32_t)vis > n_tets) break;
  }
  out[r] = res;
  visited[r] = vis;
}

// Pinhole camera rays on the device (render.camera_rays, render.py:169-185):
// the per-camera frame (fwd, right, up2, half_w, half_h) comes from the host
// (numpy, once per frame); the per-pixel fp64 arithmetic is repeated here in
// numpy's broadcast order -- sx = ((x + .5) / W * 2 - 1) * half_w,
// sy = (1 - (y + .5) / H * 2) * half_h, d = (fwd + sx * right) + sy * up2 --
// then rounded to f32, so the rays are bit-identical to the host's.  Saves
// the 24 B/ray origin + direction upload for primary rays.
__global__ void camera_rays_kernel(int64_t width, int64_t height, const double* __restrict__ fr,
                                   const int64_t* __restrict__ pixels, int64_t n, float* __restrict__ o,
                                   float* __restrict__ d) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t pix = pixels ? pixels[i] : i;
  const double xs = (double)(pix % width), ys = (double)(pix / width);
  const double W = (double)width, H = (double)height;
  const double sx = __dmul_rn(__dsub_rn(__dmul_rn(__ddiv_rn(__dadd_rn(xs, 0.5), W), 2.0), 1.0), fr[12]);
  const double sy = __dmul_rn(__dsub_rn(1.0, __dmul_rn(__ddiv_rn(__dadd_rn(ys, 0.5), H), 2.0)), fr[13]);
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double dk = __dadd_rn(__dadd_rn(fr[k], __dmul_rn(sx, fr[3 + k])), __dmul_rn(sy, fr[6 + k]));
    d[3 * i + k] = __double2float_rn(dk);
    o[3 * i + k] = __double2float_rn(fr[9 + k]);
  }
}

// A frame's primary pass in one launch (tb_trace_camera): each lane forms
// its pixel's ray with camera_rays_kernel's fp64 arithmetic (so the ray is
// bit-identical to tb_camera_rays' output), walks it from the camera tet and
// writes the seven hit arrays -- no rays in HBM, no second launch.  The frame
// comes by value (112 B of kernel parameters: nothing to upload).  Outputs
// may be mapped pinned host memory (render-style: the hits cross PCIe as the
// warps' stores); a full block's 1-byte statuses are staged in shared memory
// and stored as one 128 B write, as cast_kernel does for host rays.
struct CamFrame {
  double f[14];
};
template <int L, bool kClamp>
__global__ void __launch_bounds__(kCastBlock, (cast_min_blocks<L, false>()))
    camera_cast_kernel(MeshView m, int64_t width, int64_t height, CamFrame fr, uint32_t cam_tet,
                       uint8_t* __restrict__ status, int32_t* __restrict__ cf, int32_t* __restrict__ tet,
                       int32_t* __restrict__ visited, int32_t* __restrict__ triangle, double* __restrict__ t,
                       int32_t* __restrict__ tet_back) {
  const int64_t n = width * height;
  const int64_t r = (int64_t)blockIdx.x * kCastBlock + threadIdx.x;
  const bool full = (int64_t)(blockIdx.x + 1) * kCastBlock <= n && (reinterpret_cast<uintptr_t>(status) & 3u) == 0;
  if (!full && r >= n) return;
  const double xs = (double)(r % width), ys = (double)(r / width);
  const double W = (double)width, H = (double)height;
  const double sx = __dmul_rn(__dsub_rn(__dmul_rn(__ddiv_rn(__dadd_rn(xs, 0.5), W), 2.0), 1.0), fr.f[12]);
  const double sy = __dmul_rn(__dsub_rn(1.0, __dmul_rn(__ddiv_rn(__dadd_rn(ys, 0.5), H), 2.0)), fr.f[13]);
  float dv[3], ov[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    dv[k] = __double2float_rn(__dadd_rn(__dadd_rn(fr.f[k], __dmul_rn(sx, fr.f[3 + k])), __dmul_rn(sy, fr.f[6 + k])));
    ov[k] = __double2float_rn(fr.f[9 + k]);
  }
  uint32_t cur = cam_tet, ref;
  int vis;
  uint8_t st;
  walk_ray<L, kClamp>(m, ov[0], ov[1], ov[2], dv[0], dv[1], dv[2], cur, ref, vis, st);
  if (full) {  // no lane of a full block returned early: the barrier is safe
    __shared__ uint32_t s_status[kCastBlock / 4];
    reinterpret_cast<uint8_t*>(s_status)[threadIdx.x] = st;
    write_result(m, r, st, ref, cur, vis, ov[0], ov[1], ov[2], dv[0], dv[1], dv[2], nullptr, cf, tet, visited,
                 triangle, t, tet_back);
    __syncthreads();
    if (threadIdx.x < kCastBlock / 4)
      reinterpret_cast<uint32_t*>(status + (int64_t)blockIdx.x * kCastBlock)[threadIdx.x] = s_status[threadIdx.x];
    return;
  }
  write_result(m, r, st, ref, cur, vis, ov[0], ov[1], ov[2], dv[0], dv[1], dv[2], status, cf, tet, visited, triangle,
               t, tet_back);
}

// Hull clipping for origins outside the mesh (traversal.cast_ray_auto,
// traversal.py:545-589): the nearest boundary face hit by the ray, tested
// brute force in fp64 (Moller-Trumbore with u, v, t bounds, det == 0
// skipped, first strictly-nearest face in hull order wins).  Hull faces are
// staged through shared memory in tiles; each lane tests its ray against
// every face.  Outputs the hull list index (-1 = no hit) and the hit t.
constexpr int kHullTile = 128;

__global__ void __launch_bounds__(kBlock) hull_clip_kernel(MeshView m, int64_t n, const float* __restrict__ o,
                                                           const float* __restrict__ d,
                                                           const int32_t* __restrict__ rays, int64_t n_hull,
                                                           const int4* __restrict__ hull,  // (tet, v0, v1, v2)
                                                           int32_t* __restrict__ best_face,
                                                           double* __restrict__ best_t) {
  __shared__ double tile[kHullTile][9];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool live = i < n;
  double O[3] = {0, 0, 0}, D[3] = {0, 0, 0};
  if (live) {
    const int64_t r = rays ? rays[i] : i;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      O[k] = (double)o[3 * r + k];
      D[k] = (double)d[3 * r + k];
    }
  }
  int32_t best = -1;
  double bt = 0.0;
  for (int64_t f0 = 0; f0 < n_hull; f0 += kHullTile) {
    __syncthreads();
    for (int k = threadIdx.x; k < kHullTile; k += blockDim.x) {
      if (f0 + k < n_hull) {
        const int4 h = hull[f0 + k];
        const int v[3] = {h.y, h.z, h.w};
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const float4 P = ldg_f4(&m.pts[v[c]]);
          tile[k][3 * c] = P.x;
          tile[k][3 * c + 1] = P.y;
          tile[k][3 * c + 2] = P.z;
        }
      }
    }
    __syncthreads();
    if (!live) continue;
    const int cnt = (int)((n_hull - f0) < kHullTile ? (n_hull - f0) : kHullTile);
    for (int k = 0; k < cnt; ++k) {
      const double* T = tile[k];
      const double e1x = __dsub_rn(T[3], T[0]), e1y = __dsub_rn(T[4], T[1]), e1z = __dsub_rn(T[5], T[2]);
      const double e2x = __dsub_rn(T[6], T[0]), e2y = __dsub_rn(T[7], T[1]), e2z = __dsub_rn(T[8], T[2]);
      const double pvx = __dsub_rn(__dmul_rn(D[1], e2z), __dmul_rn(D[2], e2y));
      const double pvy = __dsub_rn(__dmul_rn(D[2], e2x), __dmul_rn(D[0], e2z));
      const double pvz = __dsub_rn(__dmul_rn(D[0], e2y), __dmul_rn(D[1], e2x));
      const double det = __dadd_rn(__dadd_rn(__dmul_rn(e1x, pvx), __dmul_rn(e1y, pvy)), __dmul_rn(e1z, pvz));
      if (det == 0.0) continue;
      const double inv = __ddiv_rn(1.0, det);
      const double tvx = __dsub_rn(O[0], T[0]), tvy = __dsub_rn(O[1], T[1]), tvz = __dsub_rn(O[2], T[2]);
      const double u = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(tvx, pvx), __dmul_rn(tvy, pvy)), __dmul_rn(tvz, pvz)), inv);
      const double qx = __dsub_rn(__dmul_rn(tvy, e1z), __dmul_rn(tvz, e1y));
      const double qy = __dsub_rn(__dmul_rn(tvz, e1x), __dmul_rn(tvx, e1z));
      const double qz = __dsub_rn(__dmul_rn(tvx, e1y), __dmul_rn(tvy, e1x));
      const double v = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(D[0], qx), __dmul_rn(D[1], qy)), __dmul_rn(D[2], qz)), inv);
      const double tt = __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(e2x, qx), __dmul_rn(e2y, qy)), __dmul_rn(e2z, qz)), inv);
      if (u < 0.0 || v < 0.0 || __dadd_rn(u, v) > 1.0 || tt < 0.0) continue;
      if (best < 0 || tt < bt) {
        best = (int32_t)(f0 + k);
        bt = tt;
      }
    }
  }
  if (live) {
    best_face[i] = best;
    best_t[i] = bt;
  }
}

// Occlusion walks, _kernels.pyx:527-614.
template <int L, bool kClamp>
__global__ void __launch_bounds__(kBlock) shadow_kernel(MeshView m, int64_t n, const double* __restrict__ p,
                                                        const double* __restrict__ light, int light_stride,
                                                        const int32_t* __restrict__ p_tet,
                                                        const int32_t* __restrict__ light_tet, int lt_stride,
                                                        double eps, uint8_t* __restrict__ occ,
                                                        int32_t* __restrict__ visited) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  uint32_t cur = (uint32_t)p_tet[r];
  const int32_t ltet = light_tet[lt_stride * r];
  int vis = 1;
  uint8_t oc = 0;
  if ((int32_t)cur == ltet) {
    occ[r] = 0;
    visited[r] = 1;
    return;
  }
  const double* L3 = light + (int64_t)light_stride * r;
  float o32[3], d32[3];
  double o64[3], d64[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    d32[k] = __double2float_rn(__dsub_rn(L3[k], p[3 * r + k]));
    o32[k] = __double2float_rn(p[3 * r + k]);
    o64[k] = o32[k];
    d64[k] = d32[k];
  }
  Basis b;
  uint32_t idx[3];
  float pw[6];
  const int j = init_ray(m, o32[0], o32[1], o32[2], d32[0], d32[1], d32[2], (int)cur, b, idx, pw);
  uint32_t ref = pick4u(__ldg(&m.sn[cur]), j);
  const uint32_t n_tets = (uint32_t)m.n_tets;
  const uint32_t lt_u = (uint32_t)ltet;  // -1 (light outside) never equals a tet
  const double one_m_eps = __dsub_rn(1.0, eps);
  const float4* __restrict__ P = ray_points(m, b);
  while (true) {
    // fast path: plain references that are not the light's tet, 4x unrolled
    // while the guard cannot trip (same steps as the general loop below)
    while (ref < n_tets && ref != lt_u && vis + 4 <= (int)n_tets) {
      uint32_t nxt = ref;
      ref = advance<L, kClamp>(m, P, b, idx, pw, nxt, cur);
      cur = nxt;
      if (ref >= n_tets || ref == lt_u) { vis += 1; break; }
      nxt = ref;
      ref = advance<L, kClamp>(m, P, b, idx, pw, nxt, cur);
      cur = nxt;
      if (ref >= n_tets || ref == lt_u) { vis += 2; break; }
      nxt = ref;
      ref = advance<L, kClamp>(m, P, b, idx, pw, nxt, cur);
      cur = nxt;
      if (ref >= n_tets || ref == lt_u) { vis += 3; break; }
      nxt = ref;
      ref = advance<L, kClamp>(m, P, b, idx, pw, nxt, cur);
      cur = nxt;
      vis += 4;
    }
    uint32_t nxt, entry;
    if (ref == kBoundary) break;
    if (ref & kConstrained) {
      const uint32_t cfi = ref & kPayload;
      if (cfi >= (uint64_t)m.n_cf) break;  // corrupt mesh: no out-of-bounds gather
      const int32_t tri = __ldg(&m.cf_tri[cfi]);
      if ((uint32_t)tri >= (uint64_t)m.n_tri) break;
      const double tt = seg_tri_t(o64, d64, m.tri + 9 * (int64_t)tri);
      if (tt >= one_m_eps) break;
      if (tt > eps) { oc = 1; break; }
      const int2 ct = __ldg(&m.cf_tets[cfi]);
      const int32_t other = (ct.x == (int32_t)cur) ? ct.y : ct.x;
      if (other < 0) break;
      nxt = (uint32_t)other;
      entry = ref;
    } else {
      nxt = ref & kPayload;
      entry = cur;
    }
    if ((int32_t)nxt == ltet) break;
    if (nxt >= n_tets) break;
    ref = advance<L, kClamp>(m, P, b, idx, pw, nxt, entry);
    cur = nxt;
    ++vis;
    if ((uint32_t)vis > n_tets) break;
  }
  occ[r] = oc;
  visited[r] = vis;
}

// ScTP fallback walk: fp64 scalar-triple-product exit test per tet
// (traversal.sctp_exit_face, traversal.py:484-511) over the same xor-linked
// records; the entry face is the one opposite the recovered vertex i3.
template <int L>
#ifndef TB_SCTP_MIN_BLOCKS
#define TB_SCTP_MIN_BLOCKS 6  // 80 registers (r01: 1 -> 92 regs, 6 -> +5 %, 8 -> spills)
#endif
__global__ void __launch_bounds__(kBlock, TB_SCTP_MIN_BLOCKS) sctp_kernel(MeshView m, int64_t n, const float* __restrict__ o,
                                                      const float* __restrict__ d,
                                                      const int32_t* __restrict__ start,
                                                      uint8_t* __restrict__ status, int32_t* __restrict__ cf,
                                                      int32_t* __restrict__ tet, int32_t* __restrict__ visited,
                                                      int32_t* __restrict__ triangle, double* __restrict__ t,
                                                      int32_t* __restrict__ tet_back,
                                                      const int64_t* __restrict__ oidx) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  float o0, o1, o2, d0, d1, d2;
  load_xyz_warp(o, r, n, o0, o1, o2);  // whole warp participates (shuffles)
  load_xyz_warp(d, r, n, d0, d1, d2);
  if (r >= n) return;
  const double O[3] = {o0, o1, o2};
  const double D[3] = {d0, d1, d2};
  uint32_t cur = (uint32_t)start[r];
  SctpWindow w;
  const int4 qd = __ldg(&m.sv[cur]);
  const uint32_t ids[4] = {(uint32_t)qd.x, (uint32_t)qd.y, (uint32_t)qd.z, (uint32_t)qd.w};
  float4 P[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) P[i] = ldg_f4(&m.pts[ids[i]]);
  const int j = sctp_exit(P, ids, O, D, -1, __ldg(&m.orient[cur]) != 0);
  w.drop(P, ids, j);
  SctpEdges e;
  window_edges(w, {O[0], O[1], O[2]}, {D[0], D[1], D[2]}, e);
  uint32_t ref = pick4u(__ldg(&m.sn[cur]), j);
  uint32_t prev = cur;
  int vis = 1;
  uint8_t st;
  const uint32_t n_tets = (uint32_t)m.n_tets;
  while (true) {
    if (ref == kBoundary) { st = kMiss; break; }
    if (ref & kConstrained) { st = kHit; break; }
    const uint32_t nxt = ref & kPayload;
    if (nxt >= n_tets) { st = kError; break; }
    ref = sctp_advance_cached<L>(m, w, e, O, D, nxt, prev);
    prev = nxt;
    cur = nxt;
    ++vis;
    if ((uint32_t)vis > n_tets) { st = kError; break; }
  }
  write_result(m, oidx ? __ldg(oidx + r) : r, st, ref, cur, vis, o0, o1, o2, d0, d1, d2, status, cf, tet, visited, triangle, t,
               tet_back);
}

// Layout dispatch helper.
template <template <int> class K, typename... Args>
int launch_layout(int layout, unsigned grid, cudaStream_t s, Args... args) {
  switch (layout) {
    case 16: K<16>::launch(grid, s, args...); break;
    case 20: K<20>::launch(grid, s, args...); break;
    case 32: K<32>::launch(grid, s, args...); break;
    case 80: K<80>::launch(grid, s, args...); break;
    default: return set_error(TB_E_LAYOUT, "unsupported layout %d", layout);
  }
  return TB_OK;
}

template <int L>
struct CastL {
  template <typename... A>
  static void launch(unsigned g, cudaStream_t s, bool safe, bool host_rays, const int64_t* oidx, A... a) {
    const bool nc = safe && L != 80;  // validated mesh: no per-step index clamp
    const int32_t* none = nullptr;
    if (oidx != nullptr) {  // scattered outputs (device rays only)
      if (nc)
        cast_kernel<L, false, false, true><<<g, kCastBlock, 0, s>>>(a..., oidx, none, nullptr);
      else
        cast_kernel<L, true, false, true><<<g, kCastBlock, 0, s>>>(a..., oidx, none, nullptr);
    } else if (host_rays) {
      if (nc)
        cast_kernel<L, false, true, false><<<g, kCastBlock, 0, s>>>(a..., oidx, none, nullptr);
      else
        cast_kernel<L, true, true, false><<<g, kCastBlock, 0, s>>>(a..., oidx, none, nullptr);
    } else {
      if (nc)
        cast_kernel<L, false, false, false><<<g, kCastBlock, 0, s>>>(a..., oidx, none, nullptr);
      else
        cast_kernel<L, true, false, false><<<g, kCastBlock, 0, s>>>(a..., oidx, none, nullptr);
    }
  }
};
// Caller-ordered blocks (device rays, in-place results).
template <int L>
struct CastOrderedL {
  template <typename... A>
  static void launch(unsigned g, cudaStream_t s, bool safe, const int32_t* bmap, A... a) {
    const int64_t* none = nullptr;
    const int32_t* no_gather = nullptr;
    if (safe && L != 80)
      cast_kernel<L, false, false, false, false, true><<<g, kCastBlock, 0, s>>>(a..., none, no_gather, bmap);
    else
      cast_kernel<L, true, false, false, false, true><<<g, kCastBlock, 0, s>>>(a..., none, no_gather, bmap);
  }
};
// Binned walk: rays read through perm; results stored through widx (perm
// itself, or perm composed with a caller's scatter index).
template <int L>
struct CastBinnedL {
  template <typename... A>
  static void launch(unsigned g, cudaStream_t s, bool safe, const int32_t* perm, const int64_t* widx, A... a) {
    if (safe && L != 80)
      cast_kernel<L, false, false, true, true><<<g, kCastBlock, 0, s>>>(a..., widx, perm, nullptr);
    else
      cast_kernel<L, true, false, true, true><<<g, kCastBlock, 0, s>>>(a..., widx, perm, nullptr);
  }
};

template <int L>
struct CastDynL {
  // grid: one full wave of resident blocks (fewer for small batches)
  template <typename... A>
  static void launch(int64_t n, cudaStream_t s, bool safe, A... a) {
    static int per_sm[2] = {0, 0}, sms = 0;
    const bool nc = safe && L != 80;
    if (per_sm[nc] == 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (nc)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[1], cast_dyn_kernel<L, false>, kCastBlock, 0);
      else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[0], cast_dyn_kernel<L, true>, kCastBlock, 0);
      if (per_sm[nc] < 1) per_sm[nc] = 1;
    }
    const int64_t full = (int64_t)per_sm[nc] * sms;
    const int64_t need = (n + kCastBlock - 1) / kCastBlock;
    const unsigned g = (unsigned)(need < full ? need : full);
    if (nc)
      cast_dyn_kernel<L, false><<<g, kCastBlock, 0, s>>>(a...);
    else
      cast_dyn_kernel<L, true><<<g, kCastBlock, 0, s>>>(a...);
  }
};

// Stream-ordered scratch from a per-device pool that keeps its memory
// between calls (the default pool returns it to the driver at every
// synchronisation, turning each call into a fresh cudaMalloc).
int scratch_alloc(int device, size_t bytes, cudaStream_t s, char** out) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  if (device < 0 || device >= 64) return set_error(TB_E_ARG, "device %d out of range", device);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[device]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = device;
      TB_CUDA(cudaMemPoolCreate(&pools[device], &props));
      uint64_t keep = ~(uint64_t)0;
      TB_CUDA(cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &keep));
    }
  }
  TB_CUDA(cudaMallocFromPoolAsync((void**)out, bytes, pools[device], s));
  return TB_OK;
}

template <int L>
struct CastPersistL {
  // grid: one full wave of resident blocks (or fewer for small batches)
  template <typename... A>
  static void launch(unsigned g, cudaStream_t s, A... a) {
    static int per_sm = 0, sms = 0;
    if (per_sm == 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cast_persist_kernel<L>, kBlock, 0);
      if (per_sm < 1) per_sm = 1;
    }
    const unsigned full = (unsigned)(per_sm * sms);
    cast_persist_kernel<L><<<g < full ? g : full, kBlock, 0, s>>>(a...);
  }
};

// ----------------------------------------------------------------------------
#include "binning.cuh"  // direction binning: dir_bin, bin_count / bin_scan / bin_seg_scan / bin_scatter


// TETB200_SCHED: 0 = auto, 1 = one ray per lane (cast_kernel), 2 = persistent
// refill (cast_persist_kernel), 3 / 4 = block compaction with 256 / 512
// threads (cast_compact_kernel), 5 = dynamic warp chunks (cast_dyn_kernel),
// 6 = direction-binned.  TETB200_ROUND: steps per compaction round.
std::atomic<int> g_sched_mode{-1}, g_round_steps{-1};
int sched_mode() {
  int mode = g_sched_mode.load(std::memory_order_relaxed);
  if (mode < 0) {
    const char* v = getenv("TETB200_SCHED");
    mode = v ? atoi(v) : 0;
    if (mode < 0 || mode > 7) mode = 0;
    int expect = -1;
    g_sched_mode.compare_exchange_strong(expect, mode);
    mode = g_sched_mode.load();
  }
  return mode;
}
int round_steps() {
  int k = g_round_steps.load(std::memory_order_relaxed);
  if (k < 0) {
    const char* v = getenv("TETB200_ROUND");
    k = v ? atoi(v) : 32;  // r01 sweep, config 4: 8 / 16 / 32 / 48 / 64 -> best at 32
    if (k < 1) k = 1;
    int expect = -1;
    g_round_steps.compare_exchange_strong(expect, k);
    k = g_round_steps.load();
  }
  return k;
}
template <int L, int BT, bool kClamp>
struct CastCompactL {
  // grid: one full wave of resident blocks (or fewer for small batches)
  template <typename... A>
  static void launch(int64_t n, cudaStream_t s, A... a) {
    static int per_sm = 0, sms = 0;
    if (per_sm == 0) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cast_compact_kernel<L, BT, kClamp>, BT, 0);
      if (per_sm < 1) per_sm = 1;
    }
    const int64_t full = (int64_t)per_sm * sms;
    const int64_t chunks = (n + 31) / 32;
    const unsigned g = (unsigned)(chunks < full ? chunks : full);
    cast_compact_kernel<L, BT, kClamp><<<g, BT, 0, s>>>(a..., round_steps());
  }
};
template <int BT, typename... A>
int launch_compact(int layout, bool safe, int64_t n, cudaStream_t s, A... a) {
  switch (layout * 2 + (safe ? 1 : 0)) {
    case 32: CastCompactL<16, BT, true>::launch(n, s, a...); break;
    case 33: CastCompactL<16, BT, false>::launch(n, s, a...); break;
    case 40: CastCompactL<20, BT, true>::launch(n, s, a...); break;
    case 41: CastCompactL<20, BT, false>::launch(n, s, a...); break;
    case 64: CastCompactL<32, BT, true>::launch(n, s, a...); break;
    case 65: CastCompactL<32, BT, false>::launch(n, s, a...); break;
    case 160: case 161: CastCompactL<80, BT, true>::launch(n, s, a...); break;
    default: return set_error(TB_E_LAYOUT, "unsupported layout %d", layout);
  }
  return TB_OK;
}
template <int L>
struct VisitsL {
  template <typename... A>
  static void launch(unsigned g, cudaStream_t s, A... a) { visits_kernel<L><<<g, kBlock, 0, s>>>(a...); }
};
template <int L>
struct LocateL {
  template <typename... A>
  static void launch(unsigned g, cudaStream_t s, A... a) { locate_kernel<L><<<g, kBlock, 0, s>>>(a...); }
};
template <int L>
struct ShadowL {
  template <typename... A>
  static void launch(unsigned g, cudaStream_t s, bool safe, A... a) {
    if (safe && L != 80)
      shadow_kernel<L, false><<<g, kBlock, 0, s>>>(a...);
    else
      shadow_kernel<L, true><<<g, kBlock, 0, s>>>(a...);
  }
};
template <int L>
struct CameraCastL {
  template <typename... A>
  static void launch(unsigned g, cudaStream_t s, bool safe, A... a) {
    if (safe && L != 80)
      camera_cast_kernel<L, false><<<g, kCastBlock, 0, s>>>(a...);
    else
      camera_cast_kernel<L, true><<<g, kCastBlock, 0, s>>>(a...);
  }
};
template <int L>
struct SctpL {
  template <typename... A>
  static void launch(unsigned g, cudaStream_t s, A... a) { sctp_kernel<L><<<g, kBlock, 0, s>>>(a...); }
};

// L2 gather roof for the walk's access shape (SURVEY 8 d: "report against a
// measured L2 gather bandwidth" when the hot arrays fit in L2).  Each pair is
// one step's worth of gathers at independent pseudo-random indices: the
// layout's record words (exactly the loads Record<L>::load issues) and one
// float4 of a random axis-permuted point copy, 8 pairs in flight per thread
// so the loads are never latency-serialised.  Algorithmic bytes per pair
// = L + 12, the same per-step figure the bench's roofline counts.
__device__ __forceinline__ uint32_t probe_hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7FEB352Du;
  x ^= x >> 15; x *= 0x846CA68Bu;
  return x ^ (x >> 16);
}

__device__ __forceinline__ uint32_t fold4(const uint4& u) { return u.x ^ u.y ^ u.z ^ u.w; }

template <int L>
__device__ __forceinline__ uint32_t probe_fold(const Record<L>& r) {
  if constexpr (L == 16) return fold4(r.r);
  else if constexpr (L == 20) return r.v ^ fold4(r.n);
  else return fold4(r.a) ^ fold4(r.n);
}

template <int L>
__global__ void __launch_bounds__(256) gather_probe_kernel(MeshView m, int64_t n_pairs, uint32_t seed,
                                                           uint32_t* __restrict__ sink) {
  constexpr int kInFlight = 8;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nt = (uint32_t)m.n_tets, np6 = (uint32_t)(m.n_points * 6);
  uint32_t acc = 0;
  auto pair = [&](int64_t i) {
    const uint32_t h = probe_hash((uint32_t)i * 2u + seed);
    Record<L> r;
    r.load(m, __umulhi(h, nt));
    const float4 q = __ldg(&m.pts[__umulhi(probe_hash(h ^ 0x5bd1e995u), np6)]);
    return probe_fold<L>(r) ^ __float_as_uint(q.x) ^ __float_as_uint(q.y) ^ __float_as_uint(q.z);
  };
  const int64_t groups = n_pairs / kInFlight;
  for (int64_t g = tid; g < groups; g += nthreads) {
    uint32_t v[kInFlight];
#pragma unroll
    for (int k = 0; k < kInFlight; ++k) v[k] = pair(g * kInFlight + k);  // all loads issued before any use
#pragma unroll
    for (int k = 0; k < kInFlight; ++k) acc ^= v[k];
  }
  if (tid < n_pairs - groups * kInFlight) acc ^= pair(groups * kInFlight + tid);
  if (acc == 0x9E3779B9u) atomicXor(sink, acc);  // keeps the loads live; practically never stores
}

// Launch order of a batch's blocks, longest walk first, from a previous
// similar batch's per-ray visited counts (tb_block_order).  A block's key is
// its largest visited count (a block holds its slot until its slowest warp
// ends), bucketed in kOrderBuckets log-spaced classes.  Pass 1: one warp per
// block takes the key and adds it to the bucket histogram (warp-aggregated
// atomics); pass 2: every CTA scans the small histogram in shared memory and
// scatters its blocks, longest bucket first, through per-bucket atomic
// cursors.  The order inside a bucket follows the atomics: it decides where a
// block runs, never what it computes.
constexpr int kOrderBuckets = 64;

__device__ __forceinline__ int order_bucket(int v) {
  // 0..15 exact, then 4 classes per power of two, descending ids for longer walks
  int b;
  if (v < 16) {
    b = v;
  } else {
    const int e = 31 - __clz(v);               // >= 4
    b = 16 + (e - 4) * 4 + ((v >> (e - 2)) & 3);
  }
  return kOrderBuckets - 1 - min(b, kOrderBuckets - 1);
}

__global__ void block_key_kernel(const int32_t* __restrict__ visited, int64_t n, int64_t nb,
                                 uint8_t* __restrict__ key, int* __restrict__ hist) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nb) return;
  int mx = 0;
  for (int k = lane; k < kCastBlock; k += 32) {
    const int64_t r = w * kCastBlock + k;
    if (r < n) mx = max(mx, __ldg(visited + r));
  }
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) {
    const int b = order_bucket(mx);
    key[w] = (uint8_t)b;
    atomicAdd(hist + b, 1);
  }
}

__global__ void block_scatter_kernel(const uint8_t* __restrict__ key, int64_t nb, const int* __restrict__ hist,
                                     int* __restrict__ cursor, int32_t* __restrict__ order, int64_t b0 = 0) {
  __shared__ int base[kOrderBuckets];
  if (threadIdx.x < 32) {  // exclusive scan of the histogram, 2 buckets per lane
    const int a = hist[2 * threadIdx.x], c = hist[2 * threadIdx.x + 1];
    int pre = a + c;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, pre, o);
      if ((int)threadIdx.x >= o) pre += v;
    }
    base[2 * threadIdx.x] = pre - a - c;
    base[2 * threadIdx.x + 1] = pre - c;
  }
  __syncthreads();
  const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const int k = key[b];
  // warp-aggregated cursor bumps: one atomic per distinct bucket in the warp
  const unsigned peers = __match_any_sync(__activemask(), k);
  const int leader = __ffs(peers) - 1;
  const int rank = __popc(peers & ((1u << (threadIdx.x & 31)) - 1u));
  int pos = 0;
  if ((int)(threadIdx.x & 31) == leader) pos = atomicAdd(cursor + k, __popc(peers));
  pos = __shfl_sync(peers, pos, leader);
  order[base[k] + pos + rank] = (int32_t)(b0 + b);
}

// Sampled cost pre-pass of schedule 7 ("sampled"): one ray per block -- the
// block's middle ray -- walked at most `cap` steps; its step count, exact
// below kOrderBuckets, is the block's key for the longest-first order.  A
// single ray per block, capped at 32 steps, orders a 1080p frame as well as
// the blocks' full walk lengths do (r02 probe): the blocks that matter are
// the ones whose rays run long, and any ray past 32 steps marks one.
template <int L, bool kClamp>
__global__ void __launch_bounds__(64) block_probe_kernel(MeshView m, int64_t n, const float* __restrict__ o,
                                                         const float* __restrict__ d,
                                                         const int32_t* __restrict__ start, int64_t b0, int64_t nb,
                                                         int cap, uint8_t* __restrict__ key, int* __restrict__ hist) {
  // blocks b0 .. nb-1 (the ordered tail of a split launch; b0 = 0: all)
  const int64_t b = b0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool in = b < nb;
  int steps = 0;
  if (in) {
    int64_t r = b * kCastBlock + kCastBlock / 2;
    if (r >= n) r = n - 1;
    uint32_t cur = (uint32_t)__ldg(start + r);
    Basis bs;
    uint32_t idx[3];
    float p[6];
    const int j = init_ray(m, __ldg(o + 3 * r), __ldg(o + 3 * r + 1), __ldg(o + 3 * r + 2), __ldg(d + 3 * r),
                           __ldg(d + 3 * r + 1), __ldg(d + 3 * r + 2), (int)cur, bs, idx, p);
    uint32_t ref = pick4u(__ldg(&m.sn[cur]), j);
    const float4* __restrict__ P = ray_points(m, bs);
    const uint32_t live = kClamp ? (uint32_t)m.n_tets : kBoundary;
    steps = 1;
    while (ref < live && steps < cap) {
      const uint32_t nxt = ref;
#ifndef TB_PROBE_NO_PREFETCH
      if constexpr (L == 20) {
        // The walk here is a lone latency chain over a cold L2.  The tet's four
        // neighbours are the next step's only candidates: their records go to
        // L2 while this step decides, and -- from their vx words, prefetched one
        // step earlier and so L2 hits now -- so do the point copies of the
        // vertex each would add (vx[n_k] ^ vx[t] ^ v_k, v_k the tet's k-th
        // smallest vertex, across from n_k).  Each step then finds its record
        // and its point in L2 instead of two DRAM round trips.
        const uint4 nb4 = __ldg(&m.rec4[nxt]);
        const uint32_t vt = __ldg(&m.vx[nxt]);
        const uint32_t a[4] = {idx[0], idx[1], idx[2], idx[0] ^ idx[1] ^ idx[2] ^ vt};
        uint32_t v[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          int r = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) r += (a[j] < a[i]) ? 1 : 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) v[k] = (r == k) ? a[i] : v[k];
        }
        const uint32_t nbs[4] = {nb4.x, nb4.y, nb4.z, nb4.w};
        const uint32_t last_point = (uint32_t)m.n_points - 1u;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (nbs[k] < (uint32_t)m.n_tets) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(m.vx + nbs[k]));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(m.rec4 + nbs[k]));
            const uint32_t nv = min(__ldg(&m.vx[nbs[k]]) ^ vt ^ v[k], last_point);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(P + nv));
          }
      }
#endif
      ref = advance<L, kClamp>(m, P, bs, idx, p, nxt, cur);
      cur = nxt;
      ++steps;
    }
  }
  const int k = kOrderBuckets - 1 - min(steps, kOrderBuckets - 1);
  if (in) key[b - b0] = (uint8_t)k;
  const unsigned act = __ballot_sync(0xffffffffu, in);
  if (!in) return;
  const unsigned peers = __match_any_sync(act, k);
  if ((int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(hist + k, __popc(peers));
}

template <int L>
struct BlockProbeL {
  template <typename... A>
  static void launch(unsigned g, cudaStream_t s, bool safe, A... a) {
    if (safe && L != 80)
      block_probe_kernel<L, false><<<g, 64, 0, s>>>(a...);
    else
      block_probe_kernel<L, true><<<g, 64, 0, s>>>(a...);
  }
};

// Blocks per wave of the walk on `device` (SMs x the 10 resident blocks of
// the 48-register walks).
int64_t cast_wave(int device) {
  static std::atomic<int> sms[64];
  int c = device >= 0 && device < 64 ? sms[device].load(std::memory_order_relaxed) : 148;
  if (c == 0) {
    if (cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || c <= 0) c = 148;
    sms[device].store(c, std::memory_order_relaxed);
  }
  return (int64_t)c * TB_CAST_MIN_BLOCKS;
}

// Schedule 7's split (cast_dispatch): the first head_blocks() blocks walk in
// launch order while the pre-pass orders the rest, which then launch longest
// first on a high-priority side stream.  The head must outlast the pre-pass
// (~20-25 us, a lone latency chain): at least kHeadWaves waves.  The ordered
// tail is ~65 % of the launch, at most kTailWaves waves: only the last waves'
// order shapes the SM-idle tail, and a longer sorted stretch only trades away
// the frame order's L2 locality.  r02 A/B (profiles/r02_experiments.md):
// config 2 (11 waves) tail 50 / 65 / 80 % -> 0.1776 / 0.1715 / 0.1836 ms;
// config 3 (44 waves) tail 35 / 50 / 65 % -> 0.7209 / 0.7225 / 0.7306 ms;
// 1 M rays (5.5 waves) tail 50 / 60 % -> 0.0975 / 0.114 ms.
// TETB200_ORDER_TAIL (percent of the blocks, experiment knob) overrides.
constexpr int64_t kHeadWaves = 3, kTailWaves = 16;
int64_t head_blocks(int device, int64_t nb) {
  static const int pct = [] {
    const char* v = getenv("TETB200_ORDER_TAIL");
    return v ? std::min(100, std::max(1, atoi(v))) : 0;
  }();
  if (pct) return nb - std::max<int64_t>(1, nb * pct / 100);
  const int64_t wave = cast_wave(device);
  const int64_t tail = std::min(nb * 65 / 100, kTailWaves * wave);
  const int64_t head = std::max(nb - tail, kHeadWaves * wave);
  return head >= nb ? 0 : head;  // too short to split: order every block, pre-pass first
}

// Schedule 0 ("auto") for device-resident batches: the sampled longest-first
// order (7) for launches of kSampledMinWaves .. kSampledMaxWaves waves, one
// ray per lane (1) otherwise.  Short launches cannot hide the pre-pass under a
// head (262 K / 524 K rays: lane 0.068 / 0.080 ms, sampled 0.089 / 0.098);
// long ones have a diluted tail and lose frame-order locality (config 5, 146
// waves: -0.6 %).  Config 2 (11 waves) +18 %, config 3 (44 waves) +2.5 %
// (r02 A/B).  Incoherent batches ask for "binned".
constexpr int64_t kSampledMinWaves = 6, kSampledMaxWaves = 48;
int auto_schedule(int device, int64_t n) {
  if (device < 0 || device >= 64) return 1;
  const int64_t nb = (n + kCastBlock - 1) / kCastBlock;
  const int64_t wave = cast_wave(device);
  return nb >= kSampledMinWaves * wave && nb <= kSampledMaxWaves * wave ? 7 : 1;
}

int probe_cap() {
  static const int cap = [] {
    const char* v = getenv("TETB200_PROBE_CAP");  // experiment knob
    const int c = v ? atoi(v) : 32;
    return c < 2 ? 2 : (c > 63 ? 63 : c);
  }();
  return cap;
}

int check_mesh(const tb_mesh* m) {
  if (m == nullptr) return set_error(TB_E_ARG, "mesh handle is NULL");
  return TB_OK;
}

// Launch the traversal with an explicit schedule (see sched_mode).
// Schedule 7's side stream (highest priority: once the tail's order exists,
// its blocks take the SM slots the head's retiring blocks free, so the long
// blocks start early and the head's remainder fills in behind them -- at
// default priority the tail waited for the whole head: config 2 0.1959 vs
// 0.1784 ms at a 60 % tail) and a fork / join event pair, per (host thread,
// device).
struct OrderSide {
  cudaStream_t s[64] = {};
  cudaEvent_t fork[64] = {}, join[64] = {};
  ~OrderSide() {
    for (int dv = 0; dv < 64; ++dv) {
      if (!s[dv]) continue;
      int prev = -1;
      cudaGetDevice(&prev);
      cudaSetDevice(dv);
      cudaStreamSynchronize(s[dv]);
      cudaEventDestroy(fork[dv]);
      cudaEventDestroy(join[dv]);
      cudaStreamDestroy(s[dv]);
      if (prev >= 0) cudaSetDevice(prev);
    }
    cudaGetLastError();
  }
};
int order_side(int device, cudaStream_t* side, cudaEvent_t* fork, cudaEvent_t* join) {
  static thread_local OrderSide o;
  if (device < 0 || device >= 64) return set_error(TB_E_ARG, "device %d out of range", device);
  if (!o.s[device]) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    if (cudaStreamCreateWithPriority(&o.s[device], cudaStreamNonBlocking, greatest) != cudaSuccess ||
        cudaEventCreateWithFlags(&o.fork[device], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&o.join[device], cudaEventDisableTiming) != cudaSuccess)
      return set_error(TB_E_CUDA, "side stream for the sampled schedule: %s", cudaGetErrorString(cudaGetLastError()));
  }
  *side = o.s[device];
  *fork = o.fork[device];
  *join = o.join[device];
  return TB_OK;
}
// TETB200_BIN_SPLIT=0 keeps the binned schedule on the caller's stream in one
// piece (A/B; results are identical either way)
#ifndef TB_BIN_SPLIT_DEFAULT
#define TB_BIN_SPLIT_DEFAULT 1
#endif
bool bin_split() {
  static const int v = [] {
    const char* e = getenv("TETB200_BIN_SPLIT");
    return e ? atoi(e) : TB_BIN_SPLIT_DEFAULT;
  }();
  return v > 0;
}
int cast_dispatch(tb_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start, uint8_t* status,
                  int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle, double* t, int32_t* tet_back,
                  cudaStream_t s, int mode, bool host_rays = false, const int64_t* oidx = nullptr) {
  DeviceGuard g(m->device);
  const MeshView v = m->view();
  int e = TB_OK;
  // Scattered outputs (multi-GPU frame assembly): one ray per lane or the
  // binned walk (its permutation composed with oidx); the compaction and
  // refill schedules have no scatter variant and run one ray per lane.
  if (oidx != nullptr && mode != 6) mode = 1;
  if (mode == 0 && !host_rays) mode = auto_schedule(m->device, n);
  if ((mode == 3 || mode == 4) && n < (int64_t)1 << 32) {
    e = mode == 3 ? launch_compact<256>(m->layout, m->safe, n, s, v, n, o, d, start, status, cf, tet, visited,
                                        triangle, t, tet_back)
                  : launch_compact<512>(m->layout, m->safe, n, s, v, n, o, d, start, status, cf, tet, visited,
                                        triangle, t, tet_back);
  } else if (mode == 6 && !host_rays && n < ((int64_t)1 << 31)) {
    // direction binning (stable counting sort of ray indices by direction cell), then
    // the walk in binned order, reading rays and storing results by index
    const int n_tiles = (int)((n + kBinTile - 1) / kBinTile);
    const int S = bin_tile() / kBinTile;  // tiles per sorting segment, 0 = one global sort
    const int n_segs = S ? (n_tiles + S - 1) / S : 1;
    // hist: kBins counts per tile (padded to whole segments in tile-local mode), then the 96 totals
    const size_t hist_n = (size_t)(S ? n_segs * S : n_tiles) * kBins;
    const size_t hist_b = ((hist_n + kBins) * 4 + 255) & ~(size_t)255;
    char* scratch = nullptr;
    const size_t widx_b = oidx ? (size_t)n * 8 : 0;  // perm composed with the caller's scatter index
    if (int e2 = scratch_alloc(m->device, hist_b + widx_b + (size_t)n * 4 + (size_t)n, s, &scratch)) return e2;
    int32_t* hist = reinterpret_cast<int32_t*>(scratch);
    int32_t* totals = hist + hist_n;
    int64_t* widx = oidx ? reinterpret_cast<int64_t*>(scratch + hist_b) : nullptr;  // null: results to perm[r]
    int32_t* perm = reinterpret_cast<int32_t*>(scratch + hist_b + widx_b);
    uint8_t* bins = reinterpret_cast<uint8_t*>(scratch + hist_b + widx_b + (size_t)n * 4);
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    const int seg_mid = (n_segs + 1) / 2;
    if (S && !oidx && n_segs >= 2 && bin_split() && order_side(m->device, &side, &fork, &join) == TB_OK) {
      // Two chunks of whole segments (the sort is segment-local): chunk 0 is
      // binned on the caller's stream and walks there; chunk 1 is binned on the
      // high-priority side stream beside chunk 0's walk and then walks there
      // too, so only half of the binning passes precede any walk.
      const int ta = std::min(seg_mid * S, n_tiles);
      const int64_t ra = std::min<int64_t>((int64_t)ta * kBinTile, n);
      cudaError_t ce = cudaMemsetAsync(hist, 0, hist_n * 4, s);
      if (ce == cudaSuccess) {
        bin_count_kernel<<<ta, kBinThreads, 0, s>>>(d, n, hist, n_tiles, S, bins, 0);
        bin_seg_scan_kernel<<<seg_mid, 1024, 0, s>>>(hist, S, 0);
        bin_scatter_kernel<<<ta, kBinThreads, 0, s>>>(bins, n, hist, totals, n_tiles, S, perm, 0);
        ce = cudaEventRecord(fork, s);
      }
      if (ce == cudaSuccess) ce = cudaStreamWaitEvent(side, fork, 0);
      if (ce != cudaSuccess) {
        cudaFreeAsync(scratch, s);
        return set_error(TB_E_CUDA, "binned schedule fork: %s", cudaGetErrorString(ce));
      }
      bin_count_kernel<<<n_tiles - ta, kBinThreads, 0, side>>>(d, n, hist, n_tiles, S, bins, ta);
      bin_seg_scan_kernel<<<n_segs - seg_mid, 1024, 0, side>>>(hist, S, seg_mid);
      bin_scatter_kernel<<<n_tiles - ta, kBinThreads, 0, side>>>(bins, n, hist, totals, n_tiles, S, perm, ta);
      e = launch_layout<CastBinnedL>(m->layout, grid_for(ra, kCastBlock), s, m->safe, (const int32_t*)perm,
                                     (const int64_t*)nullptr, v, ra, o, d, start, status, cf, tet, visited, triangle,
                                     t, tet_back);
      if (!e)
        e = launch_layout<CastBinnedL>(m->layout, grid_for(n - ra, kCastBlock), side, m->safe,
                                       (const int32_t*)(perm + ra), (const int64_t*)nullptr, v, n - ra, o, d, start,
                                       status, cf, tet, visited, triangle, t, tet_back);
      const bool ok = cudaEventRecord(join, side) == cudaSuccess && cudaStreamWaitEvent(s, join, 0) == cudaSuccess;
      if (!ok && !e) e = set_error(TB_E_CUDA, "binned schedule join: %s", cudaGetErrorString(cudaGetLastError()));
    } else {
      if (S) {
        if (cudaError_t me = cudaMemsetAsync(hist, 0, hist_n * 4, s)) {  // the ragged segment's missing tiles count 0
          cudaFreeAsync(scratch, s);
          return set_error(TB_E_CUDA, "binning scratch memset: %s", cudaGetErrorString(me));
        }
        bin_count_kernel<<<n_tiles, kBinThreads, 0, s>>>(d, n, hist, n_tiles, S, bins);
        bin_seg_scan_kernel<<<n_segs, 1024, 0, s>>>(hist, S);
      } else {
        bin_count_kernel<<<n_tiles, kBinThreads, 0, s>>>(d, n, hist, n_tiles, 0, bins);
        bin_scan_kernel<<<kBins, 1024, 0, s>>>(hist, n_tiles, totals);
      }
      bin_scatter_kernel<<<n_tiles, kBinThreads, 0, s>>>(bins, n, hist, totals, n_tiles, S, perm);
      if (oidx) compose_index_kernel<<<grid_for(n, 256), 256, 0, s>>>(perm, oidx, n, widx);
      e = launch_layout<CastBinnedL>(m->layout, grid_for(n, kCastBlock), s, m->safe, perm, widx, v, n, o, d, start,
                                     status, cf, tet, visited, triangle, t, tet_back);
    }
    cudaFreeAsync(scratch, s);
  } else if (mode == 7 && !host_rays && oidx == nullptr) {
    // sampled longest-first: a capped walk of one ray per block orders the
    // blocks (block_probe_kernel -> block_scatter_kernel), then the full walk
    // launches them in that order, rays and results in place.  Split (b0 > 0):
    // the head's blocks walk in launch order on the caller's stream while the
    // side stream probes and orders the tail, which launches longest first at
    // high priority; the caller's stream joins the side stream at the end.
    const int64_t nb = (n + kCastBlock - 1) / kCastBlock;
    const int64_t b0 = head_blocks(m->device, nb);  // first block of the ordered tail
    const int64_t nt = nb - b0;
    const size_t kb = ((size_t)nt + 255) / 256 * 256, hb = 2 * kOrderBuckets * sizeof(int);
    char* scratch = nullptr;
    if (int e2 = scratch_alloc(m->device, kb + hb + (size_t)nt * 4, s, &scratch)) return e2;
    uint8_t* key = reinterpret_cast<uint8_t*>(scratch);
    int* hist = reinterpret_cast<int*>(scratch + kb);
    int32_t* order = reinterpret_cast<int32_t*>(scratch + kb + hb);
    cudaStream_t side = s;
    cudaEvent_t fork = nullptr, join = nullptr;
    if (b0 > 0) {  // split launch: fork the side stream off the caller's
      if (int e2 = order_side(m->device, &side, &fork, &join)) {
        cudaFreeAsync(scratch, s);
        return e2;
      }
      if (cudaEventRecord(fork, s) != cudaSuccess || cudaStreamWaitEvent(side, fork, 0) != cudaSuccess) {
        cudaFreeAsync(scratch, s);
        return set_error(TB_E_CUDA, "sampled schedule fork: %s", cudaGetErrorString(cudaGetLastError()));
      }
    }
    if (cudaError_t me = cudaMemsetAsync(hist, 0, hb, side)) {
      e = set_error(TB_E_CUDA, "sampled schedule memset: %s", cudaGetErrorString(me));
    } else {
      e = launch_layout<BlockProbeL>(m->layout, grid_for(nt, 64), side, m->safe, v, n, o, d, start, b0, nb,
                                     probe_cap(), key, hist);
    }
    if (!e && b0 > 0)  // the head, in launch order, on the caller's stream
      e = launch_layout<CastL>(m->layout, (unsigned)b0, s, m->safe, false, (const int64_t*)nullptr, v,
                               b0 * kCastBlock, o, d, start, status, cf, tet, visited, triangle, t, tet_back);
    if (!e) {
      block_scatter_kernel<<<grid_for(nt, 256), 256, 0, side>>>(key, nt, hist, hist + kOrderBuckets, order, b0);
      e = launch_layout<CastOrderedL>(m->layout, (unsigned)nt, side, m->safe, (const int32_t*)order, v, n, o, d,
                                      start, status, cf, tet, visited, triangle, t, tet_back);
    }
    if (b0 > 0) {  // join (also on error: nothing may stay queued on the side stream past the free)
      const bool ok = cudaEventRecord(join, side) == cudaSuccess && cudaStreamWaitEvent(s, join, 0) == cudaSuccess;
      if (!ok && !e) e = set_error(TB_E_CUDA, "sampled schedule join: %s", cudaGetErrorString(cudaGetLastError()));
    }
    cudaFreeAsync(scratch, s);
  } else if (mode == 5 && !host_rays) {
    char* scratch = nullptr;
    if (int e2 = scratch_alloc(m->device, 256, s, &scratch)) return e2;
    unsigned long long* next = reinterpret_cast<unsigned long long*>(scratch);
    if (cudaError_t me = cudaMemsetAsync(next, 0, sizeof(*next), s)) {
      cudaFreeAsync(scratch, s);
      return set_error(TB_E_CUDA, "dynamic schedule counter: %s", cudaGetErrorString(me));
    }
    switch (m->layout) {
      case 16: CastDynL<16>::launch(n, s, m->safe, v, n, o, d, start, status, cf, tet, visited, triangle, t, tet_back, next); break;
      case 20: CastDynL<20>::launch(n, s, m->safe, v, n, o, d, start, status, cf, tet, visited, triangle, t, tet_back, next); break;
      case 32: CastDynL<32>::launch(n, s, m->safe, v, n, o, d, start, status, cf, tet, visited, triangle, t, tet_back, next); break;
      case 80: CastDynL<80>::launch(n, s, m->safe, v, n, o, d, start, status, cf, tet, visited, triangle, t, tet_back, next); break;
      default: e = set_error(TB_E_LAYOUT, "unsupported layout %d", m->layout);
    }
    cudaFreeAsync(scratch, s);
  } else if (mode == 2) {
    e = launch_layout<CastPersistL>(m->layout, grid_for(n, kBlock), s, v, n, o, d, start, status, cf, tet, visited,
                                    triangle, t, tet_back);
  } else {
    e = launch_layout<CastL>(m->layout, grid_for(n, kCastBlock), s, m->safe, host_rays, oidx, v, n, o, d, start,
                             status, cf, tet, visited, triangle, t, tet_back);
  }
  if (e) return e;
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}


// Stream-ordered scratch for the *_host entry points.
struct Scratch {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
};

}  // namespace

// ============================================================================
// C ABI
extern "C" {

int tb_abi_version(void) { return TB_ABI_VERSION; }

const char* tb_last_error(void) { return g_last_error.c_str(); }

int tb_mesh_create(int device, int layout, int64_t n_points, const float* points_xyz, int64_t n_tets,
                   const uint32_t* records, const int32_t* side_verts, const uint32_t* side_neighbors,
                   int64_t n_cf, const int32_t* cf_triangle, const int32_t* cf_tets, int64_t n_tri,
                   const double* tri_coords, tb_mesh** out) {
  if (out == nullptr) return set_error(TB_E_ARG, "out is NULL");
  *out = nullptr;
  if (layout != 16 && layout != 20 && layout != 32 && layout != 80)
    return set_error(TB_E_LAYOUT, "unknown layout %d (expected 16, 20, 32 or 80)", layout);
  if (n_points <= 0 || n_tets <= 0 || n_cf < 0 || n_tri < 0)
    return set_error(TB_E_ARG, "bad sizes n_points=%lld n_tets=%lld n_cf=%lld n_tri=%lld",
                     (long long)n_points, (long long)n_tets, (long long)n_cf, (long long)n_tri);
  if (n_tets >= (int64_t)0x7FFFFFFF || n_points >= (int64_t)0x7FFFFFFF)
    return set_error(TB_E_ARG, "mesh too large for 31-bit references");
  if (!points_xyz || !side_verts || !side_neighbors || (layout != 80 && !records))
    return set_error(TB_E_ARG, "NULL mesh array");
  if (n_cf > 0 && (!cf_triangle || !cf_tets)) return set_error(TB_E_ARG, "NULL constrained-face array");
  if (n_tri > 0 && !tri_coords) return set_error(TB_E_ARG, "NULL triangle coordinates");
  int ndev = 0;
  TB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return set_error(TB_E_ARG, "device %d out of range (%d)", device, ndev);
  DeviceGuard g(device);

  tb_mesh* m = new tb_mesh();
  m->device = device;
  m->layout = layout;
  m->n_points = n_points;
  m->n_tets = n_tets;
  m->n_cf = n_cf;
  m->n_tri = n_tri;
  auto fail = [&](int code) {
    tb_mesh_destroy(m);
    return code;
  };
#define TB_MC(call)                                                                      \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(set_error(e_ == cudaErrorMemoryAllocation ? TB_E_OOM : TB_E_CUDA,      \
                            "%s failed: %s", #call, cudaGetErrorString(e_)));            \
  } while (0)

  float* tmp_xyz = nullptr;
  TB_MC(cudaMalloc(&m->pts, 6 * n_points * sizeof(float4)));
  TB_MC(cudaMalloc(&tmp_xyz, n_points * 3 * sizeof(float)));
  TB_MC(cudaMemcpy(tmp_xyz, points_xyz, n_points * 3 * sizeof(float), cudaMemcpyHostToDevice));
  pad_points_kernel<<<grid_for(n_points, 256), 256>>>(tmp_xyz, m->pts, n_points);
  TB_MC(cudaGetLastError());
  TB_MC(cudaDeviceSynchronize());
  cudaFree(tmp_xyz);

  TB_MC(cudaMalloc(&m->sv, n_tets * sizeof(int4)));
  TB_MC(cudaMemcpy(m->sv, side_verts, n_tets * sizeof(int4), cudaMemcpyHostToDevice));
  TB_MC(cudaMalloc(&m->sn, n_tets * sizeof(uint4)));
  TB_MC(cudaMemcpy(m->sn, side_neighbors, n_tets * sizeof(uint4), cudaMemcpyHostToDevice));
  TB_MC(cudaMalloc(&m->orient, n_tets));
  orient_kernel<<<grid_for(n_tets, 256), 256>>>(m->sv, m->pts, m->orient, n_tets, n_points);
  TB_MC(cudaGetLastError());

  int64_t rec_bytes = 0;
  if (layout == 16) {
    rec_bytes = n_tets * 16;
    TB_MC(cudaMalloc(&m->rec4, rec_bytes));
    TB_MC(cudaMemcpy(m->rec4, records, rec_bytes, cudaMemcpyHostToDevice));
  } else if (layout == 32) {
    rec_bytes = n_tets * 32;
    TB_MC(cudaMalloc(&m->rec4, rec_bytes));
    TB_MC(cudaMemcpy(m->rec4, records, rec_bytes, cudaMemcpyHostToDevice));
  } else if (layout == 20) {
    rec_bytes = n_tets * 20;
    uint32_t* tmp = nullptr;
    TB_MC(cudaMalloc(&m->vx, n_tets * sizeof(uint32_t)));
    TB_MC(cudaMalloc(&m->rec4, n_tets * sizeof(uint4)));
    TB_MC(cudaMalloc(&tmp, rec_bytes));
    TB_MC(cudaMemcpy(tmp, records, rec_bytes, cudaMemcpyHostToDevice));
    split_tet20_kernel<<<grid_for(n_tets, 256), 256>>>(tmp, m->vx, m->rec4, n_tets);
    TB_MC(cudaGetLastError());
    TB_MC(cudaDeviceSynchronize());
    cudaFree(tmp);
  } else {  // 80
    rec_bytes = n_tets * 80;
    TB_MC(cudaMalloc(&m->rec4, rec_bytes));
    build_tet80_kernel<<<grid_for(n_tets, 256), 256>>>(m->sv, m->sn, m->pts, m->rec4, n_tets);
    TB_MC(cudaGetLastError());
    TB_MC(cudaDeviceSynchronize());
  }

  if (n_cf > 0) {
    TB_MC(cudaMalloc(&m->cf_tri, n_cf * sizeof(int32_t)));
    TB_MC(cudaMemcpy(m->cf_tri, cf_triangle, n_cf * sizeof(int32_t), cudaMemcpyHostToDevice));
    TB_MC(cudaMalloc(&m->cf_tets, n_cf * sizeof(int2)));
    TB_MC(cudaMemcpy(m->cf_tets, cf_tets, n_cf * sizeof(int2), cudaMemcpyHostToDevice));
  }
  {
    unsigned int* bad = nullptr;
    unsigned int hbad = 1;
    TB_MC(cudaMalloc(&bad, sizeof(unsigned int)));
    TB_MC(cudaMemset(bad, 0, sizeof(unsigned int)));
    validate_kernel<<<grid_for(n_tets, 256), 256>>>(layout, m->sv, m->sn, m->rec4, m->vx, n_tets, n_points, m->cf_tri,
                                                    m->cf_tets, n_cf, n_tri, bad);
    TB_MC(cudaGetLastError());
    TB_MC(cudaMemcpy(&hbad, bad, sizeof(unsigned int), cudaMemcpyDeviceToHost));
    cudaFree(bad);
    m->safe = hbad == 0 && layout != 80;
  }

  if (n_tri > 0) {
    TB_MC(cudaMalloc(&m->tri, n_tri * 9 * sizeof(double)));
    TB_MC(cudaMemcpy(m->tri, tri_coords, n_tri * 9 * sizeof(double), cudaMemcpyHostToDevice));
  }
#undef TB_MC
  m->hbm_bytes = n_points * 16 * 6 + n_tets * 33 + rec_bytes + n_cf * 12 + n_tri * 72;
  // Hot bytes the walk actually gathers from on this device: the records plus
  // the six axis-permuted float4 point copies (96 B per point; a ray reads one
  // copy, an incoherent batch all six).  TetMesh-80 reads only its records.
  // (The reference's accelerator -- records + 12 B f32 points -- is reported
  // beside it by bench.py as mesh_bytes.reference_accelerator_bytes.)
  m->hot_bytes = (layout == 80) ? rec_bytes : rec_bytes + n_points * 16 * 6;
  *out = m;
  return TB_OK;
}

// Device-to-device copy of an uploaded mesh (SURVEY 8 e: "mesh replicated --
// upload from pinned host memory, or broadcast from GPU 0").  Every device
// array is copied peer to peer (NVLink on a node); nothing is rebuilt or
// revalidated, so a replica costs one HBM-to-HBM copy of the mesh.
int tb_mesh_replicate(const tb_mesh* src, int device, tb_mesh** out) {
  if (int e = check_mesh(src)) return e;
  if (!out) return set_error(TB_E_ARG, "out is NULL");
  *out = nullptr;
  const int64_t np = src->n_points, nt = src->n_tets;
  const int64_t rec_bytes = src->layout == 16 ? nt * 16 : src->layout == 32 ? nt * 32 : src->layout == 20 ? nt * 16
                                                                                                            : nt * 80;
  tb_mesh* m = new tb_mesh();
  m->device = device;
  m->layout = src->layout;
  m->n_points = np; m->n_tets = nt; m->n_cf = src->n_cf; m->n_tri = src->n_tri;
  m->safe = src->safe;
  m->hbm_bytes = src->hbm_bytes;
  m->hot_bytes = src->hot_bytes;
  int err = TB_OK;
  auto copy = [&](auto*& dst, const void* from, int64_t bytes) {
    if (err != TB_OK || from == nullptr || bytes <= 0) return;
    DeviceGuard g(device);
    cudaError_t e = cudaMalloc((void**)&dst, (size_t)bytes);
    if (e == cudaSuccess) e = cudaMemcpyPeer(dst, device, from, src->device, (size_t)bytes);
    if (e != cudaSuccess)
      err = set_error(e == cudaErrorMemoryAllocation ? TB_E_OOM : TB_E_CUDA, "replicate to device %d: %s", device,
                      cudaGetErrorString(e));
  };
  copy(m->pts, src->pts, 6 * np * 16);
  copy(m->rec4, src->rec4, rec_bytes);
  copy(m->vx, src->vx, src->layout == 20 ? nt * 4 : 0);
  copy(m->sv, src->sv, nt * 16);
  copy(m->sn, src->sn, nt * 16);
  copy(m->orient, src->orient, nt);
  copy(m->cf_tri, src->cf_tri, src->n_cf * 4);
  copy(m->cf_tets, src->cf_tets, src->n_cf * 8);
  copy(m->tri, src->tri, src->n_tri * 72);
  if (err != TB_OK) {
    tb_mesh_destroy(m);
    return err;
  }
  *out = m;
  return TB_OK;
}

int tb_mesh_destroy(tb_mesh* m) {
  if (m == nullptr) return TB_OK;
  DeviceGuard g(m->device);
  cudaFree(m->pts);
  cudaFree(m->rec4);
  cudaFree(m->vx);
  cudaFree(m->sv);
  cudaFree(m->sn);
  cudaFree(m->cf_tri);
  cudaFree(m->cf_tets);
  cudaFree(m->tri);
  cudaFree(m->orient);
  delete m;
  return TB_OK;
}

int tb_mesh_info(const tb_mesh* m, int* device, int* layout, int64_t* n_points, int64_t* n_tets,
                 int64_t* n_cf, int64_t* hbm_bytes, int64_t* hot_bytes) {
  if (int e = check_mesh(m)) return e;
  if (device) *device = m->device;
  if (layout) *layout = m->layout;
  if (n_points) *n_points = m->n_points;
  if (n_tets) *n_tets = m->n_tets;
  if (n_cf) *n_cf = m->n_cf;
  if (hbm_bytes) *hbm_bytes = m->hbm_bytes;
  if (hot_bytes) *hot_bytes = m->hot_bytes;
  return TB_OK;
}

int tb_mesh_validated(const tb_mesh* m, int* validated) {
  if (int e = check_mesh(m)) return e;
  if (!validated) return set_error(TB_E_ARG, "validated is NULL");
  *validated = m->safe ? 1 : 0;
  return TB_OK;
}

int tb_probe_gather(tb_mesh* m, int64_t n_pairs, uint32_t seed, uint32_t* sink, void* stream) {
  if (int e = check_mesh(m)) return e;
  if (n_pairs < 0) return set_error(TB_E_ARG, "negative pair count");
  if (!sink) return set_error(TB_E_ARG, "sink is NULL");
  if (n_pairs == 0 || m->n_tets == 0 || m->n_points == 0) return TB_OK;
  DeviceGuard g(m->device);
  int sms = 0;
  TB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device));
  const unsigned grid = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((int64_t)sms * 16, (n_pairs + 256 * 8 - 1) / (256 * 8)));
  const cudaStream_t s = (cudaStream_t)stream;
  const MeshView v = m->view();
  switch (m->layout) {
    case 32: gather_probe_kernel<32><<<grid, 256, 0, s>>>(v, n_pairs, seed, sink); break;
    case 20: gather_probe_kernel<20><<<grid, 256, 0, s>>>(v, n_pairs, seed, sink); break;
    case 16: gather_probe_kernel<16><<<grid, 256, 0, s>>>(v, n_pairs, seed, sink); break;
    default: return set_error(TB_E_LAYOUT, "gather probe: layout %d has no separate point array", m->layout);
  }
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_cast_rays(tb_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                 uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle, double* t,
                 int32_t* tet_back, void* stream) {
  if (int e = check_mesh(m)) return e;
  if (n < 0) return set_error(TB_E_ARG, "negative ray count");
  if (n == 0) return TB_OK;
  if (!o || !d || !start || !status || !cf || !tet || !visited) return set_error(TB_E_ARG, "NULL ray buffer");
  // device pointers: auto = tb_auto_schedule (sampled longest-first for
  // launches of few waves, else one ray per lane; deciding coherence would
  // need a host round trip -- callers that know their batch is incoherent
  // select "binned")
  return cast_dispatch(m, n, o, d, start, status, cf, tet, visited, triangle, t, tet_back, (cudaStream_t)stream,
                       sched_mode());
}

int tb_cast_rays_scatter(tb_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                         const int64_t* out_index, uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited,
                         int32_t* triangle, double* t, int32_t* tet_back, void* stream) {
  if (int e = check_mesh(m)) return e;
  if (n < 0) return set_error(TB_E_ARG, "negative ray count");
  if (n == 0) return TB_OK;
  if (!o || !d || !start || !out_index || !status || !cf || !tet || !visited)
    return set_error(TB_E_ARG, "NULL ray buffer");
  return cast_dispatch(m, n, o, d, start, status, cf, tet, visited, triangle, t, tet_back, (cudaStream_t)stream, 1,
                       false, out_index);
}

int tb_cast_rays_scatter_sched(tb_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                               const int64_t* out_index, uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited,
                               int32_t* triangle, double* t, int32_t* tet_back, int schedule, void* stream) {
  if (int e = check_mesh(m)) return e;
  if (n < 0) return set_error(TB_E_ARG, "negative ray count");
  if (schedule < 0 || schedule > 7) return set_error(TB_E_ARG, "schedule %d not in 0..7", schedule);
  if (n == 0) return TB_OK;
  if (!o || !d || !start || !out_index || !status || !cf || !tet || !visited)
    return set_error(TB_E_ARG, "NULL ray buffer");
  return cast_dispatch(m, n, o, d, start, status, cf, tet, visited, triangle, t, tet_back, (cudaStream_t)stream,
                       schedule == 0 ? sched_mode() : schedule, false, out_index);
}

int tb_sctp_cast_rays_scatter(tb_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                              const int64_t* out_index, uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited,
                              int32_t* triangle, double* t, int32_t* tet_back, void* stream) {
  if (int e = check_mesh(m)) return e;
  if (n < 0) return set_error(TB_E_ARG, "negative ray count");
  if (n == 0) return TB_OK;
  if (!o || !d || !start || !out_index || !status || !cf || !tet || !visited)
    return set_error(TB_E_ARG, "NULL ray buffer");
  DeviceGuard g(m->device);
  if (int e = launch_layout<SctpL>(m->layout, grid_for(n, kBlock), (cudaStream_t)stream, m->view(), n, o, d, start,
                                   status, cf, tet, visited, triangle, t, tet_back, out_index))
    return e;
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

// Single-process multi-GPU trace (SURVEY 8 b's tb_trace_multi).  The frame's
// 16 x 16-pixel tiles (render.py:496-514 order) go round-robin to the meshes;
// every mesh's device walks its tiles straight from the frame's ray arrays on
// meshes[0]'s device and stores each result into the frame's output arrays
// there (cast_kernel's kGather + kScatter path: P2P loads and stores over
// NVLink for the other devices, no staging copies, no collective).
namespace {
struct ShardKey {
  int device;
  int64_t width, height;
  int parts, part;
  bool operator<(const ShardKey& o) const {
    return std::tie(device, width, height, parts, part) < std::tie(o.device, o.width, o.height, o.parts, o.part);
  }
};
std::mutex g_shard_mu;
std::map<ShardKey, std::pair<int32_t*, int64_t>> g_shards;  // device index arrays, kept for the process

int shard_indices(int device, int64_t W, int64_t H, int parts, int part, const int32_t** idx, int64_t* count) {
  std::lock_guard<std::mutex> lk(g_shard_mu);
  const ShardKey key{device, W, H, parts, part};
  auto it = g_shards.find(key);
  if (it == g_shards.end()) {
    if (W * H > INT32_MAX) return set_error(TB_E_ARG, "frame of %lld pixels: pixel indices exceed int32", (long long)(W * H));
    std::vector<int32_t> h;
    const int64_t tx = (W + 15) / 16, ty = (H + 15) / 16;
    for (int64_t k = part; k < tx * ty; k += parts) {
      const int64_t x0 = (k % tx) * 16, y0 = (k / tx) * 16;
      for (int64_t y = y0; y < std::min(H, y0 + 16); ++y)
        for (int64_t x = x0; x < std::min(W, x0 + 16); ++x) h.push_back((int32_t)(y * W + x));
    }
    int32_t* dptr = nullptr;
    if (!h.empty()) {
      DeviceGuard g(device);
      TB_CUDA(cudaMalloc((void**)&dptr, h.size() * sizeof(int32_t)));
      TB_CUDA(cudaMemcpy(dptr, h.data(), h.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    it = g_shards.emplace(key, std::make_pair(dptr, (int64_t)h.size())).first;
  }
  *idx = it->second.first;
  *count = it->second.second;
  return TB_OK;
}

// one non-blocking stream per (host thread, device) for the non-root devices
// Per host thread and device; destroyed when the thread exits.
struct MultiStreams {
  cudaStream_t s[64] = {};
  ~MultiStreams() {
    for (int dv = 0; dv < 64; ++dv) {
      if (!s[dv]) continue;
      int prev = -1;
      cudaGetDevice(&prev);
      cudaSetDevice(dv);
      cudaStreamSynchronize(s[dv]);
      cudaStreamDestroy(s[dv]);
      if (prev >= 0) cudaSetDevice(prev);
    }
    cudaGetLastError();  // teardown errors (runtime already unloading) are not reportable
  }
};
cudaStream_t multi_stream(int device) {
  static thread_local MultiStreams streams;
  if (device < 0 || device >= 64) return nullptr;
  if (!streams.s[device]) {
    DeviceGuard g(device);
    cudaStreamCreateWithFlags(&streams.s[device], cudaStreamNonBlocking);
  }
  return streams.s[device];
}
}  // namespace

int tb_trace_multi(int n_meshes, tb_mesh* const* meshes, int64_t width, int64_t height, const float* o,
                   const float* d, const int32_t* start, uint8_t* status, int32_t* cf, int32_t* tet,
                   int32_t* visited, int32_t* triangle, double* t, int32_t* tet_back, void* stream) {
  if (n_meshes < 1 || n_meshes > 64 || !meshes) return set_error(TB_E_ARG, "n_meshes %d not in 1..64", n_meshes);
  if (width < 0 || height < 0 || width * height >= ((int64_t)1 << 40)) return set_error(TB_E_ARG, "bad frame size");
  if (width * height == 0) return TB_OK;
  if (!o || !d || !start || !status || !cf || !tet || !visited) return set_error(TB_E_ARG, "NULL ray buffer");
  for (int k = 0; k < n_meshes; ++k) {
    if (int e = check_mesh(meshes[k])) return e;
    if (meshes[k]->layout != meshes[0]->layout || meshes[k]->n_tets != meshes[0]->n_tets)
      return set_error(TB_E_ARG, "mesh %d is not a replica of mesh 0 (layout / size differ)", k);
  }
  const int d0 = meshes[0]->device;
  const cudaStream_t s0 = (cudaStream_t)stream;
  cudaEvent_t ready = nullptr;
  {
    DeviceGuard g(d0);
    TB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    TB_CUDA(cudaEventRecord(ready, s0));  // the rays are written on the caller's stream
  }
  int err = TB_OK;
  std::vector<cudaEvent_t> done;
  for (int k = 0; k < n_meshes && err == TB_OK; ++k) {
    tb_mesh* m = meshes[k];
    const int32_t* idx = nullptr;
    int64_t count = 0;
    if ((err = shard_indices(m->device, width, height, n_meshes, k, &idx, &count)) != TB_OK || count == 0) continue;
    DeviceGuard g(m->device);
    if (m->device != d0) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, m->device, d0);
      if (!can) {
        err = set_error(TB_E_CUDA, "device %d cannot access device %d's memory (no P2P)", m->device, d0);
        break;
      }
      const cudaError_t pe = cudaDeviceEnablePeerAccess(d0, 0);
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) {
        err = set_error(TB_E_CUDA, "enable peer access %d -> %d: %s", m->device, d0, cudaGetErrorString(pe));
        break;
      }
      cudaGetLastError();
    }
    const cudaStream_t sk = m->device == d0 ? s0 : multi_stream(m->device);
    if (sk != s0 && cudaStreamWaitEvent(sk, ready, 0) != cudaSuccess) {
      err = set_error(TB_E_CUDA, "cross-device wait failed");
      break;
    }
    if ((err = launch_layout<CastBinnedL>(m->layout, grid_for(count, kCastBlock), sk, m->safe, idx, nullptr, m->view(), count, o,
                                          d, start, status, cf, tet, visited, triangle, t, tet_back)) != TB_OK)
      break;
    if (sk != s0) {
      cudaEvent_t ev = nullptr;
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess || cudaEventRecord(ev, sk) != cudaSuccess) {
        err = set_error(TB_E_CUDA, "event on device %d failed", m->device);
        break;
      }
      done.push_back(ev);
    }
  }
  {
    DeviceGuard g(d0);
    for (cudaEvent_t ev : done) {
      if (cudaStreamWaitEvent(s0, ev, 0) != cudaSuccess && err == TB_OK) err = set_error(TB_E_CUDA, "join failed");
      cudaEventDestroy(ev);  // released once the wait has been enqueued
    }
    cudaEventDestroy(ready);
  }
  if (err == TB_OK) {
    DeviceGuard g(d0);
    TB_CUDA(cudaGetLastError());
  }
  return err;
}

int tb_cast_epilogue(tb_mesh* m, int64_t n, const float* o, const float* d, const int32_t* cf, const int32_t* tet,
                     int32_t* triangle, double* t, int32_t* tet_back, void* stream) {
  if (int e = check_mesh(m)) return e;
  if (n < 0) return set_error(TB_E_ARG, "negative ray count");
  if (n == 0) return TB_OK;
  if (!o || !d || !cf || !tet) return set_error(TB_E_ARG, "NULL buffer");
  DeviceGuard g(m->device);
  epilogue_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(m->view(), n, o, d, cf, tet, triangle, t,
                                                                         tet_back);
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_device_alloc(size_t bytes, int device, void** out) {
  if (!out) return set_error(TB_E_ARG, "out is NULL");
  DeviceGuard g(device);
  TB_CUDA(cudaMalloc(out, bytes ? bytes : 1));
  return TB_OK;
}

int tb_device_free(void* ptr) {
  if (ptr) TB_CUDA(cudaFree(ptr));
  return TB_OK;
}

int tb_ipc_get_handle(const void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return set_error(TB_E_ARG, "NULL pointer");
  cudaIpcMemHandle_t h;
  TB_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  memcpy(handle_out, &h, sizeof(h));
  return TB_OK;
}

int tb_ipc_open(const void* handle, int device, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return set_error(TB_E_ARG, "NULL pointer");
  DeviceGuard g(device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  TB_CUDA(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return TB_OK;
}

int tb_ipc_close(void* dev_ptr) {
  if (dev_ptr) TB_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return TB_OK;
}

int tb_cast_rays_sched(tb_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                       uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle, double* t,
                       int32_t* tet_back, int schedule, void* stream) {
  if (int e = check_mesh(m)) return e;
  if (n < 0) return set_error(TB_E_ARG, "negative ray count");
  if (schedule < 0 || schedule > 7) return set_error(TB_E_ARG, "schedule %d not in 0..7", schedule);
  if (n == 0) return TB_OK;
  if (!o || !d || !start || !status || !cf || !tet || !visited) return set_error(TB_E_ARG, "NULL ray buffer");
  return cast_dispatch(m, n, o, d, start, status, cf, tet, visited, triangle, t, tet_back, (cudaStream_t)stream,
                       schedule == 0 ? sched_mode() : schedule);
}

int tb_cast_block_size(void) { return kCastBlock; }

int tb_auto_schedule(int device, int64_t n) { return n < 0 ? -1 : auto_schedule(device, n); }

int tb_binned_pieces(int64_t n) {
  if (n < 0) return -1;
  const int n_tiles = (int)((n + kBinTile - 1) / kBinTile);
  const int S = bin_tile() / kBinTile;
  return (S && (n_tiles + S - 1) / S >= 2 && bin_split()) ? 2 : 1;
}

int64_t tb_sampled_head_blocks(int device, int64_t n) {
  return n < 0 ? -1 : head_blocks(device, (n + kCastBlock - 1) / kCastBlock);
}

int tb_block_order(int64_t n, const int32_t* visited, int32_t* order, int64_t n_blocks, void* stream) {
  if (n < 0) return set_error(TB_E_ARG, "negative ray count");
  const int64_t nb = (n + kCastBlock - 1) / kCastBlock;
  if (n_blocks != nb) return set_error(TB_E_ARG, "order must hold the %lld blocks of %d rays", (long long)nb,
                                       kCastBlock);
  if (nb == 0) return TB_OK;
  if (!visited || !order) return set_error(TB_E_ARG, "NULL buffer");
  if (nb > (int64_t)INT32_MAX) return set_error(TB_E_ARG, "too many blocks");
  int dev = 0;
  TB_CUDA(cudaGetDevice(&dev));
  const cudaStream_t s = (cudaStream_t)stream;
  // scratch: keys + histogram + cursors, from the per-device pool that keeps its memory
  const size_t kb = ((size_t)nb + 255) / 256 * 256, hb = 2 * kOrderBuckets * sizeof(int);
  char* scratch = nullptr;
  if (int e = scratch_alloc(dev, kb + hb, s, &scratch)) return e;
  uint8_t* key = reinterpret_cast<uint8_t*>(scratch);
  int* hist = reinterpret_cast<int*>(scratch + kb);
  int* cursor = hist + kOrderBuckets;
  cudaMemsetAsync(hist, 0, hb, s);
  block_key_kernel<<<grid_for(nb * 32, 256), 256, 0, s>>>(visited, n, nb, key, hist);
  block_scatter_kernel<<<grid_for(nb, 256), 256, 0, s>>>(key, nb, hist, cursor, order);
  const cudaError_t e = cudaGetLastError();
  cudaFreeAsync(scratch, s);
  TB_CUDA(e);
  return TB_OK;
}

int tb_cast_rays_ordered(tb_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                         const int32_t* block_order, int64_t n_blocks, uint8_t* status, int32_t* cf, int32_t* tet,
                         int32_t* visited, int32_t* triangle, double* t, int32_t* tet_back, void* stream) {
  if (int e = check_mesh(m)) return e;
  if (n < 0) return set_error(TB_E_ARG, "negative ray count");
  if (n == 0) return TB_OK;
  if (!o || !d || !start || !status || !cf || !tet || !visited) return set_error(TB_E_ARG, "NULL ray buffer");
  const int64_t nb = (n + kCastBlock - 1) / kCastBlock;
  if (!block_order || n_blocks != nb)
    return set_error(TB_E_ARG, "block_order must list the %lld blocks of %d rays (got %lld)", (long long)nb,
                     kCastBlock, (long long)n_blocks);
  DeviceGuard g(m->device);
  // the order is a permutation of [0, nb) (the caller's contract; an entry
  // out of range only reads past the rays' blocks, which r >= n guards)
  int e = launch_layout<CastOrderedL>(m->layout, (unsigned)nb, (cudaStream_t)stream, m->safe, block_order, m->view(),
                                      n, o, d, start, status, cf, tet, visited, triangle, t, tet_back);
  if (e) return e;
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_sctp_cast_rays(tb_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                      uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle,
                      double* t, int32_t* tet_back, void* stream) {
  if (int e = check_mesh(m)) return e;
  if (n < 0) return set_error(TB_E_ARG, "negative ray count");
  if (n == 0) return TB_OK;
  if (!o || !d || !start || !status || !cf || !tet || !visited) return set_error(TB_E_ARG, "NULL ray buffer");
  DeviceGuard g(m->device);
  const cudaStream_t s = (cudaStream_t)stream;
  if (int e = launch_layout<SctpL>(m->layout, grid_for(n, kBlock), s, m->view(), n, o, d, start, status, cf,
                                   tet, visited, triangle, t, tet_back, (const int64_t*)nullptr))
    return e;
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_cast_rays_visits(tb_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                        const int64_t* offsets, int32_t* seq, void* stream) {
  if (int e = check_mesh(m)) return e;
  if (n < 0) return set_error(TB_E_ARG, "negative ray count");
  if (n == 0) return TB_OK;
  if (!o || !d || !start || !offsets || !seq) return set_error(TB_E_ARG, "NULL buffer");
  DeviceGuard g(m->device);
  const cudaStream_t s = (cudaStream_t)stream;
  if (int e = launch_layout<VisitsL>(m->layout, grid_for(n, kBlock), s, m->view(), n, o, d, start, offsets, seq))
    return e;
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_camera_rays(int64_t width, int64_t height, const double* frame, const int64_t* pixels, int64_t n, float* o,
                   float* d, void* stream) {
  if (width <= 0 || height <= 0 || n < 0) return set_error(TB_E_ARG, "bad camera size");
  if (n == 0) return TB_OK;
  if (!frame || !o || !d) return set_error(TB_E_ARG, "NULL buffer");
  camera_rays_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(width, height, frame, pixels, n, o, d);
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_trace_camera(tb_mesh* m, int64_t width, int64_t height, const double* frame, int32_t cam_tet, uint8_t* status,
                    int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle, double* t, int32_t* tet_back,
                    void* stream) {
  if (int e = check_mesh(m)) return e;
  if (width <= 0 || height <= 0) return set_error(TB_E_ARG, "bad camera size");
  if (!frame || !status || !cf || !tet || !visited) return set_error(TB_E_ARG, "NULL buffer");
  if (cam_tet < 0 || cam_tet >= m->n_tets) return set_error(TB_E_ARG, "camera tet %d out of range", cam_tet);
  CamFrame fr;
  for (int k = 0; k < 14; ++k) fr.f[k] = frame[k];
  DeviceGuard g(m->device);
  const int64_t n = width * height;
  if (int e = launch_layout<CameraCastL>(m->layout, grid_for(n, kCastBlock), (cudaStream_t)stream, m->safe, m->view(),
                                         width, height, fr, (uint32_t)cam_tet, status, cf, tet, visited, triangle, t,
                                         tet_back))
    return e;
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_hull_clip(tb_mesh* m, int64_t n, const float* o, const float* d, const int32_t* rays, int64_t n_hull,
                 const int32_t* hull, int32_t* best_face, double* best_t, void* stream) {
  if (int e = check_mesh(m)) return e;
  if (n < 0 || n_hull < 0) return set_error(TB_E_ARG, "negative count");
  if (n == 0) return TB_OK;
  if (!o || !d || !best_face || !best_t || (n_hull > 0 && !hull)) return set_error(TB_E_ARG, "NULL buffer");
  DeviceGuard g(m->device);
  hull_clip_kernel<<<grid_for(n, kBlock), kBlock, 0, (cudaStream_t)stream>>>(
      m->view(), n, o, d, rays, n_hull, reinterpret_cast<const int4*>(hull), best_face, best_t);
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_locate_points(tb_mesh* m, int64_t n, const double* q, const int32_t* hints, int32_t* tet,
                     int32_t* visited, void* stream) {
  if (int e = check_mesh(m)) return e;
  if (n < 0) return set_error(TB_E_ARG, "negative point count");
  if (n == 0) return TB_OK;
  if (!q || !hints || !tet || !visited) return set_error(TB_E_ARG, "NULL buffer");
  DeviceGuard g(m->device);
  const cudaStream_t s = (cudaStream_t)stream;
  if (int e = launch_layout<LocateL>(m->layout, grid_for(n, kBlock), s, m->view(), n, q, hints, tet, visited))
    return e;
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

int tb_shadow_rays(tb_mesh* m, int64_t n, const double* p, const double* light, int light_stride,
                   const int32_t* p_tet, const int32_t* light_tet, int light_tet_stride, double eps,
                   uint8_t* occluded, int32_t* visited, void* stream) {
  if (int e = check_mesh(m)) return e;
  if (n < 0) return set_error(TB_E_ARG, "negative ray count");
  if (n == 0) return TB_OK;
  if (!p || !light || !p_tet || !light_tet || !occluded || !visited) return set_error(TB_E_ARG, "NULL buffer");
  if ((light_stride != 0 && light_stride != 3) || (light_tet_stride != 0 && light_tet_stride != 1))
    return set_error(TB_E_ARG, "bad light strides %d/%d", light_stride, light_tet_stride);
  DeviceGuard g(m->device);
  const cudaStream_t s = (cudaStream_t)stream;
  if (int e = launch_layout<ShadowL>(m->layout, grid_for(n, kBlock), s, m->safe, m->view(), n, p, light, light_stride,
                                     p_tet, light_tet, light_tet_stride, eps, occluded, visited))
    return e;
  TB_CUDA(cudaGetLastError());
  return TB_OK;
}

// ----------------------------------------------------------------------------
// Host-buffer entry points (what the kernel-module protocol calls: numpy
// arrays in, numpy arrays out).  Streams and staging come from a
// process-wide pool of slots per device, checked out per call and returned
// after it -- never owned by a host thread -- so a renderer whose tile pool
// creates and joins threads every frame (render.py:538-541) pays no
// per-thread allocation, stream creation or implicit device synchronisation
// at thread exit (r01's per-thread contexts made 256..65536-ray calls 2-3x
// slower than the CPU reference; bench small_batch).  Pageable buffers are
// staged through the slot's pinned, mapped host memory and the kernels read
// and write that memory over PCIe themselves: one launch and one sync per
// chunk, chunks double-buffered so host memcpy overlaps the GPU.
}  // extern "C"
namespace {

inline size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }

struct HostSlot {
  int device = -1;
  cudaStream_t s = nullptr;
  char* h = nullptr;   // pinned, mapped host staging
  char* hd = nullptr;  // its device alias
  size_t h_bytes = 0;
  int host(size_t b) {
    if (h_bytes >= b) return TB_OK;
    if (h) {
      cudaStreamSynchronize(s);
      cudaFreeHost(h);
    }
    h = hd = nullptr;
    h_bytes = 0;
    const size_t want = std::max(b, (size_t)1 << 20);
    TB_CUDA(cudaHostAlloc((void**)&h, want, cudaHostAllocMapped | cudaHostAllocPortable));
    if (cudaError_t e = cudaHostGetDevicePointer((void**)&hd, h, 0)) {
      cudaFreeHost(h);
      h = nullptr;
      return set_error(TB_E_CUDA, "mapped staging: %s", cudaGetErrorString(e));
    }
    h_bytes = want;
    return TB_OK;
  }
  // device alias of a pointer into h
  template <typename T>
  T* dev(T* p) const { return reinterpret_cast<T*>(hd + (reinterpret_cast<char*>(p) - h)); }
};

std::mutex g_slot_mu;
std::vector<HostSlot*> g_free_slots[64];

int slot_get(int device, HostSlot** out) {
  if (device < 0 || device >= 64) return set_error(TB_E_ARG, "device %d out of range", device);
  {
    std::lock_guard<std::mutex> lk(g_slot_mu);
    if (!g_free_slots[device].empty()) {
      *out = g_free_slots[device].back();
      g_free_slots[device].pop_back();
      return TB_OK;
    }
  }
  HostSlot* sl = new HostSlot();
  sl->device = device;
  DeviceGuard g(device);
  if (cudaError_t e = cudaStreamCreateWithFlags(&sl->s, cudaStreamNonBlocking)) {
    delete sl;
    return set_error(TB_E_CUDA, "host-path stream: %s", cudaGetErrorString(e));
  }
  *out = sl;
  return TB_OK;
}

// Returns the slot to the pool after draining its stream (error paths
// included: nothing queued may still touch the staging afterwards).
struct SlotLease {
  HostSlot* p = nullptr;
  SlotLease() = default;
  SlotLease(const SlotLease&) = delete;
  SlotLease& operator=(const SlotLease&) = delete;
  ~SlotLease() {
    if (!p) return;
    cudaStreamSynchronize(p->s);
    std::lock_guard<std::mutex> lk(g_slot_mu);
    g_free_slots[p->device].push_back(p);
  }
};

// Device-staged copy pipeline (TETB200_E2E=1 only: an A/B knob against the
// zero-copy path): three streams, each with HBM staging for one chunk.
struct PipeCtx {
  static constexpr int kStreams = 3;
  static constexpr int64_t kChunk = 1 << 18;  // rays per pipeline chunk
  int device = -1;
  struct Slot {
    cudaStream_t s = nullptr;
    char* base = nullptr;
    float *o = nullptr, *d = nullptr;
    int32_t *st = nullptr, *cf = nullptr, *tet = nullptr, *vis = nullptr, *tri = nullptr, *back = nullptr;
    uint8_t* status = nullptr;
    double* t = nullptr;
  } slot[kStreams];
};

std::vector<PipeCtx*> g_free_pipes[64];

int pipe_get(int device, PipeCtx** out) {
  if (device < 0 || device >= 64) return set_error(TB_E_ARG, "device %d out of range", device);
  {
    std::lock_guard<std::mutex> lk(g_slot_mu);
    if (!g_free_pipes[device].empty()) {
      *out = g_free_pipes[device].back();
      g_free_pipes[device].pop_back();
      return TB_OK;
    }
  }
  PipeCtx* c = new PipeCtx();
  c->device = device;
  const size_t k = (size_t)PipeCtx::kChunk;
  for (int i = 0; i < PipeCtx::kStreams; ++i) {
    PipeCtx::Slot& sl = c->slot[i];
    cudaError_t e = cudaStreamCreateWithFlags(&sl.s, cudaStreamNonBlocking);
    const size_t total = al256(k * 12) * 2 + al256(k * 4) * 6 + al256(k) + al256(k * 8);
    if (e == cudaSuccess) e = cudaMalloc((void**)&sl.base, total);
    if (e != cudaSuccess) {
      for (PipeCtx::Slot& x : c->slot) {
        if (x.s) cudaStreamDestroy(x.s);
        if (x.base) cudaFree(x.base);
      }
      delete c;
      return set_error(e == cudaErrorMemoryAllocation ? TB_E_OOM : TB_E_CUDA, "host-path staging: %s",
                       cudaGetErrorString(e));
    }
    char* p = sl.base;
    auto take = [&](size_t bytes) { char* q = p; p += al256(bytes); return q; };
    sl.o = reinterpret_cast<float*>(take(k * 12));
    sl.d = reinterpret_cast<float*>(take(k * 12));
    sl.st = reinterpret_cast<int32_t*>(take(k * 4));
    sl.status = reinterpret_cast<uint8_t*>(take(k));
    sl.cf = reinterpret_cast<int32_t*>(take(k * 4));
    sl.tet = reinterpret_cast<int32_t*>(take(k * 4));
    sl.vis = reinterpret_cast<int32_t*>(take(k * 4));
    sl.tri = reinterpret_cast<int32_t*>(take(k * 4));
    sl.t = reinterpret_cast<double*>(take(k * 8));
    sl.back = reinterpret_cast<int32_t*>(take(k * 4));
  }
  *out = c;
  return TB_OK;
}

struct PipeLease {
  PipeCtx* p = nullptr;
  ~PipeLease() {
    if (!p) return;
    for (PipeCtx::Slot& sl : p->slot) cudaStreamSynchronize(sl.s);
    std::lock_guard<std::mutex> lk(g_slot_mu);
    g_free_pipes[p->device].push_back(p);
  }
};

// Device address of a mapped pinned host buffer (false for pageable memory).
bool mapped_ptr(const void* p, void** dev) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a.type != cudaMemoryTypeHost || a.devicePointer == nullptr) return false;
  *dev = a.devicePointer;
  return true;
}

// TETB200_E2E: 0 = auto (zero-copy: mapped pinned buffers directly, pageable
// ones through pinned staging), 1 = the device-staged copy pipeline.
int e2e_mode() {
  const char* v = getenv("TETB200_E2E");
  return v ? atoi(v) : 0;
}

// Rays per pinned staging chunk for pageable buffers (double-buffered).
constexpr int64_t kHostChunk = 1 << 17;

// Per-ray staging of one cast chunk of C rays in a slot's pinned memory.
struct CastStage {
  float *o, *d;
  int32_t* st;
  uint8_t* status;
  int32_t *cf, *tet, *vis, *tri, *back;
  double* t;
  static size_t bytes(size_t C) {
    return al256(C * 12) * 2 + al256(C * 4) * 6 + al256(C) + al256(C * 8);
  }
  CastStage(char* base, size_t C) {
    char* p = base;
    auto take = [&](size_t b) { char* q = p; p += al256(b); return q; };
    o = reinterpret_cast<float*>(take(C * 12));
    d = reinterpret_cast<float*>(take(C * 12));
    st = reinterpret_cast<int32_t*>(take(C * 4));
    status = reinterpret_cast<uint8_t*>(take(C));
    cf = reinterpret_cast<int32_t*>(take(C * 4));
    tet = reinterpret_cast<int32_t*>(take(C * 4));
    vis = reinterpret_cast<int32_t*>(take(C * 4));
    tri = reinterpret_cast<int32_t*>(take(C * 4));
    t = reinterpret_cast<double*>(take(C * 8));
    back = reinterpret_cast<int32_t*>(take(C * 4));
  }
};

}  // namespace

extern "C" {

}  // extern "C"

namespace {

// Host-buffer traversal (both walks).
int cast_host(tb_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start, uint8_t* status,
              int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle, double* t, int32_t* tet_back,
              bool sctp) {
  if (int e = check_mesh(m)) return e;
  if (n < 0) return set_error(TB_E_ARG, "negative ray count");
  if (n == 0) return TB_OK;
  if (!o || !d || !start || !status || !cf || !tet || !visited) return set_error(TB_E_ARG, "NULL ray buffer");
  DeviceGuard g(m->device);
  const int mode = e2e_mode();
  // Host batches run one ray per lane unless a schedule is set: the walk
  // hides under PCIe time here, and the zero-copy path depends on
  // cast_kernel's warp-cooperative coalesced ray loads (r01: config 4 e2e
  // 1354 Mrays/s zero-copy lane vs 1156 staged compaction; zero-copy
  // compaction, whose refills and epilogue read rays lane by lane over
  // PCIe, 64 Mrays/s).
  const int sched = sched_mode();
  auto launch = [&](int64_t k, const float* ko, const float* kd, const int32_t* ks, uint8_t* kst, int32_t* kcf,
                    int32_t* ktet, int32_t* kvis, int32_t* ktri, double* kt, int32_t* kback, cudaStream_t s,
                    bool host_rays) {
    return sctp ? tb_sctp_cast_rays(m, k, ko, kd, ks, kst, kcf, ktet, kvis, ktri, kt, kback, s)
                : cast_dispatch(m, k, ko, kd, ks, kst, kcf, ktet, kvis, ktri, kt, kback, s, sched, host_rays);
  };
  // Zero-copy path: when every buffer is mapped pinned host memory
  // (cudaHostAlloc / torch pin_memory under UVA), the trace kernel reads the
  // rays and writes the hits straight over PCIe -- one launch, no staging
  // copies; reads and writes use the two link directions concurrently.
  void *dO, *dD, *dS, *dSt, *dCf, *dTet, *dVis, *dTri = nullptr, *dT = nullptr, *dBack = nullptr;
  const bool outs_mapped = mapped_ptr(status, &dSt) && mapped_ptr(cf, &dCf) && mapped_ptr(tet, &dTet) &&
                           mapped_ptr(visited, &dVis) && (!triangle || mapped_ptr(triangle, &dTri)) &&
                           (!t || mapped_ptr(t, &dT)) && (!tet_back || mapped_ptr(tet_back, &dBack));
  const bool ins_mapped = mapped_ptr(o, &dO) && mapped_ptr(d, &dD) && mapped_ptr(start, &dS);
  if (mode == 0 && outs_mapped && ins_mapped) {
    SlotLease L;
    if (int e = slot_get(m->device, &L.p)) return e;
    if (int e = launch(n, (const float*)dO, (const float*)dD, (const int32_t*)dS, (uint8_t*)dSt, (int32_t*)dCf,
                       (int32_t*)dTet, (int32_t*)dVis, (int32_t*)dTri, (double*)dT, (int32_t*)dBack, L.p->s, true))
      return e;
    TB_CUDA(cudaStreamSynchronize(L.p->s));
    return TB_OK;
  }
  if (mode == 0) {
    // Pageable buffers: chunks staged through pinned, mapped slots (two,
    // alternating, when the batch spans several chunks) -- the caller's
    // thread copies chunk c in while the GPU walks chunk c-1 straight from
    // / into the other slot's pinned memory.
    const int64_t C = n < kHostChunk ? n : kHostChunk;
    const int k = n > C ? 2 : 1;
    SlotLease L[2];
    for (int i = 0; i < k; ++i) {
      if (int e = slot_get(m->device, &L[i].p)) return e;
      if (int e = L[i].p->host(CastStage::bytes((size_t)C))) return e;
    }
    int64_t c_start[2] = {-1, -1}, c_len[2] = {0, 0};
    auto drain = [&](int i) -> int {
      if (c_start[i] < 0) return TB_OK;
      TB_CUDA(cudaStreamSynchronize(L[i].p->s));
      const CastStage v(L[i].p->h, (size_t)C);
      const int64_t a = c_start[i];
      const size_t len = (size_t)c_len[i];
      memcpy(status + a, v.status, len);
      memcpy(cf + a, v.cf, len * 4);
      memcpy(tet + a, v.tet, len * 4);
      memcpy(visited + a, v.vis, len * 4);
      if (triangle) memcpy(triangle + a, v.tri, len * 4);
      if (t) memcpy(t + a, v.t, len * 8);
      if (tet_back) memcpy(tet_back + a, v.back, len * 4);
      c_start[i] = -1;
      return TB_OK;
    };
    for (int64_t c0 = 0, c = 0; c0 < n; c0 += C, ++c) {
      const int i = (int)(c % k);
      if (int e = drain(i)) return e;
      const int64_t len = (n - c0 < C) ? (n - c0) : C;
      HostSlot& sl = *L[i].p;
      const CastStage v(sl.h, (size_t)C);
      memcpy(v.o, o + 3 * c0, (size_t)len * 12);
      memcpy(v.d, d + 3 * c0, (size_t)len * 12);
      memcpy(v.st, start + c0, (size_t)len * 4);
      if (int e = launch(len, sl.dev(v.o), sl.dev(v.d), sl.dev(v.st), sl.dev(v.status), sl.dev(v.cf), sl.dev(v.tet),
                         sl.dev(v.vis), triangle ? sl.dev(v.tri) : nullptr, t ? sl.dev(v.t) : nullptr,
                         tet_back ? sl.dev(v.back) : nullptr, sl.s, true))
        return e;
      c_start[i] = c0;
      c_len[i] = len;
    }
    for (int i = 0; i < k; ++i)
      if (int e = drain(i)) return e;
    return TB_OK;
  }
  // TETB200_E2E=1: chunked 3-stream copy pipeline through HBM staging --
  // chunk c's H2D, kernel and D2H are ordered on stream c % 3, so copies of
  // one chunk overlap the trace of the previous one (an A/B knob; r01 chose
  // zero copy).
  PipeLease P;
  if (int e = pipe_get(m->device, &P.p)) return e;
  PipeCtx* ctx = P.p;
  int64_t chunk = PipeCtx::kChunk;
  if (const char* v = getenv("TETB200_CHUNK")) {  // experiment knob: rays per chunk (<= kChunk)
    const int64_t c = atoll(v);
    if (c > 0 && c < chunk) chunk = c;
  }
#define TB_CUDA_PIPE(call)                                                                          \
  do {                                                                                              \
    cudaError_t e_ = (call);                                                                        \
    if (e_ != cudaSuccess) return set_error(TB_E_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
  for (int64_t c0 = 0, c = 0; c0 < n; c0 += chunk, ++c) {
    const int64_t k = (n - c0 < chunk) ? (n - c0) : chunk;
    const size_t uk = (size_t)k;
    PipeCtx::Slot& sl = ctx->slot[c % PipeCtx::kStreams];
    const cudaStream_t s = sl.s;
    TB_CUDA_PIPE(cudaMemcpyAsync(sl.o, o + 3 * c0, uk * 12, cudaMemcpyHostToDevice, s));
    TB_CUDA_PIPE(cudaMemcpyAsync(sl.d, d + 3 * c0, uk * 12, cudaMemcpyHostToDevice, s));
    TB_CUDA_PIPE(cudaMemcpyAsync(sl.st, start + c0, uk * 4, cudaMemcpyHostToDevice, s));
    if (int e = launch(k, sl.o, sl.d, sl.st, sl.status, sl.cf, sl.tet, sl.vis, triangle ? sl.tri : nullptr,
                       t ? sl.t : nullptr, tet_back ? sl.back : nullptr, s, false))
      return e;
    TB_CUDA_PIPE(cudaMemcpyAsync(status + c0, sl.status, uk, cudaMemcpyDeviceToHost, s));
    TB_CUDA_PIPE(cudaMemcpyAsync(cf + c0, sl.cf, uk * 4, cudaMemcpyDeviceToHost, s));
    TB_CUDA_PIPE(cudaMemcpyAsync(tet + c0, sl.tet, uk * 4, cudaMemcpyDeviceToHost, s));
    TB_CUDA_PIPE(cudaMemcpyAsync(visited + c0, sl.vis, uk * 4, cudaMemcpyDeviceToHost, s));
    if (triangle) TB_CUDA_PIPE(cudaMemcpyAsync(triangle + c0, sl.tri, uk * 4, cudaMemcpyDeviceToHost, s));
    if (t) TB_CUDA_PIPE(cudaMemcpyAsync(t + c0, sl.t, uk * 8, cudaMemcpyDeviceToHost, s));
    if (tet_back) TB_CUDA_PIPE(cudaMemcpyAsync(tet_back + c0, sl.back, uk * 4, cudaMemcpyDeviceToHost, s));
  }
#undef TB_CUDA_PIPE
  for (int i = 0; i < PipeCtx::kStreams; ++i) TB_CUDA(cudaStreamSynchronize(ctx->slot[i].s));
  return TB_OK;
}

}  // namespace

extern "C" {

int tb_cast_rays_host(tb_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                      uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle,
                      double* t, int32_t* tet_back) {
  return cast_host(m, n, o, d, start, status, cf, tet, visited, triangle, t, tet_back, false);
}

int tb_sctp_cast_rays_host(tb_mesh* m, int64_t n, const float* o, const float* d, const int32_t* start,
                           uint8_t* status, int32_t* cf, int32_t* tet, int32_t* visited, int32_t* triangle,
                           double* t, int32_t* tet_back) {
  return cast_host(m, n, o, d, start, status, cf, tet, visited, triangle, t, tet_back, true);
}

// Point location / shadow rays on host buffers: the same pooled slots, inputs
// memcpy'd into pinned mapped staging, the kernel reading and writing it over
// PCIe, one launch + one sync per chunk (renderers call these per tile).
int tb_locate_points_host(tb_mesh* m, int64_t n, const double* q, const int32_t* hints, int32_t* tet,
                          int32_t* visited) {
  if (int e = check_mesh(m)) return e;
  if (n < 0) return set_error(TB_E_ARG, "negative point count");
  if (n == 0) return TB_OK;
  if (!q || !hints || !tet || !visited) return set_error(TB_E_ARG, "NULL buffer");
  DeviceGuard g(m->device);
  SlotLease L;
  if (int e = slot_get(m->device, &L.p)) return e;
  const size_t C = (size_t)(n < kHostChunk ? n : kHostChunk);
  if (int e = L.p->host(al256(C * 24) + al256(C * 4) * 3)) return e;
  HostSlot& sl = *L.p;
  double* hq = reinterpret_cast<double*>(sl.h);
  int32_t* hh = reinterpret_cast<int32_t*>(sl.h + al256(C * 24));
  int32_t* ht = reinterpret_cast<int32_t*>(sl.h + al256(C * 24) + al256(C * 4));
  int32_t* hv = reinterpret_cast<int32_t*>(sl.h + al256(C * 24) + al256(C * 4) * 2);
  for (int64_t c0 = 0; c0 < n; c0 += (int64_t)C) {
    const size_t len = (size_t)((n - c0 < (int64_t)C) ? (n - c0) : (int64_t)C);
    memcpy(hq, q + 3 * c0, len * 24);
    memcpy(hh, hints + c0, len * 4);
    if (int e = tb_locate_points(m, (int64_t)len, sl.dev(hq), sl.dev(hh), sl.dev(ht), sl.dev(hv), sl.s)) return e;
    TB_CUDA(cudaStreamSynchronize(sl.s));
    memcpy(tet + c0, ht, len * 4);
    memcpy(visited + c0, hv, len * 4);
  }
  return TB_OK;
}

int tb_shadow_rays_host(tb_mesh* m, int64_t n, const double* p, const double* light, int light_stride,
                        const int32_t* p_tet, const int32_t* light_tet, int light_tet_stride, double eps,
                        uint8_t* occluded, int32_t* visited) {
  if (int e = check_mesh(m)) return e;
  if (n < 0) return set_error(TB_E_ARG, "negative ray count");
  if (n == 0) return TB_OK;
  if (!p || !light || !p_tet || !light_tet || !occluded || !visited) return set_error(TB_E_ARG, "NULL buffer");
  if ((light_stride != 0 && light_stride != 3) || (light_tet_stride != 0 && light_tet_stride != 1))
    return set_error(TB_E_ARG, "bad light strides %d/%d", light_stride, light_tet_stride);
  DeviceGuard g(m->device);
  SlotLease L;
  if (int e = slot_get(m->device, &L.p)) return e;
  const size_t C = (size_t)(n < kHostChunk ? n : kHostChunk);
  const size_t CL = light_stride ? C : 1, CLT = light_tet_stride ? C : 1;
  if (int e = L.p->host(al256(C * 24) + al256(CL * 24) + al256(C * 4) * 2 + al256(CLT * 4) + al256(C))) return e;
  HostSlot& sl = *L.p;
  char* b = sl.h;
  double* hp = reinterpret_cast<double*>(b);
  b += al256(C * 24);
  double* hl = reinterpret_cast<double*>(b);
  b += al256(CL * 24);
  int32_t* hpt = reinterpret_cast<int32_t*>(b);
  b += al256(C * 4);
  int32_t* hlt = reinterpret_cast<int32_t*>(b);
  b += al256(CLT * 4);
  int32_t* hv = reinterpret_cast<int32_t*>(b);
  b += al256(C * 4);
  uint8_t* ho = reinterpret_cast<uint8_t*>(b);
  if (!light_stride) memcpy(hl, light, 24);
  if (!light_tet_stride) memcpy(hlt, light_tet, 4);
  for (int64_t c0 = 0; c0 < n; c0 += (int64_t)C) {
    const size_t len = (size_t)((n - c0 < (int64_t)C) ? (n - c0) : (int64_t)C);
    memcpy(hp, p + 3 * c0, len * 24);
    memcpy(hpt, p_tet + c0, len * 4);
    if (light_stride) memcpy(hl, light + 3 * c0, len * 24);
    if (light_tet_stride) memcpy(hlt, light_tet + c0, len * 4);
    if (int e = tb_shadow_rays(m, (int64_t)len, sl.dev(hp), sl.dev(hl), light_stride, sl.dev(hpt), sl.dev(hlt),
                               light_tet_stride, eps, sl.dev(ho), sl.dev(hv), sl.s))
      return e;
    TB_CUDA(cudaStreamSynchronize(sl.s));
    memcpy(occluded + c0, ho, len);
    memcpy(visited + c0, hv, len * 4);
  }
  return TB_OK;
}

int tb_set_schedule(int mode, int steps_per_round) {
  if (mode > 7) return set_error(TB_E_ARG, "schedule mode %d not in 0..7", mode);
  if (steps_per_round == 0) return set_error(TB_E_ARG, "steps_per_round must be >= 1");
  if (mode >= 0) g_sched_mode.store(mode);
  if (steps_per_round > 0) g_round_steps.store(steps_per_round);
  return TB_OK;
}

int tb_get_schedule(int* mode, int* steps_per_round) {
  if (mode) *mode = sched_mode();
  if (steps_per_round) *steps_per_round = round_steps();
  return TB_OK;
}

int tb_host_alloc(size_t bytes, void** out) {
  if (!out) return set_error(TB_E_ARG, "out is NULL");
  TB_CUDA(cudaMallocHost(out, bytes ? bytes : 1));
  return TB_OK;
}

int tb_host_free(void* ptr) {
  if (ptr) TB_CUDA(cudaFreeHost(ptr));
  return TB_OK;
}

}  // extern "C"
