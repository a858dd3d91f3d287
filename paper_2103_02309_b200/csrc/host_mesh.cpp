// host_mesh.cpp -- native host-side mesh building for the traversal engine.
//
// The GPU walks the compact records; these routines build them on the host,
// once per scene, in plain C++ (no CUDA): Hilbert keys for the locality
// reorder, the sorted-slot side tables, the layout records and the id
// remapping of a reorder.  They reproduce the reference's numpy results bit
// for bit (tetmesh.py:299-371, :437-507; hilbert.py:14-73) -- the Python
// layer (tetmesh.py, hilbert.py) wraps them -- and run in one pass per
// array instead of numpy's many temporaries (50 M-tet scenes).
// Built with -ffp-contract=off: the quantization and centroid arithmetic
// must round exactly as numpy's elementwise float64 operations do.
#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/tetb200.h"

namespace {

constexpr uint32_t kConstrainedBit = 0x80000000u;
constexpr uint32_t kBoundaryRef = 0x7FFFFFFFu;

// Skilling, "Programming the Hilbert curve" (AIP Conf. Proc. 707, 2004):
// AxesToTranspose on one cell, then the transposed bits interleaved with
// axis 0 most significant.
uint64_t hilbert_key(uint32_t x0, uint32_t x1, uint32_t x2, int order) {
  uint32_t x[3] = {x0, x1, x2};
  const uint32_t top = 1u << (order - 1);
  for (uint32_t q = top; q > 1; q >>= 1) {
    const uint32_t low = q - 1;
    for (int i = 0; i < 3; ++i) {
      if (x[i] & q) {
        x[0] ^= low;  // invert the low bits of axis 0
      } else {
        const uint32_t swap = (x[0] ^ x[i]) & low;  // exchange the low bits
        x[0] ^= swap;
        x[i] ^= swap;
      }
    }
  }
  x[1] ^= x[0];
  x[2] ^= x[1];
  uint32_t flip = 0;
  for (uint32_t q = top; q > 1; q >>= 1)
    if (x[2] & q) flip ^= q - 1;
  for (int i = 0; i < 3; ++i) x[i] ^= flip;
  uint64_t key = 0;
  for (int b = order - 1; b >= 0; --b)
    key = (key << 3) | (uint64_t)((x[0] >> b) & 1u) << 2 | (uint64_t)((x[1] >> b) & 1u) << 1 |
          (uint64_t)((x[2] >> b) & 1u);
  return key;
}

bool plain_ref(uint32_t r) { return (r & kConstrainedBit) == 0 && r != kBoundaryRef; }

}  // namespace

extern "C" {

int tb_hilbert_keys(const int64_t* cells, int64_t n, int order, uint64_t* keys) {
  if (order < 1 || order > 20) return TB_E_ARG;
  if (n < 0 || (n > 0 && (!cells || !keys))) return TB_E_ARG;
  const int64_t lim = int64_t(1) << order;
  for (int64_t i = 0; i < 3 * n; ++i)
    if (cells[i] < 0 || cells[i] >= lim) return TB_E_ARG;
  for (int64_t i = 0; i < n; ++i)
    keys[i] = hilbert_key((uint32_t)cells[3 * i], (uint32_t)cells[3 * i + 1], (uint32_t)cells[3 * i + 2], order);
  return TB_OK;
}

int tb_hilbert_quantize(const double* pts, int64_t n, const double* lo, const double* hi, int order,
                        int64_t* cells) {
  if (order < 1 || order > 20 || n < 0 || (n > 0 && (!pts || !cells)) || !lo || !hi) return TB_E_ARG;
  const double scale = (double)((int64_t(1) << order) - 1);
  const int64_t top = (int64_t(1) << order) - 1;
  double extent[3];
  for (int k = 0; k < 3; ++k) extent[k] = hi[k] > lo[k] ? hi[k] - lo[k] : 1.0;
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < 3; ++k) {
      const double v = std::floor(((pts[3 * i + k] - lo[k]) / extent[k]) * scale);
      int64_t c;
      if (std::isnan(v))
        c = INT64_MIN;  // numpy's float64 -> int64 cast of NaN, then clipped to 0 below
      else if (v >= 9.2e18)
        c = INT64_MAX;
      else if (v <= -9.2e18)
        c = INT64_MIN;
      else
        c = (int64_t)v;
      cells[3 * i + k] = c < 0 ? 0 : (c > top ? top : c);
    }
  }
  return TB_OK;
}

int tb_tet_centroids(const double* pts, int64_t n_points, const int32_t* quads, int64_t n, double* out) {
  if (n < 0 || (n > 0 && (!pts || !quads || !out))) return TB_E_ARG;
  for (int64_t t = 0; t < n; ++t) {
    const int32_t* q = quads + 4 * t;
    for (int k = 0; k < 4; ++k)
      if (q[k] < 0 || q[k] >= n_points) return TB_E_ARG;
    for (int c = 0; c < 3; ++c) {
      // numpy's mean over the 4 rows: sequential sum, then one division
      double s = pts[3 * (int64_t)q[0] + c];
      s += pts[3 * (int64_t)q[1] + c];
      s += pts[3 * (int64_t)q[2] + c];
      s += pts[3 * (int64_t)q[3] + c];
      out[3 * t + c] = s / 4.0;
    }
  }
  return TB_OK;
}

int tb_build_side_tables(int64_t n, const int32_t* verts, const uint32_t* refs, const int64_t* row_of,
                         const int64_t* vert_map, int64_t n_vert_map, const int64_t* tet_map, int64_t n_tet_map,
                         int32_t* sv_out, uint32_t* sn_out) {
  if (n < 0 || (n > 0 && (!verts || !refs || !sv_out || !sn_out))) return TB_E_ARG;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t src = row_of ? row_of[i] : i;
    int64_t v[4];
    uint32_t r[4];
    for (int k = 0; k < 4; ++k) {
      const int32_t vv = verts[4 * src + k];
      if (vert_map) {
        if (vv < 0 || vv >= n_vert_map) return TB_E_ARG;
        v[k] = vert_map[vv];
      } else {
        v[k] = vv;
      }
      uint32_t rr = refs[4 * src + k];
      if (tet_map && plain_ref(rr)) {
        if ((int64_t)rr >= n_tet_map) return TB_E_ARG;
        rr = (uint32_t)tet_map[rr];
      }
      r[k] = rr;
    }
    // stable insertion sort of the 4 slots by vertex id, refs alongside
    for (int a = 1; a < 4; ++a) {
      const int64_t kv = v[a];
      const uint32_t kr = r[a];
      int b = a - 1;
      while (b >= 0 && v[b] > kv) {
        v[b + 1] = v[b];
        r[b + 1] = r[b];
        --b;
      }
      v[b + 1] = kv;
      r[b + 1] = kr;
    }
    for (int k = 0; k < 4; ++k) {
      sv_out[4 * i + k] = (int32_t)v[k];
      sn_out[4 * i + k] = r[k];
    }
  }
  return TB_OK;
}

int tb_pack_records(int layout, int64_t n, const int32_t* sv, const uint32_t* sn, uint32_t* words) {
  if (layout != 32 && layout != 20 && layout != 16) return TB_E_LAYOUT;
  if (n < 0 || (n > 0 && (!sv || !sn || !words))) return TB_E_ARG;
  const int w = layout / 4;
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t* v = reinterpret_cast<const uint32_t*>(sv + 4 * i);
    const uint32_t* r = sn + 4 * i;
    uint32_t* out = words + w * i;
    const uint32_t x = v[0] ^ v[1] ^ v[2] ^ v[3];
    if (layout == 32) {
      out[0] = v[0]; out[1] = v[1]; out[2] = v[2]; out[3] = x;
      out[4] = r[0]; out[5] = r[1]; out[6] = r[2]; out[7] = r[3];
    } else if (layout == 20) {
      out[0] = x;
      out[1] = r[0]; out[2] = r[1]; out[3] = r[2]; out[4] = r[3];
    } else {
      out[0] = x;
      out[1] = r[0] ^ r[3]; out[2] = r[1] ^ r[3]; out[3] = r[2] ^ r[3];
    }
  }
  return TB_OK;
}

}  // extern "C"
