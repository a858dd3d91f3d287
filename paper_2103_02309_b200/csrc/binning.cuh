// binning.cuh -- direction binning for incoherent batches (schedule 6).
// Included by tetb200.cu inside its anonymous namespace (one translation
// unit): the kernels use tetb200.cu's error helpers only through the
// dispatch code that stays there.
#pragma once

// Direction binning for incoherent batches (schedule 6).  A stable counting
// sort of the ray indices by direction cell: the dominant axis and its sign
// pick a cube-map face, a 4 x 4 grid over the face's other two coordinates
// (divided by the dominant one) the cell -- 96 bins.  Rays of one cell cross
// the mesh in nearly parallel directions, so after binning a warp's rays
// (still in the caller's order inside their cell -- image order for
// secondaries spawned from a frame) share tets and L1 lines.  The walk then
// reads each ray through the permutation and stores its results at the
// original index (cast_kernel's kScatter + kGather path): outputs unchanged.
// r01 (config 4, 16.7 M diffuse secondaries; tools/bin_probe.py): walk
// 7.14 ms unbinned, 6.47 by octant (8 bins), 6.05 by face, 5.13 by 4 x 4
// cells per face, 5.47 by 8 x 8.  Any deterministic cell function is exact:
// only the order of the walks changes.
#ifndef TB_BIN_FACE
#define TB_BIN_FACE 4
#endif
constexpr int kBinFace = TB_BIN_FACE;                // cells per cube-face edge
constexpr int kBins = 6 * kBinFace * kBinFace;       // 96
static_assert(kBins <= 255, "bin ids are stored as bytes (kBins itself marks a dead lane)");
constexpr int kBinTile = 4096;                       // rays per binning block
constexpr int kBinThreads = 256;                     // 8 warps; one ray per thread per round

__device__ __forceinline__ int dir_bin(const float* __restrict__ d, int64_t r) {
  const float x = __ldg(d + 3 * r), y = __ldg(d + 3 * r + 1), z = __ldg(d + 3 * r + 2);
  const float ax = fabsf(x), ay = fabsf(y), az = fabsf(z);
  int a;
  float m, u, v;
  if (ax >= ay && ax >= az) {
    a = 0; m = x; u = y; v = z;
  } else if (ay >= az) {
    a = 1; m = y; u = x; v = z;
  } else {
    a = 2; m = z; u = x; v = y;
  }
  const float s = __fdividef(0.5f * kBinFace, fabsf(m));  // NaN / inf directions land in some cell: still exact
  const int cu = min(max((int)((u + fabsf(m)) * s), 0), kBinFace - 1);
  const int cv = min(max((int)((v + fabsf(m)) * s), 0), kBinFace - 1);
  return ((2 * a + (m < 0.f)) * kBinFace + cu) * kBinFace + cv;
}

// Lanes of the (full) warp holding the same bin id (< 128, kBins included):
// seven ballots over the id's bits instead of __match_any_sync, whose
// MATCH.ANY is slow enough to matter once a pass matches twice per ray (r02:
// config 4, a two-barrier scatter variant with two matches per ray +53 us per
// step with MATCH.ANY, +0 with ballots; see profiles/r02_experiments.md).
__device__ __forceinline__ unsigned bin_peers(int bin) {
#ifdef TB_BIN_MATCH_ANY
  return __match_any_sync(0xffffffffu, bin);
#else
  static_assert(kBins < 128, "bin ids (and the dead-lane id kBins) fit 7 bits");
  unsigned m = 0xffffffffu;
#pragma unroll
  for (int b = 0; b < 7; ++b) {
    const unsigned v = __ballot_sync(0xffffffffu, (bin >> b) & 1);
    m &= ((bin >> b) & 1) ? v : ~v;
  }
  return m;
#endif
}

// Histogram index of (bin b, tile t): global sort (S == 0) bin-major over
// all tiles; tile-local sort (S = tiles per segment) segment-major, then
// bin, then the tile within the segment -- so one exclusive scan per segment
// yields absolute positions inside the segment's own range of rays.
__device__ __forceinline__ int64_t hist_at(int b, int t, int n_tiles, int S) {
  return S ? ((int64_t)(t / S) * kBins + b) * S + (t % S) : (int64_t)b * n_tiles + t;
}

// hist[hist_at(b, tile)] = rays of bin b in the tile; bins[r] = ray r's bin
// (so the scatter pass reads 1 byte per ray instead of the direction).
__global__ void __launch_bounds__(kBinThreads) bin_count_kernel(const float* __restrict__ d, int64_t n,
                                                                int32_t* __restrict__ hist, int n_tiles, int S,
                                                                uint8_t* __restrict__ bins, int tile0 = 0) {
  __shared__ int cnt[kBins];
  for (int b = threadIdx.x; b < kBins; b += kBinThreads) cnt[b] = 0;
  __syncthreads();
  const int tile = tile0 + (int)blockIdx.x;  // tile0: first tile of a chunk of segments
  const int64_t base = (int64_t)tile * kBinTile;
  for (int i = threadIdx.x; i < kBinTile; i += kBinThreads) {  // warp-uniform trip count
    const int64_t r = base + i;
    const int bin = r < n ? dir_bin(d, r) : kBins;
    if (r < n) bins[r] = (uint8_t)bin;
    const unsigned peers = bin_peers(bin);  // one shared-memory atomic per bin per warp
    if (bin < kBins && (peers & ((1u << (threadIdx.x & 31)) - 1u)) == 0) atomicAdd(&cnt[bin], __popc(peers));
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kBins; b += kBinThreads) hist[hist_at(b, tile, n_tiles, S)] = cnt[b];
}

// Segmented mode: one block per segment, exclusive scan of its kBins * S
// counts in place, offset by the segment's first ray.
__global__ void __launch_bounds__(1024) bin_seg_scan_kernel(int32_t* __restrict__ hist, int S, int seg0 = 0) {
  __shared__ int32_t warp_sum[32];
  __shared__ int32_t carry;
  const int len = kBins * S;
  const int seg = seg0 + (int)blockIdx.x;
  int32_t* row = hist + (int64_t)seg * len;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int32_t seg_base = seg * S * kBinTile;
  for (int base = 0; base < len; base += 1024) {
    const int i = base + threadIdx.x;
    const int32_t v = i < len ? row[i] : 0;
    int32_t x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) warp_sum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int32_t w = warp_sum[lane];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, w, off);
        if (lane >= off) w += y;
      }
      warp_sum[lane] = w;
    }
    __syncthreads();
    if (i < len) row[i] = seg_base + carry + (warp ? warp_sum[warp - 1] : 0) + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sum[31];
    __syncthreads();
  }
}

// Global mode (TETB200_BIN_TILE=0): one block per bin, exclusive scan of the bin's per-tile counts in place
// (coalesced 1024-entry chunks, warp-shuffle scans, running carry); the
// bin's total goes to totals[bin].
__global__ void __launch_bounds__(1024) bin_scan_kernel(int32_t* __restrict__ hist, int n_tiles,
                                                        int32_t* __restrict__ totals) {
  __shared__ int32_t warp_sum[32];
  __shared__ int32_t carry;
  int32_t* row = hist + (int64_t)blockIdx.x * n_tiles;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n_tiles; base += 1024) {
    const int i = base + threadIdx.x;
    const int32_t v = i < n_tiles ? row[i] : 0;
    int32_t x = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) warp_sum[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int32_t w = warp_sum[lane];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, w, off);
        if (lane >= off) w += y;
      }
      warp_sum[lane] = w;
    }
    __syncthreads();
    if (i < n_tiles) row[i] = carry + (warp ? warp_sum[warp - 1] : 0) + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

// Stable scatter of the permutation: perm[start of bin b + offset of the
// tile within bin b + rank of ray r among the tile's bin-b rays, in caller
// order] = r.  Ranks within a warp come from bin_peers().
__global__ void __launch_bounds__(kBinThreads) bin_scatter_kernel(const uint8_t* __restrict__ bins, int64_t n,
                                                                  const int32_t* __restrict__ offs,
                                                                  const int32_t* __restrict__ totals, int n_tiles,
                                                                  int S, int32_t* __restrict__ perm, int tile0 = 0) {
  __shared__ int warp_cnt[kBinThreads / 32][kBins];
  const int tile = tile0 + (int)blockIdx.x;
  __shared__ int running[kBins];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {  // global sort: bin starts = exclusive prefix of the 96 totals
    int acc = 0;
    for (int b = 0; b < kBins; ++b) {
      running[b] = acc;
      acc += S ? 0 : totals[b];
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kBins; b += kBinThreads) running[b] += offs[hist_at(b, tile, n_tiles, S)];
  const int64_t base = (int64_t)tile * kBinTile;
  for (int round = 0; round < kBinTile / kBinThreads; ++round) {
    if (base + round * kBinThreads >= n) break;  // block-uniform
    for (int k = threadIdx.x; k < (kBinThreads / 32) * kBins; k += kBinThreads) (&warp_cnt[0][0])[k] = 0;
    __syncthreads();
    const int64_t r = base + round * kBinThreads + threadIdx.x;
    const bool live = r < n;
    const int bin = live ? (int)__ldg(bins + r) : kBins;
    const unsigned peers = bin_peers(bin);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (live && rank == 0) warp_cnt[warp][bin] = __popc(peers);
    __syncthreads();
    if (live) {
      int pos = running[bin] + rank;
      for (int w = 0; w < warp; ++w) pos += warp_cnt[w][bin];
      perm[pos] = (int32_t)r;
    }
    __syncthreads();
    for (int b = threadIdx.x; b < kBins; b += kBinThreads) {
      int add = 0;
      for (int w = 0; w < kBinThreads / 32; ++w) add += warp_cnt[w][b];
      running[b] += add;
    }
    __syncthreads();
  }
}

// Scatter target of a binned walk whose results go to a caller's index
// (multi-GPU frame assembly): widx[r] = oidx[perm[r]].
__global__ void compose_index_kernel(const int32_t* __restrict__ perm, const int64_t* __restrict__ oidx, int64_t n,
                                     int64_t* __restrict__ widx) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) widx[r] = __ldg(oidx + __ldg(perm + r));
}

// Sorting segments (r01, bench.py device values): binning sorts within
// segments of 262144 consecutive rays rather than over the whole batch.  A
// global permutation scatters every ray's gathered reads and result stores
// over the whole batch, and the partial sectors thrash L2 (ncu, config 4
// global: 9.4 GB DRAM read + 3.6 GB write per walk, L2 hit 25 %); within a
// segment those spans stay L2-resident while coherence is kept.  Config 4
// (16.7 M rays): global 3097 Mrays/s; segments of 64 K / 128 K / 256 K /
// 512 K / 1 M / 2 M rays 3335 / 3347 / 3359 / 3373 / 3367 / 3330.  Config-2
// secondaries (2.07 M): global 2265, 256 K segments 2398.  TETB200_BIN_TILE
// overrides (0 = one global sort).
int bin_tile() {
  static int env = -2;
  if (env == -2) {
    const char* v = getenv("TETB200_BIN_TILE");
    env = v ? (atoi(v) <= 0 ? 0 : ((atoi(v) + kBinTile - 1) / kBinTile) * kBinTile) : -1;  // whole tiles
  }
  return env >= 0 ? env : 262144;
}
