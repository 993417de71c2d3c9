// Forward kernels of rasterize_meshes on sm_100a.
//
//   K0 k_face_setup   prepare_faces (MR:100-131): cull + EXACT integer pixel-range bbox per face
//   K1 k_bin_faces    pass 1 (MR:237-264): coarse binning, warp-aggregated atomics into fixed-capacity bins
//   K2 k_fine         pass 2 (MR:265-282) + test_pixel_face/PixelHeap/emit_pixel (MR:133-197): one CTA per
//                     (mesh, bin); faces staged in shared memory; per-pixel top-K on the (z, id) key
//
// The binned and naive (bin_size == 0, MR:214-232) paths share K2; they differ only in where a CTA takes its
// candidate faces from (its bin list vs. the whole mesh). A bin whose list overflowed max_faces_per_bin is
// rasterized from the whole mesh as well (spill path), so results never depend on the capacity.
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cstdint>
#include <algorithm>
#include <type_traits>
#include <utility>
#include <vector>

#include "raster_kernels.cuh"
#include "raster_math.cuh"

#ifndef DR_STATS
#define DR_STATS 0
#endif
#if DR_STATS
// debug build only (tools/fine_stats.py): work counters of K2
__device__ unsigned long long g_stats[12];
#define STAT_ADD(i, v) do { const unsigned long long sv_ = (unsigned long long)(v); if ((threadIdx.x & 31) == 0) atomicAdd(&g_stats[i], sv_); } while (0)
#else
#define STAT_ADD(i, v) do { } while (0)
#endif

namespace drb {

// ------------------------------------------------------------------------------------------------
// exact integer pixel ranges

// smallest j in [0, W] with pixel_x(W, j) >= L
__device__ __forceinline__ int first_col_ge(double L, int W) {
  double e = ((L + 1.0) * W - 1.0) * 0.5;
  int j = !(e > 0.0) ? 0 : (e >= (double)W ? W : (int)ceil(e));
  while (j > 0 && pixel_x(W, j - 1) >= L) --j;
  while (j < W && pixel_x(W, j) < L) ++j;
  return j;
}
// largest j in [-1, W-1] with pixel_x(W, j) <= U
__device__ __forceinline__ int last_col_le(double U, int W) {
  double e = ((U + 1.0) * W - 1.0) * 0.5;
  int j = !(e < (double)(W - 1)) ? W - 1 : (e < 0.0 ? -1 : (int)floor(e));
  while (j < W - 1 && pixel_x(W, j + 1) <= U) ++j;
  while (j >= 0 && pixel_x(W, j) > U) --j;
  return j;
}
// smallest i in [0, H] with pixel_y(H, i) <= U   (pixel_y decreases with i)
__device__ __forceinline__ int first_row_le(double U, int H) {
  double e = ((1.0 - U) * H - 1.0) * 0.5;
  int i = !(e > 0.0) ? 0 : (e >= (double)H ? H : (int)ceil(e));
  while (i > 0 && pixel_y(H, i - 1) <= U) --i;
  while (i < H && pixel_y(H, i) > U) ++i;
  return i;
}
// largest i in [-1, H-1] with pixel_y(H, i) >= L
__device__ __forceinline__ int last_row_ge(double L, int H) {
  double e = ((1.0 - L) * H - 1.0) * 0.5;
  int i = !(e < (double)(H - 1)) ? H - 1 : (e < 0.0 ? -1 : (int)floor(e));
  while (i < H - 1 && pixel_y(H, i + 1) >= L) ++i;
  while (i >= 0 && pixel_y(H, i) < L) --i;
  return i;
}

// ------------------------------------------------------------------------------------------------
// K0: face setup

__device__ __forceinline__ void face_setup_one(const double* __restrict__ fv, int64_t f, int H, int W, double inflate,
                                               double znear, int clip_nonpositive_z, int cull_backfaces,
                                               int4* __restrict__ ibbox, float* __restrict__ zkey) {
  const double* p = fv + 9 * f;
  double v[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) v[k] = __ldg(p + k);
  int4 out = make_int4(1, 0, 1, 0);  // empty
  float key = __int_as_float(0x7f800000);  // +inf: culled faces are never candidates
  bool keep = true;
#pragma unroll
  for (int k = 0; k < 9; ++k) keep = keep && isfinite(v[k]);  // builder-defined: non-finite faces are culled
  if (keep) {
    double z0 = v[2], z1 = v[5], z2 = v[8];
    if (clip_nonpositive_z && (z0 <= 0 || z1 <= 0 || z2 <= 0)) keep = false;  // MR:112
    if (z0 < znear && z1 < znear && z2 < znear) keep = false;                 // MR:113
    V2 a{v[0], v[1]}, b{v[3], v[4]}, c{v[6], v[7]};
    double area = signed_area2(a, b, c);
    if (fabs(area) < kDegenerateArea) keep = false;  // MR:114
    if (cull_backfaces && area > 0) keep = false;    // builder-defined
    if (keep) {
      // MR:123-126 (std::min({..}) / std::max({..}))
      double mnx = a.x, mny = a.y, mxx = a.x, mxy = a.y;
      mnx = b.x < mnx ? b.x : mnx;
      mnx = c.x < mnx ? c.x : mnx;
      mny = b.y < mny ? b.y : mny;
      mny = c.y < mny ? c.y : mny;
      mxx = mxx < b.x ? b.x : mxx;
      mxx = mxx < c.x ? c.x : mxx;
      mxy = mxy < b.y ? b.y : mxy;
      mxy = mxy < c.y ? c.y : mxy;
      double bx0 = mnx - inflate, by0 = mny - inflate, bx1 = mxx + inflate, by1 = mxy + inflate;
      // pixel (i,j) passes MR:168-169 iff j in [j0,j1] and i in [i0,i1]
      int j0 = first_col_ge(bx0, W), j1 = last_col_le(bx1, W);
      int i0 = first_row_le(by1, H), i1 = last_row_ge(by0, H);
      if (j0 <= j1 && i0 <= i1) out = make_int4(i0, i1, j0, j1);
      // Depth key: with clamped barycentrics (MR:172) every candidate z = RN(RN(w0 z0) + RN(w1 z1)) + RN(w2 z2)
      // (MR:173) has w_i >= 0 and |sum w_i - 1| <= 4 ulp, so z >= zmin - 8 ulp(|zmin|) - (underflow, 3 * 2^-1074);
      // the key subtracts a far larger margin and rounds down to fp32, so it is a strict lower bound.
      double zmin = z0 < z1 ? z0 : z1;
      zmin = z2 < zmin ? z2 : zmin;
      key = __double2float_rd(zmin - fabs(zmin) * 1e-9 - 1e-300);
    }
  }
  ibbox[f] = out;
  if (zkey) zkey[f] = key;
}

// Only the batch's own faces are set up (a mesh-sharded rank passes its meshes' ranges of the whole packed batch):
// k_face_setup_range covers one merged interval of the ranges; k_face_setup (grid (x, N), blockIdx.y = mesh) is
// used when the ranges fall into many intervals. Overlapping ranges write identical values.
__global__ void __launch_bounds__(256) k_face_setup_range(const double* __restrict__ fv, int64_t f_lo, int64_t f_hi,
                                                          int H, int W, double inflate, double znear,
                                                          int clip_nonpositive_z, int cull_backfaces,
                                                          int4* __restrict__ ibbox, float* __restrict__ zkey) {
  const int64_t f = f_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f < f_hi) face_setup_one(fv, f, H, W, inflate, znear, clip_nonpositive_z, cull_backfaces, ibbox, zkey);
}

__global__ void __launch_bounds__(256) k_face_setup(const double* __restrict__ fv, const int64_t* __restrict__ first,
                                                    const int64_t* __restrict__ num, int H, int W, double inflate,
                                                    double znear, int clip_nonpositive_z, int cull_backfaces,
                                                    int4* __restrict__ ibbox, float* __restrict__ zkey) {
  const int64_t nf = num[blockIdx.y], f0 = first[blockIdx.y];
  for (int64_t lf = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; lf < nf; lf += (int64_t)gridDim.x * blockDim.x)
    face_setup_one(fv, f0 + lf, H, W, inflate, znear, clip_nonpositive_z, cull_backfaces, ibbox, zkey);
}

// ------------------------------------------------------------------------------------------------
// K1: coarse binning (pass 1, MR:237-264) into EXACT-size lists: count -> exclusive scan -> fill.
// Each warp walks 32 consecutive faces of one mesh; the bins a face touches form a rectangle of the bin grid.
// Lanes that target the same bin in the same round are grouped with __match_any_sync and reserve their slots
// with ONE atomicAdd (leader), so adjacent faces of a mesh (which mostly share bins) cost one global atomic per
// (warp, bin). Order inside a bin is irrelevant: the K smallest under the strict total order (z, id) do not
// depend on it (MR:138-140). The lists live in one pool sized from F (workspace is planned before the counts
// are known); a bin that does not fit the pool, or exceeds the caller's max_faces_per_bin, takes the spill
// path in K2 (its micro-tiles scan the whole mesh), so results never depend on either capacity.

// A bin entry carries everything K2 needs to decide whether a face touches a micro-tile (one coalesced 16-byte
// load per entry instead of a dependent ibbox gather): {face id, zkey bits, i0 | i1 << 16, j0 | j1 << 16}.
// Pixel indices fit 16 bits (image side <= 32768, checked by make_plan).
__device__ __forceinline__ int4 make_bin_entry(int32_t fid, float key, int4 ib) {
  return make_int4(fid, __float_as_int(key), (ib.x & 0xffff) | (ib.y << 16), (ib.z & 0xffff) | (ib.w << 16));
}
__device__ __forceinline__ int4 entry_ibbox(int4 e) {
  return make_int4(e.z & 0xffff, (int)((unsigned)e.z >> 16), e.w & 0xffff, (int)((unsigned)e.w >> 16));
}

template <bool kFill>
__global__ void __launch_bounds__(256) k_bin_faces(const int4* __restrict__ ibbox, const int64_t* __restrict__ first,
                                                   const int64_t* __restrict__ num, int bs, int nbx, int nby,
                                                   int* __restrict__ counts, const int64_t* __restrict__ off,
                                                   int* __restrict__ cursor, int64_t pool,
                                                   const float* __restrict__ zkey, int4* __restrict__ entries) {
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int64_t nf = num[b], f0 = first[b];
  const int nbins = nbx * nby;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t bin0 = (int64_t)b * nbins;
  for (int64_t base = warp * 32; base < nf; base += nwarps * 32) {
    int64_t lf = base + lane;
    int4 ib = lf < nf ? ibbox[f0 + lf] : make_int4(1, 0, 1, 0);
    int bi0 = 0, bj0 = 0, bw = 0, n = 0;
    if (ib.x <= ib.y) {
      bi0 = ib.x / bs;
      bj0 = ib.z / bs;
      bw = ib.w / bs - bj0 + 1;
      n = (ib.y / bs - bi0 + 1) * bw;
    }
    for (int k = 0; __any_sync(0xffffffffu, k < n); ++k) {
      bool active = k < n;
      int key = active ? (bi0 + k / bw) * nbx + (bj0 + k % bw) : -1 - lane;
      unsigned peers = __match_any_sync(0xffffffffu, key);
      int leader = __ffs(peers) - 1;
      int rank = __popc(peers & ((1u << lane) - 1u));
      if constexpr (!kFill) {
        if (active && lane == leader) atomicAdd(counts + bin0 + key, __popc(peers));
      } else {
        int64_t pos = -1;
        if (active && lane == leader) {
          const int64_t o = off[bin0 + key];
          if (o + counts[bin0 + key] <= pool) pos = o + atomicAdd(cursor + bin0 + key, __popc(peers));
        }
        pos = __shfl_sync(0xffffffffu, pos, leader);
        if (active && pos >= 0) entries[pos + rank] = make_bin_entry((int32_t)(f0 + lf), zkey ? zkey[f0 + lf] : 0.f, ib);
      }
    }
  }
}

// Shared-memory histogram form of the same two passes, used for point clouds (at most kBinSmemMax bins per
// cloud): a CTA takes kBinChunk consecutive items of one cloud, counts their (item, bin) pairs with shared-memory
// atomics, then issues ONE global atomic per non-empty bin (count pass: the count; fill pass: the reservation of
// the CTA's run of the bin's list, after which each pair takes its place with a shared-memory atomic). Per-pair
// global atomics were the binning's cost wherever neighbouring items do not share bins (random point clouds: the
// warp-level __match_any_sync aggregation of k_bin_faces finds no peers there): points binning 0.44 -> 0.10 ms.
// Meshes keep k_bin_faces: their faces come in spatial order (the warp aggregation works), and the changed entry
// order within a depth bucket cost K2 up to +3 % (C5) against 0.05 ms saved in binning (C4).
constexpr int kBinSmemMax = 2048;
constexpr int kBinChunk = 2048;

template <bool kFill>
__global__ void __launch_bounds__(256) k_bin_faces_smem(const int4* __restrict__ ibbox,
                                                        const int64_t* __restrict__ first,
                                                        const int64_t* __restrict__ num, int bs, int nbx, int nby,
                                                        int* __restrict__ counts, const int64_t* __restrict__ off,
                                                        int* __restrict__ cursor, int64_t pool,
                                                        const float* __restrict__ zkey, int4* __restrict__ entries) {
  __shared__ int hist[kBinSmemMax];
  __shared__ long long runs[kFill ? kBinSmemMax : 1];  // fill: start of this CTA's run in each bin's list (-1: none)
  const int b = blockIdx.y;
  const int64_t nf = num[b], f0 = first[b];
  const int64_t c0 = (int64_t)blockIdx.x * kBinChunk;
  if (c0 >= nf) return;  // (uniform per CTA)
  const int64_t c1 = nf < c0 + kBinChunk ? nf : c0 + kBinChunk;
  const int nbins = nbx * nby;
  const int64_t bin0 = (int64_t)b * nbins;
  for (int t = threadIdx.x; t < nbins; t += blockDim.x) hist[t] = 0;
  __syncthreads();
  for (int64_t lf = c0 + threadIdx.x; lf < c1; lf += blockDim.x) {
    const int4 ib = ibbox[f0 + lf];
    if (ib.x > ib.y) continue;
    const int bi1 = ib.y / bs, bj0 = ib.z / bs, bj1 = ib.w / bs;
    for (int bi = ib.x / bs; bi <= bi1; ++bi)
      for (int bj = bj0; bj <= bj1; ++bj) atomicAdd(&hist[bi * nbx + bj], 1);
  }
  __syncthreads();
  if constexpr (!kFill) {
    for (int t = threadIdx.x; t < nbins; t += blockDim.x) {
      const int c = hist[t];
      if (c) atomicAdd(counts + bin0 + t, c);
    }
  } else {
    for (int t = threadIdx.x; t < nbins; t += blockDim.x) {
      const int c = hist[t];
      long long r = -1;
      if (c) {
        const int64_t o = off[bin0 + t];
        if (o + counts[bin0 + t] <= pool) r = o + atomicAdd(cursor + bin0 + t, c);  // the whole bin fits the pool
      }
      runs[t] = r;
      hist[t] = 0;
    }
    __syncthreads();
    for (int64_t lf = c0 + threadIdx.x; lf < c1; lf += blockDim.x) {
      const int4 ib = ibbox[f0 + lf];
      if (ib.x > ib.y) continue;
      const int4 e = make_bin_entry((int32_t)(f0 + lf), zkey ? zkey[f0 + lf] : 0.f, ib);
      const int bi1 = ib.y / bs, bj0 = ib.z / bs, bj1 = ib.w / bs;
      for (int bi = ib.x / bs; bi <= bi1; ++bi)
        for (int bj = bj0; bj <= bj1; ++bj) {
          const int t = bi * nbx + bj;
          const long long r = runs[t];
          if (r >= 0) entries[r + atomicAdd(&hist[t], 1)] = e;
        }
    }
  }
}

// exclusive scan of the bin counts without extra workspace: (1) every CTA scans a segment of kScanSeg counts
// locally (exclusive, into off); (2) every CTA adds the sum of all earlier segments to its elements except the
// segment's last one — it reads those sums back as off[last] + counts[last] of each earlier segment, values no
// block of this pass modifies; (3) one thread walks the segments and fixes their last elements in order.
constexpr int kScanThreads = 1024;
constexpr int kScanPer = 4;
constexpr int kScanSeg = kScanThreads * kScanPer;

__global__ void __launch_bounds__(kScanThreads) k_scan_local(const int* __restrict__ counts, int64_t n,
                                                             int64_t* __restrict__ off) {
  __shared__ int64_t warp_tot[kScanThreads / 32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t base = (int64_t)blockIdx.x * kScanSeg + (int64_t)t * kScanPer;
  int c[kScanPer];
  int64_t sum = 0;
#pragma unroll
  for (int u = 0; u < kScanPer; ++u) {
    c[u] = base + u < n ? counts[base + u] : 0;
    sum += c[u];
  }
  int64_t incl = sum;  // warp inclusive scan of the per-thread sums
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    int64_t x = warp_tot[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int64_t v = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += v;
    }
    warp_tot[lane] = x;
  }
  __syncthreads();
  int64_t run = incl - sum + (w > 0 ? warp_tot[w - 1] : 0);
#pragma unroll
  for (int u = 0; u < kScanPer; ++u) {
    if (base + u < n) off[base + u] = run;
    run += c[u];
  }
}

__global__ void __launch_bounds__(256) k_scan_fix(const int* __restrict__ counts, int64_t n,
                                                  int64_t* __restrict__ off) {
  __shared__ int64_t red[256];
  const int seg = blockIdx.x;
  if (seg == 0) return;
  int64_t s = 0;
  for (int q = threadIdx.x; q < seg; q += 256) {  // totals of the earlier segments
    const int64_t last = (int64_t)(q + 1) * kScanSeg - 1;
    s += off[last] + counts[last];
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int d = 128; d > 0; d >>= 1) {
    if (threadIdx.x < d) red[threadIdx.x] += red[threadIdx.x + d];
    __syncthreads();
  }
  const int64_t prefix = red[0];
  const int64_t lo = (int64_t)seg * kScanSeg, hi = min(n, lo + kScanSeg - 1);  // the last element: k_scan_last
  for (int64_t i = lo + threadIdx.x; i < hi; i += 256) off[i] += prefix;
}

__global__ void k_scan_last(const int* __restrict__ counts, int64_t n, int64_t* __restrict__ off) {
  int64_t prefix = 0;
  for (int64_t last = kScanSeg - 1; last < n; last += kScanSeg) {
    const int64_t tot = off[last] + counts[last];  // still the segment-local value
    off[last] += prefix;
    prefix += tot;
  }
}

// ------------------------------------------------------------------------------------------------
// K1b: depth-order each bin list so K2 meets the nearest faces first: its K-th-depth cull then rejects most of
// the list before the exact test. One CTA per bin: keys to shared memory, the bin's depth range, a 1024-bucket
// counting sort (histogram, scan, scatter back in place). Measured against the exact bitonic sort of (key, id) it
// replaced: C4 sort 0.39 -> 0.18 ms with the same K2 time, C3 0.24 -> 0.04 ms; C5 (K=50) K2 +1 %. The
// selection K2 makes is order-independent (strict total order, MR:138-140): the order changes only its work.

constexpr int kSortThreads = 256;
constexpr int kSortBuckets = kSortThreads * kSortBpt;
static_assert(kSortBuckets == kSortBucketsH, "bucket count shared with the point fine stage");

// Short bins (<= kWarpSortMax entries, most of them): one WARP per bin, no CTA barrier. The warp reads the bin's
// (id, key) pairs into registers (8 per lane), reduces the depth range with shuffles, counts kWarpSortBuckets
// linear buckets in its own shared-memory histogram, scans it (8 buckets per lane), scatters the re-packed entries
// back in place. Bucket map (lo, scale) as for the CTA sort, so the point stage's exit bound stays valid.
constexpr int kWarpSortMax = 256;
constexpr int kWarpSortPer = kWarpSortMax / 32;
constexpr int kWarpSortBuckets = 256;
constexpr int kWarpSortWarps = 8;
__global__ void __launch_bounds__(kWarpSortWarps * 32) k_sort_bins_warp(const int* __restrict__ counts,
                                                                     const int64_t* __restrict__ off,
                                                                     int4* __restrict__ entries,
                                                                     const int4* __restrict__ ibbox,
                                                                     int64_t nbins_total, int64_t pool, int cap,
                                                                     float2* __restrict__ brange) {
  __shared__ unsigned hist_all[kWarpSortWarps][kWarpSortBuckets];
  const int lane = threadIdx.x & 31;
  unsigned* hist = hist_all[threadIdx.x >> 5];
  const int64_t nwarps = (int64_t)gridDim.x * kWarpSortWarps;
  // warp w owns bins w, w + nwarps, ...; 32 of its counts are read at once and the in-range ones kept
  for (int64_t k0 = (int64_t)blockIdx.x * kWarpSortWarps + (threadIdx.x >> 5); k0 < nbins_total; k0 += 32 * nwarps) {
    const int64_t mybin = k0 + (int64_t)lane * nwarps;
    bool in = false;
    if (mybin < nbins_total) {
      const int c = counts[mybin];
      in = c > 0 && c <= kWarpSortMax && bin_is_sorted(off[mybin], c, pool, cap);
    }
    unsigned todo = __ballot_sync(0xffffffffu, in);
    while (todo) {
      const int64_t bin = k0 + (int64_t)(__ffs(todo) - 1) * nwarps;
      todo &= todo - 1;
      const int c = counts[bin];
      int4* L = entries + off[bin];
      int fid[kWarpSortPer];
      float key[kWarpSortPer];
      float lo = __int_as_float(0x7f800000), hi = -lo;
#pragma unroll
      for (int t = 0; t < kWarpSortPer; ++t) {
        const int i = t * 32 + lane;
        fid[t] = -1;
        key[t] = 0.f;
        if (i < c) {
          const int2 fk = *reinterpret_cast<const int2*>(L + i);  // {face id, zkey bits}
          fid[t] = fk.x;
          key[t] = __int_as_float(fk.y);
          lo = fminf(lo, key[t]);
          hi = fmaxf(hi, key[t]);
        }
      }
      for (int d = 16; d; d >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, d));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, d));
      }
      const float scale = hi > lo ? (float)kWarpSortBuckets * 0.99999f / (hi - lo) : 0.f;
      if (brange && lane == 0) brange[bin] = make_float2(lo, scale);  // the bucket map (sort_bucket stays < 256)
#pragma unroll
      for (int j = 0; j < kWarpSortBuckets / 32; ++j) hist[lane * (kWarpSortBuckets / 32) + j] = 0;
      __syncwarp();
      int bk[kWarpSortPer];
#pragma unroll
      for (int t = 0; t < kWarpSortPer; ++t) {
        bk[t] = min(kWarpSortBuckets - 1, sort_bucket(key[t], lo, scale));
        if (fid[t] >= 0) atomicAdd(&hist[bk[t]], 1u);
      }
      __syncwarp();
      {  // exclusive scan: lane l holds buckets [8 l, 8 l + 8)
        constexpr int PB = kWarpSortBuckets / 32;
        unsigned v[PB], tot = 0;
#pragma unroll
        for (int j = 0; j < PB; ++j) { v[j] = hist[lane * PB + j]; tot += v[j]; }
        unsigned x = tot;
        for (int d = 1; d < 32; d <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, x, d);
          if (lane >= d) x += y;
        }
        unsigned base = x - tot;
#pragma unroll
        for (int j = 0; j < PB; ++j) { hist[lane * PB + j] = base; base += v[j]; }
      }
      __syncwarp();
#pragma unroll
      for (int t = 0; t < kWarpSortPer; ++t) {
        if (fid[t] >= 0) {
          const int pos = (int)atomicAdd(&hist[bk[t]], 1u);
          L[pos] = make_bin_entry(fid[t], key[t], __ldg(ibbox + fid[t]));
        }
      }
      __syncwarp();
    }
  }
}

// MAXN = shared-memory capacity in entries; bins with (MINN, MAXN] entries are sorted by this instantiation
template <int MAXN, int MINN, bool kDyn>
__global__ void __launch_bounds__(kSortThreads) k_sort_bins(const int* __restrict__ counts,
                                                            const int64_t* __restrict__ off,
                                                            int4* __restrict__ entries,
                                                            const int4* __restrict__ ibbox, int64_t nbins_total,
                                                            int64_t pool, int cap, float2* __restrict__ brange) {
  __shared__ unsigned long long s_static[kDyn ? 1 : MAXN];
  __shared__ unsigned sel_mask;
  __shared__ unsigned hist[kSortBuckets];
  __shared__ unsigned wsum[kSortThreads / 32];
  __shared__ float red_lo[kSortThreads / 32], red_hi[kSortThreads / 32];
  extern __shared__ unsigned long long s_dyn[];
  unsigned long long* s = kDyn ? s_dyn : s_static;
  // CTA b owns bins b, b + grid, b + 2 grid, ... (round robin: adjacent large bins land on different CTAs);
  // warp 0 reads 32 of its counts at once and keeps the ones in this instantiation's size range, so a CTA does
  // not walk the (mostly out-of-range) bins one by one
  const int64_t stride = gridDim.x;
  for (int64_t k0 = 0; (int64_t)blockIdx.x + k0 * stride < nbins_total; k0 += 32) {
    if (threadIdx.x < 32) {
      const int64_t bin = (int64_t)blockIdx.x + (k0 + threadIdx.x) * stride;
      bool in = false;
      if (bin < nbins_total) {
        const int c = counts[bin];
        in = c > MINN && c <= MAXN && bin_is_sorted(off[bin], c, pool, cap);  // spill bins are never read as lists
      }
      const unsigned m = __ballot_sync(0xffffffffu, in);
      if (threadIdx.x == 0) sel_mask = m;
    }
    __syncthreads();
    unsigned todo = sel_mask;
    __syncthreads();
  while (todo) {
    const int64_t bin = (int64_t)blockIdx.x + (k0 + __ffs(todo) - 1) * stride;
    todo &= todo - 1;
    const int c = counts[bin];
    const int64_t o = off[bin];
    int4* L = entries + o;
    // depth-bucket order: keys in smem, bin depth range, 256 linear buckets (histogram, scan, scatter). Order
    // inside a bucket is arbitrary (K2 is order-independent); one pass of O(c) instead of O(c log^2 c).
    float lo = __int_as_float(0x7f800000), hi = -lo;
    for (int i = threadIdx.x; i < c; i += kSortThreads) {
      const int2 fk = *reinterpret_cast<const int2*>(L + i);  // {face id, zkey bits}
      s[i] = ((unsigned long long)(uint32_t)fk.y << 32) | (uint32_t)fk.x;
      const float z = __int_as_float(fk.y);
      lo = fminf(lo, z);
      hi = fmaxf(hi, z);
    }
    for (int d = 16; d; d >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, d));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, d));
    }
    const int wid = threadIdx.x >> 5, ln = threadIdx.x & 31;
    if (ln == 0) { red_lo[wid] = lo; red_hi[wid] = hi; }
#pragma unroll
    for (int j = 0; j < kSortBpt; ++j) hist[threadIdx.x * kSortBpt + j] = 0;
    __syncthreads();
    lo = red_lo[0]; hi = red_hi[0];
#pragma unroll
    for (int w = 1; w < kSortThreads / 32; ++w) { lo = fminf(lo, red_lo[w]); hi = fmaxf(hi, red_hi[w]); }
    const float scale = sort_bucket_scale(lo, hi);
    if (brange && threadIdx.x == 0) brange[bin] = make_float2(lo, scale);  // the bucket map, for an exit bound
    auto bucket = [&](unsigned long long e) { return sort_bucket(__uint_as_float((uint32_t)(e >> 32)), lo, scale); };
    for (int i = threadIdx.x; i < c; i += kSortThreads) atomicAdd(&hist[bucket(s[i])], 1u);
    __syncthreads();
    {  // exclusive scan of the bucket counts (kSortBpt consecutive ones per thread)
      unsigned v[kSortBpt], tot = 0;
#pragma unroll
      for (int j = 0; j < kSortBpt; ++j) { v[j] = hist[threadIdx.x * kSortBpt + j]; tot += v[j]; }
      unsigned x = tot;
      for (int d = 1; d < 32; d <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, d);
        if (ln >= d) x += y;
      }
      if (ln == 31) wsum[wid] = x;
      __syncthreads();
      unsigned base = x - tot;
      for (int w = 0; w < wid; ++w) base += wsum[w];
#pragma unroll
      for (int j = 0; j < kSortBpt; ++j) { hist[threadIdx.x * kSortBpt + j] = base; base += v[j]; }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < c; i += kSortThreads) {
      const unsigned long long e = s[i];
      const int pos = (int)atomicAdd(&hist[bucket(e)], 1u);
      const int32_t f = (int32_t)(uint32_t)e;
      L[pos] = make_bin_entry(f, __uint_as_float((uint32_t)(e >> 32)), __ldg(ibbox + f));
    }
    __syncthreads();
  }
  }
}

// ------------------------------------------------------------------------------------------------
// K2: fine rasterization — warp-autonomous, (face, pixel) pairs evaluated lane-parallel
//
// Work item = one 8x4 pixel micro-tile of one bin of one mesh. Warps of a persistent grid pull items from a
// global counter (consecutive items = micro-tiles of the same bin, so concurrently running warps share the
// bin's list in L1/L2), and never synchronise with each other: no CTA barrier, no idle lanes while a slow
// neighbour finishes.
//
// Per item the warp streams the bin's face list (or the whole mesh: naive mode / overflowed bin) 32 faces
// at a time: each lane intersects one face's exact integer pixel range (K0) with the micro-tile; faces that
// touch it are compacted (ballot + popc) into a warp-private ring in shared memory together with their
// per-face invariants (structure-of-arrays) and their covered pixel rectangle. Every 32 staged faces the warp
// enumerates their (face, pixel) pairs — prefix sum of the rectangle areas across lanes, then 32 pairs per
// step, one per lane (the pair's face from a ballot and the block's face-start bits) — so every lane evaluates a pair
// (MR:166-176) regardless of how small the triangles are. Passing candidates go into the pixel's sorted
// (z, id) list in shared memory; lanes that hit the same pixel in one step insert one after another
// (__match_any_sync ranks). Winners' bary / dists are recomputed with the identical operation sequence at
// emit time (MR:178-197), so the payload carries exactly the bits the candidate test produced.

constexpr int kPairQ = 64;  // < 32 pending + one enumeration step of 32
// (measured and removed: an early exit of a depth-ordered list once its next key exceeds every pixel's K-th depth
// — the per-chunk test cost more than the chunks it skipped and forced register spills)
constexpr int kRing = 48;  // staged faces per warp: < 32 pending + newly staged (>= 17); 64 measured the same
// Staged fp64 fields per face: only a, b, c, z, area are stored and the edge vectors / squared edge lengths are
// recomputed per pair (same expressions on the same operands => same bits), trading ~15 fp64 ops per pair for 2x
// less shared memory per warp (more resident warps) than staging all 19 invariants.
constexpr int kNF = 10;

enum : int { F_AX, F_AY, F_BX, F_BY, F_CX, F_CY, F_Z0, F_Z1, F_Z2, F_AREA };

// one warp's shared memory: staged-face ring (SoA) + top-K lists of its 32 pixels
// buffered candidates per pixel before the owner lane merges them into its list. Measured: 12 instead of 8 on the
// register path (C4 k_fine 6.16 -> 6.00 ms: fewer overflow merges); on the shared-memory list path 12 costs
// shared memory per warp (C5 6.70 -> 8.52 ms) and 6 is no better (6.74), so 8 there
constexpr int kBufSmem = 8, kBufReg = 12;
__host__ __device__ constexpr int buf_cap(int K) { return K <= 8 ? kBufReg : kBufSmem; }
template <int KMAX>
constexpr int kBufT = KMAX == 0 ? kBufSmem : kBufReg;

struct WarpSmem {
  double* d;        // [kNF][kRing]
  int32_t* fid;     // [kRing]
  uint32_t* rect;   // [kRing] covered rectangle in the micro-tile: r0 | c0<<4 | h<<8 | w<<12 | recip(w)<<16
  float* fkey;      // [kRing] depth key (zkey) of the staged face
  double* tz;       // [K][32]      sorted top-K lists, column p = pixel p of the micro-tile
  int32_t* tid;     // [K][32]
  double* bz;       // [buf_cap(K)][32]   unsorted per-pixel candidate buffers (merged by the owner lane)
  int32_t* bid;     // [buf_cap(K)][32]
  int32_t* bcnt;    // [32]
  double* pxy;      // [12] pixel-centre NDC coordinates of the micro-tile: x of its 8 columns, y of its 4 rows
  uint32_t* pairq;  // [kPairQ] queued (ring slot << 5 | pixel) pairs awaiting evaluation
  int32_t* tcnt;    // [32] entries held by each pixel's list (shared-memory list path, KMAX == 0)
  int ls;           // pixel-major list stride K + 1

  // element (slot s, pixel p) of the top-K lists. kPM: pixel-major rows padded to K + 1 entries, so both the
  // owner-lane accesses (32 pixels, same s) and the transposed emit (consecutive s of a few pixels) hit distinct
  // banks; otherwise slot-major [K][32] (shift-and-add indexing; the emit's same-column reads conflict 8-way).
  // Measured: pixel-major pays for the shared-memory lists (K > 8, C5 k_fine 6.84 -> 6.73 ms) but not for the
  // register-merge path (C4 6.18 -> 6.21 ms), so it is used where KMAX == 0 only.
  template <bool kPM>
  __device__ __forceinline__ int li(int s, int p) const {
    return kPM ? p * ls + s : s * 32 + p;
  }
  // element c of pixel p's candidate buffer, [cap][32] (a pixel-major, conflict-free layout measured 0.4 %
  // slower: the index math costs more than the conflicts of same-pixel appends)
  __device__ __forceinline__ int bi(int c, int p) const { return c * 32 + p; }

  __device__ __forceinline__ double get(int f, int k) const { return d[f * kRing + k]; }
  __device__ __forceinline__ void put(int f, int k, double v) const { d[f * kRing + k] = v; }
  __device__ __forceinline__ FaceGeom geom(int k) const {
    FaceGeom g;
    g.a = V2{get(F_AX, k), get(F_AY, k)};
    g.b = V2{get(F_BX, k), get(F_BY, k)};
    g.c = V2{get(F_CX, k), get(F_CY, k)};
    g.z0 = get(F_Z0, k);
    g.z1 = get(F_Z1, k);
    g.z2 = get(F_Z2, k);
    g.area = get(F_AREA, k);
    g.ab = g.b - g.a;
    g.bc = g.c - g.b;
    g.ca = g.a - g.c;
    g.len_ab = norm2(g.ab);
    g.len_bc = norm2(g.bc);
    g.len_ca = norm2(g.ca);
    return g;
  }
  __device__ __forceinline__ void stage(int k, const double* fv, int32_t f, uint32_t r, float key) const {
    double v[9];
    const double* p = fv + 9 * (int64_t)f;
#pragma unroll
    for (int t = 0; t < 9; ++t) v[t] = __ldg(p + t);
    const FaceGeom g = make_face_geom(v);
    put(F_AX, k, g.a.x); put(F_AY, k, g.a.y); put(F_BX, k, g.b.x); put(F_BY, k, g.b.y);
    put(F_CX, k, g.c.x); put(F_CY, k, g.c.y); put(F_Z0, k, g.z0); put(F_Z1, k, g.z1); put(F_Z2, k, g.z2);
    put(F_AREA, k, g.area);
    fid[k] = f;
    rect[k] = r;
    fkey[k] = key;
  }
};

// per-warp layout, 8-byte aligned pieces first: d | tz | bz | pxy | fid | tid | bid | rect | fkey | bcnt | pairq |
// tcnt
template <int CAP>
__host__ __device__ constexpr size_t warp_smem_bytes_cap(int K) {
  return (size_t)kNF * kRing * sizeof(double) + (size_t)(K + 1) * 32 * sizeof(double) +
         (size_t)CAP * 32 * sizeof(double) + 12 * sizeof(double) + (size_t)kRing * sizeof(int32_t) +
         (size_t)(K + 1) * 32 * sizeof(int32_t) + (size_t)CAP * 32 * sizeof(int32_t) +
         (size_t)kRing * (sizeof(uint32_t) + sizeof(float)) + 32 * sizeof(int32_t) + kPairQ * sizeof(uint32_t) +
         32 * sizeof(int32_t) + 8;  // + pad keeps the next warp's base 8-byte aligned
}
// (the kernel uses the compile-time-capacity form: a runtime select in the warp's base offset cost ptxas ~20
// registers and spills)
// The register-list instantiations (KMAX = 1, 4, 8: the launcher's K thresholds) lay their lists out for KMAX
// entries, so every per-warp array sits at a compile-time offset from the warp's base (one base register, immediate
// offsets) instead of K-dependent run-time pointers the compiler rematerialises in the loops.
__host__ __device__ constexpr int list_kmax(int K) { return K == 1 ? 1 : (K <= 4 ? 4 : (K <= 8 ? 8 : 0)); }
__host__ __device__ constexpr int layout_k(int K) { return list_kmax(K) ? list_kmax(K) : K; }
__host__ __device__ constexpr size_t warp_smem_bytes(int K) {
  return K <= 8 ? warp_smem_bytes_cap<kBufReg>(layout_k(K)) : warp_smem_bytes_cap<kBufSmem>(K);
}

// Rectangle of the micro-tile (rows i0..i0+3, cols j0..j0+7, limited to vh x vw existing pixels) covered by
// the pixel range `ib`; 0 if none. Packed as r0 | c0<<4 | h<<8 | w<<12 | ceil(256/w)<<16: the pair
// rank -> (rank / w, rank % w) split uses (rank * ceil(256/w)) >> 8, exact for rank < 32 and w <= 8.
__device__ __forceinline__ uint32_t cover_rect(int4 ib, int i0, int j0, int vh, int vw) {
  const int r0 = max(ib.x - i0, 0), r1 = min(ib.y - i0, vh - 1);
  const int c0 = max(ib.z - j0, 0), c1 = min(ib.w - j0, vw - 1);
  if (ib.x > ib.y || r0 > r1 || c0 > c1) return 0u;
  const uint32_t h = (uint32_t)(r1 - r0 + 1), w = (uint32_t)(c1 - c0 + 1);
  return (uint32_t)r0 | ((uint32_t)c0 << 4) | (h << 8) | (w << 12) | (((255u + w) / w) << 16);
}

__device__ __forceinline__ double pos_inf() { return __longlong_as_double(0x7ff0000000000000LL); }

template <typename OutT>
__device__ __forceinline__ void emit_slot(const FineArgs<OutT>& A, int64_t slot, bool occupied, double z,
                                          int32_t fid, const double* v, double px, double py, bool persp,
                                          bool clip) {
  if (occupied) {
    const FaceGeom g = make_face_geom(v);
    PixelFaceResult r;
    // fp64 payload: the identical operation sequence => the bits the candidate test produced; fp32 payload: the
    // same formulas with fdiv_payload divisions (~2^-46 relative), rounded once to fp32 (selection is decided)
    eval_pixel_face<true, std::is_same<OutT, double>::value ? 1 : 2>(V2{px, py}, g, A.blur, A.znear, persp, clip, r);
    A.p2f[slot] = fid;
    A.zbuf[slot] = (OutT)z;
    A.bary[3 * slot + 0] = (OutT)r.bary[0];
    A.bary[3 * slot + 1] = (OutT)r.bary[1];
    A.bary[3 * slot + 2] = (OutT)r.bary[2];
    A.dists[slot] = (OutT)r.dist;
  } else {  // MR:191-195
    A.p2f[slot] = -1;
    A.zbuf[slot] = (OutT)-1.0;
    A.bary[3 * slot + 0] = (OutT)0.0;
    A.bary[3 * slot + 1] = (OutT)0.0;
    A.bary[3 * slot + 2] = (OutT)0.0;
    A.dists[slot] = (OutT)0.0;
  }
}

// silhouette_blend's per-slot opacity (shading.cpp:82-83): sigmoid(-dist / sigma) of the slot's signed squared
// distance, recomputed from the face (fast divisions: the value is consumed within tolerance, not selected on)
// (inv_sigma = 1 / sigma: a product and a fast quotient instead of two IEEE divisions per slot)
__device__ __forceinline__ double silhouette_prob(const double* v, double px, double py, double inv_sigma) {
  const FaceGeom g = make_face_geom(v);
  const V2 p{px, py};
  const DistResult dr = point_triangle_dist2<false>(p, g, p - g.a, p - g.b, p - g.c);
  return fdiv(1.0, 1.0 + exp(dr.dist * inv_sigma));  // sigmoid(-dist / sigma)
}

// softmax_blend's clamped inverse depth (shading.cpp:136-137): (zfar - clamp(z, znear, zfar)) / (zfar - znear)
__device__ __forceinline__ double blend_zinv(double z, const BlendArgs& bl) {
  const double zc = z < bl.znear ? bl.znear : (bl.zfar < z ? bl.zfar : z);  // std::clamp
  return (bl.zfar - zc) * bl.inv_zr;
}

// one occupied slot of the softmax render: interpolate_face_attributes of the vertex colours with the slot's
// clamped barycentrics (shading.cpp:11-32: o[d] += w_i * a_i[d], i = 0..2) and the slot's opacity
// sigmoid(-dists / sigma) (shading.cpp:146); fast divisions (values are consumed within tolerance)
template <typename OutT>
__device__ __forceinline__ void softmax_slot(const FineArgs<OutT>& A, const double* v, int32_t f, double px,
                                             double py, double c[3], double& prob) {
  const FaceGeom g = make_face_geom(v);
  PixelFaceResult r;
  eval_pixel_face<true, false>(V2{px, py}, g, A.blur, A.znear, A.persp, A.clip, r);
  c[0] = c[1] = c[2] = 0.0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int64_t vi = A.blend.faces[3 * (int64_t)f + i];
    const double* a = A.blend.vert_colors + 3 * vi;
    c[0] += r.bary[i] * __ldg(a);
    c[1] += r.bary[i] * __ldg(a + 1);
    c[2] += r.bary[i] * __ldg(a + 2);
  }
  prob = fdiv(1.0, 1.0 + exp(r.dist * A.blend.inv_sigma));  // sigmoid(-dists / sigma)
}

// Insert (zc, f) into pixel p's sorted list (column p of [K][32]) in shared memory: shifting loop.
// kCounted (the shared-memory list path, KMAX == 0): ws.tcnt[p] = entries held, so a list that is not full grows
// at its end instead of shifting +inf padding down from slot K-1 (for K = 50 that padding walk was most of the
// fine stage's time). The register path (KMAX > 0, K <= 8) does not maintain tcnt and walks from K-1.
template <bool kCounted>
__device__ __forceinline__ void list_insert(const WarpSmem& ws, int K, int p, double zc, int32_t f) {
  const int n = kCounted ? ws.tcnt[p] : K;
  const int tail = ws.li<kCounted>(K - 1, p);
  if (n < K || cand_less(zc, f, ws.tz[tail], ws.tid[tail])) {
    int s = n < K ? n : K - 1;
    if (kCounted && n < K) ws.tcnt[p] = n + 1;
    while (s > 0) {
      const double zp = ws.tz[ws.li<kCounted>(s - 1, p)];
      const int32_t ip = ws.tid[ws.li<kCounted>(s - 1, p)];
      if (!cand_less(zc, f, zp, ip)) break;
      ws.tz[ws.li<kCounted>(s, p)] = zp;
      ws.tid[ws.li<kCounted>(s, p)] = ip;
      --s;
    }
    ws.tz[ws.li<kCounted>(s, p)] = zc;
    ws.tid[ws.li<kCounted>(s, p)] = f;
  }
}

// Every lane merges the buffered candidates of ITS pixel (p = lane) into its sorted list: all 32 lanes work
// at once, and for K <= KMAX the list lives in registers during the merge (fully unrolled insertion: no
// shared-memory load -> compare -> branch chain). The merge runs outside the fp64 evaluation, so these
// registers do not add to the evaluation's pressure.
// (an out-of-line merge measured slower: 11.76 vs 10.30 ms)
template <int KMAX>
__device__ __forceinline__ void merge_buffers(const WarpSmem& ws, int K, int lane) {
  const int n = ws.bcnt[lane];
#if DR_STATS
  STAT_ADD(8, __reduce_add_sync(0xffffffffu, (unsigned)n));
  STAT_ADD(9, 1);
  unsigned below = 0;
#endif
  if (n > 0) {
    if constexpr (KMAX == 0) {
      for (int c = 0; c < n; ++c) list_insert<true>(ws, K, lane, ws.bz[ws.bi(c, lane)], ws.bid[ws.bi(c, lane)]);
    } else {
      double z[KMAX];
      int32_t id[KMAX];
#pragma unroll
      for (int s = 0; s < KMAX; ++s) {
        z[s] = s < K ? ws.tz[ws.li<(KMAX == 0)>(s, lane)] : pos_inf();
        id[s] = s < K ? ws.tid[ws.li<(KMAX == 0)>(s, lane)] : INT_MAX;
      }
      for (int c = 0; c < n; ++c) {
        const double zc = ws.bz[ws.bi(c, lane)];
        const int32_t ic = ws.bid[ws.bi(c, lane)];
        if (!cand_less(zc, ic, z[KMAX - 1], id[KMAX - 1])) continue;  // not below the list tail
#if DR_STATS
        ++below;
#endif
#pragma unroll
        for (int s = KMAX - 1; s >= 0; --s) {
          const int sp = s > 0 ? s - 1 : 0;
          const bool lt_prev = s > 0 && cand_less(zc, ic, z[sp], id[sp]);
          const bool lt_cur = cand_less(zc, ic, z[s], id[s]);
          if (lt_prev) {
            z[s] = z[sp];
            id[s] = id[sp];
          } else if (lt_cur) {
            z[s] = zc;
            id[s] = ic;
          }
        }
      }
#pragma unroll
      for (int s = 0; s < KMAX; ++s) {
        if (s < K) {
          ws.tz[ws.li<(KMAX == 0)>(s, lane)] = z[s];
          ws.tid[ws.li<(KMAX == 0)>(s, lane)] = id[s];
        }
      }
    }
    ws.bcnt[lane] = 0;
  }
#if DR_STATS
  STAT_ADD(10, __reduce_add_sync(0xffffffffu, below));
#endif
}

// Append a passing candidate to its pixel's buffer (merging every buffer first if one would overflow).
// Append passing candidates to their pixels' buffers with shared-memory atomics on the buffer counts (no
// match_any grouping); when a buffer is full the warp merges every buffer and the overflowed candidates retry.
// Insertion order is irrelevant: the K smallest under the strict (z, id) order do not depend on it (MR:138-140).
// (It replaced __match_any_sync grouping of same-pixel lanes with ranks from the group mask: C4 k_fine 5.42 ->
// 5.06 ms, C5 6.19 -> 5.68 ms.)
template <int KMAX, typename OutT>
__device__ __forceinline__ void insert_candidate(const FineArgs<OutT>& A, const WarpSmem& ws, bool pass, int p,
                                                 int32_t f, double z, int lane) {
  const int K = A.K;
  bool todo = pass;
  while (__any_sync(0xffffffffu, todo)) {
    const int pos = todo ? atomicAdd(&ws.bcnt[p], 1) : 0;
    const bool ok = todo && pos < kBufT<KMAX>;
    if (ok) {
      ws.bz[ws.bi(pos, p)] = z;
      ws.bid[ws.bi(pos, p)] = f;
    }
    todo = todo && !ok;
    if (__any_sync(0xffffffffu, todo)) {  // a buffer is full: merge them all, then retry the rest
      __syncwarp();
      STAT_ADD(11, 1);
      if (todo && pos == kBufT<KMAX>) ws.bcnt[p] = kBufT<KMAX>;  // undo the failed increments (one writer)
      __syncwarp();
      merge_buffers<KMAX>(ws, K, lane);
    }
    __syncwarp();
  }
}

// Evaluate the first n (<= 32) queued (face slot, pixel) pairs, one per lane, and insert the survivors.
template <int KMAX, typename OutT>
__device__ __forceinline__ void eval_pairs(const FineArgs<OutT>& A, const WarpSmem& ws, int n, int lane,
                                           bool persp, bool clip) {
  const uint32_t e = lane < n ? ws.pairq[lane] : 0x80000000u;
  const bool act = lane < n;
  bool pass = false;
  int p = 0;
  int32_t f = 0;
  PixelFaceResult res;
  if (act) {
    const int k = (int)(e >> 5);
    p = (int)(e & 31u);
    const FaceGeom fg = ws.geom(k);
    const V2 pix{ws.pxy[p & 7], ws.pxy[8 + (p >> 3)]};
    pass = eval_pixel_face<false>(pix, fg, A.blur, A.znear, persp, clip, res);
    f = ws.fid[k];
  }
  STAT_ADD(3, __popc(__ballot_sync(0xffffffffu, act)));
  STAT_ADD(4, __popc(__ballot_sync(0xffffffffu, pass)));
  STAT_ADD(7, 1);
  insert_candidate<KMAX>(A, ws, pass, p, f, res.z, lane);
}


// Enumerate the (face, pixel) pairs of ring slots [head, head+G) (mod kRing): prefix sum of the covered
// rectangle areas across lanes, then 32 pairs per step, one per lane (the pair's face from the block's face-start
// bits). Pairs the K-th-depth cull cannot rule out are compacted (ballot) into the warp's pair queue and
// evaluated 32 at a time, so culled pairs cost no fp64 work and evaluation steps keep every lane busy. The
// queue is drained before returning (its entries name ring slots the caller recycles).
template <int KMAX, typename OutT>
__device__ __forceinline__ void process_group(const FineArgs<OutT>& A, const WarpSmem& ws, int head, int G,
                                              int lane, bool persp, bool clip) {
  const int K = A.K;
  const int slot_l = (head + lane) % kRing;
  const uint32_t rl = lane < G ? ws.rect[slot_l] : 0u;
  const int cnt = (int)(((rl >> 8) & 15u) * ((rl >> 12) & 15u));
  int incl = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  int qn = 0;  // queued pairs (< 32 between steps)
  int base = 0;
  // one loop, one inlined copy of eval_pairs (instruction-cache footprint is a first-order cost here)
  for (;;) {
    if (base < total) {
      const int j = base + lane;
      const bool act = j < total;
      // face lane = first lane whose inclusive prefix exceeds j
      // = (faces starting at or before `base`) - 1 + (faces starting in (base, j]): one ballot, one OR-reduction
      // of the start bits of this block of 32 pairs, one popc per lane (staged faces are lanes < G, cnt >= 1).
      // (It replaced a 5-step shuffle binary search over the prefix: C4 k_fine -1.3 %, C5 -3.2 %.)
      const int excl_l = incl - cnt;
      const int f0 = __popc(__ballot_sync(0xffffffffu, cnt > 0 && excl_l <= base)) - 1;
      const unsigned starts = __reduce_or_sync(
          0xffffffffu, (cnt > 0 && excl_l > base && excl_l < base + 32) ? (1u << (excl_l - base)) : 0u);
      const int lo = min(max(f0 + __popc(starts & ((2u << lane) - 1u)), 0), 31);
      const int excl = __shfl_sync(0xffffffffu, incl - cnt, lo);
      const uint32_t r = __shfl_sync(0xffffffffu, rl, lo);
      bool keep = false;
      uint32_t entry = 0;
      if (act) {
        const int rank = j - excl;
        const int w = (int)((r >> 12) & 15u);
        const int dr = (rank * (int)(r >> 16)) >> 8;
        const int row = (int)(r & 15u) + dr;
        const int col = (int)((r >> 4) & 15u) + (rank - dr * w);
        const int p = row * 8 + col;
        const int k = (head + lo) % kRing;
        // K-th-depth cull: every z this face can produce is > its key; if the key already exceeds the pixel's
        // current K-th candidate the face cannot enter the pixel's list (strict (z, id) order, MR:138-140)
        keep = !clip || !((double)ws.fkey[k] > ws.tz[ws.li<(KMAX == 0)>(K - 1, p)]);  // zsort == clip
        entry = ((uint32_t)k << 5) | (uint32_t)p;
      }
      STAT_ADD(2, __popc(__ballot_sync(0xffffffffu, act)));
      const unsigned kb = __ballot_sync(0xffffffffu, keep);
      if (keep) ws.pairq[qn + __popc(kb & ((1u << lane) - 1u))] = entry;
      qn += __popc(kb);
      base += 32;
      __syncwarp();
    }
    const bool drain = base >= total;
    if (qn >= 32 || (drain && qn > 0)) {
      const int n = min(qn, 32);
      eval_pairs<KMAX>(A, ws, n, lane, persp, clip);
      qn -= n;
      if (qn > 0) {  // move the remainder to the front
        const uint32_t t = lane < qn ? ws.pairq[32 + lane] : 0u;
        __syncwarp();
        if (lane < qn) ws.pairq[lane] = t;
      }
      __syncwarp();
    }
    if (drain && qn == 0) break;
  }
}

// 128 registers per thread (16 resident warps per SM) is the measured sweet spot: capping lower spills, and
// fewer resident warps cannot hide the fp64 dependency latency (profiles/r01/README.md).
// kMode: 0 = the fragment payload; 1 = fused silhouette emit (alpha, optional pix_to_face); 2 = fused softmax
// render emit (interpolated vertex colours + softmax_blend -> image, optional pix_to_face) — separate
// instantiations so the fragment path's code (and register allocation) does not carry them
// kPC: perspective_correct fixed at compile time (0 / 1) for the fragment instantiations, read from A (2) for the
// fused consumers (their own instantiations already multiply the kernel count)
// kExactK: K == KMAX (the register path's common case), so every loop over the list has a compile-time trip count
template <typename OutT, int NW, int KMAX, int kMode, int kPC = 2, int kCL = 2, bool kExactK = false>
__global__ void __launch_bounds__(NW * 32, 16 / NW) k_fine(FineArgs<OutT> A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int K = kExactK ? KMAX : A.K;
  const bool persp = kPC == 2 ? A.persp : kPC == 1;
  // clip_barycentric_coords; the depth-ordered bins and K-th-depth culling are on exactly when it is (make_plan)
  const bool clip = kCL == 2 ? A.clip : kCL == 1;
  WarpSmem ws;
  {
    const int KL = KMAX > 0 ? KMAX : K;  // list layout (compile-time on the register path)
    unsigned char* base = smem_raw + (size_t)wid * warp_smem_bytes_cap<kBufT<KMAX>>(KL);
    ws.d = reinterpret_cast<double*>(base);
    ws.tz = ws.d + kNF * kRing;
    ws.bz = ws.tz + (KL + 1) * 32;
    ws.ls = K + 1;
    ws.pxy = ws.bz + kBufT<KMAX> * 32;  // == buf_cap(K): KMAX == 0 exactly when K > 8
    ws.fid = reinterpret_cast<int32_t*>(ws.pxy + 12);
    ws.tid = ws.fid + kRing;
    ws.bid = ws.tid + (KL + 1) * 32;
    ws.rect = reinterpret_cast<uint32_t*>(ws.bid + kBufT<KMAX> * 32);
    ws.fkey = reinterpret_cast<float*>(ws.rect + kRing);
    ws.bcnt = reinterpret_cast<int32_t*>(ws.fkey + kRing);
    ws.pairq = reinterpret_cast<uint32_t*>(ws.bcnt + 32);
    ws.tcnt = reinterpret_cast<int32_t*>(ws.pairq + kPairQ);
  }
  const int nbins = A.nbx * A.nby;
  const int mtx = (A.bs + 7) >> 3, mty = (A.bs + 3) >> 2;  // micro-tiles per bin row / column
  const int mt_per_bin = mtx * mty;
  const int64_t n_items = (int64_t)A.N * nbins * mt_per_bin;

  for (;;) {
    int64_t item = 0;
    if (lane == 0) item = (int64_t)atomicAdd(A.work_counter, 1ull);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= n_items) break;
    int mt, bin, b;
    if (n_items <= 0xffffffffll) {  // (uniform) 32-bit decode with precomputed reciprocals
      const uint32_t it = (uint32_t)item, q1 = A.div_mt.div(it), q2 = A.div_bins.div(q1);
      mt = (int)(it - q1 * (uint32_t)mt_per_bin);
      bin = (int)(q1 - q2 * (uint32_t)nbins);
      b = (int)q2;
    } else {
      mt = (int)(item % mt_per_bin);
      const int64_t bb = item / mt_per_bin;
      bin = (int)(bb % nbins);
      b = (int)(bb / nbins);
    }
    const int by = (int)A.div_nbx.div((uint32_t)bin), bx = bin - by * A.nbx;
    const int bi0 = by * A.bs, bj0 = bx * A.bs;
    const int bi1 = min(A.H, bi0 + A.bs) - 1, bj1 = min(A.W, bj0 + A.bs) - 1;
    const int mtr = (int)A.div_mtx.div((uint32_t)mt);
    const int mi0 = bi0 + mtr * 4, mj0 = bj0 + (mt - mtr * mtx) * 8;
    const int vh = min(4, bi1 - mi0 + 1), vw = min(8, bj1 - mj0 + 1);  // existing pixels of the micro-tile
    if (vh <= 0 || vw <= 0) continue;
    STAT_ADD(5, 1);

    // candidate faces: the bin list, or the whole mesh (naive mode / overflowed bin)
    const int64_t f0 = A.first[b], nf = A.num[b];
    const int4* list = nullptr;
    int64_t nsrc = nf;
    if (A.binned) {
      const int64_t gb = (int64_t)b * nbins + bin;
      const int c = A.bin_counts[gb];
      const int64_t o = A.bin_off[gb];
      if (bin_fits(o, c, A.pool, A.cap)) {
        list = A.bin_entries + o;
        nsrc = c;
      }
    }
    for (int s = 0; s < K; ++s) {
      ws.tz[ws.li<(KMAX == 0)>(s, lane)] = pos_inf();
      ws.tid[ws.li<(KMAX == 0)>(s, lane)] = INT_MAX;
    }
    ws.bcnt[lane] = 0;
    ws.tcnt[lane] = 0;
    if (lane < 8) ws.pxy[lane] = pixel_x(A.W, mj0 + lane);               // camera.cpp:100-102, once per
    else if (lane < 12) ws.pxy[lane] = pixel_y(A.H, mi0 + (lane - 8));   // micro-tile instead of per pair
    __syncwarp();

    const bool valid_px = (lane >> 3) < vh && (lane & 7) < vw;
    double T = pos_inf();  // max over the micro-tile's pixels of the K-th candidate depth (+inf: a list not full)
    int head = 0, pending = 0;
    // the next 32 list entries are loaded while the current ones are staged and evaluated
    int4 e_next = make_int4(-1, 0, 0, 0);
    if (list && lane < nsrc) e_next = list[lane];
    for (int64_t c0 = 0; c0 < nsrc; c0 += 32) {
      const int64_t ci = c0 + lane;
      uint32_t r = 0u;
      int32_t fid = -1;
      float key = 0.f;
      const int4 e_cur = e_next;
      if (list && ci + 32 < nsrc) e_next = list[ci + 32];
      STAT_ADD(0, __popc(__ballot_sync(0xffffffffu, ci < nsrc)));
      if (ci < nsrc) {
        int4 ib;
        if (list) {
          const int4 e = e_cur;
          fid = e.x;
          key = __int_as_float(e.y);
          ib = entry_ibbox(e);
        } else {
          fid = (int32_t)(f0 + ci);
          key = clip ? A.zkey[fid] : 0.f;
          ib = A.ibbox[fid];
        }
        if (!clip || !((double)key > T)) r = cover_rect(ib, mi0, mj0, vh, vw);
      }
      unsigned todo = __ballot_sync(0xffffffffu, r != 0u);
      const bool last = c0 + 32 >= nsrc;
      do {
        // stage as many of the remaining faces as the ring has room for (room >= 17 since pending < 32)
        const int room = kRing - pending;
        const int rank = __popc(todo & ((1u << lane) - 1u));
        const bool mine = ((todo >> lane) & 1u) && rank < room;
        const unsigned take = __ballot_sync(0xffffffffu, mine);
        if (mine) ws.stage((head + pending + rank) % kRing, A.fv, fid, r, key);
        pending += __popc(take);
        STAT_ADD(1, __popc(take));
        todo &= ~take;
        __syncwarp();
        bool ran = false;
        while (pending >= 32 || (last && todo == 0u && pending > 0)) {
          const int G = min(pending, 32);
          process_group<KMAX>(A, ws, head, G, lane, persp, clip);
          head = (head + G) % kRing;
          pending -= G;
          ran = true;
        }
        if (ran) {  // merge the buffered candidates (the only merge site besides a buffer overflow), refresh T
          __syncwarp();
          merge_buffers<KMAX>(ws, K, lane);
          __syncwarp();
          if (clip) {  // max of the K-th depths (the list tails alone are a valid, looser threshold)
            double t = valid_px ? ws.tz[ws.li<(KMAX == 0)>(K - 1, lane)] : -pos_inf();
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, d));
            T = t;
          }
        }
      } while (todo);
    }
    // every group's candidates were merged after it ran: the buffers are empty here
    __syncwarp();
    if constexpr (kMode == 0) {
      // fragment payload (MR:178-197), lanes over (pixel, slot) in output order: q = (row * 8 + col) * K + s, so
      // one step writes whole runs of consecutive slots of a micro-tile row (coalesced stores); the next step's
      // face_verts are fetched before the current slot is evaluated. A lane's (pixel, slot) advances by 32 slots per
      // step incrementally (no integer division by K per step) and its output slot is the micro-tile's base plus
      // 32-bit offsets.
      const int64_t slot_base = (((int64_t)b * A.H + mi0) * A.W + mj0) * K;
      const int row_stride = A.W * K;
      const int dpix = 32 / K, ds = 32 - dpix * K;
      int fpix = lane / K, fs = lane - fpix * K;  // (pixel, slot) of this lane's next fetch
      auto fetch = [&](int32_t& f, double* v, int64_t& slot, double& z, double& qx, double& qy) {
        const int pix = fpix, s = fs;
        fs += ds;
        fpix += dpix;
        if (fs >= K) {
          fs -= K;
          ++fpix;
        }
        f = INT_MAX;
        slot = -1;
        if (pix >= 32) return;
        const int row = pix >> 3, col = pix & 7;
        if (row >= vh || col >= vw) return;
        slot = slot_base + (int64_t)(row * row_stride + col * K + s);
        f = ws.tid[ws.li<(KMAX == 0)>(s, pix)];
        z = ws.tz[ws.li<(KMAX == 0)>(s, pix)];
        qx = ws.pxy[col];
        qy = ws.pxy[8 + row];
        if (f != INT_MAX) {
#pragma unroll
          for (int t = 0; t < 9; ++t) v[t] = __ldg(A.fv + 9 * (int64_t)f + t);
        }
      };
      if constexpr (KMAX > 0) {
        // register-list path (K <= 8, <= 256 (pixel, slot) entries): empty slots get their constant payload here and
        // the occupied ones (typically ~45 %) are compacted (ballot) into the idle candidate-id buffer, so the fp64
        // payload recompute below runs on full warps instead of under a ~45 %-active lane mask (C4 k_fine 4.72 ->
        // 4.63 ms)
        int n = 0;
        for (int q0 = 0; q0 < 32 * K; q0 += 32) {
          const int pix = fpix, sl = fs;
          fs += ds;
          fpix += dpix;
          if (fs >= K) {
            fs -= K;
            ++fpix;
          }
          const int row = pix >> 3, col = pix & 7;
          const bool valid = pix < 32 && row < vh && col < vw;
          const int32_t f = valid ? ws.tid[ws.li<false>(sl, pix)] : INT_MAX;
          if (valid && f == INT_MAX) {
            const double vz[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
            emit_slot<OutT>(A, slot_base + (int64_t)(row * row_stride + col * K + sl), false, 0.0, f, vz, 0.0, 0.0,
                            persp, clip);
          }
          const bool occ = valid && f != INT_MAX;
          const unsigned m = __ballot_sync(0xffffffffu, occ);
          if (occ) ws.bid[n + __popc(m & ((1u << lane) - 1u))] = (pix << 8) | sl;
          n += __popc(m);
        }
        __syncwarp();
        auto fetch_c = [&](int i, int32_t& f, double* v, int64_t& slot, double& z, double& qx, double& qy) {
          f = INT_MAX;
          slot = -1;
          if (i >= n) return;
          const int e = ws.bid[i], pix = e >> 8, sl = e & 255, row = pix >> 3, col = pix & 7;
          slot = slot_base + (int64_t)(row * row_stride + col * K + sl);
          f = ws.tid[ws.li<false>(sl, pix)];
          z = ws.tz[ws.li<false>(sl, pix)];
          qx = ws.pxy[col];
          qy = ws.pxy[8 + row];
#pragma unroll
          for (int t = 0; t < 9; ++t) v[t] = __ldg(A.fv + 9 * (int64_t)f + t);
        };
        int32_t fn;
        double vn[9], zn = 0.0, xn = 0.0, yn = 0.0;
        int64_t sn;
        fetch_c(lane, fn, vn, sn, zn, xn, yn);
        for (int b0 = 0; b0 < n; b0 += 32) {
          const int32_t f = fn;
          const int64_t slot = sn;
          const double z = zn, qx = xn, qy = yn;
          double v[9];
#pragma unroll
          for (int t = 0; t < 9; ++t) v[t] = vn[t];
          fetch_c(b0 + 32 + lane, fn, vn, sn, zn, xn, yn);
          if (slot >= 0) emit_slot<OutT>(A, slot, true, z, f, v, qx, qy, persp, clip);
        }
        __syncwarp();
        continue;
      }
      // shared-memory list path (K > 8): occupancy is higher there and the streamed form of the compaction (no
      // face_verts prefetch) measured slower (C5 5.42 -> 5.55 ms), so this path keeps the transposed loop
      int32_t fn;
      double vn[9], zn = 0.0, xn = 0.0, yn = 0.0;
      int64_t sn;
      fetch(fn, vn, sn, zn, xn, yn);
      for (int q0 = 0; q0 < 32 * K; q0 += 32) {
        const int32_t f = fn;
        const int64_t slot = sn;
        const double z = zn, qx = xn, qy = yn;
        double v[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) v[t] = vn[t];
        fetch(fn, vn, sn, zn, xn, yn);
        if (slot >= 0) emit_slot<OutT>(A, slot, f != INT_MAX, z, f, v, qx, qy, persp, clip);
      }
      __syncwarp();
      continue;
    }
    // emit this lane's pixel (MR:178-197); the next occupied slot's face_verts are fetched before the current
    // slot is evaluated so the global-load latency overlaps the fp64 work
    const int row = lane >> 3, col = lane & 7;
    if (row < vh && col < vw) {
      const int pi = mi0 + row, pj = mj0 + col;
      const double px = pixel_x(A.W, pj), py = pixel_y(A.H, pi);
      const int64_t slot0 = (((int64_t)b * A.H + pi) * A.W + pj) * K;
      double vnext[9];
      int32_t fnext = ws.tid[ws.li<(KMAX == 0)>(0, lane)];
      if (fnext != INT_MAX) {
#pragma unroll
        for (int t = 0; t < 9; ++t) vnext[t] = __ldg(A.fv + 9 * (int64_t)fnext + t);
      }
      double keep = 1.0;  // silhouette mode: prod over occupied slots of (1 - prob)
      const double inv_sigma = kMode == 1 ? 1.0 / A.sigma : 0.0;
      // softmax mode (shading.cpp:123-160): zinv_max over the occupied slots from the exact depths in the list
      double zinv_max = -1.0, wsum = 0.0, acc[3] = {0.0, 0.0, 0.0};
      bool any = false;
      if constexpr (kMode == 2) {
        for (int s = 0; s < K; ++s) {
          if (ws.tid[ws.li<(KMAX == 0)>(s, lane)] == INT_MAX) continue;
          any = true;
          const double zi = blend_zinv(ws.tz[ws.li<(KMAX == 0)>(s, lane)], A.blend);
          zinv_max = zinv_max < zi ? zi : zinv_max;  // std::max(zinv_max, zinv)
        }
      }
      for (int s = 0; s < K; ++s) {
        const int32_t f = fnext;
        double v[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) v[t] = vnext[t];
        fnext = s + 1 < K ? ws.tid[ws.li<(KMAX == 0)>(s + 1, lane)] : INT_MAX;
        if (fnext != INT_MAX) {
#pragma unroll
          for (int t = 0; t < 9; ++t) vnext[t] = __ldg(A.fv + 9 * (int64_t)fnext + t);
        }
        if constexpr (kMode == 1) {
          if (A.p2f) A.p2f[slot0 + s] = f != INT_MAX ? (int64_t)f : -1;
          if (f != INT_MAX) keep *= 1.0 - silhouette_prob(v, px, py, inv_sigma);
        } else if constexpr (kMode == 2) {
          if (A.p2f) A.p2f[slot0 + s] = f != INT_MAX ? (int64_t)f : -1;
          if (f != INT_MAX) {
            double c[3], prob;
            softmax_slot(A, v, f, px, py, c, prob);
            const double zi = blend_zinv(ws.tz[ws.li<(KMAX == 0)>(s, lane)], A.blend);
            const double w = prob * exp((zi - zinv_max) * A.blend.inv_gamma);
            wsum += w;
            acc[0] += c[0] * w;  // Vec3 += Vec3 * double
            acc[1] += c[1] * w;
            acc[2] += c[2] * w;
          }
        } else {
          emit_slot<OutT>(A, slot0 + s, f != INT_MAX, ws.tz[ws.li<(KMAX == 0)>(s, lane)], f, v, px, py, persp,
                          clip);
        }
      }
      if constexpr (kMode == 1) A.alpha[((int64_t)b * A.H + pi) * A.W + pj] = (OutT)(1.0 - keep);  // shading.cpp:86
      if constexpr (kMode == 2) {
        OutT* img = A.image + 3 * (((int64_t)b * A.H + pi) * A.W + pj);
        if (!any) {
          img[0] = (OutT)A.blend.background[0];  // shading.cpp:130, 141
          img[1] = (OutT)A.blend.background[1];
          img[2] = (OutT)A.blend.background[2];
        } else {
          const double inv = 1.0 / wsum;  // image = acc * (1.0 / wsum), shading.cpp:153
          img[0] = (OutT)(acc[0] * inv);
          img[1] = (OutT)(acc[1] * inv);
          img[2] = (OutT)(acc[2] * inv);
        }
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------------------
// host-side launchers (called from capi.cu)

void launch_face_setup(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t max_faces,
                       const std::vector<std::pair<int64_t, int64_t>>& intervals, int H, int W, double inflate,
                       double znear, int clip_z, int cull, int4* ibbox, float* zkey, cudaStream_t st) {
  if (max_faces <= 0) return;
  if (intervals.size() <= 8) {  // one launch per merged interval of the ranges (one for a whole packed batch)
    for (const auto& iv : intervals)
      k_face_setup_range<<<(unsigned)((iv.second - iv.first + 255) / 256), 256, 0, st>>>(
          fv, iv.first, iv.second, H, W, inflate, znear, clip_z, cull, ibbox, zkey);
    return;
  }
  const unsigned gx = (unsigned)std::min<int64_t>((max_faces + 255) / 256, 65535);
  k_face_setup<<<dim3(gx, (unsigned)N), 256, 0, st>>>(fv, first, num, H, W, inflate, znear, clip_z, cull, ibbox,
                                                      zkey);
}

void launch_bin_faces(const int4* ibbox, const int64_t* first, const int64_t* num, int64_t N, int64_t max_faces,
                      int bs, int nbx, int nby, int* counts, cudaStream_t st, bool smem_hist) {
  if (max_faces <= 0) return;
  if (smem_hist && (int64_t)nbx * nby <= kBinSmemMax && (max_faces + kBinChunk - 1) / kBinChunk <= 65535) {
    const unsigned gx = (unsigned)((max_faces + kBinChunk - 1) / kBinChunk);
    k_bin_faces_smem<false><<<dim3(gx, (unsigned)N), 256, 0, st>>>(ibbox, first, num, bs, nbx, nby, counts, nullptr,
                                                                  nullptr, 0, nullptr, nullptr);
    return;
  }
  unsigned gx = (unsigned)std::min<int64_t>((max_faces + 255) / 256, 65535);
  k_bin_faces<false><<<dim3(gx, (unsigned)N), 256, 0, st>>>(ibbox, first, num, bs, nbx, nby, counts, nullptr, nullptr,
                                                           0, nullptr, nullptr);
}

void launch_scan_bins(const int* counts, int64_t nbins_total, int64_t* off, cudaStream_t st) {
  if (nbins_total <= 0) return;
  const unsigned nseg = (unsigned)((nbins_total + kScanSeg - 1) / kScanSeg);
  k_scan_local<<<nseg, kScanThreads, 0, st>>>(counts, nbins_total, off);
  if (nseg > 1) {
    k_scan_fix<<<nseg, 256, 0, st>>>(counts, nbins_total, off);
    k_scan_last<<<1, 1, 0, st>>>(counts, nbins_total, off);
  }
}

void launch_fill_bins(const int4* ibbox, const int64_t* first, const int64_t* num, int64_t N, int64_t max_faces,
                      int bs, int nbx, int nby, const int* counts, const int64_t* off, int* cursor, int64_t pool,
                      const float* zkey, int4* entries, cudaStream_t st, bool smem_hist) {
  if (max_faces <= 0) return;
  if (smem_hist && (int64_t)nbx * nby <= kBinSmemMax && (max_faces + kBinChunk - 1) / kBinChunk <= 65535) {
    const unsigned gx = (unsigned)((max_faces + kBinChunk - 1) / kBinChunk);
    k_bin_faces_smem<true><<<dim3(gx, (unsigned)N), 256, 0, st>>>(ibbox, first, num, bs, nbx, nby,
                                                                 const_cast<int*>(counts), off, cursor, pool, zkey,
                                                                 entries);
    return;
  }
  unsigned gx = (unsigned)std::min<int64_t>((max_faces + 255) / 256, 65535);
  k_bin_faces<true><<<dim3(gx, (unsigned)N), 256, 0, st>>>(ibbox, first, num, bs, nbx, nby,
                                                          const_cast<int*>(counts), off, cursor, pool, zkey, entries);
}

cudaError_t launch_sort_bins(const int* counts, const int64_t* off, int4* entries, const int4* ibbox,
                             int64_t nbins_total, int64_t pool, int cap, cudaStream_t st, float2* bin_range) {
  if (nbins_total <= 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<int64_t>(nbins_total, 148 * 16);
  k_sort_bins_warp<<<(unsigned)std::min<int64_t>((nbins_total + kWarpSortWarps - 1) / kWarpSortWarps, 148 * 8),
                     kWarpSortWarps * 32, 0, st>>>(counts, off, entries, ibbox, nbins_total, pool, cap, bin_range);
  k_sort_bins<kSortMax, kWarpSortMax, false><<<grid, kSortThreads, 0, st>>>(counts, off, entries, ibbox,
                                                                            nbins_total, pool, cap, bin_range);
  auto big = k_sort_bins<kSortMaxBig, kSortMax, true>;
  const int smem = kSortMaxBig * (int)sizeof(unsigned long long);
  cudaError_t e = cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  big<<<(unsigned)std::min<int64_t>(nbins_total, 148), kSortThreads, smem, st>>>(counts, off, entries, ibbox,
                                                                                  nbins_total, pool, cap, bin_range);
  return cudaGetLastError();
}

template <typename OutT>
static cudaError_t launch_fine_t(const FineArgs<OutT>& A, int nw, cudaStream_t st) {
  const size_t smem = (size_t)nw * warp_smem_bytes(A.K);
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    kern<<<(unsigned)(sms * per_sm), nw * 32, smem, st>>>(A);  // persistent: warps pull micro-tiles
    return cudaGetLastError();
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  // the fused consumers at K == 8 on the register path (the headline K): flags and K fixed at compile time too
  auto consumer_k8 = [&](auto mode_c) -> cudaError_t {
    constexpr int M = decltype(mode_c)::value;
    auto f = [&](auto pc, auto cl) -> cudaError_t {
      return go(k_fine<OutT, 8, 8, M, decltype(pc)::value, decltype(cl)::value, true>);
    };
    if (A.persp) return A.clip ? f(I1{}, I1{}) : f(I1{}, I0{});
    return A.clip ? f(I0{}, I1{}) : f(I0{}, I0{});
  };
  auto by_k = [&](auto nw_c) -> cudaError_t {
    constexpr int NW = decltype(nw_c)::value;
    // register-resident merge for small K, shared-memory shifting loop otherwise
    if (A.alpha) {  // fused silhouette: fp32 alpha, or fp64 for the fit loop (fit.py)
      if constexpr (NW == 8) {
        if (A.K == 8) return consumer_k8(std::integral_constant<int, 1>{});
      }
      if (A.K == 1) return go(k_fine<OutT, NW, 1, 1>);
      if (A.K <= 4) return go(k_fine<OutT, NW, 4, 1>);
      if (A.K <= 8) return go(k_fine<OutT, NW, 8, 1>);
      return go(k_fine<OutT, NW, 0, 1>);
    }
    if (A.image) {
      if constexpr (std::is_same<OutT, float>::value) {  // the fused softmax render writes an fp32 image only
        if constexpr (NW == 8) {
          if (A.K == 8) return consumer_k8(std::integral_constant<int, 2>{});
        }
        if (A.K == 1) return go(k_fine<OutT, NW, 1, 2>);
        if (A.K <= 4) return go(k_fine<OutT, NW, 4, 2>);
        if (A.K <= 8) return go(k_fine<OutT, NW, 8, 2>);
        return go(k_fine<OutT, NW, 0, 2>);
      } else {
        return cudaErrorInvalidValue;
      }
    }
    // fragment payload: one instantiation per (perspective_correct, clip_barycentric_coords)
    auto by_flags = [&](auto pc, auto cl) -> cudaError_t {
      constexpr int PC = decltype(pc)::value, CL = decltype(cl)::value;
      if constexpr (NW == 8) {  // (the register path always runs 8-warp CTAs)
        if (A.K == 1) return go(k_fine<OutT, NW, 1, 0, PC, CL, true>);
        if (A.K == 4) return go(k_fine<OutT, NW, 4, 0, PC, CL, true>);
        if (A.K == 8) return go(k_fine<OutT, NW, 8, 0, PC, CL, true>);
      }
      if (A.K == 1) return go(k_fine<OutT, NW, 1, 0, PC, CL>);
      if (A.K <= 4) return go(k_fine<OutT, NW, 4, 0, PC, CL>);
      if (A.K <= 8) return go(k_fine<OutT, NW, 8, 0, PC, CL>);
      return go(k_fine<OutT, NW, 0, 0, PC, CL>);
    };
    if (A.persp) return A.clip ? by_flags(I1{}, I1{}) : by_flags(I1{}, I0{});
    return A.clip ? by_flags(I0{}, I1{}) : by_flags(I0{}, I0{});
  };
  if (nw == 8) return by_k(std::integral_constant<int, 8>{});
  return by_k(std::integral_constant<int, 2>{});
}

size_t fine_warp_smem_bytes(int K) { return warp_smem_bytes(K); }

cudaError_t launch_fine(const FineArgs<float>& A, int nwarps, cudaStream_t st) { return launch_fine_t(A, nwarps, st); }
cudaError_t launch_fine(const FineArgs<double>& A, int nwarps, cudaStream_t st) { return launch_fine_t(A, nwarps, st); }

}  // namespace drb

#if DR_STATS
extern "C" int dr_debug_stats(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_stats, sizeof(unsigned long long) * 12);
  if (reset) {
    unsigned long long z[12] = {};
    cudaMemcpyToSymbol(g_stats, z, sizeof(z));
  }
  return 0;
}
#endif
