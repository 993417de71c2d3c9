// Point rasterizer on sm_100a: rasterize_points / rasterize_points_naive
// (/root/reference/proj/src/point_render.cpp, "PR" below, :105-155 / :82-103) and the backward of its
// fragments to the projected points (PyTorch3D's rasterize_points backward; the reference's
// splat_position_backward, PR:302-338, is this with d_dists2 = -d_alpha / radius^2, d_zbuf = 0).
//
//   P0 k_point_setup    prepare_points (PR:17-31): cull (clipped, z_view < znear, non-finite) + the EXACT range of
//                       tiles whose reference rectangle test keeps the point (PR:125-134), found by binary search
//                       on per-tile bound tables computed with the reference's expressions
//   P1                  count -> scan -> fill into exact-size bin lists (the face coarse stage's kernels: a point's
//                       tile range is handed over as a pixel range)
//   P2 k_points_fine    one CTA per (cloud, bin, <=16x16 pixel block), one thread per pixel; the bin's points are
//                       staged through shared memory 256 at a time and each pixel keeps its K nearest (z, id) in
//                       registers (PR:140-148, PixelHeap PR:44-58); dists2 is recomputed at emit with the same ops
//   P3 k_points_backward per occupied slot: d points_ndc += (-2 (px - x) g_d, -2 (py - y) g_d, g_z), warp-aggregated
//                       fp64 atomics per point
//
// Exactness: selection and payload use the reference's operations in its order (Vec2 `pix - xy`, norm2, `<= r2`),
// compiled with -fmad=false, so idx / zbuf / dists2 are bit-identical to the reference (fp64 entry point).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdint>

#include "raster_kernels.cuh"
#include "raster_math.cuh"

namespace drb {

// ------------------------------------------------------------------------------------------------
// tile bound tables (PR:125-132): x bounds per tile column, y bounds per tile row

__global__ void k_point_tile_bounds(int H, int W, int ts, int nbx, int nby, double radius, double* __restrict__ bx_min,
                                    double* __restrict__ bx_max, double* __restrict__ by_min,
                                    double* __restrict__ by_max) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < nbx) {
    const int j0 = t * ts, j1 = min(W, j0 + ts) - 1;
    const double tl = pixel_x(W, j0), br = pixel_x(W, j1);
    bx_min[t] = (tl < br ? tl : br) - radius;  // std::min(tl.x, br.x) - s.radius
    bx_max[t] = (tl < br ? br : tl) + radius;  // std::max(tl.x, br.x) + s.radius
  }
  if (t < nby) {
    const int i0 = t * ts, i1 = min(H, i0 + ts) - 1;
    const double tl = pixel_y(H, i0), br = pixel_y(H, i1);
    by_min[t] = (tl < br ? tl : br) - radius;
    by_max[t] = (tl < br ? br : tl) + radius;
  }
}

// ------------------------------------------------------------------------------------------------
// P0: point setup. A point is kept in tile (tx, ty) iff !(x < bx_min || x > bx_max || y < by_min || y > by_max)
// (PR:133-134). bx_min/bx_max grow with tx and by_min/by_max shrink with ty, so the kept tiles form a rectangle.

__global__ void __launch_bounds__(256) k_point_setup(const double* __restrict__ pts, int64_t p_lo, int64_t p_hi,
                                                     int ts, int nbx, int nby, double znear, int clip_z,
                                                     const double* __restrict__ bx_min,
                                                     const double* __restrict__ bx_max,
                                                     const double* __restrict__ by_min,
                                                     const double* __restrict__ by_max, int4* __restrict__ ibbox,
                                                     float* __restrict__ zkey) {
  const int64_t p = p_lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= p_hi) return;
  const double x = pts[3 * p], y = pts[3 * p + 1], z = pts[3 * p + 2];
  int4 out = make_int4(1, 0, 1, 0);  // empty
  bool keep = isfinite(x) && isfinite(y) && isfinite(z);  // a NaN point never passes d2 <= r2 (PR:145)
  if (clip_z && !(z > 0)) keep = false;                   // NdcPoint.clipped (camera.cpp:44-47)
  if (z < znear) keep = false;                            // PR:26
  if (keep) {
    // first tx with x <= bx_max[tx]; last tx with bx_min[tx] <= x
    int lo = 0, hi = nbx;
    while (lo < hi) {
      const int m = (lo + hi) >> 1;
      if (bx_max[m] < x) lo = m + 1; else hi = m;
    }
    const int tx0 = lo;
    lo = -1;
    hi = nbx - 1;
    while (lo < hi) {
      const int m = (lo + hi + 1) >> 1;
      if (bx_min[m] <= x) lo = m; else hi = m - 1;
    }
    const int tx1 = lo;
    // first ty with by_min[ty] <= y; last ty with y <= by_max[ty]
    lo = 0;
    hi = nby;
    while (lo < hi) {
      const int m = (lo + hi) >> 1;
      if (by_min[m] > y) lo = m + 1; else hi = m;
    }
    const int ty0 = lo;
    lo = -1;
    hi = nby - 1;
    while (lo < hi) {
      const int m = (lo + hi + 1) >> 1;
      if (y <= by_max[m]) lo = m; else hi = m - 1;
    }
    const int ty1 = lo;
    if (tx0 <= tx1 && ty0 <= ty1) out = make_int4(ty0 * ts, ty1 * ts, tx0 * ts, tx1 * ts);  // as pixel ranges
  }
  ibbox[p] = out;
  zkey[p] = keep ? __double2float_rd(z) : __int_as_float(0x7f800000);  // <= z: a point's depth IS its candidate z
}

// ------------------------------------------------------------------------------------------------
// P2: fine stage

constexpr int kPtThreads = 256;  // one thread per pixel of a <= 16x16 block
constexpr int kPtTab = 2048;     // backward pixel-centre table (W + H entries)

__device__ __forceinline__ bool pt_less(double za, int32_t ia, double zb, int32_t ib) {  // PR:37
  return za != zb ? za < zb : ia < ib;
}

constexpr int kPtMaxK = 128;  // points_per_pixel limit of the generic (local-memory list) instantiation

template <typename OutT, int KMAX>
__global__ void __launch_bounds__(kPtThreads) k_points_fine(PointFineArgs<OutT> A) {
  __shared__ double sx[kPtThreads], sy[kPtThreads], sz[kPtThreads];
  __shared__ int32_t sid[kPtThreads];
  __shared__ double s_kth[kPtThreads / 32];
  __shared__ uint16_t s_wl[kPtThreads / 32][kPtThreads];  // per warp: staged points that can reach its two rows
  // per-pixel sorted (z, id) list: KMAX > 0 => registers (fully unrolled, +inf padded), else local memory
  constexpr int KL = KMAX > 0 ? KMAX : kPtMaxK;
  double lz[KL];
  int32_t lid[KL];
  const int K = A.K;
  const int nbins = A.nbx * A.nby;
  const int subs = A.sub_x * A.sub_y;
  const int64_t n_items = (int64_t)A.N * nbins * subs;
  for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int sub = (int)(item % subs);
    const int64_t bb = item / subs;
    const int bin = (int)(bb % nbins);
    const int b = (int)(bb / nbins);
    const int by = bin / A.nbx, bx = bin % A.nbx;
    const int bi0 = by * A.bs + (sub / A.sub_x) * 16, bj0 = bx * A.bs + (sub % A.sub_x) * 16;
    const int bi1 = min(min(A.H, by * A.bs + A.bs), bi0 + 16), bj1 = min(min(A.W, bx * A.bs + A.bs), bj0 + 16);
    if (bi0 >= bi1 || bj0 >= bj1) continue;
    const int i = bi0 + (int)(threadIdx.x >> 4), j = bj0 + (int)(threadIdx.x & 15);
    const bool valid = i < bi1 && j < bj1;
    const double px = pixel_x(A.W, j), py = pixel_y(A.H, i);  // pixel_center_ndc (camera.cpp:100-102)
    // the warp's two pixel rows (threads 16r .. 16r+15 hold row r of the block)
    const int wi0 = bi0 + 2 * (int)(threadIdx.x >> 5);
    const double wpy0 = pixel_y(A.H, wi0), wpy1 = pixel_y(A.H, wi0 + 1);
    // candidate points: the bin list, or the whole cloud (naive / spilled bin)
    const int64_t p0 = A.first[b], np = A.num[b];
    const int4* list = nullptr;
    bool sorted = false;
    int64_t nsrc = np;
    if (A.binned) {
      const int64_t gb = (int64_t)b * nbins + bin;
      const int c = A.bin_counts[gb];
      const int64_t o = A.bin_off[gb];
      if (bin_fits(o, c, A.pool, 0)) {
        list = A.bin_entries + o;
        nsrc = c;
        sorted = A.sorted && bin_is_sorted(o, c, A.pool, 0);  // longer bins stay unsorted (k_sort_bins)
      }
    }
    int n = 0;  // candidates held (generic path)
    if constexpr (KMAX > 0) {
#pragma unroll
      for (int s = 0; s < KMAX; ++s) {
        lz[s] = __longlong_as_double(0x7ff0000000000000LL);
        lid[s] = INT_MAX;
      }
    }
    for (int64_t c0 = 0; c0 < nsrc; c0 += kPtThreads) {
      // depth-ordered bin: once every pixel of the block holds K points nearer than a lower bound of every
      // remaining depth key, no later point can enter any list (strict (z, id) order, PR:37). The bound is the
      // lower edge of the bucket two below the next entry's (rounding in the float bucket map stays under one
      // bucket width); the sort wrote this bin's bucket map because bin_is_sorted holds for it
      if (sorted) {
        double kth = -__longlong_as_double(0x7ff0000000000000LL);
        if (valid) {
          if constexpr (KMAX > 0) kth = lz[KMAX - 1];  // >= the K-th depth (== it when K == KMAX)
          else kth = n < K ? __longlong_as_double(0x7ff0000000000000LL) : lz[K - 1];
        }
        for (int d = 16; d >= 1; d >>= 1) kth = fmax(kth, __shfl_xor_sync(0xffffffffu, kth, d));
        __syncthreads();
        if ((threadIdx.x & 31) == 0) s_kth[threadIdx.x >> 5] = kth;
        __syncthreads();
        double T = s_kth[0];
        for (int w = 1; w < kPtThreads / 32; ++w) T = fmax(T, s_kth[w]);
        const float key = __int_as_float(list[c0].y);
        // the sort's bucket map (lo, scale) of this bin, loaded here: nothing stays live
        const float2 br = A.brange[(int64_t)b * nbins + bin];
        const int bk = sort_bucket(key, br.x, br.y);
        // lo + (bk - 2) / scale with both roundings downward: a lower bound of every key in buckets >= bk
        const double bound =
            br.y > 0.f && bk >= 2 ? (double)__fadd_rd(br.x, __fdiv_rd((float)(bk - 2), br.y)) : (double)br.x;
        if (bound > T) break;
      }
      __syncthreads();
      const int64_t ci = c0 + threadIdx.x;
      if (ci < nsrc) {
        int32_t pid;
        bool live = true;
        if (list) {
          pid = list[ci].x;
        } else {
          pid = (int32_t)(p0 + ci);
          if (A.binned) {  // spilled bin: the point must pass this tile's inflated bounds test (PR:133-134)
            const int4 ib = A.ibbox[pid];  // kept tiles as pixel ranges (multiples of bs)
            const int ti = by * A.bs, tj = bx * A.bs;
            live = ib.x <= ti && ti <= ib.y && ib.z <= tj && tj <= ib.w;
          } else {  // rasterize_points_naive has no tile test: prepare_points liveness only (PR:17-31, 82-103)
            live = A.zkey[pid] != __int_as_float(0x7f800000);
          }
        }
        sx[threadIdx.x] = A.pts[3 * (int64_t)pid];
        sy[threadIdx.x] = A.pts[3 * (int64_t)pid + 1];
        sz[threadIdx.x] = A.pts[3 * (int64_t)pid + 2];
        sid[threadIdx.x] = live ? pid : -1;
      }
      __syncthreads();
      const int m = (int)(nsrc - c0 < kPtThreads ? nsrc - c0 : kPtThreads);
      // warp filter: a staged point can pass PR:145 at one of the warp's pixels only if its own y term alone does:
      // the test's d2 = fl(fl(vx * vx) + fl(vy * vy)) >= fl(vy * vy) (rounding is monotone, vx * vx >= 0), and vy is
      // computed here exactly as the test computes it. The warp then walks only those points (~1/4 of the batch
      // for a radius of a pixel or two in a 16-row block) instead of all of them.
      int wn = 0;
      uint16_t* wl = s_wl[threadIdx.x >> 5];
      {
        const int lane = threadIdx.x & 31;
        for (int q0 = 0; q0 < m; q0 += 32) {
          const int q = q0 + lane;
          bool keep = false;
          if (q < m && sid[q] >= 0) {
            const double vy0 = wpy0 - sy[q], vy1 = wpy1 - sy[q];
            keep = vy0 * vy0 <= A.r2 || vy1 * vy1 <= A.r2;
          }
          const unsigned kb = __ballot_sync(0xffffffffu, keep);
          if (keep) wl[wn + __popc(kb & ((1u << lane) - 1u))] = (uint16_t)q;
          wn += __popc(kb);
        }
        __syncwarp();
      }
      if (valid) {
        for (int k = 0; k < wn; ++k) {
          const int q = wl[k];
          const int32_t pid = sid[q];
          const double vx = px - sx[q], vy = py - sy[q];  // pix - pr.xy
          const double d2 = vx * vx + vy * vy;            // Vec2::norm2 (core.hpp:66)
          if (pid < 0 || !(d2 <= A.r2)) continue;         // PR:145
          const double zc = sz[q];
          // sorted insertion (the K smallest under (z, id) are order-independent, PR:37-58)
          if constexpr (KMAX > 0) {
            if (!pt_less(zc, pid, lz[KMAX - 1], lid[KMAX - 1])) continue;
#pragma unroll
            for (int s = KMAX - 1; s >= 0; --s) {
              const int sp = s > 0 ? s - 1 : 0;
              const bool lt_prev = s > 0 && pt_less(zc, pid, lz[sp], lid[sp]);
              if (lt_prev) {
                lz[s] = lz[sp];
                lid[s] = lid[sp];
              } else if (pt_less(zc, pid, lz[s], lid[s])) {
                lz[s] = zc;
                lid[s] = pid;
              }
            }
          } else {
            if (n == K && !pt_less(zc, pid, lz[K - 1], lid[K - 1])) continue;
            int s = n < K ? n : K - 1;
            if (n < K) ++n;
            while (s > 0 && pt_less(zc, pid, lz[s - 1], lid[s - 1])) {
              lz[s] = lz[s - 1];
              lid[s] = lid[s - 1];
              --s;
            }
            lz[s] = zc;
            lid[s] = pid;
          }
        }
      }
    }
    if (valid) {  // emit_pixel (PR:71-80); empty slots: alloc_fragments (PR:60-69)
      const int64_t slot0 = (((int64_t)b * A.H + i) * A.W + j) * K;
      auto emit = [&](int s, double z, int32_t pid, bool occ) {
        if (occ) {
          const double vx = px - A.pts[3 * (int64_t)pid], vy = py - A.pts[3 * (int64_t)pid + 1];
          A.idx[slot0 + s] = pid;
          A.zbuf[slot0 + s] = (OutT)z;
          A.dists2[slot0 + s] = (OutT)(vx * vx + vy * vy);  // the bits the selection compared
        } else {
          A.idx[slot0 + s] = -1;
          A.zbuf[slot0 + s] = (OutT)-1.0;
          A.dists2[slot0 + s] = (OutT)0.0;
        }
      };
      if constexpr (KMAX > 0) {
#pragma unroll
        for (int s = 0; s < KMAX; ++s)
          if (s < K) emit(s, lz[s], lid[s], lid[s] != INT_MAX);
      } else {
        for (int s = 0; s < K; ++s) emit(s, s < n ? lz[s] : 0.0, s < n ? lid[s] : -1, s < n);
      }
    }
  }
}

// ------------------------------------------------------------------------------------------------
// P3: backward of (zbuf, dists2) to points_ndc

template <typename InT>
__global__ void __launch_bounds__(256) k_points_backward(const double* __restrict__ pts, const int64_t* __restrict__ idx,
                                                         const InT* __restrict__ g_zbuf,
                                                         const InT* __restrict__ g_dists2, int64_t S, int64_t P, int H,
                                                         int W, int K, double* __restrict__ grad, FastDivU32 divK,
                                                         FastDivU32 divHW, FastDivU32 divW) {
  // pixel centres from a shared table (pixel_x(W, j) for j < W, then pixel_y(H, i)) and slot -> (pixel, i, j) by
  // precomputed reciprocals when the indices fit 32 bits: no 64-bit divisions and no fp64 division per slot
  __shared__ double tab[kPtTab];
  const bool use_tab = W + H <= kPtTab;
  if (use_tab)
    for (int t = threadIdx.x; t < W + H; t += blockDim.x) tab[t] = t < W ? pixel_x(W, t) : pixel_y(H, t - W);
  __syncthreads();
  const bool s32 = S <= 0xffffffffll;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < S; base += stride) {
    const int64_t slot = base + threadIdx.x;
    int32_t pid = -1;
    double g[3] = {0.0, 0.0, 0.0};
    if (slot < S) {
      const int64_t p = idx[slot];
      if (p >= 0 && p < P) {
        pid = (int32_t)p;
        int i, j;
        if (s32) {
          const uint32_t pix = divK.div((uint32_t)slot);
          const uint32_t rem = pix - divHW.div(pix) * divHW.d;
          i = (int)divW.div(rem);
          j = (int)rem - i * W;
        } else {
          const int64_t pix = slot / K;
          const int rem = (int)(pix % ((int64_t)H * W));
          i = rem / W;
          j = rem - i * W;
        }
        const double gd = (double)g_dists2[slot];
        const double cx = use_tab ? tab[j] : pixel_x(W, j), cy = use_tab ? tab[W + i] : pixel_y(H, i);
        g[0] = -2.0 * (cx - pts[3 * p]) * gd;      // d|pix - xy|^2 / dx
        g[1] = -2.0 * (cy - pts[3 * p + 1]) * gd;
        g[2] = (double)g_zbuf[slot];                          // zbuf = z_view
      }
    }
    // lanes of the warp hitting the same point: shuffle-sum, one lane issues the atomics
    const int key = pid >= 0 ? pid : -1 - lane;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    unsigned rel = __popc(peers & ((1u << lane) - 1u));
    unsigned rem_p = peers & ~((2u << lane) - 1u);
    while (__any_sync(0xffffffffu, rem_p != 0)) {
      const int next = __ffs(rem_p);
      const int src = next ? next - 1 : lane;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double t = __shfl_sync(0xffffffffu, g[k], src);
        if (next) g[k] += t;
      }
      rem_p &= ~__ballot_sync(0xffffffffu, rel & 1u);
      rel >>= 1;
    }
    if (pid >= 0 && (peers & ((1u << lane) - 1u)) == 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (g[k] != 0.0) atomicAdd(grad + 3 * (int64_t)pid + k, g[k]);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// launchers

cudaError_t launch_point_setup(const double* pts, int64_t p_lo, int64_t p_hi, int H, int W, int ts, int nbx, int nby,
                               double radius, double znear, int clip_z, double* bounds, int4* ibbox, float* zkey,
                               cudaStream_t st) {
  const int nt = std::max(nbx, nby);
  double* bx_min = bounds;
  double* bx_max = bounds + nbx;
  double* by_min = bounds + 2 * nbx;
  double* by_max = bounds + 2 * nbx + nby;
  k_point_tile_bounds<<<(nt + 255) / 256, 256, 0, st>>>(H, W, ts, nbx, nby, radius, bx_min, bx_max, by_min, by_max);
  if (p_hi > p_lo)
    k_point_setup<<<(unsigned)((p_hi - p_lo + 255) / 256), 256, 0, st>>>(pts, p_lo, p_hi, ts, nbx, nby, znear, clip_z,
                                                                         bx_min, bx_max, by_min, by_max, ibbox,
                                                                         zkey);
  return cudaGetLastError();
}

template <typename OutT>
static cudaError_t launch_points_fine_t(const PointFineArgs<OutT>& A, cudaStream_t st) {
  const int64_t items = (int64_t)A.N * A.nbx * A.nby * A.sub_x * A.sub_y;
  if (items <= 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<int64_t>(items, 148 * 32);
  if (A.K == 1) k_points_fine<OutT, 1><<<grid, kPtThreads, 0, st>>>(A);
  else if (A.K <= 8) k_points_fine<OutT, 8><<<grid, kPtThreads, 0, st>>>(A);
  else if (A.K <= 16) k_points_fine<OutT, 16><<<grid, kPtThreads, 0, st>>>(A);
  else k_points_fine<OutT, 0><<<grid, kPtThreads, 0, st>>>(A);
  return cudaGetLastError();
}

cudaError_t launch_points_fine(const PointFineArgs<float>& A, cudaStream_t st) { return launch_points_fine_t(A, st); }
cudaError_t launch_points_fine(const PointFineArgs<double>& A, cudaStream_t st) { return launch_points_fine_t(A, st); }

template <typename InT>
static cudaError_t launch_points_backward_t(const double* pts, const int64_t* idx, const InT* gz, const InT* gd,
                                            int64_t S, int64_t P, int H, int W, int K, double* grad,
                                            cudaStream_t st) {
  if (S <= 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<int64_t>((S + 255) / 256, 148 * 16);
  const bool s32 = S <= 0xffffffffll;  // the kernel's 32-bit path (then H * W < 2^32 as well)
  k_points_backward<InT><<<grid, 256, 0, st>>>(pts, idx, gz, gd, S, P, H, W, K, grad,
                                                s32 ? FastDivU32((uint32_t)K) : FastDivU32(),
                                                s32 ? FastDivU32((uint32_t)((int64_t)H * W)) : FastDivU32(),
                                                s32 ? FastDivU32((uint32_t)W) : FastDivU32());
  return cudaGetLastError();
}
cudaError_t launch_points_backward(const double* pts, const int64_t* idx, const float* gz, const float* gd, int64_t S,
                                   int64_t P, int H, int W, int K, double* grad, cudaStream_t st) {
  return launch_points_backward_t(pts, idx, gz, gd, S, P, H, W, K, grad, st);
}
cudaError_t launch_points_backward(const double* pts, const int64_t* idx, const double* gz, const double* gd,
                                   int64_t S, int64_t P, int H, int W, int K, double* grad, cudaStream_t st) {
  return launch_points_backward_t(pts, idx, gz, gd, S, P, H, W, K, grad, st);
}

}  // namespace drb
