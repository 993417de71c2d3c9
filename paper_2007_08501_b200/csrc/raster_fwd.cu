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

#include "raster_kernels.cuh"
#include "raster_math.cuh"

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

__global__ void __launch_bounds__(256) k_face_setup(const double* __restrict__ fv, int64_t F, int H, int W,
                                                    double inflate, double znear, int clip_nonpositive_z,
                                                    int cull_backfaces, int4* __restrict__ ibbox) {
  int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const double* p = fv + 9 * f;
  double v[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) v[k] = __ldg(p + k);
  int4 out = make_int4(1, 0, 1, 0);  // empty
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
    }
  }
  ibbox[f] = out;
}

// ------------------------------------------------------------------------------------------------
// K1: coarse binning. Each warp walks 32 consecutive faces of one mesh; the bins a face touches form a
// rectangle of the bin grid. Lanes that target the same bin in the same round are grouped with
// __match_any_sync and reserve their slots with ONE atomicAdd (leader), so adjacent faces of a mesh
// (which mostly share bins) cost one global atomic per (warp, bin). Order inside a bin is irrelevant:
// the K smallest under the strict total order (z, id) do not depend on it (MR:138-140).

__global__ void __launch_bounds__(256) k_bin_faces(const int4* __restrict__ ibbox, const int64_t* __restrict__ first,
                                                   const int64_t* __restrict__ num, int bs, int nbx, int nby, int cap,
                                                   int* __restrict__ counts, int32_t* __restrict__ lists) {
  const int b = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int64_t nf = num[b], f0 = first[b];
  const int nbins = nbx * nby;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int* cnt = counts + (int64_t)b * nbins;
  int32_t* lst = lists + (int64_t)b * nbins * cap;
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
      int base_slot = 0;
      if (active && lane == leader) base_slot = atomicAdd(cnt + key, __popc(peers));
      base_slot = __shfl_sync(0xffffffffu, base_slot, leader);
      if (active && base_slot + rank < cap) lst[(int64_t)key * cap + base_slot + rank] = (int32_t)(f0 + lf);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// K2: fine rasterization

// Staged face: geometry + invariants (FaceGeom) + integer pixel range. Every lane of a warp reads the same
// record at the same time (shared-memory broadcast), so array-of-structs costs no bank conflicts.
struct __align__(16) StagedFace {
  double ax, ay, bx, by, cx, cy;
  double z0, z1, z2;
  double abx, aby, bcx, bcy, cax, cay;
  double lab, lbc, lca;
  double area;
  int32_t fid;
  int32_t _pad;
  int4 ib;
};

__device__ __forceinline__ void stage_face(StagedFace& s, const double* fv, int32_t fid, int4 ib) {
  double v[9];
  const double* p = fv + 9 * (int64_t)fid;
#pragma unroll
  for (int k = 0; k < 9; ++k) v[k] = __ldg(p + k);
  FaceGeom g = make_face_geom(v);
  s.ax = g.a.x; s.ay = g.a.y; s.bx = g.b.x; s.by = g.b.y; s.cx = g.c.x; s.cy = g.c.y;
  s.z0 = g.z0; s.z1 = g.z1; s.z2 = g.z2;
  s.abx = g.ab.x; s.aby = g.ab.y; s.bcx = g.bc.x; s.bcy = g.bc.y; s.cax = g.ca.x; s.cay = g.ca.y;
  s.lab = g.len_ab; s.lbc = g.len_bc; s.lca = g.len_ca;
  s.area = g.area;
  s.fid = fid;
  s.ib = ib;
}

__device__ __forceinline__ FaceGeom load_geom(const StagedFace& s) {
  FaceGeom g;
  g.a = V2{s.ax, s.ay}; g.b = V2{s.bx, s.by}; g.c = V2{s.cx, s.cy};
  g.z0 = s.z0; g.z1 = s.z1; g.z2 = s.z2;
  g.ab = V2{s.abx, s.aby}; g.bc = V2{s.bcx, s.bcy}; g.ca = V2{s.cax, s.cay};
  g.len_ab = s.lab; g.len_bc = s.lbc; g.len_ca = s.lca;
  g.area = s.area;
  return g;
}

// Register-resident bounded sorted list of the K smallest (z, id) keys, KMAX >= K at compile time.
// Unused slots hold the sentinel (+inf, INT_MAX), which compares greater than any real candidate; all
// indexing is compile-time (fully unrolled) so the list never spills to local memory.
template <int KMAX>
struct RegTopK {
  double z[KMAX];
  int32_t id[KMAX];
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int s = 0; s < KMAX; ++s) {
      z[s] = __longlong_as_double(0x7ff0000000000000LL);
      id[s] = INT_MAX;
    }
  }
  // insertion into a sorted array, walking from the tail: slot s takes slot s-1 if the candidate sorts
  // before it, else the candidate if it sorts before the old slot s. Slots >= K are never written.
  __device__ __forceinline__ void insert(double zc, int32_t ic, int K) {
#pragma unroll
    for (int s = KMAX - 1; s >= 0; --s) {
      if (s < K) {
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
  }
};

// Shared-memory bounded sorted list (large K): column `tid` of [K][nthreads] arrays.
struct SmemTopK {
  double* z;
  int32_t* id;
  int stride;
  int n;
  __device__ __forceinline__ void reset() { n = 0; }
  __device__ __forceinline__ void insert(double zc, int32_t ic, int K) {
    int m = n;
    if (m == K) {
      if (!cand_less(zc, ic, z[(K - 1) * stride], id[(K - 1) * stride])) return;
      m = K - 1;
    }
    int pos = m;
    while (pos > 0) {
      double zp = z[(pos - 1) * stride];
      int32_t ip = id[(pos - 1) * stride];
      if (!cand_less(zc, ic, zp, ip)) break;
      z[pos * stride] = zp;
      id[pos * stride] = ip;
      --pos;
    }
    z[pos * stride] = zc;
    id[pos * stride] = ic;
    n = m + 1;
  }
};

template <typename OutT>
__device__ __forceinline__ void emit_slot(const FineArgs<OutT>& A, int64_t slot, bool occupied, double z,
                                          int32_t fid, double px, double py) {
  if (occupied) {
    double v[9];
    const double* p = A.fv + 9 * (int64_t)fid;
#pragma unroll
    for (int k = 0; k < 9; ++k) v[k] = __ldg(p + k);
    FaceGeom g = make_face_geom(v);
    PixelFaceResult r;
    eval_pixel_face<true>(V2{px, py}, g, A.blur, A.znear, A.persp, A.clip, r);  // same ops => same bits
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

// emit_pixel (MR:178-197): slots in ascending (z, id); bary/dists of the winners are recomputed with the
// identical operation sequence, so they carry the bits the candidate test produced.
template <typename OutT, int KMAX>
__device__ __forceinline__ void emit_pixel(const FineArgs<OutT>& A, const RegTopK<KMAX>& tk, int b, int i, int j,
                                           double px, double py) {
  const int64_t slot0 = (((int64_t)b * A.H + i) * A.W + j) * A.K;
#pragma unroll
  for (int s = 0; s < KMAX; ++s)
    if (s < A.K) emit_slot<OutT>(A, slot0 + s, tk.id[s] != INT_MAX, tk.z[s], tk.id[s], px, py);
}
template <typename OutT>
__device__ __forceinline__ void emit_pixel(const FineArgs<OutT>& A, const SmemTopK& tk, int b, int i, int j,
                                           double px, double py) {
  const int64_t slot0 = (((int64_t)b * A.H + i) * A.W + j) * A.K;
  for (int s = 0; s < A.K; ++s) {
    const bool occ = s < tk.n;
    emit_slot<OutT>(A, slot0 + s, occ, occ ? tk.z[s * tk.stride] : 0.0, occ ? tk.id[s * tk.stride] : -1, px, py);
  }
}

// One CTA per (mesh b, bin). The bin is covered by sub-tiles of stw x sth pixels; each warp owns an 8x4
// micro-tile of the sub-tile (compact footprint => lanes share the faces they test). For every sub-tile the
// CTA streams its candidate faces through shared memory in chunks of blockDim faces, keeping only those
// whose integer pixel range meets the sub-tile (ballot + popc compaction), then every lane tests the staged
// faces against its pixel and keeps its top-K.
template <typename OutT, typename TopK, int KMAX>
__global__ void __launch_bounds__(256) k_fine(FineArgs<OutT> A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  StagedFace* staged = reinterpret_cast<StagedFace*>(smem_raw);
  __shared__ int warp_cnt[8];

  const int nbins = A.nbx * A.nby;
  const int b = blockIdx.x / nbins;
  const int bin = blockIdx.x % nbins;
  const int by = bin / A.nbx, bx = bin % A.nbx;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nthreads = blockDim.x;
  const int nwarps = nthreads >> 5;

  // bin pixel rectangle (clipped to the image)
  const int bi0 = by * A.bs, bj0 = bx * A.bs;
  const int bi1 = min(A.H, bi0 + A.bs) - 1, bj1 = min(A.W, bj0 + A.bs) - 1;

  // candidate face source
  const int64_t f0 = A.first[b], nf = A.num[b];
  const int32_t* list = nullptr;
  int64_t nsrc = nf;
  if (A.binned) {
    int c = A.bin_counts[(int64_t)b * nbins + bin];
    if (c <= A.cap) {
      list = A.bin_lists + ((int64_t)b * nbins + bin) * A.cap;
      nsrc = c;
    }
  }

  TopK tk;
  if constexpr (KMAX == 0) {
    double* zs = reinterpret_cast<double*>(smem_raw + A.staged_bytes);
    tk.z = zs + tid;
    tk.id = reinterpret_cast<int32_t*>(zs + (size_t)A.K * nthreads) + tid;
    tk.stride = nthreads;
  }

  const int mt_w = A.stw >> 3;  // micro-tiles per sub-tile row
  for (int si = bi0; si <= bi1; si += A.sth) {
    for (int sj = bj0; sj <= bj1; sj += A.stw) {
      const int si1 = min(bi1, si + A.sth - 1), sj1 = min(bj1, sj + A.stw - 1);
      const int i = si + (wid / mt_w) * 4 + (lane >> 3);
      const int j = sj + (wid % mt_w) * 8 + (lane & 7);
      const bool valid = i <= si1 && j <= sj1;
      const double px = pixel_x(A.W, j), py = pixel_y(A.H, i);
      tk.reset();

      for (int64_t c0 = 0; c0 < nsrc; c0 += nthreads) {
        // ---- stage: filter candidates against the sub-tile, compact, load geometry
        const int64_t ci = c0 + tid;
        int32_t fid = -1;
        int4 ib = make_int4(1, 0, 1, 0);
        if (ci < nsrc) {
          fid = list ? list[ci] : (int32_t)(f0 + ci);
          ib = A.ibbox[fid];
        }
        const bool keep = ib.x <= ib.y && ib.y >= si && ib.x <= si1 && ib.w >= sj && ib.z <= sj1;
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) warp_cnt[wid] = __popc(bal);
        __syncthreads();
        int off = 0, tot = 0;
        for (int w = 0; w < nwarps; ++w) {
          int cw = warp_cnt[w];
          off += w < wid ? cw : 0;
          tot += cw;
        }
        if (keep) stage_face(staged[off + __popc(bal & ((1u << lane) - 1u))], A.fv, fid, ib);
        __syncthreads();
        // ---- test the staged faces against this lane's pixel
        if (valid) {
          for (int k = 0; k < tot; ++k) {
            const int4 fb = staged[k].ib;
            if (i < fb.x || i > fb.y || j < fb.z || j > fb.w) continue;
            const FaceGeom g = load_geom(staged[k]);
            PixelFaceResult r;
            if (eval_pixel_face<false>(V2{px, py}, g, A.blur, A.znear, A.persp, A.clip, r))
              tk.insert(r.z, staged[k].fid, A.K);
          }
        }
        __syncthreads();
      }
      if (valid) emit_pixel(A, tk, b, i, j, px, py);
    }
  }
}

// ------------------------------------------------------------------------------------------------
// host-side launchers (called from capi.cu)

void launch_face_setup(const double* fv, int64_t F, int H, int W, double inflate, double znear, int clip_z,
                       int cull, int4* ibbox, cudaStream_t st) {
  if (F <= 0) return;
  unsigned grid = (unsigned)((F + 255) / 256);
  k_face_setup<<<grid, 256, 0, st>>>(fv, F, H, W, inflate, znear, clip_z, cull, ibbox);
}

void launch_bin_faces(const int4* ibbox, const int64_t* first, const int64_t* num, int64_t N, int64_t max_faces,
                      int bs, int nbx, int nby, int cap, int* counts, int32_t* lists, cudaStream_t st) {
  if (max_faces <= 0) return;
  unsigned gx = (unsigned)std::min<int64_t>((max_faces + 255) / 256, 65535);
  dim3 grid(gx, (unsigned)N);
  k_bin_faces<<<grid, 256, 0, st>>>(ibbox, first, num, bs, nbx, nby, cap, counts, lists);
}

template <typename OutT>
static cudaError_t launch_fine_t(const FineArgs<OutT>& A, int64_t nblocks, cudaStream_t st) {
  const int nthreads = (A.stw / 8) * (A.sth / 4) * 32;
  size_t smem = A.staged_bytes;
  const int K = A.K;
  auto go = [&](auto kern, size_t extra) -> cudaError_t {
    size_t total = smem + extra;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)total);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)nblocks, nthreads, total, st>>>(A);
    return cudaGetLastError();
  };
  if (K <= 1) return go(k_fine<OutT, RegTopK<1>, 1>, 0);
  if (K <= 2) return go(k_fine<OutT, RegTopK<2>, 2>, 0);
  if (K <= 4) return go(k_fine<OutT, RegTopK<4>, 4>, 0);
  if (K <= 8) return go(k_fine<OutT, RegTopK<8>, 8>, 0);
  if (K <= 16) return go(k_fine<OutT, RegTopK<16>, 16>, 0);
  return go(k_fine<OutT, SmemTopK, 0>, (size_t)K * nthreads * (sizeof(double) + sizeof(int32_t)));
}

cudaError_t launch_fine(const FineArgs<float>& A, int64_t nblocks, cudaStream_t st) {
  return launch_fine_t(A, nblocks, st);
}
cudaError_t launch_fine(const FineArgs<double>& A, int64_t nblocks, cudaStream_t st) {
  return launch_fine_t(A, nblocks, st);
}

size_t staged_face_bytes() { return sizeof(StagedFace); }

}  // namespace drb
