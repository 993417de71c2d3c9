// C-ABI of libdr_raster_b200.so (include/dr_raster.h): validation, workspace planning, launch sequence,
// error reporting, launch counting and optional per-kernel event timing.
//
// Error behaviour mirrors the reference's exceptions as status codes:
//   empty batch                          -> DR_ERR_SHAPE (MeshBatch ctor "empty mesh batch", batching.cpp:14)
//   negative face counts                 -> DR_ERR_SHAPE
//   mesh face range outside [0, F)       -> DR_ERR_INDEX (cf. IndexError, batching.cpp:17-21)
//   image size / K / bin size out of range -> DR_ERR_RANGE
//   null pointers / short workspace      -> DR_ERR_USAGE / DR_ERR_OOM
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dr_raster.h"
#include "raster_kernels.cuh"

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(DR_ERR_CUDA, "CUDA error in %s: %s", where, cudaGetErrorString(e));
}

// ---- optional per-kernel timing ring ----
const char* kKernelNames[] = {"k_face_setup",  "k_bin_faces",   "k_fine",        "k_backward",
                              "memset",        "k_camera",      "k_batching",    "k_sort_bins",
                              "k_silhouette_backward", "k_point_setup", "k_points_fine", "k_points_backward",
                              "k_softmax_backward"};
enum {
  KN_SETUP = 0, KN_BIN = 1, KN_FINE = 2, KN_BWD = 3, KN_MEMSET = 4, KN_CAMERA = 5, KN_BATCH = 6, KN_SORT = 7,
  KN_SIL_BWD = 8, KN_PT_SETUP = 9, KN_PT_FINE = 10, KN_PT_BWD = 11, KN_SOFT_BWD = 12
};
struct ProfEntry {
  int kernel;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
std::atomic<bool> g_prof_on{false};
std::vector<ProfEntry> g_prof;

struct ProfScope {
  cudaStream_t st;
  int kernel;
  cudaEvent_t a = nullptr, b = nullptr;
  ProfScope(cudaStream_t s, int k) : st(s), kernel(k) {
    if (g_prof_on.load()) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st);
    }
    if (k != KN_MEMSET) g_launches.fetch_add(1);
  }
  ~ProfScope() {
    if (a) {
      cudaEventRecord(b, st);
      std::lock_guard<std::mutex> lk(g_prof_mu);
      g_prof.push_back({kernel, a, b});
    }
  }
};

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

struct Plan {
  int64_t N = 0, F = 0;
  int H = 0, W = 0, K = 0;
  int bs = 0;  // bin side used by the fine stage (16 when naive)
  bool binned = false;
  int nbx = 0, nby = 0, cap = 0;
  bool zsort = false;  // depth-ordered bins + K-th-depth culling (clip_barycentric_coords only)
  int64_t nbins_total = 0, pool = 0;  // N * bins; list-pool capacity (entries)
  size_t off_ibbox = 0, off_zkey = 0, off_counter = 0, off_counts = 0, off_cursor = 0, off_binoff = 0, off_lists = 0,
         total = 0;
};

// list-pool capacity: the workspace is planned before the bin counts exist; 8 entries per face covers every
// benchmark scene (faces touch 1-2 bins on average); bins past the pool take the exact spill path
int64_t pool_entries(int64_t F) { return 8 * F + 65536; }

int make_plan(int64_t N, int64_t F, const dr_raster_settings* s, Plan& p) {
  if (!s) return fail(DR_ERR_USAGE, "settings pointer is null");
  if (N < 1) return fail(DR_ERR_SHAPE, "empty mesh batch (N=%lld)", (long long)N);
  if (N > 65535) return fail(DR_ERR_RANGE, "N=%lld meshes exceeds 65535", (long long)N);
  if (F < 0) return fail(DR_ERR_SHAPE, "negative face count F=%lld", (long long)F);
  if (F > INT32_MAX - 1) return fail(DR_ERR_RANGE, "F=%lld exceeds the int32 face-id range", (long long)F);
  if (s->image_h < 1 || s->image_w < 1 || s->image_h > 32768 || s->image_w > 32768)
    return fail(DR_ERR_RANGE, "image size %dx%d outside [1, 32768]", s->image_h, s->image_w);
  if (s->faces_per_pixel < 1 || s->faces_per_pixel > 1024)
    return fail(DR_ERR_RANGE, "faces_per_pixel=%d outside [1, 1024]", s->faces_per_pixel);
  if (s->bin_size < 0) return fail(DR_ERR_RANGE, "bin_size=%d < 0", s->bin_size);
  if (s->max_faces_per_bin < 0) return fail(DR_ERR_RANGE, "max_faces_per_bin=%d < 0", s->max_faces_per_bin);
  if (std::isnan(s->blur_radius) || std::isnan(s->znear)) return fail(DR_ERR_RANGE, "blur_radius/znear is NaN");
  p.N = N;
  p.F = F;
  p.H = s->image_h;
  p.W = s->image_w;
  p.K = s->faces_per_pixel;
  p.binned = s->bin_size > 0;
  p.bs = p.binned ? s->bin_size : 16;
  p.nbx = (p.W + p.bs - 1) / p.bs;
  p.nby = (p.H + p.bs - 1) / p.bs;
  p.cap = p.binned ? s->max_faces_per_bin : 0;  // 0 = unlimited (the reference's bins are unbounded, MR:244)
  p.zsort = s->clip_barycentric_coords != 0;
  size_t off = 0;
  p.off_ibbox = off;
  off = align_up(off + sizeof(int4) * (size_t)std::max<int64_t>(F, 1));
  p.off_zkey = off;
  off = align_up(off + sizeof(float) * (size_t)std::max<int64_t>(F, 1));
  p.off_counter = off;
  off = align_up(off + sizeof(unsigned long long));
  p.off_counts = off;
  if (p.binned) {
    p.nbins_total = N * (int64_t)p.nbx * p.nby;
    p.pool = pool_entries(F);
    off = align_up(off + sizeof(int) * (size_t)p.nbins_total);
    p.off_cursor = off;
    off = align_up(off + sizeof(int) * (size_t)p.nbins_total);
    p.off_binoff = off;
    off = align_up(off + sizeof(int64_t) * (size_t)p.nbins_total);
    p.off_lists = off;  // 16-byte entries: face id, zkey, packed pixel range
    off = align_up(off + sizeof(int4) * (size_t)p.pool);
  }
  p.total = off;
  return DR_OK;
}

// host copy of the mesh ranges: validation + grid sizing (N is small; one D2H per call)
// `host_first/host_num`: optional host copies of the same arrays (the *_hr entry points); without them the
// device arrays are read back, which synchronises `st`.
int read_ranges(const int64_t* first, const int64_t* num, int64_t N, int64_t F, cudaStream_t st,
                int64_t* max_faces, std::vector<int64_t>* out = nullptr, const int64_t* host_first = nullptr,
                const int64_t* host_num = nullptr) {
  std::vector<int64_t> h(2 * (size_t)N);
  if (host_first && host_num) {
    std::memcpy(h.data(), host_first, sizeof(int64_t) * N);
    std::memcpy(h.data() + N, host_num, sizeof(int64_t) * N);
  } else {
    cudaError_t e = cudaMemcpyAsync(h.data(), first, sizeof(int64_t) * N, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h.data() + N, num, sizeof(int64_t) * N, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "reading mesh_to_face_first_idx / num_faces_per_mesh");
  }
  int64_t mx = 0;
  for (int64_t b = 0; b < N; ++b) {
    int64_t f0 = h[b], n = h[N + b];
    if (n < 0) return fail(DR_ERR_SHAPE, "num_faces_per_mesh[%lld] = %lld < 0", (long long)b, (long long)n);
    if (f0 < 0 || f0 > F || f0 + n > F)
      return fail(DR_ERR_INDEX, "mesh %lld face range [%lld, %lld) outside [0, %lld)", (long long)b, (long long)f0,
                  (long long)(f0 + n), (long long)F);
    mx = std::max(mx, n);
  }
  *max_faces = mx;
  if (out) *out = std::move(h);
  return DR_OK;
}

// The union of the batch's item ranges as sorted, merged [lo, hi) intervals (h = first[N] then num[N]).
std::vector<std::pair<int64_t, int64_t>> merged_ranges(const std::vector<int64_t>& h, int64_t N) {
  std::vector<std::pair<int64_t, int64_t>> iv, out;
  for (int64_t b = 0; b < N; ++b)
    if (h[N + b] > 0) iv.push_back({h[b], h[b] + h[N + b]});
  std::sort(iv.begin(), iv.end());
  for (const auto& x : iv) {
    if (!out.empty() && x.first <= out.back().second) out.back().second = std::max(out.back().second, x.second);
    else out.push_back(x);
  }
  return out;
}

// Zero grad rows (`row` doubles per packed item) on the union of the batch's item ranges only (merged
// intervals), so a caller may run the backward on disjoint groups of one packed buffer concurrently.
cudaError_t zero_rows(double* grad, int row, const std::vector<int64_t>& h, int64_t N, cudaStream_t st) {
  for (const auto& iv : merged_ranges(h, N)) {
    cudaError_t e = cudaMemsetAsync(grad + (int64_t)row * iv.first, 0,
                                    sizeof(double) * row * (size_t)(iv.second - iv.first), st);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// alpha != nullptr selects the fused silhouette emit (p2f optional, zbuf/bary/dists unused)
template <typename OutT>
int fwd_impl(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
             const dr_raster_settings* s, int64_t* p2f, OutT* zbuf, OutT* bary, OutT* dists, void* ws, size_t ws_bytes,
             cudaStream_t st, const int64_t* host_first = nullptr, const int64_t* host_num = nullptr,
             OutT* alpha = nullptr, double sigma = 0.0, OutT* image = nullptr, const drb::BlendArgs* blend = nullptr) {
  Plan p;
  int rc = make_plan(N, F, s, p);
  if (rc) return rc;
  if (!first || !num || (F > 0 && !fv)) return fail(DR_ERR_USAGE, "null input pointer");
  if ((alpha || image) ? false : (!p2f || !zbuf || !bary || !dists)) return fail(DR_ERR_USAGE, "null output pointer");
  if (alpha && !(sigma > 0.0)) return fail(DR_ERR_RANGE, "silhouette sigma must be > 0 (got %g)", sigma);
  if (!ws || ws_bytes < p.total)
    return fail(DR_ERR_OOM, "workspace too small: %zu bytes given, %zu needed", ws_bytes, p.total);
  int64_t max_faces = 0;
  std::vector<int64_t> ranges;
  rc = read_ranges(first, num, N, F, st, &max_faces, &ranges, host_first, host_num);
  if (rc) return rc;

  char* base = static_cast<char*>(ws);
  int4* ibbox = reinterpret_cast<int4*>(base + p.off_ibbox);
  int* counts = reinterpret_cast<int*>(base + p.off_counts);
  int4* entries = reinterpret_cast<int4*>(base + p.off_lists);
  int* cursor = reinterpret_cast<int*>(base + p.off_cursor);
  int64_t* bin_off = reinterpret_cast<int64_t*>(base + p.off_binoff);
  float* zkey = reinterpret_cast<float*>(base + p.off_zkey);
  const double inflate = std::sqrt(std::max(0.0, s->blur_radius));  // MR:103

  {
    ProfScope ps(st, KN_SETUP);
    drb::launch_face_setup(fv, first, num, N, max_faces, merged_ranges(ranges, N), p.H, p.W, inflate, s->znear,
                           s->clip_nonpositive_z, s->cull_backfaces, ibbox, zkey, st);
  }
  if (p.binned) {
    {
      ProfScope ps(st, KN_MEMSET);
      cudaError_t e = cudaMemsetAsync(counts, 0, sizeof(int) * (size_t)p.nbins_total, st);
      if (e == cudaSuccess) e = cudaMemsetAsync(cursor, 0, sizeof(int) * (size_t)p.nbins_total, st);
      if (e != cudaSuccess) return cuda_fail(e, "zeroing bin counts");
    }
    {
      ProfScope ps(st, KN_BIN);  // count -> scan -> fill: exact-size lists
      drb::launch_bin_faces(ibbox, first, num, N, max_faces, p.bs, p.nbx, p.nby, counts, st);
      drb::launch_scan_bins(counts, p.nbins_total, bin_off, st);
      drb::launch_fill_bins(ibbox, first, num, N, max_faces, p.bs, p.nbx, p.nby, counts, bin_off, cursor, p.pool,
                            p.zsort ? zkey : nullptr, entries, st);
    }
    // depth order of the bins (measured: skipping it costs C4 +9 % and C5 +170 % in K2)
    if (p.zsort) {
      ProfScope ps(st, KN_SORT);
      cudaError_t e = drb::launch_sort_bins(counts, bin_off, entries, ibbox, p.nbins_total, p.pool, p.cap, st);
      if (e != cudaSuccess) return cuda_fail(e, "sorting bins");
    }
  }
  drb::FineArgs<OutT> A;
  A.fv = fv;
  A.ibbox = ibbox;
  A.first = first;
  A.num = num;
  A.bin_counts = counts;
  A.bin_entries = entries;
  A.bin_off = bin_off;
  A.pool = p.pool;
  A.zkey = zkey;
  A.zsort = p.zsort ? 1 : 0;
  A.binned = p.binned ? 1 : 0;
  A.cap = p.cap;
  A.bs = p.bs;
  A.nbx = p.nbx;
  A.nby = p.nby;
  A.H = p.H;
  A.W = p.W;
  A.K = p.K;
  A.blur = s->blur_radius;
  A.znear = s->znear;
  A.persp = s->perspective_correct != 0;
  A.clip = s->clip_barycentric_coords != 0;
  // K2 is a persistent grid of warps pulling 8x4 micro-tiles; pick the CTA size (warps) that fits the most
  // warps per SM given each warp's shared memory (staged-face ring + K*32 top-K entries).
  const size_t per_warp = drb::fine_warp_smem_bytes(p.K);
  int nw = 0, best = 0;
  for (int cand : {8, 2}) {  // CTA sizes K2 is instantiated for
    size_t cta = (size_t)cand * per_warp + 1024;
    int ctas = (int)std::min<size_t>(228 * 1024 / cta, 32);
    if (cand * per_warp > 227 * 1024) ctas = 0;
    if (ctas * cand > best) {
      best = ctas * cand;
      nw = cand;
    }
  }
  if (nw == 0) return fail(DR_ERR_RANGE, "faces_per_pixel=%d too large for the shared-memory top-K", p.K);
  A.N = (int)N;
  A.work_counter = reinterpret_cast<unsigned long long*>(base + p.off_counter);
  {
    const int mtx = (p.bs + 7) >> 3, mty = (p.bs + 3) >> 2;  // micro-tiles per bin row / column (k_fine)
    A.div_mt = drb::FastDivU32((uint32_t)(mtx * mty));
    A.div_bins = drb::FastDivU32((uint32_t)(p.nbx * p.nby));
    A.div_nbx = drb::FastDivU32((uint32_t)p.nbx);
    A.div_mtx = drb::FastDivU32((uint32_t)mtx);
  }
  A.p2f = p2f;
  A.zbuf = zbuf;
  A.bary = bary;
  A.dists = dists;
  A.alpha = alpha;
  A.sigma = sigma;
  A.image = image;
  if (blend) A.blend = *blend;
  cudaError_t e = cudaMemsetAsync(A.work_counter, 0, sizeof(unsigned long long), st);
  if (e == cudaSuccess) {
    ProfScope ps(st, KN_FINE);
    e = drb::launch_fine(A, nw, st);
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "rasterize_meshes forward");
  return DR_OK;
}

template <typename InT>
int bwd_impl(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
             const dr_raster_settings* s, const int64_t* p2f, const InT* bary, const InT* dz, const InT* db,
             const InT* dd, double* grad, cudaStream_t st, const int64_t* host_first = nullptr,
             const int64_t* host_num = nullptr) {
  Plan p;
  int rc = make_plan(N, F, s, p);
  if (rc) return rc;
  if (!first || !num || !p2f || !bary || !dz || !db || !dd || (F > 0 && (!fv || !grad)))
    return fail(DR_ERR_USAGE, "null input/output pointer");
  // cotangents in host memory would fault in the kernel (pageable) or crawl over PCIe (page-locked: measured
  // slower than copying them): both are rejected
  for (const void* ptr : {static_cast<const void*>(dz), static_cast<const void*>(db), static_cast<const void*>(dd)}) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess ||
        (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)) {
      cudaGetLastError();
      return fail(DR_ERR_USAGE, "cotangent pointer is not device memory");
    }
  }
  int64_t mx;
  std::vector<int64_t> ranges;
  rc = read_ranges(first, num, N, F, st, &mx, &ranges, host_first, host_num);
  if (rc) return rc;
  if (F == 0) return DR_OK;
  cudaError_t e;
  {
    ProfScope ps(st, KN_MEMSET);
    e = zero_rows(grad, 9, ranges, N, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "zeroing grad_face_verts");
  drb::BwdArgs<InT> A;
  A.fv = fv;
  A.p2f = p2f;
  A.bary = bary;
  A.d_zbuf = dz;
  A.d_bary = db;
  A.d_dists = dd;
  A.grad = grad;
  A.S = N * (int64_t)p.H * p.W * p.K;
  A.F = F;
  A.H = p.H;
  A.W = p.W;
  A.K = p.K;
  A.persp = s->perspective_correct != 0;
  A.clip = s->clip_barycentric_coords != 0;
  A.divK = drb::FastDivU32((uint32_t)p.K);
  A.divW = drb::FastDivU32((uint32_t)p.W);
  {
    ProfScope ps(st, KN_BWD);
    e = drb::launch_backward(A, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "rasterize_meshes backward");
  return DR_OK;
}

int sil_bwd_impl(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
                 const dr_raster_settings* s, double sigma, const int64_t* p2f, const float* d_alpha, double* grad,
                 cudaStream_t st, const double* d_alpha64 = nullptr, const int64_t* host_first = nullptr,
                 const int64_t* host_num = nullptr) {
  Plan p;
  int rc = make_plan(N, F, s, p);
  if (rc) return rc;
  if (!first || !num || !p2f || (!d_alpha && !d_alpha64) || (F > 0 && (!fv || !grad)))
    return fail(DR_ERR_USAGE, "null input/output pointer");
  if (!(sigma > 0.0)) return fail(DR_ERR_RANGE, "silhouette sigma must be > 0 (got %g)", sigma);
  int64_t mx;
  std::vector<int64_t> ranges;
  rc = read_ranges(first, num, N, F, st, &mx, &ranges, host_first, host_num);
  if (rc) return rc;
  if (F == 0) return DR_OK;
  cudaError_t e;
  {
    ProfScope ps(st, KN_MEMSET);
    e = zero_rows(grad, 9, ranges, N, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "zeroing grad_face_verts");
  drb::SilBwdArgs A;
  A.fv = fv;
  A.p2f = p2f;
  A.d_alpha = d_alpha;
  A.d_alpha64 = d_alpha64;
  A.grad = grad;
  A.npix = N * (int64_t)p.H * p.W;
  A.F = F;
  A.H = p.H;
  A.W = p.W;
  A.K = p.K;
  A.sigma = sigma;
  {
    ProfScope ps(st, KN_SIL_BWD);
    e = drb::launch_silhouette_backward(A, st);
  }
  if (e == cudaErrorInvalidConfiguration)
    return fail(DR_ERR_RANGE, "faces_per_pixel=%d too large for the fused silhouette backward", p.K);
  if (e != cudaSuccess) return cuda_fail(e, "rasterize_silhouette backward");
  return DR_OK;
}

// ---- point rasterizer (point_render.cpp:105-155) ----
struct PointPlan {
  int64_t N = 0, P = 0;
  int H = 0, W = 0, K = 0, bs = 16, nbx = 0, nby = 0;
  bool binned = false;
  int64_t nbins_total = 0, pool = 0;
  size_t off_ibbox = 0, off_zkey = 0, off_bounds = 0, off_counts = 0, off_cursor = 0, off_binoff = 0, off_lists = 0,
         off_brange = 0, total = 0;
};

int make_point_plan(int64_t N, int64_t P, const dr_point_raster_settings* s, PointPlan& p) {
  if (!s) return fail(DR_ERR_USAGE, "settings pointer is null");
  if (N < 1) return fail(DR_ERR_SHAPE, "empty point cloud batch (N=%lld)", (long long)N);
  if (N > 65535) return fail(DR_ERR_RANGE, "N=%lld clouds exceeds 65535", (long long)N);
  if (P < 0) return fail(DR_ERR_SHAPE, "negative point count P=%lld", (long long)P);
  if (P > INT32_MAX - 1) return fail(DR_ERR_RANGE, "P=%lld exceeds the int32 point-id range", (long long)P);
  if (s->image_h < 1 || s->image_w < 1 || s->image_h > 32768 || s->image_w > 32768)
    return fail(DR_ERR_RANGE, "image size %dx%d outside [1, 32768]", s->image_h, s->image_w);
  if (s->points_per_pixel < 1 || s->points_per_pixel > 128)
    return fail(DR_ERR_RANGE, "points_per_pixel=%d outside [1, 128]", s->points_per_pixel);
  if (s->bin_size < 0) return fail(DR_ERR_RANGE, "bin_size=%d < 0", s->bin_size);
  if (std::isnan(s->radius) || std::isnan(s->znear)) return fail(DR_ERR_RANGE, "radius/znear is NaN");
  p.N = N;
  p.P = P;
  p.H = s->image_h;
  p.W = s->image_w;
  p.K = s->points_per_pixel;
  p.binned = s->bin_size > 0;
  p.bs = p.binned ? s->bin_size : 16;
  p.nbx = (p.W + p.bs - 1) / p.bs;
  p.nby = (p.H + p.bs - 1) / p.bs;
  size_t off = 0;
  p.off_ibbox = off;
  off = align_up(off + sizeof(int4) * (size_t)std::max<int64_t>(P, 1));
  p.off_zkey = off;
  off = align_up(off + sizeof(float) * (size_t)std::max<int64_t>(P, 1));
  p.off_bounds = off;
  off = align_up(off + sizeof(double) * 2 * (size_t)(p.nbx + p.nby));
  p.off_counts = off;
  if (p.binned) {
    p.nbins_total = N * (int64_t)p.nbx * p.nby;
    // list-pool capacity from the radius: a point lands in the tiles its radius-inflated tile test keeps
    // (PR:125-134), about (r W / bs + 2) x (r H / bs + 2) of them (tile side 2 bs / W in NDC), so a wide radius
    // does not push most bins onto the unsorted whole-cloud spill path. Clamped to keep the workspace bounded;
    // bins past the pool still rasterize correctly (spill path).
    const double r = std::max(0.0, s->radius);
    const double tx = std::min<double>(p.nbx, std::floor(r * p.W / p.bs) + 2.0);
    const double ty = std::min<double>(p.nby, std::floor(r * p.H / p.bs) + 2.0);
    const double want = (double)P * std::max(1.0, tx * ty);
    const double cap = std::max<double>(8.0 * P, (double)(1ll << 28));
    p.pool = (int64_t)std::min(want, cap) + 65536;
    off = align_up(off + sizeof(int) * (size_t)p.nbins_total);
    p.off_cursor = off;
    off = align_up(off + sizeof(int) * (size_t)p.nbins_total);
    p.off_binoff = off;
    off = align_up(off + sizeof(int64_t) * (size_t)p.nbins_total);
    p.off_lists = off;
    off = align_up(off + sizeof(int4) * (size_t)p.pool);
    p.off_brange = off;
    off = align_up(off + sizeof(float2) * (size_t)p.nbins_total);
  }
  p.total = off;
  return DR_OK;
}

template <typename OutT>
int points_fwd_impl(const double* pts, const int64_t* first, const int64_t* num, int64_t N, int64_t P,
                    const dr_point_raster_settings* s, int64_t* idx, OutT* zbuf, OutT* dists2, void* ws,
                    size_t ws_bytes, cudaStream_t st) {
  PointPlan p;
  int rc = make_point_plan(N, P, s, p);
  if (rc) return rc;
  if (!first || !num || !idx || !zbuf || !dists2 || (P > 0 && !pts)) return fail(DR_ERR_USAGE, "null pointer");
  if (!ws || ws_bytes < p.total)
    return fail(DR_ERR_OOM, "workspace too small: %zu bytes given, %zu needed", ws_bytes, p.total);
  int64_t max_pts = 0;
  std::vector<int64_t> ranges;
  rc = read_ranges(first, num, N, P, st, &max_pts, &ranges);
  if (rc) return rc;
  int64_t p_lo = P, p_hi = 0;
  for (int64_t b = 0; b < N; ++b)
    if (ranges[N + b] > 0) {
      p_lo = std::min(p_lo, ranges[b]);
      p_hi = std::max(p_hi, ranges[b] + ranges[N + b]);
    }
  char* base = static_cast<char*>(ws);
  int4* ibbox = reinterpret_cast<int4*>(base + p.off_ibbox);
  double* bounds = reinterpret_cast<double*>(base + p.off_bounds);
  float* zkey = reinterpret_cast<float*>(base + p.off_zkey);
  int* counts = reinterpret_cast<int*>(base + p.off_counts);
  int* cursor = reinterpret_cast<int*>(base + p.off_cursor);
  int64_t* bin_off = reinterpret_cast<int64_t*>(base + p.off_binoff);
  int4* entries = reinterpret_cast<int4*>(base + p.off_lists);
  float2* brange = reinterpret_cast<float2*>(base + p.off_brange);
  cudaError_t e;
  {
    ProfScope ps(st, KN_PT_SETUP);
    e = drb::launch_point_setup(pts, p_lo, p_hi, p.H, p.W, p.bs, p.nbx, p.nby, s->radius, s->znear,
                                s->clip_nonpositive_z, bounds, ibbox, zkey, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "rasterize_points setup");
  if (p.binned) {
    {
      ProfScope ps(st, KN_MEMSET);
      e = cudaMemsetAsync(counts, 0, sizeof(int) * (size_t)p.nbins_total, st);
      if (e == cudaSuccess) e = cudaMemsetAsync(cursor, 0, sizeof(int) * (size_t)p.nbins_total, st);
      if (e != cudaSuccess) return cuda_fail(e, "zeroing point bin counts");
    }
    ProfScope ps(st, KN_BIN);
    drb::launch_bin_faces(ibbox, first, num, N, max_pts, p.bs, p.nbx, p.nby, counts, st, /*smem_hist=*/true);
    drb::launch_scan_bins(counts, p.nbins_total, bin_off, st);
    drb::launch_fill_bins(ibbox, first, num, N, max_pts, p.bs, p.nbx, p.nby, counts, bin_off, cursor, p.pool, zkey,
                          entries, st, /*smem_hist=*/true);
  }
  const bool sorted = p.binned;
  if (sorted) {
    ProfScope ps(st, KN_SORT);
    // the point fine stage stops streaming a bin once a lower bound of its remaining keys exceeds every pixel's
    // K-th depth; that bound comes from the bin's bucket map (brange), written by the sort for every bin the
    // fine stage treats as sorted (drb::bin_is_sorted with cap 0)
    e = drb::launch_sort_bins(counts, bin_off, entries, ibbox, p.nbins_total, p.pool, 0, st, brange);
    if (e != cudaSuccess) return cuda_fail(e, "sorting point bins");
  }
  drb::PointFineArgs<OutT> A;
  A.pts = pts;
  A.ibbox = ibbox;
  A.zkey = zkey;
  A.first = first;
  A.num = num;
  A.bin_counts = counts;
  A.bin_off = bin_off;
  A.bin_entries = entries;
  A.pool = p.pool;
  A.binned = p.binned ? 1 : 0;
  A.bs = p.bs;
  A.nbx = p.nbx;
  A.nby = p.nby;
  A.sorted = sorted ? 1 : 0;
  A.brange = sorted ? brange : nullptr;
  A.sub_x = (p.bs + 15) / 16;
  A.sub_y = (p.bs + 15) / 16;
  A.H = p.H;
  A.W = p.W;
  A.K = p.K;
  A.r2 = s->radius * s->radius;  // point_render.cpp:112
  A.N = (int)N;
  A.idx = idx;
  A.zbuf = zbuf;
  A.dists2 = dists2;
  {
    ProfScope ps(st, KN_PT_FINE);
    e = drb::launch_points_fine(A, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "rasterize_points");
  return DR_OK;
}

template <typename InT>
int points_bwd_impl(const double* pts, const int64_t* first, const int64_t* num, int64_t N, int64_t P,
                    const dr_point_raster_settings* s, const int64_t* idx, const InT* gz, const InT* gd, double* grad,
                    cudaStream_t st) {
  PointPlan p;
  int rc = make_point_plan(N, P, s, p);
  if (rc) return rc;
  if (!first || !num || !idx || !gz || !gd || (P > 0 && (!pts || !grad))) return fail(DR_ERR_USAGE, "null pointer");
  int64_t mx;
  std::vector<int64_t> ranges;
  rc = read_ranges(first, num, N, P, st, &mx, &ranges);
  if (rc) return rc;
  if (P == 0) return DR_OK;
  cudaError_t e;
  {
    ProfScope ps(st, KN_MEMSET);
    e = zero_rows(grad, 3, ranges, N, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "zeroing grad_points");
  {
    ProfScope ps(st, KN_PT_BWD);
    e = drb::launch_points_backward(pts, idx, gz, gd, N * (int64_t)p.H * p.W * p.K, P, p.H, p.W, p.K, grad, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "rasterize_points backward");
  return DR_OK;
}

drb::BlendArgs blend_args(const dr_blend_params* bp, const double* vert_colors, const int64_t* faces, int64_t V) {
  drb::BlendArgs b;
  b.vert_colors = vert_colors;
  b.faces = faces;
  b.V = V;
  b.sigma = bp->sigma;
  b.gamma = bp->gamma;
  for (int c = 0; c < 3; ++c) b.background[c] = bp->background[c];
  b.znear = bp->znear;
  b.zfar = bp->zfar;
  b.inv_sigma = 1.0 / b.sigma;
  b.inv_gamma = 1.0 / b.gamma;
  b.inv_zr = 1.0 / (b.zfar - b.znear);
  return b;
}

int check_blend(const dr_blend_params* bp, const double* vert_colors, const int64_t* faces, int64_t V, int64_t F) {
  if (!bp) return fail(DR_ERR_USAGE, "blend params pointer is null");
  if (!(bp->sigma > 0.0) || !(bp->gamma > 0.0))
    return fail(DR_ERR_RANGE, "blend sigma/gamma must be > 0 (got %g, %g)", bp->sigma, bp->gamma);
  if (!(bp->zfar > bp->znear)) return fail(DR_ERR_RANGE, "zfar (%g) must exceed znear (%g)", bp->zfar, bp->znear);
  if (V < 0) return fail(DR_ERR_SHAPE, "negative vertex count");
  if (F > 0 && (!vert_colors || !faces)) return fail(DR_ERR_USAGE, "null vertex colours / faces");
  return DR_OK;
}

}  // namespace

extern "C" {

int dr_rasterize_softmax_fwd(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
                             const dr_raster_settings* s, const dr_blend_params* bp, const double* vert_colors,
                             const int64_t* faces, int64_t V, int64_t* p2f, float* image, void* ws, size_t ws_bytes,
                             dr_stream_t stream) {
  if (!image) return fail(DR_ERR_USAGE, "image is null");
  int rc = check_blend(bp, vert_colors, faces, V, F);
  if (rc) return rc;
  const drb::BlendArgs b = blend_args(bp, vert_colors, faces, V);
  return fwd_impl<float>(fv, first, num, N, F, s, p2f, nullptr, nullptr, nullptr, ws, ws_bytes,
                         reinterpret_cast<cudaStream_t>(stream), nullptr, nullptr, nullptr, 0.0, image, &b);
}

int dr_rasterize_softmax_bwd(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
                             const dr_raster_settings* s, const dr_blend_params* bp, const double* vert_colors,
                             const int64_t* faces, int64_t V, const int64_t* p2f, const float* grad_image,
                             double* grad_face_verts, double* grad_vert_colors, dr_stream_t stream) {
  Plan p;
  int rc = make_plan(N, F, s, p);
  if (rc) return rc;
  rc = check_blend(bp, vert_colors, faces, V, F);
  if (rc) return rc;
  if (!first || !num || !p2f || !grad_image || (F > 0 && (!fv || !grad_face_verts)) || (V > 0 && !grad_vert_colors))
    return fail(DR_ERR_USAGE, "null input/output pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int64_t mx;
  std::vector<int64_t> ranges;
  rc = read_ranges(first, num, N, F, st, &mx, &ranges);
  if (rc) return rc;
  cudaError_t e;
  {
    ProfScope ps(st, KN_MEMSET);
    e = zero_rows(grad_face_verts, 9, ranges, N, st);
    if (e == cudaSuccess && V > 0) e = cudaMemsetAsync(grad_vert_colors, 0, sizeof(double) * 3 * (size_t)V, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "zeroing gradients");
  if (F == 0) return DR_OK;
  drb::SoftBwdArgs A;
  A.fv = fv;
  A.p2f = p2f;
  A.d_image = grad_image;
  A.grad = grad_face_verts;
  A.grad_colors = grad_vert_colors;
  A.npix = N * (int64_t)p.H * p.W;
  A.F = F;
  A.H = p.H;
  A.W = p.W;
  A.K = p.K;
  A.persp = s->perspective_correct != 0;
  A.clip = s->clip_barycentric_coords != 0;
  A.blur = s->blur_radius;
  A.znear = s->znear;
  A.blend = blend_args(bp, vert_colors, faces, V);
  {
    ProfScope ps(st, KN_SOFT_BWD);
    e = drb::launch_softmax_backward(A, st);
  }
  if (e == cudaErrorInvalidConfiguration)
    return fail(DR_ERR_RANGE, "faces_per_pixel=%d too large for the fused softmax backward (<= 64)", p.K);
  if (e != cudaSuccess) return cuda_fail(e, "rasterize_softmax backward");
  return DR_OK;
}

void dr_point_raster_settings_default(dr_point_raster_settings* s) {
  if (!s) return;
  std::memset(s, 0, sizeof(*s));
  s->image_h = s->image_w = 64;  // PointRasterSettings{} (point_render.hpp:14-19)
  s->points_per_pixel = 8;
  s->bin_size = 16;
  s->radius = 0.05;
  s->znear = 0.1;
  s->clip_nonpositive_z = 1;
}

size_t dr_rasterize_points_workspace_bytes(int64_t N, int64_t P, const dr_point_raster_settings* s) {
  PointPlan p;
  if (make_point_plan(N, P, s, p)) return 0;
  return p.total;
}

int dr_rasterize_points_fwd(const double* pts, const int64_t* first, const int64_t* num, int64_t N, int64_t P,
                            const dr_point_raster_settings* s, int64_t* idx, float* zbuf, float* dists2, void* ws,
                            size_t ws_bytes, dr_stream_t stream) {
  return points_fwd_impl<float>(pts, first, num, N, P, s, idx, zbuf, dists2, ws, ws_bytes,
                                reinterpret_cast<cudaStream_t>(stream));
}

int dr_rasterize_points_fwd_f64(const double* pts, const int64_t* first, const int64_t* num, int64_t N, int64_t P,
                                const dr_point_raster_settings* s, int64_t* idx, double* zbuf, double* dists2,
                                void* ws, size_t ws_bytes, dr_stream_t stream) {
  return points_fwd_impl<double>(pts, first, num, N, P, s, idx, zbuf, dists2, ws, ws_bytes,
                                 reinterpret_cast<cudaStream_t>(stream));
}

int dr_rasterize_points_bwd(const double* pts, const int64_t* first, const int64_t* num, int64_t N, int64_t P,
                            const dr_point_raster_settings* s, const int64_t* idx, const float* grad_zbuf,
                            const float* grad_dists2, double* grad_points, dr_stream_t stream) {
  return points_bwd_impl<float>(pts, first, num, N, P, s, idx, grad_zbuf, grad_dists2, grad_points,
                                reinterpret_cast<cudaStream_t>(stream));
}

int dr_rasterize_points_bwd_f64(const double* pts, const int64_t* first, const int64_t* num, int64_t N, int64_t P,
                                const dr_point_raster_settings* s, const int64_t* idx, const double* grad_zbuf,
                                const double* grad_dists2, double* grad_points, dr_stream_t stream) {
  return points_bwd_impl<double>(pts, first, num, N, P, s, idx, grad_zbuf, grad_dists2, grad_points,
                                 reinterpret_cast<cudaStream_t>(stream));
}

int dr_rasterize_silhouette_fwd(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
                                const dr_raster_settings* s, double sigma, int64_t* p2f, float* alpha, void* ws,
                                size_t ws_bytes, dr_stream_t stream) {
  if (!alpha) return fail(DR_ERR_USAGE, "alpha is null");
  return fwd_impl<float>(fv, first, num, N, F, s, p2f, nullptr, nullptr, nullptr, ws, ws_bytes,
                         reinterpret_cast<cudaStream_t>(stream), nullptr, nullptr, alpha, sigma);
}

int dr_rasterize_silhouette_bwd(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
                                const dr_raster_settings* s, double sigma, const int64_t* p2f, const float* d_alpha,
                                double* grad, dr_stream_t stream) {
  return sil_bwd_impl(fv, first, num, N, F, s, sigma, p2f, d_alpha, grad, reinterpret_cast<cudaStream_t>(stream));
}

int dr_rasterize_silhouette_fwd_f64(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
                                    const dr_raster_settings* s, double sigma, int64_t* p2f, double* alpha, void* ws,
                                    size_t ws_bytes, dr_stream_t stream) {
  if (!alpha) return fail(DR_ERR_USAGE, "alpha is null");
  return fwd_impl<double>(fv, first, num, N, F, s, p2f, nullptr, nullptr, nullptr, ws, ws_bytes,
                          reinterpret_cast<cudaStream_t>(stream), nullptr, nullptr, alpha, sigma);
}

int dr_rasterize_silhouette_bwd_f64(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
                                    const dr_raster_settings* s, double sigma, const int64_t* p2f,
                                    const double* d_alpha, double* grad, dr_stream_t stream) {
  return sil_bwd_impl(fv, first, num, N, F, s, sigma, p2f, nullptr, grad, reinterpret_cast<cudaStream_t>(stream),
                      d_alpha);
}

int dr_rasterize_silhouette_fwd_f64_hr(const double* fv, const int64_t* first, const int64_t* num, int64_t N,
                                       int64_t F, const dr_raster_settings* s, double sigma, int64_t* p2f,
                                       double* alpha, void* ws, size_t ws_bytes, dr_stream_t stream,
                                       const int64_t* host_first, const int64_t* host_num) {
  if (!alpha) return fail(DR_ERR_USAGE, "alpha is null");
  if (!host_first || !host_num) return fail(DR_ERR_USAGE, "host ranges are null");
  return fwd_impl<double>(fv, first, num, N, F, s, p2f, nullptr, nullptr, nullptr, ws, ws_bytes,
                          reinterpret_cast<cudaStream_t>(stream), host_first, host_num, alpha, sigma);
}

int dr_rasterize_silhouette_bwd_f64_hr(const double* fv, const int64_t* first, const int64_t* num, int64_t N,
                                       int64_t F, const dr_raster_settings* s, double sigma, const int64_t* p2f,
                                       const double* d_alpha, double* grad, dr_stream_t stream,
                                       const int64_t* host_first, const int64_t* host_num) {
  if (!host_first || !host_num) return fail(DR_ERR_USAGE, "host ranges are null");
  return sil_bwd_impl(fv, first, num, N, F, s, sigma, p2f, nullptr, grad, reinterpret_cast<cudaStream_t>(stream),
                      d_alpha, host_first, host_num);
}

void dr_raster_settings_default(dr_raster_settings* s) {
  if (!s) return;
  std::memset(s, 0, sizeof(*s));
  s->image_h = s->image_w = 64;  // RasterSettings{} (mesh_raster.hpp:18-23)
  s->faces_per_pixel = 1;
  s->bin_size = 16;
  s->blur_radius = 1e-4;
  s->znear = 0.1;  // Camera{} (camera.hpp:26)
  s->clip_nonpositive_z = 1;
  s->clip_barycentric_coords = 1;
}

size_t dr_rasterize_meshes_workspace_bytes(int64_t N, int64_t F, const dr_raster_settings* s) {
  Plan p;
  if (make_plan(N, F, s, p)) return 0;
  return p.total;
}

int dr_rasterize_meshes_fwd(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
                            const dr_raster_settings* s, int64_t* p2f, float* zbuf, float* bary, float* dists,
                            void* ws, size_t ws_bytes, dr_stream_t stream) {
  return fwd_impl<float>(fv, first, num, N, F, s, p2f, zbuf, bary, dists, ws, ws_bytes,
                         reinterpret_cast<cudaStream_t>(stream));
}

int dr_rasterize_meshes_fwd_hr(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
                               const dr_raster_settings* s, int64_t* p2f, float* zbuf, float* bary, float* dists,
                               void* ws, size_t ws_bytes, dr_stream_t stream, const int64_t* host_first,
                               const int64_t* host_num) {
  if (!host_first || !host_num) return fail(DR_ERR_USAGE, "host ranges are null");
  return fwd_impl<float>(fv, first, num, N, F, s, p2f, zbuf, bary, dists, ws, ws_bytes,
                         reinterpret_cast<cudaStream_t>(stream), host_first, host_num);
}

int dr_rasterize_meshes_bwd_hr(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
                               const dr_raster_settings* s, const int64_t* p2f, const float* bary, const float* dz,
                               const float* db, const float* dd, double* grad, dr_stream_t stream,
                               const int64_t* host_first, const int64_t* host_num) {
  if (!host_first || !host_num) return fail(DR_ERR_USAGE, "host ranges are null");
  return bwd_impl<float>(fv, first, num, N, F, s, p2f, bary, dz, db, dd, grad, reinterpret_cast<cudaStream_t>(stream),
                         host_first, host_num);
}

int dr_rasterize_meshes_fwd_f64(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
                                const dr_raster_settings* s, int64_t* p2f, double* zbuf, double* bary,
                                double* dists, void* ws, size_t ws_bytes, dr_stream_t stream) {
  return fwd_impl<double>(fv, first, num, N, F, s, p2f, zbuf, bary, dists, ws, ws_bytes,
                          reinterpret_cast<cudaStream_t>(stream));
}

int dr_rasterize_meshes_bwd(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
                            const dr_raster_settings* s, const int64_t* p2f, const float* bary, const float* dz,
                            const float* db, const float* dd, double* grad, dr_stream_t stream) {
  return bwd_impl<float>(fv, first, num, N, F, s, p2f, bary, dz, db, dd, grad, reinterpret_cast<cudaStream_t>(stream));
}

int dr_rasterize_meshes_bwd_f64(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t F,
                                const dr_raster_settings* s, const int64_t* p2f, const double* bary,
                                const double* dz, const double* db, const double* dd, double* grad,
                                dr_stream_t stream) {
  return bwd_impl<double>(fv, first, num, N, F, s, p2f, bary, dz, db, dd, grad,
                          reinterpret_cast<cudaStream_t>(stream));
}

static drb::CameraArgs camera_args(const dr_camera* cam) {
  drb::CameraArgs a;
  for (int i = 0; i < 9; ++i) a.r[i] = cam->rotation[i];
  for (int i = 0; i < 3; ++i) a.t[i] = cam->translation[i];
  a.focal = cam->focal_length;
  a.pp[0] = cam->principal_point[0];
  a.pp[1] = cam->principal_point[1];
  a.ortho[0] = cam->ortho_scale[0];
  a.ortho[1] = cam->ortho_scale[1];
  a.perspective = cam->perspective != 0;
  return a;
}

int dr_world_to_face_verts(const double* verts, int64_t V, const int64_t* faces, int64_t F, const dr_camera* cam,
                           double* face_verts, dr_stream_t stream) {
  if (!cam) return fail(DR_ERR_USAGE, "camera pointer is null");
  if (V < 0 || F < 0) return fail(DR_ERR_SHAPE, "negative vertex/face count");
  if (F == 0) return DR_OK;
  if (!verts || !faces || !face_verts) return fail(DR_ERR_USAGE, "null input/output pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int* flag = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&flag), sizeof(int), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(flag, 0, sizeof(int), st);
  if (e == cudaSuccess) {
    ProfScope ps(st, KN_CAMERA);
    e = drb::launch_world_to_face_verts(verts, V, faces, F, camera_args(cam), face_verts, flag, st);
  }
  int bad = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, flag, sizeof(int), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (flag) cudaFreeAsync(flag, st);
  if (e != cudaSuccess) return cuda_fail(e, "world_to_face_verts");
  if (bad) return fail(DR_ERR_INDEX, "face vertex index out of range [0, %lld)", (long long)V);
  return DR_OK;
}

int dr_world_to_face_verts_async(const double* verts, int64_t V, const int64_t* faces, int64_t F,
                                 const dr_camera* cam, double* face_verts, int* bad_index, dr_stream_t stream) {
  if (!cam) return fail(DR_ERR_USAGE, "camera pointer is null");
  if (V < 0 || F < 0) return fail(DR_ERR_SHAPE, "negative vertex/face count");
  if (F == 0) return DR_OK;
  if (!verts || !faces || !face_verts) return fail(DR_ERR_USAGE, "null input/output pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  {
    ProfScope ps(st, KN_CAMERA);
    e = drb::launch_world_to_face_verts(verts, V, faces, F, camera_args(cam), face_verts, bad_index, st);
  }
  return e == cudaSuccess ? DR_OK : cuda_fail(e, "world_to_face_verts");
}

int dr_face_verts_backward(const double* verts, int64_t V, const int64_t* faces, int64_t F, const dr_camera* cam,
                           const double* gfv, double* gverts, dr_stream_t stream) {
  if (!cam) return fail(DR_ERR_USAGE, "camera pointer is null");
  if (V < 0 || F < 0) return fail(DR_ERR_SHAPE, "negative vertex/face count");
  if (V == 0) return DR_OK;
  if (!verts || !gverts || (F > 0 && (!faces || !gfv))) return fail(DR_ERR_USAGE, "null input/output pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  {
    ProfScope ps(st, KN_CAMERA);
    e = drb::launch_face_verts_backward(verts, V, faces, F, camera_args(cam), gfv, gverts, st);
  }
  if (e != cudaSuccess) return cuda_fail(e, "face_verts_backward");
  return DR_OK;
}

int dr_world_to_points_ndc(const double* points, int64_t P, const dr_camera* cam, double* points_ndc,
                           dr_stream_t stream) {
  if (!cam) return fail(DR_ERR_USAGE, "camera pointer is null");
  if (P < 0) return fail(DR_ERR_SHAPE, "negative point count");
  if (P == 0) return DR_OK;
  if (!points || !points_ndc) return fail(DR_ERR_USAGE, "null input/output pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  {
    ProfScope ps(st, KN_CAMERA);
    e = drb::launch_world_to_points_ndc(points, P, camera_args(cam), points_ndc, st);
  }
  return e == cudaSuccess ? DR_OK : cuda_fail(e, "world_to_points_ndc");
}

int dr_points_ndc_backward(const double* points, int64_t P, const dr_camera* cam, const double* grad_points_ndc,
                           double* grad_points, dr_stream_t stream) {
  if (!cam) return fail(DR_ERR_USAGE, "camera pointer is null");
  if (P < 0) return fail(DR_ERR_SHAPE, "negative point count");
  if (P == 0) return DR_OK;
  if (!points || !grad_points_ndc || !grad_points) return fail(DR_ERR_USAGE, "null input/output pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  {
    ProfScope ps(st, KN_CAMERA);
    e = drb::launch_points_ndc_backward(points, P, camera_args(cam), grad_points_ndc, grad_points, st);
  }
  return e == cudaSuccess ? DR_OK : cuda_fail(e, "points_ndc_backward");
}

int dr_packed_to_padded(const void* packed, const int64_t* first, const int64_t* num, int64_t N, int64_t max_count,
                        int64_t row_bytes, const void* pad_row, void* padded, dr_stream_t stream) {
  if (N < 0 || max_count < 0 || row_bytes <= 0) return fail(DR_ERR_SHAPE, "packed_to_padded: bad sizes");
  if (row_bytes > drb::kMaxPadRow && pad_row)
    return fail(DR_ERR_RANGE, "packed_to_padded: pad row larger than %d bytes", drb::kMaxPadRow);
  if (N * max_count > 0 && (!first || !num || !packed || !padded))
    return fail(DR_ERR_USAGE, "packed_to_padded: null pointer");
  drb::PadRow pad;
  std::memset(pad.bytes, 0, sizeof(pad.bytes));
  if (pad_row) std::memcpy(pad.bytes, pad_row, (size_t)row_bytes);
  else if (row_bytes > drb::kMaxPadRow) return fail(DR_ERR_RANGE, "packed_to_padded: rows above 256 bytes unsupported");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  {
    ProfScope ps(st, KN_BATCH);
    e = drb::launch_packed_to_padded(packed, first, num, N, max_count, row_bytes, pad, padded, st);
  }
  return e == cudaSuccess ? DR_OK : cuda_fail(e, "packed_to_padded");
}

int dr_padded_to_packed(const void* padded, const int64_t* first, const int64_t* num, int64_t N, int64_t max_count,
                        int64_t row_bytes, void* packed, dr_stream_t stream) {
  if (N < 0 || max_count < 0 || row_bytes <= 0) return fail(DR_ERR_SHAPE, "padded_to_packed: bad sizes");
  if (N * max_count > 0 && (!first || !num || !packed || !padded))
    return fail(DR_ERR_USAGE, "padded_to_packed: null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  {
    ProfScope ps(st, KN_BATCH);
    e = drb::launch_padded_to_packed(padded, first, num, N, max_count, row_bytes, packed, st);
  }
  return e == cudaSuccess ? DR_OK : cuda_fail(e, "padded_to_packed");
}

int dr_packed_item_to_element(const int64_t* first, const int64_t* num, int64_t N, int64_t total, int32_t* out,
                              dr_stream_t stream) {
  if (N < 0 || total < 0) return fail(DR_ERR_SHAPE, "item_to_element: bad sizes");
  if ((N > 0 && (!first || !num)) || (total > 0 && !out)) return fail(DR_ERR_USAGE, "item_to_element: null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  {
    ProfScope ps(st, KN_BATCH);
    e = drb::launch_item_to_element(first, num, N, total, out, st);
  }
  return e == cudaSuccess ? DR_OK : cuda_fail(e, "item_to_element");
}

const char* dr_last_error(void) { return g_err.c_str(); }

// used by the host-only translation units of this library (shard.cu) to report through dr_last_error()
int dr_set_error(int status, const char* msg) { return fail(status, "%s", msg); }

int dr_rasterize_meshes_bin_stats(int64_t N, int64_t F, const dr_raster_settings* s, const void* ws,
                                  dr_stream_t stream, int64_t out[4]) {
  Plan p;
  int rc = make_plan(N, F, s, p);
  if (rc) return rc;
  if (!p.binned) return fail(DR_ERR_USAGE, "bin_stats: bin_size == 0 (naive path has no bins)");
  if (!ws || !out) return fail(DR_ERR_USAGE, "null pointer");
  size_t nb = (size_t)p.nbins_total;
  std::vector<int> h(nb);
  std::vector<int64_t> ho(nb);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(h.data(), static_cast<const char*>(ws) + p.off_counts, sizeof(int) * nb,
                                  cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(ho.data(), static_cast<const char*>(ws) + p.off_binoff, sizeof(int64_t) * nb,
                        cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "bin_stats");
  int64_t over = 0, tot = 0, mx = 0;
  for (size_t i = 0; i < nb; ++i) {
    over += !drb::bin_fits(ho[i], h[i], p.pool, p.cap);
    tot += h[i];
    mx = std::max<int64_t>(mx, h[i]);
  }
  out[0] = (int64_t)nb;
  out[1] = over;
  out[2] = tot;
  out[3] = mx;
  return DR_OK;
}

uint64_t dr_launch_count(void) { return g_launches.load(); }

void dr_profile_enable(int enable) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& e : g_prof) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  g_prof.clear();
  g_prof_on.store(enable != 0);
}

int dr_profile_read(int* kernel_idx, float* ms, int cap) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  int n = 0;
  for (auto& e : g_prof) {
    if (n >= cap) break;
    cudaEventSynchronize(e.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, e.a, e.b);
    kernel_idx[n] = e.kernel;
    ms[n] = t;
    ++n;
  }
  return n;
}

const char* dr_profile_kernel_name(int idx) {
  if (idx < 0 || idx >= (int)(sizeof(kKernelNames) / sizeof(kKernelNames[0]))) return "";
  return kKernelNames[idx];
}

}  // extern "C"
