// Kernel argument blocks and launcher declarations shared by raster_fwd.cu, raster_bwd.cu and capi.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <utility>
#include <vector>

namespace drb {

// softmax render (shading.cpp:123-230 over interpolate_face_attributes, shading.cpp:11-73; grad.cpp:177-209)
struct BlendArgs {
  const double* vert_colors = nullptr;  // [V,3] packed per-vertex colours
  const int64_t* faces = nullptr;       // [F,3] packed faces, global vertex ids
  int64_t V = 0;
  double sigma = 1e-4, gamma = 1e-4;    // BlendParams (shading.hpp:13-17)
  double background[3] = {0.0, 0.0, 0.0};
  double znear = 0.1, zfar = 100.0;     // Camera.znear / zfar
  // 1 / sigma, 1 / gamma, 1 / (zfar - znear), computed once on the host: the render's per-slot blend values are
  // products with these instead of IEEE divisions (tolerance values, never selected on)
  double inv_sigma = 1e4, inv_gamma = 1e4, inv_zr = 1.0 / 99.9;
};

// Unsigned 32-bit division by a run-time invariant divisor with one multiply-high (Granlund & Montgomery,
// "Division by invariant integers using multiplication", Fig. 4.1): exact for every 32-bit dividend.
struct FastDivU32 {
  uint32_t d = 1, m = 1;
  int sh1 = 0, sh2 = 0;
  FastDivU32() = default;
  explicit FastDivU32(uint32_t div) : d(div) {
    int l = 0;
    while (l < 32 && (1ull << l) < div) ++l;  // l = ceil(log2 d)
    m = (uint32_t)(((1ull << 32) * ((1ull << l) - div)) / div + 1);
    sh1 = l < 1 ? l : 1;
    sh2 = l - 1 > 0 ? l - 1 : 0;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    const uint32_t t1 = __umulhi(m, n);
    return (t1 + ((n - t1) >> sh1)) >> sh2;
  }
};

template <typename OutT>
struct FineArgs {
  const double* fv;         // [F,3,3] face_verts
  const int4* ibbox;        // [F] (i0, i1, j0, j1) exact pixel ranges; empty if i0 > i1
  const int64_t* first;     // [N] mesh_to_face_first_idx
  const int64_t* num;       // [N] num_faces_per_mesh
  const int* bin_counts;    // [N, nby, nbx] entries per bin
  const int64_t* bin_off;   // [N, nby, nbx] start of each bin's list in the pool (exclusive scan of counts)
  const int4* bin_entries;  // [pool] bin after bin: {face id, zkey bits, i0 | i1 << 16, j0 | j1 << 16}
  const float* zkey;        // [F] lower bound on any z the face can produce at any pixel (zsort only)
  int64_t pool;             // list pool capacity (entries); a bin that does not fit takes the spill path
  int zsort;                // 1 => depth-ordered bins (ascending zkey) + K-th-depth culling (clip_barycentric_coords)
  int binned;               // 0 => naive: every CTA scans its whole mesh
  int cap;                  // max_faces_per_bin: 0 = unlimited; longer bins take the spill path
  int bs, nbx, nby;         // bin (tile) side in pixels, bins per row / column
  int H, W, K;
  double blur, znear;
  bool persp, clip;
  int N;
  unsigned long long* work_counter;  // zeroed before launch; warps pull micro-tiles from it
  // micro-tile index -> (mesh, bin, micro-tile) without integer division instructions (set by the launcher)
  FastDivU32 div_mt, div_bins, div_nbx, div_mtx;
  int64_t* p2f;
  OutT* zbuf;
  OutT* bary;
  OutT* dists;
  OutT* alpha;   // non-null => fused silhouette_blend (shading.cpp:75-91): alpha [N,H,W] (+ p2f if non-null)
  double sigma;  // silhouette opacity falloff (BlendParams.sigma)
  OutT* image;   // non-null => fused softmax render: image [N,H,W,3] (+ p2f if non-null)
  BlendArgs blend;
};


template <typename InT>
struct BwdArgs {
  const double* fv;
  const int64_t* p2f;
  const InT* bary;
  const InT* d_zbuf;
  const InT* d_bary;
  const InT* d_dists;
  double* grad;  // [F,3,3]
  int64_t S;     // slots
  int64_t F;
  int H, W, K;
  bool persp, clip;
  FastDivU32 divK, divW;  // slot -> pixel -> (i, j) without integer division instructions
  int cpc = 32;           // K3: 512-slot chunks per CTA (set by the launcher from the slot count)
};

// fused silhouette_blend_backward + rasterize_backward (shading.cpp:93-121, MR:329-403 with d_zbuf = d_bary = 0)
struct SilBwdArgs {
  const double* fv;
  const int64_t* p2f;     // [N,H,W,K]
  const float* d_alpha;   // [N,H,W]
  const double* d_alpha64;  // [N,H,W] fp64 cotangent (used instead of d_alpha when non-null; exact exp)
  double* grad;           // [F,3,3]
  int64_t npix;           // N*H*W
  int64_t F;
  int H, W, K;
  double sigma;
  FastDivU32 divK;  // slot -> pixel in the slot-compacted kernel (set by the launcher)
};

// point rasterizer (raster_points.cu)
template <typename OutT>
struct PointFineArgs {  // rasterize_points (point_render.cpp:105-155)
  const double* pts;
  const int4* ibbox;
  const float* zkey;        // [P] +inf: culled by prepare_points (PR:17-31), else <= the point's depth
  const int64_t* first;
  const int64_t* num;
  const int* bin_counts;
  const int64_t* bin_off;
  const int4* bin_entries;
  int64_t pool;
  int binned, bs, nbx, nby, sub_x, sub_y;  // sub_x/sub_y: 16x16 blocks per bin row / column
  int sorted;                              // bins depth-ordered (early exit)
  const float2* brange = nullptr;          // bucket-ordered bins: per-bin (lo, scale) of the bucket map
  int H, W, K;
  double r2;
  int N;
  int64_t* idx;
  OutT* zbuf;
  OutT* dists2;
};

cudaError_t launch_point_setup(const double* pts, int64_t p_lo, int64_t p_hi, int H, int W, int ts, int nbx, int nby,
                               double radius, double znear, int clip_z, double* bounds /*[2*nbx + 2*nby]*/,
                               int4* ibbox, float* zkey, cudaStream_t st);
cudaError_t launch_points_fine(const PointFineArgs<float>& A, cudaStream_t st);
cudaError_t launch_points_fine(const PointFineArgs<double>& A, cudaStream_t st);
cudaError_t launch_points_backward(const double* pts, const int64_t* idx, const float* gz, const float* gd, int64_t S,
                                   int64_t P, int H, int W, int K, double* grad, cudaStream_t st);
cudaError_t launch_points_backward(const double* pts, const int64_t* idx, const double* gz, const double* gd,
                                   int64_t S, int64_t P, int H, int W, int K, double* grad, cudaStream_t st);

// fused softmax render backward (grad.cpp:195-206: softmax_blend_backward -> interpolate_face_attributes_backward
// -> rasterize_backward)
struct SoftBwdArgs {
  const double* fv;
  const int64_t* p2f;      // [N,H,W,K]
  const float* d_image;    // [N,H,W,3]
  double* grad;            // [F,3,3] face_verts cotangent
  double* grad_colors;     // [V,3] vertex-colour cotangent
  int64_t npix, F;
  int H, W, K;
  bool persp, clip;
  double blur, znear;      // raster settings (exact re-evaluation of each slot)
  BlendArgs blend;
  FastDivU32 divK;         // slot -> pixel in the slot-compacted kernel (set by the launcher)
};
cudaError_t launch_softmax_backward(const SoftBwdArgs& A, cudaStream_t st);

// Camera (dr_camera / dr::Camera, camera.hpp:19-35) as kernel arguments.
struct CameraArgs {
  double r[9];      // world -> view rotation, row-major
  double t[3];      // world -> view translation
  double focal;     // perspective focal length
  double pp[2];     // principal point (NDC)
  double ortho[2];  // orthographic scale
  int perspective;
};

cudaError_t launch_world_to_face_verts(const double* verts, int64_t V, const int64_t* faces, int64_t F,
                                       const CameraArgs& c, double* fv, int* bad_index, cudaStream_t st);
cudaError_t launch_world_to_points_ndc(const double* points, int64_t P, const CameraArgs& c, double* out,
                                       cudaStream_t st);
cudaError_t launch_points_ndc_backward(const double* points, int64_t P, const CameraArgs& c, const double* g_ndc,
                                       double* g_world, cudaStream_t st);
cudaError_t launch_face_verts_backward(const double* verts, int64_t V, const int64_t* faces, int64_t F,
                                       const CameraArgs& c, const double* gfv, double* gverts, cudaStream_t st);
// pad row of packed_to_padded (passed by value in the kernel parameters)
constexpr int kMaxPadRow = 256;
struct PadRow {
  unsigned char bytes[kMaxPadRow];
};
cudaError_t launch_packed_to_padded(const void* packed, const int64_t* first, const int64_t* num, int64_t N,
                                    int64_t max_count, int64_t row_bytes, const PadRow& pad, void* padded,
                                    cudaStream_t st);
cudaError_t launch_padded_to_packed(const void* padded, const int64_t* first, const int64_t* num, int64_t N,
                                    int64_t max_count, int64_t row_bytes, void* packed, cudaStream_t st);
cudaError_t launch_item_to_element(const int64_t* first, const int64_t* num, int64_t N, int64_t total, int32_t* out,
                                   cudaStream_t st);

void launch_face_setup(const double* fv, const int64_t* first, const int64_t* num, int64_t N, int64_t max_faces,
                       const std::vector<std::pair<int64_t, int64_t>>& intervals, int H, int W, double inflate,
                       double znear, int clip_z, int cull, int4* ibbox, float* zkey, cudaStream_t st);
constexpr int kSortMax = 4096;      // bins up to this length are sorted by k_sort_bins (32 KB shared memory)
constexpr int kSortMaxBig = 16384;  // ... up to this one by its 128 KB variant; longer bins stay unsorted
// bin usable as a list: fits the pool and the caller's max_faces_per_bin (0 = unlimited)
__host__ __device__ __forceinline__ bool bin_fits(int64_t off, int cnt, int64_t pool, int cap) {
  return off + cnt <= pool && (cap <= 0 || cnt <= cap);
}
void launch_bin_faces(const int4* ibbox, const int64_t* first, const int64_t* num, int64_t N, int64_t max_faces,
                      int bs, int nbx, int nby, int* counts, cudaStream_t st,
                      bool smem_hist = false);  // count pass
void launch_scan_bins(const int* counts, int64_t nbins_total, int64_t* off, cudaStream_t st);
void launch_fill_bins(const int4* ibbox, const int64_t* first, const int64_t* num, int64_t N, int64_t max_faces,
                      int bs, int nbx, int nby, const int* counts, const int64_t* off, int* cursor, int64_t pool,
                      const float* zkey, int4* entries, cudaStream_t st, bool smem_hist = false);
// smem_hist: the CTA-level shared-memory histogram form (k_bin_faces_smem), for items in no spatial order (points)
// The bins k_sort_bins depth-orders: every non-empty bin of at most kSortMaxBig entries that is read as a list.
// The fine stages treat exactly these bins as sorted (the point stage reads their bucket map for its exit bound),
// so the sort and both fine stages share this one predicate.
__host__ __device__ __forceinline__ bool bin_is_sorted(int64_t off, int cnt, int64_t pool, int cap) {
  return cnt > 0 && cnt <= kSortMaxBig && bin_fits(off, cnt, pool, cap);
}
// Depth-bucket order of a bin (k_sort_bins): keys [lo, hi] map linearly onto kSortBucketsH buckets.
// Shared with the point fine stage, which bounds the keys of the rest of a bin from the bucket of its next entry.
constexpr int kSortBpt = 4;  // bucket counts per thread of the sort's scan (256 threads)
constexpr int kSortBucketsH = 256 * kSortBpt;
__device__ __forceinline__ float sort_bucket_scale(float lo, float hi) {
  return hi > lo ? (float)kSortBucketsH * 0.99999f / (hi - lo) : 0.f;
}
__device__ __forceinline__ int sort_bucket(float key, float lo, float scale) {
  return min(kSortBucketsH - 1, max(0, __float2int_rz((key - lo) * scale)));  // NaN/inf range -> bucket 0
}

cudaError_t launch_sort_bins(const int* counts, const int64_t* off, int4* entries, const int4* ibbox,
                             int64_t nbins_total, int64_t pool, int cap, cudaStream_t st,
                             float2* bin_range = nullptr);
cudaError_t launch_fine(const FineArgs<float>& A, int nwarps, cudaStream_t st);
cudaError_t launch_fine(const FineArgs<double>& A, int nwarps, cudaStream_t st);
cudaError_t launch_backward(const BwdArgs<float>& A, cudaStream_t st);
cudaError_t launch_backward(const BwdArgs<double>& A, cudaStream_t st);
cudaError_t launch_silhouette_backward(const SilBwdArgs& A, cudaStream_t st);
size_t fine_warp_smem_bytes(int K);  // shared memory one warp of K2 needs

}  // namespace drb
