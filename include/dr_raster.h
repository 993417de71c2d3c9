/*
 * dr_raster.h — C-ABI of the B200-native rasterize_meshes hot path (libdr_raster_b200.so).
 *
 * Replaces, on the north-star boundary (BASELINE.json):
 *   dr::rasterize_meshes        /root/reference/proj/include/dr/mesh_raster.hpp:41  (src/mesh_raster.cpp:234-285)
 *   dr::rasterize_meshes_naive  /root/reference/proj/include/dr/mesh_raster.hpp:44  (src/mesh_raster.cpp:214-232)
 *   dr::rasterize_backward      /root/reference/proj/include/dr/mesh_raster.hpp:66-69 (src/mesh_raster.cpp:329-403)
 *   dr::RasterSettings          /root/reference/proj/include/dr/mesh_raster.hpp:18-23
 *   dr::MeshFragments           /root/reference/proj/include/dr/mesh_raster.hpp:28-39
 *
 * The reference consumes MeshBatch + Camera; this ABI consumes what the reference derives from them:
 *   face_verts [F,3,3] fp64       per face vertex (x_ndc, y_ndc, z_view) = world_to_ndc (camera.cpp:36-70)
 *                                 gathered through MeshBatch::faces_packed (batching.hpp:100-103)
 *   mesh_to_face_first_idx [N]    MeshBatch::faces_packed().offsets[0..N)   (batching.hpp:20-27)
 *   num_faces_per_mesh [N]        MeshBatch::num_faces_per_mesh()           (batching.hpp:98)
 * Camera knowledge that face_verts cannot carry travels in the settings (znear, clip_nonpositive_z).
 *
 * Conventions
 *   - All array pointers are DEVICE pointers, caller-owned, stream-ordered on `stream`.
 *   - Fragment layout is the reference's row-major [N,H,W,K] (mesh_raster.hpp:36-38):
 *     slot = ((b*H + i)*W + j)*K + s; bary_coords has a trailing dimension of 3.
 *   - Empty slots: pix_to_face -1, zbuf -1, bary 0, pix_dists 0 (mesh_raster.cpp:191-195, 205-208).
 *   - No exceptions cross the ABI: every entry point returns a dr_status; dr_last_error() holds a
 *     thread-local message for the last failure on the calling thread.
 *   - Reentrant: no global state besides the per-thread error message, the launch counter and the
 *     optional profiling ring (dr_profile_*), which are diagnostics only.
 *   - There is no CPU fallback: without a usable CUDA device every compute entry point fails with
 *     DR_ERR_CUDA.
 */
#ifndef DR_RASTER_H
#define DR_RASTER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ABI-compatible with cudaStream_t without requiring CUDA headers (NULL = legacy default stream). */
typedef struct CUstream_st* dr_stream_t;

typedef enum {
  DR_OK = 0,
  DR_ERR_SHAPE = 1, /* dr::ShapeError  (batching.cpp:10-31, mesh_raster.cpp:333-336) */
  DR_ERR_INDEX = 2, /* dr::IndexError  (batching.cpp:17-21) */
  DR_ERR_RANGE = 3, /* dr::RangeError  (core.hpp:38-40): settings out of range */
  DR_ERR_CUDA = 4,  /* CUDA runtime failure / no device */
  DR_ERR_OOM = 5,   /* workspace too small or allocation failure */
  DR_ERR_USAGE = 6  /* dr::UsageError (core.hpp:47-49): null pointers, bad arguments */
} dr_status;

/* RasterSettings (mesh_raster.hpp:18-23) plus the north-star parameters. Zero-initialise, then set. */
typedef struct dr_raster_settings {
  int32_t image_h, image_w;    /* RasterSettings.image_h / image_w, >= 1 */
  int32_t faces_per_pixel;     /* K >= 1 (RasterSettings.faces_per_pixel) */
  int32_t bin_size;            /* 0 => naive semantics (mesh_raster.cpp:214); > 0 => coarse-to-fine with
                                  bins of bin_size x bin_size pixels (RasterSettings.tile_size) */
  int32_t max_faces_per_bin;   /* longest bin list the fast path uses; 0 => unlimited (lists are sized
                                  exactly: count -> scan -> fill). A longer bin (or one past the list pool)
                                  is rasterized by the spill path: results never change (reference bins
                                  are unbounded, mesh_raster.cpp:244) */
  int32_t _reserved0;          /* must be 0 */
  double blur_radius;          /* squared NDC distance (RasterSettings.blur_radius) */
  double znear;                /* Camera.znear (camera.hpp:26): all-behind cull (mesh_raster.cpp:113) and the
                                  per-pixel z cut (mesh_raster.cpp:174) */
  uint8_t clip_nonpositive_z;  /* 1 for perspective cameras: drop faces with any vertex z_view <= 0
                                  (world_to_ndc's `clipped`, camera.cpp:44-47, mesh_raster.cpp:112) */
  uint8_t perspective_correct; /* 0 = reference behaviour; 1 = builder-defined correction */
  uint8_t clip_barycentric_coords; /* 1 = reference behaviour (always clamps, mesh_raster.cpp:172) */
  uint8_t cull_backfaces;      /* 0 = reference; 1 = drop faces whose NDC signed_area2 > 0 */
  uint8_t _reserved1[4];       /* must be 0 */
} dr_raster_settings;

/* Fill `s` with the reference defaults (RasterSettings{} + Camera{} + perspective): 64x64, K=1,
 * blur 1e-4, bin 16, znear 0.1, clip_nonpositive_z=1, clip_barycentric_coords=1, others 0. */
void dr_raster_settings_default(dr_raster_settings* s);

/* Workspace bytes the forward needs for (N meshes, F packed faces, settings). */
size_t dr_rasterize_meshes_workspace_bytes(int64_t N, int64_t F, const dr_raster_settings* s);

/* Forward (rasterize_meshes): fp32 fragment payload (zbuf, bary, dists), int64 pix_to_face.
 * pix_to_face/zbuf/pix_dists: [N,H,W,K]; bary_coords: [N,H,W,K,3]. Every slot is written. */
int dr_rasterize_meshes_fwd(const double* face_verts, const int64_t* mesh_to_face_first_idx,
                            const int64_t* num_faces_per_mesh, int64_t N, int64_t F,
                            const dr_raster_settings* s, int64_t* pix_to_face, float* zbuf,
                            float* bary_coords, float* pix_dists, void* workspace, size_t workspace_bytes,
                            dr_stream_t stream);

/* Same contract with fp64 payload: bit-identical to the reference MeshFragments (mesh_raster.hpp:28-39). */
int dr_rasterize_meshes_fwd_f64(const double* face_verts, const int64_t* mesh_to_face_first_idx,
                                const int64_t* num_faces_per_mesh, int64_t N, int64_t F,
                                const dr_raster_settings* s, int64_t* pix_to_face, double* zbuf,
                                double* bary_coords, double* pix_dists, void* workspace,
                                size_t workspace_bytes, dr_stream_t stream);

/* Backward (rasterize_backward, mesh_raster.cpp:345-378): cotangents on zbuf [N,H,W,K], bary [N,H,W,K,3],
 * dists [N,H,W,K] pulled back to grad_face_verts [F,3,3] = d(x_ndc, y_ndc, z_view) per face vertex.
 * The rows of the batch's face ranges are overwritten; rows of faces outside every mesh range are left
 * untouched (so disjoint groups of meshes of one packed buffer can be processed by separate calls).
 * pix_to_face / bary_coords are the forward's outputs for the same batch (the reference reads frag.bary,
 * mesh_raster.cpp:359).
 * Accumulation uses fp64 atomics: the summation order is not fixed, results agree to ~1e-15 relative.
 * The cotangents must be device memory (DR_ERR_USAGE otherwise, page-locked host memory included). */
int dr_rasterize_meshes_bwd(const double* face_verts, const int64_t* mesh_to_face_first_idx,
                            const int64_t* num_faces_per_mesh, int64_t N, int64_t F,
                            const dr_raster_settings* s, const int64_t* pix_to_face, const float* bary_coords,
                            const float* grad_zbuf, const float* grad_bary, const float* grad_dists,
                            double* grad_face_verts, dr_stream_t stream);

/* fp64 variant (bary and cotangents in fp64, as the reference's std::vector<double>). */
int dr_rasterize_meshes_bwd_f64(const double* face_verts, const int64_t* mesh_to_face_first_idx,
                                const int64_t* num_faces_per_mesh, int64_t N, int64_t F,
                                const dr_raster_settings* s, const int64_t* pix_to_face,
                                const double* bary_coords, const double* grad_zbuf, const double* grad_bary,
                                const double* grad_dists, double* grad_face_verts, dr_stream_t stream);

/* Asynchronous variants: identical contracts, plus HOST copies of mesh_to_face_first_idx / num_faces_per_mesh
 * (validation and grid sizing then need no device read-back, so the call does not synchronise `stream` and
 * can be enqueued ahead in a copy/compute pipeline). The device arrays must hold the same values. */
int dr_rasterize_meshes_fwd_hr(const double* face_verts, const int64_t* mesh_to_face_first_idx,
                               const int64_t* num_faces_per_mesh, int64_t N, int64_t F, const dr_raster_settings* s,
                               int64_t* pix_to_face, float* zbuf, float* bary_coords, float* pix_dists,
                               void* workspace, size_t workspace_bytes, dr_stream_t stream,
                               const int64_t* host_first, const int64_t* host_num);
int dr_rasterize_meshes_bwd_hr(const double* face_verts, const int64_t* mesh_to_face_first_idx,
                               const int64_t* num_faces_per_mesh, int64_t N, int64_t F, const dr_raster_settings* s,
                               const int64_t* pix_to_face, const float* bary_coords, const float* grad_zbuf,
                               const float* grad_bary, const float* grad_dists, double* grad_face_verts,
                               dr_stream_t stream, const int64_t* host_first, const int64_t* host_num);

/* ---- camera side of the path: MeshBatch + Camera <-> face_verts on the GPU ---- */

/* dr::Camera (camera.hpp:19-35). */
typedef struct dr_camera {
  int32_t perspective;        /* 1 = ProjectionKind::Perspective, 0 = Orthographic */
  int32_t _reserved0;
  double rotation[9];         /* world -> view, row-major */
  double translation[3];      /* world -> view */
  double focal_length;        /* perspective */
  double principal_point[2];  /* perspective, NDC units */
  double ortho_scale[2];      /* orthographic, per axis */
  double znear, zfar;
} dr_camera;

/* world_to_ndc (camera.cpp:36-70) of every packed vertex gathered per face (prepare_faces,
 * mesh_raster.cpp:100-122): verts [V,3] world space, faces [F,3] packed GLOBAL vertex indices
 * (MeshBatch::faces_packed) -> face_verts [F,3,3] (x_ndc, y_ndc, z_view); a clipped vertex (perspective,
 * z_view <= 0) gets xy = (0,0) like the reference. Bit-identical to the reference's NdcPoints.
 * Out-of-range vertex indices -> DR_ERR_INDEX (synchronises the stream to report it). */
int dr_world_to_face_verts(const double* verts, int64_t V, const int64_t* faces, int64_t F, const dr_camera* cam,
                           double* face_verts, dr_stream_t stream);
/* Same without the synchronising index check: a face with a vertex index outside [0, V) sets *bad_index = 1
 * (device int, may be NULL) and that vertex's face_verts entries are NaN (the face is culled downstream). For callers that validated the topology
 * once (a fit loop) and for CUDA-graph capture. */
int dr_world_to_face_verts_async(const double* verts, int64_t V, const int64_t* faces, int64_t F,
                                 const dr_camera* cam, double* face_verts, int* bad_index, dr_stream_t stream);

/* Reverse of the above (mesh_raster.cpp:380-401): grad_face_verts [F,3,3] scattered to vertices and pulled
 * through world_to_ndc_backward (camera.cpp:72-85) -> grad_verts [V,3] world space (overwritten). */
int dr_face_verts_backward(const double* verts, int64_t V, const int64_t* faces, int64_t F, const dr_camera* cam,
                           const double* grad_face_verts, double* grad_verts, dr_stream_t stream);

/* ---- packed <-> padded batch bookkeeping (batching.hpp:20-27, 48-75) on the GPU ---- */

/* padded[b, j, :] = packed[first[b] + j, :] for j < num[b], else pad_row (NULL = zeros). Rows are opaque
 * row_bytes-byte records; padded is [N, max_count, row_bytes]. first/num are device arrays. */
int dr_packed_to_padded(const void* packed, const int64_t* first, const int64_t* num, int64_t N, int64_t max_count,
                        int64_t row_bytes, const void* pad_row, void* padded, dr_stream_t stream);
/* packed[first[b] + j, :] = padded[b, j, :] for j < num[b]. */
int dr_padded_to_packed(const void* padded, const int64_t* first, const int64_t* num, int64_t N, int64_t max_count,
                        int64_t row_bytes, void* packed, dr_stream_t stream);
/* out[i] = the batch element owning packed row i (PackedView::item_to_element), -1 for rows in no range. */
int dr_packed_item_to_element(const int64_t* first, const int64_t* num, int64_t N, int64_t total, int32_t* out,
                              dr_stream_t stream);

/* ---- streamed host pipeline (the reference's host-in / host-out calling convention, mesh_raster.hpp:41,66-69) ----
 * rasterize_meshes forward (+ backward) between HOST buffers and the GPU: the batch is cut into contiguous groups
 * of meshes balanced by PCIe bytes (smaller groups at both ends, `ramp`) and run on three streams so H2D of
 * group g+1, the kernels of group g and D2H of group g-1 overlap; group g's H2D waits for the D2H of group
 * g - lookahead (0: no gating). Host ranges: ordered, non-overlapping mesh ranges of the packed batch (host
 * arrays). The pipeline owns its device buffers (one allocation) and streams; run() is stream-ordered: it
 * enqueues everything and makes `stream` wait for completion. Host buffers should be page-locked for the copies
 * to overlap. fp32 payload / cotangents (the dr_rasterize_meshes_fwd / _bwd layouts), fp64 grad_face_verts. */
typedef struct dr_host_pipeline* dr_host_pipeline_t;
int dr_host_pipeline_create(const int64_t* host_first, const int64_t* host_num, int64_t N, int64_t F,
                            const dr_raster_settings* s, int32_t n_groups, int32_t ramp, int32_t lookahead,
                            int32_t backward, dr_host_pipeline_t* out);
/* Number of groups; writes up to cap [g0, g1) mesh ranges into bounds[2 * g], bounds[2 * g + 1]. */
int dr_host_pipeline_groups(dr_host_pipeline_t p, int64_t* bounds, int64_t cap);
int dr_host_pipeline_run(dr_host_pipeline_t p, const double* face_verts, int64_t* pix_to_face, float* zbuf,
                         float* bary_coords, float* pix_dists, const float* grad_zbuf, const float* grad_bary,
                         const float* grad_dists, double* grad_face_verts, dr_stream_t stream);
int dr_host_pipeline_destroy(dr_host_pipeline_t p);

/* ---- fused fragment consumer: silhouette ----
 * dr_rasterize_silhouette_fwd = silhouette_blend(rasterize_meshes(...), sigma)
 *   (shading.cpp:75-91 over mesh_raster.cpp:234): alpha [N,H,W] fp32 = 1 - prod_k (1 - sigmoid(-dist_k / sigma))
 *   over the occupied slots of each pixel; pix_to_face [N,H,W,K] (may be NULL) is bit-exact with
 *   dr_rasterize_meshes_fwd. zbuf / bary / dists are never written to memory. Same workspace as the forward.
 * dr_rasterize_silhouette_bwd = rasterize_backward(..., d_zbuf = 0, d_bary = 0,
 *   silhouette_blend_backward(frag, sigma, d_alpha)) (shading.cpp:93-121, mesh_raster.cpp:329-403): the
 *   reference fit loop's step (pipeline.cpp:153-162); grad_face_verts [F,3,3] is overwritten on the batch's
 *   face ranges. sigma must be > 0 (DR_ERR_RANGE). */
int dr_rasterize_silhouette_fwd(const double* face_verts, const int64_t* mesh_to_face_first_idx,
                                const int64_t* num_faces_per_mesh, int64_t N, int64_t F, const dr_raster_settings* s,
                                double sigma, int64_t* pix_to_face, float* alpha, void* workspace,
                                size_t workspace_bytes, dr_stream_t stream);
int dr_rasterize_silhouette_bwd(const double* face_verts, const int64_t* mesh_to_face_first_idx,
                                const int64_t* num_faces_per_mesh, int64_t N, int64_t F, const dr_raster_settings* s,
                                double sigma, const int64_t* pix_to_face, const float* grad_alpha,
                                double* grad_face_verts, dr_stream_t stream);
/* fp64 alpha / fp64 cotangent variants (the fit loop, pipeline.cpp:100-205, where Adam's per-coordinate
 * normalisation amplifies fp32 rounding in near-zero gradients): alpha matches silhouette_blend of the fp64
 * MeshFragments to a few ulps; the backward evaluates the sigmoid in fp64. */
int dr_rasterize_silhouette_fwd_f64(const double* face_verts, const int64_t* mesh_to_face_first_idx,
                                    const int64_t* num_faces_per_mesh, int64_t N, int64_t F,
                                    const dr_raster_settings* s, double sigma, int64_t* pix_to_face, double* alpha,
                                    void* workspace, size_t workspace_bytes, dr_stream_t stream);
int dr_rasterize_silhouette_bwd_f64(const double* face_verts, const int64_t* mesh_to_face_first_idx,
                                    const int64_t* num_faces_per_mesh, int64_t N, int64_t F,
                                    const dr_raster_settings* s, double sigma, const int64_t* pix_to_face,
                                    const double* grad_alpha, double* grad_face_verts, dr_stream_t stream);
/* Asynchronous fp64 silhouette (host copies of the mesh ranges, as dr_rasterize_meshes_fwd_hr): no call
 * synchronises or allocates, so a whole fit iteration can be captured into one CUDA graph (fit.py). */
int dr_rasterize_silhouette_fwd_f64_hr(const double* face_verts, const int64_t* mesh_to_face_first_idx,
                                       const int64_t* num_faces_per_mesh, int64_t N, int64_t F,
                                       const dr_raster_settings* s, double sigma, int64_t* pix_to_face,
                                       double* alpha, void* workspace, size_t workspace_bytes, dr_stream_t stream,
                                       const int64_t* host_first, const int64_t* host_num);
int dr_rasterize_silhouette_bwd_f64_hr(const double* face_verts, const int64_t* mesh_to_face_first_idx,
                                       const int64_t* num_faces_per_mesh, int64_t N, int64_t F,
                                       const dr_raster_settings* s, double sigma, const int64_t* pix_to_face,
                                       const double* grad_alpha, double* grad_face_verts, dr_stream_t stream,
                                       const int64_t* host_first, const int64_t* host_num);

/* ---- fused fragment consumer: softmax render ----
 * The reference's differentiable softmax render (grad.cpp:177-209): rasterize_meshes -> interpolate_face_attributes
 * of per-vertex colours with the clamped barycentrics (shading.cpp:11-32) -> softmax_blend (shading.cpp:123-160).
 * dr_rasterize_softmax_fwd writes image [N,H,W,3] fp32 (and pix_to_face, may be NULL); no fragment payload is
 * materialised. dr_rasterize_softmax_bwd chains softmax_blend_backward (shading.cpp:162-230) ->
 * interpolate_face_attributes_backward (shading.cpp:35-73) -> rasterize_backward (mesh_raster.cpp:329-378):
 * grad_face_verts [F,3,3] (overwritten on the batch's face ranges) and grad_vert_colors [V,3] (overwritten).
 * faces [F,3] = MeshBatch::faces_packed() global vertex ids (must be valid: they are not re-checked here);
 * vert_colors [V,3] fp64. faces_per_pixel <= 64 for the backward. */
typedef struct dr_blend_params {
  double sigma;          /* BlendParams.sigma (shading.hpp:14), > 0 */
  double gamma;          /* BlendParams.gamma (shading.hpp:15), > 0 */
  double background[3];  /* BlendParams.background_color */
  double znear, zfar;    /* Camera.znear / zfar (softmax_blend's depth normalisation) */
} dr_blend_params;
int dr_rasterize_softmax_fwd(const double* face_verts, const int64_t* mesh_to_face_first_idx,
                             const int64_t* num_faces_per_mesh, int64_t N, int64_t F, const dr_raster_settings* s,
                             const dr_blend_params* blend, const double* vert_colors, const int64_t* faces, int64_t V,
                             int64_t* pix_to_face, float* image, void* workspace, size_t workspace_bytes,
                             dr_stream_t stream);
int dr_rasterize_softmax_bwd(const double* face_verts, const int64_t* mesh_to_face_first_idx,
                             const int64_t* num_faces_per_mesh, int64_t N, int64_t F, const dr_raster_settings* s,
                             const dr_blend_params* blend, const double* vert_colors, const int64_t* faces, int64_t V,
                             const int64_t* pix_to_face, const float* grad_image, double* grad_face_verts,
                             double* grad_vert_colors, dr_stream_t stream);

/* ---- point rasterizer ----
 * Replaces dr::rasterize_points / rasterize_points_naive (point_render.hpp:33-36, point_render.cpp:82-155) on the
 * same boundary as the meshes: points_ndc [P,3] fp64 = world_to_ndc (x_ndc, y_ndc, z_view) of the packed points
 * (PointCloudBatch::points_packed, batching.hpp:138), cloud_to_packed_first_idx / num_points_per_cloud [N] int64.
 * Outputs PointFragments (point_render.hpp:21-30): idx int64 [N,H,W,K] (packed point id, -1 empty), zbuf
 * [N,H,W,K] (z_view, -1 empty), dists2 [N,H,W,K] (squared NDC distance, 0 empty); occupied slots ascending in
 * (z, id). fp32 payload, or fp64 (_f64, bit-identical to the reference). */
typedef struct dr_point_raster_settings {
  int32_t image_h, image_w;   /* PointRasterSettings.image_h / image_w */
  int32_t points_per_pixel;   /* K in [1, 128] */
  int32_t bin_size;           /* 0 => rasterize_points_naive; > 0 => tiled (PointRasterSettings.tile_size) */
  double radius;              /* splat radius in NDC (PointRasterSettings.radius); r2 = radius * radius */
  double znear;               /* Camera.znear: points with z_view < znear are dropped (point_render.cpp:26) */
  uint8_t clip_nonpositive_z; /* 1 for perspective cameras: drop points with z_view <= 0 (NdcPoint.clipped) */
  uint8_t _reserved[7];       /* must be 0 */
} dr_point_raster_settings;

void dr_point_raster_settings_default(dr_point_raster_settings* s);
size_t dr_rasterize_points_workspace_bytes(int64_t N, int64_t P, const dr_point_raster_settings* s);
int dr_rasterize_points_fwd(const double* points_ndc, const int64_t* cloud_to_packed_first_idx,
                            const int64_t* num_points_per_cloud, int64_t N, int64_t P,
                            const dr_point_raster_settings* s, int64_t* idx, float* zbuf, float* dists2,
                            void* workspace, size_t workspace_bytes, dr_stream_t stream);
int dr_rasterize_points_fwd_f64(const double* points_ndc, const int64_t* cloud_to_packed_first_idx,
                                const int64_t* num_points_per_cloud, int64_t N, int64_t P,
                                const dr_point_raster_settings* s, int64_t* idx, double* zbuf, double* dists2,
                                void* workspace, size_t workspace_bytes, dr_stream_t stream);
/* grad_points_ndc [P,3] (overwritten on the batch's point ranges) = sum over occupied slots of
 * (-2 (px - x) g_dists2, -2 (py - y) g_dists2, g_zbuf). The reference's splat_position_backward
 * (point_render.cpp:302-338) is this with g_dists2 = -d_alpha / radius^2, g_zbuf = 0, then dr_points_ndc_backward. */
int dr_rasterize_points_bwd(const double* points_ndc, const int64_t* cloud_to_packed_first_idx,
                            const int64_t* num_points_per_cloud, int64_t N, int64_t P,
                            const dr_point_raster_settings* s, const int64_t* idx, const float* grad_zbuf,
                            const float* grad_dists2, double* grad_points_ndc, dr_stream_t stream);
int dr_rasterize_points_bwd_f64(const double* points_ndc, const int64_t* cloud_to_packed_first_idx,
                                const int64_t* num_points_per_cloud, int64_t N, int64_t P,
                                const dr_point_raster_settings* s, const int64_t* idx, const double* grad_zbuf,
                                const double* grad_dists2, double* grad_points_ndc, dr_stream_t stream);
/* world_to_ndc (camera.cpp:36-70) of P packed points -> points_ndc [P,3], and its backward (camera.cpp:72-85). */
int dr_world_to_points_ndc(const double* points, int64_t P, const dr_camera* cam, double* points_ndc,
                           dr_stream_t stream);
int dr_points_ndc_backward(const double* points, int64_t P, const dr_camera* cam, const double* grad_points_ndc,
                           double* grad_points, dr_stream_t stream);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char* dr_last_error(void);

/* ---- diagnostics (not part of the reference surface) ---- */

/* Reads the coarse-stage counters a forward left in `workspace` (synchronises `stream`):
 * out[0] = bins, out[1] = bins on the spill path (longer than max_faces_per_bin or past the list pool),
 * out[2] = total bin entries,
 * out[3] = largest bin. Returns DR_ERR_USAGE for bin_size == 0. */
int dr_rasterize_meshes_bin_stats(int64_t N, int64_t F, const dr_raster_settings* s, const void* workspace,
                                  dr_stream_t stream, int64_t out[4]);

/* Device self-test of the grouped exact division every selection-path quotient uses (raster_math.cuh xdiv_*):
 * compares it bit for bit with IEEE a/b on n pseudo-random hard-case triples. Writes the mismatch count (and the
 * first mismatching a, b) and returns 0, or DR_ERR_CUDA. Synchronous. */
int dr_selftest_division(uint64_t n, uint64_t seed, uint64_t* mismatches, double first_bad_ab[2]);

/* Number of kernels this library has launched in this process. */
uint64_t dr_launch_count(void);

/* Optional per-kernel CUDA-event timing (on the launching stream). enable=1 starts recording (clears the
 * ring); dr_profile_read synchronises and returns up to `cap` entries (name index, milliseconds).
 * Names: dr_profile_kernel_name(idx). */
void dr_profile_enable(int enable);
int dr_profile_read(int* kernel_idx, float* ms, int cap);
const char* dr_profile_kernel_name(int idx);

#ifdef __cplusplus
}
#endif
#endif /* DR_RASTER_H */
