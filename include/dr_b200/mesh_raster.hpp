// dr_b200 — C++ host mirror of the reference's rasterizer interface, running on the B200 C-ABI.
//
// Same names, argument meaning and error behaviour as the reference (/root/reference/proj):
//   MeshBatch            include/dr/batching.hpp:86-125   (validation: ShapeError / IndexError, batching.cpp:10-31)
//   Camera               include/dr/camera.hpp:19-35
//   RasterSettings       include/dr/mesh_raster.hpp:18-23 (+ the north-star flags, reference defaults)
//   MeshFragments        include/dr/mesh_raster.hpp:28-39 (fp64 payload: bit-identical to the reference)
//   rasterize_meshes / rasterize_meshes_naive / rasterize_backward   include/dr/mesh_raster.hpp:41,44,66-69
// so code written against dr:: ports by changing the namespace. Every call runs on the current CUDA device:
// vertices and faces go to HBM, world_to_ndc + the face gather, the rasterizer and its backward, the vertex
// scatter and world_to_ndc_backward all run as sm_100a kernels (include/dr_raster.h); results come back to
// host vectors like the reference's by-value returns. There is no CPU fallback (CudaError without a GPU).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace dr_b200 {

struct ShapeError : std::runtime_error {
  explicit ShapeError(const std::string& m) : std::runtime_error("ShapeError: " + m) {}
};
struct IndexError : std::runtime_error {
  explicit IndexError(const std::string& m) : std::runtime_error("IndexError: " + m) {}
};
struct RangeError : std::runtime_error {
  explicit RangeError(const std::string& m) : std::runtime_error("RangeError: " + m) {}
};
struct UsageError : std::runtime_error {
  explicit UsageError(const std::string& m) : std::runtime_error("UsageError: " + m) {}
};
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& m) : std::runtime_error("CudaError: " + m) {}
};

struct Vec2 {
  double x = 0, y = 0;
};
struct Vec3 {
  double x = 0, y = 0, z = 0;
};
struct Face {
  int64_t a = 0, b = 0, c = 0;
};
struct Mat3 {
  double m[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  static Mat3 identity() { return {}; }
};

template <typename T>
struct PackedView {
  std::vector<T> data;
  std::vector<int64_t> offsets;  // B+1
};

class MeshBatch {
 public:
  // ShapeError on mismatched list lengths, an empty batch or a zero-vertex mesh; IndexError on an
  // out-of-range face index. Zero-face meshes are legal (batching.cpp:10-31).
  MeshBatch(std::vector<std::vector<Vec3>> verts_list, std::vector<std::vector<Face>> faces_list);

  int size() const { return int(verts_list_.size()); }
  const std::vector<std::vector<Vec3>>& verts_list() const { return verts_list_; }
  const std::vector<std::vector<Face>>& faces_list() const { return faces_list_; }
  const std::vector<int64_t>& num_verts_per_mesh() const { return num_verts_; }
  const std::vector<int64_t>& num_faces_per_mesh() const { return num_faces_; }
  const PackedView<Vec3>& verts_packed() const { return verts_packed_; }
  const PackedView<Face>& faces_packed() const { return faces_packed_; }  // globally offset indices
  int64_t total_verts() const { return verts_packed_.offsets.back(); }
  int64_t total_faces() const { return faces_packed_.offsets.back(); }
  MeshBatch with_verts(const std::vector<Vec3>& new_verts_packed) const;

 private:
  std::vector<std::vector<Vec3>> verts_list_;
  std::vector<std::vector<Face>> faces_list_;
  std::vector<int64_t> num_verts_, num_faces_;
  PackedView<Vec3> verts_packed_;
  PackedView<Face> faces_packed_;
};

enum class ProjectionKind { Orthographic, Perspective };

struct Camera {
  Mat3 rotation;
  Vec3 translation;
  ProjectionKind kind = ProjectionKind::Perspective;
  double focal_length = 1.0;
  Vec2 principal_point{};
  Vec2 ortho_scale{1.0, 1.0};
  double znear = 0.1;
  double zfar = 100.0;

  static Camera orthographic(Mat3 r, Vec3 t, Vec2 scale = {1, 1}, double znear = 0.1, double zfar = 100.0);
  static Camera perspective(Mat3 r, Vec3 t, double focal = 1.0, Vec2 pp = {}, double znear = 0.1,
                            double zfar = 100.0);
  static Camera look_from_distance(double d, ProjectionKind kind, double focal = 1.0);
};

struct RasterSettings {
  int image_h = 64, image_w = 64;
  int faces_per_pixel = 1;       // K
  double blur_radius = 1e-4;     // squared NDC distance
  int tile_size = 16;            // bin side in pixels (north-star `bin_size`)
  // north-star parameters (defaults = the reference's only behaviour)
  int max_faces_per_bin = 0;     // 0 = unlimited (exact-size lists); overflow never changes results
  bool perspective_correct = false;
  bool clip_barycentric_coords = true;
  bool cull_backfaces = false;
};

struct MeshFragments {
  int batch = 0, h = 0, w = 0, k = 0;
  std::vector<int64_t> pix_to_face;
  std::vector<double> zbuf;
  std::vector<double> bary;   // ... x K x 3
  std::vector<double> dists;  // signed squared NDC distance

  int64_t slots() const { return int64_t(batch) * h * w * k; }
  int64_t slot(int b, int i, int j, int s) const { return ((int64_t(b) * h + i) * w + j) * k + s; }
};

// Page-locked host memory for the streamed pipeline's buffers (cudaHostAlloc): copies from / to it overlap the
// kernels; from pageable std::vector memory they would serialise.
template <typename T>
struct PinnedAllocator {
  using value_type = T;
  PinnedAllocator() = default;
  template <typename U>
  PinnedAllocator(const PinnedAllocator<U>&) {}
  T* allocate(size_t n);
  void deallocate(T* p, size_t) noexcept;
  template <typename U>
  bool operator==(const PinnedAllocator<U>&) const { return true; }
  template <typename U>
  bool operator!=(const PinnedAllocator<U>&) const { return false; }
};
template <typename T>
using pinned_vector = std::vector<T, PinnedAllocator<T>>;

// fp32-payload fragments in page-locked host memory (the layout of MeshFragments, floats instead of doubles):
// what HostPipeline streams back. pix_to_face is bit-identical to MeshFragments'; zbuf / bary / dists are the
// fp64 values rounded once (within 1e-5 relative / 1e-6 absolute of the reference, BASELINE north_star).
struct MeshFragments32 {
  int batch = 0, h = 0, w = 0, k = 0;
  pinned_vector<int64_t> pix_to_face;
  pinned_vector<float> zbuf;
  pinned_vector<float> bary;
  pinned_vector<float> dists;
  int64_t slots() const { return int64_t(batch) * h * w * k; }
  void resize(int b, int hh, int ww, int kk);
};

// The streamed host path (include/dr_raster.h dr_host_pipeline_*): forward + backward of one fixed batch layout
// between page-locked host buffers and the GPU, mesh groups pipelined over three CUDA streams (H2D of group g+1,
// kernels of g, D2H of g-1). Construct once per (batch layout, settings); run() per step. Inputs are the
// north-star boundary (packed face_verts [F,3,3] = world_to_ndc per face vertex, e.g. from face_verts_packed);
// outputs land in `out` / `grad_face_verts` when run() returns (it synchronises its stream).
class HostPipeline {
 public:
  HostPipeline(const std::vector<int64_t>& mesh_to_face_first_idx, const std::vector<int64_t>& num_faces_per_mesh,
               int64_t num_faces, const RasterSettings& s, const Camera& c, int n_groups = 24, int ramp = 2,
               int lookahead = 3, bool backward = true);
  ~HostPipeline();
  HostPipeline(const HostPipeline&) = delete;
  HostPipeline& operator=(const HostPipeline&) = delete;
  // face_verts [F*9]; cotangents fp32 in the fragment layout (bary x3); grad_face_verts [F*9] (fp64)
  void run(const pinned_vector<double>& face_verts, MeshFragments32& out, const pinned_vector<float>& d_zbuf,
           const pinned_vector<float>& d_bary, const pinned_vector<float>& d_dists,
           pinned_vector<double>& grad_face_verts);
  int groups() const;

 private:
  void* handle_ = nullptr;
  void* stream_ = nullptr;
  int n_ = 0, h_ = 0, w_ = 0, k_ = 0;
  int64_t f_ = 0;
  bool backward_ = true;
};

// world_to_ndc of every packed vertex gathered per face (the north-star face_verts [F,3,3]) into host memory.
pinned_vector<double> face_verts_packed(const MeshBatch& m, const Camera& c);

MeshFragments rasterize_meshes(const MeshBatch& m, const Camera& c, const RasterSettings& s);
MeshFragments rasterize_meshes_naive(const MeshBatch& m, const Camera& c, const RasterSettings& s);
std::vector<Vec3> rasterize_backward(const MeshBatch& m, const Camera& c, const RasterSettings& s,
                                     const MeshFragments& frag, const std::vector<double>& d_zbuf,
                                     const std::vector<double>& d_bary, const std::vector<double>& d_dists);

}  // namespace dr_b200
