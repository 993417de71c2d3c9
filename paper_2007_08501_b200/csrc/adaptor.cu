// dr_b200:: host adaptor (include/dr_b200/*.hpp): the reference's C++ surface on top of the C-ABI.
//
// rasterize_meshes:  verts/faces -> HBM -> dr_world_to_face_verts -> dr_rasterize_meshes_fwd_f64 -> host
// rasterize_backward: fragments + cotangents -> HBM -> dr_rasterize_meshes_bwd_f64 -> dr_face_verts_backward -> host
// rasterize_silhouette(_backward): the same with the fused silhouette entry points
// rasterize_points / splat_position_backward: points -> HBM -> dr_world_to_points_ndc -> dr_rasterize_points_*
// Error codes from the C-ABI are rethrown as the reference's exception types.
#include <cuda_runtime.h>

#include <cstring>
#include <new>
#include <string>
#include <utility>

#include "../../include/dr_b200/mesh_raster.hpp"
#include "../../include/dr_b200/point_render.hpp"
#include "../../include/dr_b200/shading.hpp"
#include "../../include/dr_raster.h"

namespace dr_b200 {

namespace {

[[noreturn]] void throw_status(int rc, const char* what) {
  std::string msg = std::string(what) + ": " + dr_last_error();
  switch (rc) {
    case DR_ERR_SHAPE: throw ShapeError(msg);
    case DR_ERR_INDEX: throw IndexError(msg);
    case DR_ERR_RANGE: throw RangeError(msg);
    case DR_ERR_USAGE: throw UsageError(msg);
    default: throw CudaError(msg);
  }
}

void check(int rc, const char* what) {
  if (rc != DR_OK) throw_status(rc, what);
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// RAII device buffer
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) {
    if (bytes) cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

template <typename T>
void upload(DevBuf& d, const T* h, size_t n) {
  if (n) cuda_check(cudaMemcpy(d.p, h, n * sizeof(T), cudaMemcpyHostToDevice), "H2D");
}
template <typename T>
void download(T* h, const DevBuf& d, size_t n) {
  if (n) cuda_check(cudaMemcpy(h, d.p, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
}

dr_camera to_c(const Camera& c) {
  dr_camera o;
  std::memset(&o, 0, sizeof(o));
  o.perspective = c.kind == ProjectionKind::Perspective ? 1 : 0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o.rotation[3 * i + j] = c.rotation.m[i][j];
  o.translation[0] = c.translation.x;
  o.translation[1] = c.translation.y;
  o.translation[2] = c.translation.z;
  o.focal_length = c.focal_length;
  o.principal_point[0] = c.principal_point.x;
  o.principal_point[1] = c.principal_point.y;
  o.ortho_scale[0] = c.ortho_scale.x;
  o.ortho_scale[1] = c.ortho_scale.y;
  o.znear = c.znear;
  o.zfar = c.zfar;
  return o;
}

dr_raster_settings to_c(const RasterSettings& s, const Camera& c, bool naive) {
  dr_raster_settings o;
  std::memset(&o, 0, sizeof(o));
  o.image_h = s.image_h;
  o.image_w = s.image_w;
  o.faces_per_pixel = s.faces_per_pixel;
  o.bin_size = naive ? 0 : s.tile_size;
  o.max_faces_per_bin = s.max_faces_per_bin;
  o.blur_radius = s.blur_radius;
  o.znear = c.znear;
  o.clip_nonpositive_z = c.kind == ProjectionKind::Perspective ? 1 : 0;
  o.perspective_correct = s.perspective_correct ? 1 : 0;
  o.clip_barycentric_coords = s.clip_barycentric_coords ? 1 : 0;
  o.cull_backfaces = s.cull_backfaces ? 1 : 0;
  return o;
}

// verts [V,3] and packed faces [F,3] on the device, projected to face_verts [F,3,3]
struct DeviceMesh {
  int64_t V, F, N;
  DevBuf verts, faces, fv, first, num;
  DeviceMesh(const MeshBatch& m, const Camera& c)
      : V(m.total_verts()),
        F(m.total_faces()),
        N(m.size()),
        verts(sizeof(double) * 3 * V),
        faces(sizeof(int64_t) * 3 * F),
        fv(sizeof(double) * 9 * F),
        first(sizeof(int64_t) * N),
        num(sizeof(int64_t) * N) {
    static_assert(sizeof(Vec3) == 3 * sizeof(double) && sizeof(Face) == 3 * sizeof(int64_t), "packed layout");
    upload(verts, reinterpret_cast<const double*>(m.verts_packed().data.data()), 3 * (size_t)V);
    upload(faces, reinterpret_cast<const int64_t*>(m.faces_packed().data.data()), 3 * (size_t)F);
    upload(first, m.faces_packed().offsets.data(), (size_t)N);  // offsets[0..N) = mesh_to_face_first_idx
    upload(num, m.num_faces_per_mesh().data(), (size_t)N);
    dr_camera cam = to_c(c);
    check(dr_world_to_face_verts(verts.as<double>(), V, faces.as<int64_t>(), F, &cam, fv.as<double>(), nullptr),
          "world_to_ndc");
  }
};

MeshFragments run_forward(const MeshBatch& m, const Camera& c, const RasterSettings& s, bool naive) {
  DeviceMesh d(m, c);
  dr_raster_settings rs = to_c(s, c, naive);
  size_t ws_bytes = dr_rasterize_meshes_workspace_bytes(d.N, d.F, &rs);
  if (ws_bytes == 0) throw_status(DR_ERR_RANGE, "rasterize_meshes");
  MeshFragments frag;
  frag.batch = m.size();
  frag.h = s.image_h;
  frag.w = s.image_w;
  frag.k = s.faces_per_pixel;
  const size_t S = (size_t)frag.slots();
  DevBuf ws(ws_bytes), p2f(sizeof(int64_t) * S), zbuf(sizeof(double) * S), bary(sizeof(double) * 3 * S),
      dists(sizeof(double) * S);
  check(dr_rasterize_meshes_fwd_f64(d.fv.as<double>(), d.first.as<int64_t>(), d.num.as<int64_t>(), d.N, d.F, &rs,
                                    p2f.as<int64_t>(), zbuf.as<double>(), bary.as<double>(), dists.as<double>(),
                                    ws.p, ws_bytes, nullptr),
        "rasterize_meshes");
  frag.pix_to_face.resize(S);
  frag.zbuf.resize(S);
  frag.bary.resize(3 * S);
  frag.dists.resize(S);
  download(frag.pix_to_face.data(), p2f, S);
  download(frag.zbuf.data(), zbuf, S);
  download(frag.bary.data(), bary, 3 * S);
  download(frag.dists.data(), dists, S);
  return frag;
}

}  // namespace

MeshBatch::MeshBatch(std::vector<std::vector<Vec3>> verts_list, std::vector<std::vector<Face>> faces_list)
    : verts_list_(std::move(verts_list)), faces_list_(std::move(faces_list)) {
  if (verts_list_.size() != faces_list_.size())
    throw ShapeError("verts_list and faces_list lengths differ: " + std::to_string(verts_list_.size()) + " vs " +
                     std::to_string(faces_list_.size()));
  if (verts_list_.empty()) throw ShapeError("empty mesh batch");
  const size_t n = verts_list_.size();
  num_verts_.resize(n);
  num_faces_.resize(n);
  verts_packed_.offsets.assign(n + 1, 0);
  faces_packed_.offsets.assign(n + 1, 0);
  for (size_t i = 0; i < n; ++i) {
    const int64_t nv = int64_t(verts_list_[i].size());
    if (nv == 0) throw ShapeError("mesh " + std::to_string(i) + " has zero vertices");
    num_verts_[i] = nv;
    num_faces_[i] = int64_t(faces_list_[i].size());
    for (const Face& f : faces_list_[i])
      for (int64_t idx : {f.a, f.b, f.c})
        if (idx < 0 || idx >= nv)
          throw IndexError("face index " + std::to_string(idx) + " out of range for mesh " + std::to_string(i) +
                           " with " + std::to_string(nv) + " verts");
    verts_packed_.offsets[i + 1] = verts_packed_.offsets[i] + nv;
    faces_packed_.offsets[i + 1] = faces_packed_.offsets[i] + num_faces_[i];
  }
  verts_packed_.data.reserve(size_t(verts_packed_.offsets.back()));
  faces_packed_.data.reserve(size_t(faces_packed_.offsets.back()));
  for (size_t i = 0; i < n; ++i) {
    verts_packed_.data.insert(verts_packed_.data.end(), verts_list_[i].begin(), verts_list_[i].end());
    const int64_t off = verts_packed_.offsets[i];
    for (const Face& f : faces_list_[i]) faces_packed_.data.push_back({f.a + off, f.b + off, f.c + off});
  }
}

MeshBatch MeshBatch::with_verts(const std::vector<Vec3>& new_verts_packed) const {
  if (int64_t(new_verts_packed.size()) != total_verts())
    throw ShapeError("with_verts: expected " + std::to_string(total_verts()) + " packed verts, got " +
                     std::to_string(new_verts_packed.size()));
  std::vector<std::vector<Vec3>> lists(verts_list_.size());
  for (size_t i = 0; i < verts_list_.size(); ++i) {
    auto b = new_verts_packed.begin() + verts_packed_.offsets[i];
    lists[i].assign(b, b + num_verts_[i]);
  }
  return MeshBatch(std::move(lists), faces_list_);
}

Camera Camera::orthographic(Mat3 r, Vec3 t, Vec2 scale, double znear, double zfar) {
  Camera c;
  c.rotation = r;
  c.translation = t;
  c.kind = ProjectionKind::Orthographic;
  c.ortho_scale = scale;
  c.znear = znear;
  c.zfar = zfar;
  return c;
}

Camera Camera::perspective(Mat3 r, Vec3 t, double focal, Vec2 pp, double znear, double zfar) {
  Camera c;
  c.rotation = r;
  c.translation = t;
  c.kind = ProjectionKind::Perspective;
  c.focal_length = focal;
  c.principal_point = pp;
  c.znear = znear;
  c.zfar = zfar;
  return c;
}

Camera Camera::look_from_distance(double d, ProjectionKind kind, double focal) {
  return kind == ProjectionKind::Perspective ? perspective(Mat3::identity(), {0, 0, d}, focal)
                                             : orthographic(Mat3::identity(), {0, 0, d});
}

MeshFragments rasterize_meshes(const MeshBatch& m, const Camera& c, const RasterSettings& s) {
  return run_forward(m, c, s, /*naive=*/s.tile_size <= 0);
}

template <typename T>
T* PinnedAllocator<T>::allocate(size_t n) {
  void* p = nullptr;
  if (n && cudaHostAlloc(&p, n * sizeof(T), cudaHostAllocDefault) != cudaSuccess) throw std::bad_alloc();
  return static_cast<T*>(p);
}
template <typename T>
void PinnedAllocator<T>::deallocate(T* p, size_t) noexcept {
  if (p) cudaFreeHost(p);
}
template struct PinnedAllocator<int64_t>;
template struct PinnedAllocator<float>;
template struct PinnedAllocator<double>;

void MeshFragments32::resize(int b, int hh, int ww, int kk) {
  batch = b;
  h = hh;
  w = ww;
  k = kk;
  const size_t S = (size_t)slots();
  pix_to_face.resize(S);
  zbuf.resize(S);
  bary.resize(3 * S);
  dists.resize(S);
}

pinned_vector<double> face_verts_packed(const MeshBatch& m, const Camera& c) {
  DeviceMesh d(m, c);
  pinned_vector<double> out(9 * (size_t)d.F);
  download(out.data(), d.fv, 9 * (size_t)d.F);
  return out;
}

HostPipeline::HostPipeline(const std::vector<int64_t>& first, const std::vector<int64_t>& num, int64_t num_faces,
                           const RasterSettings& s, const Camera& c, int n_groups, int ramp, int lookahead,
                           bool backward)
    : n_((int)num.size()), h_(s.image_h), w_(s.image_w), k_(s.faces_per_pixel), f_(num_faces), backward_(backward) {
  if (first.size() != num.size()) throw ShapeError("HostPipeline: first / num lengths differ");
  dr_raster_settings rs = to_c(s, c, s.tile_size <= 0);
  dr_host_pipeline_t h = nullptr;
  check(dr_host_pipeline_create(first.data(), num.data(), (int64_t)num.size(), num_faces, &rs, n_groups, ramp,
                                lookahead, backward ? 1 : 0, &h),
        "HostPipeline");
  handle_ = h;
  cudaStream_t st = nullptr;
  cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "HostPipeline stream");
  stream_ = st;
}

HostPipeline::~HostPipeline() {
  dr_host_pipeline_destroy(static_cast<dr_host_pipeline_t>(handle_));
  if (stream_) cudaStreamDestroy(static_cast<cudaStream_t>(stream_));
}

int HostPipeline::groups() const {
  return dr_host_pipeline_groups(static_cast<dr_host_pipeline_t>(handle_), nullptr, 0);
}

void HostPipeline::run(const pinned_vector<double>& face_verts, MeshFragments32& out,
                       const pinned_vector<float>& d_zbuf, const pinned_vector<float>& d_bary,
                       const pinned_vector<float>& d_dists, pinned_vector<double>& grad_face_verts) {
  const int64_t S = (int64_t)n_ * h_ * w_ * k_;
  if ((int64_t)face_verts.size() != 9 * f_) throw ShapeError("HostPipeline::run: face_verts is not [F,3,3]");
  if (backward_ && ((int64_t)d_zbuf.size() != S || (int64_t)d_bary.size() != 3 * S || (int64_t)d_dists.size() != S))
    throw ShapeError("HostPipeline::run: cotangent shapes do not match the fragments");  // mesh_raster.cpp:333-336
  if (out.batch != n_ || out.h != h_ || out.w != w_ || out.k != k_) out.resize(n_, h_, w_, k_);
  if (backward_) grad_face_verts.resize(9 * (size_t)f_);
  auto st = static_cast<cudaStream_t>(stream_);
  check(dr_host_pipeline_run(static_cast<dr_host_pipeline_t>(handle_), face_verts.data(), out.pix_to_face.data(),
                             out.zbuf.data(), out.bary.data(), out.dists.data(), backward_ ? d_zbuf.data() : nullptr,
                             backward_ ? d_bary.data() : nullptr, backward_ ? d_dists.data() : nullptr,
                             backward_ ? grad_face_verts.data() : nullptr, reinterpret_cast<dr_stream_t>(st)),
        "HostPipeline::run");
  cuda_check(cudaStreamSynchronize(st), "HostPipeline::run");
}

MeshFragments rasterize_meshes_naive(const MeshBatch& m, const Camera& c, const RasterSettings& s) {
  return run_forward(m, c, s, /*naive=*/true);
}

std::vector<Vec3> rasterize_backward(const MeshBatch& m, const Camera& c, const RasterSettings& s,
                                     const MeshFragments& frag, const std::vector<double>& d_zbuf,
                                     const std::vector<double>& d_bary, const std::vector<double>& d_dists) {
  const int64_t ns = frag.slots();
  if (int64_t(d_zbuf.size()) != ns || int64_t(d_dists.size()) != ns || int64_t(d_bary.size()) != ns * 3)
    throw ShapeError("rasterize_backward: cotangent shapes do not match fragments");  // mesh_raster.cpp:333-336
  if (int64_t(frag.pix_to_face.size()) != ns || int64_t(frag.bary.size()) != 3 * ns)
    throw ShapeError("rasterize_backward: fragment buffers do not match their dimensions");
  if (frag.batch != m.size() || frag.h != s.image_h || frag.w != s.image_w || frag.k != s.faces_per_pixel)
    throw ShapeError("rasterize_backward: fragments were not produced with these settings");
  DeviceMesh d(m, c);
  dr_raster_settings rs = to_c(s, c, false);
  DevBuf p2f(sizeof(int64_t) * ns), bary(sizeof(double) * 3 * ns), dz(sizeof(double) * ns),
      db(sizeof(double) * 3 * ns), dd(sizeof(double) * ns), gfv(sizeof(double) * 9 * d.F),
      gv(sizeof(double) * 3 * d.V);
  upload(p2f, frag.pix_to_face.data(), (size_t)ns);
  upload(bary, frag.bary.data(), 3 * (size_t)ns);
  upload(dz, d_zbuf.data(), (size_t)ns);
  upload(db, d_bary.data(), 3 * (size_t)ns);
  upload(dd, d_dists.data(), (size_t)ns);
  check(dr_rasterize_meshes_bwd_f64(d.fv.as<double>(), d.first.as<int64_t>(), d.num.as<int64_t>(), d.N, d.F, &rs,
                                    p2f.as<int64_t>(), bary.as<double>(), dz.as<double>(), db.as<double>(),
                                    dd.as<double>(), gfv.as<double>(), nullptr),
        "rasterize_backward");
  dr_camera cam = to_c(c);
  check(dr_face_verts_backward(d.verts.as<double>(), d.V, d.faces.as<int64_t>(), d.F, &cam, gfv.as<double>(),
                               gv.as<double>(), nullptr),
        "world_to_ndc_backward");
  std::vector<Vec3> out(size_t(d.V));
  download(reinterpret_cast<double*>(out.data()), gv, 3 * (size_t)d.V);
  return out;
}

// ---- fused silhouette (pipeline.cpp:153-162) ----

SilhouetteFragments rasterize_silhouette(const MeshBatch& m, const Camera& c, const RasterSettings& s, double sigma) {
  DeviceMesh d(m, c);
  dr_raster_settings rs = to_c(s, c, s.tile_size <= 0);
  size_t ws_bytes = dr_rasterize_meshes_workspace_bytes(d.N, d.F, &rs);
  if (ws_bytes == 0) throw_status(DR_ERR_RANGE, "rasterize_silhouette");
  SilhouetteFragments out;
  out.batch = m.size();
  out.h = s.image_h;
  out.w = s.image_w;
  out.k = s.faces_per_pixel;
  const size_t npix = (size_t)out.batch * out.h * out.w, S = npix * (size_t)out.k;
  DevBuf ws(ws_bytes), p2f(sizeof(int64_t) * S), alpha(sizeof(float) * npix);
  check(dr_rasterize_silhouette_fwd(d.fv.as<double>(), d.first.as<int64_t>(), d.num.as<int64_t>(), d.N, d.F, &rs,
                                    sigma, p2f.as<int64_t>(), alpha.as<float>(), ws.p, ws_bytes, nullptr),
        "rasterize_silhouette");
  out.pix_to_face.resize(S);
  download(out.pix_to_face.data(), p2f, S);
  std::vector<float> a(npix);
  download(a.data(), alpha, npix);
  out.alpha.assign(a.begin(), a.end());
  return out;
}

std::vector<Vec3> rasterize_silhouette_backward(const MeshBatch& m, const Camera& c, const RasterSettings& s,
                                                double sigma, const SilhouetteFragments& frag,
                                                const std::vector<double>& d_alpha) {
  const size_t npix = (size_t)frag.batch * frag.h * frag.w;
  if (d_alpha.size() != npix) throw ShapeError("silhouette_blend_backward: cotangent shape mismatch");  // SH:98
  if (frag.batch != m.size() || frag.h != s.image_h || frag.w != s.image_w || frag.k != s.faces_per_pixel ||
      frag.pix_to_face.size() != npix * (size_t)frag.k)
    throw ShapeError("rasterize_silhouette_backward: fragments were not produced with these settings");
  DeviceMesh d(m, c);
  dr_raster_settings rs = to_c(s, c, false);
  DevBuf p2f(sizeof(int64_t) * npix * frag.k), da(sizeof(float) * npix), gfv(sizeof(double) * 9 * d.F),
      gv(sizeof(double) * 3 * d.V);
  upload(p2f, frag.pix_to_face.data(), npix * (size_t)frag.k);
  std::vector<float> da32(d_alpha.begin(), d_alpha.end());
  upload(da, da32.data(), npix);
  check(dr_rasterize_silhouette_bwd(d.fv.as<double>(), d.first.as<int64_t>(), d.num.as<int64_t>(), d.N, d.F, &rs,
                                    sigma, p2f.as<int64_t>(), da.as<float>(), gfv.as<double>(), nullptr),
        "rasterize_silhouette_backward");
  dr_camera cam = to_c(c);
  check(dr_face_verts_backward(d.verts.as<double>(), d.V, d.faces.as<int64_t>(), d.F, &cam, gfv.as<double>(),
                               gv.as<double>(), nullptr),
        "world_to_ndc_backward");
  std::vector<Vec3> out(size_t(d.V));
  download(reinterpret_cast<double*>(out.data()), gv, 3 * (size_t)d.V);
  return out;
}

// ---- point clouds (point_render.cpp) ----

PointCloudBatch::PointCloudBatch(std::vector<std::vector<Vec3>> points_list) : points_list_(std::move(points_list)) {
  if (points_list_.empty()) throw ShapeError("empty point cloud batch");
  const size_t n = points_list_.size();
  num_points_.resize(n);
  points_packed_.offsets.assign(n + 1, 0);
  for (size_t i = 0; i < n; ++i) {
    num_points_[i] = int64_t(points_list_[i].size());
    points_packed_.offsets[i + 1] = points_packed_.offsets[i] + num_points_[i];
  }
  points_packed_.data.reserve(size_t(points_packed_.offsets.back()));
  for (const auto& l : points_list_) points_packed_.data.insert(points_packed_.data.end(), l.begin(), l.end());
}

PointCloudBatch PointCloudBatch::with_points(const std::vector<Vec3>& new_points_packed) const {
  if (int64_t(new_points_packed.size()) != total_points())
    throw ShapeError("with_points: expected " + std::to_string(total_points()) + " packed points, got " +
                     std::to_string(new_points_packed.size()));
  std::vector<std::vector<Vec3>> lists(points_list_.size());
  for (size_t i = 0; i < points_list_.size(); ++i) {
    auto b = new_points_packed.begin() + points_packed_.offsets[i];
    lists[i].assign(b, b + num_points_[i]);
  }
  return PointCloudBatch(std::move(lists));
}

namespace {

struct DevicePoints {
  int64_t P, N;
  DevBuf pts, ndc, first, num;
  DevicePoints(const PointCloudBatch& pc, const Camera& c)
      : P(pc.total_points()),
        N(pc.size()),
        pts(sizeof(double) * 3 * P),
        ndc(sizeof(double) * 3 * P),
        first(sizeof(int64_t) * N),
        num(sizeof(int64_t) * N) {
    upload(pts, reinterpret_cast<const double*>(pc.points_packed().data.data()), 3 * (size_t)P);
    upload(first, pc.points_packed().offsets.data(), (size_t)N);
    upload(num, pc.num_points_per_cloud().data(), (size_t)N);
    dr_camera cam = to_c(c);
    check(dr_world_to_points_ndc(pts.as<double>(), P, &cam, ndc.as<double>(), nullptr), "world_to_ndc");
  }
};

dr_point_raster_settings to_c(const PointRasterSettings& s, const Camera& c, bool naive) {
  dr_point_raster_settings o;
  std::memset(&o, 0, sizeof(o));
  o.image_h = s.image_h;
  o.image_w = s.image_w;
  o.points_per_pixel = s.points_per_pixel;
  o.bin_size = naive ? 0 : s.tile_size;
  o.radius = s.radius;
  o.znear = c.znear;
  o.clip_nonpositive_z = c.kind == ProjectionKind::Perspective ? 1 : 0;
  return o;
}

PointFragments run_points(const PointCloudBatch& pc, const Camera& c, const PointRasterSettings& s, bool naive) {
  DevicePoints d(pc, c);
  dr_point_raster_settings rs = to_c(s, c, naive);
  size_t ws_bytes = dr_rasterize_points_workspace_bytes(d.N, d.P, &rs);
  if (ws_bytes == 0) throw_status(DR_ERR_RANGE, "rasterize_points");
  PointFragments f;
  f.batch = pc.size();
  f.h = s.image_h;
  f.w = s.image_w;
  f.k = s.points_per_pixel;
  const size_t S = (size_t)f.slots();
  DevBuf ws(ws_bytes), idx(sizeof(int64_t) * S), zb(sizeof(double) * S), d2(sizeof(double) * S);
  check(dr_rasterize_points_fwd_f64(d.ndc.as<double>(), d.first.as<int64_t>(), d.num.as<int64_t>(), d.N, d.P, &rs,
                                    idx.as<int64_t>(), zb.as<double>(), d2.as<double>(), ws.p, ws_bytes, nullptr),
        "rasterize_points");
  f.idx.resize(S);
  f.zbuf.resize(S);
  f.dists2.resize(S);
  download(f.idx.data(), idx, S);
  download(f.zbuf.data(), zb, S);
  download(f.dists2.data(), d2, S);
  return f;
}

}  // namespace

PointFragments rasterize_points(const PointCloudBatch& pc, const Camera& c, const PointRasterSettings& s) {
  return run_points(pc, c, s, /*naive=*/s.tile_size <= 0);
}

PointFragments rasterize_points_naive(const PointCloudBatch& pc, const Camera& c, const PointRasterSettings& s) {
  return run_points(pc, c, s, /*naive=*/true);
}

std::vector<double> splat_opacity(const PointFragments& frag, double radius) {
  std::vector<double> alpha(size_t(frag.slots()), 0.0);  // point_render.cpp:157-168
  const double inv_r2 = 1.0 / (radius * radius);
  for (size_t slot = 0; slot < alpha.size(); ++slot)
    if (frag.idx[slot] >= 0) alpha[slot] = 1.0 - frag.dists2[slot] * inv_r2;
  return alpha;
}

std::vector<Vec3> splat_position_backward(const PointCloudBatch& pc, const Camera& c, const PointRasterSettings& s,
                                          const PointFragments& frag, const std::vector<double>& d_alphas) {
  if (int64_t(d_alphas.size()) != frag.slots())
    throw ShapeError("splat_position_backward: cotangent shape mismatch");  // point_render.cpp:305-306
  DevicePoints d(pc, c);
  dr_point_raster_settings rs = to_c(s, c, false);
  const size_t S = (size_t)frag.slots();
  // alpha = 1 - dists2 / r^2  =>  d dists2 = -d_alpha / r^2; zbuf carries no gradient here
  const double inv_r2 = 1.0 / (s.radius * s.radius);
  std::vector<double> gd(S, 0.0), gz(S, 0.0);
  for (size_t slot = 0; slot < S; ++slot)
    if (frag.idx[slot] >= 0) gd[slot] = -d_alphas[slot] * inv_r2;
  DevBuf idx(sizeof(int64_t) * S), dgz(sizeof(double) * S), dgd(sizeof(double) * S), gndc(sizeof(double) * 3 * d.P),
      gw(sizeof(double) * 3 * d.P);
  upload(idx, frag.idx.data(), S);
  upload(dgz, gz.data(), S);
  upload(dgd, gd.data(), S);
  check(dr_rasterize_points_bwd_f64(d.ndc.as<double>(), d.first.as<int64_t>(), d.num.as<int64_t>(), d.N, d.P, &rs,
                                    idx.as<int64_t>(), dgz.as<double>(), dgd.as<double>(), gndc.as<double>(), nullptr),
        "rasterize_points_backward");
  dr_camera cam = to_c(c);
  check(dr_points_ndc_backward(d.pts.as<double>(), d.P, &cam, gndc.as<double>(), gw.as<double>(), nullptr),
        "world_to_ndc_backward");
  std::vector<Vec3> out(size_t(d.P));
  download(reinterpret_cast<double*>(out.data()), gw, 3 * (size_t)d.P);
  return out;
}

}  // namespace dr_b200
