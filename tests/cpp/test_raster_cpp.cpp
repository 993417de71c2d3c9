// C++ parity test: the reference's own rasterizer tests (proj/tests/test_raster.cpp) re-run against the
// B200 host mirror dr_b200:: (include/dr_b200/mesh_raster.hpp), plus direct bit-for-bit comparison with the
// reference library dr:: (oracle/_ref/libdr3d_ref.so, the unmodified reference sources) on the same inputs.
// Built by the top-level Makefile (target `cpptest`, needs /root/reference headers at build time) and run by
// tests/test_cpp_mirror.py on a GPU box. Prints one line per case; exit code = number of failed checks.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <vector>

#include "dr/batching.hpp"
#include "dr/camera.hpp"
#include "dr/mesh_raster.hpp"
#include "dr/point_render.hpp"
#include "dr/shading.hpp"
#include "dr/templates.hpp"
#include "dr_b200/mesh_raster.hpp"
#include "dr_b200/point_render.hpp"
#include "dr_b200/shading.hpp"

namespace ref = dr;
namespace gpu = dr_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      ++g_fail;                                                                  \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
    }                                                                            \
  } while (0)

static gpu::MeshBatch to_gpu(const ref::MeshBatch& m) {
  std::vector<std::vector<gpu::Vec3>> v(size_t(m.size()));
  std::vector<std::vector<gpu::Face>> f(size_t(m.size()));
  for (int b = 0; b < m.size(); ++b) {
    for (const auto& p : m.verts_list()[size_t(b)]) v[size_t(b)].push_back({p.x, p.y, p.z});
    for (const auto& q : m.faces_list()[size_t(b)]) f[size_t(b)].push_back({q.a, q.b, q.c});
  }
  return gpu::MeshBatch(v, f);
}

static gpu::Camera to_gpu(const ref::Camera& c) {
  gpu::Camera o;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o.rotation.m[i][j] = c.rotation.m[i][j];
  o.translation = {c.translation.x, c.translation.y, c.translation.z};
  o.kind = c.kind == ref::ProjectionKind::Perspective ? gpu::ProjectionKind::Perspective
                                                      : gpu::ProjectionKind::Orthographic;
  o.focal_length = c.focal_length;
  o.principal_point = {c.principal_point.x, c.principal_point.y};
  o.ortho_scale = {c.ortho_scale.x, c.ortho_scale.y};
  o.znear = c.znear;
  o.zfar = c.zfar;
  return o;
}

static gpu::RasterSettings to_gpu(const ref::RasterSettings& s) {
  gpu::RasterSettings o;
  o.image_h = s.image_h;
  o.image_w = s.image_w;
  o.faces_per_pixel = s.faces_per_pixel;
  o.blur_radius = s.blur_radius;
  o.tile_size = s.tile_size;
  return o;
}

static bool same(const ref::MeshFragments& a, const gpu::MeshFragments& b) {
  return a.pix_to_face == b.pix_to_face && a.zbuf == b.zbuf && a.bary == b.bary && a.dists == b.dists;
}

// test_raster.cpp:113-125
static ref::MeshBatch random_soup(ref::Rng& rng, int batch, int max_faces) {
  std::vector<std::vector<ref::Vec3>> verts(static_cast<size_t>(batch));
  std::vector<std::vector<ref::Face>> faces(static_cast<size_t>(batch));
  for (int b = 0; b < batch; ++b) {
    int64_t nv = 6 + rng.uniform_int(20);
    verts[size_t(b)].resize(size_t(nv));
    for (auto& v : verts[size_t(b)]) v = rng.normal_vec3() * 0.6;
    int64_t nf = 1 + rng.uniform_int(max_faces);
    for (int64_t f = 0; f < nf; ++f)
      faces[size_t(b)].push_back({rng.uniform_int(nv), rng.uniform_int(nv), rng.uniform_int(nv)});
  }
  return ref::MeshBatch(verts, faces);
}

static void tiled_equals_naive_equals_reference() {
  // test_raster.cpp:127-149, both GPU paths compared with the reference bit for bit
  ref::Rng rng(57);
  for (int trial = 0; trial < 20; ++trial) {
    ref::MeshBatch m = random_soup(rng, 1 + int(rng.uniform_int(2)), 25);
    ref::RasterSettings s;
    int sizes[] = {32, 64};
    int ks[] = {1, 10, 50};
    double blurs[] = {0.0, 1e-4};
    s.image_h = s.image_w = sizes[rng.uniform_int(2)];
    s.faces_per_pixel = ks[rng.uniform_int(3)];
    s.blur_radius = blurs[rng.uniform_int(2)];
    s.tile_size = rng.uniform_int(2) == 0 ? 16 : 8;
    ref::Camera cam = rng.uniform_int(2) == 0 ? ref::Camera::look_from_distance(3.0, ref::ProjectionKind::Perspective, 1.5)
                                              : ref::Camera::look_from_distance(3.0, ref::ProjectionKind::Orthographic);
    ref::MeshFragments want = ref::rasterize_meshes(m, cam, s);
    gpu::MeshBatch gm = to_gpu(m);
    gpu::MeshFragments t = gpu::rasterize_meshes(gm, to_gpu(cam), to_gpu(s));
    gpu::MeshFragments n = gpu::rasterize_meshes_naive(gm, to_gpu(cam), to_gpu(s));
    CHECK(same(want, t));
    CHECK(same(want, n));
  }
}

static void slot_invariants() {
  // test_raster.cpp:151-192
  gpu::MeshBatch m = to_gpu(ref::ico_sphere(1));
  gpu::RasterSettings s;
  s.image_h = s.image_w = 48;
  s.faces_per_pixel = 8;
  s.blur_radius = 1e-3;
  gpu::Camera cam = gpu::Camera::look_from_distance(3.0, gpu::ProjectionKind::Perspective, 2.0);
  gpu::MeshFragments f = gpu::rasterize_meshes(m, cam, s);
  bool any = false;
  for (int i = 0; i < s.image_h; ++i)
    for (int j = 0; j < s.image_w; ++j) {
      bool seen_empty = false;
      for (int k = 0; k < s.faces_per_pixel; ++k) {
        int64_t slot = f.slot(0, i, j, k);
        int64_t face = f.pix_to_face[size_t(slot)];
        if (face < 0) {
          seen_empty = true;
          continue;
        }
        any = true;
        CHECK(!seen_empty);
        CHECK(f.dists[size_t(slot)] <= s.blur_radius);
        CHECK(f.zbuf[size_t(slot)] >= cam.znear);
        double w0 = f.bary[size_t(slot * 3)], w1 = f.bary[size_t(slot * 3 + 1)], w2 = f.bary[size_t(slot * 3 + 2)];
        CHECK(w0 >= 0 && w1 >= 0 && w2 >= 0);
        CHECK(std::fabs(w0 + w1 + w2 - 1.0) <= 1e-9);
        if (k > 0) {
          int64_t prev = f.slot(0, i, j, k - 1);
          CHECK(f.zbuf[size_t(prev)] < f.zbuf[size_t(slot)] ||
                (f.zbuf[size_t(prev)] == f.zbuf[size_t(slot)] && f.pix_to_face[size_t(prev)] < face));
        }
      }
    }
  CHECK(any);
}

static void blur_grows_coverage() {
  // test_raster.cpp:194-208
  gpu::MeshBatch m = to_gpu(ref::ico_sphere(1));
  gpu::Camera cam = gpu::Camera::look_from_distance(3.0, gpu::ProjectionKind::Perspective, 2.0);
  gpu::RasterSettings tight, loose;
  tight.image_h = tight.image_w = loose.image_h = loose.image_w = 64;
  tight.blur_radius = 0.0;
  loose.blur_radius = 5e-3;
  auto count = [&](const gpu::RasterSettings& s) {
    gpu::MeshFragments f = gpu::rasterize_meshes(m, cam, s);
    int64_t n = 0;
    for (int64_t v : f.pix_to_face) n += v >= 0;
    return n;
  };
  CHECK(count(loose) > count(tight));
}

static void backward_matches_fd_and_reference() {
  // test_raster.cpp:210-254 + direct comparison with dr::rasterize_backward
  ref::MeshBatch rm({{{-0.8, -0.6, 0.1}, {0.9, -0.5, 0.3}, {0.0, 0.8, -0.2}}}, {{{0, 1, 2}}});
  ref::Camera rcam = ref::Camera::look_from_distance(3.0, ref::ProjectionKind::Perspective, 1.3);
  ref::RasterSettings rs;
  rs.image_h = rs.image_w = 12;
  rs.faces_per_pixel = 2;
  rs.blur_radius = 0.03;
  gpu::MeshBatch m = to_gpu(rm);
  gpu::Camera cam = to_gpu(rcam);
  gpu::RasterSettings s = to_gpu(rs);
  gpu::MeshFragments base = gpu::rasterize_meshes(m, cam, s);
  ref::Rng rng(61);
  std::vector<double> wz(size_t(base.slots())), wb(size_t(base.slots() * 3)), wd(size_t(base.slots()));
  for (auto& v : wz) v = rng.normal();
  for (auto& v : wb) v = rng.normal();
  for (auto& v : wd) v = rng.normal();
  auto scalar = [&](const std::vector<gpu::Vec3>& verts) {
    gpu::MeshFragments f = gpu::rasterize_meshes(m.with_verts(verts), cam, s);
    double acc = 0;
    for (int64_t i = 0; i < f.slots(); ++i) {
      if (f.pix_to_face[size_t(i)] < 0) continue;
      acc += wz[size_t(i)] * f.zbuf[size_t(i)] + wd[size_t(i)] * f.dists[size_t(i)];
      for (int c = 0; c < 3; ++c) acc += wb[size_t(i * 3 + c)] * f.bary[size_t(i * 3 + c)];
    }
    return acc;
  };
  std::vector<gpu::Vec3> g = gpu::rasterize_backward(m, cam, s, base, wz, wb, wd);
  ref::MeshFragments rbase = ref::rasterize_meshes(rm, rcam, rs);
  std::vector<ref::Vec3> gr = ref::rasterize_backward(rm, rcam, rs, rbase, wz, wb, wd);
  std::vector<gpu::Vec3> v0 = m.verts_packed().data;
  const double eps = 1e-6;
  for (size_t i = 0; i < v0.size(); ++i) {
    for (int axis = 0; axis < 3; ++axis) {
      std::vector<gpu::Vec3> vp = v0, vm = v0;
      double* cp = axis == 0 ? &vp[i].x : (axis == 1 ? &vp[i].y : &vp[i].z);
      double* cm = axis == 0 ? &vm[i].x : (axis == 1 ? &vm[i].y : &vm[i].z);
      *cp += eps;
      *cm -= eps;
      double fd = (scalar(vp) - scalar(vm)) / (2 * eps);
      double an = axis == 0 ? g[i].x : (axis == 1 ? g[i].y : g[i].z);
      double rf = axis == 0 ? gr[i].x : (axis == 1 ? gr[i].y : gr[i].z);
      CHECK(std::fabs(fd - an) / std::fmax(std::fmax(std::fabs(fd), std::fabs(an)), 1e-6) <= 2e-3);
      CHECK(std::fabs(rf - an) <= 1e-12 * std::fmax(1.0, std::fabs(rf)));
    }
  }
}

static void errors_mirror_reference() {
  bool threw = false;
  try {
    gpu::MeshBatch bad({}, {});
  } catch (const gpu::ShapeError&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    gpu::MeshBatch bad({{{0, 0, 0}, {1, 0, 0}, {0, 1, 0}}}, {{{0, 1, 3}}});
  } catch (const gpu::IndexError&) {
    threw = true;
  }
  CHECK(threw);
  gpu::MeshBatch m({{{0, 0, 0}, {1, 0, 0}, {0, 1, 0}}}, {{{0, 1, 2}}});
  gpu::RasterSettings s;
  gpu::MeshFragments f = gpu::rasterize_meshes(m, gpu::Camera::look_from_distance(3.0, gpu::ProjectionKind::Perspective), s);
  threw = false;
  try {
    gpu::rasterize_backward(m, gpu::Camera{}, s, f, std::vector<double>(3), f.bary, f.dists);
  } catch (const gpu::ShapeError&) {
    threw = true;
  }
  CHECK(threw);
}

static double max_rel(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 1e-300;
  for (size_t i = 0; i < a.size() && i < b.size(); ++i) {
    num = std::fmax(num, std::fabs(a[i] - b[i]));
    den = std::fmax(den, std::fabs(b[i]));
  }
  return a.size() == b.size() ? num / den : 1e300;
}

static std::vector<double> flat(const std::vector<gpu::Vec3>& v) {
  std::vector<double> o;
  for (const auto& p : v) o.insert(o.end(), {p.x, p.y, p.z});
  return o;
}
static std::vector<double> flat(const std::vector<ref::Vec3>& v) {
  std::vector<double> o;
  for (const auto& p : v) o.insert(o.end(), {p.x, p.y, p.z});
  return o;
}

// test_point_render.cpp:24-43 against the GPU mirror: tiled == naive == reference, bit for bit
static void points_tiled_naive_reference() {
  ref::Rng rng(83);
  for (int trial = 0; trial < 15; ++trial) {
    int b = 1 + int(rng.uniform_int(3));
    std::vector<std::vector<ref::Vec3>> clouds(static_cast<size_t>(b));
    for (auto& cl : clouds) {  // tests/helpers.hpp:23-33
      int64_t n = 1 + rng.uniform_int(200);
      for (int64_t i = 0; i < n; ++i) cl.push_back(rng.normal_vec3());
    }
    ref::PointRasterSettings s;
    s.image_h = s.image_w = rng.uniform_int(2) == 0 ? 32 : 64;
    s.points_per_pixel = rng.uniform_int(2) == 0 ? 1 : 8;
    s.radius = rng.uniform(0.02, 0.15);
    s.tile_size = rng.uniform_int(2) == 0 ? 16 : 8;
    ref::Camera cam = rng.uniform_int(2) == 0 ? ref::Camera::look_from_distance(3.0, ref::ProjectionKind::Perspective, 1.5)
                                              : ref::Camera::look_from_distance(3.0, ref::ProjectionKind::Orthographic);
    ref::PointFragments want = ref::rasterize_points(ref::PointCloudBatch(clouds), cam, s);
    std::vector<std::vector<gpu::Vec3>> gc(clouds.size());
    for (size_t i = 0; i < clouds.size(); ++i)
      for (const auto& p : clouds[i]) gc[i].push_back({p.x, p.y, p.z});
    gpu::PointCloudBatch pc(gc);
    gpu::PointRasterSettings gs;
    gs.image_h = s.image_h;
    gs.image_w = s.image_w;
    gs.points_per_pixel = s.points_per_pixel;
    gs.radius = s.radius;
    gs.tile_size = s.tile_size;
    gpu::PointFragments t = gpu::rasterize_points(pc, to_gpu(cam), gs);
    gpu::PointFragments n = gpu::rasterize_points_naive(pc, to_gpu(cam), gs);
    CHECK(t.idx == want.idx && t.zbuf == want.zbuf && t.dists2 == want.dists2);
    CHECK(n.idx == want.idx && n.zbuf == want.zbuf && n.dists2 == want.dists2);
    if (trial == 0) {  // splat_opacity -> splat_position_backward vs the reference
      std::vector<double> da(size_t(want.slots()));
      for (auto& x : da) x = rng.normal();
      std::vector<ref::Vec3> gr = ref::splat_position_backward(ref::PointCloudBatch(clouds), cam, s, want, da);
      std::vector<gpu::Vec3> gg = gpu::splat_position_backward(pc, to_gpu(cam), gs, t, da);
      CHECK(max_rel(flat(gg), flat(gr)) < 1e-10);
      CHECK(gpu::splat_opacity(t, s.radius) == ref::splat_opacity(want, s.radius));
    }
  }
}

// the reference fit step (pipeline.cpp:153-162) vs the fused GPU silhouette calls
static void fused_silhouette_matches_reference_fit_step() {
  ref::MeshBatch m = ref::ico_sphere(2);
  ref::Camera cam = ref::Camera::look_from_distance(3.0, ref::ProjectionKind::Perspective, 2.0);
  ref::RasterSettings s;
  s.image_h = s.image_w = 64;
  s.faces_per_pixel = 4;
  s.blur_radius = 2e-4;
  const double sigma = 1e-4;
  ref::MeshFragments frag = ref::rasterize_meshes(m, cam, s);
  std::vector<double> alpha = ref::silhouette_blend(frag, sigma);
  gpu::SilhouetteFragments g = gpu::rasterize_silhouette(to_gpu(m), to_gpu(cam), to_gpu(s), sigma);
  CHECK(g.pix_to_face == frag.pix_to_face);
  CHECK(max_rel(g.alpha, alpha) < 1e-6);
  std::vector<double> da(alpha.size());
  for (size_t i = 0; i < da.size(); ++i) da[i] = alpha[i] - 0.5;
  std::vector<double> dd = ref::silhouette_blend_backward(frag, sigma, da);
  std::vector<ref::Vec3> want = ref::rasterize_backward(m, cam, s, frag, std::vector<double>(frag.zbuf.size(), 0.0),
                                                        std::vector<double>(frag.bary.size(), 0.0), dd);
  std::vector<gpu::Vec3> got = gpu::rasterize_silhouette_backward(to_gpu(m), to_gpu(cam), to_gpu(s), sigma, g, da);
  CHECK(max_rel(flat(got), flat(want)) < 1e-4);
}

// The streamed host pipeline (dr_b200::HostPipeline, include/dr_raster.h dr_host_pipeline_*) on a synthetic batch:
// pix_to_face bit-identical to the reference dr::rasterize_meshes, the fp32 payload within the north-star
// tolerance of the reference's fp64 one, and the same gradients whether the batch streams as 1 or 5 mesh groups.
static void host_pipeline_matches_reference() {
  ref::MeshBatch m = ref::synthetic_batch(3000.0, 1500.0, 6, 3);
  ref::Camera cam = ref::Camera::look_from_distance(3.0, ref::ProjectionKind::Perspective, 2.0);
  ref::RasterSettings s;
  s.image_h = s.image_w = 64;
  s.faces_per_pixel = 4;
  s.blur_radius = 1e-4;
  ref::MeshFragments want = ref::rasterize_meshes(m, cam, s);
  gpu::MeshBatch gm = to_gpu(m);
  const int64_t F = gm.total_faces();
  std::vector<int64_t> first(gm.faces_packed().offsets.begin(), gm.faces_packed().offsets.end() - 1);
  gpu::pinned_vector<double> fv = gpu::face_verts_packed(gm, to_gpu(cam));
  const size_t S = size_t(want.slots());
  ref::Rng rng(5);
  gpu::pinned_vector<float> dz(S), db(3 * S), dd(S);
  for (auto& x : dz) x = float(rng.normal());
  for (auto& x : db) x = float(rng.normal());
  for (auto& x : dd) x = float(rng.normal());
  gpu::pinned_vector<double> g1, g5;
  for (int groups : {1, 5}) {
    gpu::HostPipeline pipe(first, gm.num_faces_per_mesh(), F, to_gpu(s), to_gpu(cam), groups, 1, 2, true);
    CHECK(pipe.groups() >= 1 && pipe.groups() <= groups);
    gpu::MeshFragments32 out;
    for (int rep = 0; rep < 2; ++rep) pipe.run(fv, out, dz, db, dd, groups == 1 ? g1 : g5);
    CHECK(std::equal(want.pix_to_face.begin(), want.pix_to_face.end(), out.pix_to_face.begin()));
    bool close = true;
    for (size_t i = 0; i < S; ++i) {
      close = close && std::fabs(out.zbuf[i] - want.zbuf[i]) <= 1e-6 + 1e-5 * std::fabs(want.zbuf[i]);
      close = close && std::fabs(out.dists[i] - want.dists[i]) <= 1e-6 + 1e-5 * std::fabs(want.dists[i]);
    }
    for (size_t i = 0; i < 3 * S; ++i) close = close && std::fabs(out.bary[i] - want.bary[i]) <= 1e-6 + 1e-5 * std::fabs(want.bary[i]);
    CHECK(close);
  }
  std::vector<double> a(g1.begin(), g1.end()), b(g5.begin(), g5.end());
  CHECK(max_rel(a, b) < 1e-12);
  double mx = 0;
  for (double x : a) mx = std::max(mx, std::fabs(x));
  CHECK(mx > 0);
}

int main() {
  struct Case {
    const char* name;
    std::function<void()> fn;
  } cases[] = {{"tiled_equals_naive_equals_reference", tiled_equals_naive_equals_reference},
               {"slot_invariants", slot_invariants},
               {"blur_grows_coverage", blur_grows_coverage},
               {"backward_matches_fd_and_reference", backward_matches_fd_and_reference},
               {"errors_mirror_reference", errors_mirror_reference},
               {"points_tiled_naive_reference", points_tiled_naive_reference},
               {"fused_silhouette_matches_reference_fit_step", fused_silhouette_matches_reference_fit_step},
               {"host_pipeline_matches_reference", host_pipeline_matches_reference}};
  for (auto& c : cases) {
    int before = g_fail;
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  exception: %s\n", e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", c.name);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail;
}
