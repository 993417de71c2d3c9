// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the *unmodified* reference `dr3d` library
// (/root/reference/proj/src/{core,batching,camera,mesh_raster,templates}.cpp), compiled
// by oracle/Makefile into oracle/_ref/libdr3d_ref.so. It lets the Python tests and the
// bench's reference arm call the reference's own rasterizer and generators:
//   dr::rasterize_meshes / rasterize_meshes_naive   (mesh_raster.hpp:41,44)
//   dr::rasterize_backward                          (mesh_raster.hpp:66-69)
//   dr::world_to_ndc                                (camera.hpp:50)
//   dr::ico_sphere / cube / synthetic_batch         (templates.hpp:12-24)
//   dr::silhouette_blend / silhouette_blend_backward (shading.hpp:37-41)
//   the softmax render op of grad.cpp:177-209 (interpolate_face_attributes + softmax_blend and their backwards)
//   dr::rasterize_points / _naive, splat_position_backward (point_render.hpp:33-36, 66-68)
//   dr::fit_silhouette (pipeline.hpp:91-95, pipeline.cpp:100-205) and its regularizers / loss
//   (geometry.hpp:96-107)
//   dr::packed_to_padded / padded_to_packed (batching.hpp:48-75) over fixed-size rows
// Errors are caught and reported through ref_last_error() (the reference throws).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "dr/batching.hpp"
#include "dr/camera.hpp"
#include "dr/core.hpp"
#include "dr/geometry.hpp"
#include "dr/mesh_raster.hpp"
#include "dr/pipeline.hpp"
#include "dr/point_render.hpp"
#include "dr/shading.hpp"
#include "dr/templates.hpp"

namespace {
thread_local std::string g_err;

// cam: [kind(0 ortho,1 persp), R(9 row-major), t(3), focal, ppx, ppy, sx, sy, znear, zfar]
dr::Camera make_camera(const double* cam) {
  dr::Mat3 r;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) r.m[i][j] = cam[1 + 3 * i + j];
  dr::Vec3 t{cam[10], cam[11], cam[12]};
  if (cam[0] != 0.0)
    return dr::Camera::perspective(r, t, cam[13], {cam[14], cam[15]}, cam[18], cam[19]);
  return dr::Camera::orthographic(r, t, {cam[16], cam[17]}, cam[18], cam[19]);
}

dr::RasterSettings make_settings(const int32_t* si, double blur) {
  dr::RasterSettings s;
  s.image_h = si[0];
  s.image_w = si[1];
  s.faces_per_pixel = si[2];
  s.tile_size = si[3];
  s.blur_radius = blur;
  return s;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
void ref_set_num_threads(int n) { dr::set_num_threads(n); }
int ref_num_threads(void) { return dr::num_threads(); }

// ---- mesh batches (opaque handles) ----
void* ref_batch_from_arrays(const double* verts, const int64_t* faces_local, const int64_t* vert_counts,
                            const int64_t* face_counts, int32_t n) {
  dr::MeshBatch* out = nullptr;
  int rc = guarded([&] {
    std::vector<std::vector<dr::Vec3>> vl(size_t(n > 0 ? n : 0));
    std::vector<std::vector<dr::Face>> fl(size_t(n > 0 ? n : 0));
    int64_t vo = 0, fo = 0;
    for (int32_t b = 0; b < n; ++b) {
      for (int64_t v = 0; v < vert_counts[b]; ++v, ++vo)
        vl[size_t(b)].push_back({verts[3 * vo], verts[3 * vo + 1], verts[3 * vo + 2]});
      for (int64_t f = 0; f < face_counts[b]; ++f, ++fo)
        fl[size_t(b)].push_back({faces_local[3 * fo], faces_local[3 * fo + 1], faces_local[3 * fo + 2]});
    }
    out = new dr::MeshBatch(std::move(vl), std::move(fl));
  });
  return rc == 0 ? out : nullptr;
}
void* ref_ico_sphere(int level) {
  dr::MeshBatch* out = nullptr;
  guarded([&] { out = new dr::MeshBatch(dr::ico_sphere(level)); });
  return out;
}
void* ref_cube(double half, int n) {
  dr::MeshBatch* out = nullptr;
  guarded([&] { out = new dr::MeshBatch(dr::cube(half, n)); });
  return out;
}
void* ref_synthetic_batch(double mean_faces, double sigma, int batch, uint64_t seed) {
  dr::MeshBatch* out = nullptr;
  guarded([&] { out = new dr::MeshBatch(dr::synthetic_batch(mean_faces, sigma, batch, seed)); });
  return out;
}
void ref_batch_free(void* h) { delete static_cast<dr::MeshBatch*>(h); }
// sizes: [N, total_verts, total_faces]
void ref_batch_sizes(void* h, int64_t* out3) {
  auto* m = static_cast<dr::MeshBatch*>(h);
  out3[0] = m->size();
  out3[1] = m->total_verts();
  out3[2] = m->total_faces();
}
// packed verts [V,3], packed faces with GLOBAL indices [F,3], per-mesh counts
void ref_batch_export(void* h, double* verts, int64_t* faces_packed, int64_t* vert_counts,
                      int64_t* face_counts) {
  auto* m = static_cast<dr::MeshBatch*>(h);
  const auto& v = m->verts_packed().data;
  for (size_t i = 0; i < v.size(); ++i) {
    verts[3 * i] = v[i].x;
    verts[3 * i + 1] = v[i].y;
    verts[3 * i + 2] = v[i].z;
  }
  const auto& f = m->faces_packed().data;
  for (size_t i = 0; i < f.size(); ++i) {
    faces_packed[3 * i] = f[i].a;
    faces_packed[3 * i + 1] = f[i].b;
    faces_packed[3 * i + 2] = f[i].c;
  }
  for (int b = 0; b < m->size(); ++b) {
    vert_counts[b] = m->num_verts_per_mesh()[size_t(b)];
    face_counts[b] = m->num_faces_per_mesh()[size_t(b)];
  }
}

// ---- camera ----
int ref_world_to_ndc(const double* cam, const double* pts, int64_t n, double* xy, double* zv,
                     uint8_t* clipped) {
  return guarded([&] {
    dr::Camera c = make_camera(cam);
    for (int64_t i = 0; i < n; ++i) {
      dr::NdcPoint p = dr::world_to_ndc(c, dr::Vec3{pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]});
      xy[2 * i] = p.xy.x;
      xy[2 * i + 1] = p.xy.y;
      zv[i] = p.z_view;
      clipped[i] = p.clipped ? 1 : 0;
    }
  });
}
int ref_world_to_ndc_backward(const double* cam, const double* pts, const double* d_xy,
                              const double* d_z, int64_t n, double* d_world) {
  return guarded([&] {
    dr::Camera c = make_camera(cam);
    for (int64_t i = 0; i < n; ++i) {
      dr::Vec3 g = dr::world_to_ndc_backward(c, {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]},
                                             {d_xy[2 * i], d_xy[2 * i + 1]}, d_z[i]);
      d_world[3 * i] = g.x;
      d_world[3 * i + 1] = g.y;
      d_world[3 * i + 2] = g.z;
    }
  });
}

// ---- the hot path ----
// si: [H, W, K, tile]; outputs sized N*H*W*K (bary x3)
int ref_rasterize(void* h, const double* cam, const int32_t* si, double blur, int naive,
                  int64_t* p2f, double* zbuf, double* bary, double* dists) {
  return guarded([&] {
    auto* m = static_cast<dr::MeshBatch*>(h);
    dr::Camera c = make_camera(cam);
    dr::RasterSettings s = make_settings(si, blur);
    dr::MeshFragments f = naive ? dr::rasterize_meshes_naive(*m, c, s) : dr::rasterize_meshes(*m, c, s);
    std::memcpy(p2f, f.pix_to_face.data(), f.pix_to_face.size() * sizeof(int64_t));
    std::memcpy(zbuf, f.zbuf.data(), f.zbuf.size() * sizeof(double));
    std::memcpy(bary, f.bary.data(), f.bary.size() * sizeof(double));
    std::memcpy(dists, f.dists.data(), f.dists.size() * sizeof(double));
  });
}

// silhouette blend over fragments (dr::silhouette_blend / _backward, shading.hpp:37-41); only pix_to_face and
// dists are read by the reference
int ref_silhouette_blend(const int64_t* p2f, const double* dists, int32_t nbatch, int32_t h, int32_t w, int32_t k,
                         double sigma, double* alpha) {
  return guarded([&] {
    dr::MeshFragments f;
    f.batch = nbatch;
    f.h = h;
    f.w = w;
    f.k = k;
    size_t ns = size_t(f.slots());
    f.pix_to_face.assign(p2f, p2f + ns);
    f.dists.assign(dists, dists + ns);
    f.zbuf.assign(ns, 0.0);
    f.bary.assign(3 * ns, 0.0);
    std::vector<double> a = dr::silhouette_blend(f, sigma);
    std::memcpy(alpha, a.data(), a.size() * sizeof(double));
  });
}
int ref_silhouette_blend_backward(const int64_t* p2f, const double* dists, int32_t nbatch, int32_t h, int32_t w,
                                  int32_t k, double sigma, const double* d_alpha, double* d_dists) {
  return guarded([&] {
    dr::MeshFragments f;
    f.batch = nbatch;
    f.h = h;
    f.w = w;
    f.k = k;
    size_t ns = size_t(f.slots());
    f.pix_to_face.assign(p2f, p2f + ns);
    f.dists.assign(dists, dists + ns);
    f.zbuf.assign(ns, 0.0);
    f.bary.assign(3 * ns, 0.0);
    std::vector<double> da(d_alpha, d_alpha + ns / size_t(k));
    std::vector<double> dd = dr::silhouette_blend_backward(f, sigma, da);
    std::memcpy(d_dists, dd.data(), dd.size() * sizeof(double));
  });
}

// ---- softmax render (grad.cpp:177-209 composed from the reference's own functions) ----
// vert_colors [V,3]; blend = [sigma, gamma, bg_r, bg_g, bg_b]; image [n*H*W*3]; p2f [S]
int ref_softmax_render(void* h, const double* cam, const int32_t* si, double blur, const double* vert_colors,
                       const double* blend, double* image, int64_t* p2f) {
  return guarded([&] {
    auto* m = static_cast<dr::MeshBatch*>(h);
    dr::Camera c = make_camera(cam);
    dr::RasterSettings s = make_settings(si, blur);
    dr::BlendParams p;
    p.sigma = blend[0];
    p.gamma = blend[1];
    p.background_color = {blend[2], blend[3], blend[4]};
    dr::MeshFragments frag = dr::rasterize_meshes(*m, c, s);
    std::vector<double> attr(vert_colors, vert_colors + 3 * m->total_verts());
    std::vector<double> interp = dr::interpolate_face_attributes(*m, frag, attr, 3);
    std::vector<dr::Vec3> colors(size_t(frag.slots()));
    for (size_t i = 0; i < colors.size(); ++i) colors[i] = {interp[3 * i], interp[3 * i + 1], interp[3 * i + 2]};
    std::vector<dr::Vec3> img = dr::softmax_blend(frag, colors, p, c.znear, c.zfar);
    for (size_t i = 0; i < img.size(); ++i) {
      image[3 * i] = img[i].x;
      image[3 * i + 1] = img[i].y;
      image[3 * i + 2] = img[i].z;
    }
    std::memcpy(p2f, frag.pix_to_face.data(), frag.pix_to_face.size() * sizeof(int64_t));
  });
}
// vjp: d_image [n*H*W*3] -> world d_verts [V,3] and d_vert_colors [V,3]
int ref_softmax_render_backward(void* h, const double* cam, const int32_t* si, double blur, const double* vert_colors,
                                const double* blend, const double* d_image, double* d_verts, double* d_colors) {
  return guarded([&] {
    auto* m = static_cast<dr::MeshBatch*>(h);
    dr::Camera c = make_camera(cam);
    dr::RasterSettings s = make_settings(si, blur);
    dr::BlendParams p;
    p.sigma = blend[0];
    p.gamma = blend[1];
    p.background_color = {blend[2], blend[3], blend[4]};
    dr::MeshFragments frag = dr::rasterize_meshes(*m, c, s);
    std::vector<double> attr(vert_colors, vert_colors + 3 * m->total_verts());
    std::vector<double> interp = dr::interpolate_face_attributes(*m, frag, attr, 3);
    std::vector<dr::Vec3> colors(size_t(frag.slots()));
    for (size_t i = 0; i < colors.size(); ++i) colors[i] = {interp[3 * i], interp[3 * i + 1], interp[3 * i + 2]};
    const size_t npix = size_t(frag.slots() / frag.k);
    std::vector<dr::Vec3> dimg(npix);
    for (size_t i = 0; i < npix; ++i) dimg[i] = {d_image[3 * i], d_image[3 * i + 1], d_image[3 * i + 2]};
    dr::SoftmaxBlendGrads bg = dr::softmax_blend_backward(frag, colors, p, c.znear, c.zfar, dimg);
    std::vector<double> flat_dc(3 * bg.d_colors.size());
    for (size_t i = 0; i < bg.d_colors.size(); ++i) {
      flat_dc[3 * i] = bg.d_colors[i].x;
      flat_dc[3 * i + 1] = bg.d_colors[i].y;
      flat_dc[3 * i + 2] = bg.d_colors[i].z;
    }
    dr::InterpolateGrads ig = dr::interpolate_face_attributes_backward(*m, frag, attr, 3, flat_dc);
    std::vector<dr::Vec3> g = dr::rasterize_backward(*m, c, s, frag, bg.d_zbuf, ig.d_bary, bg.d_dists);
    for (size_t i = 0; i < g.size(); ++i) {
      d_verts[3 * i] = g[i].x;
      d_verts[3 * i + 1] = g[i].y;
      d_verts[3 * i + 2] = g[i].z;
    }
    std::memcpy(d_colors, ig.d_attrs.data(), ig.d_attrs.size() * sizeof(double));
  });
}

// ---- point clouds ----
// points [P,3] world, counts [n]; si: [H, W, K, tile]; outputs [n,H,W,K]
int ref_rasterize_points(const double* pts, const int64_t* counts, int32_t n, const double* cam, const int32_t* si,
                         double radius, int naive, int64_t* idx, double* zbuf, double* dists2) {
  return guarded([&] {
    std::vector<std::vector<dr::Vec3>> pl(size_t(n > 0 ? n : 0));
    int64_t o = 0;
    for (int32_t b = 0; b < n; ++b)
      for (int64_t i = 0; i < counts[b]; ++i, ++o) pl[size_t(b)].push_back({pts[3 * o], pts[3 * o + 1], pts[3 * o + 2]});
    dr::PointCloudBatch pc(std::move(pl));
    dr::Camera c = make_camera(cam);
    dr::PointRasterSettings s;
    s.image_h = si[0];
    s.image_w = si[1];
    s.points_per_pixel = si[2];
    s.tile_size = si[3];
    s.radius = radius;
    dr::PointFragments f = naive ? dr::rasterize_points_naive(pc, c, s) : dr::rasterize_points(pc, c, s);
    std::memcpy(idx, f.idx.data(), f.idx.size() * sizeof(int64_t));
    std::memcpy(zbuf, f.zbuf.data(), f.zbuf.size() * sizeof(double));
    std::memcpy(dists2, f.dists2.data(), f.dists2.size() * sizeof(double));
  });
}
// splat_opacity -> d_alphas -> splat_position_backward (world-space d_points [P,3])
int ref_splat_position_backward(const double* pts, const int64_t* counts, int32_t n, const double* cam,
                                const int32_t* si, double radius, const int64_t* idx, const double* zbuf,
                                const double* dists2, const double* d_alphas, double* d_points) {
  return guarded([&] {
    std::vector<std::vector<dr::Vec3>> pl(size_t(n > 0 ? n : 0));
    int64_t o = 0;
    for (int32_t b = 0; b < n; ++b)
      for (int64_t i = 0; i < counts[b]; ++i, ++o) pl[size_t(b)].push_back({pts[3 * o], pts[3 * o + 1], pts[3 * o + 2]});
    dr::PointCloudBatch pc(std::move(pl));
    dr::Camera c = make_camera(cam);
    dr::PointRasterSettings s;
    s.image_h = si[0];
    s.image_w = si[1];
    s.points_per_pixel = si[2];
    s.tile_size = si[3];
    s.radius = radius;
    dr::PointFragments f;
    f.batch = n;
    f.h = s.image_h;
    f.w = s.image_w;
    f.k = s.points_per_pixel;
    size_t ns = size_t(f.slots());
    f.idx.assign(idx, idx + ns);
    f.zbuf.assign(zbuf, zbuf + ns);
    f.dists2.assign(dists2, dists2 + ns);
    std::vector<double> da(d_alphas, d_alphas + ns);
    std::vector<dr::Vec3> g = dr::splat_position_backward(pc, c, s, f, da);
    for (size_t i = 0; i < g.size(); ++i) {
      d_points[3 * i] = g[i].x;
      d_points[3 * i + 1] = g[i].y;
      d_points[3 * i + 2] = g[i].z;
    }
  });
}

// fragments in, world-space d_verts [V,3] out (dr::rasterize_backward, mesh_raster.hpp:66-69)
int ref_rasterize_backward(void* h, const double* cam, const int32_t* si, double blur, int32_t nbatch,
                           const int64_t* p2f, const double* zbuf, const double* bary,
                           const double* dists, const double* d_zbuf, const double* d_bary,
                           const double* d_dists, double* d_verts) {
  return guarded([&] {
    auto* m = static_cast<dr::MeshBatch*>(h);
    dr::Camera c = make_camera(cam);
    dr::RasterSettings s = make_settings(si, blur);
    dr::MeshFragments f;
    f.batch = nbatch;
    f.h = s.image_h;
    f.w = s.image_w;
    f.k = s.faces_per_pixel;
    size_t ns = size_t(f.slots());
    f.pix_to_face.assign(p2f, p2f + ns);
    f.zbuf.assign(zbuf, zbuf + ns);
    f.bary.assign(bary, bary + 3 * ns);
    f.dists.assign(dists, dists + ns);
    std::vector<double> dz(d_zbuf, d_zbuf + ns), db(d_bary, d_bary + 3 * ns), dd(d_dists, d_dists + ns);
    std::vector<dr::Vec3> g = dr::rasterize_backward(*m, c, s, f, dz, db, dd);
    for (size_t i = 0; i < g.size(); ++i) {
      d_verts[3 * i] = g[i].x;
      d_verts[3 * i + 1] = g[i].y;
      d_verts[3 * i + 2] = g[i].z;
    }
  });
}

// kernel-level helpers for the known-answer tests (mesh_raster.hpp:51-64)
double ref_point_triangle_dist2(const double* p, const double* a, const double* b, const double* c) {
  return dr::point_triangle_dist2({p[0], p[1]}, {a[0], a[1]}, {b[0], b[1]}, {c[0], c[1]});
}
void ref_barycentric(const double* p, const double* a, const double* b, const double* c, double* w) {
  dr::Vec3 r = dr::barycentric_coords({p[0], p[1]}, {a[0], a[1]}, {b[0], b[1]}, {c[0], c[1]});
  w[0] = r.x;
  w[1] = r.y;
  w[2] = r.z;
}
void ref_clamp_barycentric(const double* w, double* out) {
  dr::Vec3 r = dr::clamp_barycentric({w[0], w[1], w[2]});
  out[0] = r.x;
  out[1] = r.y;
  out[2] = r.z;
}
void ref_point_triangle_dist2_backward(const double* p, const double* a, const double* b, const double* c,
                                       double d_out, double* g6) {
  dr::Vec2 da{}, db{}, dc{};
  dr::point_triangle_dist2_backward({p[0], p[1]}, {a[0], a[1]}, {b[0], b[1]}, {c[0], c[1]}, d_out, da, db,
                                    dc);
  g6[0] = da.x; g6[1] = da.y; g6[2] = db.x; g6[3] = db.y; g6[4] = dc.x; g6[5] = dc.y;
}
// ---- fit_silhouette (pipeline.cpp:100-205) ----
// cfg_i: [template_level, num_views, iterations, image_size, faces_per_pixel]
// cfg_d: [target_scale, step_size, lambda_laplacian, lambda_edge, coarse_blur_radius, coarse_sigma,
//         coarse_fraction, blur_radius, sigma, camera_distance, focal_length]
// trace: [iterations, 5] (iter, l_s, l_l, l_e, total); verts_out: the fitted packed verts [V,3] (V <= vcap)
int ref_fit_silhouette(const char* target_spec, const int32_t* ci, const double* cd, double* trace, double* final_loss,
                       double* verts_out, int64_t vcap, int64_t* nverts) {
  return guarded([&] {
    dr::FitConfig c;
    c.target_spec = target_spec;
    c.template_level = ci[0];
    c.num_views = ci[1];
    c.iterations = ci[2];
    c.image_size = ci[3];
    c.faces_per_pixel = ci[4];
    c.target_scale = cd[0];
    c.step_size = cd[1];
    c.lambda_laplacian = cd[2];
    c.lambda_edge = cd[3];
    c.coarse_blur_radius = cd[4];
    c.coarse_sigma = cd[5];
    c.coarse_fraction = cd[6];
    c.blur_radius = cd[7];
    c.sigma = cd[8];
    c.camera_distance = cd[9];
    c.focal_length = cd[10];
    dr::FitResult r = dr::fit_silhouette(c);
    for (size_t i = 0; i < r.trace.size(); ++i) {
      const auto& t = r.trace[i];
      trace[5 * i] = t.iter;
      trace[5 * i + 1] = t.l_s;
      trace[5 * i + 2] = t.l_l;
      trace[5 * i + 3] = t.l_e;
      trace[5 * i + 4] = t.total;
    }
    *final_loss = r.final_silhouette_loss;
    const auto& v = r.mesh.verts_packed().data;
    *nverts = int64_t(v.size());
    for (size_t i = 0; i < v.size() && int64_t(i) < vcap; ++i) {
      verts_out[3 * i] = v[i].x;
      verts_out[3 * i + 1] = v[i].y;
      verts_out[3 * i + 2] = v[i].z;
    }
  });
}

// mesh regularizers of a batch: out2 = [edge_length_loss mean, laplacian_loss mean]; d_edge / d_lap [V,3] for
// d_mean = 1 (geometry.cpp:556-649)
int ref_mesh_losses(void* h, double* out2, double* d_edge, double* d_lap) {
  return guarded([&] {
    const auto& m = *static_cast<dr::MeshBatch*>(h);
    out2[0] = dr::edge_length_loss(m).mean;
    out2[1] = dr::laplacian_loss(m).mean;
    std::vector<dr::Vec3> g;
    dr::edge_length_loss_backward(m, 1.0, g);
    for (size_t i = 0; i < g.size(); ++i) {
      d_edge[3 * i] = g[i].x;
      d_edge[3 * i + 1] = g[i].y;
      d_edge[3 * i + 2] = g[i].z;
    }
    dr::laplacian_loss_backward(m, 1.0, g);
    for (size_t i = 0; i < g.size(); ++i) {
      d_lap[3 * i] = g[i].x;
      d_lap[3 * i + 1] = g[i].y;
      d_lap[3 * i + 2] = g[i].z;
    }
  });
}

// silhouette_iou_loss and its backward (geometry.cpp:651-682)
int ref_silhouette_iou(const double* pred, const double* gt, int64_t n, double d_loss, double* loss, double* grad) {
  return guarded([&] {
    std::vector<double> p(pred, pred + n), g(gt, gt + n);
    *loss = dr::silhouette_iou_loss(p, g);
    std::vector<double> d = dr::silhouette_iou_loss_backward(p, g, d_loss);
    std::memcpy(grad, d.data(), sizeof(double) * size_t(n));
  });
}

// dr::packed_to_padded / padded_to_packed (batching.hpp:48-75) over rows of `row` doubles (T = a fixed-size row)
extern "C++" {
namespace {
template <int R>
struct Row {
  double v[R];
};
template <int R>
void p2pad(const double* data, const int64_t* offsets, int64_t B, double pad, double* out) {
  dr::PackedView<Row<R>> pv;
  pv.offsets.assign(offsets, offsets + B + 1);
  pv.data.resize(size_t(offsets[B]));
  std::memcpy(pv.data.data(), data, sizeof(double) * R * size_t(offsets[B]));
  Row<R> p;
  for (int k = 0; k < R; ++k) p.v[k] = pad;
  std::vector<Row<R>> o = dr::packed_to_padded(pv, p);
  std::memcpy(out, o.data(), sizeof(double) * R * o.size());
}
template <int R>
void pad2p(const double* padded, int64_t B, int64_t max_count, const int64_t* counts, double* out, int32_t* ite) {
  std::vector<Row<R>> pd(size_t(B * max_count));
  std::memcpy(pd.data(), padded, sizeof(double) * R * pd.size());
  dr::PackedView<Row<R>> pv = dr::padded_to_packed(pd, std::vector<int64_t>(counts, counts + B));
  std::memcpy(out, pv.data.data(), sizeof(double) * R * pv.data.size());
  for (size_t i = 0; i < pv.item_to_element.size(); ++i) ite[i] = pv.item_to_element[i];
}
}  // namespace
}  // extern "C++"

// row = 1 or 9 doubles per packed item; out = [B, max_count, row] (max over the element counts)
int ref_packed_to_padded(const double* data, const int64_t* offsets, int64_t B, int32_t row, double pad, double* out) {
  return guarded([&] {
    if (row == 9) p2pad<9>(data, offsets, B, pad, out);
    else p2pad<1>(data, offsets, B, pad, out);
  });
}
int ref_padded_to_packed(const double* padded, int64_t B, int64_t max_count, const int64_t* counts, int32_t row,
                         double* out, int32_t* item_to_element) {
  return guarded([&] {
    if (row == 9) pad2p<9>(padded, B, max_count, counts, out, item_to_element);
    else pad2p<1>(padded, B, max_count, counts, out, item_to_element);
  });
}

}  // extern "C"
