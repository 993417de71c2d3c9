/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the rasterize_meshes hot path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this file's
 * shared library (oracle/liboracle.so), and only as the CHECKER. The product path
 * (paper_2007_08501_b200/) never links or calls it.
 *
 * A plain-C restatement of the reference `dr3d` rasterizer (/root/reference/proj/src/mesh_raster.cpp,
 * "MR" below) on the north-star boundary: packed face_verts [F,3,3] = (x_ndc, y_ndc, z_view) per
 * face vertex plus mesh_to_face_first_idx / num_faces_per_mesh, instead of MeshBatch + Camera.
 *
 * Parity pin: with perspective_correct=0, clip_barycentric_coords=1, cull_backfaces=0 the forward is
 * checked BIT-IDENTICAL against the reference's own rasterize_meshes / rasterize_meshes_naive (built
 * from the reference sources into oracle/_ref by oracle/Makefile) on the reference's test scenes
 * (tests/test_oracle_pin.py) and against committed golden vectors (tests/golden/). The backward is
 * checked end-to-end (per-face grads -> vertex scatter -> world_to_ndc_backward) against the
 * reference's rasterize_backward.
 * perspective_correct=1, cull_backfaces=1 and clip_barycentric_coords=0 do not exist in the reference:
 * their semantics are defined HERE (builder-defined, "parity pinned only by our restatement").
 *
 * Evaluation order is the reference's, operation by operation (core.hpp:61-70 Vec2 ops), compiled with
 * -ffp-contract=off so no FMA contraction changes a rounding.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Same layout as dr_raster_settings in include/dr_raster.h. */
typedef struct {
  int32_t image_h, image_w;
  int32_t faces_per_pixel;
  int32_t bin_size;
  int32_t max_faces_per_bin;
  int32_t _pad;
  double blur_radius;
  double znear;
  uint8_t clip_nonpositive_z;
  uint8_t perspective_correct;
  uint8_t clip_barycentric_coords;
  uint8_t cull_backfaces;
  uint8_t _pad2[4];
} orc_settings;

typedef struct {
  double x, y;
} v2;

#define K_DEGENERATE_AREA 1e-10 /* MR:10 */
#define K_PERSP_EPS 1e-8        /* builder-defined denominator floor for perspective_correct */

static inline v2 sub(v2 a, v2 b) { v2 r = {a.x - b.x, a.y - b.y}; return r; }
static inline v2 add(v2 a, v2 b) { v2 r = {a.x + b.x, a.y + b.y}; return r; }
static inline v2 mul(v2 a, double s) { v2 r = {a.x * s, a.y * s}; return r; }
static inline double dot(v2 a, v2 b) { return a.x * b.x + a.y * b.y; }    /* core.hpp:65 */
static inline double norm2(v2 a) { return a.x * a.x + a.y * a.y; }        /* core.hpp:66 */
static inline double cross(v2 a, v2 b) { return a.x * b.y - a.y * b.x; }  /* core.hpp:68 */
static inline v2 perp(v2 a) { v2 r = {a.y, -a.x}; return r; }             /* core.hpp:70 */
static inline double clamp01(double v) { return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v); } /* std::clamp */

/* MR:12-14 */
static inline double signed_area2(v2 a, v2 b, v2 c) { return cross(sub(b, a), sub(c, a)); }

/* MR:17-24 */
static inline double point_segment_dist2(v2 p, v2 a, v2 b, double* t_out) {
  v2 ab = sub(b, a);
  double len2 = norm2(ab);
  double t = len2 > 0 ? clamp01(dot(sub(p, a), ab) / len2) : 0.0;
  v2 q = add(a, mul(ab, t));
  *t_out = t;
  return norm2(sub(p, q));
}

/* MR:26-34 */
static inline int inside_triangle(v2 p, v2 a, v2 b, v2 c) {
  double area = signed_area2(a, b, c);
  if (fabs(area) < K_DEGENERATE_AREA) return 0;
  double e0 = signed_area2(a, b, p);
  double e1 = signed_area2(b, c, p);
  double e2 = signed_area2(c, a, p);
  if (area > 0) return e0 >= 0 && e1 >= 0 && e2 >= 0;
  return e0 <= 0 && e1 <= 0 && e2 <= 0;
}

/* MR:38-44 */
double orc_point_triangle_dist2_v(v2 p, v2 a, v2 b, v2 c) {
  double t;
  double d = point_segment_dist2(p, a, b, &t);
  double d1 = point_segment_dist2(p, b, c, &t);
  d = d1 < d ? d1 : d; /* std::min(d, d1) returns d unless d1 < d */
  double d2 = point_segment_dist2(p, c, a, &t);
  d = d2 < d ? d2 : d;
  return inside_triangle(p, a, b, c) ? -d : d;
}

/* MR:71-77 */
static inline void barycentric_coords(v2 p, v2 a, v2 b, v2 c, double w[3]) {
  double area = signed_area2(a, b, c);
  w[0] = signed_area2(p, b, c) / area;
  w[1] = signed_area2(p, c, a) / area;
  w[2] = signed_area2(p, a, b) / area;
}

/* MR:79-84 */
static inline void clamp_barycentric(const double w[3], double o[3]) {
  double t0 = clamp01(w[0]), t1 = clamp01(w[1]), t2 = clamp01(w[2]);
  double s = t0 + t1 + t2;
  if (s <= 0) {
    o[0] = o[1] = o[2] = 1.0 / 3;
    return;
  }
  double inv = 1.0 / s;
  o[0] = t0 * inv;
  o[1] = t1 * inv;
  o[2] = t2 * inv;
}

/* Builder-defined perspective correction (PyTorch3D's formula; no reference counterpart). */
static inline double persp_correct(const double w[3], const double z[3], double u[3]) {
  double top0 = w[0] * z[1] * z[2];
  double top1 = w[1] * z[0] * z[2];
  double top2 = w[2] * z[0] * z[1];
  double den = top0 + top1 + top2;
  double denc = den > K_PERSP_EPS ? den : K_PERSP_EPS;
  u[0] = top0 / denc;
  u[1] = top1 / denc;
  u[2] = top2 / denc;
  return den;
}

/* camera.cpp:100-102 */
static inline v2 pixel_center_ndc(int h, int w, int i, int j) {
  v2 r = {(2.0 * j + 1.0) / w - 1.0, 1.0 - (2.0 * i + 1.0) / h};
  return r;
}

/* ------------------------------------------------------------------------------------------ */
/* exported known-answer helpers (mesh_raster.hpp:51-64)                                       */

double orc_point_triangle_dist2(const double* p, const double* a, const double* b, const double* c) {
  v2 P = {p[0], p[1]}, A = {a[0], a[1]}, B = {b[0], b[1]}, C = {c[0], c[1]};
  return orc_point_triangle_dist2_v(P, A, B, C);
}
void orc_barycentric(const double* p, const double* a, const double* b, const double* c, double* w) {
  v2 P = {p[0], p[1]}, A = {a[0], a[1]}, B = {b[0], b[1]}, C = {c[0], c[1]};
  barycentric_coords(P, A, B, C, w);
}
void orc_clamp_barycentric(const double* w, double* o) { clamp_barycentric(w, o); }
void orc_pixel_center_ndc(int h, int w, int i, int j, double* xy) {
  v2 r = pixel_center_ndc(h, w, i, j);
  xy[0] = r.x;
  xy[1] = r.y;
}

/* MR:46-69: envelope gradient; nearest edge (first strict min), t and sign frozen */
static void point_triangle_dist2_backward(v2 p, const v2 v[3], double d_out, v2 g[3]) {
  double best = 0, best_t = 0;
  int best_e = -1;
  for (int e = 0; e < 3; ++e) {
    double t;
    double d = point_segment_dist2(p, v[e], v[(e + 1) % 3], &t);
    if (best_e < 0 || d < best) {
      best = d;
      best_t = t;
      best_e = e;
    }
  }
  double sign = inside_triangle(p, v[0], v[1], v[2]) ? -1.0 : 1.0;
  v2 ea = v[best_e], eb = v[(best_e + 1) % 3];
  v2 q = add(ea, mul(sub(eb, ea), best_t));
  v2 gg = mul(sub(q, p), 2.0 * sign * d_out);
  g[best_e] = add(g[best_e], mul(gg, 1.0 - best_t));
  g[(best_e + 1) % 3] = add(g[(best_e + 1) % 3], mul(gg, best_t));
}
void orc_point_triangle_dist2_backward(const double* p, const double* a, const double* b, const double* c,
                                       double d_out, double* g6) {
  v2 P = {p[0], p[1]};
  v2 v[3] = {{a[0], a[1]}, {b[0], b[1]}, {c[0], c[1]}};
  v2 g[3] = {{0, 0}, {0, 0}, {0, 0}};
  point_triangle_dist2_backward(P, v, d_out, g);
  for (int i = 0; i < 3; ++i) {
    g6[2 * i] = g[i].x;
    g6[2 * i + 1] = g[i].y;
  }
}

/* MR:290-306 */
static void barycentric_backward(v2 p, v2 a, v2 b, v2 c, const double dw[3], v2 g[3]) {
  double area = signed_area2(a, b, c);
  double w[3];
  barycentric_coords(p, a, b, c, w);
  v2 grad_d_a = perp(sub(b, c));
  v2 grad_d_b = perp(sub(c, a));
  v2 grad_d_c = perp(sub(a, b));
  v2 gn0_b = perp(sub(c, p)), gn0_c = perp(sub(p, b));
  v2 gn1_c = perp(sub(a, p)), gn1_a = perp(sub(p, c));
  v2 gn2_a = perp(sub(b, p)), gn2_b = perp(sub(p, a));
  double inv = 1.0 / area;
  double wd = w[0] * dw[0] + w[1] * dw[1] + w[2] * dw[2];
  g[0] = add(g[0], mul(sub(add(mul(gn1_a, dw[1]), mul(gn2_a, dw[2])), mul(grad_d_a, wd)), inv));
  g[1] = add(g[1], mul(sub(add(mul(gn0_b, dw[0]), mul(gn2_b, dw[2])), mul(grad_d_b, wd)), inv));
  g[2] = add(g[2], mul(sub(add(mul(gn0_c, dw[0]), mul(gn1_c, dw[1])), mul(grad_d_c, wd)), inv));
}

/* MR:309-325 */
static void clamp_barycentric_backward(const double wr[3], const double dc[3], double out[3]) {
  double t[3] = {clamp01(wr[0]), clamp01(wr[1]), clamp01(wr[2])};
  double s = t[0] + t[1] + t[2];
  if (s <= 0) {
    out[0] = out[1] = out[2] = 0.0;
    return;
  }
  double hat[3] = {t[0] / s, t[1] / s, t[2] / s};
  double d = dc[0] * hat[0] + dc[1] * hat[1] + dc[2] * hat[2];
  for (int i = 0; i < 3; ++i) {
    double d_t = (dc[i] - d) / s;
    out[i] = (wr[i] > 0.0 && wr[i] < 1.0) ? d_t : 0.0;
  }
}

/* ------------------------------------------------------------------------------------------ */
/* face setup: MR:100-131 (prepare_faces) restated on face_verts                               */

typedef struct {
  int64_t face_id;
  v2 v[3];
  double z[3];
  v2 bb_min, bb_max;
} face_rec;

/* returns 1 if the face survives culling; fills rec */
static int prepare_face(const double* fv, int64_t f, const orc_settings* s, double inflate, face_rec* rec) {
  const double* p = fv + 9 * f;
  for (int k = 0; k < 9; ++k)
    if (!isfinite(p[k])) return 0; /* builder-defined: non-finite faces are culled */
  v2 a = {p[0], p[1]}, b = {p[3], p[4]}, c = {p[6], p[7]};
  double z0 = p[2], z1 = p[5], z2 = p[8];
  if (s->clip_nonpositive_z && (z0 <= 0 || z1 <= 0 || z2 <= 0)) return 0;    /* MR:112 */
  if (z0 < s->znear && z1 < s->znear && z2 < s->znear) return 0;             /* MR:113 */
  double area = signed_area2(a, b, c);
  if (fabs(area) < K_DEGENERATE_AREA) return 0;                              /* MR:114 */
  if (s->cull_backfaces && area > 0) return 0;                               /* builder-defined */
  rec->face_id = f;
  rec->v[0] = a;
  rec->v[1] = b;
  rec->v[2] = c;
  rec->z[0] = z0;
  rec->z[1] = z1;
  rec->z[2] = z2;
  /* MR:123-126; std::min({..}) / std::max({..}) */
  double mnx = a.x, mny = a.y, mxx = a.x, mxy = a.y;
  if (b.x < mnx) mnx = b.x;
  if (c.x < mnx) mnx = c.x;
  if (b.y < mny) mny = b.y;
  if (c.y < mny) mny = c.y;
  if (mxx < b.x) mxx = b.x;
  if (mxx < c.x) mxx = c.x;
  if (mxy < b.y) mxy = b.y;
  if (mxy < c.y) mxy = c.y;
  rec->bb_min.x = mnx - inflate;
  rec->bb_min.y = mny - inflate;
  rec->bb_max.x = mxx + inflate;
  rec->bb_max.y = mxy + inflate;
  return 1;
}

/* ------------------------------------------------------------------------------------------ */
/* per-pixel selection: MR:133-197                                                             */

typedef struct {
  double z;
  int64_t face;
  double bary[3];
  double dist;
} cand;

static inline int cand_less(const cand* x, const cand* y) { /* MR:138-140 */
  return x->z != y->z ? x->z < y->z : x->face < y->face;
}

/* Bounded selection of the K smallest candidates under (z, face id), kept sorted ascending. The
 * reference keeps a max-heap and sorts at emit (MR:144-161); the selected set and its sorted order are
 * the same because (z, id) is a strict total order. */
static inline void offer(cand* arr, int* n, int k, const cand* c) {
  int m = *n;
  if (m == k) {
    if (!cand_less(c, &arr[k - 1])) return;
    m = k - 1;
  }
  int pos = m;
  while (pos > 0 && cand_less(c, &arr[pos - 1])) {
    arr[pos] = arr[pos - 1];
    --pos;
  }
  arr[pos] = *c;
  *n = m + 1;
}

/* MR:166-176 plus the builder-defined flags */
static inline void test_pixel_face(v2 pix, const face_rec* fr, const orc_settings* s, cand* arr, int* n) {
  if (pix.x < fr->bb_min.x || pix.x > fr->bb_max.x || pix.y < fr->bb_min.y || pix.y > fr->bb_max.y) return;
  double dist = orc_point_triangle_dist2_v(pix, fr->v[0], fr->v[1], fr->v[2]);
  if (dist > s->blur_radius) return;
  double w[3], u[3], bary[3];
  barycentric_coords(pix, fr->v[0], fr->v[1], fr->v[2], w);
  if (s->perspective_correct) {
    persp_correct(w, fr->z, u);
  } else {
    u[0] = w[0];
    u[1] = w[1];
    u[2] = w[2];
  }
  if (s->clip_barycentric_coords) {
    clamp_barycentric(u, bary);
  } else {
    bary[0] = u[0];
    bary[1] = u[1];
    bary[2] = u[2];
  }
  double z = bary[0] * fr->z[0] + bary[1] * fr->z[1] + bary[2] * fr->z[2];
  if (z < s->znear) return; /* MR:174 */
  cand c;
  c.z = z;
  c.face = fr->face_id;
  c.bary[0] = bary[0];
  c.bary[1] = bary[1];
  c.bary[2] = bary[2];
  c.dist = dist;
  offer(arr, n, s->faces_per_pixel, &c);
}

/* conservative pixel window for a bbox; the exact fp64 test (MR:168-169) still runs per pixel */
static void pixel_window(double lo, double hi, int n, int* a, int* b) {
  /* x_j = (2j+1)/n - 1  =>  j = ((x+1)n - 1)/2 */
  double ja = ((lo + 1.0) * n - 1.0) * 0.5 - 2.0;
  double jb = ((hi + 1.0) * n - 1.0) * 0.5 + 2.0;
  if (ja < 0) ja = 0;
  if (jb > n - 1) jb = n - 1;
  if (!(ja <= jb)) {
    *a = 1;
    *b = 0;
    return;
  }
  *a = (int)floor(ja);
  *b = (int)ceil(jb);
  if (*b > n - 1) *b = n - 1;
}

/* Return codes follow include/dr_raster.h: 0 OK, 1 SHAPE, 2 INDEX, 3 RANGE, 5 OOM. */
int orc_rasterize_fwd(const double* face_verts, const int64_t* first, const int64_t* num, int64_t n_meshes,
                      int64_t n_faces, const orc_settings* s, int64_t* p2f, double* zbuf, double* bary,
                      double* dists) {
  if (n_meshes < 1) return 1;
  if (s->image_h <= 0 || s->image_w <= 0 || s->faces_per_pixel < 1) return 3;
  for (int64_t b = 0; b < n_meshes; ++b)
    if (num[b] < 0 || first[b] < 0 || first[b] + num[b] > n_faces) return 2;
  const int H = s->image_h, W = s->image_w, K = s->faces_per_pixel;
  const double inflate = sqrt(s->blur_radius > 0.0 ? s->blur_radius : 0.0); /* MR:103 */
  cand* heaps = (cand*)malloc(sizeof(cand) * (size_t)H * W * K);
  int* counts = (int*)malloc(sizeof(int) * (size_t)H * W);
  if (!heaps || !counts) {
    free(heaps);
    free(counts);
    return 5;
  }
  for (int64_t b = 0; b < n_meshes; ++b) {
    memset(counts, 0, sizeof(int) * (size_t)H * W);
    /* Face-major traversal in ascending packed id. MR:214-232 is pixel-major; the K smallest under the
     * strict total order (z, id) do not depend on the visiting order (the reference's own tiled == naive
     * property, test_raster.cpp:127-149). */
    for (int64_t f = first[b]; f < first[b] + num[b]; ++f) {
      face_rec fr;
      if (!prepare_face(face_verts, f, s, inflate, &fr)) continue;
      int j0, j1, i0, i1;
      pixel_window(fr.bb_min.x, fr.bb_max.x, W, &j0, &j1);
      /* y_i = 1 - (2i+1)/H  =>  i = ((1-y)H - 1)/2 ; y decreasing in i */
      pixel_window(-fr.bb_max.y, -fr.bb_min.y, H, &i0, &i1);
      for (int i = i0; i <= i1; ++i)
        for (int j = j0; j <= j1; ++j) {
          v2 pix = pixel_center_ndc(H, W, i, j);
          size_t px = (size_t)i * W + j;
          test_pixel_face(pix, &fr, s, heaps + px * K, &counts[px]);
        }
    }
    /* emit: MR:178-197 */
    for (size_t px = 0; px < (size_t)H * W; ++px) {
      const cand* h = heaps + px * K;
      for (int k = 0; k < K; ++k) {
        size_t slot = ((size_t)b * H * W + px) * K + k;
        if (k < counts[px]) {
          p2f[slot] = h[k].face;
          zbuf[slot] = h[k].z;
          bary[3 * slot] = h[k].bary[0];
          bary[3 * slot + 1] = h[k].bary[1];
          bary[3 * slot + 2] = h[k].bary[2];
          dists[slot] = h[k].dist;
        } else {
          p2f[slot] = -1; /* MR:192-194, alloc_fragments MR:205-208 */
          zbuf[slot] = -1.0;
          bary[3 * slot] = bary[3 * slot + 1] = bary[3 * slot + 2] = 0.0;
          dists[slot] = 0.0;
        }
      }
    }
  }
  free(heaps);
  free(counts);
  return 0;
}

/* Backward restated per slot (MR:345-378); the per-slot vertex cotangents are accumulated into
 * grad_face_verts [F,3,3] = d(x_ndc, y_ndc, z_view) of each face vertex, in slot order (the reference
 * scatters the same per-slot values to vertices in slot order, MR:383-392). bary is the forward's bary
 * (the reference reads frag.bary for the z path, MR:359-375). */
int orc_rasterize_bwd(const double* face_verts, const int64_t* first, const int64_t* num, int64_t n_meshes,
                      int64_t n_faces, const orc_settings* s, const int64_t* p2f, const double* bary,
                      const double* d_zbuf, const double* d_bary, const double* d_dists, double* grad_fv) {
  (void)first;
  (void)num;
  if (n_meshes < 1) return 1;
  if (s->image_h <= 0 || s->image_w <= 0 || s->faces_per_pixel < 1) return 3;
  const int H = s->image_h, W = s->image_w, K = s->faces_per_pixel;
  memset(grad_fv, 0, sizeof(double) * 9 * (size_t)n_faces);
  const int64_t ns = n_meshes * (int64_t)H * W * K;
  for (int64_t slot = 0; slot < ns; ++slot) {
    int64_t fid = p2f[slot];
    if (fid < 0) continue;
    if (fid >= n_faces) return 2;
    const double* q = face_verts + 9 * fid;
    v2 v[3] = {{q[0], q[1]}, {q[3], q[4]}, {q[6], q[7]}};
    double z[3] = {q[2], q[5], q[8]};
    int64_t pix = slot / K;
    int64_t rem = pix % ((int64_t)H * W);
    v2 p = pixel_center_ndc(H, W, (int)(rem / W), (int)(rem % W));
    double w_hat[3] = {bary[3 * slot], bary[3 * slot + 1], bary[3 * slot + 2]};
    double dz = d_zbuf[slot];
    double d_hat[3] = {d_bary[3 * slot] + dz * z[0], d_bary[3 * slot + 1] + dz * z[1],
                       d_bary[3 * slot + 2] + dz * z[2]};
    double w_raw[3];
    barycentric_coords(p, v[0], v[1], v[2], w_raw);
    double dzv[3] = {0.0, 0.0, 0.0}; /* extra z-cotangents from perspective correction */
    double d_w[3];
    if (s->perspective_correct) {
      double u[3], d_u[3], d_top[3];
      double den = persp_correct(w_raw, z, u);
      if (s->clip_barycentric_coords)
        clamp_barycentric_backward(u, d_hat, d_u);
      else {
        d_u[0] = d_hat[0];
        d_u[1] = d_hat[1];
        d_u[2] = d_hat[2];
      }
      if (den > K_PERSP_EPS) {
        double du_u = d_u[0] * u[0] + d_u[1] * u[1] + d_u[2] * u[2];
        for (int i = 0; i < 3; ++i) d_top[i] = (d_u[i] - du_u) / den;
      } else {
        for (int i = 0; i < 3; ++i) d_top[i] = d_u[i] / K_PERSP_EPS;
      }
      /* top0 = w0 z1 z2, top1 = w1 z0 z2, top2 = w2 z0 z1 */
      d_w[0] = d_top[0] * z[1] * z[2];
      d_w[1] = d_top[1] * z[0] * z[2];
      d_w[2] = d_top[2] * z[0] * z[1];
      dzv[0] = d_top[1] * w_raw[1] * z[2] + d_top[2] * w_raw[2] * z[1];
      dzv[1] = d_top[0] * w_raw[0] * z[2] + d_top[2] * w_raw[2] * z[0];
      dzv[2] = d_top[0] * w_raw[0] * z[1] + d_top[1] * w_raw[1] * z[0];
    } else if (s->clip_barycentric_coords) {
      clamp_barycentric_backward(w_raw, d_hat, d_w); /* MR:367 */
    } else {
      d_w[0] = d_hat[0];
      d_w[1] = d_hat[1];
      d_w[2] = d_hat[2];
    }
    v2 dxy[3] = {{0, 0}, {0, 0}, {0, 0}};
    barycentric_backward(p, v[0], v[1], v[2], d_w, dxy);              /* MR:370 */
    point_triangle_dist2_backward(p, v, d_dists[slot], dxy);         /* MR:371-372 */
    double* g = grad_fv + 9 * fid;
    for (int i = 0; i < 3; ++i) {
      g[3 * i + 0] += dxy[i].x;
      g[3 * i + 1] += dxy[i].y;
      g[3 * i + 2] += dz * w_hat[i] + dzv[i]; /* MR:375 */
    }
  }
  return 0;
}

/* ---- silhouette blend (/root/reference/proj/src/shading.cpp, "SH") on fragments ----
 * orc_silhouette_blend:          SH:75-91  alpha[px] = 1 - prod over occupied slots (in slot order) of
 *                                          (1 - sigmoid(-dists / sigma)), sigmoid(x) = 1 / (1 + exp(-x)) (SH:9)
 * orc_silhouette_blend_backward: SH:93-121 d_dists[slot] = d_alpha * prod_{other occupied} (1 - p) *
 *                                          (-p (1 - p) / sigma); pixels with d_alpha == 0 and empty slots get 0 */
static inline double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

void orc_silhouette_blend(const int64_t* p2f, const double* dists, int64_t npix, int k, double sigma,
                          double* alpha) {
  for (int64_t px = 0; px < npix; ++px) {
    double keep = 1.0;
    for (int s = 0; s < k; ++s) {
      int64_t slot = px * k + s;
      if (p2f[slot] < 0) continue;
      double prob = sigmoid(-dists[slot] / sigma);
      keep *= 1.0 - prob;
    }
    alpha[px] = 1.0 - keep;
  }
}

void orc_silhouette_blend_backward(const int64_t* p2f, const double* dists, int64_t npix, int k, double sigma,
                                   const double* d_alpha, double* d_dists) {
  for (int64_t i = 0; i < npix * k; ++i) d_dists[i] = 0.0;
  for (int64_t px = 0; px < npix; ++px) {
    double da = d_alpha[px];
    if (da == 0) continue;
    for (int s = 0; s < k; ++s) {
      int64_t slot = px * k + s;
      if (p2f[slot] < 0) continue;
      double prob_s = sigmoid(-dists[slot] / sigma);
      double rest = 1.0;
      for (int s2 = 0; s2 < k; ++s2) {
        if (s2 == s) continue;
        int64_t slot2 = px * k + s2;
        if (p2f[slot2] < 0) continue;
        rest *= 1.0 - sigmoid(-dists[slot2] / sigma);
      }
      d_dists[slot] = da * rest * (-prob_s * (1.0 - prob_s) / sigma);
    }
  }
}

/* ---- point rasterizer (/root/reference/proj/src/point_render.cpp, "PR") on the points_ndc boundary ----
 * points_ndc [P,3] = (x_ndc, y_ndc, z_view) per packed point; tile = 0 selects rasterize_points_naive (PR:82-103),
 * tile > 0 rasterize_points (PR:105-155). Outputs [N,H,W,K]: idx (-1 empty), zbuf (-1 empty), dists2 (0 empty). */
typedef struct {
  double z;
  int64_t point;
  double dist2;
} pcand;

static inline int pcand_less(const pcand* x, const pcand* y) { /* PR:37 */
  return x->z != y->z ? x->z < y->z : x->point < y->point;
}

static inline void poffer(pcand* arr, int* n, int k, const pcand* c) {
  int m = *n;
  if (m == k) {
    if (!pcand_less(c, &arr[k - 1])) return;
    m = k - 1;
  }
  int pos = m;
  while (pos > 0 && pcand_less(c, &arr[pos - 1])) {
    arr[pos] = arr[pos - 1];
    --pos;
  }
  arr[pos] = *c;
  *n = m + 1;
}

static void pemit(int64_t* idx, double* zbuf, double* d2, int64_t slot0, int k, const pcand* arr, int n) {
  for (int s = 0; s < k; ++s) { /* PR:60-80 */
    if (s < n) {
      idx[slot0 + s] = arr[s].point;
      zbuf[slot0 + s] = arr[s].z;
      d2[slot0 + s] = arr[s].dist2;
    } else {
      idx[slot0 + s] = -1;
      zbuf[slot0 + s] = -1.0;
      d2[slot0 + s] = 0.0;
    }
  }
}

int orc_rasterize_points(const double* pts, const int64_t* first, const int64_t* num, int64_t n_clouds, int64_t P,
                         int h, int w, int k, int tile, double radius, double znear, int clip_nonpositive_z,
                         int64_t* idx, double* zbuf, double* dists2) {
  double r2 = radius * radius; /* PR:112 */
  pcand* arr = (pcand*)malloc(sizeof(pcand) * (size_t)k);
  int64_t* keep = (int64_t*)malloc(sizeof(int64_t) * (size_t)(P > 0 ? P : 1));
  if (!arr || !keep) {
    free(arr);
    free(keep);
    return 5;
  }
  for (int64_t b = 0; b < n_clouds; ++b) {
    /* prepare_points (PR:17-31): clipped (perspective z_view <= 0) or z_view < znear are dropped */
    int64_t nk = 0;
    for (int64_t p = first[b]; p < first[b] + num[b]; ++p) {
      double z = pts[3 * p + 2];
      if (clip_nonpositive_z && z <= 0) continue;
      if (z < znear) continue;
      keep[nk++] = p;
    }
    int tiles_x = tile > 0 ? (w + tile - 1) / tile : 1, tiles_y = tile > 0 ? (h + tile - 1) / tile : 1;
    for (int ty = 0; ty < tiles_y; ++ty) {
      for (int tx = 0; tx < tiles_x; ++tx) {
        int i0 = tile > 0 ? ty * tile : 0, i1 = tile > 0 ? (h < i0 + tile ? h : i0 + tile) : h;
        int j0 = tile > 0 ? tx * tile : 0, j1 = tile > 0 ? (w < j0 + tile ? w : j0 + tile) : w;
        double min_x = 0, max_x = 0, min_y = 0, max_y = 0;
        if (tile > 0) { /* PR:125-132 */
          v2 tl = pixel_center_ndc(h, w, i0, j0), br = pixel_center_ndc(h, w, i1 - 1, j1 - 1);
          min_x = (tl.x < br.x ? tl.x : br.x) - radius;
          max_x = (tl.x < br.x ? br.x : tl.x) + radius;
          min_y = (tl.y < br.y ? tl.y : br.y) - radius;
          max_y = (tl.y < br.y ? br.y : tl.y) + radius;
        }
        for (int i = i0; i < i1; ++i) {
          for (int j = j0; j < j1; ++j) {
            v2 pix = pixel_center_ndc(h, w, i, j);
            int n = 0;
            for (int64_t q = 0; q < nk; ++q) {
              int64_t p = keep[q];
              double x = pts[3 * p], y = pts[3 * p + 1];
              if (tile > 0 && (x < min_x || x > max_x || y < min_y || y > max_y)) continue; /* PR:133-134 */
              v2 xy = {x, y};
              double d2 = norm2(sub(pix, xy)); /* PR:145 */
              if (d2 <= r2) {
                pcand c = {pts[3 * p + 2], p, d2};
                poffer(arr, &n, k, &c);
              }
            }
            pemit(idx, zbuf, dists2, (((int64_t)b * h + i) * w + j) * k, k, arr, n);
          }
        }
      }
    }
  }
  free(arr);
  free(keep);
  return 0;
}

/* d points_ndc [P,3] from per-slot cotangents on zbuf and dists2 (dists2 = |pix - xy|^2, zbuf = z_view) */
void orc_rasterize_points_bwd(const double* pts, int64_t P, int64_t n_clouds, int h, int w, int k, const int64_t* idx,
                              const double* g_zbuf, const double* g_d2, double* grad) {
  for (int64_t i = 0; i < 3 * P; ++i) grad[i] = 0.0;
  int64_t S = n_clouds * h * w * k;
  for (int64_t slot = 0; slot < S; ++slot) {
    int64_t p = idx[slot];
    if (p < 0) continue;
    int64_t px = slot / k, rem = px % ((int64_t)h * w);
    v2 pix = pixel_center_ndc(h, w, (int)(rem / w), (int)(rem % w));
    grad[3 * p] += -2.0 * (pix.x - pts[3 * p]) * g_d2[slot];
    grad[3 * p + 1] += -2.0 * (pix.y - pts[3 * p + 1]) * g_d2[slot];
    grad[3 * p + 2] += g_zbuf[slot];
  }
}
