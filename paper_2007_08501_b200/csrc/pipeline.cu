// Streamed host pipeline (include/dr_raster.h dr_host_pipeline_*): rasterize_meshes forward + backward between
// HOST buffers and the GPU, the way a reference caller uses the path (MeshFragments returned by value and the
// backward fed from host vectors, /root/reference/proj/include/dr/mesh_raster.hpp:41,66-69).
//
// A host caller pays H2D for face_verts (72 B/face) and the cotangents (20 B/slot, fp32) and D2H for the
// fragments (28 B/slot) and grad_face_verts (72 B/face) — C4: 7.4 GB per step, far more than the kernels' own
// time. Meshes are independent (mesh_raster.cpp:240-283), so the batch is cut into contiguous groups of meshes
// and run on three streams:
//
//   h2d  : group g+1's face_verts rows and cotangents        (overlaps)
//   comp : forward + backward of group g                     (overlaps)
//   d2h  : group g-1's fragments and grad_face_verts rows    (overlaps)
//
// Groups balance PCIe bytes (the e2e bound), with geometrically smaller groups at both ends (`ramp`) so the
// pipeline's fill and drain are short. The device->host direction carries more bytes than host->device, and both
// share the link's bidirectional budget: group g's H2D waits for the D2H of group g - lookahead, so inputs arrive
// just in time instead of taking half the link while outputs queue. Every group's calls use the FULL packed
// face_verts with the group's global mesh ranges (face ids stay global; each backward writes only its group's
// rows) and pass host copies of the ranges, so nothing synchronises and the host thread runs ahead.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dr_raster.h"

extern "C" int dr_set_error(int status, const char* msg);

struct dr_host_pipeline {
  int64_t N = 0, F = 0, HWK = 0;
  dr_raster_settings s{};
  int backward = 1, lookahead = 3;
  std::vector<int64_t> first, num;
  std::vector<std::pair<int64_t, int64_t>> groups;  // mesh ranges [g0, g1)
  size_t ws_bytes = 0;
  void* mem = nullptr;  // one device allocation, carved below
  double* fv = nullptr;
  int64_t *d_first = nullptr, *d_num = nullptr, *p2f = nullptr;
  float *zbuf = nullptr, *bary = nullptr, *dists = nullptr, *dz = nullptr, *db = nullptr, *dd = nullptr;
  double* grad = nullptr;
  void* ws = nullptr;
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> ev;  // per group: in, fwd, out, d2h, fv_in
  cudaEvent_t ev_start = nullptr, ev_end[3] = {nullptr, nullptr, nullptr};
};

namespace {

int err(int status, const char* msg) { return dr_set_error(status, msg); }

int cuda_err(cudaError_t e, const char* where) {
  std::string m = std::string("CUDA error in host pipeline ") + where + ": " + cudaGetErrorString(e);
  return dr_set_error(DR_ERR_CUDA, m.c_str());
}

void release(dr_host_pipeline* p) {
  if (!p) return;
  for (cudaEvent_t e : p->ev)
    if (e) cudaEventDestroy(e);
  if (p->ev_start) cudaEventDestroy(p->ev_start);
  for (cudaEvent_t e : p->ev_end)
    if (e) cudaEventDestroy(e);
  for (cudaStream_t s : {p->h2d, p->comp, p->d2h})
    if (s) cudaStreamDestroy(s);
  if (p->mem) cudaFree(p->mem);
  delete p;
}

// contiguous runs of meshes of roughly equal cost; the first and last `ramp` groups are 1/2, 1/4, ... of a full one
std::vector<std::pair<int64_t, int64_t>> contiguous_groups(const std::vector<double>& cost, int n_groups, int ramp) {
  const int64_t n = (int64_t)cost.size();
  n_groups = (int)std::max<int64_t>(1, std::min<int64_t>(n_groups, n));
  const int r = std::max(0, std::min(ramp, (n_groups - 1) / 2));
  std::vector<double> rel((size_t)n_groups, 1.0);
  for (int i = 0; i < r; ++i) rel[(size_t)(r - 1 - i)] = rel[(size_t)(n_groups - r + i)] = std::ldexp(1.0, -(i + 1));
  double tot_rel = 0, tot = 0;
  for (double x : rel) tot_rel += x;
  for (double x : cost) tot += x;
  std::vector<double> bounds((size_t)n_groups);
  double acc_rel = 0;
  for (int g = 0; g < n_groups; ++g) bounds[(size_t)g] = (acc_rel += rel[(size_t)g]) / tot_rel * tot;
  std::vector<std::pair<int64_t, int64_t>> out;
  int64_t start = 0;
  double acc = 0;
  for (int64_t b = 0; b < n; ++b) {
    acc += cost[(size_t)b];
    const bool cut = (int)out.size() < n_groups - 1 && acc >= bounds[out.size()] - 1e-9 * tot;
    if (cut || b == n - 1) {
      out.push_back({start, b + 1});
      start = b + 1;
    }
  }
  return out;
}

template <typename T>
T* carve(char*& cur, int64_t count) {
  T* p = reinterpret_cast<T*>(cur);
  cur += ((size_t)std::max<int64_t>(count, 1) * sizeof(T) + 255) / 256 * 256;
  return p;
}

}  // namespace

extern "C" {

int dr_host_pipeline_create(const int64_t* host_first, const int64_t* host_num, int64_t N, int64_t F,
                            const dr_raster_settings* s, int32_t n_groups, int32_t ramp, int32_t lookahead,
                            int32_t backward, dr_host_pipeline_t* out) {
  if (!out) return err(DR_ERR_USAGE, "dr_host_pipeline_create: out is null");
  *out = nullptr;
  if (!s || !host_first || !host_num) return err(DR_ERR_USAGE, "dr_host_pipeline_create: null pointer");
  if (N < 1 || F < 0) return err(DR_ERR_SHAPE, "dr_host_pipeline_create: empty batch or negative face count");
  for (int64_t b = 0; b < N; ++b) {
    if (host_num[b] < 0 || host_first[b] < 0 || host_first[b] + host_num[b] > F)
      return err(DR_ERR_INDEX, "dr_host_pipeline_create: mesh range outside [0, F)");
    if (b > 0 && host_first[b] < host_first[b - 1] + host_num[b - 1])
      return err(DR_ERR_USAGE, "dr_host_pipeline_create: mesh ranges must be ordered and non-overlapping");
  }
  auto* p = new dr_host_pipeline;
  p->N = N;
  p->F = F;
  p->s = *s;
  p->backward = backward != 0;
  p->lookahead = std::max(0, (int)lookahead);
  p->first.assign(host_first, host_first + N);
  p->num.assign(host_num, host_num + N);
  p->HWK = (int64_t)s->image_h * s->image_w * s->faces_per_pixel;
  // PCIe bytes per mesh of one step: face_verts in + fragments out (+ cotangents in + grad rows out)
  std::vector<double> cost((size_t)N);
  for (int64_t b = 0; b < N; ++b)
    cost[(size_t)b] = 72.0 * (double)p->num[(size_t)b] * (p->backward ? 2 : 1) + (p->backward ? 48.0 : 28.0) * p->HWK;
  p->groups = contiguous_groups(cost, n_groups, ramp);
  for (const auto& g : p->groups) {
    const size_t b = dr_rasterize_meshes_workspace_bytes(g.second - g.first, F, s);
    if (b == 0) {
      release(p);
      return err(DR_ERR_RANGE, (std::string("dr_host_pipeline_create: ") + dr_last_error()).c_str());
    }
    p->ws_bytes = std::max(p->ws_bytes, b);
  }
  const int64_t S = N * p->HWK;
  const size_t bytes = 256 * 16 + 72 * (size_t)F + 16 * (size_t)N + S * (8 + 4 + 12 + 4) +
                       (p->backward ? S * 20 + 72 * (size_t)F : 0) + p->ws_bytes;
  cudaError_t e = cudaMalloc(&p->mem, bytes);
  if (e != cudaSuccess) {
    release(p);
    return err(DR_ERR_OOM, "dr_host_pipeline_create: device allocation failed");
  }
  char* cur = static_cast<char*>(p->mem);
  p->fv = carve<double>(cur, 9 * F);
  p->d_first = carve<int64_t>(cur, N);
  p->d_num = carve<int64_t>(cur, N);
  p->p2f = carve<int64_t>(cur, S);
  p->zbuf = carve<float>(cur, S);
  p->bary = carve<float>(cur, 3 * S);
  p->dists = carve<float>(cur, S);
  if (p->backward) {
    p->dz = carve<float>(cur, S);
    p->db = carve<float>(cur, 3 * S);
    p->dd = carve<float>(cur, S);
    p->grad = carve<double>(cur, 9 * F);
  }
  p->ws = carve<char>(cur, (int64_t)p->ws_bytes);
  e = cudaMemcpy(p->d_first, host_first, sizeof(int64_t) * N, cudaMemcpyHostToDevice);
  // rows of faces in no mesh range (gaps between ranges) are copied back with their group: keep them zero
  if (e == cudaSuccess && p->backward) e = cudaMemset(p->grad, 0, sizeof(double) * 9 * (size_t)std::max<int64_t>(F, 1));
  if (e == cudaSuccess) e = cudaMemcpy(p->d_num, host_num, sizeof(int64_t) * N, cudaMemcpyHostToDevice);
  for (cudaStream_t* st : {&p->h2d, &p->comp, &p->d2h})
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(st, cudaStreamNonBlocking);
  p->ev.assign(5 * p->groups.size(), nullptr);
  for (cudaEvent_t& ev : p->ev)
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_start, cudaEventDisableTiming);
  for (cudaEvent_t& ev : p->ev_end)
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    release(p);
    return cuda_err(e, "create");
  }
  *out = p;
  return DR_OK;
}

int dr_host_pipeline_groups(dr_host_pipeline_t p, int64_t* bounds, int64_t cap) {
  if (!p) return 0;
  for (size_t g = 0; g < p->groups.size() && (int64_t)g < cap && bounds; ++g) {
    bounds[2 * g] = p->groups[g].first;
    bounds[2 * g + 1] = p->groups[g].second;
  }
  return (int)p->groups.size();
}

int dr_host_pipeline_run(dr_host_pipeline_t p, const double* face_verts, int64_t* pix_to_face, float* zbuf,
                         float* bary_coords, float* pix_dists, const float* grad_zbuf, const float* grad_bary,
                         const float* grad_dists, double* grad_face_verts, dr_stream_t stream) {
  if (!p) return err(DR_ERR_USAGE, "dr_host_pipeline_run: null pipeline");
  if ((p->F > 0 && !face_verts) || !pix_to_face || !zbuf || !bary_coords || !pix_dists)
    return err(DR_ERR_USAGE, "dr_host_pipeline_run: null host buffer");
  if (p->backward && (!grad_zbuf || !grad_bary || !grad_dists || (p->F > 0 && !grad_face_verts)))
    return err(DR_ERR_USAGE, "dr_host_pipeline_run: null cotangent / gradient buffer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaEventRecord(p->ev_start, st);
  for (cudaStream_t s : {p->h2d, p->comp, p->d2h})
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, p->ev_start, 0);
  if (e != cudaSuccess) return cuda_err(e, "start");
  const int64_t HWK = p->HWK;
  for (size_t gi = 0; gi < p->groups.size(); ++gi) {
    const int64_t g0 = p->groups[gi].first, g1 = p->groups[gi].second, n = g1 - g0;
    const int64_t lo = p->first[(size_t)g0], hi = p->first[(size_t)(g1 - 1)] + p->num[(size_t)(g1 - 1)];
    const int64_t s0 = g0 * HWK, ns = n * HWK;
    cudaEvent_t ev_in = p->ev[5 * gi], ev_fwd = p->ev[5 * gi + 1], ev_out = p->ev[5 * gi + 2],
                ev_d2h = p->ev[5 * gi + 3], ev_fv = p->ev[5 * gi + 4];
    if (p->lookahead > 0 && gi >= (size_t)p->lookahead) {
      e = cudaStreamWaitEvent(p->h2d, p->ev[5 * (gi - p->lookahead) + 3], 0);
      if (e != cudaSuccess) return cuda_err(e, "lookahead");
    }
    // h2d
    if (hi > lo) e = cudaMemcpyAsync(p->fv + 9 * lo, face_verts + 9 * lo, sizeof(double) * 9 * (hi - lo),
                                     cudaMemcpyHostToDevice, p->h2d);
    // the forward needs only the face_verts rows: it starts (and its fragments leave) while the cotangents arrive
    if (e == cudaSuccess) e = cudaEventRecord(ev_fv, p->h2d);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->comp, ev_fv, 0);
    if (p->backward) {
      if (e == cudaSuccess) e = cudaMemcpyAsync(p->dz + s0, grad_zbuf + s0, sizeof(float) * ns, cudaMemcpyHostToDevice, p->h2d);
      if (e == cudaSuccess) e = cudaMemcpyAsync(p->db + 3 * s0, grad_bary + 3 * s0, sizeof(float) * 3 * ns, cudaMemcpyHostToDevice, p->h2d);
      if (e == cudaSuccess) e = cudaMemcpyAsync(p->dd + s0, grad_dists + s0, sizeof(float) * ns, cudaMemcpyHostToDevice, p->h2d);
    }
    if (e == cudaSuccess) e = cudaEventRecord(ev_in, p->h2d);
    if (e != cudaSuccess) return cuda_err(e, "h2d");
    // comp
    int rc = dr_rasterize_meshes_fwd_hr(p->fv, p->d_first + g0, p->d_num + g0, n, p->F, &p->s, p->p2f + s0,
                                        p->zbuf + s0, p->bary + 3 * s0, p->dists + s0, p->ws, p->ws_bytes,
                                        reinterpret_cast<dr_stream_t>(p->comp), p->first.data() + g0,
                                        p->num.data() + g0);
    if (rc) return rc;
    e = cudaEventRecord(ev_fwd, p->comp);
    if (e != cudaSuccess) return cuda_err(e, "forward event");
    if (p->backward) {
      e = cudaStreamWaitEvent(p->comp, ev_in, 0);  // the group's cotangents
      if (e != cudaSuccess) return cuda_err(e, "cotangent wait");
      rc = dr_rasterize_meshes_bwd_hr(p->fv, p->d_first + g0, p->d_num + g0, n, p->F, &p->s, p->p2f + s0,
                                      p->bary + 3 * s0, p->dz + s0, p->db + 3 * s0, p->dd + s0, p->grad,
                                      reinterpret_cast<dr_stream_t>(p->comp), p->first.data() + g0,
                                      p->num.data() + g0);
      if (rc) return rc;
    }
    e = cudaEventRecord(ev_out, p->comp);
    // d2h: fragments as soon as the forward is done, gradients after the backward
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->d2h, ev_fwd, 0);
    if (e == cudaSuccess) e = cudaMemcpyAsync(pix_to_face + s0, p->p2f + s0, sizeof(int64_t) * ns, cudaMemcpyDeviceToHost, p->d2h);
    if (e == cudaSuccess) e = cudaMemcpyAsync(zbuf + s0, p->zbuf + s0, sizeof(float) * ns, cudaMemcpyDeviceToHost, p->d2h);
    if (e == cudaSuccess) e = cudaMemcpyAsync(bary_coords + 3 * s0, p->bary + 3 * s0, sizeof(float) * 3 * ns, cudaMemcpyDeviceToHost, p->d2h);
    if (e == cudaSuccess) e = cudaMemcpyAsync(pix_dists + s0, p->dists + s0, sizeof(float) * ns, cudaMemcpyDeviceToHost, p->d2h);
    if (p->backward && hi > lo) {
      if (e == cudaSuccess) e = cudaStreamWaitEvent(p->d2h, ev_out, 0);
      if (e == cudaSuccess) e = cudaMemcpyAsync(grad_face_verts + 9 * lo, p->grad + 9 * lo, sizeof(double) * 9 * (hi - lo),
                                                cudaMemcpyDeviceToHost, p->d2h);
    }
    if (e == cudaSuccess) e = cudaEventRecord(ev_d2h, p->d2h);
    if (e != cudaSuccess) return cuda_err(e, "d2h");
  }
  // the caller's stream waits for all three
  cudaStream_t ss[3] = {p->h2d, p->comp, p->d2h};
  for (int i = 0; i < 3 && e == cudaSuccess; ++i) {
    e = cudaEventRecord(p->ev_end[i], ss[i]);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, p->ev_end[i], 0);
  }
  return e == cudaSuccess ? DR_OK : cuda_err(e, "end");
}

int dr_host_pipeline_destroy(dr_host_pipeline_t p) {
  if (p) {
    cudaStreamSynchronize(p->h2d);
    cudaStreamSynchronize(p->comp);
    cudaStreamSynchronize(p->d2h);
  }
  release(p);
  return DR_OK;
}

}  // extern "C"
