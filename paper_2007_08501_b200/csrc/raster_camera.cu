// Camera side of the path, GPU-resident:
//
//   k_world_to_face_verts   world_to_ndc (camera.cpp:36-70) per face vertex, gathered through the packed faces
//                           (MeshBatch::faces_packed, batching.cpp:33-43) into face_verts [F,3,3] — what
//                           prepare_faces reads (mesh_raster.cpp:100-122)
//   k_scatter_face_grads    per-face-vertex cotangents -> per-vertex (d_xy, d_z) (mesh_raster.cpp:380-392)
//   k_world_to_ndc_backward world_to_ndc_backward (camera.cpp:72-85) per vertex (mesh_raster.cpp:394-401)
//
// Compiled with -fmad=false like the rasterizer: Mat3::apply is evaluated left to right (core.hpp:113-117)
// and the perspective divide as (f*x)/z + pp, so face_verts are bit-identical to the reference's NdcPoints.
// The scatter uses fp64 atomics (the reference sums in slot order on one thread).
#include <cuda_runtime.h>

#include <cstdint>

#include "raster_kernels.cuh"

namespace drb {

struct View {
  double x, y, z;
};

__device__ __forceinline__ View world_to_view(const CameraArgs& c, double px, double py, double pz) {
  // Mat3::apply (core.hpp:113-117) + translation (camera.cpp:36-38)
  View v;
  v.x = c.r[0] * px + c.r[1] * py + c.r[2] * pz + c.t[0];
  v.y = c.r[3] * px + c.r[4] * py + c.r[5] * pz + c.t[1];
  v.z = c.r[6] * px + c.r[7] * py + c.r[8] * pz + c.t[2];
  return v;
}

// one output point per thread: face vertex t = faces[t] (n = 3F), or point t itself when faces == nullptr (n = P)
__global__ void k_world_to_face_verts(const double* __restrict__ verts, int64_t V, const int64_t* __restrict__ faces,
                                      int64_t n, CameraArgs c, double* __restrict__ fv, int* __restrict__ bad_index) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t vi = faces ? faces[t] : t;
  double x = 0.0, y = 0.0, z = 0.0;
  if (vi < 0 || vi >= V) {
    if (bad_index) atomicExch(bad_index, 1);
    x = y = z = __longlong_as_double(0x7ff8000000000000LL);  // NaN: the face is culled downstream
  } else {
    const View v = world_to_view(c, verts[3 * vi], verts[3 * vi + 1], verts[3 * vi + 2]);
    z = v.z;  // NdcPoint.z_view (camera.cpp:42)
    if (c.perspective) {
      if (!(v.z <= 0)) {  // camera.cpp:44-50; a clipped point keeps xy = (0, 0)
        x = c.focal * v.x / v.z + c.pp[0];
        y = c.focal * v.y / v.z + c.pp[1];
      }
    } else {
      x = c.ortho[0] * v.x;  // camera.cpp:52
      y = c.ortho[1] * v.y;
    }
  }
  fv[3 * t + 0] = x;
  fv[3 * t + 1] = y;
  fv[3 * t + 2] = z;
}

__global__ void k_scatter_face_grads(const int64_t* __restrict__ faces, int64_t F, int64_t V,
                                     const double* __restrict__ gfv, double* __restrict__ acc /*[V,3]*/) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 3 * F) return;
  const int64_t vi = faces[t];
  if (vi < 0 || vi >= V) return;
  const double gx = gfv[3 * t], gy = gfv[3 * t + 1], gz = gfv[3 * t + 2];
  if (gx != 0.0) atomicAdd(acc + 3 * vi, gx);
  if (gy != 0.0) atomicAdd(acc + 3 * vi + 1, gy);
  if (gz != 0.0) atomicAdd(acc + 3 * vi + 2, gz);
}

__global__ void k_world_to_ndc_backward(const double* __restrict__ verts, int64_t V, CameraArgs c,
                                        double* __restrict__ acc /*[V,3] in: (d_x, d_y, d_z) out: d_world*/) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const View pv = world_to_view(c, verts[3 * i], verts[3 * i + 1], verts[3 * i + 2]);
  const double dx = acc[3 * i], dy = acc[3 * i + 1], dz = acc[3 * i + 2];
  double vx, vy, vz;
  if (c.perspective) {
    if (pv.z <= 0) {  // clipped points get zero gradient (camera.cpp:76)
      acc[3 * i] = acc[3 * i + 1] = acc[3 * i + 2] = 0.0;
      return;
    }
    const double f = c.focal;
    vx = dx * f / pv.z;
    vy = dy * f / pv.z;
    vz = -f * (dx * pv.x + dy * pv.y) / (pv.z * pv.z) + dz;
  } else {
    vx = dx * c.ortho[0];
    vy = dy * c.ortho[1];
    vz = dz;
  }
  // Mat3::apply_transposed (core.hpp:118-122)
  acc[3 * i + 0] = c.r[0] * vx + c.r[3] * vy + c.r[6] * vz;
  acc[3 * i + 1] = c.r[1] * vx + c.r[4] * vy + c.r[7] * vz;
  acc[3 * i + 2] = c.r[2] * vx + c.r[5] * vy + c.r[8] * vz;
}

cudaError_t launch_world_to_face_verts(const double* verts, int64_t V, const int64_t* faces, int64_t F,
                                       const CameraArgs& c, double* fv, int* bad_index, cudaStream_t st) {
  if (F <= 0) return cudaSuccess;
  const int64_t n = 3 * F;
  k_world_to_face_verts<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(verts, V, faces, n, c, fv, bad_index);
  return cudaGetLastError();
}

// point clouds: world_to_ndc of every packed point (prepare_points, point_render.cpp:17-31)
cudaError_t launch_world_to_points_ndc(const double* points, int64_t P, const CameraArgs& c, double* out,
                                       cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  k_world_to_face_verts<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(points, P, nullptr, P, c, out, nullptr);
  return cudaGetLastError();
}

// world_to_ndc_backward per point (point_render.cpp:333-337)
cudaError_t launch_points_ndc_backward(const double* points, int64_t P, const CameraArgs& c, const double* g_ndc,
                                       double* g_world, cudaStream_t st) {
  if (P <= 0) return cudaSuccess;
  cudaError_t e = cudaMemcpyAsync(g_world, g_ndc, sizeof(double) * 3 * (size_t)P, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  k_world_to_ndc_backward<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(points, P, c, g_world);
  return cudaGetLastError();
}

cudaError_t launch_face_verts_backward(const double* verts, int64_t V, const int64_t* faces, int64_t F,
                                       const CameraArgs& c, const double* gfv, double* gverts, cudaStream_t st) {
  if (V <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(gverts, 0, sizeof(double) * 3 * (size_t)V, st);
  if (e != cudaSuccess) return e;
  if (F > 0) {
    const int64_t n = 3 * F;
    k_scatter_face_grads<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(faces, F, V, gfv, gverts);
  }
  k_world_to_ndc_backward<<<(unsigned)((V + 255) / 256), 256, 0, st>>>(verts, V, c, gverts);
  return cudaGetLastError();
}

}  // namespace drb
