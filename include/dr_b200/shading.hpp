// dr_b200 — the reference's silhouette fit step (/root/reference/proj/src/pipeline.cpp:153-162) as two fused GPU
// calls on the B200 C-ABI (include/dr_raster.h):
//
//   rasterize_silhouette          = dr::silhouette_blend(dr::rasterize_meshes(m, c, s), sigma)   shading.hpp:37
//   rasterize_silhouette_backward = dr::rasterize_backward(m, c, s, frag, 0, 0,
//                                       dr::silhouette_blend_backward(frag, sigma, d_alpha))    shading.hpp:39-41
//
// The [B,H,W,K] zbuf / bary / dists (and their cotangents) never exist; pix_to_face is the only per-slot state.
#pragma once

#include <vector>

#include "mesh_raster.hpp"

namespace dr_b200 {

struct SilhouetteFragments {
  int batch = 0, h = 0, w = 0, k = 0;
  std::vector<int64_t> pix_to_face;  // [B,H,W,K], bit-identical to rasterize_meshes
  std::vector<double> alpha;         // [B,H,W] = 1 - prod_k (1 - sigmoid(-dists_k / sigma)) (fp32 on the GPU)
};

SilhouetteFragments rasterize_silhouette(const MeshBatch& m, const Camera& c, const RasterSettings& s, double sigma);

// world-space packed vertex gradients of sum(d_alpha * alpha)
std::vector<Vec3> rasterize_silhouette_backward(const MeshBatch& m, const Camera& c, const RasterSettings& s,
                                                double sigma, const SilhouetteFragments& frag,
                                                const std::vector<double>& d_alpha);

}  // namespace dr_b200
