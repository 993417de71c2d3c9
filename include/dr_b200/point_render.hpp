// dr_b200 — C++ host mirror of the reference's point rasterizer (/root/reference/proj/include/dr/point_render.hpp
// and PointCloudBatch from dr/batching.hpp:127-157), running on the B200 C-ABI (include/dr_raster.h).
//
//   PointCloudBatch                 batching.hpp:127-157 (points only; features are the compositor's business)
//   PointRasterSettings             point_render.hpp:14-19
//   PointFragments                  point_render.hpp:21-30 (fp64 payload: bit-identical to the reference)
//   rasterize_points / _naive       point_render.hpp:33-36
//   splat_opacity                   point_render.hpp:39
//   splat_position_backward         point_render.hpp:66-68
// Projection, rasterization and the backward run as sm_100a kernels; results come back as host vectors.
#pragma once

#include <vector>

#include "mesh_raster.hpp"

namespace dr_b200 {

class PointCloudBatch {
 public:
  // ShapeError on an empty batch (batching.cpp PointCloudBatch constructor)
  explicit PointCloudBatch(std::vector<std::vector<Vec3>> points_list);

  int size() const { return int(points_list_.size()); }
  const std::vector<std::vector<Vec3>>& points_list() const { return points_list_; }
  const std::vector<int64_t>& num_points_per_cloud() const { return num_points_; }
  const PackedView<Vec3>& points_packed() const { return points_packed_; }
  int64_t total_points() const { return points_packed_.offsets.back(); }
  PointCloudBatch with_points(const std::vector<Vec3>& new_points_packed) const;

 private:
  std::vector<std::vector<Vec3>> points_list_;
  std::vector<int64_t> num_points_;
  PackedView<Vec3> points_packed_;
};

struct PointRasterSettings {
  int image_h = 64, image_w = 64;
  int points_per_pixel = 8;  // K (<= 128 on the GPU path)
  double radius = 0.05;      // splat radius in NDC
  int tile_size = 16;        // 0 => naive
};

struct PointFragments {
  int batch = 0, h = 0, w = 0, k = 0;
  std::vector<int64_t> idx;      // packed point ids, -1 empty
  std::vector<double> zbuf;      // z_view, -1 empty
  std::vector<double> dists2;    // squared NDC distance pixel centre -> splat centre, 0 empty

  int64_t slots() const { return int64_t(batch) * h * w * k; }
};

PointFragments rasterize_points(const PointCloudBatch& pc, const Camera& c, const PointRasterSettings& s);
PointFragments rasterize_points_naive(const PointCloudBatch& pc, const Camera& c, const PointRasterSettings& s);

// alpha = 1 - dists2 / radius^2; empty slots get 0 (point_render.cpp:157-168)
std::vector<double> splat_opacity(const PointFragments& frag, double radius);

// slot alpha cotangents -> packed world-space point gradients (point_render.cpp:302-338)
std::vector<Vec3> splat_position_backward(const PointCloudBatch& pc, const Camera& c, const PointRasterSettings& s,
                                          const PointFragments& frag, const std::vector<double>& d_alphas);

}  // namespace dr_b200
