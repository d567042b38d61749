// Drop-in check: a C++ caller written against the reference's voxplane API
// names (reference include paths, types and functions) replays a VXPF stream
// through the B200 library twice:
//   1. Pipeline::frame  — one run_frames iteration per frame (pipeline.cpp:199-213)
//   2. the per-stage API — VoxelGrid::clear_rays / integrate_frame / recenter,
//      estimate_normals, classify_steppable, build_adjacency, label_components,
//      filter_clusters, fit_planes, refine_plane, make_polygon
//      (the loop of acceptance.cpp:287-336 / voxel_frame_polygons)
// and writes both final polygon sets in the golden-file format.
// Usage: drop_in_replay frames.bin out_dir seed extent
// (compiled by __graft_entry__.build() against oracle/eigen_shim, the test
// build's stand-in for the Eigen the reference's users already have)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "voxplane/pipeline.hpp"
#include "voxplane/plane_fit.hpp"
#include "voxplane/polygonize.hpp"
#include "voxplane/segmentation.hpp"
#include "voxplane/voxel_grid.hpp"

using namespace voxplane;

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s frames.bin out_dir seed extent\n", argv[0]);
    return 2;
  }
  const std::vector<SensorFrame> frames = read_frames_binary(argv[1]);
  const std::string out = argv[2];
  const uint64_t seed = std::strtoull(argv[3], nullptr, 10);
  const int e = std::atoi(argv[4]);
  const double res = 0.01;
  const Vec3i extent(e, e, e);
  const Vec3 start = frames.front().pose.translation;

  SegmentConfig cfg;
  cfg.ransac.seed = seed;
  cfg.refine_exact = true;

  // 1. run_frames through the Pipeline object
  {
    Pipeline pl(res, extent, start, cfg);
    std::vector<PlanePolygon> polys;
    for (const SensorFrame& f : frames) polys = pl.frame(f);
    write_polygons(out + "/polygons_pipeline.txt", polys);
  }

  // 2. the same loop spelled with the per-stage reference API
  VoxelGrid grid(res, extent, start);
  auto global_cell = [&](const Vec3& p) {  // pipeline.cpp:37-41
    return Vec3i(static_cast<int>(std::floor(p.x() / res)), static_cast<int>(std::floor(p.y() / res)),
                 static_cast<int>(std::floor(p.z() / res)));
  };
  Vec3i last = global_cell(start);
  std::vector<PlanePolygon> polys;
  for (const SensorFrame& f : frames) {
    grid.clear_rays(f);
    grid.integrate_frame(f);
    const Vec3i cell = global_cell(f.pose.translation);
    if (cell != last) {
      grid.recenter(f.pose.translation);
      last = cell;
    }
    polys.clear();
    if (grid.occupied_count() == 0) continue;
    const std::vector<SurfaceEstimate> est = estimate_normals(grid, cfg.segmentation);
    const SteppablePartition part = classify_steppable(grid, est, cfg.segmentation);
    const Adjacency adj = build_adjacency(part.steppable, cfg.segmentation, res);
    const ClusterSet set = label_components(part.steppable, adj);
    const std::vector<Cluster> clusters = filter_clusters(set, cfg.segmentation.min_cluster_size);
    const std::vector<ClusterFit> fits = fit_planes(clusters, cfg.ransac);
    for (const ClusterFit& fit : fits) {
      PlaneModel model = refine_plane(fit.inliers, fit.model, cfg.ransac.up);
      model.inlier_count = fit.model.inlier_count;
      model.cluster_label = fit.model.cluster_label;
      auto poly = make_polygon(model, fit.inliers);
      if (poly && poly->area >= cfg.min_polygon_area) polys.push_back(std::move(*poly));
    }
  }
  write_polygons(out + "/polygons_stages.txt", polys);
  std::printf("ok %zu frames\n", frames.size());
  return 0;
}
