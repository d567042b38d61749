// voxplane/pipeline.hpp -- run_frames (reference pipeline.hpp:17-33,
// pipeline.cpp:157-245) and the configuration / timing / IoU types it uses
// (config.hpp, metrics.hpp), over the B200 library.
//
// run_frames drives vp_pipeline_run_frames: the whole frame list is one
// device-resident run with several frames in flight (frame k+1's mapping
// overlaps frame k's fitting), and every frame's polygons are packed on the
// device into mapped host memory -- so per_frame_polygons, the per-frame
// FrameTiming spans (CUDA-event device time) and the final polygons come back
// without a host round trip per frame. Outputs equal calling Pipeline::frame
// per frame (tests/test_gpu_parity.py, tests/test_gpu_fullsize.py).
// run.baseline selects the height-map path (vp_hm_*), as the reference does.
#pragma once

#include <chrono>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "voxplane/voxplane.hpp"

namespace voxplane {

// ------------------------------------------------------ scene_sim.hpp types
enum class SceneKind { Stair5, SingleStage, Overhang, SmallObstacle };

struct SceneParams {
  double stair_rise = 0.17;
  double stair_run = 0.29;
  double stair_width = 1.2;
  double approach_length = 1.2;
  double floor_size = 0.88;
  double stage_size = 0.40;
  double stage_height = 0.20;
  double overhang_floor_x = 1.4;
  double overhang_floor_y = 0.9;
  double overhang_clearance = 0.5;
  double overhang_depth = 0.4;
  Vec3 obstacle_size = Vec3(0.07, 0.10, 0.08);
  Vec3 obstacle_center_xy = Vec3(0.3, 0.0, 0.0);
  double obstacle_floor_size = 1.2;
};

struct SensorSpec {
  enum class Kind { PinholeDepth, RayPattern };
  Kind kind = Kind::PinholeDepth;
  int width = 720;
  int height = 480;
  double hfov_deg = 87.0;
  double vfov_deg = 58.0;
  std::vector<Vec3f> pattern;
  double rate_hz = 30.0;
  double max_range = 10.0;
  double noise_sigma = 0.003;
};

// ------------------------------------------------------------- config.hpp
struct OutputConfig {
  std::string dir = "out";
  bool per_frame_polygons = false;
  bool timing_csv = true;
  bool emit_frames = false;
  bool dump_labels = false;
  double min_polygon_area = 0.002;  // m^2
};

struct RunConfig {
  int frames = 100;
  std::uint64_t seed = 1234;
  int threads = 0;        // the reference's CPU pool size; unused on the device
  bool baseline = false;  // height-map path instead of the voxel pipeline
  bool refine = true;
};

struct PipelineConfig {
  SceneKind scene_kind = SceneKind::SingleStage;
  SceneParams scene;
  std::string sensor_kind = "pinhole";
  int pattern_rays = 20000;
  SensorSpec sensor;
  double grid_resolution = 0.01;
  Vec3i grid_extent = Vec3i(200, 200, 200);
  SegmentationParams segmentation;
  RansacParams ransac;
  OutputConfig output;
  RunConfig run;
  // B200 extensions: the device, and bit-identical sequential refine sums
  // (default: the deterministic tree reduction, within 1e-4 rad / 1e-4 m)
  int device = 0;
  bool refine_exact = false;
};

inline PipelineConfig default_config() { return PipelineConfig{}; }

// ------------------------------------------------------------ metrics.hpp
struct PlaneMatch {
  int detected_id = -1;
  int truth_id = -1;
  double iou = 0.0;
};

struct IoUReport {
  std::vector<PlaneMatch> matches;  // truth id ascending
  std::size_t truth_count = 0;
  std::size_t detected_count = 0;
  std::size_t unmatched_truth = 0;
  std::size_t unmatched_detected = 0;
  double mean_iou = 0.0;
  double area_weighted_iou = 0.0;
};

namespace detail {
// PlanePolygon list -> the C ABI's polygon set (views into `store`)
struct PolySet {
  std::vector<vp_polygon> polys;
  std::vector<double> store;
  vp_polygons_t view{};
  explicit PolySet(std::span<const PlanePolygon> ps) {
    size_t nv = 0;
    for (const PlanePolygon& p : ps) nv += p.vertices3d.size();
    store.resize(5 * nv);
    size_t o = 0;
    for (const PlanePolygon& p : ps) {
      vp_polygon q{};
      q.plane = to_c(p.plane);
      q.nverts = static_cast<uint32_t>(p.vertices3d.size());
      q.v2d = store.data() + o;
      for (size_t k = 0; k < p.vertices3d.size(); ++k) {
        store[o + 2 * k] = k < p.vertices2d.size() ? p.vertices2d[k].x() : 0.0;
        store[o + 2 * k + 1] = k < p.vertices2d.size() ? p.vertices2d[k].y() : 0.0;
      }
      q.v3d = store.data() + o + 2 * q.nverts;
      for (size_t k = 0; k < p.vertices3d.size(); ++k)
        for (int c = 0; c < 3; ++c) store[o + 2 * q.nverts + 3 * k + c] = p.vertices3d[k][c];
      o += 5 * q.nverts;
      q.area = p.area;
      polys.push_back(q);
    }
    view.count = polys.size();
    view.polys = polys.data();
  }
};
}  // namespace detail

/// match_planes (metrics.cpp:71-160): plane IoU rasterised on the device
/// (default 0.005 m), greedy one-to-one matching by descending IoU.
inline IoUReport match_planes(std::span<const PlanePolygon> detected, std::span<const PlanePolygon> truth,
                              double raster_res = 0.005, int device = 0) {
  detail::PolySet d(detected), t(truth);
  vp_iou_report r{};
  std::vector<vp_plane_match> m(std::max<size_t>(1, std::min(detected.size(), truth.size())));
  detail::check(vp_match_planes(&d.view, &t.view, raster_res, device, &r, m.data()));
  IoUReport out;
  out.truth_count = r.truth_count;
  out.detected_count = r.detected_count;
  out.unmatched_truth = r.unmatched_truth;
  out.unmatched_detected = r.unmatched_detected;
  out.mean_iou = r.mean_iou;
  out.area_weighted_iou = r.area_weighted_iou;
  for (uint64_t i = 0; i < r.matched; ++i) out.matches.push_back({m[i].detected_id, m[i].truth_id, m[i].iou});
  return out;
}

/// write_iou_report (metrics.cpp:162-185): the reference's key/value text.
inline void write_iou_report(const std::string& path, const IoUReport& report) {
  vp_iou_report r{};
  r.truth_count = report.truth_count;
  r.detected_count = report.detected_count;
  r.matched = report.matches.size();
  r.unmatched_truth = report.unmatched_truth;
  r.unmatched_detected = report.unmatched_detected;
  r.mean_iou = report.mean_iou;
  r.area_weighted_iou = report.area_weighted_iou;
  std::vector<vp_plane_match> m;
  for (const PlaneMatch& x : report.matches) m.push_back({x.detected_id, x.truth_id, x.iou});
  if (vp_write_iou_report(path.c_str(), &r, m.data()) != VP_OK) throw OutputError(vp_last_error());
}

struct FrameTiming {
  std::size_t frame = 0;
  double mapping_ms = 0.0;   // clear + integrate + recenter
  double classify_ms = 0.0;  // normals + steppability
  double cluster_ms = 0.0;   // adjacency + CCL
  double ransac_ms = 0.0;
  double hull_ms = 0.0;
  double total_ms = 0.0;
  std::size_t points = 0;
  std::size_t voxels = 0;
  std::size_t clusters = 0;
};

struct TimingReport {
  std::vector<FrameTiming> frames;
  FrameTiming mean;
};

/// timeline (metrics.cpp:233-258): per-stage means; counts averaged and rounded.
inline TimingReport timeline(std::vector<FrameTiming> frames) {
  TimingReport r;
  r.frames = std::move(frames);
  if (r.frames.empty()) return r;
  FrameTiming& m = r.mean;
  double pts = 0.0, vox = 0.0, clu = 0.0;
  for (const FrameTiming& f : r.frames) {
    m.mapping_ms += f.mapping_ms;
    m.classify_ms += f.classify_ms;
    m.cluster_ms += f.cluster_ms;
    m.ransac_ms += f.ransac_ms;
    m.hull_ms += f.hull_ms;
    m.total_ms += f.total_ms;
    pts += static_cast<double>(f.points);
    vox += static_cast<double>(f.voxels);
    clu += static_cast<double>(f.clusters);
  }
  const double n = static_cast<double>(r.frames.size());
  m.mapping_ms /= n;
  m.classify_ms /= n;
  m.cluster_ms /= n;
  m.ransac_ms /= n;
  m.hull_ms /= n;
  m.total_ms /= n;
  m.points = static_cast<std::size_t>(std::llround(pts / n));
  m.voxels = static_cast<std::size_t>(std::llround(vox / n));
  m.clusters = static_cast<std::size_t>(std::llround(clu / n));
  return r;
}

/// write_timing_csv (metrics.cpp:262-280): one row per frame, then the mean.
inline void write_timing_csv(const std::string& path, const TimingReport& report) {
  std::ofstream os(path);
  if (!os) throw OutputError("timing csv: cannot open for write: " + path);
  os << "frame,points,voxels,clusters,mapping_ms,classify_ms,cluster_ms,ransac_ms,hull_ms,total_ms\n";
  char buf[256];
  auto row = [&](const std::string& tag, const FrameTiming& f) {
    std::snprintf(buf, sizeof buf, "%s,%zu,%zu,%zu,%.3f,%.3f,%.3f,%.3f,%.3f,%.3f\n", tag.c_str(), f.points,
                  f.voxels, f.clusters, f.mapping_ms, f.classify_ms, f.cluster_ms, f.ransac_ms, f.hull_ms,
                  f.total_ms);
    os << buf;
  };
  for (const FrameTiming& f : report.frames) row(std::to_string(f.frame), f);
  if (!report.frames.empty()) row("mean", report.mean);
}

// ----------------------------------------------------------- pipeline.hpp
struct PipelineResult {
  std::vector<PlanePolygon> polygons;  // final frame
  std::optional<IoUReport> iou;        // when ground truth was available
  TimingReport timing;
  std::size_t frames_processed = 0;
  std::string polygons_path;
  std::string iou_report_path;
  std::string timing_csv_path;
};

namespace detail {
inline std::string ensure_out_dir(const PipelineConfig& config) {  // pipeline.cpp:21-36
  namespace fs = std::filesystem;
  const fs::path dir(config.output.dir);
  std::error_code ec;
  fs::create_directories(dir, ec);
  if (ec) throw OutputError("output: cannot create directory " + dir.string());
  const fs::path probe = dir / ".write_probe";
  if (FILE* f = std::fopen(probe.string().c_str(), "w")) {
    std::fclose(f);
    fs::remove(probe, ec);
  } else {
    throw OutputError("output: directory not writable: " + dir.string());
  }
  return dir.string();
}

inline vp_pipeline_params run_params(const PipelineConfig& c) {
  vp_pipeline_params p{};
  p.seg = to_c(c.segmentation);
  p.ransac = to_c(c.ransac);
  p.refine = c.run.refine ? 1 : 0;
  p.min_polygon_area = c.output.min_polygon_area;
  p.refine_exact = c.refine_exact ? 1 : 0;
  return p;
}

struct PolyList {  // owns the vp_polygons_t results of a run
  std::vector<vp_polygons_t*> v;
  ~PolyList() {
    for (auto* p : v) vp_polygons_free(p);
  }
};
}  // namespace detail

/// run_frames (pipeline.cpp:157-245): every frame clear -> integrate ->
/// recenter -> classify -> cluster -> fit -> polygonize; final polygons, IoU
/// report (with ground truth), per-frame polygons and timing CSV land in
/// config.output.dir, as the reference writes them.
inline PipelineResult run_frames(const PipelineConfig& config, const std::vector<SensorFrame>& frames,
                                 const std::vector<PlanePolygon>* ground_truth) {
  namespace fs = std::filesystem;
  const std::string out_dir = detail::ensure_out_dir(config);
  const Vec3 start = frames.empty() ? Vec3::Zero() : frames.front().pose.translation;
  const vp_pipeline_params p = detail::run_params(config);
  PipelineResult result;
  std::vector<FrameTiming> timings(frames.size());
  std::vector<std::vector<PlanePolygon>> per_frame;
  const size_t nf = frames.size();
  if (config.run.baseline) {
    // height map, fixed window around the scene origin (pipeline.cpp:167-194)
    const int32_t e2[2] = {config.grid_extent.x(), config.grid_extent.y()};
    const double c2[2] = {0.0, 0.0};
    vp_heightmap* hm = nullptr;
    detail::check(vp_heightmap_create(config.grid_resolution, e2, c2, config.device, &hm));
    std::unique_ptr<vp_heightmap, void (*)(vp_heightmap*)> hold(hm, vp_heightmap_destroy);
    for (size_t k = 0; k < nf; ++k) {
      const SensorFrame& f = frames[k];
      FrameTiming& t = timings[k];
      t.frame = k;
      t.points = f.points.size();
      const auto t0 = std::chrono::steady_clock::now();
      double R[9], tt[3];
      detail::pose_arrays(f.pose, R, tt);
      detail::check(vp_hm_integrate(hm, detail::frame_xyz(f), f.points.size(), R, tt));
      const auto t1 = std::chrono::steady_clock::now();
      vp_polygons_t* out = nullptr;
      detail::check(vp_hm_segment(hm, &p, &out));
      result.polygons = detail::take(out);
      const auto t2 = std::chrono::steady_clock::now();
      t.mapping_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
      t.cluster_ms = std::chrono::duration<double, std::milli>(t2 - t1).count();
      t.total_ms = std::chrono::duration<double, std::milli>(t2 - t0).count();
      t.clusters = result.polygons.size();
      if (config.output.per_frame_polygons) per_frame.push_back(result.polygons);
    }
  } else if (nf) {
    const int32_t e[3] = {config.grid_extent.x(), config.grid_extent.y(), config.grid_extent.z()};
    const double c[3] = {start.x(), start.y(), start.z()};
    vp_pipeline* pl = nullptr;
    detail::check(vp_pipeline_create(config.grid_resolution, e, c, &p, config.device, &pl));
    std::unique_ptr<vp_pipeline, void (*)(vp_pipeline*)> hold(pl, vp_pipeline_destroy);
    std::vector<const float*> xyz(nf);
    std::vector<uint64_t> n(nf);
    std::vector<double> R(9 * nf), t(3 * nf);
    for (size_t k = 0; k < nf; ++k) {
      xyz[k] = detail::frame_xyz(frames[k]);
      n[k] = frames[k].points.size();
      detail::pose_arrays(frames[k].pose, &R[9 * k], &t[3 * k]);
    }
    std::vector<vp_frame_timing> tm(nf);
    detail::PolyList pf;
    pf.v.assign(nf, nullptr);
    vp_run_outputs ex{};
    ex.timings = tm.data();
    if (config.output.per_frame_polygons) ex.per_frame = pf.v.data();
    vp_polygons_t* last = nullptr;
    detail::check(vp_pipeline_run_frames(pl, nf, xyz.data(), n.data(), R.data(), t.data(), 0, &last, &ex));
    result.polygons = detail::take(last);
    for (size_t k = 0; k < nf; ++k) {
      FrameTiming& ft = timings[k];
      ft.frame = k;
      ft.mapping_ms = tm[k].mapping_ms;
      ft.classify_ms = tm[k].classify_ms;
      ft.cluster_ms = tm[k].cluster_ms;
      ft.ransac_ms = tm[k].ransac_ms;
      ft.hull_ms = tm[k].hull_ms;
      ft.total_ms = tm[k].total_ms;
      ft.points = tm[k].points;
      ft.voxels = tm[k].voxels;
      ft.clusters = tm[k].clusters;
      if (config.output.per_frame_polygons) {
        per_frame.push_back(detail::take(pf.v[k]));
        pf.v[k] = nullptr;
      }
    }
    if (config.output.dump_labels) {
      // the final frame's cluster set (pipeline.cpp:208-212): the grid holds
      // the final map, and segmentation is a pure function of it
      VoxelGrid grid = VoxelGrid::borrow(vp_pipeline_grid(pl), config.grid_resolution, config.grid_extent);
      ClusterSet set;
      if (grid.occupied_count() > 0) {
        const auto est = estimate_normals(grid, config.segmentation);
        const auto part = classify_steppable(grid, est, config.segmentation);
        set = detail::group_labels(part.steppable, label_components_device(part.steppable, config.segmentation,
                                                                           config.grid_resolution,
                                                                           config.device));
      }
      dump_labeled_points((fs::path(out_dir) / "labels_final.txt").string(), set);
    }
  }
  for (size_t k = 0; k < per_frame.size(); ++k) {
    char name[48];
    std::snprintf(name, sizeof name, "polygons_%04zu.txt", k);
    write_polygons((fs::path(out_dir) / name).string(), per_frame[k]);
  }
  result.frames_processed = nf;
  result.timing = timeline(std::move(timings));
  result.polygons_path = (fs::path(out_dir) / "polygons_final.txt").string();
  write_polygons(result.polygons_path, result.polygons);
  if (ground_truth) {
    result.iou = match_planes(result.polygons, *ground_truth, 0.005, config.device);
    result.iou_report_path = (fs::path(out_dir) / "iou_report.txt").string();
    write_iou_report(result.iou_report_path, *result.iou);
  }
  if (config.output.timing_csv) {
    result.timing_csv_path = (fs::path(out_dir) / "timing.csv").string();
    write_timing_csv(result.timing_csv_path, result.timing);
  }
  return result;
}

/// replay_pipeline (pipeline.cpp:291-302): run_frames on a recorded stream,
/// with the IoU report when a truth file is given.
inline PipelineResult replay_pipeline(const PipelineConfig& config, const std::string& frames_path,
                                      const std::string& truth_path = {}) {
  namespace fs = std::filesystem;
  if (!fs::exists(frames_path)) throw MissingInputError("replay: no such file: " + frames_path);
  const std::vector<SensorFrame> frames = read_frames_binary(frames_path);
  std::vector<PlanePolygon> truth;
  if (!truth_path.empty()) {
    if (!fs::exists(truth_path)) throw MissingInputError("replay: no such file: " + truth_path);
    truth = read_polygons(truth_path);
  }
  return run_frames(config, frames, truth_path.empty() ? nullptr : &truth);
}

}  // namespace voxplane
