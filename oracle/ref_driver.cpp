// oracle/_ref driver — TEST INFRASTRUCTURE ONLY (never linked by the product).
//
// A C ABI over the UNMODIFIED reference sources in /root/reference/proj/core
// (compiled by oracle/Makefile against oracle/eigen_shim). It exists to pin
// the C restatement (oracle/voxplane_oracle.c) and to serve as the CPU
// baseline (`bench.py --impl reference`, cpu_baseline.kind = "reference"):
//   ref_session_*   the per-frame body of run_frames (pipeline.cpp:176-213)
//                   with a stage trace in the voxplane_trace.h format
//   ref_run_named   the reference's own test_pipeline.cpp runs, to reproduce
//                   the golden files in proj/test_scratch byte for byte
//   ref_render      render_frame (scene_sim.cpp:186-236) for arbitrary scenes,
//                   to pin the product's input generator
//   ref_replay      replay_pipeline (pipeline.cpp:291-302) on a VXPF file
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "voxplane/config.hpp"
#include "voxplane/frame_io.hpp"
#include "voxplane/metrics.hpp"
#include "voxplane/parallel.hpp"
#include "voxplane/pipeline.hpp"
#include "voxplane/plane_fit.hpp"
#include "voxplane/polygon_io.hpp"
#include "voxplane/polygonize.hpp"
#include "voxplane/scene_sim.hpp"
#include "voxplane/segmentation.hpp"
#include "voxplane/voxel_grid.hpp"
#include "voxplane_b200.h"
#include "voxplane_trace.h"

using namespace voxplane;

namespace {

thread_local std::string g_err;

struct Writer {
  std::vector<uint8_t> b;
  template <typename T>
  void put(const T& v) {
    const auto* p = reinterpret_cast<const uint8_t*>(&v);
    b.insert(b.end(), p, p + sizeof(T));
  }
  void put3(const Vec3& v) {
    put(v.x());
    put(v.y());
    put(v.z());
  }
  void put3i(const Vec3i& v) {
    put<int32_t>(v.x());
    put<int32_t>(v.y());
    put<int32_t>(v.z());
  }
};

SegmentationParams seg_from(const vp_seg_params& s) {
  SegmentationParams p;
  p.neighbor_radius = s.neighbor_radius;
  p.min_neighbors = s.min_neighbors;
  p.max_angle_deg = s.max_angle_deg;
  p.adjacency_angle_deg = s.adjacency_angle_deg;
  p.distance_th = s.distance_th;
  p.min_cluster_size = s.min_cluster_size;
  p.up = Vec3(s.up[0], s.up[1], s.up[2]);
  return p;
}

RansacParams ransac_from(const vp_ransac_params& r) {
  RansacParams p;
  p.iterations = r.iterations;
  p.inlier_eps = r.inlier_eps;
  p.seed = r.seed;
  p.up = Vec3(r.up[0], r.up[1], r.up[2]);
  p.execution = r.execution ? RansacExecution::PerClusterSerial : RansacExecution::ClusterParallel;
  return p;
}

// pipeline.cpp:37-41 (file-static in the reference)
Vec3i global_cell(const Vec3& p, double resolution) {
  return Vec3i(static_cast<int>(std::floor(p.x() / resolution)),
               static_cast<int>(std::floor(p.y() / resolution)),
               static_cast<int>(std::floor(p.z() / resolution)));
}

SensorFrame make_frame(const float* xyz, uint64_t n, const double* R, const double* t) {
  SensorFrame f;
  f.points.resize(n);
  for (uint64_t i = 0; i < n; ++i) f.points[i] = Vec3f(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) f.pose.rotation(r, c) = R[3 * r + c];
    f.pose.translation[r] = t[r];
  }
  return f;
}

struct Session {
  VoxelGrid grid;
  vp_pipeline_params params;
  Vec3i last_cell;
  uint32_t frame = 0;
  bool fixed = false;  // fixed window, never recentered
  Session(double res, const Vec3i& ext, const Vec3& c, const vp_pipeline_params& p)
      : grid(res, ext, c), params(p), last_cell(global_cell(c, res)) {}
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_free(void* p) { std::free(p); }

void ref_set_threads(int n) { set_thread_count(n <= 0 ? default_thread_count() : unsigned(n)); }

void* ref_session_create(double res, const int32_t ext[3], const double center[3],
                         const vp_pipeline_params* p) {
  try {
    return new Session(res, Vec3i(ext[0], ext[1], ext[2]), Vec3(center[0], center[1], center[2]), *p);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_session_destroy(void* s) { delete static_cast<Session*>(s); }

// Fixed-window mode: clear_rays + integrate_frame + voxel_frame_polygons per
// frame with no recenter (the C5 map and the slab path).
void ref_session_set_fixed(void* s, int fixed) { static_cast<Session*>(s)->fixed = fixed != 0; }

// One run_frames iteration (pipeline.cpp:199-213) with every stage of
// voxel_frame_polygons (pipeline.cpp:43-85) serialised.
int ref_session_frame(void* sp, const float* xyz, uint64_t n, const double R[9], const double t[3],
                      uint8_t** out, uint64_t* out_len) {
  auto* s = static_cast<Session*>(sp);
  try {
    const SensorFrame frame = make_frame(xyz, n, R, t);
    Writer w;
    w.b.insert(w.b.end(), {'V', 'P', 'T', 'R'});
    w.put<uint32_t>(VP_TRACE_VERSION);
    w.put<uint32_t>(s->frame++);

    const ClearStats cs = s->grid.clear_rays(frame);
    const UpdateStats us = s->grid.integrate_frame(frame);
    const double res = s->grid.resolution();
    const Vec3i cell = global_cell(frame.pose.translation, res);
    ShiftStats ss;
    uint8_t recentered = 0;
    if (!s->fixed && cell != s->last_cell) {
      ss = s->grid.recenter(frame.pose.translation);
      s->last_cell = cell;
      recentered = 1;
    }
    w.put<uint64_t>(cs.voxels_cleared);
    w.put<uint64_t>(cs.voxels_freed);
    w.put<uint64_t>(us.voxels_touched);
    w.put<uint64_t>(us.points_discarded);
    w.put(recentered);
    w.put3i(ss.shift);
    w.put<uint64_t>(ss.voxels_dropped);
    w.put3(s->grid.origin());
    w.put<uint64_t>(s->grid.occupied_count());

    const vp_pipeline_params& P = s->params;
    const SegmentationParams seg = seg_from(P.seg);
    const RansacParams rp = ransac_from(P.ransac);
    if (s->grid.occupied_count() == 0) {
      for (int k = 0; k < 5; ++k) w.put<uint64_t>(0);  // V, S, K, skipped, unfit
      w.put<uint64_t>(0);                              // F
      w.put<uint64_t>(0);                              // P
      // layout: V | S | K | skipped unfit F | P
    } else {
      const std::vector<OccupiedVoxel> occ = s->grid.occupied_voxels();
      w.put<uint64_t>(occ.size());
      for (const auto& v : occ) w.put3i(v.index);
      for (const auto& v : occ) w.put3(v.mean);
      for (const auto& v : occ) w.put<uint32_t>(v.count);
      for (const auto& v : occ) w.put<uint8_t>(static_cast<uint8_t>(v.status));

      const std::vector<SurfaceEstimate> est = estimate_normals(s->grid, seg);
      for (const auto& e : est) w.put3(e.normal);
      for (const auto& e : est) w.put<int32_t>(e.neighbor_count);
      for (const auto& e : est) w.put<uint8_t>(e.valid ? 1 : 0);

      const SteppablePartition part = classify_steppable(s->grid, est, seg);
      w.put<uint64_t>(part.steppable.size());
      for (const auto& p : part.steppable) w.put3i(p.voxel);
      for (const auto& p : part.steppable) w.put3(p.mean);
      for (const auto& p : part.steppable) w.put3(p.normal);

      const Adjacency adj = build_adjacency(part.steppable, seg, res);
      const ClusterSet set = label_components(part.steppable, adj);
      for (int32_t l : set.labels) w.put<int32_t>(l);
      const std::vector<Cluster> clusters = filter_clusters(set, seg.min_cluster_size);
      w.put<uint64_t>(clusters.size());
      for (const auto& c : clusters) {
        w.put<int32_t>(c.label);
        w.put<uint64_t>(c.members.size());
      }

      FitStats fs;
      const std::vector<ClusterFit> fits = fit_planes(clusters, rp, &fs);
      w.put<uint64_t>(fs.clusters_skipped_small);
      w.put<uint64_t>(fs.clusters_unfit);
      w.put<uint64_t>(fits.size());
      for (const auto& f : fits) {
        w.put3(f.model.normal);
        w.put(f.model.offset);
        w.put<int32_t>(f.model.inlier_count);
        w.put<int32_t>(f.model.cluster_label);
        w.put<uint64_t>(f.inliers.size());
        for (const auto& q : f.inliers) w.put3(q);
      }
      std::vector<PlanePolygon> polys;
      for (const auto& f : fits) {
        PlaneModel model = f.model;
        if (P.refine) {  // pipeline.cpp:74-78
          model = refine_plane(f.inliers, model, rp.up);
          model.inlier_count = f.model.inlier_count;
          model.cluster_label = f.model.cluster_label;
        }
        w.put3(model.normal);
        w.put(model.offset);
        auto poly = make_polygon(model, f.inliers);  // pipeline.cpp:79-81
        if (poly && poly->area >= P.min_polygon_area) polys.push_back(std::move(*poly));
      }
      w.put<uint64_t>(polys.size());
      for (const auto& p : polys) {
        w.put3(p.plane.normal);
        w.put(p.plane.offset);
        w.put<int32_t>(p.plane.inlier_count);
        w.put<int32_t>(p.plane.cluster_label);
        w.put<uint64_t>(p.vertices2d.size());
        for (const auto& q : p.vertices2d) {
          w.put(q.x());
          w.put(q.y());
        }
        for (const auto& q : p.vertices3d) w.put3(q);
        w.put(p.area);
      }
    }
    *out_len = w.b.size();
    *out = static_cast<uint8_t*>(std::malloc(w.b.size()));
    std::memcpy(*out, w.b.data(), w.b.size());
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return VP_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VP_ECUDA;
  }
}

// One run_frames iteration (pipeline.cpp:199-213) without serialisation:
// the CPU-baseline step. Returns wall milliseconds in *ms.
int ref_session_step(void* sp, const float* xyz, uint64_t n, const double R[9], const double t[3],
                     double* ms, uint64_t* npolys) {
  auto* s = static_cast<Session*>(sp);
  try {
    const SensorFrame frame = make_frame(xyz, n, R, t);
    StageTimer timer;
    timer.start();
    s->grid.clear_rays(frame);
    s->grid.integrate_frame(frame);
    const Vec3i cell = global_cell(frame.pose.translation, s->grid.resolution());
    if (!s->fixed && cell != s->last_cell) {
      s->grid.recenter(frame.pose.translation);
      s->last_cell = cell;
    }
    std::vector<PlanePolygon> polygons;
    const vp_pipeline_params& P = s->params;
    if (s->grid.occupied_count() > 0) {  // voxel_frame_polygons (pipeline.cpp:43-85)
      const SegmentationParams seg = seg_from(P.seg);
      const RansacParams rp = ransac_from(P.ransac);
      const std::vector<SurfaceEstimate> est = estimate_normals(s->grid, seg);
      const SteppablePartition part = classify_steppable(s->grid, est, seg);
      const Adjacency adj = build_adjacency(part.steppable, seg, s->grid.resolution());
      const ClusterSet set = label_components(part.steppable, adj);
      const std::vector<Cluster> clusters = filter_clusters(set, seg.min_cluster_size);
      const std::vector<ClusterFit> fits = fit_planes(clusters, rp);
      for (const ClusterFit& fit : fits) {
        PlaneModel model = fit.model;
        if (P.refine) {
          model = refine_plane(fit.inliers, model, rp.up);
          model.inlier_count = fit.model.inlier_count;
          model.cluster_label = fit.model.cluster_label;
        }
        auto poly = make_polygon(model, fit.inliers);
        if (poly && poly->area >= P.min_polygon_area) polygons.push_back(std::move(*poly));
      }
    }
    *ms = timer.stop_ms();
    if (npolys) *npolys = polygons.size();
    s->frame++;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VP_EINVAL;
  }
}

// Raw grid state for state-parity tests on small windows: sums (C x 3),
// counts (C), statuses (C), window (logical) x-major order.
int ref_session_cells(void* sp, double* sums, uint32_t* counts, uint8_t* status) {
  auto* s = static_cast<Session*>(sp);
  const Vec3i e = s->grid.extent();
  std::size_t f = 0;
  for (int x = 0; x < e.x(); ++x)
    for (int y = 0; y < e.y(); ++y)
      for (int z = 0; z < e.z(); ++z, ++f) {
        const auto& c = s->grid.cell(Vec3i(x, y, z));
        sums[3 * f] = c.sx;
        sums[3 * f + 1] = c.sy;
        sums[3 * f + 2] = c.sz;
        counts[f] = c.count;
        status[f] = static_cast<uint8_t>(c.status);
      }
  return 0;
}

// The reference's own test runs (proj/tests/test_pipeline.cpp) whose outputs
// are the golden files in proj/test_scratch.
int ref_run_named(const char* name, const char* outdir) {
  try {
    const std::string n(name);
    PipelineConfig c = default_config();
    auto tiny = [&]() {  // test_pipeline.cpp:15-26
      c.scene_kind = SceneKind::SmallObstacle;
      c.sensor.width = 96;
      c.sensor.height = 72;
      c.grid_extent = Vec3i(140, 140, 140);
      c.run.frames = 6;
      c.run.seed = 77;
      c.ransac.seed = 77;
    };
    if (n == "t1" || n == "t3" || n == "live") {
      tiny();
      if (n == "t1") c.run.threads = 1;
      if (n == "t3") c.run.threads = 3;
      if (n == "live") c.output.emit_frames = true;
    } else if (n == "smallobs") {  // :55-62
      tiny();
      c.sensor.width = 160;
      c.sensor.height = 120;
      c.run.frames = 10;
      c.output.dump_labels = true;
    } else if (n == "stair") {  // :77-88
      c.scene_kind = SceneKind::Stair5;
      c.sensor.width = 240;
      c.sensor.height = 180;
      c.grid_extent = Vec3i(200, 200, 200);
      c.run.frames = 25;
      c.run.seed = 5;
      c.ransac.seed = 5;
    } else if (n == "rosette") {  // :110-121
      c.scene_kind = SceneKind::SmallObstacle;
      c.sensor_kind = "rosette";
      c.pattern_rays = 12000;
      c.grid_extent = Vec3i(200, 200, 200);
      c.run.frames = 30;
      c.run.seed = 5;
      c.ransac.seed = 5;
    } else if (n == "baseline") {  // :183-192
      tiny();
      c.run.baseline = true;
      c.run.frames = 4;
      c.output.emit_frames = true;  // the stream, for the height-map parity test
    } else {
      g_err = "unknown run " + n;
      return VP_EINVAL;
    }
    c.output.dir = outdir;
    run_pipeline(c);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VP_ECUDA;
  }
}

// replay_pipeline (pipeline.cpp:291-302) with a JSON config
// (config.cpp:132-232); output.dir is overridden by outdir.
int ref_replay(const char* config_json, const char* frames_path, const char* outdir,
               int threads) {
  try {
    PipelineConfig c = config_json && *config_json ? load_config_file(config_json) : default_config();
    c.output.dir = outdir;
    if (threads >= 0) c.run.threads = threads;
    replay_pipeline(c, frames_path);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VP_ECUDA;
  }
}

// render_frame (scene_sim.cpp:186-236) over a pose list, for an arbitrary
// scene: boxes (6 per box: min xyz, max xyz), rects (14 per rect: R row-major
// 9, t 3, half_u, half_v). sensor_kind 0 = pinhole, 1 = ray pattern.
// Writes a VXPF stream (frame_io.cpp:110-125).
int ref_render(const double* boxes, int nb, const double* rects, int nr, int sensor_kind,
               int width, int height, double hfov, double vfov, const float* pattern,
               int npattern, double rate_hz, double max_range, double noise_sigma,
               const double* poses, int nframes, uint64_t seed, const char* frames_path) {
  try {
    Scene scene;
    for (int i = 0; i < nb; ++i)
      scene.boxes.push_back({Vec3(boxes[6 * i], boxes[6 * i + 1], boxes[6 * i + 2]),
                             Vec3(boxes[6 * i + 3], boxes[6 * i + 4], boxes[6 * i + 5])});
    for (int i = 0; i < nr; ++i) {
      Rect r;
      const double* q = rects + 14 * i;
      for (int a = 0; a < 3; ++a) {
        for (int b = 0; b < 3; ++b) r.pose.rotation(a, b) = q[3 * a + b];
        r.pose.translation[a] = q[9 + a];
      }
      r.half_u = q[12];
      r.half_v = q[13];
      scene.rects.push_back(r);
    }
    SensorSpec spec;
    spec.kind = sensor_kind == 0 ? SensorSpec::Kind::PinholeDepth : SensorSpec::Kind::RayPattern;
    spec.width = width;
    spec.height = height;
    spec.hfov_deg = hfov;
    spec.vfov_deg = vfov;
    for (int i = 0; i < npattern; ++i)
      spec.pattern.push_back(Vec3f(pattern[3 * i], pattern[3 * i + 1], pattern[3 * i + 2]));
    spec.rate_hz = rate_hz;
    spec.max_range = max_range;
    spec.noise_sigma = noise_sigma;
    std::vector<SensorFrame> frames;
    for (int f = 0; f < nframes; ++f) {
      Pose p;
      const double* q = poses + 12 * f;
      for (int a = 0; a < 3; ++a) {
        for (int b = 0; b < 3; ++b) p.rotation(a, b) = q[3 * a + b];
        p.translation[a] = q[9 + a];
      }
      frames.push_back(render_frame(scene, spec, p, seed, static_cast<uint64_t>(f)));
    }
    write_frames_binary(frames_path, frames);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VP_ECUDA;
  }
}

// Stock scenes and trajectories: build_scene (scene_sim.cpp:43-114) boxes /
// rects, and default_trajectory (pipeline.cpp:89-155) poses for a scene kind
// (0 Stair5, 1 SingleStage, 2 Overhang, 3 SmallObstacle) and frame count.
int ref_stock_scene(int kind, double* boxes, int* nb, double* rects, int* nr) {
  const Scene s = build_scene(static_cast<SceneKind>(kind), SceneParams{});
  *nb = static_cast<int>(s.boxes.size());
  *nr = static_cast<int>(s.rects.size());
  for (std::size_t i = 0; i < s.boxes.size(); ++i)
    for (int k = 0; k < 3; ++k) {
      boxes[6 * i + k] = s.boxes[i].min[k];
      boxes[6 * i + 3 + k] = s.boxes[i].max[k];
    }
  for (std::size_t i = 0; i < s.rects.size(); ++i) {
    double* q = rects + 14 * i;
    for (int a = 0; a < 3; ++a) {
      for (int b = 0; b < 3; ++b) q[3 * a + b] = s.rects[i].pose.rotation(a, b);
      q[9 + a] = s.rects[i].pose.translation[a];
    }
    q[12] = s.rects[i].half_u;
    q[13] = s.rects[i].half_v;
  }
  return 0;
}

int ref_default_trajectory(int kind, int frames, double rate_hz, double* poses) {
  PipelineConfig c = default_config();
  c.scene_kind = static_cast<SceneKind>(kind);
  c.run.frames = frames;
  c.sensor.rate_hz = rate_hz;
  const std::vector<Pose> ps = default_trajectory(c);
  for (std::size_t f = 0; f < ps.size(); ++f) {
    double* q = poses + 12 * f;
    for (int a = 0; a < 3; ++a) {
      for (int b = 0; b < 3; ++b) q[3 * a + b] = ps[f].rotation(a, b);
      q[9 + a] = ps[f].translation[a];
    }
  }
  return static_cast<int>(ps.size());
}

int ref_spherical_pattern(int n, float* out) {
  const auto v = make_spherical_pattern(n);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) out[3 * i + k] = v[i][k];
  return n;
}

int ref_rosette_pattern(int n, float* out) {
  const auto v = make_rosette_pattern(n);
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) out[3 * i + k] = v[i][k];
  return n;
}

}  // extern "C"

// ---- reference utilities for the drop-in API checks (TEST INFRASTRUCTURE) ----
#include "voxplane/jacobi.hpp"
#include "voxplane/rng.hpp"

extern "C" {

// hull_filter / monotone_chain / convex_hull (polygonize.cpp:50-144):
// op 0 / 1 / 2 on n 2-D points; out has room for 2n doubles.
int ref_hull(int op, const double* pts, uint64_t n, int directions, double* out, uint64_t* m) {
  std::vector<Vec2> p(n);
  for (uint64_t i = 0; i < n; ++i) p[i] = Vec2(pts[2 * i], pts[2 * i + 1]);
  const std::vector<Vec2> r = op == 0 ? hull_filter(p, directions) : op == 1 ? monotone_chain(p)
                                                                              : convex_hull(p, directions);
  for (size_t i = 0; i < r.size(); ++i) {
    out[2 * i] = r[i].x();
    out[2 * i + 1] = r[i].y();
  }
  *m = r.size();
  return 0;
}

// jacobi_eigen_sym3 (jacobi.cpp:46-81): a row-major, vecs column-major.
void ref_jacobi(const double a[9], double vals[3], double vecs[9]) {
  Mat3 m;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) m(r, c) = a[3 * r + c];
  const EigenSym3 e = jacobi_eigen_sym3(m);
  for (int k = 0; k < 3; ++k) {
    vals[k] = e.eigenvalues[k];
    for (int r = 0; r < 3; ++r) vecs[3 * k + r] = e.eigenvectors(r, k);
  }
}

// CounterRng (rng.hpp:13-64) streams: count draws of each kind from fresh
// generators keyed (seed, k1, k2).
void ref_rng(uint64_t seed, uint64_t k1, uint64_t k2, uint64_t count, uint32_t below_n, uint64_t* raw,
             double* uni, uint32_t* below, double* normals) {
  CounterRng a(seed, k1, k2), b(seed, k1, k2), c(seed, k1, k2), d(seed, k1, k2);
  for (uint64_t i = 0; i < count; ++i) {
    raw[i] = a.next_u64();
    uni[i] = b.uniform();
    below[i] = c.below(below_n);
    normals[i] = d.normal();
  }
}

// label_components(steppable, adjacency) (segmentation.cpp:147-194) on CSR lists.
int ref_label_adjacency(uint64_t n, const uint64_t* rows, const int32_t* cols, int32_t* labels) {
  std::vector<SteppablePoint> st(n);
  Adjacency adj(n);
  for (uint64_t i = 0; i < n; ++i) adj[i].assign(cols + rows[i], cols + rows[i + 1]);
  const ClusterSet set = label_components(st, adj);
  for (uint64_t i = 0; i < n; ++i) labels[i] = set.labels[i];
  return 0;
}

}  // extern "C"
