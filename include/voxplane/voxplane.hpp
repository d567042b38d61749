// voxplane C++ API on the B200 library — the drop-in for the reference's
// proj/core hot path (namespace voxplane, same type and function names and
// argument meaning as /root/reference/proj/core/include/voxplane/*.hpp),
// implemented header-only over the C ABI in voxplane_b200.h. Link with
// -lvoxplane_b200. Like the reference it is written against Eigen 3
// (<Eigen/Dense> from the including project).
//
// Differences a caller can observe, all deliberate:
//   * VoxelGrid::cell() returns the Cell by value (the map lives in HBM);
//   * every grid takes an optional CUDA device index (default 0);
//   * segment() is the exported form of the reference's file-static
//     voxel_frame_polygons (pipeline.cpp:43-85), and Pipeline::frame() is one
//     iteration of run_frames (pipeline.cpp:199-213).
// Errors are reported with the reference's exception types.
#pragma once

#include <Eigen/Dense>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <numeric>
#include <optional>
#include <sstream>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "voxplane_b200.h"

namespace voxplane {

// ----------------------------------------------------------- types.hpp
using Vec3 = Eigen::Vector3d;
using Vec3f = Eigen::Vector3f;
using Vec3i = Eigen::Vector3i;
using Vec2 = Eigen::Vector2d;
using Mat3 = Eigen::Matrix3d;

enum class VoxelStatus : std::uint8_t { Free = 0, Occupied = 1, Steppable = 2 };

struct OccupiedVoxel {
  Vec3i index;
  Vec3 mean;
  std::uint32_t count = 0;
  VoxelStatus status = VoxelStatus::Free;
};

struct Pose {
  Mat3 rotation = Mat3::Identity();
  Vec3 translation = Vec3::Zero();
  Vec3 apply(const Vec3& p) const { return rotation * p + translation; }
};

constexpr double kRadToDeg = 57.295779513082320876798;
constexpr double kDegToRad = 0.017453292519943295769237;

inline Vec3 orient_up(const Vec3& n, const Vec3& up) {  // types.hpp:43-52
  const double d = n.dot(up);
  if (d < 0.0) return -n;
  if (d > 0.0) return n;
  for (int k = 0; k < 3; ++k) {
    if (n[k] > 0.0) return n;
    if (n[k] < 0.0) return -n;
  }
  return n;
}

struct SensorFrame {
  std::vector<Vec3f> points;
  Pose pose;
  double timestamp = 0.0;
};

struct UpdateStats {
  std::size_t voxels_touched = 0;
  std::size_t points_discarded = 0;
};
struct ClearStats {
  std::size_t voxels_cleared = 0;
  std::size_t voxels_freed = 0;
};
struct ShiftStats {
  Vec3i shift = Vec3i::Zero();
  std::size_t voxels_dropped = 0;
};

// ----------------------------------------------------------- errors.hpp
struct MissingInputError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct OutputError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int rc) {
  if (rc == VP_OK) return;
  const std::string msg = vp_last_error();
  if (rc == VP_EINVAL || rc == VP_EEMPTY) throw std::invalid_argument(msg);
  if (rc == VP_ENOMEM) throw std::bad_alloc();
  throw std::runtime_error("voxplane_b200: " + msg);
}
inline void pose_arrays(const Pose& p, double R[9], double t[3]) {
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) R[3 * r + c] = p.rotation(r, c);
    t[r] = p.translation[r];
  }
}
inline const float* frame_xyz(const SensorFrame& f) {
  static_assert(sizeof(Vec3f) == 3 * sizeof(float), "Vec3f must be 3 packed floats");
  return f.points.empty() ? nullptr : reinterpret_cast<const float*>(f.points.data());
}
}  // namespace detail

// ------------------------------------------------------ segmentation.hpp
struct SegmentationParams {
  int neighbor_radius = 1;
  int min_neighbors = 3;
  double max_angle_deg = 15.0;
  double adjacency_angle_deg = 15.0;
  double distance_th = 0.05;
  int min_cluster_size = 30;
  Vec3 up = Vec3::UnitZ();
};

struct SurfaceEstimate {
  Vec3i voxel;
  Vec3 mean = Vec3::Zero();
  Vec3 normal = Vec3::Zero();
  int neighbor_count = 0;
  double angle_to_up_deg = 0.0;
  bool valid = false;
};

struct SteppablePoint {
  Vec3i voxel;
  Vec3 mean;
  Vec3 normal;
};

struct SteppablePartition {
  std::vector<SteppablePoint> steppable;
  std::vector<Vec3i> objects;
};

using Adjacency = std::vector<std::vector<std::int32_t>>;

struct Cluster {
  std::int32_t label = 0;
  std::vector<SteppablePoint> members;
};

struct ClusterSet {
  std::vector<std::int32_t> labels;
  std::vector<Cluster> clusters;
};

// --------------------------------------------------------- plane_fit.hpp
struct PlaneModel {
  Vec3 normal = Vec3::UnitZ();
  double offset = 0.0;
  int inlier_count = 0;
  std::int32_t cluster_label = -1;
};

enum class RansacExecution { ClusterParallel, PerClusterSerial };

struct RansacParams {
  int iterations = 100;
  double inlier_eps = 0.01;
  std::uint64_t seed = 0;
  Vec3 up = Vec3::UnitZ();
  RansacExecution execution = RansacExecution::ClusterParallel;
};

struct ClusterFit {
  PlaneModel model;
  std::vector<Vec3> inliers;
};

struct FitStats {
  std::size_t clusters_skipped_small = 0;
  std::size_t clusters_unfit = 0;
};

// -------------------------------------------------------- polygonize.hpp
struct PlaneBasis {
  Vec3 u;
  Vec3 v;
  Vec3 origin;
};

struct PlanePolygon {
  PlaneModel plane;
  std::vector<Vec2> vertices2d;
  std::vector<Vec3> vertices3d;
  double area = 0.0;
};

namespace detail {
inline vp_seg_params to_c(const SegmentationParams& p) {
  vp_seg_params s{};
  s.neighbor_radius = p.neighbor_radius;
  s.min_neighbors = p.min_neighbors;
  s.max_angle_deg = p.max_angle_deg;
  s.adjacency_angle_deg = p.adjacency_angle_deg;
  s.distance_th = p.distance_th;
  s.min_cluster_size = p.min_cluster_size;
  for (int k = 0; k < 3; ++k) s.up[k] = p.up[k];
  return s;
}
inline vp_ransac_params to_c(const RansacParams& p) {
  vp_ransac_params r{};
  r.iterations = p.iterations;
  r.inlier_eps = p.inlier_eps;
  r.seed = p.seed;
  for (int k = 0; k < 3; ++k) r.up[k] = p.up[k];
  r.execution = p.execution == RansacExecution::PerClusterSerial ? 1 : 0;
  return r;
}
inline PlaneModel from_c(const vp_plane& q) {
  PlaneModel m;
  m.normal = Vec3(q.normal[0], q.normal[1], q.normal[2]);
  m.offset = q.offset;
  m.inlier_count = q.inlier_count;
  m.cluster_label = q.cluster_label;
  return m;
}
inline vp_plane to_c(const PlaneModel& m) {
  vp_plane q{};
  for (int k = 0; k < 3; ++k) q.normal[k] = m.normal[k];
  q.offset = m.offset;
  q.inlier_count = m.inlier_count;
  q.cluster_label = m.cluster_label;
  return q;
}
inline std::vector<PlanePolygon> take(vp_polygons_t* out, bool keep_empty = false) {
  std::vector<PlanePolygon> v;
  for (size_t i = 0; i < out->count; ++i) {
    const vp_polygon& q = out->polys[i];
    if (!q.nverts && !keep_empty) continue;
    PlanePolygon p;
    p.plane = from_c(q.plane);
    for (uint32_t k = 0; k < q.nverts; ++k) {
      p.vertices2d.emplace_back(q.v2d[2 * k], q.v2d[2 * k + 1]);
      p.vertices3d.emplace_back(q.v3d[3 * k], q.v3d[3 * k + 1], q.v3d[3 * k + 2]);
    }
    p.area = q.area;
    v.push_back(std::move(p));
  }
  vp_polygons_free(out);
  return v;
}
}  // namespace detail

// -------------------------------------------------------- voxel_grid.hpp
/// Robot-centric dense 3D voxel map, resident in HBM (voxel_grid.hpp:17-91).
class VoxelGrid {
 public:
  struct Cell {
    double sx = 0.0, sy = 0.0, sz = 0.0;
    std::uint32_t count = 0;
    VoxelStatus status = VoxelStatus::Free;
  };

  VoxelGrid(double resolution, const Vec3i& extent, const Vec3& center, int device = 0)
      : resolution_(resolution), extent_(extent) {
    const int32_t e[3] = {extent.x(), extent.y(), extent.z()};
    const double c[3] = {center.x(), center.y(), center.z()};
    detail::check(vp_grid_create(resolution, e, c, device, &g_));
    owned_ = true;
  }
  ~VoxelGrid() {
    if (owned_) vp_grid_destroy(g_);
  }
  VoxelGrid(const VoxelGrid&) = delete;
  VoxelGrid& operator=(const VoxelGrid&) = delete;

  double resolution() const { return resolution_; }
  const Vec3i& extent() const { return extent_; }
  Vec3 origin() const {
    double o[3];
    detail::check(vp_grid_info(g_, o, nullptr, nullptr, nullptr));
    return Vec3(o[0], o[1], o[2]);
  }
  Vec3 world_center() const { return origin() + extent_.cast<double>() * (0.5 * resolution_); }
  bool in_bounds(const Vec3i& idx) const {
    return (idx.array() >= 0).all() && (idx.array() < extent_.array()).all();
  }
  Vec3i world_to_index(const Vec3& p) const {
    const Vec3 o = origin();
    return Vec3i(static_cast<int>(std::floor((p.x() - o.x()) / resolution_)),
                 static_cast<int>(std::floor((p.y() - o.y()) / resolution_)),
                 static_cast<int>(std::floor((p.z() - o.z()) / resolution_)));
  }
  Vec3 index_to_center(const Vec3i& idx) const {
    return origin() + (idx.cast<double>() + Vec3::Constant(0.5)) * resolution_;
  }
  std::size_t flat(const Vec3i& idx) const {
    return (static_cast<std::size_t>(idx.x()) * extent_.y() + idx.y()) * extent_.z() + idx.z();
  }
  Vec3i unflat(std::size_t f) const {
    const std::size_t ze = extent_.z(), ye = extent_.y();
    return Vec3i(static_cast<int>(f / (ze * ye)), static_cast<int>((f / ze) % ye),
                 static_cast<int>(f % ze));
  }
  Cell cell(const Vec3i& idx) const {
    const int32_t i[3] = {idx.x(), idx.y(), idx.z()};
    double s[3];
    Cell c;
    uint8_t st = 0;
    detail::check(vp_get_cell(g_, i, s, &c.count, &st));
    c.sx = s[0];
    c.sy = s[1];
    c.sz = s[2];
    c.status = static_cast<VoxelStatus>(st);
    return c;
  }
  std::size_t cell_count() const {
    return static_cast<std::size_t>(extent_.x()) * extent_.y() * extent_.z();
  }
  std::size_t occupied_count() const {
    uint64_t n = 0;
    detail::check(vp_grid_info(g_, nullptr, nullptr, nullptr, &n));
    return n;
  }
  void merge_point(const Vec3i& idx, const Vec3& p) {
    const int32_t i[3] = {idx.x(), idx.y(), idx.z()};
    const double q[3] = {p.x(), p.y(), p.z()};
    detail::check(vp_merge_point(g_, i, q));
  }
  UpdateStats integrate_frame(const SensorFrame& frame) {
    double R[9], t[3];
    detail::pose_arrays(frame.pose, R, t);
    vp_update_stats s{};
    detail::check(vp_integrate_frame(g_, detail::frame_xyz(frame), frame.points.size(), R, t, &s));
    return UpdateStats{s.voxels_touched, s.points_discarded};
  }
  ClearStats clear_rays(const SensorFrame& frame) {
    double R[9], t[3];
    detail::pose_arrays(frame.pose, R, t);
    vp_clear_stats s{};
    detail::check(vp_clear_rays(g_, detail::frame_xyz(frame), frame.points.size(), R, t, &s));
    return ClearStats{s.voxels_cleared, s.voxels_freed};
  }
  ShiftStats recenter(const Vec3& new_center) {
    const double c[3] = {new_center.x(), new_center.y(), new_center.z()};
    vp_shift_stats s{};
    detail::check(vp_recenter(g_, c, &s));
    ShiftStats out;
    out.shift = Vec3i(s.shift[0], s.shift[1], s.shift[2]);
    out.voxels_dropped = s.voxels_dropped;
    return out;
  }
  std::vector<OccupiedVoxel> occupied_voxels() const {
    vp_occupied_t* o = nullptr;
    detail::check(vp_occupied_voxels(g_, &o));
    std::vector<OccupiedVoxel> v(o->count);
    for (size_t i = 0; i < o->count; ++i) {
      v[i].index = Vec3i(o->idx[3 * i], o->idx[3 * i + 1], o->idx[3 * i + 2]);
      v[i].mean = Vec3(o->mean[3 * i], o->mean[3 * i + 1], o->mean[3 * i + 2]);
      v[i].count = o->npts[i];
      v[i].status = static_cast<VoxelStatus>(o->status[i]);
    }
    vp_occupied_free(o);
    return v;
  }
  void set_status(const Vec3i& idx, VoxelStatus s) {
    const int32_t i[3] = {idx.x(), idx.y(), idx.z()};
    detail::check(vp_set_status(g_, i, static_cast<uint8_t>(s)));
  }
  static Vec3 cell_mean(const Cell& c) {
    return Vec3(c.sx, c.sy, c.sz) / static_cast<double>(c.count);
  }
  vp_grid* handle() const { return g_; }
  /// A non-owning view of a library-owned grid (e.g. a pipeline's map).
  static VoxelGrid borrow(vp_grid* g, double resolution, const Vec3i& extent) {
    return VoxelGrid(g, resolution, extent);
  }

 private:
  friend class Pipeline;
  VoxelGrid(vp_grid* borrowed, double res, const Vec3i& ext)
      : resolution_(res), extent_(ext), g_(borrowed), owned_(false) {}
  double resolution_;
  Vec3i extent_;
  vp_grid* g_ = nullptr;
  bool owned_ = false;
};

// ------------------------------------------------------ segmentation API
/// estimate_normals (segmentation.cpp:19-67); throws on an empty grid.
inline std::vector<SurfaceEstimate> estimate_normals(const VoxelGrid& grid,
                                                     const SegmentationParams& params) {
  const vp_seg_params sp = detail::to_c(params);
  vp_estimates_t* e = nullptr;
  detail::check(vp_estimate_normals(grid.handle(), &sp, &e));
  std::vector<SurfaceEstimate> v(e->count);
  for (size_t i = 0; i < e->count; ++i) {
    v[i].voxel = Vec3i(e->idx[3 * i], e->idx[3 * i + 1], e->idx[3 * i + 2]);
    v[i].mean = Vec3(e->mean[3 * i], e->mean[3 * i + 1], e->mean[3 * i + 2]);
    v[i].normal = Vec3(e->normal[3 * i], e->normal[3 * i + 1], e->normal[3 * i + 2]);
    v[i].neighbor_count = e->neighbor_count[i];
    v[i].angle_to_up_deg = e->angle_to_up_deg[i];
    v[i].valid = e->valid[i] != 0;
  }
  vp_estimates_free(e);
  return v;
}

/// classify_steppable (segmentation.cpp:69-85) over the given estimates: the
/// predicate (valid, neighbor_count >= min_neighbors, angle_to_up_deg <=
/// max_angle_deg) runs on the device, which also writes the statuses into the
/// grid; the partition keeps the estimates' order.
inline SteppablePartition classify_steppable(VoxelGrid& grid,
                                             const std::vector<SurfaceEstimate>& estimates,
                                             const SegmentationParams& params) {
  const size_t n = estimates.size();
  std::vector<int32_t> idx(3 * n), nc(n);
  std::vector<double> ang(n);
  std::vector<uint8_t> valid(n), st(n);
  for (size_t i = 0; i < n; ++i) {
    const SurfaceEstimate& e = estimates[i];
    idx[3 * i] = e.voxel.x();
    idx[3 * i + 1] = e.voxel.y();
    idx[3 * i + 2] = e.voxel.z();
    nc[i] = e.neighbor_count;
    ang[i] = e.angle_to_up_deg;
    valid[i] = e.valid ? 1 : 0;
  }
  const vp_seg_params sp = detail::to_c(params);
  detail::check(vp_classify_estimates(grid.handle(), &sp, n, idx.data(), nc.data(), ang.data(), valid.data(),
                                      st.data()));
  SteppablePartition part;
  for (size_t i = 0; i < n; ++i) {
    const SurfaceEstimate& e = estimates[i];
    if (st[i] == 2)
      part.steppable.push_back({e.voxel, e.mean, e.normal});
    else
      part.objects.push_back(e.voxel);
  }
  return part;
}

namespace detail {
struct StepArrays {
  std::vector<int32_t> idx;
  std::vector<double> mean, normal;
  vp_steppable_t view{};
  explicit StepArrays(const std::vector<SteppablePoint>& s) {
    for (const SteppablePoint& p : s) {
      idx.insert(idx.end(), {p.voxel.x(), p.voxel.y(), p.voxel.z()});
      mean.insert(mean.end(), {p.mean.x(), p.mean.y(), p.mean.z()});
      normal.insert(normal.end(), {p.normal.x(), p.normal.y(), p.normal.z()});
    }
    view.count = s.size();
    view.idx = idx.data();
    view.mean = mean.data();
    view.normal = normal.data();
  }
};
}  // namespace detail

/// build_adjacency (segmentation.cpp:87-132), lists ascending.
inline Adjacency build_adjacency(const std::vector<SteppablePoint>& steppable,
                                 const SegmentationParams& params, double resolution,
                                 int device = 0) {
  detail::StepArrays a(steppable);
  const vp_seg_params sp = detail::to_c(params);
  uint64_t* rows = nullptr;
  int32_t* cols = nullptr;
  uint64_t ne = 0;
  detail::check(vp_build_adjacency(&a.view, &sp, resolution, device, &rows, &cols, &ne));
  Adjacency adj(steppable.size());
  for (size_t i = 0; i < steppable.size(); ++i) adj[i].assign(cols + rows[i], cols + rows[i + 1]);
  vp_free(rows);
  vp_free(cols);
  return adj;
}

namespace detail {
// ClusterSet from canonical labels: clusters in ascending label order,
// members in ascending ordinal (segmentation.cpp:182-193)
inline ClusterSet group_labels(const std::vector<SteppablePoint>& steppable, std::vector<int32_t> labels) {
  ClusterSet set;
  const size_t n = steppable.size();
  std::vector<int64_t> slot(n, -1);
  for (size_t i = 0; i < n; ++i) {
    const int32_t l = labels[i];
    if (slot[l] < 0) {
      slot[l] = static_cast<int64_t>(set.clusters.size());
      set.clusters.emplace_back();
      set.clusters.back().label = l;
    }
    set.clusters[slot[l]].members.push_back(steppable[i]);
  }
  set.labels = std::move(labels);
  return set;
}
}  // namespace detail

/// label_components (segmentation.cpp:147-194) on a given adjacency: a
/// device union-find over the lists; labels are the canonical component
/// minima.
inline ClusterSet label_components(const std::vector<SteppablePoint>& steppable,
                                   const Adjacency& adjacency, int device = 0) {
  const size_t n = steppable.size();
  std::vector<uint64_t> rows(n + 1, 0);
  for (size_t i = 0; i < n; ++i) rows[i + 1] = rows[i] + adjacency[i].size();
  std::vector<int32_t> cols;
  cols.reserve(rows[n]);
  for (const auto& l : adjacency) cols.insert(cols.end(), l.begin(), l.end());
  std::vector<int32_t> labels(n);
  detail::check(vp_label_components_adjacency(n, rows.data(), cols.data(), device, labels.data()));
  return detail::group_labels(steppable, std::move(labels));
}

/// Fused build_adjacency + label_components on the device (no adjacency lists).
inline std::vector<int32_t> label_components_device(const std::vector<SteppablePoint>& steppable,
                                                    const SegmentationParams& params,
                                                    double resolution, int device = 0) {
  detail::StepArrays a(steppable);
  const vp_seg_params sp = detail::to_c(params);
  std::vector<int32_t> labels(steppable.size());
  detail::check(vp_label_components(&a.view, &sp, resolution, device, labels.data()));
  return labels;
}

inline std::vector<Cluster> filter_clusters(const ClusterSet& set, int min_size) {
  std::vector<Cluster> out;
  for (const Cluster& c : set.clusters)
    if (static_cast<int>(c.members.size()) >= min_size) out.push_back(c);
  return out;
}

inline void dump_labeled_points(const std::string& path, const ClusterSet& set) {
  std::ofstream os(path);
  if (!os) throw std::runtime_error("dump_labeled_points: cannot open " + path);
  char buf[160];
  for (const Cluster& c : set.clusters)
    for (const SteppablePoint& p : c.members) {
      std::snprintf(buf, sizeof buf, "%.9g %.9g %.9g %d %.9g %.9g %.9g\n", p.mean.x(), p.mean.y(),
                    p.mean.z(), c.label, p.normal.x(), p.normal.y(), p.normal.z());
      os << buf;
    }
}

// --------------------------------------------------------- plane fitting
/// fit_planes (plane_fit.cpp:55-131): cluster-parallel RANSAC on the device.
inline std::vector<ClusterFit> fit_planes(const std::vector<Cluster>& clusters,
                                          const RansacParams& params, FitStats* stats = nullptr,
                                          int device = 0) {
  std::vector<int32_t> labels;
  std::vector<uint64_t> offs{0};
  std::vector<double> means;
  for (const Cluster& c : clusters) {
    labels.push_back(c.label);
    for (const SteppablePoint& p : c.members) means.insert(means.end(), {p.mean.x(), p.mean.y(), p.mean.z()});
    offs.push_back(offs.back() + c.members.size());
  }
  const vp_ransac_params rp = detail::to_c(params);
  vp_fits_t* f = nullptr;
  detail::check(vp_fit_planes(clusters.size(), labels.data(), offs.data(), means.data(), &rp, device, &f));
  std::vector<ClusterFit> fits(f->count);
  for (size_t i = 0; i < f->count; ++i) {
    fits[i].model = detail::from_c(f->models[i]);
    for (uint64_t k = f->offsets[i]; k < f->offsets[i + 1]; ++k)
      fits[i].inliers.emplace_back(f->inliers[3 * k], f->inliers[3 * k + 1], f->inliers[3 * k + 2]);
  }
  if (stats) {
    stats->clusters_skipped_small = f->clusters_skipped_small;
    stats->clusters_unfit = f->clusters_unfit;
  }
  vp_fits_free(f);
  return fits;
}

/// refine_plane (plane_fit.cpp:133-154), bit-identical sequential sums.
inline PlaneModel refine_plane(std::span<const Vec3> inliers, const PlaneModel& initial,
                               const Vec3& up = Vec3::UnitZ(), int device = 0) {
  std::vector<double> pts;
  for (const Vec3& p : inliers) pts.insert(pts.end(), {p.x(), p.y(), p.z()});
  vp_plane model = detail::to_c(initial);
  uint64_t offs[2] = {0, inliers.size()};
  vp_fits_t f{};
  f.count = 1;
  f.models = &model;
  f.offsets = offs;
  f.inliers = pts.data();
  const double u[3] = {up.x(), up.y(), up.z()};
  vp_plane out{};
  detail::check(vp_refine_planes(&f, u, 1, device, &out));
  return detail::from_c(out);
}

// ------------------------------------------------------------ polygonize
inline PlaneBasis plane_basis(const PlaneModel& plane) {  // polygonize.cpp:21-34
  const Vec3& n = plane.normal;
  int least = 0;
  for (int k = 1; k < 3; ++k)
    if (std::abs(n[k]) < std::abs(n[least])) least = k;
  Vec3 axis = Vec3::Zero();
  axis[least] = 1.0;
  PlaneBasis basis;
  basis.u = (axis - n.dot(axis) * n).normalized();
  basis.v = n.cross(basis.u);
  basis.origin = plane.offset * n;
  return basis;
}

inline std::vector<Vec2> project_to_plane(const PlaneModel& plane, std::span<const Vec3> points) {
  const PlaneBasis basis = plane_basis(plane);
  std::vector<Vec2> out(points.size());
  for (size_t i = 0; i < points.size(); ++i) {
    const Vec3 d = points[i] - basis.origin;
    out[i] = Vec2(d.dot(basis.u), d.dot(basis.v));
  }
  return out;
}

inline Vec3 lift_from_plane(const PlaneBasis& basis, const Vec2& q) {
  return basis.origin + q.x() * basis.u + q.y() * basis.v;
}

inline double polygon_area(std::span<const Vec2> ring) {  // polygonize.cpp:146-154
  double twice = 0.0;
  for (size_t i = 0; i < ring.size(); ++i) {
    const Vec2& a = ring[i];
    const Vec2& b = ring[(i + 1) % ring.size()];
    twice += a.x() * b.y() - b.x() * a.y();
  }
  return 0.5 * twice;
}

namespace detail {
inline std::vector<double> flat2(std::span<const Vec2> pts) {
  std::vector<double> a(2 * pts.size());
  for (size_t i = 0; i < pts.size(); ++i) {
    a[2 * i] = pts[i].x();
    a[2 * i + 1] = pts[i].y();
  }
  return a;
}
inline std::vector<Vec2> take2(double* out, uint64_t m) {
  std::vector<Vec2> v(m);
  for (uint64_t i = 0; i < m; ++i) v[i] = Vec2(out[2 * i], out[2 * i + 1]);
  vp_free(out);
  return v;
}
}  // namespace detail

/// hull_filter (polygonize.cpp:50-114) on the device: survivors in input order.
inline std::vector<Vec2> hull_filter(std::span<const Vec2> points, int directions = 16, int device = 0) {
  const std::vector<double> a = detail::flat2(points);
  double* out = nullptr;
  uint64_t m = 0;
  detail::check(vp_hull_filter(a.data(), points.size(), directions, device, &out, &m));
  return detail::take2(out, m);
}

/// monotone_chain (polygonize.cpp:116-139) on the device: strict CCW hull from
/// the lexicographic minimum, empty when all points are collinear.
inline std::vector<Vec2> monotone_chain(std::span<const Vec2> points, int device = 0) {
  const std::vector<double> a = detail::flat2(points);
  double* out = nullptr;
  uint64_t m = 0;
  detail::check(vp_monotone_chain(a.data(), points.size(), device, &out, &m));
  return detail::take2(out, m);
}

/// convex_hull (polygonize.cpp:141-144): hull_filter then monotone_chain.
inline std::vector<Vec2> convex_hull(std::span<const Vec2> points, int directions = 16, int device = 0) {
  const std::vector<double> a = detail::flat2(points);
  double* out = nullptr;
  uint64_t m = 0;
  detail::check(vp_convex_hull(a.data(), points.size(), directions, device, &out, &m));
  return detail::take2(out, m);
}

inline bool point_in_convex(std::span<const Vec2> ring, const Vec2& p, double slack = 0.0) {
  for (size_t i = 0; i < ring.size(); ++i) {
    const Vec2& a = ring[i];
    const Vec2& b = ring[(i + 1) % ring.size()];
    const double len = (b - a).norm();
    const double c = (b.x() - a.x()) * (p.y() - a.y()) - (b.y() - a.y()) * (p.x() - a.x());
    if (c < -slack * (len > 0.0 ? len : 1.0)) return false;
  }
  return true;
}

/// make_polygon (polygonize.cpp:166-182) for many planes at once on the device;
/// entries that are nullopt in the reference come back empty.
inline std::vector<std::optional<PlanePolygon>> make_polygons(
    const std::vector<PlaneModel>& planes, const std::vector<std::vector<Vec3>>& inliers,
    int filter_directions = 16, int device = 0) {
  std::vector<vp_plane> pl;
  std::vector<uint64_t> offs{0};
  std::vector<double> pts;
  for (size_t i = 0; i < planes.size(); ++i) {
    pl.push_back(detail::to_c(planes[i]));
    for (const Vec3& p : inliers[i]) pts.insert(pts.end(), {p.x(), p.y(), p.z()});
    offs.push_back(offs.back() + inliers[i].size());
  }
  vp_polygons_t* out = nullptr;
  detail::check(vp_make_polygons(planes.size(), pl.data(), offs.data(), pts.data(),
                                 filter_directions, device, &out));
  std::vector<std::optional<PlanePolygon>> res;
  for (PlanePolygon& p : detail::take(out, true)) {
    if (p.vertices3d.empty()) res.emplace_back(std::nullopt);
    else res.emplace_back(std::move(p));
  }
  return res;
}

inline std::optional<PlanePolygon> make_polygon(const PlaneModel& plane,
                                                std::span<const Vec3> inliers,
                                                int filter_directions = 16) {
  return make_polygons({plane}, {std::vector<Vec3>(inliers.begin(), inliers.end())},
                       filter_directions)[0];
}

// -------------------------------------------------------------- pipeline
/// Everything voxel_frame_polygons reads from PipelineConfig.
struct SegmentConfig {
  SegmentationParams segmentation;
  RansacParams ransac;
  bool refine = true;
  double min_polygon_area = 0.002;
  bool refine_exact = false;  // true: refine sums bit-identical to the reference
};

namespace detail {
inline vp_pipeline_params to_c(const SegmentConfig& c) {
  vp_pipeline_params p{};
  p.seg = to_c(c.segmentation);
  p.ransac = to_c(c.ransac);
  p.refine = c.refine ? 1 : 0;
  p.min_polygon_area = c.min_polygon_area;
  p.refine_exact = c.refine_exact ? 1 : 0;
  return p;
}
}  // namespace detail

/// segment(): voxel_frame_polygons (pipeline.cpp:43-85) on the device grid.
inline std::vector<PlanePolygon> segment(VoxelGrid& grid, const SegmentConfig& config) {
  const vp_pipeline_params p = detail::to_c(config);
  vp_polygons_t* out = nullptr;
  detail::check(vp_segment(grid.handle(), &p, &out, nullptr));
  return detail::take(out);
}

/// run_frames state (pipeline.cpp:157-245): frame() is one iteration of its
/// loop (clear_rays, integrate_frame, recenter on a global-cell change,
/// voxel_frame_polygons), returning the frame's polygons.
class Pipeline {
 public:
  Pipeline(double resolution, const Vec3i& extent, const Vec3& start_center,
           const SegmentConfig& config, int device = 0)
      : resolution_(resolution), extent_(extent) {
    const int32_t e[3] = {extent.x(), extent.y(), extent.z()};
    const double c[3] = {start_center.x(), start_center.y(), start_center.z()};
    const vp_pipeline_params p = detail::to_c(config);
    detail::check(vp_pipeline_create(resolution, e, c, &p, device, &pl_));
  }
  ~Pipeline() { vp_pipeline_destroy(pl_); }
  Pipeline(const Pipeline&) = delete;
  Pipeline& operator=(const Pipeline&) = delete;

  std::vector<PlanePolygon> frame(const SensorFrame& f, vp_frame_timing* timing = nullptr) {
    double R[9], t[3];
    detail::pose_arrays(f.pose, R, t);
    vp_polygons_t* out = nullptr;
    detail::check(vp_pipeline_frame(pl_, detail::frame_xyz(f), f.points.size(), R, t, &out, timing));
    return detail::take(out);
  }
  VoxelGrid grid() { return VoxelGrid(vp_pipeline_grid(pl_), resolution_, extent_); }

 private:
  double resolution_;
  Vec3i extent_;
  vp_pipeline* pl_ = nullptr;
};

// ------------------------------------------------------------- frame / polygon I/O
/// read_frames_binary (frame_io.cpp:127-152): VXPF stream.
inline std::vector<SensorFrame> read_frames_binary(const std::string& path) {
  std::ifstream is(path, std::ios::binary);
  if (!is) throw MissingInputError("frame stream: cannot open: " + path);
  auto u32 = [&]() {
    unsigned char b[4];
    is.read(reinterpret_cast<char*>(b), 4);
    if (!is) throw std::runtime_error("frame stream: truncated file");
    return static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[1]) << 8) |
           (static_cast<uint32_t>(b[2]) << 16) | (static_cast<uint32_t>(b[3]) << 24);
  };
  auto f32 = [&]() {
    const uint32_t u = u32();
    float v;
    std::memcpy(&v, &u, 4);
    return v;
  };
  char magic[4];
  is.read(magic, 4);
  if (!is || std::string(magic, 4) != "VXPF") throw std::runtime_error("frame stream: bad magic in " + path);
  if (u32() != 1) throw std::runtime_error("frame stream: unsupported version");
  std::vector<SensorFrame> frames;
  while (is.peek() != EOF) {
    SensorFrame f;
    const uint32_t n = u32();
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) f.pose.rotation(r, c) = f32();
      f.pose.translation[r] = f32();
    }
    f.points.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
      const float x = f32(), y = f32(), z = f32();
      f.points[i] = Vec3f(x, y, z);
    }
    f.timestamp = static_cast<double>(frames.size());
    frames.push_back(std::move(f));
  }
  return frames;
}

/// quantize_pose (frame_io.cpp:64-72): the pose through the file format's f32.
inline Pose quantize_pose(const Pose& pose) {
  Pose q;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) q.rotation(r, c) = static_cast<double>(static_cast<float>(pose.rotation(r, c)));
    q.translation[r] = static_cast<double>(static_cast<float>(pose.translation[r]));
  }
  return q;
}

/// write_frames_binary (frame_io.cpp:74-89): a VXPF stream.
inline void write_frames_binary(const std::string& path, const std::vector<SensorFrame>& frames) {
  std::vector<const float*> xyz(frames.size());
  std::vector<uint64_t> n(frames.size());
  std::vector<double> R(9 * frames.size()), t(3 * frames.size());
  for (size_t k = 0; k < frames.size(); ++k) {
    xyz[k] = detail::frame_xyz(frames[k]);
    n[k] = frames[k].points.size();
    detail::pose_arrays(frames[k].pose, &R[9 * k], &t[3 * k]);
  }
  const int rc = vp_write_frames_binary(path.c_str(), frames.size(), xyz.data(), n.data(), R.data(), t.data());
  if (rc != VP_OK) throw OutputError(vp_last_error());
}

/// write_frames_text / read_frames_text (frame_io.cpp:118-196): the
/// hand-written fixture format ("frame n", "pose" + 12 numbers, n "x y z").
inline void write_frames_text(const std::string& path, const std::vector<SensorFrame>& frames) {
  std::ofstream os(path);
  if (!os) throw OutputError("frame stream: cannot open for write: " + path);
  char buf[96];
  for (const SensorFrame& f : frames) {
    os << "frame " << f.points.size() << '\n' << "pose";
    for (int r = 0; r < 3; ++r) {
      std::snprintf(buf, sizeof buf, " %.9g %.9g %.9g %.9g", f.pose.rotation(r, 0), f.pose.rotation(r, 1),
                    f.pose.rotation(r, 2), f.pose.translation[r]);
      os << buf;
    }
    os << '\n';
    for (const Vec3f& p : f.points) {
      std::snprintf(buf, sizeof buf, "%.9g %.9g %.9g\n", static_cast<double>(p.x()), static_cast<double>(p.y()),
                    static_cast<double>(p.z()));
      os << buf;
    }
  }
  if (!os) throw OutputError("frame stream: write failed: " + path);
}

namespace detail {
inline bool content_line(std::istream& is, std::string& line) {
  while (std::getline(is, line)) {
    const size_t i = line.find_first_not_of(" \t\r");
    if (i == std::string::npos || line[i] == '#') continue;
    return true;
  }
  return false;
}
}  // namespace detail

inline std::vector<SensorFrame> read_frames_text(const std::string& path) {
  std::ifstream is(path);
  if (!is) throw MissingInputError("frame stream: cannot open: " + path);
  std::vector<SensorFrame> frames;
  std::string line;
  while (detail::content_line(is, line)) {
    std::istringstream h(line);
    std::string kw;
    size_t n = 0;
    h >> kw >> n;
    if (kw != "frame" || !h) throw std::runtime_error("frame stream: expected 'frame <count>' in " + path);
    if (!detail::content_line(is, line)) throw std::runtime_error("frame stream: missing pose line in " + path);
    std::istringstream ps(line);
    ps >> kw;
    if (kw != "pose") throw std::runtime_error("frame stream: expected 'pose' in " + path);
    SensorFrame f;
    for (int r = 0; r < 3; ++r) {
      double v[4];
      ps >> v[0] >> v[1] >> v[2] >> v[3];
      for (int c = 0; c < 3; ++c) f.pose.rotation(r, c) = v[c];
      f.pose.translation[r] = v[3];
    }
    if (!ps) throw std::runtime_error("frame stream: malformed pose in " + path);
    f.points.resize(n);
    for (size_t i = 0; i < n; ++i) {
      if (!detail::content_line(is, line))
        throw std::runtime_error("frame stream: truncated point list in " + path);
      std::istringstream vs(line);
      float x, y, z;
      vs >> x >> y >> z;
      if (!vs) throw std::runtime_error("frame stream: malformed point in " + path);
      f.points[i] = Vec3f(x, y, z);
    }
    f.timestamp = static_cast<double>(frames.size());
    frames.push_back(std::move(f));
  }
  return frames;
}

/// write_polygons (polygon_io.cpp:30-47): the golden-file format.
inline void write_polygons(const std::string& path, const std::vector<PlanePolygon>& polygons) {
  std::ofstream os(path);
  if (!os) throw OutputError("polygons: cannot open for write: " + path);
  auto fmt = [](double v) {
    char buf[48];
    std::snprintf(buf, sizeof buf, "%.9g", v);
    return std::string(buf);
  };
  os << "# voxplane polygons v1\n";
  for (const PlanePolygon& p : polygons) {
    os << "polygon\n";
    os << "normal " << fmt(p.plane.normal.x()) << ' ' << fmt(p.plane.normal.y()) << ' '
       << fmt(p.plane.normal.z()) << '\n';
    os << "offset " << fmt(p.plane.offset) << '\n';
    os << "vertices " << p.vertices3d.size() << '\n';
    for (const Vec3& v : p.vertices3d) os << fmt(v.x()) << ' ' << fmt(v.y()) << ' ' << fmt(v.z()) << '\n';
    os << "area " << fmt(p.area) << '\n';
    os << "label " << p.plane.cluster_label << '\n';
    os << "inliers " << p.plane.inlier_count << '\n';
  }
  if (!os) throw OutputError("polygons: write failed: " + path);
}

/// read_polygons (polygon_io.cpp:50-127): the golden-file format back; the
/// in-plane ring is recomputed from the 3-D vertices with plane_basis.
inline std::vector<PlanePolygon> read_polygons(const std::string& path) {
  std::ifstream is(path);
  if (!is) throw MissingInputError("polygons: cannot open: " + path);
  std::vector<PlanePolygon> out;
  std::string line;
  auto field = [&](const char* name) {
    if (!detail::content_line(is, line))
      throw std::runtime_error(std::string("polygons: missing '") + name + "' in " + path);
    std::istringstream ss(line);
    std::string kw;
    ss >> kw;
    if (kw != name)
      throw std::runtime_error(std::string("polygons: expected '") + name + "', got '" + kw + "' in " + path);
    return ss;
  };
  while (detail::content_line(is, line)) {
    std::istringstream h(line);
    std::string kw;
    h >> kw;
    if (kw != "polygon") throw std::runtime_error("polygons: expected 'polygon' in " + path);
    PlanePolygon p;
    {
      auto ss = field("normal");
      ss >> p.plane.normal.x() >> p.plane.normal.y() >> p.plane.normal.z();
      if (!ss) throw std::runtime_error("polygons: malformed normal in " + path);
    }
    {
      auto ss = field("offset");
      ss >> p.plane.offset;
      if (!ss) throw std::runtime_error("polygons: malformed offset in " + path);
    }
    size_t k = 0;
    {
      auto ss = field("vertices");
      ss >> k;
      if (!ss) throw std::runtime_error("polygons: malformed vertex count in " + path);
    }
    p.vertices3d.resize(k);
    for (size_t i = 0; i < k; ++i) {
      if (!detail::content_line(is, line)) throw std::runtime_error("polygons: truncated vertex list in " + path);
      std::istringstream vs(line);
      vs >> p.vertices3d[i].x() >> p.vertices3d[i].y() >> p.vertices3d[i].z();
      if (!vs) throw std::runtime_error("polygons: malformed vertex in " + path);
    }
    field("area") >> p.area;
    field("label") >> p.plane.cluster_label;
    field("inliers") >> p.plane.inlier_count;
    const PlaneBasis b = plane_basis(p.plane);
    for (const Vec3& v : p.vertices3d) {
      const Vec3 d = v - b.origin;
      p.vertices2d.emplace_back(d.dot(b.u), d.dot(b.v));
    }
    out.push_back(std::move(p));
  }
  return out;
}

}  // namespace voxplane
