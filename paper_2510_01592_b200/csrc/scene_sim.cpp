// Synthetic frame source (include/voxplane_scene.h): a host restatement of
// /root/reference/proj/core/src/scene_sim.cpp and the default trajectories of
// pipeline.cpp:89-155, so benchmarks and tests can produce the reference's
// exact input frames without the reference. Compiled with -ffp-contract=off;
// vector expressions follow the Eigen 3.4 evaluation order used throughout
// (3-term dots (a0b0 + a1b1) + a2b2, 3x3*vec3 row 2 as r0v0 + (r1v1 + r2v2)).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "voxplane_b200.h"
#include "voxplane_scene.h"

namespace {

constexpr double kPi = 3.14159265358979323846;  // glibc M_PI
constexpr double kDegToRad = 0.017453292519943295769237;
constexpr double kRayEps = 1e-9;

struct V3 {
  double x, y, z;
  double operator[](int k) const { return k == 0 ? x : (k == 1 ? y : z); }
};
V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
V3 scl(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
double dot(V3 a, V3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
V3 cross(V3 a, V3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
V3 normalized(V3 a) {
  const double z = dot(a, a);
  return z > 0.0 ? V3{a.x / std::sqrt(z), a.y / std::sqrt(z), a.z / std::sqrt(z)} : a;
}
double norm(V3 a) { return std::sqrt(dot(a, a)); }

struct M3 {
  double m[9];  // row-major
};
V3 col(const M3& r, int c) { return {r.m[c], r.m[3 + c], r.m[6 + c]}; }
V3 matvec(const M3& r, V3 p) {
  return {(r.m[0] * p.x + r.m[1] * p.y) + r.m[2] * p.z, (r.m[3] * p.x + r.m[4] * p.y) + r.m[5] * p.z,
          r.m[6] * p.x + (r.m[7] * p.y + r.m[8] * p.z)};
}

bool valid_rotation(const M3& R) {
  double t[3][3], p[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t[i][j] = R.m[3 * j + i];
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i)
      p[i][j] = i < 2 ? (t[i][0] * R.m[j] + t[i][1] * R.m[3 + j]) + t[i][2] * R.m[6 + j]
                      : t[i][0] * R.m[j] + (t[i][1] * R.m[3 + j] + t[i][2] * R.m[6 + j]);
  double mx = 0.0;
  bool first = true;
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i) {
      double v = p[i][j] - (i == j ? 1.0 : 0.0);
      v = v < 0.0 ? -v : v;
      if (first || mx < v) mx = v;
      first = false;
    }
  if (mx > 1e-6) return false;
  auto m = [&](int r, int c) { return R.m[3 * r + c]; };
  auto h = [&](int a, int b, int c) { return m(0, a) * (m(1, b) * m(2, c) - m(1, c) * m(2, b)); };
  return std::abs((h(0, 1, 2) - h(1, 0, 2) + h(2, 0, 1)) - 1.0) <= 1e-6;
}

// CounterRng (rng.hpp:13-64)
struct Rng {
  uint64_t s;
  double cached = 0.0;
  bool has = false;
  static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  Rng(uint64_t seed, uint64_t k1, uint64_t k2) {
    s = mix(seed + 0x9e3779b97f4a7c15ULL);
    s = mix(s ^ mix(k1 + 0xbf58476d1ce4e5b9ULL));
    s = mix(s ^ mix(k2 + 0x94d049bb133111ebULL));
  }
  uint64_t next() {
    s += 0x9e3779b97f4a7c15ULL;
    return mix(s);
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double normal() {
    if (has) {
      has = false;
      return cached;
    }
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    cached = r * std::sin(a);
    has = true;
    return r * std::cos(a);
  }
};

// scene_sim.cpp:121-157
double cast_ray(const vp_box* boxes, size_t nb, const vp_rect* rects, size_t nr, V3 o, V3 d,
                double max_range) {
  double best = std::numeric_limits<double>::infinity();
  for (size_t b = 0; b < nb; ++b) {
    double t0 = 0.0, t1 = std::numeric_limits<double>::infinity();
    bool miss = false;
    for (int k = 0; k < 3 && !miss; ++k) {
      if (d[k] == 0.0) {
        if (o[k] < boxes[b].min[k] || o[k] > boxes[b].max[k]) miss = true;
        continue;
      }
      double ta = (boxes[b].min[k] - o[k]) / d[k];
      double tb = (boxes[b].max[k] - o[k]) / d[k];
      if (ta > tb) std::swap(ta, tb);
      t0 = std::max(t0, ta);
      t1 = std::min(t1, tb);
      if (t0 > t1) miss = true;
    }
    if (miss) continue;
    const double t = t0 > kRayEps ? t0 : t1;
    if (t > kRayEps && t < best) best = t;
  }
  for (size_t i = 0; i < nr; ++i) {
    M3 R;
    std::memcpy(R.m, rects[i].R, sizeof R.m);
    const V3 tr{rects[i].t[0], rects[i].t[1], rects[i].t[2]};
    const V3 n = col(R, 2);
    const double denom = dot(n, d);
    if (std::abs(denom) < 1e-12) continue;
    const double t = dot(n, sub(tr, o)) / denom;
    if (t <= kRayEps || t >= best) continue;
    const V3 q = sub(add(o, scl(t, d)), tr);
    if (std::abs(dot(q, col(R, 0))) <= rects[i].half_u && std::abs(dot(q, col(R, 1))) <= rects[i].half_v)
      best = t;
  }
  return best <= max_range ? best : std::numeric_limits<double>::infinity();
}

// scene_sim.cpp:238-250
M3 look_pose(V3 forward) {
  const V3 f = normalized(forward);
  V3 left = cross(V3{0.0, 0.0, 1.0}, f);
  if (norm(left) < 1e-6) left = cross(V3{1.0, 0.0, 0.0}, f);
  left = normalized(left);
  const V3 up = cross(f, left);
  M3 R;
  R.m[0] = f.x; R.m[3] = f.y; R.m[6] = f.z;
  R.m[1] = left.x; R.m[4] = left.y; R.m[7] = left.z;
  R.m[2] = up.x; R.m[5] = up.y; R.m[8] = up.z;
  return R;
}

struct Spec {
  int kind = 0;  // 0 Straight, 1 Orbit, 2 StairAscent
  double duration = 5.0, rate = 20.0;
  V3 start{-1.0, 0.0, 0.5}, end{0.0, 0.0, 0.5};
  double pitch0 = -25.0, pitch1 = -25.0;
  V3 center{0.0, 0.0, 0.0};
  double radius = 0.5, height = 0.5, start_angle = 0.0, revolutions = 1.0;
  double rise = 0.17, run = 0.29, x0 = 0.0;
};

void put_pose(std::vector<double>& out, const M3& R, V3 t) {
  out.insert(out.end(), R.m, R.m + 9);
  out.push_back(t.x);
  out.push_back(t.y);
  out.push_back(t.z);
}

// scene_sim.cpp:252-298
std::vector<double> scripted(const Spec& s) {
  const size_t n = static_cast<size_t>(std::floor(s.duration * s.rate + 1e-9));
  std::vector<double> out;
  for (size_t i = 0; i < n; ++i) {
    const double u = n > 1 ? static_cast<double>(i) / static_cast<double>(n - 1) : 0.0;
    if (s.kind == 0) {
      const V3 pos = add(s.start, scl(u, sub(s.end, s.start)));
      const double pitch = (s.pitch0 + u * (s.pitch1 - s.pitch0)) * kDegToRad;
      V3 dir = sub(s.end, s.start);
      dir.z = 0.0;
      if (norm(dir) < 1e-9) dir = V3{1.0, 0.0, 0.0};
      dir = normalized(dir);
      const V3 fwd{dir.x * std::cos(pitch), dir.y * std::cos(pitch), std::sin(pitch)};
      put_pose(out, look_pose(fwd), pos);
    } else if (s.kind == 1) {
      const double a = s.start_angle * kDegToRad + 2.0 * kPi * s.revolutions * u;
      const V3 pos = add(s.center, V3{s.radius * std::cos(a), s.radius * std::sin(a), s.height});
      put_pose(out, look_pose(sub(s.center, pos)), pos);
    } else {
      const V3 flat = add(s.start, scl(u, sub(s.end, s.start)));
      const double climb = std::max(0.0, (flat.x - s.x0) / s.run) * s.rise;
      const V3 pos = add(flat, V3{0.0, 0.0, climb});
      const double pitch = (s.pitch0 + u * (s.pitch1 - s.pitch0)) * kDegToRad;
      const V3 fwd{std::cos(pitch), 0.0, std::sin(pitch)};
      put_pose(out, look_pose(fwd), pos);
    }
  }
  return out;
}

// SceneParams defaults (scene_sim.hpp:35-50)
struct SceneParams {
  double stair_rise = 0.17, stair_run = 0.29, stair_width = 1.2, approach_length = 1.2;
  double floor_size = 0.88, stage_size = 0.40, stage_height = 0.20;
  double overhang_floor_x = 1.4, overhang_floor_y = 0.9, overhang_clearance = 0.5,
         overhang_depth = 0.4;
  V3 obstacle_size{0.07, 0.10, 0.08};
  V3 obstacle_center_xy{0.3, 0.0, 0.0};
  double obstacle_floor_size = 1.2;
};

vp_rect hrect(V3 c, double hx, double hy) {
  vp_rect r{};
  r.R[0] = r.R[4] = r.R[8] = 1.0;
  r.t[0] = c.x;
  r.t[1] = c.y;
  r.t[2] = c.z;
  r.half_u = hx;
  r.half_v = hy;
  return r;
}

thread_local std::string t_err;

}  // namespace

extern "C" {

int vp_stock_scene(int kind, vp_box* boxes, size_t* nb, vp_rect* rects, size_t* nr) {
  const SceneParams p;
  *nb = 0;
  *nr = 0;
  switch (kind) {
    case 0: {  // Stair5 (scene_sim.cpp:46-65)
      const double w = 0.5 * p.stair_width;
      rects[(*nr)++] = hrect(V3{-0.5 * p.approach_length, 0, 0}, 0.5 * p.approach_length, w);
      for (int k = 0; k < 5; ++k) {
        const double x0 = k * p.stair_run, x1 = (k + 1) * p.stair_run, z1 = (k + 1) * p.stair_rise;
        boxes[(*nb)++] = vp_box{{x0, -w, 0.0}, {x1, w, z1}};
      }
      return 0;
    }
    case 1: {  // SingleStage (:66-80)
      const double f = 0.5 * p.floor_size;
      rects[(*nr)++] = hrect(V3{0, 0, 0}, f, f);
      const double s = 0.5 * p.stage_size, cx = f - s;
      rects[(*nr)++] = hrect(V3{cx, 0, p.stage_height}, s, f);
      return 0;
    }
    case 2: {  // Overhang (:81-95)
      const double fx = 0.5 * p.overhang_floor_x, fy = 0.5 * p.overhang_floor_y;
      rects[(*nr)++] = hrect(V3{0, 0, 0}, fx, fy);
      const double ox = 0.5 * p.overhang_depth, cx = fx - ox;
      rects[(*nr)++] = hrect(V3{cx, 0, p.overhang_clearance}, ox, fy);
      return 0;
    }
    case 3: {  // SmallObstacle (:96-111)
      const double f = 0.5 * p.obstacle_floor_size;
      rects[(*nr)++] = hrect(V3{0, 0, 0}, f, f);
      const V3 half = scl(0.5, p.obstacle_size);
      const V3 c{p.obstacle_center_xy.x, p.obstacle_center_xy.y, 0.0};
      boxes[(*nb)++] = vp_box{{c.x - half.x, c.y - half.y, c.z - 0.0},
                              {c.x + half.x, c.y + half.y, c.z + p.obstacle_size.z}};
      return 0;
    }
  }
  return VP_EINVAL;
}

int vp_scripted_trajectory(int kind, const double sp[21], double* poses, int cap) {
  Spec s;
  s.kind = kind;
  s.duration = sp[0];
  s.rate = sp[1];
  s.start = V3{sp[2], sp[3], sp[4]};
  s.end = V3{sp[5], sp[6], sp[7]};
  s.pitch0 = sp[8];
  s.pitch1 = sp[9];
  s.center = V3{sp[10], sp[11], sp[12]};
  s.radius = sp[13];
  s.height = sp[14];
  s.start_angle = sp[15];
  s.revolutions = sp[16];
  s.rise = sp[17];
  s.run = sp[18];
  s.x0 = sp[19];
  const auto v = scripted(s);
  const int n = static_cast<int>(v.size() / 12);
  std::memcpy(poses, v.data(), sizeof(double) * 12 * std::min(n, cap));
  return n;
}

int vp_default_trajectory(int kind, int frames, double rate_hz, double* poses) {
  const SceneParams p;
  const double rate = rate_hz > 0.0 ? rate_hz : 20.0;
  Spec s;
  s.rate = rate;
  std::vector<double> v;
  switch (kind) {
    case 1: {  // SingleStage (pipeline.cpp:96-121)
      const int orbit_frames = (frames * 3) / 4;
      const int over_frames = frames - orbit_frames;
      s.kind = 1;
      s.center = V3{0, 0, 0};
      s.radius = 0.5 * p.floor_size + 0.10;
      s.height = 0.5;
      s.revolutions = 1.0;
      s.duration = orbit_frames / rate;
      v = scripted(s);
      const double cx = 0.5 * (p.floor_size - p.stage_size);
      Spec o;
      o.kind = 0;
      o.rate = rate;
      o.duration = over_frames / rate;
      o.start = V3{s.radius, 0.0, s.height};
      o.end = V3{cx, 0.0, 0.9};
      o.pitch0 = -45.0;
      o.pitch1 = -75.0;
      const auto w = scripted(o);
      v.insert(v.end(), w.begin(), w.end());
      while (static_cast<int>(v.size() / 12) > frames) v.resize(v.size() - 12);
      break;
    }
    case 2:  // Overhang (:122-131)
      s.kind = 0;
      s.duration = frames / rate;
      s.start = V3{-0.6, 0.0, 0.45};
      s.end = V3{0.1, 0.0, 0.45};
      s.pitch0 = -35.0;
      s.pitch1 = 10.0;
      v = scripted(s);
      break;
    case 0:  // Stair5 (:132-143)
      s.kind = 2;
      s.duration = frames / rate;
      s.start = V3{-0.9, 0.0, 0.55};
      s.end = V3{2.5 * p.stair_run, 0.0, 0.55};
      s.pitch0 = -30.0;
      s.pitch1 = -30.0;
      s.rise = p.stair_rise;
      s.run = p.stair_run;
      s.x0 = 0.0;
      v = scripted(s);
      break;
    case 3:  // SmallObstacle (:144-152)
      s.kind = 0;
      s.duration = frames / rate;
      s.start = V3{-0.55, 0.0, 0.5};
      s.end = V3{-0.05, 0.0, 0.5};
      s.pitch0 = -40.0;
      s.pitch1 = -45.0;
      v = scripted(s);
      break;
    default:
      return -1;
  }
  std::memcpy(poses, v.data(), v.size() * sizeof(double));
  return static_cast<int>(v.size() / 12);
}

int vp_scene_truth(int kind, double* planes, double* corners, size_t* n) {
  // build_scene's add_truth regions (scene_sim.cpp:23-30, 43-114): plane_through
  // (orient_up(normal.normalized()), offset = n . first corner) + 4 corners each
  const SceneParams p;
  *n = 0;
  auto add_truth = [&](V3 nrm, std::initializer_list<V3> cs) {
    V3 u = normalized(nrm);
    const double d = dot(u, V3{0, 0, 1});  // orient_up (types.hpp:43-52)
    const double flip = d < 0.0 ? -1.0 : 1.0;
    if (d == 0.0) {
      const double c3[3] = {u.x, u.y, u.z};
      for (int k = 0; k < 3; ++k) {
        if (c3[k] > 0.0) break;
        if (c3[k] < 0.0) {
          u = scl(-1.0, u);
          break;
        }
      }
    } else if (flip < 0.0) {
      u = V3{-u.x, -u.y, -u.z};
    }
    const V3 c0 = *cs.begin();
    double* pl = planes + 4 * *n;
    pl[0] = u.x;
    pl[1] = u.y;
    pl[2] = u.z;
    pl[3] = dot(u, c0);
    int k = 0;
    for (const V3& c : cs) {
      corners[12 * *n + 3 * k] = c.x;
      corners[12 * *n + 3 * k + 1] = c.y;
      corners[12 * *n + 3 * k + 2] = c.z;
      ++k;
    }
    ++*n;
  };
  const V3 ux{1, 0, 0}, uz{0, 0, 1}, mx{-1, 0, 0};
  switch (kind) {
    case 0: {  // Stair5
      const double w = 0.5 * p.stair_width;
      add_truth(uz, {{-p.approach_length, -w, 0}, {0, -w, 0}, {0, w, 0}, {-p.approach_length, w, 0}});
      for (int k = 0; k < 5; ++k) {
        const double x0 = k * p.stair_run, x1 = (k + 1) * p.stair_run, z1 = (k + 1) * p.stair_rise;
        add_truth(uz, {{x0, -w, z1}, {x1, -w, z1}, {x1, w, z1}, {x0, w, z1}});
        const double z0 = k * p.stair_rise;
        add_truth(mx, {{x0, -w, z0}, {x0, w, z0}, {x0, w, z1}, {x0, -w, z1}});
      }
      return 0;
    }
    case 1: {  // SingleStage
      const double f = 0.5 * p.floor_size;
      add_truth(uz, {{-f, -f, 0}, {f, -f, 0}, {f, f, 0}, {-f, f, 0}});
      const double s = 0.5 * p.stage_size, cx = f - s, h = p.stage_height;
      add_truth(uz, {{cx - s, -f, h}, {cx + s, -f, h}, {cx + s, f, h}, {cx - s, f, h}});
      return 0;
    }
    case 2: {  // Overhang
      const double fx = 0.5 * p.overhang_floor_x, fy = 0.5 * p.overhang_floor_y;
      add_truth(uz, {{-fx, -fy, 0}, {fx, -fy, 0}, {fx, fy, 0}, {-fx, fy, 0}});
      const double ox = 0.5 * p.overhang_depth, oy = fy, cx = fx - ox, h = p.overhang_clearance;
      add_truth(uz, {{cx - ox, -oy, h}, {cx + ox, -oy, h}, {cx + ox, oy, h}, {cx - ox, oy, h}});
      return 0;
    }
    case 3: {  // SmallObstacle
      const double f = 0.5 * p.obstacle_floor_size;
      add_truth(uz, {{-f, -f, 0}, {f, -f, 0}, {f, f, 0}, {-f, f, 0}});
      const V3 half = scl(0.5, p.obstacle_size);
      const V3 c{p.obstacle_center_xy.x, p.obstacle_center_xy.y, 0.0};
      const double z = p.obstacle_size.z;
      add_truth(uz, {{c.x - half.x, c.y - half.y, z}, {c.x + half.x, c.y - half.y, z},
                     {c.x + half.x, c.y + half.y, z}, {c.x - half.x, c.y + half.y, z}});
      return 0;
    }
    default:
      (void)ux;
      return -1;
  }
}

int vp_quantize_pose(const double Rin[9], const double tin[3], double qR[9], double qt[3]) {
  M3 R;  // quantize_pose (frame_io.cpp:64-72)
  for (int i = 0; i < 9; ++i) R.m[i] = static_cast<double>(static_cast<float>(Rin[i]));
  if (!valid_rotation(R)) return VP_EINVAL;  // render_frame (scene_sim.cpp:188-190)
  std::memcpy(qR, R.m, sizeof R.m);
  for (int k = 0; k < 3; ++k) qt[k] = static_cast<double>(static_cast<float>(tin[k]));
  return VP_OK;
}

int vp_spherical_pattern(int n, float* out) {  // scene_sim.cpp:174-184
  const double golden = kPi * (3.0 - std::sqrt(5.0));
  for (int i = 0; i < n; ++i) {
    const double z = 1.0 - 2.0 * (i + 0.5) / n;
    const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
    const double phi = golden * i;
    out[3 * i] = static_cast<float>(r * std::cos(phi));
    out[3 * i + 1] = static_cast<float>(r * std::sin(phi));
    out[3 * i + 2] = static_cast<float>(z);
  }
  return n;
}

int vp_rosette_pattern(int n, double cone_deg, double freq_ratio, float* out) {  // :161-172
  const double half = 0.5 * cone_deg * kDegToRad;
  for (int i = 0; i < n; ++i) {
    const double s = static_cast<double>(i) / std::max(1, n - 1);
    const double rho = half * std::abs(std::sin(2.0 * kPi * freq_ratio * s));
    const double phi = 2.0 * kPi * s * 197.0;
    out[3 * i] = static_cast<float>(std::cos(rho));
    out[3 * i + 1] = static_cast<float>(std::sin(rho) * std::cos(phi));
    out[3 * i + 2] = static_cast<float>(std::sin(rho) * std::sin(phi));
  }
  return n;
}

int vp_render_frame(const vp_box* boxes, size_t nb, const vp_rect* rects, size_t nr,
                    const vp_sensor* sensor, const double Rin[9], const double tin[3], uint64_t seed,
                    uint64_t frame_index, int threads, float** points, uint64_t* n_out, double qR[9],
                    double qt[3]) {
  *points = nullptr;
  *n_out = 0;
  M3 R;  // quantize_pose (frame_io.cpp:64-72)
  for (int i = 0; i < 9; ++i) R.m[i] = static_cast<double>(static_cast<float>(Rin[i]));
  const V3 t{static_cast<double>(static_cast<float>(tin[0])), static_cast<double>(static_cast<float>(tin[1])),
             static_cast<double>(static_cast<float>(tin[2]))};
  if (!valid_rotation(R)) return VP_EINVAL;
  std::memcpy(qR, R.m, sizeof R.m);
  qt[0] = t.x;
  qt[1] = t.y;
  qt[2] = t.z;
  const double tan_h = std::tan(0.5 * sensor->hfov_deg * kDegToRad);
  const double tan_v = std::tan(0.5 * sensor->vfov_deg * kDegToRad);
  const bool pinhole = sensor->kind == 0;
  const uint64_t rays = pinhole ? static_cast<uint64_t>(sensor->width) * sensor->height : sensor->npattern;
  std::vector<float> hits(3 * rays, std::numeric_limits<float>::quiet_NaN());
  auto work = [&](uint64_t b, uint64_t e) {
    for (uint64_t i = b; i < e; ++i) {
      V3 ds;
      if (!pinhole) {
        const float* q = sensor->pattern + 3 * i;
        ds = normalized(V3{static_cast<double>(q[0]), static_cast<double>(q[1]), static_cast<double>(q[2])});
      } else {
        const int r = static_cast<int>(i) / sensor->width;
        const int c = static_cast<int>(i) % sensor->width;
        const double u = sensor->width > 1 ? 2.0 * c / (sensor->width - 1) - 1.0 : 0.0;
        const double v = sensor->height > 1 ? 2.0 * r / (sensor->height - 1) - 1.0 : 0.0;
        ds = normalized(V3{1.0, -u * tan_h, -v * tan_v});
      }
      const V3 dw = matvec(R, ds);
      const double tt = cast_ray(boxes, nb, rects, nr, t, dw, sensor->max_range);
      if (!std::isfinite(tt)) continue;
      double range = tt;
      if (sensor->noise_sigma > 0.0) {
        Rng rng(seed, frame_index, i);
        const double ns = std::clamp(sensor->noise_sigma * rng.normal(), -3.0 * sensor->noise_sigma,
                                     3.0 * sensor->noise_sigma);
        range += ns;
      }
      hits[3 * i] = static_cast<float>(ds.x * range);
      hits[3 * i + 1] = static_cast<float>(ds.y * range);
      hits[3 * i + 2] = static_cast<float>(ds.z * range);
    }
  };
  unsigned nt = threads > 0 ? static_cast<unsigned>(threads) : std::max(1u, std::thread::hardware_concurrency());
  nt = static_cast<unsigned>(std::min<uint64_t>(nt, std::max<uint64_t>(1, rays / 4096)));
  if (nt <= 1) {
    work(0, rays);
  } else {
    std::vector<std::thread> pool;
    const uint64_t chunk = (rays + nt - 1) / nt;
    for (unsigned k = 0; k < nt; ++k) {
      const uint64_t b = k * chunk, e = std::min(rays, b + chunk);
      if (b < e) pool.emplace_back(work, b, e);
    }
    for (auto& th : pool) th.join();
  }
  uint64_t n = 0;
  for (uint64_t i = 0; i < rays; ++i)
    if (std::isfinite(hits[3 * i])) ++n;
  float* out = static_cast<float*>(std::malloc(12 * n + 1));
  uint64_t k = 0;
  for (uint64_t i = 0; i < rays; ++i)
    if (std::isfinite(hits[3 * i])) {
      out[3 * k] = hits[3 * i];
      out[3 * k + 1] = hits[3 * i + 1];
      out[3 * k + 2] = hits[3 * i + 2];
      ++k;
    }
  *points = out;
  *n_out = n;
  return VP_OK;
}

}  // extern "C"
