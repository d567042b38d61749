// Plane IoU scoring (metrics.cpp:19-160, the paper's
// Table I metric): every (truth, detected) pair is gated and projected into
// the truth plane on the host (acos gate with the host libm, plane_basis and
// the shoelace exactly as the reference), rasterised on the GPU -- one block
// per pair, point_in_convex per raster cell in the reference's FP64 order
// (-fmad=false), integer counts -- and greedily matched on the host.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "voxplane_b200.h"
#include "vp_kernels.cuh"

using namespace vp;

namespace {

constexpr double kRadToDeg = 57.295779513082320876798;
constexpr double kNormalGateDeg = 20.0;  // metrics.cpp:15

struct V2 {
  double x, y;
};

struct PairJob {
  uint32_t ring_d, nd, ring_t, nt;  // offsets / sizes into the ring array
  double lox, loy, res;
  int32_t nx, ny;
};

// point_in_convex(ring, p, slack = 0) (polygonize.cpp:156-164): with slack 0
// the test is cross2(a, b, p) < -0.0, i.e. cross2 < 0
__device__ __forceinline__ bool in_convex(const double2* ring, uint32_t n, double px, double py) {
  for (uint32_t i = 0; i < n; ++i) {
    const double2 a = ring[i];
    const double2 b = ring[i + 1 == n ? 0 : i + 1];
    const double c = (b.x - a.x) * (py - a.y) - (b.y - a.y) * (px - a.x);  // cross2 (polygonize.cpp:11-13)
    if (c < -0.0) return false;
  }
  return true;
}

// plane_iou raster loop (metrics.cpp:83-95): one block per pair
__global__ void k_iou_raster(const PairJob* __restrict__ jobs, const double2* __restrict__ rings,
                             unsigned long long* counts) {
  VP_GRID_WAIT();
  const PairJob j = jobs[blockIdx.x];
  const double2* rd = rings + j.ring_d;
  const double2* rt = rings + j.ring_t;
  unsigned long long inter = 0, uni = 0;
  const uint64_t cells = static_cast<uint64_t>(j.nx) * static_cast<uint64_t>(j.ny);
  for (uint64_t c = threadIdx.x; c < cells; c += blockDim.x) {
    const int ix = static_cast<int>(c / static_cast<uint64_t>(j.ny)), iy = static_cast<int>(c % j.ny);
    const double px = j.lox + (ix + 0.5) * j.res, py = j.loy + (iy + 0.5) * j.res;
    const bool a = in_convex(rd, j.nd, px, py);
    const bool b = in_convex(rt, j.nt, px, py);
    inter += (a && b) ? 1 : 0;
    uni += (a || b) ? 1 : 0;
  }
  // block reduction (deterministic integers)
  for (int o = 16; o > 0; o >>= 1) {
    inter += __shfl_down_sync(0xffffffffu, inter, o);
    uni += __shfl_down_sync(0xffffffffu, uni, o);
  }
  __shared__ unsigned long long si[32], su[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    si[wid] = inter;
    su[wid] = uni;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long a = 0, b = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      a += si[w];
      b += su[w];
    }
    counts[2 * blockIdx.x] = a;
    counts[2 * blockIdx.x + 1] = b;
  }
}

double dot3h(const double* a, const double* b) { return (a[0] * b[0] + a[1] * b[1]) + a[2] * b[2]; }

double area2(const std::vector<V2>& r) {  // polygon_area (polygonize.cpp:146-154)
  double twice = 0.0;
  for (size_t i = 0; i < r.size(); ++i) {
    const V2& a = r[i];
    const V2& b = r[(i + 1) % r.size()];
    twice += a.x * b.y - b.x * a.y;
  }
  return 0.5 * twice;
}

// project_pair (metrics.cpp:26-52)
bool project_pair(const vp_polygon& det, const vp_polygon& tru, std::vector<V2>& pd, std::vector<V2>& pt) {
  if (det.nverts < 3 || tru.nverts < 3) return false;
  const double dot = std::clamp(dot3h(det.plane.normal, tru.plane.normal), -1.0, 1.0);
  if (std::acos(dot) * kRadToDeg > kNormalGateDeg) return false;
  // plane_basis (polygonize.cpp:21-34)
  const double* n = tru.plane.normal;
  int least = 0;
  for (int k = 1; k < 3; ++k)
    if (std::abs(n[k]) < std::abs(n[least])) least = k;
  double axis[3] = {0.0, 0.0, 0.0};
  axis[least] = 1.0;
  const double na = dot3h(n, axis);
  double u[3] = {axis[0] - na * n[0], axis[1] - na * n[1], axis[2] - na * n[2]};
  const double z = dot3h(u, u);
  if (z > 0.0) {
    const double r = std::sqrt(z);
    for (double& c : u) c = c / r;
  }
  const double v[3] = {n[1] * u[2] - n[2] * u[1], n[2] * u[0] - n[0] * u[2], n[0] * u[1] - n[1] * u[0]};
  const double o[3] = {tru.plane.offset * n[0], tru.plane.offset * n[1], tru.plane.offset * n[2]};
  auto project = [&](const vp_polygon& p, std::vector<V2>& ring) {
    ring.resize(p.nverts);
    for (uint32_t i = 0; i < p.nverts; ++i) {
      const double d[3] = {p.v3d[3 * i] - o[0], p.v3d[3 * i + 1] - o[1], p.v3d[3 * i + 2] - o[2]};
      ring[i] = V2{dot3h(d, u), dot3h(d, v)};
    }
  };
  project(det, pd);
  project(tru, pt);
  return !(std::abs(area2(pd)) < 1e-12 || std::abs(area2(pt)) < 1e-12);
}

void ckc(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
  }
}

thread_local std::string g_iou_err;

}  // namespace

extern "C" {

int vp_match_planes(const vp_polygons_t* detected, const vp_polygons_t* truth, double raster_res, int device,
                    vp_iou_report* rep, vp_plane_match* matches) {
  try {
    const size_t nd = detected ? detected->count : 0, nt = truth ? truth->count : 0;
    std::memset(rep, 0, sizeof *rep);
    rep->truth_count = nt;
    rep->detected_count = nd;
    // projected pairs (host) -> raster jobs (device)
    std::vector<PairJob> jobs;
    std::vector<double2> rings;
    std::vector<std::pair<int, int>> job_pair;  // (truth, detected)
    std::vector<V2> pd, pt;
    for (size_t t = 0; t < nt; ++t)
      for (size_t d = 0; d < nd; ++d) {
        if (!project_pair(detected->polys[d], truth->polys[t], pd, pt)) continue;
        V2 lo = pt[0], hi = pt[0];
        for (const auto* ring : {&pd, &pt})
          for (const V2& p : *ring) {  // cwiseMin / cwiseMax
            lo = V2{std::min(lo.x, p.x), std::min(lo.y, p.y)};
            hi = V2{std::max(hi.x, p.x), std::max(hi.y, p.y)};
          }
        PairJob j{};
        j.ring_d = static_cast<uint32_t>(rings.size());
        j.nd = static_cast<uint32_t>(pd.size());
        for (const V2& p : pd) rings.push_back(make_double2(p.x, p.y));
        j.ring_t = static_cast<uint32_t>(rings.size());
        j.nt = static_cast<uint32_t>(pt.size());
        for (const V2& p : pt) rings.push_back(make_double2(p.x, p.y));
        j.lox = lo.x;
        j.loy = lo.y;
        j.res = raster_res;
        j.nx = std::max(1, static_cast<int>(std::ceil((hi.x - lo.x) / raster_res)));
        j.ny = std::max(1, static_cast<int>(std::ceil((hi.y - lo.y) / raster_res)));
        jobs.push_back(j);
        job_pair.emplace_back(static_cast<int>(t), static_cast<int>(d));
      }
    std::vector<unsigned long long> counts(2 * jobs.size());
    if (!jobs.empty()) {
      ckc(cudaSetDevice(device), "cudaSetDevice");
      PairJob* dj = nullptr;
      double2* dr = nullptr;
      unsigned long long* dc = nullptr;
      ckc(cudaMalloc(&dj, jobs.size() * sizeof(PairJob)), "cudaMalloc");
      ckc(cudaMalloc(&dr, rings.size() * sizeof(double2)), "cudaMalloc");
      ckc(cudaMalloc(&dc, counts.size() * 8), "cudaMalloc");
      ckc(cudaMemcpy(dj, jobs.data(), jobs.size() * sizeof(PairJob), cudaMemcpyHostToDevice), "h2d");
      ckc(cudaMemcpy(dr, rings.data(), rings.size() * sizeof(double2), cudaMemcpyHostToDevice), "h2d");
      k_iou_raster<<<static_cast<unsigned>(jobs.size()), 256>>>(dj, dr, dc);
      ckc(cudaGetLastError(), "k_iou_raster");
      ckc(cudaMemcpy(counts.data(), dc, counts.size() * 8, cudaMemcpyDeviceToHost), "d2h");
      cudaFree(dj);
      cudaFree(dr);
      cudaFree(dc);
    }
    // match_planes (metrics.cpp:114-160)
    struct Pair {
      double iou;
      int truth_id, detected_id;
    };
    std::vector<Pair> pairs;
    for (size_t k = 0; k < jobs.size(); ++k) {
      const unsigned long long inter = counts[2 * k], uni = counts[2 * k + 1];
      const double iou = uni == 0 ? 0.0 : static_cast<double>(inter) / static_cast<double>(uni);
      if (iou > 0.0) pairs.push_back({iou, job_pair[k].first, job_pair[k].second});
    }
    std::sort(pairs.begin(), pairs.end(), [](const Pair& a, const Pair& b) {
      if (a.iou != b.iou) return a.iou > b.iou;
      if (a.truth_id != b.truth_id) return a.truth_id < b.truth_id;
      return a.detected_id < b.detected_id;
    });
    std::vector<bool> tu(nt), du(nd);
    std::vector<vp_plane_match> m;
    for (const Pair& p : pairs) {
      if (tu[p.truth_id] || du[p.detected_id]) continue;
      tu[p.truth_id] = true;
      du[p.detected_id] = true;
      m.push_back({p.detected_id, p.truth_id, p.iou});
    }
    std::sort(m.begin(), m.end(), [](const vp_plane_match& a, const vp_plane_match& b) {
      return a.truth_id < b.truth_id;
    });
    double sum = 0.0, weighted = 0.0, total = 0.0;
    std::vector<double> ti(nt, 0.0);
    for (const auto& x : m) ti[x.truth_id] = x.iou;
    for (size_t t = 0; t < nt; ++t) {
      sum += ti[t];
      weighted += ti[t] * std::abs(truth->polys[t].area);
      total += std::abs(truth->polys[t].area);
    }
    rep->matched = m.size();
    rep->mean_iou = nt == 0 ? 0.0 : sum / static_cast<double>(nt);
    rep->area_weighted_iou = total > 0.0 ? weighted / total : 0.0;
    rep->unmatched_truth = nt - m.size();
    rep->unmatched_detected = nd - m.size();
    if (matches && !m.empty()) std::memcpy(matches, m.data(), m.size() * sizeof(vp_plane_match));
    return VP_OK;
  } catch (const std::exception& e) {
    g_iou_err = e.what();
    return VP_ECUDA;
  }
}

int vp_write_iou_report(const char* path, const vp_iou_report* r, const vp_plane_match* matches) {
  FILE* f = std::fopen(path, "w");
  if (!f) return VP_EINVAL;
  std::fprintf(f, "# voxplane iou report v1\ntruth_planes %llu\ndetected_planes %llu\nmatched %llu\n"
               "unmatched_truth %llu\nunmatched_detected %llu\nmean_iou %.9g\narea_weighted_iou %.9g\n",
               static_cast<unsigned long long>(r->truth_count), static_cast<unsigned long long>(r->detected_count),
               static_cast<unsigned long long>(r->matched), static_cast<unsigned long long>(r->unmatched_truth),
               static_cast<unsigned long long>(r->unmatched_detected), r->mean_iou, r->area_weighted_iou);
  for (uint64_t i = 0; i < r->matched; ++i)
    std::fprintf(f, "match truth=%d detected=%d iou=%.9g\n", matches[i].truth_id, matches[i].detected_id,
                 matches[i].iou);
  const bool ok = std::ferror(f) == 0;
  std::fclose(f);
  return ok ? VP_OK : VP_EINVAL;
}

}  // extern "C"
