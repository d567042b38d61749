// Device frame source: render_frame (scene_sim.cpp:186-236) with cast_ray
// (scene_sim.cpp:121-157) on the GPU, so a sensor-rate stream never leaves
// HBM. One thread per ray; the geometry is the
// reference's FP64 arithmetic in its evaluation order (the library is built
// with -fmad=false), the range noise is CounterRng(seed, frame, ray).normal()
// (rng.hpp:45-59) with the device log / cos; hits are compacted in ray order.
#include <cmath>
#include <cstring>
#include <string>

#include "voxplane_b200.h"
#include "voxplane_scene.h"
#include "vp_kernels.cuh"

using namespace vp;

namespace {

constexpr double kRayEps = 1e-9;
constexpr double kDegToRad = 0.017453292519943295769237;

struct RenderDesc {
  const vp_box* boxes;
  const vp_rect* rects;
  int nb, nr;
  int pinhole, width;
  uint64_t rays;
  double tan_h, tan_v, u_den, v_den;  // u = 2c/(w-1) - 1 etc.; den <= 0: u = 0
  const float* pattern;
  double max_range, sigma;
  uint64_t seed, frame;
  double R[9], t[3];
};

__device__ __forceinline__ d3 matvec(const double* r, d3 p) {
  return mk3((r[0] * p.x + r[1] * p.y) + r[2] * p.z, (r[3] * p.x + r[4] * p.y) + r[5] * p.z,
             r[6] * p.x + (r[7] * p.y + r[8] * p.z));
}
__device__ __forceinline__ double comp(d3 v, int k) { return k == 0 ? v.x : (k == 1 ? v.y : v.z); }

// scene_sim.cpp:121-157
__device__ double cast_ray(const RenderDesc& s, d3 o, d3 d) {
  double best = CUDART_INF;
  for (int b = 0; b < s.nb; ++b) {
    double t0 = 0.0, t1 = CUDART_INF;
    bool miss = false;
    for (int k = 0; k < 3 && !miss; ++k) {
      const double dk = comp(d, k), ok = comp(o, k);
      if (dk == 0.0) {
        if (ok < s.boxes[b].min[k] || ok > s.boxes[b].max[k]) miss = true;
        continue;
      }
      double ta = (s.boxes[b].min[k] - ok) / dk;
      double tb = (s.boxes[b].max[k] - ok) / dk;
      if (ta > tb) {
        const double w = ta;
        ta = tb;
        tb = w;
      }
      t0 = t0 < ta ? ta : t0;  // std::max
      t1 = tb < t1 ? tb : t1;  // std::min
      if (t0 > t1) miss = true;
    }
    if (miss) continue;
    const double t = t0 > kRayEps ? t0 : t1;
    if (t > kRayEps && t < best) best = t;
  }
  for (int i = 0; i < s.nr; ++i) {
    const double* R = s.rects[i].R;
    const d3 tr = mk3(s.rects[i].t[0], s.rects[i].t[1], s.rects[i].t[2]);
    const d3 n = mk3(R[2], R[5], R[8]);  // rotation.col(2)
    const double denom = dot3(n, d);
    if (fabs(denom) < 1e-12) continue;
    const double t = dot3(n, sub3(tr, o)) / denom;
    if (t <= kRayEps || t >= best) continue;
    const d3 q = sub3(add3(o, scl3(t, d)), tr);
    if (fabs(dot3(q, mk3(R[0], R[3], R[6]))) <= s.rects[i].half_u &&
        fabs(dot3(q, mk3(R[1], R[4], R[7]))) <= s.rects[i].half_v)
      best = t;
  }
  return best <= s.max_range ? best : CUDART_INF;
}

__device__ __forceinline__ double rng_uniform(CounterRng& r) {
  return static_cast<double>(r.next() >> 11) * 0x1.0p-53;
}

__global__ void k_render_rays(RenderDesc s, float* hits, uint8_t* flag) {
  VP_GRID_WAIT();
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < s.rays;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    d3 ds;
    if (!s.pinhole) {
      const float* q = s.pattern + 3 * i;
      ds = normalized3(mk3(static_cast<double>(q[0]), static_cast<double>(q[1]), static_cast<double>(q[2])));
    } else {
      const int r = static_cast<int>(i) / s.width;
      const int c = static_cast<int>(i) % s.width;
      const double u = s.u_den > 0.0 ? 2.0 * c / s.u_den - 1.0 : 0.0;
      const double v = s.v_den > 0.0 ? 2.0 * r / s.v_den - 1.0 : 0.0;
      ds = normalized3(mk3(1.0, -u * s.tan_h, -v * s.tan_v));
    }
    const d3 o = mk3(s.t[0], s.t[1], s.t[2]);
    const double tt = cast_ray(s, o, matvec(s.R, ds));
    if (!isfinite(tt)) {
      flag[i] = 0;
      continue;
    }
    double range = tt;
    if (s.sigma > 0.0) {  // CounterRng(seed, frame, ray).normal(), first value (rng.hpp:45-59)
      CounterRng rng(s.seed, s.frame, i);
      double u1 = rng_uniform(rng);
      while (u1 <= 0.0) u1 = rng_uniform(rng);
      const double u2 = rng_uniform(rng);
      const double rr = sqrt(-2.0 * log(u1));
      const double a = 6.283185307179586476925286766559 * u2;
      double ns = s.sigma * (rr * cos(a));
      const double lim = 3.0 * s.sigma;
      ns = ns < -lim ? -lim : (lim < ns ? lim : ns);  // std::clamp
      range += ns;
    }
    hits[3 * i] = static_cast<float>(ds.x * range);
    hits[3 * i + 1] = static_cast<float>(ds.y * range);
    hits[3 * i + 2] = static_cast<float>(ds.z * range);
    flag[i] = 1;
  }
}

__global__ void k_render_compact(uint64_t rays, const float* __restrict__ hits, const uint8_t* __restrict__ flag,
                                 const uint32_t* __restrict__ pos, float* out) {
  VP_GRID_WAIT();
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rays;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (!flag[i]) continue;
    const uint32_t k = pos[i];
    out[3ull * k] = hits[3 * i];
    out[3ull * k + 1] = hits[3 * i + 1];
    out[3ull * k + 2] = hits[3 * i + 2];
  }
}

template <typename T>
T* alloc(size_t n) {
  void* p = nullptr;
  if (cudaMalloc(&p, (n ? n : 1) * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return static_cast<T*>(p);
}

}  // namespace

struct vp_frame_source {
  int device = 0;
  cudaStream_t stream = nullptr;
  RenderDesc d{};
  vp_box* boxes = nullptr;
  vp_rect* rects = nullptr;
  float* pattern = nullptr;
  float* hits = nullptr;
  float* out = nullptr;
  uint8_t* flag = nullptr;
  uint32_t* pos = nullptr;
  uint32_t* bsum = nullptr;
  uint32_t* nbuf = nullptr;  // [0] rays (n_ptr of the scan), [1] hits, [2] blocks done (fused scan)
  uint32_t nblocks = 0;
  ~vp_frame_source() {
    if (stream) cudaStreamSynchronize(stream);
    void* ptrs[] = {boxes, rects, pattern, hits, out, flag, pos, bsum, nbuf};
    for (void* q : ptrs)
      if (q) cudaFree(q);
    if (stream) cudaStreamDestroy(stream);
  }
};

extern "C" {

int vp_frame_source_create(const vp_box* boxes, size_t nb, const vp_rect* rects, size_t nr,
                           const vp_sensor* sensor, uint64_t seed, int device, vp_frame_source** outp) {
  *outp = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return VP_ENODEV;
  }
  if (cudaSetDevice(device) != cudaSuccess) return VP_ENODEV;
  const bool pinhole = sensor->kind == 0;
  const uint64_t rays = pinhole ? static_cast<uint64_t>(sensor->width) * sensor->height : sensor->npattern;
  if (rays >= (1ull << 31)) return VP_EINVAL;
  auto* s = new vp_frame_source();
  s->device = device;
  RenderDesc& d = s->d;
  d.nb = static_cast<int>(nb);
  d.nr = static_cast<int>(nr);
  d.pinhole = pinhole ? 1 : 0;
  d.width = sensor->width;
  d.rays = rays;
  // scene_sim.cpp:193-194, 204-206 (host libm, as the reference)
  d.tan_h = std::tan(0.5 * sensor->hfov_deg * kDegToRad);
  d.tan_v = std::tan(0.5 * sensor->vfov_deg * kDegToRad);
  d.u_den = sensor->width > 1 ? static_cast<double>(sensor->width - 1) : 0.0;
  d.v_den = sensor->height > 1 ? static_cast<double>(sensor->height - 1) : 0.0;
  d.max_range = sensor->max_range;
  d.sigma = sensor->noise_sigma;
  d.seed = seed;
  bool ok = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking) == cudaSuccess;
  s->boxes = alloc<vp_box>(nb);
  s->rects = alloc<vp_rect>(nr);
  s->pattern = alloc<float>(pinhole ? 1 : 3 * rays);
  s->hits = alloc<float>(3 * rays);
  s->out = alloc<float>(3 * rays);
  s->flag = alloc<uint8_t>(rays);
  s->pos = alloc<uint32_t>(rays);
  s->nblocks = static_cast<uint32_t>((rays + kScanPerBlock - 1) / kScanPerBlock);
  s->bsum = alloc<uint32_t>(s->nblocks + 1);
  s->nbuf = alloc<uint32_t>(3);
  ok = ok && s->boxes && s->rects && s->pattern && s->hits && s->out && s->flag && s->pos && s->bsum && s->nbuf;
  if (ok) {
    const uint32_t nr32[3] = {static_cast<uint32_t>(rays), 0u, 0u};
    ok = cudaMemcpy(s->boxes, boxes, nb * sizeof(vp_box), cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(s->rects, rects, nr * sizeof(vp_rect), cudaMemcpyHostToDevice) == cudaSuccess &&
         cudaMemcpy(s->nbuf, nr32, 12, cudaMemcpyHostToDevice) == cudaSuccess &&
         (pinhole || cudaMemcpy(s->pattern, sensor->pattern, 12 * rays, cudaMemcpyHostToDevice) == cudaSuccess);
  }
  if (!ok) {
    delete s;
    return VP_ENOMEM;
  }
  d.boxes = s->boxes;
  d.rects = s->rects;
  d.pattern = s->pattern;
  *outp = s;
  return VP_OK;
}

void vp_frame_source_destroy(vp_frame_source* s) { delete s; }

void* vp_frame_source_stream(vp_frame_source* s) { return s->stream; }

int vp_frame_source_render(vp_frame_source* s, const double R[9], const double t[3], uint64_t frame_index,
                           const float** xyz_dev, uint64_t* n, double qR[9], double qt[3]) {
  *xyz_dev = nullptr;
  *n = 0;
  const int rc = vp_quantize_pose(R, t, qR, qt);
  if (rc != VP_OK) return rc;
  cudaSetDevice(s->device);
  RenderDesc d = s->d;
  std::memcpy(d.R, qR, sizeof d.R);
  std::memcpy(d.t, qt, sizeof d.t);
  d.frame = frame_index;
  const uint64_t rays = d.rays;
  const int grid = static_cast<int>(std::min<uint64_t>((rays + 255) / 256, 148ull * 16));
  k_render_rays<<<grid > 0 ? grid : 1, 256, 0, s->stream>>>(d, s->hits, s->flag);
  k_flags_count<<<s->nblocks ? s->nblocks : 1, kScanThreads, 0, s->stream>>>(
      s->flag, s->nbuf, static_cast<uint32_t>(rays), s->bsum, s->nbuf + 1, s->nbuf + 2);  // + the block-sum scan
  k_flags_positions<<<s->nblocks ? s->nblocks : 1, kScanThreads, 0, s->stream>>>(
      s->flag, s->nbuf, static_cast<uint32_t>(rays), s->bsum, s->pos);
  k_render_compact<<<grid > 0 ? grid : 1, 256, 0, s->stream>>>(rays, s->hits, s->flag, s->pos, s->out);
  uint32_t hits = 0;
  if (cudaMemcpyAsync(&hits, s->nbuf + 1, 4, cudaMemcpyDeviceToHost, s->stream) != cudaSuccess ||
      cudaStreamSynchronize(s->stream) != cudaSuccess) {
    cudaGetLastError();
    return VP_ECUDA;
  }
  *xyz_dev = s->out;
  *n = hits;
  return VP_OK;
}

}  // extern "C"
