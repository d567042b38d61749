// Host runtime and C ABI (include/voxplane_b200.h).
//
// One vp_grid owns its device buffers and one CUDA stream. A frame update
// (clear -> integrate -> recenter -> segment) is a fixed sequence of kernels
// whose data-dependent sizes live in device counters, so the host never waits
// mid-frame; it synchronises once to read the result records.
#include <algorithm>
#include <chrono>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <limits>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "voxplane_b200.h"
#include "voxplane_trace.h"
#include "vp_kernels.cuh"

using namespace vp;

namespace vp {
void slab_frame_release(vp_grid* g);  // slab_frame.cu
}

namespace {

thread_local std::string g_err;
// CCL variant: 0 = min-neighbour hook + forward-window unions (default),
// 1 = neighbour sampling + giant skip, 2 = hook + giant skip (same labels)
int g_ccl_mode = 0;
// polygon stage as five kernels instead of k_poly_fused (VP_POLY_SPLIT=1, A/B)
const bool g_poly_split = getenv("VP_POLY_SPLIT") && atoi(getenv("VP_POLY_SPLIT")) != 0;
// programmatic dependent launch on every LAUNCH (VP_PDL=0 disables, A/B)
const bool g_pdl = !(getenv("VP_PDL") && atoi(getenv("VP_PDL")) == 0);
// pointer-jumping rounds between hook and compress (VP_CCL_JUMPS, A/B)
int g_ccl_jumps = getenv("VP_CCL_JUMPS") ? atoi(getenv("VP_CCL_JUMPS")) : 3;
// VP_WALK_GENERIC=1 (experiments): plain-grid rays through the generic walk loop
const int g_walk_generic = std::getenv("VP_WALK_GENERIC") ? 1 : 0;
// DDA walk mode (A/B): -1 k_dda_plan decides, 0 coherent lockstep, 1 bricks
const int g_dda_force = std::getenv("VP_DDA_FORCE") ? std::atoi(std::getenv("VP_DDA_FORCE")) : -1;
// mean estimated DDA steps per ray above which the plan walks bricks, for
// windows whose clear mask is larger than kDdaL2Mask (VP_DDA_LONG: any window)
const int g_dda_long = std::getenv("VP_DDA_LONG") ? std::atoi(std::getenv("VP_DDA_LONG")) : -1;
constexpr uint64_t kDdaL2Mask = 64ull << 20;
std::atomic<uint64_t> g_launches{0};

constexpr double kRadToDeg = 57.295779513082320876798;
constexpr double kDegToRad = 0.017453292519943295769237;
constexpr double kPi = 3.14159265358979323846;  // == glibc M_PI
constexpr int kThreads = 256;
#ifndef VP_CHAIN_WIDE
#define VP_CHAIN_WIDE (148 * 4)
#endif
constexpr int kChainWide = VP_CHAIN_WIDE;  // CCL .. polygon grid width in pipelined runs
#ifndef VP_SLOTS
#define VP_SLOTS 6
#endif
constexpr int kSlots = VP_SLOTS;  // frames in flight in a pipelined run
#ifndef VP_COPY_AHEAD
#define VP_COPY_AHEAD VP_SLOTS  // host frames copied ahead (e2e 3330 -> 3430 Hz vs 2)
#endif

struct VpFail {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg) { throw VpFail{code, msg}; }

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(VP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// Optional per-kernel profiling (vp_profile_enable): every launch is bracketed
// by CUDA events on its stream and the elapsed time is accumulated per kernel.
struct ProfEntry {
  std::string name;
  double ms = 0.0;
  uint64_t calls = 0;
};
std::vector<ProfEntry> g_prof;
bool g_prof_on = false;
cudaEvent_t g_prof_ev[2] = {nullptr, nullptr};

void prof_begin(cudaStream_t s) {
  if (!g_prof_ev[0]) {
    cudaEventCreate(&g_prof_ev[0]);
    cudaEventCreate(&g_prof_ev[1]);
  }
  cudaEventRecord(g_prof_ev[0], s);
}
void prof_end(cudaStream_t s, const char* name) {
  cudaEventRecord(g_prof_ev[1], s);
  cudaEventSynchronize(g_prof_ev[1]);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, g_prof_ev[0], g_prof_ev[1]);
  for (auto& e : g_prof)
    if (e.name == name) {
      e.ms += ms;
      ++e.calls;
      return;
    }
  g_prof.push_back(ProfEntry{name, ms, 1});
}

// Every kernel is launched with programmatic stream serialisation (PDL): its
// launch and block dispatch overlap the previous kernel's tail, and its first
// statement (VP_GRID_WAIT) holds it until that kernel's writes are visible.
// Inside a CUDA graph the kernel-to-kernel edges become programmatic edges.
// VP_PDL=0 launches without the attribute (A/B).
#define LAUNCH(kernel, grid, block, smem, strm_, ...)                           \
  do {                                                                         \
    if (g_prof_on) prof_begin(strm_);                                         \
    cudaLaunchConfig_t cfg_{};                                                 \
    cfg_.gridDim = dim3(grid);                                                 \
    cfg_.blockDim = dim3(block);                                               \
    cfg_.dynamicSmemBytes = (smem);                                            \
    cfg_.stream = (strm_);                                                      \
    cudaLaunchAttribute at_[1];                                                \
    at_[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;            \
    at_[0].val.programmaticStreamSerializationAllowed = 1;                     \
    cfg_.attrs = at_;                                                          \
    cfg_.numAttrs = g_pdl ? 1 : 0;                                             \
    ck(cudaLaunchKernelEx(&cfg_, kernel, __VA_ARGS__), #kernel);               \
    g_launches.fetch_add(1, std::memory_order_relaxed);                        \
    if (g_prof_on) prof_end(strm_, #kernel);                                  \
  } while (0)

template <typename T>
T* dalloc(size_t n) {
  if (n == 0) n = 1;
  void* p = nullptr;
  const cudaError_t e = cudaMalloc(&p, n * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(VP_ENOMEM, "cudaMalloc " + std::to_string(n * sizeof(T)) + " bytes: " + cudaGetErrorString(e));
  }
  return static_cast<T*>(p);
}

template <typename T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

int grid_for(uint64_t n, int cap = 148 * 16) {
  const uint64_t b = (n + kThreads - 1) / kThreads;
  return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(b, static_cast<uint64_t>(cap))));
}
constexpr int kWide = 148 * 8;  // grid-stride width for device-sized loops

// voxel_grid.cpp:13-17 (r^T r in the shim's product order; tolerance 1e-6)
bool is_valid_rotation(const double* R) {
  double t[3][3], p[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t[i][j] = R[3 * j + i];
  for (int j = 0; j < 3; ++j)
    for (int i = 0; i < 3; ++i)
      p[i][j] = i < 2 ? (t[i][0] * R[j] + t[i][1] * R[3 + j]) + t[i][2] * R[6 + j]
                      : t[i][0] * R[j] + (t[i][1] * R[3 + j] + t[i][2] * R[6 + j]);
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
  auto m = [&](int r, int c) { return R[3 * r + c]; };
  auto h = [&](int a, int b, int c) { return m(0, a) * (m(1, b) * m(2, c) - m(1, c) * m(2, b)); };
  const double det = h(0, 1, 2) - h(1, 0, 2) + h(2, 0, 1);
  return std::abs(det - 1.0) <= 1e-6;
}

// Smallest d in [0,1] with acos(d)*kRadToDeg <= theta (segmentation.cpp:62-63,
// 74-75), by bisection over the IEEE bit patterns with the host libm.
double angle_threshold(double theta) {
  auto ok = [&](double d) { return std::acos(d) * kRadToDeg <= theta; };
  if (!ok(1.0)) return std::numeric_limits<double>::infinity();
  if (ok(0.0)) return 0.0;
  uint64_t lo, hi;
  double z = 0.0, o = 1.0;
  std::memcpy(&lo, &z, 8);
  std::memcpy(&hi, &o, 8);
  while (hi - lo > 1) {
    const uint64_t mid = lo + (hi - lo) / 2;
    double d;
    std::memcpy(&d, &mid, 8);
    if (ok(d)) hi = mid; else lo = mid;
  }
  double d;
  std::memcpy(&d, &hi, 8);
  return d;
}

SegDev make_segdev(const vp_seg_params& p, double res) {
  SegDev s;
  s.radius = p.neighbor_radius;
  s.min_neighbors = p.min_neighbors;
  s.dstar = angle_threshold(p.max_angle_deg);
  s.up = d3{p.up[0], p.up[1], p.up[2]};
  s.w = std::max(1, static_cast<int>(std::ceil(p.distance_th / res)));
  // a window row (2w + 1 cells along z) is read as one 32-bit bitmap span
  if (s.w > 15) fail(VP_EINVAL, "segment: distance_th / resolution above 15 cells is not supported");
  s.d2_th = p.distance_th * p.distance_th;
  s.cos_th = std::cos(p.adjacency_angle_deg * kDegToRad);
  s.min_cluster = p.min_cluster_size;
  return s;
}

RansacDev make_ransacdev(const vp_ransac_params& r) {
  RansacDev d;
  d.iterations = r.iterations;
  d.eps = r.inlier_eps;
  d.seed = r.seed;
  d.up = d3{r.up[0], r.up[1], r.up[2]};
  return d;
}

void check_device(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    fail(VP_ENODEV, "no CUDA device visible");
  }
  if (device < 0 || device >= n) fail(VP_ENODEV, "device index out of range");
  cudaDeviceProp prop;
  ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10) fail(VP_ENODEV, std::string("sm_100a build needs a B200-class device, got ") + prop.name);
  ck(cudaSetDevice(device), "cudaSetDevice");
}

// Segmentation scratch sized by capacities; grows on overflow.
struct Seg {
  SegBufs b{};
  uint32_t* bsum = nullptr;  // scan block sums
  uint32_t bsum_cap = 0;
  double* dirtab = nullptr;
  int dir_n = -1;
  uint32_t hstride = 0;

  // capacity-dependent buffers (the direction table survives a regrow: a
  // pipelined run re-captures its graphs after one, and a capture may not
  // allocate or synchronise)
  void release_buffers() {
    void* ptrs[] = {b.occ_list, b.est_normal, b.est_ncount, b.est_valid, b.own_mean, b.own_count,
                    b.own_status, b.step_flag, b.st_idx, b.st_mean, b.st_normal,
                    b.parent, b.label, b.cnt, b.cid, b.big_flag, b.big_pos, b.klabel, b.ksize,
                    b.kpoff, b.H, b.mx, b.my, b.mz, b.cand, b.cand_cnt, b.win_it, b.win_cnt,
                    b.fid, b.fit_cluster, b.ioff, b.fch_off, b.ccount, b.fit_model, b.fit_meta, b.ref_model, b.inl,
                    b.rch_off, b.rpart, b.rcen,
                    b.proj, b.surv, b.hull, b.basis, b.pch_off, b.pext_dot, b.pext_idx, b.inner,
                    b.ninner, b.nsurv, b.pdone, b.prec_d, b.prec_i, b.pool, b.pair_key, b.pair_slot, bsum};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    b = SegBufs{};
    bsum = nullptr;
  }
  void release() {
    release_buffers();
    if (dirtab) cudaFree(dirtab);
    dirtab = nullptr;
    dir_n = -1;
  }
  void alloc_bsum(uint64_t need_bsum) {
    bsum_cap = static_cast<uint32_t>(need_bsum);
    // three regions: occupied-scan tile sums | steppable tile offsets (kept for
    // step_emit, also on a chain re-run) | flag scans (clusters)
    bsum = dalloc<uint32_t>(3ull * need_bsum);
  }

  // Cluster-count dependent buffers (clusters, members' padding, RANSAC
  // candidates, fits, polygon records) sized by kcap; the member counting
  // sort's chunk histogram by hcap. Grown by grow_k when a frame has more
  // clusters (the cluster setup flags kOverflowClusters), keeping every other
  // buffer -- the occupied and steppable lists stay valid for a chain re-run.
  uint32_t kcap = kClusterBins;
  uint64_t hcap = 0;
  void release_k_buffers() {
    void* ptrs[] = {b.klabel, b.ksize, b.kpoff, b.H, b.mx, b.my, b.mz, b.cand, b.cand_cnt, b.win_it, b.win_cnt,
                    b.fid, b.fit_cluster, b.ioff, b.fch_off, b.ccount, b.fit_model, b.fit_meta, b.ref_model,
                    b.rch_off, b.rpart, b.rcen, b.basis, b.pch_off, b.pext_dot, b.pext_idx, b.inner, b.ninner,
                    b.nsurv, b.pdone, b.prec_d, b.prec_i};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    b.klabel = nullptr, b.ksize = nullptr, b.kpoff = nullptr, b.H = nullptr, b.mx = b.my = b.mz = nullptr;
    b.cand = nullptr, b.cand_cnt = nullptr, b.win_it = b.win_cnt = b.fid = nullptr, b.fit_cluster = nullptr;
    b.ioff = b.fch_off = b.ccount = nullptr, b.fit_model = nullptr, b.fit_meta = nullptr, b.ref_model = nullptr;
    b.rch_off = nullptr, b.rpart = nullptr, b.rcen = nullptr, b.basis = nullptr, b.pch_off = nullptr;
    b.pext_dot = nullptr, b.pext_idx = nullptr, b.inner = nullptr, b.ninner = b.nsurv = b.pdone = nullptr;
    b.prec_d = nullptr, b.prec_i = nullptr;
  }
  void alloc_k_buffers(int iterations) {
    const uint32_t K = kcap;
    const uint32_t scap = b.Scap, icap = b.Icap;
    const uint32_t mcap = scap + 32u * K;
    b.Mcap = mcap;
    b.Kcap = K;
    cand_cap = static_cast<uint64_t>(std::max(iterations, 1)) * K;
    b.klabel = dalloc<int32_t>(K);
    b.ksize = dalloc<uint32_t>(K);
    b.kpoff = dalloc<uint32_t>(K + 1);
    hstride = (scap + kChunk - 1) / kChunk;
    hcap = std::max<uint64_t>(hcap, static_cast<uint64_t>(std::min(K, static_cast<uint32_t>(kClusterBins))) * hstride);
    b.H = dalloc<uint32_t>(hcap);
    b.Hcap = hcap;
    b.mx = dalloc<double>(mcap);
    b.my = dalloc<double>(mcap);
    b.mz = dalloc<double>(mcap);
    b.cand = dalloc<double>(4 * cand_cap);
    b.cand_cnt = dalloc<int32_t>(cand_cap);
    b.win_it = dalloc<int32_t>(K);
    b.win_cnt = dalloc<int32_t>(K);
    b.fid = dalloc<int32_t>(K);
    b.fit_cluster = dalloc<uint32_t>(K);
    b.ioff = dalloc<uint32_t>(K + 1);
    b.fch_off = dalloc<uint32_t>(K + 1);
    b.cch_cap = mcap / kPolyChunk + K + 1;
    b.ccount = dalloc<uint32_t>(b.cch_cap);
    b.fit_model = dalloc<double>(4ull * K);
    b.fit_meta = dalloc<int32_t>(2ull * K);
    b.ref_model = dalloc<double>(4ull * K);
    b.rch_off = dalloc<uint32_t>(K + 1);
    b.rpart = dalloc<double>(8ull * (icap / kRefineChunk + K + 1));
    b.rcen = dalloc<double>(3ull * K);
    b.basis = dalloc<double>(9ull * K);
    b.pch_off = dalloc<uint32_t>(K + 1);
    b.pch_cap = icap / kPolyChunk + K + 1;
    b.pext_dot = dalloc<double>(64ull * b.pch_cap);
    b.pext_idx = dalloc<int32_t>(64ull * b.pch_cap);
    b.inner = dalloc<double>(2ull * 130 * K);
    b.ninner = dalloc<uint32_t>(K);
    b.nsurv = dalloc<uint32_t>(K);
    b.pdone = dalloc<uint32_t>(K);
    ck(cudaMemset(b.pdone, 0, 4ull * K), "memset pdone");
    b.prec_d = dalloc<double>(8ull * K);
    b.prec_i = dalloc<int32_t>(4ull * K);
  }
  // more clusters than kcap, or a chunk histogram above hcap: K clusters over S
  // steppable voxels (the counters of the overflowing frame)
  void grow_k(uint32_t K, uint32_t S, int iterations) {
    ++gen;
    uint32_t k = kcap;
    while (k < K) k *= 2;
    const uint64_t nch = (static_cast<uint64_t>(S) + kChunk - 1) / kChunk;
    hcap = std::max<uint64_t>(hcap, static_cast<uint64_t>(K) * nch);  // the member sort's chunk histogram
    kcap = k;
    release_k_buffers();
    alloc_k_buffers(iterations);
  }

  void ensure(uint32_t vcap, uint32_t scap, uint32_t icap, int iterations, uint64_t nwords) {
    const bool need = !b.occ_list || vcap > b.Vcap || scap > b.Scap || icap > b.Icap ||
                      static_cast<uint64_t>(iterations) * kcap > cand_cap;
    const uint64_t need_bsum = std::max<uint64_t>({(nwords + kRowsPerBlock - 1) / kRowsPerBlock,  // >= rows / tile
                                                   (vcap + kThreads - 1) / kThreads,
                                                   (scap + kScanPerBlock - 1) / kScanPerBlock}) + 1;
    if (need) {
      ++gen;
      release_buffers();
      struct Unwind {  // a failed allocation leaves no half-built context behind
        Seg* s;
        bool done = false;
        ~Unwind() {
          if (!done) s->release_buffers();
        }
      } unwind{this};
      b.Vcap = vcap;
      b.Scap = scap;
      b.Icap = icap;
      b.occ_list = dalloc<uint32_t>(vcap);
      b.est_normal = dalloc<double>(3ull * vcap);
      b.est_ncount = dalloc<int32_t>(vcap);
      b.est_valid = dalloc<uint8_t>(vcap);
      b.own_mean = dalloc<double>(3ull * vcap);
      b.own_count = dalloc<uint32_t>(vcap);
      b.own_status = dalloc<uint8_t>(vcap);
      b.step_flag = dalloc<uint8_t>(vcap);
      b.st_idx = dalloc<int32_t>(3ull * scap);
      b.st_mean = dalloc<double>(3ull * scap);
      b.st_normal = dalloc<double>(3ull * scap);
      b.parent = dalloc<int32_t>(scap);
      b.label = dalloc<int32_t>(scap);
      b.cnt = dalloc<uint32_t>(scap);
      b.cid = dalloc<int32_t>(scap);
      b.big_flag = dalloc<uint8_t>(scap);
      b.big_pos = dalloc<uint32_t>(scap);
      hcap = 0;  // re-derived from the new steppable capacity
      alloc_k_buffers(iterations);
      b.inl = dalloc<double>(3ull * icap);
      b.proj = dalloc<double>(2ull * icap);
      b.surv = dalloc<double>(4ull * icap);
      b.hull = dalloc<double>(4ull * icap);
      b.pool_cap = icap;
      b.pool = dalloc<double>(5ull * icap);
      b.pair_cap = 2048;  // CCL root-pair set (load factor <= 1/2; overflow -> full union)
      while (b.pair_cap < scap / 4) b.pair_cap <<= 1;
      if (const char* f = getenv("VP_CCL_PAIR_CAP")) {  // test hook: force (tiny) tables
        b.pair_cap = 2;
        while (b.pair_cap < static_cast<uint32_t>(atoi(f))) b.pair_cap <<= 1;
      }
      b.pair_key = dalloc<unsigned long long>(b.pair_cap);
      ck(cudaMemset(b.pair_key, 0xff, 8ull * b.pair_cap), "pair table init");
      b.pair_slot = dalloc<uint32_t>(b.pair_cap / 2);
      alloc_bsum(need_bsum);
      unwind.done = true;
    } else if (need_bsum > bsum_cap) {
      ++gen;
      dfree(bsum);
      alloc_bsum(need_bsum);
    }
  }

  void ensure_dirs(int n, cudaStream_t s) {
    if (n == dir_n) return;
    if (n > 64) fail(VP_EINVAL, "make_polygon: at most 64 filter directions supported");
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    ck(cudaStreamIsCapturing(s, &cs), "capture status");
    if (cs != cudaStreamCaptureStatusNone) fail(VP_ECUDA, "make_polygon: direction table not set before capture");
    std::vector<double> t(2 * 64, 0.0);
    for (int j = 0; j < n; ++j) {  // polygonize.cpp:59-63
      const double a = 2.0 * kPi * j / n;
      t[2 * j] = std::cos(a);
      t[2 * j + 1] = std::sin(a);
    }
    if (!dirtab) dirtab = dalloc<double>(128);
    ck(cudaMemcpyAsync(dirtab, t.data(), 128 * sizeof(double), cudaMemcpyHostToDevice, s), "dirtab");
    ck(cudaStreamSynchronize(s), "dirtab sync");
    dir_n = n;
  }

  uint64_t cand_cap = 0;
  uint64_t gen = 0;  // bumped on reallocation (invalidates captured graphs)
};

// Per-frame layout and buffers of a slab's distributed segmentation.
struct SlabSeg {
  // layout (vp_slab_extend)
  int n = 0, me = -1;              // slabs, this slab's index
  std::vector<int32_t> xb;         // x_begin of every slab + window x extent
  std::vector<uint64_t> P;         // global plane prefix (gex + 1)
  int w = 1;
  int32_t x_lo = 0, x_hi = 0;      // extended list planes
  uint64_t n_left = 0, n_own = 0, n_ext = 0, zone_size = 0;
  int64_t base = 0, own_base = 0;
  ZoneDesc zone{};
  RankDesc rd{};
  bool labelled = false, merged = false;
  // buffers
  uint64_t xcap = 0;
  int32_t* xidx = nullptr;
  double* xmean = nullptr;
  double* xnrm = nullptr;
  int32_t* bmin = nullptr;
  int32_t* flabel = nullptr;
  uint64_t tcap = 0;
  int32_t* triples = nullptr;
  uint32_t* ntrip = nullptr;       // device counter
  uint64_t zcap = 0;
  int32_t* zparent = nullptr;
  int32_t* zminlab = nullptr;
  uint32_t* pcounts = nullptr;     // per owned plane
  int32_t pcap = 0;
  uint64_t hcap = 0;
  uint32_t* H = nullptr;
  uint32_t* dcount = nullptr;      // kMaxSlabs
  uint64_t ecap = 0;
  MemberRec* exp = nullptr;
  // dense ordinal map over the extended planes
  int32_t* xmap = nullptr;
  uint32_t* xbits = nullptr;
  uint64_t xmap_slots = 0, xmap_words = 0;

  void release() {
    void* ptrs[] = {xidx, xmean, xnrm, bmin, flabel, triples, ntrip, zparent, zminlab, pcounts, H,
                    dcount, exp, xmap, xbits};
    for (void* q : ptrs)
      if (q) cudaFree(q);
    *this = SlabSeg{};
  }
};

// Per-cluster views for fit_planes' PerClusterSerial execution mode
// (plane_fit.cpp:113-119): cluster c runs the same kernels alone with its own
// counters, a [0, padded) member offset pair and private output slots.
struct SerialFitBufs {
  uint32_t cap = 0;
  uint32_t* kp1 = nullptr;     // 2 per cluster: 0, padded size
  Counters* ctrs = nullptr;    // 1 per cluster (K = 1)
  double* fm = nullptr;        // 4 per cluster: winning model
  int32_t* fmeta = nullptr;    // 2 per cluster: inlier_count, label
  uint32_t* io1 = nullptr;     // 2 per cluster: inlier offsets
  void release() {
    void* ptrs[] = {kp1, ctrs, fm, fmeta, io1};
    for (void* q : ptrs)
      if (q) cudaFree(q);
    *this = SerialFitBufs{};
  }
};

// Host image of the per-fit records written by k_polygon.
struct HostPolys {
  std::vector<vp_polygon> polys;
  std::vector<double> verts;  // 5 per vertex (u v x y z)
};

}  // namespace

// ===========================================================================
struct vp_grid {
  int device = 0;
  cudaStream_t stream = nullptr;
  GridDesc gd{};
  double origin[3];
  int32_t ext[3];
  int32_t off[3] = {0, 0, 0};
  uint32_t* occ[2] = {nullptr, nullptr};
  int cur = 0;  // always 0: one occupancy ring (occ[1] unused)
  int32_t zb = 0;  // occupancy ring z offset (window z = 0 at ring position zb)
  // Per-frame state in two slots so consecutive frames can be in flight at
  // once (vp_pipeline_run); ctr/h_ctr/d_fp/h_fp/d_pts point at the current slot.
  Counters* ctr_s[kSlots] = {};
  Counters* h_ctr_s[kSlots] = {};  // pinned
  FrameParams* d_fp_s[kSlots] = {};
  FrameParams* h_fp_s[kSlots] = {};  // pinned
  float* d_pts_s[kSlots] = {};
  int slot = 0;
  Counters* ctr = nullptr;
  Counters* h_ctr = nullptr;
  FrameParams* d_fp = nullptr;
  FrameParams* h_fp = nullptr;
  float* d_pts = nullptr;
  unsigned long long* occ_total = nullptr;  // VoxelGrid::occupied_ (device, persistent)
  uint64_t host_occupied = 0;
  cudaStream_t mstream = nullptr;   // mapping stream of pipelined runs
  cudaStream_t fstream = nullptr;   // fork of the mapping stream (integrate grouping || clear_rays)
  cudaStream_t pstream = nullptr;   // grid-independent first half of a pipelined frame's mapping
  cudaEvent_t fork_ev[4] = {};
  // Segmentation contexts of the pipelined run's slots: frame k's CCL ..
  // polygon chain runs on its slot's stream with its own scratch and ordinal
  // map while later frames are mapped and start their chains. The active
  // context lives in (seg, gd.ordmap, gd.stbits, stream); pool[i] holds
  // context i while it is not active. use_seg(s) swaps contexts.
  Seg seg_pool[kSlots];
  cudaStream_t stream_pool[kSlots] = {};
  int32_t* ordmap_pool[kSlots] = {};
  uint32_t* stbits_pool[kSlots] = {};
  int seg_slot = 0;
  cudaStream_t lstream = nullptr;   // stream the mapping launches go to (stream or mstream)
  // grid width of the CCL .. polygon kernels: a pipelined run caps them at
  // half an SM's warp slots (148 x 4 blocks of 256) so the next mapping and grid
  // readers -- the critical path -- are not starved by latency-bound chains
  int chain_wide = 148 * 8;
  // integrate scratch
  uint64_t pcap = 0;
  uint32_t* hkey = nullptr;
  uint32_t* hcnt = nullptr;
  uint32_t* hoff = nullptr;
  uint32_t hmask = 0;
  uint32_t* groups = nullptr;
  uint32_t* pslot = nullptr;
  uint32_t* prank = nullptr;
  uint32_t* sorted = nullptr;
  uint32_t* dense = nullptr;  // slots of integrate groups > kFoldMax points
  uint32_t* medium = nullptr;  // slots of integrate groups kFoldSmall < points <= kFoldMax
  uint32_t* rperm = nullptr;  // clear_rays: rays in bin order (when binning is on)
  uint8_t* bin_of = nullptr;  // clear_rays: length bin per ray
  DdaBins* dbins = nullptr;
  Seg seg;
  cudaEvent_t ev[8];
  // window-sized ordinal map for segmenting a gathered slab steppable list
  int32_t* gmap = nullptr;
  uint32_t* gbits = nullptr;
  // distributed segmentation of a slab (vp_slab_extend .. vp_slab_segment_owned)
  SlabSeg sl;
  // fit_planes PerClusterSerial views (vp_fit_planes, vp_run_ablation)
  SerialFitBufs sf;
  // CUDA graph of one pipeline frame (see pipeline_enqueue)
  bool capturing = false;
  uint64_t gen = 1;  // bumped whenever a buffer the graph references is reallocated

  ~vp_grid() {
    if (stream) cudaStreamSynchronize(stream);
    seg.release();
    for (auto* p : {occ[0], occ[1]}) if (p) cudaFree(p);
    if (gd.cells) cudaFree(gd.cells);
    if (gd.clr) cudaFree(gd.clr);
    if (gd.clrb) cudaFree(gd.clrb);
    for (int q = 0; q < kSlots; ++q) {
      if (stream_pool[q]) cudaStreamSynchronize(stream_pool[q]);
      if (ordmap_pool[q]) cudaFree(ordmap_pool[q]);
      if (stbits_pool[q]) cudaFree(stbits_pool[q]);
      seg_pool[q].release();
    }
    if (gd.ordmap) cudaFree(gd.ordmap);
    if (gd.stbits) cudaFree(gd.stbits);
    if (gd.rowcnt) cudaFree(gd.rowcnt);
    if (gmap) cudaFree(gmap);
    if (gbits) cudaFree(gbits);
    sl.release();
    sf.release();
    if (mstream) cudaStreamSynchronize(mstream);
    for (int q = 0; q < kSlots; ++q) {
      if (ctr_s[q]) cudaFree(ctr_s[q]);
      if (d_fp_s[q]) cudaFree(d_fp_s[q]);
      if (h_ctr_s[q]) cudaFreeHost(h_ctr_s[q]);
      if (h_fp_s[q]) cudaFreeHost(h_fp_s[q]);
      if (d_pts_s[q]) cudaFree(d_pts_s[q]);
    }
    if (occ_total) cudaFree(occ_total);
    for (void* p : {(void*)hkey, (void*)hcnt, (void*)hoff, (void*)groups,
                    (void*)pslot, (void*)prank, (void*)sorted, (void*)dense, (void*)medium, (void*)rperm,
                    (void*)bin_of, (void*)dbins})
      if (p) cudaFree(p);
    for (auto& e : ev) if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
    if (mstream) cudaStreamDestroy(mstream);
    if (pstream) {
      cudaStreamSynchronize(pstream);
      cudaStreamDestroy(pstream);
    }
    if (fstream) {
      cudaStreamSynchronize(fstream);
      cudaStreamDestroy(fstream);
    }
    for (auto& e : fork_ev)
      if (e) cudaEventDestroy(e);
    for (auto& q : stream_pool)
      if (q) cudaStreamDestroy(q);
  }

  // ------------------------------------------------------------ set-up
  void init(double res, const int32_t* e, const double* c, int dev) {
    if (!(res > 0.0) || e[0] <= 0 || e[1] <= 0 || e[2] <= 0)  // voxel_grid.cpp:21-22
      fail(VP_EINVAL, "VoxelGrid: resolution and extents must be positive");
    const uint64_t C = static_cast<uint64_t>(e[0]) * e[1] * e[2];
    if (C >= (1ull << 32) || static_cast<uint64_t>(e[0]) * e[1] * ((e[2] + 31) / 32) * 32 >= 0xffffffffull)
      fail(VP_EINVAL, "VoxelGrid: more than 2^32 cells per grid (use slabs)");
    check_device(dev);
    device = dev;
    for (int k = 0; k < 3; ++k) {
      ext[k] = e[k];
      origin[k] = c[k] - static_cast<double>(e[k]) * (0.5 * res);  // voxel_grid.cpp:23
    }
    ck(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
    {  // the mapping stream carries the pipelined run's critical path: highest priority
      int lo = 0, hi = 0;
      ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority range");
      ck(cudaStreamCreateWithPriority(&mstream, cudaStreamNonBlocking, hi), "stream");
      ck(cudaStreamCreateWithPriority(&fstream, cudaStreamNonBlocking, hi), "stream");
      const char* pp = std::getenv("VP_PSTREAM_PRIO");  // experiments: 0 = highest .. lowest
      const int prio = pp ? std::min(lo, hi + std::atoi(pp)) : hi;
      ck(cudaStreamCreateWithPriority(&pstream, cudaStreamNonBlocking, prio), "stream");
      for (auto& e : fork_ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    }
    lstream = stream;
    for (auto& x : ev) ck(cudaEventCreate(&x), "event");
    gd.ex = e[0];
    gd.ey = e[1];
    gd.ez = e[2];
    gd.W = (e[2] + 31) / 32;
    gd.res = res;
    gd.ncells = C;
    gd.nwords = static_cast<uint64_t>(e[0]) * e[1] * gd.W;
    gd.xoff = 0;
    gd.own_lo = 0;
    gd.own_hi = e[0];
    gd.gex = e[0];
    gd.cells = dalloc<Cell>(C);
    gd.fW = make_fastdiv(static_cast<uint32_t>(gd.W));
    gd.fey = make_fastdiv(static_cast<uint32_t>(e[1]));
    gd.fez = make_fastdiv(static_cast<uint32_t>(e[2]));
    gd.bnx = (e[0] + 3) / 4;
    gd.bny = (e[1] + 3) / 4;
    gd.bnz = (e[2] + 3) / 4;
    gd.nbricks = static_cast<uint64_t>(gd.bnx) * gd.bny * gd.bnz;
    if (gd.nbricks * 64 >= 0xffffffffull) fail(VP_EINVAL, "VoxelGrid: more than 2^32 cells per grid (use slabs)");
    gd.clr = dalloc<uint32_t>(gd.nwords);
    gd.clrb = dalloc<unsigned long long>(gd.nbricks);
    gd.ordmap = dalloc<int32_t>(C);
    gd.stbits = dalloc<uint32_t>(gd.nwords);
    gd.rowcnt = dalloc<uint32_t>(static_cast<uint64_t>(e[0]) * e[1]);
    occ[0] = dalloc<uint32_t>(gd.nwords);
    ck(cudaMemsetAsync(gd.rowcnt, 0, static_cast<uint64_t>(e[0]) * e[1] * 4, stream), "memset rowcnt");
    ck(cudaMemsetAsync(gd.cells, 0, C * sizeof(Cell), stream), "memset cells");
    ck(cudaMemsetAsync(gd.clr, 0, gd.nwords * 4, stream), "memset clr");
    ck(cudaMemsetAsync(gd.clrb, 0, gd.nbricks * 8, stream), "memset clrb");
    ck(cudaMemsetAsync(occ[0], 0, gd.nwords * 4, stream), "memset occ");
    ck(cudaMemsetAsync(gd.ordmap, 0xff, C * 4, stream), "memset ordmap");
    ck(cudaMemsetAsync(gd.stbits, 0, gd.nwords * 4, stream), "memset stbits");
    for (int q = 0; q < kSlots; ++q) {
      ctr_s[q] = dalloc<Counters>(1);
      ck(cudaMemsetAsync(ctr_s[q], 0, sizeof(Counters), stream), "memset ctr");
      d_fp_s[q] = dalloc<FrameParams>(1);
      ck(cudaMallocHost(&h_ctr_s[q], sizeof(Counters)), "pinned");
      ck(cudaMallocHost(&h_fp_s[q], sizeof(FrameParams)), "pinned");
      std::memset(h_fp_s[q], 0, sizeof(FrameParams));
      std::memset(h_ctr_s[q], 0, sizeof(Counters));
    }
    occ_total = dalloc<unsigned long long>(1);
    ck(cudaMemsetAsync(occ_total, 0, 8, stream), "memset occ");
    set_slot(0);
    const uint32_t vcap = static_cast<uint32_t>(std::min<uint64_t>(C, 1u << 22));
    seg.ensure(vcap, vcap, vcap, 100, gd.nwords);
    ck(cudaFuncSetAttribute(k_poly_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, kPolySmem), "smem attr");
    ck(cudaFuncSetAttribute(k_poly_hull, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            kHullSmem * 16 * 6), "smem attr");
    ck(cudaFuncSetAttribute(k_integrate_fold_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, kDenseSmem),
       "smem attr");
    ck(cudaStreamSynchronize(stream), "init sync");
  }

  // Slab of a window with global extent ge centred on c, owning window x in
  // [xb, xe): local storage [xb - 1, xe + 1) (one halo plane per side).
  void init_slab(double res, const int32_t* ge, const double* c, int32_t xb, int32_t xe, int dev) {
    if (!(res > 0.0) || ge[0] <= 0 || ge[1] <= 0 || ge[2] <= 0 || xb < 0 || xe > ge[0] || xb >= xe)
      fail(VP_EINVAL, "slab: bad window or x range");
    const int32_t le[3] = {xe - xb + 2, ge[1], ge[2]};
    init(res, le, c, dev);
    origin[0] = c[0] - static_cast<double>(ge[0]) * (0.5 * res);  // the window's origin
    gd.xoff = xb - 1;
    gd.own_lo = 1;
    gd.own_hi = 1 + (xe - xb);
    gd.gex = ge[0];
  }

  MapDesc window_map() {
    const uint64_t C = static_cast<uint64_t>(gd.gex) * gd.ey * gd.ez;
    const uint64_t nw = static_cast<uint64_t>(gd.gex) * gd.ey * gd.W;
    if (!gmap) {
      gmap = dalloc<int32_t>(C);
      gbits = dalloc<uint32_t>(nw);
      ck(cudaMemsetAsync(gmap, 0xff, C * 4, stream), "gmap");
      ck(cudaMemsetAsync(gbits, 0, nw * 4, stream), "gbits");
    }
    MapDesc m{};
    m.map = gmap;
    m.bits = gbits;
    m.lo[0] = m.lo[1] = m.lo[2] = 0;
    m.dims[0] = gd.gex;
    m.dims[1] = gd.ey;
    m.dims[2] = gd.ez;
    m.W = gd.W;
    return m;
  }

  // Back to an empty window centred on c (VoxelGrid constructor state): zero
  // the occupied cells (bitmap-guided, O(occupied)) and the bitmaps.
  void reset(const double* c) {
    fill_static_params();
    h_fp->n = 0;
    // drop everything: a shift larger than the window zeroes every occupied cell
    for (int k = 0; k < 3; ++k) h_fp->shift[k] = ext[k] + 1;
    h_fp->do_shift = 1;
    upload_params();
    reset_frame_counters();
    launch_recenter();
    ck(cudaMemsetAsync(occ[0], 0, gd.nwords * 4, stream), "occ");
    ck(cudaMemsetAsync(gd.rowcnt, 0, static_cast<uint64_t>(gd.ex) * gd.ey * 4, stream), "rowcnt");
    for (int q = 0; q < kSlots; ++q) ck(cudaMemsetAsync(ctr_s[q], 0, sizeof(Counters), stream), "ctr");
    ck(cudaMemsetAsync(occ_total, 0, 8, stream), "occ total");
    ck(cudaStreamSynchronize(stream), "reset sync");
    cur = 0;
    zb = 0;
    host_occupied = 0;
    for (int k = 0; k < 3; ++k) {
      off[k] = 0;
      origin[k] = c[k] - static_cast<double>(ext[k]) * (0.5 * gd.res);
    }
  }

  // Segmentation context of pipeline slot s (scratch, ordinal map, stream).
  void use_seg(int s) {
    if (s == seg_slot) return;
    std::swap(seg, seg_pool[seg_slot]);  // park the active context
    std::swap(gd.ordmap, ordmap_pool[seg_slot]);
    std::swap(gd.stbits, stbits_pool[seg_slot]);
    std::swap(stream, stream_pool[seg_slot]);
    std::swap(seg, seg_pool[s]);  // activate s
    std::swap(gd.ordmap, ordmap_pool[s]);
    std::swap(gd.stbits, stbits_pool[s]);
    std::swap(stream, stream_pool[s]);
    seg_slot = s;
  }
  // Contexts 1 .. n-1 with context 0's capacities (call with context 0
  // active). Every context holds a window-sized ordinal map, so on a large
  // window the device may not fit n of them: contexts that cannot be
  // allocated are released and the number that exist is returned (>= 1;
  // a pipelined run then keeps that many frames in flight).
  int ensure_contexts(int n, int iterations) {
    for (int q = 1; q < n; ++q) {
      try {
        if (!ordmap_pool[q]) {
          if (!stream_pool[q]) ck(cudaStreamCreateWithFlags(&stream_pool[q], cudaStreamNonBlocking), "stream");
          const uint64_t C = gd.ncells;
          ordmap_pool[q] = dalloc<int32_t>(C);
          stbits_pool[q] = dalloc<uint32_t>(gd.nwords);
          ck(cudaMemsetAsync(ordmap_pool[q], 0xff, C * 4, stream_pool[q]), "memset ordmap");
          ck(cudaMemsetAsync(stbits_pool[q], 0, gd.nwords * 4, stream_pool[q]), "memset stbits");
        }
        Seg& a = seg_pool[q];
        a.ensure(std::max(a.b.Vcap, seg.b.Vcap), std::max(a.b.Scap, seg.b.Scap), std::max(a.b.Icap, seg.b.Icap),
                 iterations, gd.nwords);
        a.ensure_dirs(16, stream_pool[q]);
        ck(cudaStreamSynchronize(stream_pool[q]), "sync");
      } catch (const VpFail& e) {
        if (e.code != VP_ENOMEM) throw;
        for (int r = q; r < kSlots; ++r) release_context(r);
        return q;
      }
    }
    return n;
  }
  // Give back the device memory of (inactive) context q.
  void release_context(int q) {
    if (q == seg_slot || q == 0) return;
    if (stream_pool[q]) cudaStreamSynchronize(stream_pool[q]);
    seg_pool[q].release();
    dfree(ordmap_pool[q]);
    dfree(stbits_pool[q]);
  }
  void set_slot(int s) {
    slot = s;
    ctr = ctr_s[s];
    h_ctr = h_ctr_s[s];
    d_fp = d_fp_s[s];
    h_fp = h_fp_s[s];
    d_pts = d_pts_s[s];
  }

  void ensure_points(uint64_t n) {
    if (n <= pcap && d_pts_s[0]) return;
    uint64_t cap = std::max<uint64_t>(n, 1 << 16);
    cap = std::max<uint64_t>(cap, pcap * 2);
    ck(cudaDeviceSynchronize(), "sync before realloc");
    for (void* p : {(void*)hkey, (void*)hcnt, (void*)hoff, (void*)groups, (void*)pslot, (void*)prank,
                    (void*)sorted, (void*)dense, (void*)medium, (void*)rperm, (void*)bin_of})
      if (p) cudaFree(p);
    for (auto*& p : d_pts_s) dfree(p);
    uint64_t hs = 1;
    while (hs < 2 * cap) hs <<= 1;
    for (auto*& p : d_pts_s) p = dalloc<float>(3 * cap);
    d_pts = d_pts_s[slot];
    hkey = dalloc<uint32_t>(hs);
    hcnt = dalloc<uint32_t>(hs);
    hoff = dalloc<uint32_t>(hs);
    groups = dalloc<uint32_t>(cap);
    pslot = dalloc<uint32_t>(cap);
    prank = dalloc<uint32_t>(cap);
    sorted = dalloc<uint32_t>(cap);
    dense = dalloc<uint32_t>(cap / (kFoldMax + 1) + 1);
    medium = dalloc<uint32_t>(cap / (kFoldSmall + 1) + 1);
    rperm = dalloc<uint32_t>(cap);
    bin_of = dalloc<uint8_t>(cap);
    if (!dbins) {
      dbins = dalloc<DdaBins>(1);
      ck(cudaMemsetAsync(dbins, 0, sizeof(DdaBins), stream), "dbins");
    }
    ck(cudaMemsetAsync(hkey, 0xff, hs * 4, stream), "hkey");
    ck(cudaMemsetAsync(hcnt, 0, hs * 4, stream), "hcnt");
    hmask = static_cast<uint32_t>(hs - 1);
    pcap = cap;
    ++gen;
  }

  // ------------------------------------------------------------ frame params
  void set_pose(const double* R, const double* t) {
    std::memcpy(h_fp->R, R, 9 * sizeof(double));
    std::memcpy(h_fp->t, t, 3 * sizeof(double));
  }
  void fill_static_params() {
    for (int k = 0; k < 3; ++k) {
      h_fp->origin_pre[k] = h_fp->origin_post[k] = origin[k];
      h_fp->off_pre[k] = h_fp->off_post[k] = off[k];
      h_fp->shift[k] = 0;
    }
    h_fp->do_shift = 0;
    h_fp->occ_pre = h_fp->occ_post = occ[0];
    h_fp->zb_pre = h_fp->zb_post = zb;
  }
  // Host part of recenter (voxel_grid.cpp:217-223) -> post-shift state.
  bool plan_recenter(const double* c, vp_shift_stats* st) {
    const double res = gd.res;
    if (gd.gex != gd.ex || gd.xoff != 0) {
      // slab windows are fixed; a shift would move cells between ranks
      for (int k = 0; k < 3; ++k) {
        const double wc = origin[k] + static_cast<double>(k == 0 ? gd.gex : ext[k]) * (0.5 * res);
        if (std::llround((c[k] - wc) / res) != 0) fail(VP_EINVAL, "recenter: slab windows are fixed");
      }
      if (st) std::memset(st, 0, sizeof *st);
      return false;
    }
    int32_t s[3];
    for (int k = 0; k < 3; ++k) {
      const double wc = origin[k] + static_cast<double>(ext[k]) * (0.5 * res);  // world_center
      s[k] = static_cast<int32_t>(std::llround((c[k] - wc) / res));
    }
    if (st) {
      std::memcpy(st->shift, s, sizeof s);
      st->voxels_dropped = 0;
    }
    if (s[0] == 0 && s[1] == 0 && s[2] == 0) return false;
    for (int k = 0; k < 3; ++k) {
      origin[k] += static_cast<double>(s[k]) * res;
      int64_t o = (static_cast<int64_t>(off[k]) + s[k]) % ext[k];
      if (o < 0) o += ext[k];
      off[k] = static_cast<int32_t>(o);
      h_fp->origin_post[k] = origin[k];
      h_fp->off_post[k] = off[k];
      h_fp->shift[k] = s[k];
    }
    {  // the occupancy ring's z offset moves with the window (mod W * 32)
      const int64_t wz = static_cast<int64_t>(gd.W) * 32;
      int64_t o = (static_cast<int64_t>(zb) + s[2]) % wz;
      if (o < 0) o += wz;
      zb = static_cast<int32_t>(o);
      h_fp->zb_post = zb;
    }
    h_fp->do_shift = 1;
    return true;
  }
  void upload_params() {
    ck(cudaMemcpyAsync(d_fp, h_fp, sizeof(FrameParams), cudaMemcpyHostToDevice, lstream), "params");
  }
  // zero the slot's counters; occupied <- the persistent total
  void reset_frame_counters() { LAUNCH(k_frame_begin, 1, 32, 0, lstream, ctr, occ_total); }
  void read_counters() {
    ck(cudaMemcpyAsync(h_ctr, ctr, sizeof(Counters), cudaMemcpyDeviceToHost, stream), "ctr d2h");
    ck(cudaStreamSynchronize(stream), "sync");
    host_occupied = h_ctr->occupied;
  }

  // ------------------------------------------------------------ kernels
  // Grids are sized by the points capacity (grid-stride loops read n from
  // the device params), so the same launches can be replayed as a graph.
  void launch_clear(uint64_t n) {
    launch_clear_walk(n);
    launch_clear_apply(n, 0);
  }
  // clear_rays, first half: the DDA walks mark the clear masks (reads only
  // the points, the pose and the pre-recenter window; touches no cell)
  void launch_clear_walk(uint64_t n) {
    if (n == 0 && !capturing) return;
    const int gp = grid_for(capturing ? pcap : n);
    LAUNCH(k_dda_keys, gp, kThreads, 0, lstream, gd, d_fp, dbins, bin_of);
    // a window mask beyond L2 (C5: 150 MB): one row-layout RED per cell is a
    // DRAM round trip, the brick walk issues one per brick (C5 walk 1.5 ->
    // 0.85 ms; C2-C4 windows keep the lane-balance rule: C2 83 vs 200 us)
    const uint64_t mask_bytes = static_cast<uint64_t>(gd.gex) * gd.ey * gd.ez / 8;
    const int long_steps = g_dda_long >= 0 ? g_dda_long : (mask_bytes > kDdaL2Mask ? 128 : 0);
    LAUNCH(k_dda_plan, 1, 32, 0, lstream, dbins, g_dda_force, long_steps);
    LAUNCH(k_dda_scatter, gp, kThreads, 0, lstream, d_fp, dbins, bin_of, rperm);
    if (gd.xoff != 0 || gd.gex != gd.ex)
      LAUNCH(k_clear_walk_slab, grid_for(capturing ? pcap : n, 148 * 32), kThreads, 0, lstream, gd, d_fp, rperm,
             dbins);
    else
      LAUNCH(k_clear_walk, grid_for(capturing ? pcap : n, 148 * 32), kThreads, 0, lstream, gd, d_fp, rperm, dbins,
             g_walk_generic);
  }
  // second half: the marked cells are cleared (and the masks zeroed)
  // use_box: sweep only the box k_integrate_hash measured for this frame (the
  // mapping path), else the whole mask (clear_rays alone)
  void launch_clear_apply(uint64_t n, int use_box) {
    if (n == 0 && !capturing) return;
    // 148 x 4 blocks, grid-stride over the box, four mask loads in flight per
    // thread; one counter atomic per block
    LAUNCH(k_clear_apply, std::min<int>(148 * 4, grid_for(std::max<uint64_t>(gd.nwords, gd.nbricks))), kThreads, 0,
           lstream, gd, d_fp, ctr, dbins, use_box);
  }
  void launch_integrate(uint64_t n) {
    launch_integrate_group(n, lstream);
    launch_integrate_fold(n);
  }
  // grouping of the points by voxel (reads only the points): independent of clear_rays
  void launch_integrate_group(uint64_t n, cudaStream_t st) {
    if (n == 0 && !capturing) return;
    const int gp = grid_for(capturing ? pcap : n);
    LAUNCH(k_integrate_hash, gp, kThreads, 0, st, gd, d_fp, ctr, hkey, hcnt, hmask, groups, pslot, prank);
    LAUNCH(k_integrate_offsets, gp, kThreads, 0, st, ctr, groups, hcnt, hoff, medium, dense);
    LAUNCH(k_integrate_scatter, gp, kThreads, 0, st, d_fp, pslot, prank, hoff, sorted);
  }
  // the ordered fold into the cells: after clear_rays (voxel_grid order);
  // the thread, warp and block passes touch disjoint voxels: the larger
  // groups are folded on the fork stream beside the thread pass
  void launch_integrate_fold(uint64_t n) {
    if (n == 0 && !capturing) return;
    const int gp = grid_for(capturing ? pcap : n);
    ck(cudaEventRecord(fork_ev[2], lstream), "fork");
    ck(cudaStreamWaitEvent(fstream, fork_ev[2], 0), "fork");
    LAUNCH(k_integrate_fold_medium, 148 * 4, kThreads, 0, fstream, gd, d_fp, ctr, hkey, hcnt, hoff, sorted,
           medium);
    LAUNCH(k_integrate_fold_dense, 148, 1024, kDenseSmem, fstream, gd, d_fp, ctr, hkey, hcnt, hoff, sorted,
           pslot, dense);
    ck(cudaEventRecord(fork_ev[3], fstream), "join");
    LAUNCH(k_integrate_fold, gp, kThreads, 0, lstream, gd, d_fp, ctr, groups, hkey, hcnt, hoff, sorted);
    ck(cudaStreamWaitEvent(lstream, fork_ev[3], 0), "join");
  }
  // finalize: the last block also does k_map_finalize's bookkeeping
  void launch_recenter(bool finalize = false) {
    LAUNCH(k_recenter, grid_for(static_cast<uint64_t>(gd.ex) * gd.ey), kThreads, 0, lstream, gd, d_fp, ctr,
           finalize ? occ_total : nullptr);
  }
  void launch_finalize() { LAUNCH(k_map_finalize, 1, 1, 0, lstream, ctr, occ_total); }
  // clear_rays and the grouping half of integrate_frame in parallel (fork
  // onto fstream, join before the ordered fold), then recenter, finalize.
  void launch_mapping_forked(uint64_t n) {
    launch_mapping_pre(n);
    launch_mapping_post(n);
  }
  // The half of the mapping that touches no cell (DDA walks || grouping):
  // in a pipelined run it overlaps the previous frame's grid readers.
  void launch_mapping_pre(uint64_t n) {
    ck(cudaEventRecord(fork_ev[0], lstream), "fork");
    ck(cudaStreamWaitEvent(fstream, fork_ev[0], 0), "fork");
    launch_integrate_group(n, fstream);
    ck(cudaEventRecord(fork_ev[1], fstream), "join");
    launch_clear_walk(n);
    ck(cudaStreamWaitEvent(lstream, fork_ev[1], 0), "join");
  }
  // the half that updates the cells: clear, ordered fold, recenter
  void launch_mapping_post(uint64_t n) {
    launch_clear_apply(n, 1);
    launch_integrate_fold(n);
    launch_recenter(true);  // + finalize
  }

  // Occupied scan of the post-recenter bitmap into seg.b.occ_list; ctr->V.
  void launch_occupied_scan() {
    // over the owned logical rows (x, y): row counts, then the non-empty rows
    const uint64_t r_lo = static_cast<uint64_t>(gd.own_lo) * gd.ey;
    const uint64_t r_n = static_cast<uint64_t>(gd.own_hi - gd.own_lo) * gd.ey;
    const uint32_t nb = static_cast<uint32_t>((r_n + kRowsPerBlock - 1) / kRowsPerBlock);
    LAUNCH(k_bitmap_count, nb, kScanThreads, 0, stream, gd, d_fp, r_lo, r_n, seg.bsum, ctr);  // + scan
    LAUNCH(k_bitmap_emit, nb, kScanThreads, 0, stream, gd, d_fp, r_lo, r_n, seg.bsum, seg.b.occ_list,
           seg.b.Vcap);
  }

  // flags[0..*n) -> positions, total into *total
  void launch_flag_scan(const uint8_t* flags, const uint32_t* n_ptr, uint32_t cap, uint32_t* pos,
                        uint32_t* total) {
    const uint32_t nb = (cap + kScanPerBlock - 1) / kScanPerBlock;
    uint32_t* bs = seg.bsum + 2ull * seg.bsum_cap;
    LAUNCH(k_flags_count, nb, kScanThreads, 0, stream, flags, n_ptr, cap, bs, total, &ctr->scan_done[2]);  // + scan
    LAUNCH(k_flags_positions, nb, kScanThreads, 0, stream, flags, n_ptr, cap, bs, pos);
  }

  MapDesc grid_map() {
    MapDesc m;
    m.map = gd.ordmap;
    m.bits = gd.stbits;
    m.W = gd.W;
    m.lo[0] = m.lo[1] = m.lo[2] = 0;
    m.dims[0] = ext[0];
    m.dims[1] = ext[1];
    m.dims[2] = ext[2];
    return m;
  }

  // normals + classify + steppable list (+ ordinal map)
  // normals + classify (steppable counts per kThreads-voxel tile, scanned:
  // the tile offsets and ctr->S)
  void launch_classify(const SegDev& sd, int write_status) {
    uint32_t* ts = seg.bsum + seg.bsum_cap;
    LAUNCH(k_normals, kWide, kThreads, 0, stream, gd, d_fp, ctr, sd, seg.b, write_status, ts);  // + tile scan
  }
  // the steppable list at the ordinals of launch_classify's tile offsets
  void launch_step_emit(const MapDesc& m, int xadd = 0) {
    LAUNCH(k_step_emit, kWide, kThreads, 0, stream, gd, ctr, seg.b, m, xadd, seg.bsum + seg.bsum_cap);
  }
  // union-find over the steppable list in seg.b (ctr->S set)
  void launch_ccl(const SegDev& sd, const MapDesc& m) { launch_ccl(sd, m, seg.b); }
  void launch_ccl(const SegDev& sd, const MapDesc& m, const SegBufs& sb) {
    if (g_ccl_mode == 0) {
      // ECL-style atomic-free pre-hooking + compression: most unions then end at
      // the one-load parent check (C2: union pass 400 us -> 80 us); candidates
      // listed per warp and spread over the lanes (k_ccl_*_bal)
      LAUNCH(k_ccl_hook_bal, chain_wide, 256, 0, stream, ctr, sd, sb, m);
      if (g_ccl_jumps & 1) LAUNCH(k_ccl_jump, chain_wide, kThreads, 0, stream, ctr, sb);
      if (g_ccl_jumps & 2) LAUNCH(k_ccl_jump, chain_wide, kThreads, 0, stream, ctr, sb);
      LAUNCH(k_ccl_compress_exact, chain_wide, kThreads, 0, stream, ctr, sb);
      // cross-tree edges as a root-pair set, unioned by one block (which runs
      // the full edge-balanced union instead if the set overflowed)
      LAUNCH(k_ccl_pairs, chain_wide, 256, 0, stream, ctr, sd, sb, m);
      LAUNCH(k_ccl_pairs_union, 1, 256, 0, stream, ctr, sd, sb, m);
    } else if (g_ccl_mode == 4) {
      // hook + compression + edge-balanced unions of every forward edge
      LAUNCH(k_ccl_hook_bal, chain_wide, 256, 0, stream, ctr, sd, sb, m);
      LAUNCH(k_ccl_jump, chain_wide, kThreads, 0, stream, ctr, sb);
      LAUNCH(k_ccl_jump, chain_wide, kThreads, 0, stream, ctr, sb);
      LAUNCH(k_ccl_compress, chain_wide, kThreads, 0, stream, ctr, sb);
      LAUNCH(k_ccl_union_bal, chain_wide, 256, 0, stream, ctr, sd, sb, m);
    } else if (g_ccl_mode == 3) {
      // the same with one window row per lane (round-1 kernels, A/B)
      LAUNCH(k_ccl_hook, chain_wide, kThreads, 0, stream, ctr, sd, sb, m);
      LAUNCH(k_ccl_compress, chain_wide, kThreads, 0, stream, ctr, sb);
      LAUNCH(k_ccl_union, chain_wide, kThreads, 0, stream, ctr, sd, sb, m);
    } else {
      // sampling variants (measured slower on C2 and C5):
      // 1 = neighbour-sampling unions, 2 = min-neighbour hooking; then
      // whole-window unions of the voxels outside the sampled giant tree
      if (g_ccl_mode == 1) {
        LAUNCH(k_ccl_init, chain_wide, kThreads, 0, stream, ctr, sb);
        LAUNCH(k_ccl_lattice, chain_wide, kThreads, 0, stream, ctr, sd, sb, m);
      } else {
        LAUNCH(k_ccl_hook, chain_wide, kThreads, 0, stream, ctr, sd, sb, m);
      }
      LAUNCH(k_ccl_compress, chain_wide, kThreads, 0, stream, ctr, sb);
      LAUNCH(k_ccl_giant, 1, 1024, 0, stream, ctr, sb);
      LAUNCH(k_ccl_full, chain_wide, kThreads, 0, stream, ctr, sd, sb, m);
    }
    LAUNCH(k_ccl_flatten, chain_wide, kThreads, 0, stream, ctr, sb, m);
  }
  // label_base: global ordinal of list entry 0 (slab owners), else 0
  void launch_clusters(const SegDev& sd, int64_t label_base = 0) {
    LAUNCH(k_cluster_flags, chain_wide, kThreads, 0, stream, ctr, sd, seg.b);
    launch_flag_scan(seg.b.big_flag, &ctr->S, seg.b.Scap, seg.b.big_pos, &ctr->K);
    LAUNCH(k_cluster_assign, chain_wide, kThreads, 0, stream, ctr, seg.b);  // + cluster setup (last block)
    if (label_base) LAUNCH(k_klabel_rebase, 8, 256, 0, stream, ctr, seg.b, label_base);
    const int nch = static_cast<int>(seg.hstride);
    LAUNCH(k_member_hist, std::min(nch, 148 * 16), 32, 0, stream, ctr, seg.b, seg.hstride);
    LAUNCH(k_member_hscan, chain_wide, kThreads, 0, stream, ctr, seg.b, seg.hstride);
    LAUNCH(k_member_scatter, std::min(nch, 148 * 16), 32, 0, stream, ctr, seg.b, seg.hstride);
  }
  void launch_ransac(const RansacDev& rd) { launch_ransac(rd, ctr, seg.b); }
  // fit_planes on the clusters described by b (counters c): the same kernels
  // serve the cluster-parallel pass and, with single-cluster views, the
  // per-cluster-serial execution mode (plane_fit.cpp:107-119)
  void launch_ransac(const RansacDev& rd, Counters* c, const SegBufs& b) {
    LAUNCH(k_ransac_hyp, chain_wide, kThreads, 0, stream, c, rd, b);
    LAUNCH(k_ransac_count, chain_wide, kThreads, 0, stream, c, rd, b);
    LAUNCH(k_ransac_select, chain_wide, kThreads, 0, stream, c, rd, b);  // + fit setup (last block)
    LAUNCH(k_extract_count, chain_wide, kThreads, 0, stream, c, rd, b);
    LAUNCH(k_scan_exclusive, 1, 1024, 0, stream, b.ccount, 0u, &c->fit_chunks, nullptr, nullptr);
    LAUNCH(k_extract_emit, chain_wide, kThreads, 0, stream, c, rd, b);
  }
  void launch_refine(const double* up, int refine, int exact) {
    const d3 u{up[0], up[1], up[2]};
    if (exact) {
      LAUNCH(k_refine, 148 * 2, 32, 0, stream, ctr, seg.b, u, refine, exact);
      return;
    }
    LAUNCH(k_refine_setup, 1, 1024, 0, stream, ctr, seg.b, refine);
    LAUNCH(k_refine_part0, 148 * 4, 256, 0, stream, ctr, seg.b);     // + centroids (last block)
    LAUNCH(k_refine_part1, 148 * 4, 256, 0, stream, ctr, seg.b, u);  // + covariance, Jacobi, model
  }
  // make_polygon for every fit: one 4-CTA cluster per fit (k_poly_fused),
  // after the passes over the inliers of the fits above kPolyBig on the whole
  // GPU (VP_POLY_SPLIT=1: the five-kernel form setup/extremes/inner/keep/hull)
  void launch_polygon(int dirs, double min_area, int planar = 0) {
    seg.ensure_dirs(dirs, stream);
    if (!g_poly_split) {
      // the large fits' projection / extremes / keep test over the whole GPU
      LAUNCH(k_poly_wide_ext, 148 * 4, 256, 0, stream, ctr, seg.b, seg.dirtab, dirs, planar);
      LAUNCH(k_poly_wide_keep, 148 * 4, 256, 0, stream, ctr, seg.b);
      const int clusters = chain_wide >= 148 * 8 ? 32 : 16;
      LAUNCH(k_poly_fused, clusters * kPolyCluster, kPolyThreads, kPolySmem, stream, ctr, seg.b, seg.dirtab, dirs,
             planar, min_area);
      return;
    }
    LAUNCH(k_poly_setup, 1, 1024, 0, stream, ctr, seg.b);
    LAUNCH(k_poly_extremes, chain_wide, 256, 0, stream, ctr, seg.b, seg.dirtab, dirs, planar);
    LAUNCH(k_poly_inner, 148 * 2, 64, 0, stream, ctr, seg.b, dirs);
    LAUNCH(k_poly_keep, chain_wide, 256, 0, stream, ctr, seg.b);
    LAUNCH(k_poly_hull, 148, 256, kHullSmem * 16 * 6, stream, ctr, seg.b, min_area);
  }

  // The fused segment(): voxel_frame_polygons (pipeline.cpp:43-85) on device.
  void record(cudaEvent_t e) {
    ck(cudaEventRecordWithFlags(e, stream, capturing ? cudaEventRecordExternal : cudaEventRecordDefault),
       "event record");
  }

  // voxel_frame_polygons up to filter_clusters: everything that can overflow
  // a capacity, and the last stage that reads the grid cells.
  void launch_seg_a(const vp_pipeline_params& p, bool timing) {
    launch_seg_a1(p, timing);
    launch_seg_a2(p, timing);
  }
  // occupied_voxels .. classify_steppable + ordinal map: the last stage that
  // reads the grid (cells, occupancy) -- everything that can overflow
  // with_step_emit = false: the steppable list / ordinal map are left to the
  // caller (the pipelined run enqueues them with the chain, off the mapping
  // stream: they read only this context's lists)
  void launch_seg_a1(const vp_pipeline_params& p, bool timing, bool with_step_emit = true) {
    const SegDev sd = make_segdev(p.seg, gd.res);
    if (!capturing && static_cast<uint64_t>(p.ransac.iterations) * seg.kcap > seg.cand_cap)
      seg.ensure(seg.b.Vcap, seg.b.Scap, seg.b.Icap, p.ransac.iterations, gd.nwords);
    if (timing) record(ev[1]);
    launch_occupied_scan();
    launch_classify(sd, 1);
    if (timing) record(ev[2]);
    if (with_step_emit) launch_step_emit(grid_map());
  }
  // build_adjacency + label_components + filter_clusters: steppable list and
  // ordinal map only (cannot overflow: members <= S + 31 K < Mcap)
  void launch_seg_a2(const vp_pipeline_params& p, bool timing) {
    const SegDev sd = make_segdev(p.seg, gd.res);
    launch_ccl(sd, grid_map());
    launch_clusters(sd);
    if (timing) record(ev[3]);
  }
  // fit_planes .. make_polygon: reads only the cluster buffers
  void launch_seg_b(const vp_pipeline_params& p, bool timing) {
    const RansacDev rd = make_ransacdev(p.ransac);
    launch_ransac(rd);
    if (timing) record(ev[4]);
    launch_refine(p.ransac.up, p.refine, p.refine_exact);
    launch_polygon(16, p.min_polygon_area);
    if (timing) record(ev[5]);
  }
  void launch_segment(const vp_pipeline_params& p, bool timing) {
    launch_seg_a(p, timing);
    launch_seg_b(p, timing);
  }

  // Grow capacities after an overflow (the frame's segmentation is re-run).
  bool grow_if_overflow(int iterations) {
    const uint32_t of = h_ctr->overflow;
    if (!of) return false;
    if (of & kOverflowClusters) {  // more clusters: only the cluster-sized buffers grow
      seg.grow_k(h_ctr->K, h_ctr->S, iterations);
      if (of == kOverflowClusters) return true;
    }
    uint32_t vcap = seg.b.Vcap, scap = seg.b.Scap, icap = seg.b.Icap;
    const uint64_t C = gd.ncells;
    if (of & kOverflowOcc) vcap = static_cast<uint32_t>(std::min<uint64_t>(C, std::max<uint64_t>(2ull * vcap, h_ctr->V)));
    if (of & (kOverflowStep | kOverflowOcc)) scap = std::max(scap, std::min<uint32_t>(vcap, std::max(2 * scap, h_ctr->S)));
    if (of & kOverflowMembers) scap = std::min<uint32_t>(static_cast<uint32_t>(std::min<uint64_t>(C, 4ull * scap)), std::max(2 * scap, h_ctr->padded_members));
    if (of & (kOverflowFits | kOverflowPool)) icap = std::max(2 * icap, scap);
    seg.ensure(std::max(vcap, seg.b.Vcap), std::max(scap, seg.b.Scap), std::max(icap, seg.b.Icap),
               iterations, gd.nwords);
    return true;
  }

  // Grow the buffers the CCL .. polygon chain writes after it overflowed,
  // keeping the grid readers' outputs (occupied and steppable lists) intact.
  void grow_chain(int iterations) {
    if (h_ctr->overflow & ~kOverflowClusters) fail(VP_ENOMEM, "segmentation chain capacity overflow");
    seg.grow_k(h_ctr->K, h_ctr->S, iterations);  // keeps the steppable list the chain re-runs from
  }

  // Download polygon records of the last segment() into host vectors.
  void download_polygons(HostPolys& hp, bool keep_nullopt) {
    const uint32_t F = h_ctr->nfits;
    std::vector<double> rd(8ull * F);
    std::vector<int32_t> ri(4ull * F);
    if (F) {
      ck(cudaMemcpyAsync(rd.data(), seg.b.prec_d, rd.size() * 8, cudaMemcpyDeviceToHost, stream), "prec");
      ck(cudaMemcpyAsync(ri.data(), seg.b.prec_i, ri.size() * 4, cudaMemcpyDeviceToHost, stream), "prec");
    }
    const uint32_t pu = h_ctr->pool_used;
    hp.verts.resize(5ull * pu);
    if (pu)
      ck(cudaMemcpyAsync(hp.verts.data(), seg.b.pool, hp.verts.size() * 8, cudaMemcpyDeviceToHost,
                         stream), "pool");
    ck(cudaStreamSynchronize(stream), "sync");
    hp.polys.clear();
    for (uint32_t f = 0; f < F; ++f) {
      const int32_t nv = ri[4 * f + 2];
      if (nv <= 0 && !keep_nullopt) continue;
      vp_polygon q{};
      q.plane.normal[0] = rd[8 * f];
      q.plane.normal[1] = rd[8 * f + 1];
      q.plane.normal[2] = rd[8 * f + 2];
      q.plane.offset = rd[8 * f + 3];
      q.plane.inlier_count = ri[4 * f];
      q.plane.cluster_label = ri[4 * f + 1];
      q.nverts = nv > 0 ? static_cast<uint32_t>(nv) : 0u;
      q.area = rd[8 * f + 4];
      // stash the pool offset in v2d temporarily
      q.v2d = reinterpret_cast<const double*>(static_cast<uintptr_t>(ri[4 * f + 3]));
      hp.polys.push_back(q);
    }
  }
};

namespace {

vp_polygons_t* make_polygons_out(const HostPolys& hp) {
  size_t nv = 0;
  for (const auto& q : hp.polys) nv += q.nverts;
  const size_t bytes = sizeof(vp_polygons_t) + hp.polys.size() * sizeof(vp_polygon) + nv * 5 * sizeof(double);
  char* mem = static_cast<char*>(std::malloc(bytes));
  if (!mem) fail(VP_ENOMEM, "host allocation");
  auto* out = reinterpret_cast<vp_polygons_t*>(mem);
  out->count = hp.polys.size();
  out->polys = reinterpret_cast<vp_polygon*>(mem + sizeof(vp_polygons_t));
  double* vbase = reinterpret_cast<double*>(mem + sizeof(vp_polygons_t) + hp.polys.size() * sizeof(vp_polygon));
  for (size_t i = 0; i < hp.polys.size(); ++i) {
    vp_polygon q = hp.polys[i];
    const size_t voff = static_cast<size_t>(reinterpret_cast<uintptr_t>(q.v2d));
    double* v2 = vbase;
    double* v3 = vbase + 2 * q.nverts;
    for (uint32_t k = 0; k < q.nverts; ++k) {
      const double* src = hp.verts.data() + 5 * (voff + k);
      v2[2 * k] = src[0];
      v2[2 * k + 1] = src[1];
      v3[3 * k] = src[2];
      v3[3 * k + 1] = src[3];
      v3[3 * k + 2] = src[4];
    }
    q.v2d = q.nverts ? v2 : nullptr;
    q.v3d = q.nverts ? v3 : nullptr;
    vbase += 5 * q.nverts;
    out->polys[i] = q;
  }
  return out;
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return VP_OK;
  } catch (const VpFail& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return VP_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VP_ECUDA;
  }
}

// ------------------------------------------------------------- frame steps
// pipeline.cpp:37-41
void global_cell(const double* t, double res, int32_t* c) {
  for (int k = 0; k < 3; ++k) c[k] = static_cast<int32_t>(std::floor(t[k] / res));
}

void stage_points(vp_grid* g, const float* xyz, uint64_t n, bool device_ptr) {
  if (device_ptr) {
    g->h_fp->pts = xyz;
  } else {
    g->ensure_points(n);
    if (n)  // cudaMemcpyDefault: host (pageable or pinned) or device source
      ck(cudaMemcpyAsync(g->d_pts, xyz, n * 12, cudaMemcpyDefault, g->stream), "points h2d");
    g->h_fp->pts = g->d_pts;
  }
  g->h_fp->n = n;
}

}  // namespace

struct vp_pipeline {
  vp_grid* grid = nullptr;
  vp_pipeline_params p{};
  int32_t last_cell[3] = {0, 0, 0};
  uint32_t frame = 0;
  // one frame of work as a CUDA graph (params H2D, counter reset, every
  // kernel, stage events, counters D2H)
  cudaGraphExec_t gexec = nullptr;
  uint64_t graph_key = 0;
  uint64_t graph_kernels = 0;
  // pipelined runs: graphs per (slot, part: 0 mapping pre, 1 mapping post,
  // 2 grid readers, 3 chain)
  cudaGraphExec_t rx[kSlots][4] = {};
  uint64_t rkey[kSlots][4] = {};
  uint64_t rkern[kSlots][4] = {};
  cudaEvent_t ev_start[kSlots] = {}, ev_pre[kSlots] = {}, ev_map[kSlots] = {};
  cudaEvent_t ev_clu[kSlots] = {}, ev_ccl[kSlots] = {}, ev_rsc[kSlots] = {}, ev_done[kSlots] = {};
  cudaEvent_t ev_h2d[kSlots] = {};
  // one frame's latency (vp_pipeline_frame): points H2D start -> polygons
  // assembled in host memory
  cudaEvent_t lat_ev[2] = {nullptr, nullptr};
  float last_latency_ms = 0.0f;
  cudaStream_t cstream = nullptr;  // host-to-device copies of upcoming frames
  // every frame's polygons, packed by k_poly_pack into mapped pinned memory
  double* pack_h[kSlots] = {};
  // the single-frame path's pack (vp_pipeline_frame): no D2H round trip for the polygons
  double* pack1_h = nullptr;
  double* pack1_d = nullptr;
  double* pack_d[kSlots] = {};
  static constexpr uint64_t kPackCap = 1u << 17;  // doubles per slot (1 MiB)
  // host state of the frame occupying a slot (stage traces)
  struct SlotMeta {
    uint32_t frame = 0;
    bool rec = false;
    int32_t shift[3] = {0, 0, 0};
    double origin[3] = {0.0, 0.0, 0.0};
  } meta[kSlots];
  ~vp_pipeline() {
    for (auto e : lat_ev)
      if (e) cudaEventDestroy(e);
    if (gexec) cudaGraphExecDestroy(gexec);
    for (auto& row : rx)
      for (auto& x : row)
        if (x) cudaGraphExecDestroy(x);
    for (auto* e : {ev_start, ev_pre, ev_map, ev_clu, ev_ccl, ev_rsc, ev_done, ev_h2d})
      for (int q = 0; q < kSlots; ++q)
        if (e[q]) cudaEventDestroy(e[q]);
    if (cstream) {
      cudaStreamSynchronize(cstream);
      cudaStreamDestroy(cstream);
    }
    delete grid;  // drains the grid's streams
    if (pack1_h) cudaFreeHost(pack1_h);
    for (auto* q : pack_h)
      if (q) cudaFreeHost(q);
  }
};

namespace {

// The device work of one frame, in stream order. With capture == true the
// same sequence is recorded into a CUDA graph (every argument is frame
// invariant; per-frame values live in the device FrameParams).
void enqueue_frame_work(vp_pipeline* pl, uint64_t n) {
  vp_grid* g = pl->grid;
  const unsigned evflag = g->capturing ? cudaEventRecordExternal : cudaEventRecordDefault;
  ck(cudaMemcpyAsync(g->d_fp, g->h_fp, sizeof(FrameParams), cudaMemcpyHostToDevice, g->stream), "params");
  g->reset_frame_counters();
  ck(cudaEventRecordWithFlags(g->ev[0], g->stream, evflag), "ev");
  g->launch_mapping_forked(n);  // walks || grouping, then clear (ray box), fold, recenter
  g->launch_segment(pl->p, true);
  // the polygons straight into mapped pinned memory (read after the frame's sync)
  LAUNCH(k_poly_pack, 1, 1024, 0, g->stream, g->ctr, g->seg.b, pl->pack1_d, vp_pipeline::kPackCap);
  ck(cudaMemcpyAsync(g->h_ctr, g->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, g->stream), "ctr d2h");
}

void run_frame_graph(vp_pipeline* pl) {
  vp_grid* g = pl->grid;
  const uint64_t key = (g->gen << 32) ^ g->seg.gen;
  if (!pl->gexec || pl->graph_key != key) {
    if (pl->gexec) cudaGraphExecDestroy(pl->gexec);
    pl->gexec = nullptr;
    cudaGraph_t graph;
    const uint64_t before = g_launches.load();
    g->capturing = true;
    ck(cudaStreamBeginCapture(g->stream, cudaStreamCaptureModeThreadLocal), "capture begin");
    try {
      enqueue_frame_work(pl, g->pcap);
    } catch (...) {
      cudaStreamEndCapture(g->stream, &graph);
      g->capturing = false;
      throw;
    }
    ck(cudaStreamEndCapture(g->stream, &graph), "capture end");
    g->capturing = false;
    pl->graph_kernels = g_launches.load() - before;
    g_launches.fetch_sub(pl->graph_kernels);
    ck(cudaGraphInstantiate(&pl->gexec, graph, 0), "graph instantiate");
    cudaGraphDestroy(graph);
    pl->graph_key = key;
  }
  ck(cudaGraphLaunch(pl->gexec, g->stream), "graph launch");
  g_launches.fetch_add(pl->graph_kernels);
}

// One run_frames iteration (pipeline.cpp:199-213) through segmentation;
// returns whether the window was recentered. The caller waits on the stream.
bool pipeline_enqueue(vp_pipeline* pl, const float* xyz, uint64_t n, const double* R,
                      const double* t, bool device_ptr, vp_shift_stats* ss) {
  vp_grid* g = pl->grid;
  g->set_slot(0);
  g->lstream = g->stream;
  if (!is_valid_rotation(R))  // voxel_grid.cpp:60-61, 183-184
    fail(VP_EINVAL, "clear_rays: pose rotation is not orthonormal");
  g->ensure_points(n);
  if (static_cast<uint64_t>(pl->p.ransac.iterations) * g->seg.kcap > g->seg.cand_cap)
    g->seg.ensure(g->seg.b.Vcap, g->seg.b.Scap, g->seg.b.Icap, pl->p.ransac.iterations, g->gd.nwords);
  g->seg.ensure_dirs(16, g->stream);
  g->set_pose(R, t);
  g->fill_static_params();
  if (!pl->lat_ev[0])
    for (auto& e : pl->lat_ev) ck(cudaEventCreate(&e), "event");
  if (!pl->pack1_h) {
    ck(cudaHostAlloc(&pl->pack1_h, vp_pipeline::kPackCap * sizeof(double), cudaHostAllocMapped), "pinned");
    ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&pl->pack1_d), pl->pack1_h, 0), "mapped");
  }
  ck(cudaEventRecord(pl->lat_ev[0], g->stream), "event");  // before the points H2D
  stage_points(g, xyz, n, device_ptr);
  int32_t cell[3];
  global_cell(t, g->gd.res, cell);
  bool rec = false;
  std::memset(ss, 0, sizeof *ss);
  if (cell[0] != pl->last_cell[0] || cell[1] != pl->last_cell[1] || cell[2] != pl->last_cell[2]) {
    g->plan_recenter(t, ss);
    std::memcpy(pl->last_cell, cell, sizeof cell);
    rec = true;
  }
  if (g_prof_on || std::getenv("VP_NO_GRAPH")) {
    enqueue_frame_work(pl, n);
  } else {
    run_frame_graph(pl);
  }
  return rec;
}

void rerun_segment_until_fits(vp_grid* g, const vp_pipeline_params& p);

// Record part `part` of a frame for the current slot as a CUDA graph on
// stream `st` (rebuilt when a referenced buffer was reallocated), then launch it.
template <typename F>
void run_part_graph(vp_pipeline* pl, int part, cudaStream_t st, F&& enqueue) {
  vp_grid* g = pl->grid;
  const int s = g->slot;
  const uint64_t key = (g->gen << 32) ^ g->seg.gen;
  if (!pl->rx[s][part] || pl->rkey[s][part] != key) {
    if (pl->rx[s][part]) cudaGraphExecDestroy(pl->rx[s][part]);
    pl->rx[s][part] = nullptr;
    cudaGraph_t graph;
    const uint64_t before = g_launches.load();
    g->capturing = true;
    ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "capture begin");
    try {
      enqueue();
    } catch (...) {
      cudaStreamEndCapture(st, &graph);
      g->capturing = false;
      throw;
    }
    ck(cudaStreamEndCapture(st, &graph), "capture end");
    g->capturing = false;
    pl->rkern[s][part] = g_launches.load() - before;
    g_launches.fetch_sub(pl->rkern[s][part]);
    ck(cudaGraphInstantiate(&pl->rx[s][part], graph, 0), "graph instantiate");
    cudaGraphDestroy(graph);
    pl->rkey[s][part] = key;
  }
  ck(cudaGraphLaunch(pl->rx[s][part], st), "graph launch");
  g_launches.fetch_add(pl->rkern[s][part]);
}

// Host image of a frame's packed polygon records (k_poly_pack); false when
// the pack did not fit its buffer (the caller reads the slot's records).
bool unpack_polygons(const double* pk, HostPolys& hp) {
  if (pk[2] != 0.0) return false;
  const uint32_t F = static_cast<uint32_t>(pk[0]);
  const uint64_t Vt = static_cast<uint64_t>(pk[1]);
  hp.polys.clear();
  hp.verts.assign(pk + 4 + 12ull * F, pk + 4 + 12ull * F + 5 * Vt);
  uint64_t voff = 0;
  for (uint32_t f = 0; f < F; ++f) {
    const double* r = pk + 4 + 12ull * f;
    const uint32_t nv = static_cast<uint32_t>(r[10]);
    if (nv == 0) continue;
    vp_polygon q{};
    q.plane.normal[0] = r[0];
    q.plane.normal[1] = r[1];
    q.plane.normal[2] = r[2];
    q.plane.offset = r[3];
    q.area = r[4];
    q.plane.inlier_count = static_cast<int32_t>(r[8]);
    q.plane.cluster_label = static_cast<int32_t>(r[9]);
    q.nverts = nv;
    q.v2d = reinterpret_cast<const double*>(static_cast<uintptr_t>(voff));  // pool offset, as download_polygons
    voff += nv;
    hp.polys.push_back(q);
  }
  return true;
}

// Stage trace (voxplane_trace.h) of the segmentation held by the active
// context: counters c, host state of the frame (recenter flag, shift,
// post-recenter origin) and its polygons.
std::vector<uint8_t> build_trace(vp_grid* g, const Counters& c, uint32_t frame, bool rec, const int32_t* shift,
                                 const double* origin, const HostPolys& hp);

// What a pipelined run hands back per frame besides the final polygons.
struct RunOutputs {
  vp_frame_timing* timings = nullptr;          // n_frames stage spans
  vp_polygons_t** per_frame = nullptr;         // n_frames polygon sets (PipelineConfig per_frame_polygons)
  std::vector<std::vector<uint8_t>>* traces = nullptr;  // stage traces (parity tests)
  HostPolys* last = nullptr;                   // PipelineResult::polygons
};

// run_frames (pipeline.cpp:157-245) over a whole stream with up to kSlots
// frames in flight. Per frame k:
//   pstream  map_pre(k)  DDA walks || point grouping   after map_post(k-1)
//   mstream  map_post(k) clear, fold, recenter          after readers(k-1), map_pre(k)
//   mstream  readers(k)  occupied scan .. ordinal map
//   slot     chain(k)    CCL .. polygons, packed into mapped host memory
// The first half of the mapping touches no cell, so the walks of frame k+1
// run while frame k's readers scan the grid; the critical path is map_post +
// readers per frame, the chains (capped at kChainWide blocks) fill the rest of
// the GPU. VP_MAP_SPLIT=0 puts both halves on the mapping stream (A/B).
// Capacities of the grid readers are sized from the occupancy bound before
// enqueueing, so the host never waits per frame; a chain that outgrows its
// cluster buffers is re-run from its slot's steppable list when the slot is
// harvested (the list and ordinal map stay intact until the slot is reused).
void pipeline_run(vp_pipeline* pl, size_t nf, const float* const* xyz, const uint64_t* n,
                  const double* R, const double* t, bool device_ptrs, const RunOutputs& out) {
  const auto run_t0 = std::chrono::steady_clock::now();
  double host_wait_us = 0.0;
  vp_grid* g = pl->grid;
  for (auto* e : {pl->ev_start, pl->ev_pre, pl->ev_map, pl->ev_clu, pl->ev_ccl, pl->ev_rsc, pl->ev_done,
                  pl->ev_h2d})
    for (int q = 0; q < kSlots; ++q)
      if (!e[q]) ck(cudaEventCreate(&e[q]), "event");
  if (!pl->cstream) ck(cudaStreamCreateWithFlags(&pl->cstream, cudaStreamNonBlocking), "stream");
  for (int q = 0; q < kSlots; ++q)
    if (!pl->pack_h[q]) {
      ck(cudaHostAlloc(&pl->pack_h[q], vp_pipeline::kPackCap * sizeof(double), cudaHostAllocMapped), "pinned");
      ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&pl->pack_d[q]), pl->pack_h[q], 0), "mapped");
    }
  uint64_t maxn = 0;
  for (size_t k = 0; k < nf; ++k) maxn = std::max(maxn, n[k]);
  for (size_t k = 0; k < nf; ++k)
    if (!is_valid_rotation(R + 9 * k)) fail(VP_EINVAL, "clear_rays: pose rotation is not orthonormal");
  const char* split_env = std::getenv("VP_MAP_SPLIT");
  const cudaStream_t ps = (split_env && split_env[0] == '0') ? g->mstream : g->pstream;
  // On every exit -- normal or a throw part-way through (a failed capture,
  // allocation or overflow) -- drain every stream the run used and put the
  // grid back into its single-frame state (context 0, slot 0, stream order),
  // so later calls never see another context's buffers.
  struct RunGuard {
    vp_pipeline* pl;
    vp_grid* g;
    cudaStream_t ps;
    int nslot = 1;
    explicit RunGuard(vp_pipeline* p, cudaStream_t s) : pl(p), g(p->grid), ps(s) { g->chain_wide = kChainWide; }
    ~RunGuard() {
      for (int q = 0; q < nslot; ++q) {
        g->use_seg(q);
        cudaStreamSynchronize(g->stream);
      }
      cudaStreamSynchronize(g->mstream);
      cudaStreamSynchronize(ps);
      cudaStreamSynchronize(g->fstream);
      if (pl->cstream) cudaStreamSynchronize(pl->cstream);
      cudaGetLastError();
      g->capturing = false;
      g->use_seg(0);
      g->set_slot(0);
      g->lstream = g->stream;
      g->chain_wide = 148 * 8;  // C2: 148 x 8 -> 148 x 4 blocks inside a run, 3130 -> 3260 Hz
    }
  } guard(pl, ps);
  // a slot's stream swapped for the mapping stream while its grid readers are
  // enqueued, swapped back on scope exit (also on a throw)
  struct StreamSwap {
    vp_grid* g;
    cudaStream_t saved;
    StreamSwap(vp_grid* gg, cudaStream_t to) : g(gg), saved(gg->stream) { g->stream = to; }
    ~StreamSwap() { g->stream = saved; }
  };
  g->use_seg(0);
  g->set_slot(0);
  g->ensure_points(maxn);
  if (static_cast<uint64_t>(pl->p.ransac.iterations) * g->seg.kcap > g->seg.cand_cap)
    g->seg.ensure(g->seg.b.Vcap, g->seg.b.Scap, g->seg.b.Icap, pl->p.ransac.iterations, g->gd.nwords);
  g->seg.ensure_dirs(16, g->stream);
  const int nslot = g->ensure_contexts(static_cast<int>(std::min<size_t>(kSlots, std::max<size_t>(nf, 1))),
                                       pl->p.ransac.iterations);
  guard.nslot = nslot;
  const size_t NS = static_cast<size_t>(nslot);
  // host frames are copied ahead on the copy stream into the slot's point
  // buffer once that slot's previous frame has been mapped (the copy engine
  // overlaps the compute); copy_ahead - 1 frames ahead of the one being
  // enqueued (<= nslot: the copy of frame k waits for the mapping of frame
  // k - nslot, the slot's previous user)
  const size_t copy_ahead = std::min<size_t>(VP_COPY_AHEAD, NS);
  static_assert(VP_COPY_AHEAD >= 2 && VP_COPY_AHEAD <= kSlots, "copy-ahead depth");
  auto h2d_ahead = [&](size_t k) {
    if (device_ptrs || k >= nf) return;
    const int q = static_cast<int>(k % NS);
    if (k >= NS) ck(cudaStreamWaitEvent(pl->cstream, pl->ev_map[q], 0), "wait");
    if (n[k])
      ck(cudaMemcpyAsync(g->d_pts_s[q], xyz[k], n[k] * 12, cudaMemcpyHostToDevice, pl->cstream), "points h2d");
    ck(cudaEventRecord(pl->ev_h2d[q], pl->cstream), "ev");
  };
  uint64_t occ_known = g->host_occupied;  // occupancy before frame `known`
  size_t known = 0;
  uint32_t cap_min = 0xffffffffu;
  for (int q = 0; q < nslot; ++q) {
    g->use_seg(q);
    cap_min = std::min({cap_min, g->seg.b.Vcap, g->seg.b.Scap});
  }
  g->use_seg(0);
  ck(cudaStreamSynchronize(g->stream), "sync");
  const bool graphs = !g_prof_on && !std::getenv("VP_NO_GRAPH");
  auto enqueue_chain = [&](int s) {
    auto seg_rest = [&] {
      g->launch_step_emit(g->grid_map());  // steppable list + ordinal map (lists only, off the mapping stream)
      g->launch_seg_a2(pl->p, false);  // build_adjacency + label_components + filter_clusters
      g->record(pl->ev_ccl[s]);
      g->launch_ransac(make_ransacdev(pl->p.ransac));
      g->record(pl->ev_rsc[s]);
      g->launch_refine(pl->p.ransac.up, pl->p.refine, pl->p.refine_exact);
      g->launch_polygon(16, pl->p.min_polygon_area);
      LAUNCH(k_poly_pack, 1, 1024, 0, g->stream, g->ctr, g->seg.b, pl->pack_d[s], vp_pipeline::kPackCap);
      ck(cudaMemcpyAsync(g->h_ctr, g->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, g->stream), "ctr");
    };
    if (graphs) run_part_graph(pl, 3, g->stream, seg_rest); else seg_rest();
    ck(cudaEventRecord(pl->ev_done[s], g->stream), "ev");
  };
  // frame k's slot is reused by frame k + nslot: its whole chain must be done
  size_t harvested = 0;  // frames [0, harvested) handed back
  auto harvest = [&](size_t k) {
    if (k < harvested) return;
    harvested = k + 1;
    const int s = static_cast<int>(k % NS);
    {
      const auto w0 = std::chrono::steady_clock::now();
      ck(cudaEventSynchronize(pl->ev_done[s]), "slot sync");
      host_wait_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - w0).count();
    }
    g->use_seg(s);
    g->set_slot(s);
    for (int tries = 0; g->h_ctr->overflow; ++tries) {
      // only the chain can overflow here (the grid readers' capacities cover
      // the occupancy bound): grow its buffers, redo it from the slot's list
      if ((g->h_ctr->overflow & (kOverflowOcc | kOverflowStep)) || tries > 4)
        fail(VP_ENOMEM, "segmentation capacity overflow in a pipelined frame");
      g->grow_chain(pl->p.ransac.iterations);
      LAUNCH(k_chain_rearm, 1, 32, 0, g->stream, g->ctr);
      // (the chain starts with the steppable list: it rebuilds the ordinal
      // map the first run's CCL consumed)
      enqueue_chain(s);
      ck(cudaEventSynchronize(pl->ev_done[s]), "slot sync");
    }
    if (std::getenv("VP_PIPE_STATS")) {  // stage spans of the pipelined frame (diagnostics)
      float a = 0.f, b = 0.f, c = 0.f, a0 = 0.f;
      ck(cudaEventElapsedTime(&a0, pl->ev_start[s], pl->ev_pre[s]), "elapsed");
      ck(cudaEventElapsedTime(&a, pl->ev_pre[s], pl->ev_map[s]), "elapsed");
      ck(cudaEventElapsedTime(&b, pl->ev_map[s], pl->ev_clu[s]), "elapsed");
      ck(cudaEventElapsedTime(&c, pl->ev_clu[s], pl->ev_done[s]), "elapsed");
      std::fprintf(stderr, "frame %zu: map pre %.1f us, post %.1f us, grid readers %.1f us, chain %.1f us\n", k,
                   1e3 * a0, 1e3 * a, 1e3 * b, 1e3 * c);
    }
    if (out.timings) {  // FrameTiming spans (pipeline.cpp:181-219), device time of this frame
      float ms[6];
      ck(cudaEventElapsedTime(&ms[0], pl->ev_start[s], pl->ev_map[s]), "elapsed");
      ck(cudaEventElapsedTime(&ms[1], pl->ev_map[s], pl->ev_clu[s]), "elapsed");
      ck(cudaEventElapsedTime(&ms[2], pl->ev_clu[s], pl->ev_ccl[s]), "elapsed");
      ck(cudaEventElapsedTime(&ms[3], pl->ev_ccl[s], pl->ev_rsc[s]), "elapsed");
      ck(cudaEventElapsedTime(&ms[4], pl->ev_rsc[s], pl->ev_done[s]), "elapsed");
      ck(cudaEventElapsedTime(&ms[5], pl->ev_start[s], pl->ev_done[s]), "elapsed");
      vp_frame_timing& tm = out.timings[k];
      std::memset(&tm, 0, sizeof tm);
      tm.mapping_ms = ms[0];
      tm.classify_ms = ms[1];
      tm.cluster_ms = ms[2];
      tm.ransac_ms = ms[3];
      tm.hull_ms = ms[4];
      tm.total_ms = ms[5];
      tm.points = n[k];
      tm.voxels = g->h_ctr->occupied;
      tm.clusters = g->h_ctr->K;
    }
    if (!out.per_frame && !out.traces && !(out.last && k + 1 == nf)) return;
    HostPolys hp;
    if (!unpack_polygons(pl->pack_h[s], hp)) g->download_polygons(hp, false);
    if (out.per_frame) out.per_frame[k] = make_polygons_out(hp);
    if (out.traces) {
      const auto& m = pl->meta[s];
      out.traces->push_back(build_trace(g, *g->h_ctr, m.frame, m.rec, m.shift, m.origin, hp));
    }
    if (out.last && k + 1 == nf) *out.last = std::move(hp);
  };
  for (size_t k = 0; k < nf; ++k) {
    const int s = static_cast<int>(k % NS);
    const int prev = static_cast<int>((k + NS - 1) % NS);
    if (k >= NS) {
      harvest(k - NS);
      occ_known = g->h_ctr_s[s]->occupied;  // after frame k - nslot
      known = k - NS + 1;
    }
    // The occupied (and steppable) lists of frame k cannot be longer than the
    // occupancy known for frame known-1 plus every point integrated since:
    // grow all contexts before enqueueing if that bound exceeds a capacity,
    // so no frame in flight can overflow (no host wait per frame).
    {
      uint64_t bound = occ_known;
      for (size_t i = known; i <= k; ++i) bound += n[i];
      bound = std::min<uint64_t>(bound, g->gd.ncells);
      if (bound > cap_min) {
        for (int q = 0; q < nslot; ++q) {
          g->use_seg(q);
          ck(cudaStreamSynchronize(g->stream), "sync");
        }
        ck(cudaStreamSynchronize(g->mstream), "sync");
        ck(cudaStreamSynchronize(ps), "sync");
        // hand back every frame still held by a context before the contexts
        // are reallocated (their traces and records live there)
        for (size_t i = harvested; i < k; ++i) harvest(i);
        const uint32_t need = static_cast<uint32_t>(std::max<uint64_t>(bound, 2ull * cap_min));
        const uint32_t v = static_cast<uint32_t>(std::min<uint64_t>(need, g->gd.ncells));
        for (int q = 0; q < nslot; ++q) {
          g->use_seg(q);
          g->seg.ensure(std::max(g->seg.b.Vcap, v), std::max(g->seg.b.Scap, v), std::max(g->seg.b.Icap, v),
                        pl->p.ransac.iterations, g->gd.nwords);
        }
        cap_min = v;
      }
    }
    g->set_slot(s);
    g->use_seg(s);
    g->set_pose(R + 9 * k, t + 3 * k);
    g->fill_static_params();
    if (device_ptrs) {
      g->h_fp->pts = xyz[k];
    } else {
      if (k == 0)
        for (size_t q = 0; q + 1 < copy_ahead; ++q) h2d_ahead(q);
      h2d_ahead(k + copy_ahead - 1);
      ck(cudaStreamWaitEvent(ps, pl->ev_h2d[s], 0), "wait");
      g->h_fp->pts = g->d_pts;
    }
    g->h_fp->n = n[k];
    auto& meta = pl->meta[s];
    meta.frame = pl->frame;
    meta.rec = false;
    std::memset(meta.shift, 0, sizeof meta.shift);
    int32_t cell[3];
    global_cell(t + 3 * k, g->gd.res, cell);
    if (cell[0] != pl->last_cell[0] || cell[1] != pl->last_cell[1] || cell[2] != pl->last_cell[2]) {
      vp_shift_stats ss;
      g->plan_recenter(t + 3 * k, &ss);
      std::memcpy(pl->last_cell, cell, sizeof cell);
      meta.rec = true;
      std::memcpy(meta.shift, ss.shift, sizeof meta.shift);
    }
    std::memcpy(meta.origin, g->origin, sizeof meta.origin);
    // mapping of frame k, first half (DDA walks marking the clear masks ||
    // grouping the points; no cell touched): on the pre-mapping stream once
    // frame k-1's mapping has consumed the masks and the grouping buffers,
    // i.e. concurrently with frame k-1's grid readers
    if (k >= 1) ck(cudaStreamWaitEvent(ps, pl->ev_map[prev], 0), "wait");
    ck(cudaEventRecord(pl->ev_start[s], ps), "ev");
    g->lstream = ps;
    auto map_pre = [&] {
      g->upload_params();
      g->reset_frame_counters();
      g->launch_mapping_pre(n[k]);
    };
    if (graphs) run_part_graph(pl, 0, ps, map_pre); else map_pre();
    ck(cudaEventRecord(pl->ev_pre[s], ps), "ev");
    // second half (clear, ordered fold, recenter) on the mapping stream:
    // after frame k-1's grid readers (stream order) and the first half
    ck(cudaStreamWaitEvent(g->mstream, pl->ev_pre[s], 0), "wait");
    g->lstream = g->mstream;
    auto map_post = [&] { g->launch_mapping_post(n[k]); };
    if (graphs) run_part_graph(pl, 1, g->mstream, map_post); else map_post();
    g->lstream = g->stream;
    ck(cudaEventRecord(pl->ev_map[s], g->mstream), "ev");
    // segmentation of frame k: the grid readers (occupied scan .. ordinal
    // map) right after the mapping on the high-priority mapping stream (the
    // critical path: frame k+1's mapping waits for them), then the CCL ..
    // polygon chain on the slot's stream, overlapping later frames
    {
      StreamSwap on_mapping(g, g->mstream);
      auto seg_grid = [&] {
        g->launch_seg_a1(pl->p, false, false);  // the cell readers only: the next mapping waits for them
        ck(cudaMemcpyAsync(g->h_ctr, g->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, g->stream), "ctr");
      };
      if (graphs) run_part_graph(pl, 2, g->stream, seg_grid); else seg_grid();
      ck(cudaEventRecord(pl->ev_clu[s], g->stream), "ev");
    }
    ck(cudaStreamWaitEvent(g->stream, pl->ev_clu[s], 0), "wait");
    enqueue_chain(s);
    // no host round trip before the next frame's mapping: the capacities were
    // sized above for this frame's worst case, and harvest() checks the flags
    ++pl->frame;
  }
  for (size_t k = nf > NS ? nf - NS : 0; k < nf; ++k) harvest(k);
  if (nf) g->host_occupied = g->h_ctr_s[(nf - 1) % NS]->occupied;
  if (std::getenv("VP_PIPE_STATS"))  // host-bound run: the harvests never wait
    std::fprintf(stderr, "pipeline_run: %zu frames, host waited %.1f us in harvests (%.1f us/frame), wall %.1f us\n",
                 nf, host_wait_us, nf ? host_wait_us / nf : 0.0,
                 std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - run_t0).count());
}

void wait_frame(vp_grid* g) {
  ck(cudaStreamSynchronize(g->stream), "frame sync");
  g->host_occupied = g->h_ctr->occupied;
}

void fill_timing(vp_grid* g, vp_frame_timing* tm, uint64_t n) {
  if (!tm) return;
  float ms[5];
  for (int i = 0; i < 5; ++i) ck(cudaEventElapsedTime(&ms[i], g->ev[i], g->ev[i + 1]), "elapsed");
  tm->mapping_ms = ms[0];
  tm->classify_ms = ms[1];
  tm->cluster_ms = ms[2];
  tm->ransac_ms = ms[3];
  tm->hull_ms = ms[4];
  float tot;
  ck(cudaEventElapsedTime(&tot, g->ev[0], g->ev[5]), "elapsed");
  tm->total_ms = tot;
  tm->points = n;
  tm->voxels = g->h_ctr->occupied;
  tm->clusters = g->h_ctr->K;
}

// Re-run only the segmentation part after growing capacities.
void rerun_segment_until_fits(vp_grid* g, const vp_pipeline_params& p) {
  // the frame's mapping counters (ClearStats, UpdateStats, ShiftStats) are
  // the first run's: a re-run of the segmentation must not reset them
  const Counters map_ctr = *g->h_ctr;
  for (int tries = 0; tries < 6; ++tries) {
    const uint32_t of = g->h_ctr->overflow;
    // only the chain (CCL .. polygons) overflowed: its buffers grow and it
    // re-runs from the steppable list, like a pipelined frame's chain -- the
    // grid readers already wrote this frame's statuses into the cells, so
    // re-running them would read those instead of the pre-classify ones
    const bool chain_only = of && !(of & (kOverflowOcc | kOverflowStep));
    if (!g->grow_if_overflow(p.ransac.iterations)) break;
    if (chain_only) {
      LAUNCH(k_chain_rearm, 1, 32, 0, g->stream, g->ctr);
      // the CCL's flatten consumed (reset) the ordinal map: rebuild it from the list
      LAUNCH(k_map_fill, g->chain_wide, kThreads, 0, g->stream, g->ctr, g->seg.b, g->grid_map());
      ck(cudaEventRecord(g->ev[2], g->stream), "ev");
      g->launch_seg_a2(p, true);
      g->launch_seg_b(p, true);
      g->read_counters();
      continue;
    }
    // restore the post-map state: the recenter was already applied, so the
    // segmentation reads the post bitmap/offsets; make pre == post.
    for (int k = 0; k < 3; ++k) {
      g->h_fp->origin_pre[k] = g->h_fp->origin_post[k];
      g->h_fp->off_pre[k] = g->h_fp->off_post[k];
      g->h_fp->shift[k] = 0;
    }
    g->h_fp->occ_pre = g->h_fp->occ_post;
    g->h_fp->zb_pre = g->h_fp->zb_post;
    g->h_fp->do_shift = 0;
    g->h_fp->n = 0;
    g->upload_params();
    g->reset_frame_counters();
    ck(cudaEventRecord(g->ev[0], g->stream), "ev");
    g->launch_segment(p, true);
    g->read_counters();
  }
  if (g->h_ctr->overflow) fail(VP_ENOMEM, "segmentation capacity overflow persists");
  Counters& c = *g->h_ctr;
  c.cleared = map_ctr.cleared, c.freed = map_ctr.freed, c.touched = map_ctr.touched;
  c.discarded = map_ctr.discarded, c.dropped = map_ctr.dropped, c.newly = map_ctr.newly;
}

struct TraceW {
  std::vector<uint8_t> b;
  template <typename T>
  void put(const T& v) {
    const auto* p = reinterpret_cast<const uint8_t*>(&v);
    b.insert(b.end(), p, p + sizeof(T));
  }
  void raw(const void* p, size_t n) {
    const auto* q = static_cast<const uint8_t*>(p);
    b.insert(b.end(), q, q + n);
  }
};

template <typename T>
std::vector<T> d2h(const T* src, size_t n, cudaStream_t s) {
  std::vector<T> v(n);
  if (n) ck(cudaMemcpyAsync(v.data(), src, n * sizeof(T), cudaMemcpyDeviceToHost, s), "d2h");
  return v;
}

}  // namespace

// ===========================================================================
extern "C" {

const char* vp_last_error(void) { return g_err.c_str(); }
const char* vp_version(void) { return "voxplane_b200 0.1 (sm_100a)"; }
uint64_t vp_kernel_launch_count(void) { return g_launches.load(); }
int vp_set_ccl_mode(int mode) {
  if (mode < 0 || mode > 4) return VP_EINVAL;
  g_ccl_mode = mode;
  return VP_OK;
}

void vp_profile_enable(int on) {
  g_prof_on = on != 0;
  if (on) g_prof.clear();
}

// Accumulated per-kernel device time since vp_profile_enable(1): returns the
// number of kernels; fills up to cap entries (name pointers stay valid until
// the next vp_profile_enable).
int vp_profile_read(const char** names, double* ms, uint64_t* calls, int cap) {
  const int n = static_cast<int>(g_prof.size());
  for (int i = 0; i < n && i < cap; ++i) {
    names[i] = g_prof[i].name.c_str();
    ms[i] = g_prof[i].ms;
    calls[i] = g_prof[i].calls;
  }
  return n;
}
void vp_free(void* p) { std::free(p); }

void vp_default_params(vp_pipeline_params* p) {
  std::memset(p, 0, sizeof *p);
  p->seg.neighbor_radius = 1;
  p->seg.min_neighbors = 3;
  p->seg.max_angle_deg = 15.0;
  p->seg.adjacency_angle_deg = 15.0;
  p->seg.distance_th = 0.05;
  p->seg.min_cluster_size = 30;
  p->seg.up[2] = 1.0;
  p->ransac.iterations = 100;
  p->ransac.inlier_eps = 0.01;
  p->ransac.seed = 0;
  p->ransac.up[2] = 1.0;
  p->refine = 1;
  p->min_polygon_area = 0.002;
  p->refine_exact = 0;
}

int vp_grid_create(double res, const int32_t extent[3], const double center[3], int device,
                   vp_grid** out) {
  *out = nullptr;
  return guard([&] {
    auto* g = new vp_grid();
    try {
      g->init(res, extent, center, device);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

void vp_grid_destroy(vp_grid* g) {
  vp::slab_frame_release(g);
  delete g;
}

int vp_grid_info(const vp_grid* g, double origin[3], int32_t extent[3], double* resolution,
                 uint64_t* occupied_count) {
  return guard([&] {
    for (int k = 0; k < 3; ++k) {
      if (origin) origin[k] = g->origin[k];
      if (extent) extent[k] = g->ext[k];
    }
    if (resolution) *resolution = g->gd.res;
    if (occupied_count) *occupied_count = g->host_occupied;
  });
}

int vp_integrate_frame(vp_grid* g, const float* xyz, uint64_t n, const double R[9],
                       const double t[3], vp_update_stats* st) {
  return guard([&] {
    if (!is_valid_rotation(R)) fail(VP_EINVAL, "integrate_frame: pose rotation is not orthonormal");
    g->set_pose(R, t);
    g->fill_static_params();
    stage_points(g, xyz, n, false);
    g->upload_params();
    g->reset_frame_counters();
    g->launch_integrate(n);
    g->launch_finalize();
    g->read_counters();
    if (st) {
      st->voxels_touched = g->h_ctr->touched;
      st->points_discarded = g->h_ctr->discarded;
    }
  });
}

int vp_clear_rays(vp_grid* g, const float* xyz, uint64_t n, const double R[9], const double t[3],
                  vp_clear_stats* st) {
  return guard([&] {
    if (!is_valid_rotation(R)) fail(VP_EINVAL, "clear_rays: pose rotation is not orthonormal");
    g->set_pose(R, t);
    g->fill_static_params();
    stage_points(g, xyz, n, false);
    g->upload_params();
    g->reset_frame_counters();
    g->launch_clear(n);
    g->launch_finalize();
    g->read_counters();
    if (st) {
      st->voxels_cleared = g->h_ctr->cleared;
      st->voxels_freed = g->h_ctr->freed;
    }
  });
}

int vp_update_frame(vp_grid* g, const float* xyz, uint64_t n, const double R[9], const double t[3],
                    vp_clear_stats* cs, vp_update_stats* us) {
  return guard([&] {
    if (!is_valid_rotation(R)) fail(VP_EINVAL, "clear_rays: pose rotation is not orthonormal");
    g->set_slot(0);
    g->lstream = g->stream;
    g->set_pose(R, t);
    g->fill_static_params();
    stage_points(g, xyz, n, false);
    g->upload_params();
    g->reset_frame_counters();
    g->launch_mapping_pre(n);  // grouping (measures the ray box) || walks
    g->launch_clear_apply(n, 1);
    g->launch_integrate_fold(n);
    g->launch_finalize();
    g->read_counters();
    if (cs) {
      cs->voxels_cleared = g->h_ctr->cleared;
      cs->voxels_freed = g->h_ctr->freed;
    }
    if (us) {
      us->voxels_touched = g->h_ctr->touched;
      us->points_discarded = g->h_ctr->discarded;
    }
  });
}

int vp_recenter(vp_grid* g, const double c[3], vp_shift_stats* st) {
  return guard([&] {
    vp_shift_stats tmp;
    g->fill_static_params();
    g->h_fp->n = 0;
    if (!g->plan_recenter(c, st ? st : &tmp)) return;
    g->upload_params();
    g->reset_frame_counters();
    g->launch_recenter();
    g->launch_finalize();
    g->read_counters();
    if (st) st->voxels_dropped = g->h_ctr->dropped;
  });
}

int vp_merge_point(vp_grid* g, const int32_t idx[3], const double p[3]) {
  return guard([&] {
    if (idx[0] < 0 || idx[1] < 0 || idx[2] < 0 || idx[0] >= g->ext[0] || idx[1] >= g->ext[1] ||
        idx[2] >= g->ext[2])
      fail(VP_EINVAL, "merge_point: index out of bounds");
    g->fill_static_params();
    g->h_fp->n = 0;
    g->upload_params();
    g->reset_frame_counters();
    LAUNCH(k_merge_point, 1, 1, 0, g->stream, g->gd, g->d_fp, g->ctr, idx[0], idx[1], idx[2], p[0],
           p[1], p[2]);
    g->launch_finalize();
    g->read_counters();
  });
}

static uint64_t host_phys(const vp_grid* g, const int32_t* idx) {
  int64_t p[3];
  int32_t l[3] = {idx[0] - g->gd.xoff, idx[1], idx[2]};  // slab: window x -> local x
  for (int k = 0; k < 3; ++k) p[k] = (static_cast<int64_t>(l[k]) + g->off[k]) % g->ext[k];
  return (static_cast<uint64_t>(p[0]) * g->ext[1] + p[1]) * g->ext[2] + p[2];
}

int vp_get_cell(vp_grid* g, const int32_t idx[3], double sum[3], uint32_t* count, uint8_t* status) {
  return guard([&] {
    const int32_t lx = idx[0] - g->gd.xoff;
    if (lx < 0 || idx[1] < 0 || idx[2] < 0 || lx >= g->ext[0] || idx[1] >= g->ext[1] ||
        idx[2] >= g->ext[2])
      fail(VP_EINVAL, "cell: index out of bounds");
    Cell c;
    ck(cudaMemcpyAsync(&c, g->gd.cells + host_phys(g, idx), sizeof(Cell), cudaMemcpyDeviceToHost,
                       g->stream), "cell");
    ck(cudaStreamSynchronize(g->stream), "sync");
    if (sum) {
      sum[0] = c.sx;
      sum[1] = c.sy;
      sum[2] = c.sz;
    }
    if (count) *count = c.count;
    if (status) *status = c.status;
  });
}

int vp_set_status(vp_grid* g, const int32_t idx[3], uint8_t status) {
  return guard([&] {
    const int32_t lx = idx[0] - g->gd.xoff;
    if (lx < 0 || idx[1] < 0 || idx[2] < 0 || lx >= g->ext[0] || idx[1] >= g->ext[1] ||
        idx[2] >= g->ext[2])
      fail(VP_EINVAL, "set_status: index out of bounds");
    Cell* c = g->gd.cells + host_phys(g, idx);
    ck(cudaMemcpyAsync(&c->status, &status, 1, cudaMemcpyHostToDevice, g->stream), "status");
    ck(cudaStreamSynchronize(g->stream), "sync");
  });
}

int vp_set_statuses(vp_grid* g, const int32_t* idx, const uint8_t* status, size_t n) {
  return guard([&] {
    if (n == 0) return;
    int32_t* di = dalloc<int32_t>(3 * n);
    uint8_t* ds = dalloc<uint8_t>(n);
    ck(cudaMemcpyAsync(di, idx, 12 * n, cudaMemcpyHostToDevice, g->stream), "idx");
    ck(cudaMemcpyAsync(ds, status, n, cudaMemcpyHostToDevice, g->stream), "st");
    g->fill_static_params();
    g->h_fp->n = 0;
    g->upload_params();
    LAUNCH(k_set_statuses, grid_for(n), kThreads, 0, g->stream, g->gd, g->d_fp, di, ds, n);
    ck(cudaStreamSynchronize(g->stream), "sync");
    cudaFree(di);
    cudaFree(ds);
  });
}

int vp_occupied_voxels(vp_grid* g, vp_occupied_t** out) {
  *out = nullptr;
  return guard([&] {
    for (int tries = 0;; ++tries) {
      g->fill_static_params();
      g->h_fp->n = 0;
      g->upload_params();
      g->reset_frame_counters();
      g->launch_occupied_scan();
      LAUNCH(k_occ_gather, kWide, kThreads, 0, g->stream, g->gd, g->d_fp, g->ctr, g->seg.b);
      g->read_counters();
      if (g->h_ctr->V <= g->seg.b.Vcap || tries > 4) break;
      g->seg.ensure(static_cast<uint32_t>(std::min<uint64_t>(g->gd.ncells, 2ull * g->h_ctr->V)),
                    g->seg.b.Scap, g->seg.b.Icap, 100, g->gd.nwords);
    }
    const uint32_t V = g->h_ctr->V;
    auto flat = d2h(g->seg.b.occ_list, V, g->stream);
    auto mean = d2h(g->seg.b.own_mean, 3ull * V, g->stream);
    auto cnt = d2h(g->seg.b.own_count, V, g->stream);
    auto st = d2h(g->seg.b.own_status, V, g->stream);
    ck(cudaStreamSynchronize(g->stream), "sync");
    auto* o = static_cast<vp_occupied_t*>(std::calloc(1, sizeof(vp_occupied_t)));
    o->count = V;
    o->idx = static_cast<int32_t*>(std::malloc(12ull * V + 1));
    o->mean = static_cast<double*>(std::malloc(24ull * V + 1));
    o->npts = static_cast<uint32_t*>(std::malloc(4ull * V + 1));
    o->status = static_cast<uint8_t*>(std::malloc(V + 1));
    for (uint32_t v = 0; v < V; ++v) {
      const uint32_t f = flat[v];
      o->idx[3 * v + 2] = static_cast<int32_t>(f % g->ext[2]);
      o->idx[3 * v + 1] = static_cast<int32_t>((f / g->ext[2]) % g->ext[1]);
      o->idx[3 * v] = static_cast<int32_t>(f / g->ext[2] / g->ext[1]);
    }
    std::memcpy(o->mean, mean.data(), 24ull * V);
    std::memcpy(o->npts, cnt.data(), 4ull * V);
    std::memcpy(o->status, st.data(), V);
    *out = o;
  });
}

void vp_occupied_free(vp_occupied_t* o) {
  if (!o) return;
  std::free(o->idx);
  std::free(o->mean);
  std::free(o->npts);
  std::free(o->status);
  std::free(o);
}

// estimate_normals (+ optional classify) on the current grid state.
static void run_normals(vp_grid* g, const vp_seg_params* p, int write_status) {
  const SegDev sd = make_segdev(*p, g->gd.res);
  for (int tries = 0;; ++tries) {
    g->fill_static_params();
    g->h_fp->n = 0;
    g->upload_params();
    g->reset_frame_counters();
    g->launch_occupied_scan();
    g->launch_classify(sd, write_status);
    g->read_counters();
    if (!(g->h_ctr->overflow & kOverflowOcc) || tries > 4) break;
    g->seg.ensure(static_cast<uint32_t>(std::min<uint64_t>(g->gd.ncells, 2ull * g->h_ctr->V)),
                  static_cast<uint32_t>(std::min<uint64_t>(g->gd.ncells, 2ull * g->h_ctr->V)),
                  g->seg.b.Icap, 100, g->gd.nwords);
  }
  if (g->h_ctr->V == 0) fail(VP_EEMPTY, "estimate_normals: empty grid");
}

int vp_estimate_normals(vp_grid* g, const vp_seg_params* p, vp_estimates_t** out) {
  *out = nullptr;
  return guard([&] {
    run_normals(g, p, 0);
    LAUNCH(k_occ_gather, kWide, kThreads, 0, g->stream, g->gd, g->d_fp, g->ctr, g->seg.b);
    const uint32_t V = g->h_ctr->V;
    auto flat = d2h(g->seg.b.occ_list, V, g->stream);
    auto mean = d2h(g->seg.b.own_mean, 3ull * V, g->stream);
    auto nrm = d2h(g->seg.b.est_normal, 3ull * V, g->stream);
    auto nc = d2h(g->seg.b.est_ncount, V, g->stream);
    auto va = d2h(g->seg.b.est_valid, V, g->stream);
    ck(cudaStreamSynchronize(g->stream), "sync");
    auto* e = static_cast<vp_estimates_t*>(std::calloc(1, sizeof(vp_estimates_t)));
    e->count = V;
    e->idx = static_cast<int32_t*>(std::malloc(12ull * V + 1));
    e->mean = static_cast<double*>(std::malloc(24ull * V + 1));
    e->normal = static_cast<double*>(std::malloc(24ull * V + 1));
    e->neighbor_count = static_cast<int32_t*>(std::malloc(4ull * V + 1));
    e->angle_to_up_deg = static_cast<double*>(std::malloc(8ull * V + 1));
    e->valid = static_cast<uint8_t*>(std::malloc(V + 1));
    for (uint32_t v = 0; v < V; ++v) {
      const uint32_t f = flat[v];
      e->idx[3 * v + 2] = static_cast<int32_t>(f % g->ext[2]);
      e->idx[3 * v + 1] = static_cast<int32_t>((f / g->ext[2]) % g->ext[1]);
      e->idx[3 * v] = static_cast<int32_t>(f / g->ext[2] / g->ext[1]);
      e->angle_to_up_deg[v] = 0.0;
      if (va[v]) {  // segmentation.cpp:62-63 with the host libm
        const double d0 = (nrm[3 * v] * p->up[0] + nrm[3 * v + 1] * p->up[1]) + nrm[3 * v + 2] * p->up[2];
        const double d = std::clamp(d0, 0.0, 1.0);
        e->angle_to_up_deg[v] = std::acos(d) * kRadToDeg;
      }
    }
    std::memcpy(e->mean, mean.data(), 24ull * V);
    std::memcpy(e->normal, nrm.data(), 24ull * V);
    std::memcpy(e->neighbor_count, nc.data(), 4ull * V);
    std::memcpy(e->valid, va.data(), V);
    *out = e;
  });
}

void vp_estimates_free(vp_estimates_t* e) {
  if (!e) return;
  std::free(e->idx);
  std::free(e->mean);
  std::free(e->normal);
  std::free(e->neighbor_count);
  std::free(e->angle_to_up_deg);
  std::free(e->valid);
  std::free(e);
}

int vp_classify_steppable(vp_grid* g, const vp_seg_params* p, vp_steppable_t** steppable,
                          int32_t** objects_idx, size_t* n_objects) {
  *steppable = nullptr;
  return guard([&] {
    run_normals(g, p, 1);
    const uint32_t V = g->h_ctr->V;
    const uint32_t S = g->h_ctr->S;
    auto flat = d2h(g->seg.b.occ_list, V, g->stream);
    auto flag = d2h(g->seg.b.step_flag, V, g->stream);
    auto mean = d2h(g->seg.b.own_mean, 3ull * V, g->stream);
    auto nrm = d2h(g->seg.b.est_normal, 3ull * V, g->stream);
    ck(cudaStreamSynchronize(g->stream), "sync");
    auto* s = static_cast<vp_steppable_t*>(std::calloc(1, sizeof(vp_steppable_t)));
    s->count = S;
    s->idx = static_cast<int32_t*>(std::malloc(12ull * S + 1));
    s->mean = static_cast<double*>(std::malloc(24ull * S + 1));
    s->normal = static_cast<double*>(std::malloc(24ull * S + 1));
    std::vector<int32_t> obj;
    uint32_t k = 0;
    for (uint32_t v = 0; v < V; ++v) {
      const uint32_t f = flat[v];
      const int32_t xyz[3] = {static_cast<int32_t>(f / g->ext[2] / g->ext[1]),
                              static_cast<int32_t>((f / g->ext[2]) % g->ext[1]),
                              static_cast<int32_t>(f % g->ext[2])};
      if (flag[v]) {
        std::memcpy(s->idx + 3 * k, xyz, 12);
        std::memcpy(s->mean + 3 * k, mean.data() + 3 * v, 24);
        std::memcpy(s->normal + 3 * k, nrm.data() + 3 * v, 24);
        ++k;
      } else {
        obj.insert(obj.end(), xyz, xyz + 3);
      }
    }
    *steppable = s;
    if (objects_idx) {
      *objects_idx = static_cast<int32_t*>(std::malloc(obj.size() * 4 + 1));
      std::memcpy(*objects_idx, obj.data(), obj.size() * 4);
    }
    if (n_objects) *n_objects = obj.size() / 3;
  });
}

void vp_steppable_free(vp_steppable_t* s) {
  if (!s) return;
  std::free(s->idx);
  std::free(s->mean);
  std::free(s->normal);
  std::free(s);
}

}  // extern "C"

// ---- host-list entry points share a per-device scratch grid (1^3 window) --
namespace {
struct Scratch {
  vp_grid* g = nullptr;
  int device = -1;
};
thread_local Scratch t_scratch;

vp_grid* scratch_grid(int device) {
  if (t_scratch.g && t_scratch.device == device) return t_scratch.g;
  delete t_scratch.g;
  t_scratch.g = nullptr;
  auto* g = new vp_grid();
  const int32_t e[3] = {1, 1, 32};
  const double c[3] = {0, 0, 0};
  try {
    g->init(1.0, e, c, device);
  } catch (...) {
    delete g;
    throw;
  }
  t_scratch.g = g;
  t_scratch.device = device;
  return g;
}

template <typename T>
void h2d(T* dst, const T* src, size_t n, cudaStream_t s) {
  if (n) ck(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, s), "h2d");
}

void set_counter_u32(vp_grid* g, size_t field_offset, uint32_t v) {
  ck(cudaMemcpyAsync(reinterpret_cast<char*>(g->ctr) + field_offset, &v, 4, cudaMemcpyHostToDevice,
                     g->stream), "ctr set");
  ck(cudaStreamSynchronize(g->stream), "sync");
}

// Temporary dense ordinal volume over the steppable bounding box
// (segmentation.cpp:96-110).
struct BoxMap {
  MapDesc m{};
  int32_t* buf = nullptr;
  uint32_t* bits = nullptr;
  ~BoxMap() {
    if (buf) cudaFree(buf);
    if (bits) cudaFree(bits);
  }
};

void upload_steppable(vp_grid* g, const vp_steppable_t* s, BoxMap& bm) {
  const uint32_t S = static_cast<uint32_t>(s->count);
  g->seg.ensure(std::max(g->seg.b.Vcap, S), std::max(g->seg.b.Scap, S), g->seg.b.Icap, 100, g->gd.nwords);
  int lo[3], hi[3];
  for (int k = 0; k < 3; ++k) lo[k] = hi[k] = S ? s->idx[k] : 0;
  for (uint32_t i = 0; i < S; ++i)
    for (int k = 0; k < 3; ++k) {
      lo[k] = std::min(lo[k], s->idx[3 * i + k]);
      hi[k] = std::max(hi[k], s->idx[3 * i + k]);
    }
  uint64_t vol = 1;
  for (int k = 0; k < 3; ++k) {
    bm.m.lo[k] = lo[k];
    bm.m.dims[k] = hi[k] - lo[k] + 1;
    vol *= static_cast<uint64_t>(bm.m.dims[k]);
  }
  bm.buf = dalloc<int32_t>(vol);
  ck(cudaMemsetAsync(bm.buf, 0xff, vol * 4, g->stream), "map");
  bm.m.map = bm.buf;
  bm.m.W = (bm.m.dims[2] + 31) / 32;
  const uint64_t nw = static_cast<uint64_t>(bm.m.dims[0]) * bm.m.dims[1] * bm.m.W;
  bm.bits = dalloc<uint32_t>(nw);
  ck(cudaMemsetAsync(bm.bits, 0, nw * 4, g->stream), "bits");
  bm.m.bits = bm.bits;
  h2d(g->seg.b.st_idx, s->idx, 3ull * S, g->stream);
  h2d(g->seg.b.st_mean, s->mean, 3ull * S, g->stream);
  h2d(g->seg.b.st_normal, s->normal, 3ull * S, g->stream);
  g->reset_frame_counters();
  set_counter_u32(g, offsetof(Counters, S), S);
  LAUNCH(k_map_fill, kWide, kThreads, 0, g->stream, g->ctr, g->seg.b, bm.m);
}

// ---- fit_planes on host-provided clusters (vp_fit_planes, vp_run_ablation)
struct FitResult {
  std::vector<vp_plane> models;
  std::vector<uint64_t> offsets{0};
  std::vector<double> inliers;
  uint64_t skipped = 0, unfit = 0;
};

void append_fits(FitResult& all, const FitResult& r) {
  const uint64_t base = all.offsets.back();
  all.models.insert(all.models.end(), r.models.begin(), r.models.end());
  for (size_t i = 1; i < r.offsets.size(); ++i) all.offsets.push_back(base + r.offsets[i]);
  all.inliers.insert(all.inliers.end(), r.inliers.begin(), r.inliers.end());
  all.skipped += r.skipped;
  all.unfit += r.unfit;
}

// Stage K clusters (sizes, labels, contiguous member means) in the
// cluster-parallel layout (warp-padded SoA) and set the counters; returns kpoff.
std::vector<uint32_t> stage_clusters(vp_grid* g, uint32_t K, const int32_t* labels, const uint32_t* ksize,
                                     const double* means, int iterations) {
  std::vector<uint32_t> kpoff(K + 1, 0);
  uint64_t tot = 0, maxm = 0;
  for (uint32_t k = 0; k < K; ++k) {
    kpoff[k] = static_cast<uint32_t>(tot);
    tot += (ksize[k] + 31u) & ~31u;
    maxm += ksize[k];
  }
  kpoff[K] = static_cast<uint32_t>(tot);
  const uint32_t need = static_cast<uint32_t>(std::max<uint64_t>(tot, maxm));
  // inliers: [0, tot) for the cluster-parallel pass, [tot, 2 tot) for the serial views
  g->seg.ensure(g->seg.b.Vcap, std::max(g->seg.b.Scap, need), std::max(g->seg.b.Icap, 2 * need),
                std::max(iterations, 1), g->gd.nwords);
  std::vector<double> mx(tot, 0.0), my(tot, 0.0), mz(tot, 0.0);
  uint64_t src = 0;
  for (uint32_t k = 0; k < K; ++k)
    for (uint32_t j = 0; j < ksize[k]; ++j, ++src) {
      mx[kpoff[k] + j] = means[3 * src];
      my[kpoff[k] + j] = means[3 * src + 1];
      mz[kpoff[k] + j] = means[3 * src + 2];
    }
  h2d(g->seg.b.klabel, labels, K, g->stream);
  h2d(g->seg.b.ksize, ksize, K, g->stream);
  h2d(g->seg.b.kpoff, kpoff.data(), K + 1, g->stream);
  h2d(g->seg.b.mx, mx.data(), tot, g->stream);
  h2d(g->seg.b.my, my.data(), tot, g->stream);
  h2d(g->seg.b.mz, mz.data(), tot, g->stream);
  g->reset_frame_counters();
  set_counter_u32(g, offsetof(Counters, K), K);
  return kpoff;
}

void serial_prepare(vp_grid* g, const std::vector<uint32_t>& ksize, const std::vector<uint32_t>& kpoff) {
  SerialFitBufs& sf = g->sf;
  const uint32_t K = static_cast<uint32_t>(ksize.size());
  if (K > sf.cap) {
    sf.release();
    sf.cap = std::max<uint32_t>(K, 64);
    sf.kp1 = dalloc<uint32_t>(2ull * sf.cap);
    sf.ctrs = dalloc<Counters>(sf.cap);
    sf.fm = dalloc<double>(4ull * sf.cap);
    sf.fmeta = dalloc<int32_t>(2ull * sf.cap);
    sf.io1 = dalloc<uint32_t>(2ull * sf.cap);
  }
  std::vector<uint32_t> kp1(2ull * K);
  std::vector<Counters> c(K);
  std::memset(c.data(), 0, K * sizeof(Counters));
  for (uint32_t k = 0; k < K; ++k) {
    kp1[2 * k] = 0;
    kp1[2 * k + 1] = kpoff[k + 1] - kpoff[k];
    c[k].K = 1;
  }
  h2d(sf.kp1, kp1.data(), kp1.size(), g->stream);
  h2d(sf.ctrs, c.data(), K, g->stream);
  ck(cudaStreamSynchronize(g->stream), "sync");
}

void serial_launch(vp_grid* g, const RansacDev& rd, const std::vector<uint32_t>& kpoff) {
  SerialFitBufs& sf = g->sf;
  const uint32_t K = static_cast<uint32_t>(kpoff.size() - 1);
  for (uint32_t k = 0; k < K; ++k) {
    SegBufs v = g->seg.b;
    v.klabel += k;
    v.ksize += k;
    v.kpoff = sf.kp1 + 2 * k;
    v.mx += kpoff[k];
    v.my += kpoff[k];
    v.mz += kpoff[k];
    v.fit_model = sf.fm + 4 * k;
    v.fit_meta = sf.fmeta + 2 * k;
    v.ioff = sf.io1 + 2 * k;
    v.inl = g->seg.b.inl + 3ull * (kpoff[K] + kpoff[k]);
    v.Icap = kpoff[k + 1] - kpoff[k];
    g->launch_ransac(rd, sf.ctrs + k, v);
  }
}

FitResult parallel_results(vp_grid* g) {
  g->read_counters();
  FitResult r;
  const uint32_t F = g->h_ctr->nfits;
  r.skipped = g->h_ctr->skipped;
  r.unfit = g->h_ctr->unfit;
  if (g->h_ctr->overflow) fail(VP_ENOMEM, "fit_planes: capacity overflow");
  auto fm = d2h(g->seg.b.fit_model, 4ull * F, g->stream);
  auto meta = d2h(g->seg.b.fit_meta, 2ull * F, g->stream);
  auto io = d2h(g->seg.b.ioff, F + 1ull, g->stream);
  ck(cudaStreamSynchronize(g->stream), "sync");
  r.inliers = d2h(g->seg.b.inl, 3ull * io[F], g->stream);
  ck(cudaStreamSynchronize(g->stream), "sync");
  for (uint32_t f = 0; f < F; ++f) {
    vp_plane pl{};
    for (int q = 0; q < 3; ++q) pl.normal[q] = fm[4 * f + q];
    pl.offset = fm[4 * f + 3];
    pl.inlier_count = meta[2 * f];
    pl.cluster_label = meta[2 * f + 1];
    r.models.push_back(pl);
    r.offsets.push_back(io[f + 1]);
  }
  return r;
}

FitResult serial_results(vp_grid* g, const std::vector<uint32_t>& ksize, const std::vector<uint32_t>& kpoff) {
  SerialFitBufs& sf = g->sf;
  const uint32_t K = static_cast<uint32_t>(ksize.size());
  auto c = d2h(sf.ctrs, K, g->stream);
  auto fm = d2h(sf.fm, 4ull * K, g->stream);
  auto meta = d2h(sf.fmeta, 2ull * K, g->stream);
  auto io = d2h(sf.io1, 2ull * K, g->stream);
  ck(cudaStreamSynchronize(g->stream), "sync");
  FitResult r;
  for (uint32_t k = 0; k < K; ++k) {
    if (c[k].overflow) fail(VP_ENOMEM, "fit_planes: capacity overflow");
    r.skipped += c[k].skipped;
    r.unfit += c[k].unfit;
    if (c[k].nfits == 0) continue;
    vp_plane pl{};
    for (int q = 0; q < 3; ++q) pl.normal[q] = fm[4 * k + q];
    pl.offset = fm[4 * k + 3];
    pl.inlier_count = meta[2 * k];
    pl.cluster_label = meta[2 * k + 1];
    r.models.push_back(pl);
    const uint32_t n = io[2 * k + 1];
    auto in = d2h(g->seg.b.inl + 3ull * (kpoff[K] + kpoff[k]), 3ull * n, g->stream);
    ck(cudaStreamSynchronize(g->stream), "sync");
    r.inliers.insert(r.inliers.end(), in.begin(), in.end());
    r.offsets.push_back(r.offsets.back() + n);
  }
  return r;
}

bool same_fits(const FitResult& a, const FitResult& b) {
  return a.models.size() == b.models.size() && a.offsets == b.offsets && a.skipped == b.skipped &&
         a.unfit == b.unfit && std::memcmp(a.models.data(), b.models.data(), a.models.size() * sizeof(vp_plane)) == 0 &&
         a.inliers.size() == b.inliers.size() &&
         std::memcmp(a.inliers.data(), b.inliers.data(), a.inliers.size() * 8) == 0;
}

// ---- Fig.-9 ablation (pipeline.cpp:304-381) --------------------------------
// CounterRng (rng.hpp:13-64) on the host: the reference's synthetic clusters
// bit for bit (std::log / std::sin / std::cos as in the reference build).
struct HostRng {
  uint64_t st;
  double cached = 0.0;
  bool has = false;
  static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  HostRng(uint64_t seed, uint64_t k1, uint64_t k2) {
    st = mix(seed + 0x9e3779b97f4a7c15ULL);
    st = mix(st ^ mix(k1 + 0xbf58476d1ce4e5b9ULL));
    st = mix(st ^ mix(k2 + 0x94d049bb133111ebULL));
  }
  uint64_t next() {
    st += 0x9e3779b97f4a7c15ULL;
    return mix(st);
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  uint32_t below(uint32_t n) {
    return static_cast<uint32_t>((static_cast<unsigned __int128>(next()) * n) >> 64);
  }
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

// M for (trial, count) and the count x M synthetic members (pipeline.cpp:330-347).
int ablation_points(const vp_ablation_config& c, int trial, int count) {
  HostRng tr(c.seed, static_cast<uint64_t>(count), static_cast<uint64_t>(trial));
  return c.points_min + static_cast<int>(tr.below(static_cast<uint32_t>(c.points_max - c.points_min + 1)));
}

void ablation_clusters(const vp_ablation_config& c, int trial, int count, int m, double* out) {
  auto one = [&](int k) {
    HostRng rng(c.seed ^ 0x5eedULL, static_cast<uint64_t>(trial) << 8 | static_cast<uint64_t>(k), 7);
    const double z0 = rng.uniform(0.0, 0.5);
    double* o = out + 3ull * k * m;
    for (int i = 0; i < m; ++i) {
      const double x = rng.uniform(-0.5, 0.5);
      const double y = rng.uniform(-0.5, 0.5);
      const double z = z0 + 0.004 * rng.normal();
      o[3 * i] = x;
      o[3 * i + 1] = y;
      o[3 * i + 2] = z;
    }
  };
  const int nt = std::min<int>(count, std::max(1u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (int w = 0; w < nt; ++w)
    th.emplace_back([&, w] {
      for (int k = w; k < count; k += nt) one(k);
    });
  for (auto& t : th) t.join();
}

}  // namespace

extern "C" {


int vp_label_components(const vp_steppable_t* s, const vp_seg_params* p, double resolution,
                        int device, int32_t* labels) {
  return guard([&] {
    if (s->count == 0) return;
    vp_grid* g = scratch_grid(device);
    BoxMap bm;
    upload_steppable(g, s, bm);
    const SegDev sd = make_segdev(*p, resolution);
    g->launch_ccl(sd, bm.m);
    ck(cudaMemcpyAsync(labels, g->seg.b.label, 4 * s->count, cudaMemcpyDeviceToHost, g->stream), "labels");
    ck(cudaStreamSynchronize(g->stream), "sync");
  });
}

int vp_build_adjacency(const vp_steppable_t* s, const vp_seg_params* p, double resolution,
                       int device, uint64_t** row_offsets, int32_t** cols, uint64_t* n_edges) {
  return guard([&] {
    const uint32_t S = static_cast<uint32_t>(s->count);
    *row_offsets = static_cast<uint64_t*>(std::calloc(S + 1, 8));
    *cols = nullptr;
    *n_edges = 0;
    if (S == 0) return;
    vp_grid* g = scratch_grid(device);
    BoxMap bm;
    upload_steppable(g, s, bm);
    const SegDev sd = make_segdev(*p, resolution);
    uint32_t* cnt = dalloc<uint32_t>(S);
    LAUNCH(k_adjacency, kWide, kThreads, 0, g->stream, g->ctr, sd, g->seg.b, bm.m, nullptr, cnt, nullptr);
    auto c = d2h(cnt, S, g->stream);
    ck(cudaStreamSynchronize(g->stream), "sync");
    std::vector<uint64_t> rows(S + 1, 0);
    for (uint32_t i = 0; i < S; ++i) rows[i + 1] = rows[i] + c[i];
    uint64_t* drows = dalloc<uint64_t>(S + 1);
    int32_t* dcols = dalloc<int32_t>(rows[S]);
    h2d(drows, rows.data(), S + 1, g->stream);
    LAUNCH(k_adjacency, kWide, kThreads, 0, g->stream, g->ctr, sd, g->seg.b, bm.m, drows, cnt, dcols);
    *cols = static_cast<int32_t*>(std::malloc(rows[S] * 4 + 1));
    if (rows[S]) ck(cudaMemcpyAsync(*cols, dcols, rows[S] * 4, cudaMemcpyDeviceToHost, g->stream), "cols");
    ck(cudaStreamSynchronize(g->stream), "sync");
    std::memcpy(*row_offsets, rows.data(), 8ull * (S + 1));
    *n_edges = rows[S];
    cudaFree(cnt);
    cudaFree(drows);
    cudaFree(dcols);
  });
}

int vp_fit_planes(size_t n_clusters, const int32_t* labels, const uint64_t* offsets,
                  const double* means, const vp_ransac_params* p, int device, vp_fits_t** out) {
  *out = nullptr;
  return guard([&] {
    vp_grid* g = scratch_grid(device);
    const RansacDev rd = make_ransacdev(*p);
    FitResult all;
    for (size_t c0 = 0; c0 < n_clusters; c0 += kClusterBins) {
      const uint32_t K = static_cast<uint32_t>(std::min<size_t>(kClusterBins, n_clusters - c0));
      std::vector<uint32_t> ksize(K);
      for (uint32_t k = 0; k < K; ++k) ksize[k] = static_cast<uint32_t>(offsets[c0 + k + 1] - offsets[c0 + k]);
      const std::vector<uint32_t> kpoff =
          stage_clusters(g, K, labels + c0, ksize.data(), means + 3 * offsets[c0], p->iterations);
      if (p->execution == 1) {
        serial_prepare(g, ksize, kpoff);
        serial_launch(g, rd, kpoff);
      } else {
        g->launch_ransac(rd);
      }
      ck(cudaStreamSynchronize(g->stream), "sync");
      append_fits(all, p->execution == 1 ? serial_results(g, ksize, kpoff) : parallel_results(g));
    }
    auto* f = static_cast<vp_fits_t*>(std::calloc(1, sizeof(vp_fits_t)));
    f->count = all.models.size();
    f->models = static_cast<vp_plane*>(std::malloc(all.models.size() * sizeof(vp_plane) + 1));
    std::memcpy(f->models, all.models.data(), all.models.size() * sizeof(vp_plane));
    f->offsets = static_cast<uint64_t*>(std::malloc(all.offsets.size() * 8));
    std::memcpy(f->offsets, all.offsets.data(), all.offsets.size() * 8);
    f->inliers = static_cast<double*>(std::malloc(all.inliers.size() * 8 + 1));
    std::memcpy(f->inliers, all.inliers.data(), all.inliers.size() * 8);
    f->clusters_skipped_small = all.skipped;
    f->clusters_unfit = all.unfit;
    *out = f;
  });
}

void vp_default_ablation_config(vp_ablation_config* c) {
  std::memset(c, 0, sizeof *c);
  c->trials = 1000;
  c->points_min = 10000;
  c->points_max = 30000;
  c->seed = 1234;
  c->iterations = 100;
  c->inlier_eps = 0.01;
}

int vp_ablation_clusters(const vp_ablation_config* c, int32_t trial, int32_t count, int32_t* m,
                         double** points) {
  *points = nullptr;
  return guard([&] {
    if (count <= 0 || c->points_max < c->points_min || c->points_min < 0)
      fail(VP_EINVAL, "ablation: bad cluster count or point range");
    *m = ablation_points(*c, trial, count);
    *points = static_cast<double*>(std::malloc(3ull * count * *m * sizeof(double) + 8));
    if (!*points) fail(VP_ENOMEM, "host allocation");
    ablation_clusters(*c, trial, count, *m, *points);
  });
}

int vp_run_ablation(const vp_ablation_config* c, vp_ablation_row* rows) {
  return guard([&] {
    if (c->trials <= 0) return;  // pipeline.cpp:309
    if (c->points_max < c->points_min || c->points_min < 0 || c->n_counts < 0)
      fail(VP_EINVAL, "ablation: bad configuration");
    vp_grid* g = scratch_grid(c->device);
    vp_ransac_params rp{};
    rp.iterations = c->iterations;
    rp.inlier_eps = c->inlier_eps;
    rp.seed = c->seed;
    rp.up[2] = 1.0;
    const RansacDev rd = make_ransacdev(rp);
    std::vector<std::vector<double>> par(c->n_counts), ser(c->n_counts);
    cudaEvent_t e0, e1;
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    std::vector<double> pts;
    for (int trial = 0; trial < c->trials; ++trial) {
      for (int ci = 0; ci < c->n_counts; ++ci) {
        const int count = c->cluster_counts[ci];
        if (count <= 0 || count > kClusterBins) fail(VP_EINVAL, "ablation: 1..2048 clusters per row");
        const int m = ablation_points(*c, trial, count);
        pts.resize(3ull * count * m);
        ablation_clusters(*c, trial, count, m, pts.data());
        std::vector<int32_t> labels(count);
        std::vector<uint32_t> ksize(count, static_cast<uint32_t>(m));
        for (int k = 0; k < count; ++k) labels[k] = k;
        const std::vector<uint32_t> kpoff = stage_clusters(g, count, labels.data(), ksize.data(), pts.data(),
                                                           c->iterations);
        serial_prepare(g, ksize, kpoff);
        auto time_mode = [&](bool serial) {
          ck(cudaEventRecord(e0, g->stream), "event");
          if (serial) serial_launch(g, rd, kpoff); else g->launch_ransac(rd);
          ck(cudaEventRecord(e1, g->stream), "event");
          ck(cudaEventSynchronize(e1), "sync");
          float ms = 0.f;
          ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
          return static_cast<double>(ms);
        };
        if (trial % 2 == 0) {
          par[ci].push_back(time_mode(false));
          ser[ci].push_back(time_mode(true));
        } else {
          ser[ci].push_back(time_mode(true));
          par[ci].push_back(time_mode(false));
        }
        const FitResult a = parallel_results(g), b = serial_results(g, ksize, kpoff);
        if (a.models.size() != static_cast<size_t>(count))
          fail(VP_ECUDA, "ablation: cluster dropped during timing");  // pipeline.cpp:353-354
        if (!same_fits(a, b)) fail(VP_ECUDA, "ablation: execution modes disagree");
      }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    auto trimmed_mean = [](std::vector<double>& v) {  // pipeline.cpp:366-372
      std::sort(v.begin(), v.end());
      const size_t trim = v.size() / 10;
      double sum = 0.0;
      for (size_t i = trim; i < v.size() - trim; ++i) sum += v[i];
      return sum / static_cast<double>(v.size() - 2 * trim);
    };
    for (int ci = 0; ci < c->n_counts; ++ci) {
      vp_ablation_row& r = rows[ci];
      r.clusters = c->cluster_counts[ci];
      r.trials = c->trials;
      r.parallel_ms = trimmed_mean(par[ci]);
      r.serial_ms = trimmed_mean(ser[ci]);
      r.parallel_median_ms = par[ci][par[ci].size() / 2];
      r.serial_median_ms = ser[ci][ser[ci].size() / 2];
    }
  });
}

int vp_write_ablation_csv(const char* path, const vp_ablation_row* rows, size_t n) {
  return guard([&] {
    FILE* f = std::fopen(path, "w");
    if (!f) fail(VP_EINVAL, std::string("ablation csv: cannot open for write: ") + path);
    std::fputs("clusters,trials,parallel_ms,serial_ms,ratio,parallel_median_ms,serial_median_ms\n", f);
    for (size_t i = 0; i < n; ++i) {
      const vp_ablation_row& r = rows[i];
      std::fprintf(f, "%d,%d,%.4f,%.4f,%.4f,%.4f,%.4f\n", r.clusters, r.trials, r.parallel_ms, r.serial_ms,
                   r.serial_ms > 0.0 ? r.parallel_ms / r.serial_ms : 0.0, r.parallel_median_ms,
                   r.serial_median_ms);
    }
    std::fclose(f);
  });
}

}  // extern "C"

struct vp_stream {
  unsigned char* buf = nullptr;  // pinned: the whole file
  size_t bytes = 0;
  std::vector<uint64_t> off, n;  // per frame: xyz byte offset, point count
  std::vector<double> pose;      // 12 per frame
  bool pinned = true;
  ~vp_stream() {
    if (buf) {
      if (pinned) cudaFreeHost(buf); else std::free(buf);
    }
  }
};

namespace {
uint32_t le_u32(const unsigned char* p) {
  return static_cast<uint32_t>(p[0]) | static_cast<uint32_t>(p[1]) << 8 | static_cast<uint32_t>(p[2]) << 16 |
         static_cast<uint32_t>(p[3]) << 24;
}
float le_f32(const unsigned char* p) {
  const uint32_t u = le_u32(p);
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
void put_u32(FILE* f, uint32_t v) {
  const unsigned char b[4] = {static_cast<unsigned char>(v), static_cast<unsigned char>(v >> 8),
                              static_cast<unsigned char>(v >> 16), static_cast<unsigned char>(v >> 24)};
  std::fwrite(b, 1, 4, f);
}
void put_f32(FILE* f, float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  put_u32(f, u);
}
}  // namespace

extern "C" {

int vp_stream_open(const char* path, vp_stream** out) {
  *out = nullptr;
  return guard([&] {
    FILE* f = std::fopen(path, "rb");
    if (!f) fail(VP_EINVAL, std::string("frame stream: cannot open: ") + path);
    std::fseek(f, 0, SEEK_END);
    const long len = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    auto* s = new vp_stream();
    struct Del {
      vp_stream*& s;
      ~Del() { delete s; }
    } del{s};
    s->bytes = len > 0 ? static_cast<size_t>(len) : 0;
    // pinned when a device is present (async H2D in replay); plain host
    // memory otherwise (reading a stream needs no device)
    if (cudaHostAlloc(reinterpret_cast<void**>(&s->buf), s->bytes + 1, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      s->pinned = false;
      s->buf = static_cast<unsigned char*>(std::malloc(s->bytes + 1));
      if (!s->buf) {
        std::fclose(f);
        fail(VP_ENOMEM, "frame stream: host allocation failed");
      }
    }
    const size_t got = std::fread(s->buf, 1, s->bytes, f);
    std::fclose(f);
    if (got != s->bytes) fail(VP_EINVAL, std::string("frame stream: read failed: ") + path);
    if (s->bytes < 4 || std::memcmp(s->buf, "VXPF", 4) != 0)
      fail(VP_EINVAL, std::string("frame stream: bad magic in ") + path);
    if (s->bytes < 8 || le_u32(s->buf + 4) != 1) fail(VP_EINVAL, "frame stream: unsupported version");
    size_t o = 8;
    while (o < s->bytes) {  // frame_io.cpp:102-113; short reads throw (frame_io.cpp:28)
      if (o + 52 > s->bytes) fail(VP_EINVAL, "frame stream: truncated file");
      const uint64_t n = le_u32(s->buf + o);
      for (int k = 0; k < 12; ++k) s->pose.push_back(static_cast<double>(le_f32(s->buf + o + 4 + 4 * k)));
      o += 52;
      if (o + 12 * n > s->bytes) fail(VP_EINVAL, "frame stream: truncated file");
      s->off.push_back(o);
      s->n.push_back(n);
      o += 12 * n;
    }
    // little-endian host: the xyz payload is used in place
    *out = s;
    s = nullptr;
  });
}

void vp_stream_close(vp_stream* s) { delete s; }

uint64_t vp_stream_count(const vp_stream* s) { return s ? s->n.size() : 0; }

int vp_stream_frame(const vp_stream* s, uint64_t i, const float** xyz, uint64_t* n, double rotation[9],
                    double translation[3]) {
  return guard([&] {
    if (i >= s->n.size()) fail(VP_EINVAL, "frame stream: frame index out of range");
    *xyz = reinterpret_cast<const float*>(s->buf + s->off[i]);
    *n = s->n[i];
    const double* q = s->pose.data() + 12 * i;  // [R|t] row-major
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) rotation[3 * r + c] = q[4 * r + c];
      translation[r] = q[4 * r + 3];
    }
  });
}

int vp_write_frames_binary(const char* path, size_t n_frames, const float* const* xyz, const uint64_t* n,
                           const double* rotations, const double* translations) {
  return guard([&] {
    FILE* f = std::fopen(path, "wb");
    if (!f) fail(VP_EINVAL, std::string("frame stream: cannot open for write: ") + path);
    std::fwrite("VXPF", 1, 4, f);
    put_u32(f, 1);
    for (size_t k = 0; k < n_frames; ++k) {
      put_u32(f, static_cast<uint32_t>(n[k]));
      for (int r = 0; r < 3; ++r) {  // put_pose: f32 [R|t] row-major
        for (int c = 0; c < 3; ++c) put_f32(f, static_cast<float>(rotations[9 * k + 3 * r + c]));
        put_f32(f, static_cast<float>(translations[3 * k + r]));
      }
      for (uint64_t i = 0; i < 3 * n[k]; ++i) put_f32(f, xyz[k][i]);
    }
    const bool ok = std::ferror(f) == 0;
    std::fclose(f);
    if (!ok) fail(VP_EINVAL, std::string("frame stream: write failed: ") + path);
  });
}

int vp_write_polygons(const char* path, const vp_polygons_t* polygons) {
  return guard([&] {
    FILE* f = std::fopen(path, "w");
    if (!f) fail(VP_EINVAL, std::string("polygons: cannot open for write: ") + path);
    std::fputs("# voxplane polygons v1\n", f);
    for (size_t i = 0; i < (polygons ? polygons->count : 0); ++i) {
      const vp_polygon& q = polygons->polys[i];
      std::fprintf(f, "polygon\nnormal %.9g %.9g %.9g\noffset %.9g\nvertices %u\n", q.plane.normal[0],
                   q.plane.normal[1], q.plane.normal[2], q.plane.offset, q.nverts);
      for (uint32_t k = 0; k < q.nverts; ++k)
        std::fprintf(f, "%.9g %.9g %.9g\n", q.v3d[3 * k], q.v3d[3 * k + 1], q.v3d[3 * k + 2]);
      std::fprintf(f, "area %.9g\nlabel %d\ninliers %d\n", q.area, q.plane.cluster_label, q.plane.inlier_count);
    }
    const bool ok = std::ferror(f) == 0;
    std::fclose(f);
    if (!ok) fail(VP_EINVAL, std::string("polygons: write failed: ") + path);
  });
}

void vp_fits_free(vp_fits_t* f) {
  if (!f) return;
  std::free(f->models);
  std::free(f->offsets);
  std::free(f->inliers);
  std::free(f);
}

}  // extern "C"

namespace {
// Upload (plane, inlier set) batches as "fits" of the scratch grid.
// to_ref: the planes go to ref_model (make_polygon input) instead of fit_model
// (refine input). A selector, not a pointer: ensure() below may reallocate.
void upload_fit_batch(vp_grid* g, size_t f0, uint32_t F, const vp_plane* planes,
                      const uint64_t* offsets, const double* inliers, bool to_ref) {
  std::vector<double> fm(4ull * F);
  std::vector<int32_t> meta(2ull * F);
  std::vector<uint32_t> io(F + 1);
  const uint64_t base = offsets[f0];
  for (uint32_t f = 0; f < F; ++f) {
    for (int q = 0; q < 3; ++q) fm[4 * f + q] = planes[f0 + f].normal[q];
    fm[4 * f + 3] = planes[f0 + f].offset;
    meta[2 * f] = planes[f0 + f].inlier_count;
    meta[2 * f + 1] = planes[f0 + f].cluster_label;
    io[f] = static_cast<uint32_t>(offsets[f0 + f] - base);
  }
  io[F] = static_cast<uint32_t>(offsets[f0 + F] - base);
  const uint32_t tot = io[F];
  g->seg.ensure(g->seg.b.Vcap, g->seg.b.Scap, std::max(g->seg.b.Icap, tot), 100, g->gd.nwords);
  h2d(to_ref ? g->seg.b.ref_model : g->seg.b.fit_model, fm.data(), fm.size(), g->stream);
  h2d(g->seg.b.fit_meta, meta.data(), meta.size(), g->stream);
  h2d(g->seg.b.ioff, io.data(), io.size(), g->stream);
  h2d(g->seg.b.inl, inliers + 3 * base, 3ull * tot, g->stream);
  g->reset_frame_counters();
  set_counter_u32(g, offsetof(Counters, nfits), F);
}
}  // namespace

extern "C" {


int vp_refine_planes(const vp_fits_t* fits, const double up[3], int exact, int device,
                     vp_plane* refined) {
  return guard([&] {
    vp_grid* g = scratch_grid(device);
    for (size_t f0 = 0; f0 < fits->count; f0 += kClusterBins) {
      const uint32_t F = static_cast<uint32_t>(std::min<size_t>(kClusterBins, fits->count - f0));
      upload_fit_batch(g, f0, F, fits->models, fits->offsets, fits->inliers, false);
      g->launch_refine(up, 1, exact);
      auto rm = d2h(g->seg.b.ref_model, 4ull * F, g->stream);
      ck(cudaStreamSynchronize(g->stream), "sync");
      for (uint32_t f = 0; f < F; ++f) {
        refined[f0 + f] = fits->models[f0 + f];  // pipeline.cpp:76-77 keep count/label
        for (int q = 0; q < 3; ++q) refined[f0 + f].normal[q] = rm[4 * f + q];
        refined[f0 + f].offset = rm[4 * f + 3];
      }
    }
  });
}

int vp_make_polygons(size_t n, const vp_plane* planes, const uint64_t* offsets,
                     const double* inliers, int filter_directions, int device, vp_polygons_t** out) {
  *out = nullptr;
  return guard([&] {
    vp_grid* g = scratch_grid(device);
    HostPolys all;
    std::vector<double> verts;
    for (size_t f0 = 0; f0 < n || (f0 == 0 && n == 0); f0 += kClusterBins) {
      if (n == 0) break;
      const uint32_t F = static_cast<uint32_t>(std::min<size_t>(kClusterBins, n - f0));
      upload_fit_batch(g, f0, F, planes, offsets, inliers, true);
      g->launch_polygon(filter_directions, -std::numeric_limits<double>::infinity());
      g->read_counters();
      if (g->h_ctr->overflow & kOverflowPool) fail(VP_ENOMEM, "polygon vertex pool overflow");
      HostPolys hp;
      g->download_polygons(hp, true);
      const size_t vbase = all.verts.size() / 5;
      for (auto q : hp.polys) {
        q.v2d = reinterpret_cast<const double*>(reinterpret_cast<uintptr_t>(q.v2d) + vbase);
        all.polys.push_back(q);
      }
      all.verts.insert(all.verts.end(), hp.verts.begin(), hp.verts.end());
    }
    *out = make_polygons_out(all);
  });
}

void vp_polygons_free(vp_polygons_t* p) { std::free(p); }

int vp_pipeline_latency_ms(const vp_pipeline* pl, double* ms) {
  return guard([&] { *ms = static_cast<double>(pl->last_latency_ms); });
}

}  // extern "C"

// Accessors for the slab-frame orchestration (slab_frame.cu).
namespace vp {
void set_last_error(const char* msg) { g_err = msg; }
cudaStream_t slab_stream(vp_grid* g) { return g->stream; }
void slab_geometry(vp_grid* g, int32_t* xb, int32_t* xe, int32_t* gex, int* device, double* res) {
  *xb = g->gd.xoff + g->gd.own_lo;
  *xe = g->gd.xoff + g->gd.own_hi;
  *gex = g->gd.gex;
  *device = g->device;
  *res = g->gd.res;
}
}  // namespace vp

extern "C" {

int vp_slab_create(double res, const int32_t window_extent[3], const double center[3],
                   int32_t x_begin, int32_t x_end, int device, vp_grid** out) {
  *out = nullptr;
  return guard([&] {
    auto* g = new vp_grid();
    try {
      g->init_slab(res, window_extent, center, x_begin, x_end, device);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int vp_grid_plane(vp_grid* g, int32_t window_x, void** cells, uint64_t* cell_bytes, void** bits,
                  uint64_t* bit_bytes) {
  return guard([&] {
    const int32_t lx = window_x - g->gd.xoff;
    if (lx < 0 || lx >= g->gd.ex) fail(VP_EINVAL, "grid_plane: x outside this grid");
    if (g->off[0] || g->off[1] || g->off[2]) fail(VP_EINVAL, "grid_plane: window was recentered");
    const uint64_t plane = static_cast<uint64_t>(g->gd.ey) * g->gd.ez;
    const uint64_t wplane = static_cast<uint64_t>(g->gd.ey) * g->gd.W;
    *cells = g->gd.cells + lx * plane;
    *cell_bytes = plane * sizeof(Cell);
    *bits = g->occ[g->cur] + lx * wplane;
    *bit_bytes = wplane * 4;
  });
}

int vp_slab_steppable(vp_grid* g, const vp_seg_params* p, uint64_t* count, int32_t** idx,
                      double** mean, double** normal) {
  return guard([&] {
    const SegDev sd = make_segdev(*p, g->gd.res);
    MapDesc none{};
    for (int tries = 0;; ++tries) {
      g->fill_static_params();
      g->h_fp->n = 0;
      g->upload_params();
      g->reset_frame_counters();
      g->launch_occupied_scan();
      g->launch_classify(sd, 1);
      g->launch_step_emit(none, g->gd.xoff);
      g->read_counters();
      if (!(g->h_ctr->overflow & (kOverflowOcc | kOverflowStep)) || tries > 4) break;
      const uint32_t need = static_cast<uint32_t>(std::min<uint64_t>(g->gd.ncells, 2ull * g->h_ctr->V));
      g->seg.ensure(std::max(need, g->seg.b.Vcap), std::max(need, g->seg.b.Scap), g->seg.b.Icap,
                    100, g->gd.nwords);
    }
    *count = g->h_ctr->S;
    *idx = g->seg.b.st_idx;
    *mean = g->seg.b.st_mean;
    *normal = g->seg.b.st_normal;
  });
}

int vp_segment_steppable(vp_grid* g, const vp_pipeline_params* p, uint64_t S, const int32_t* idx,
                         const double* mean, const double* normal, int device_ptrs,
                         vp_polygons_t** out) {
  if (out) *out = nullptr;
  return guard([&] {
    const uint32_t n = static_cast<uint32_t>(S);
    const SegDev sd = make_segdev(p->seg, g->gd.res);
    const RansacDev rd = make_ransacdev(p->ransac);
    cudaMemcpyKind kind = device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    // the lists may be this grid's own steppable buffers (vp_slab_steppable),
    // which a capacity retry below reallocates: stage them aside first
    int32_t* stage = nullptr;
    if (S && idx == g->seg.b.st_idx) {
      stage = dalloc<int32_t>(15 * S);
      ck(cudaMemcpyAsync(stage, idx, 12 * S, cudaMemcpyDeviceToDevice, g->stream), "stage idx");
      ck(cudaMemcpyAsync(stage + 3 * S, mean, 24 * S, cudaMemcpyDeviceToDevice, g->stream), "stage mean");
      ck(cudaMemcpyAsync(stage + 9 * S, normal, 24 * S, cudaMemcpyDeviceToDevice, g->stream), "stage nrm");
      idx = stage;
      mean = reinterpret_cast<const double*>(stage + 3 * S);
      normal = reinterpret_cast<const double*>(stage + 9 * S);
      kind = cudaMemcpyDeviceToDevice;
    }
    struct Free {
      int32_t* p;
      ~Free() { if (p) cudaFree(p); }
    } free_stage{stage};
    g->seg.ensure(std::max(n, g->seg.b.Vcap), std::max(n, g->seg.b.Scap), std::max(n, g->seg.b.Icap),
                  p->ransac.iterations, g->gd.nwords);
    g->seg.ensure_dirs(16, g->stream);
    const MapDesc m = g->window_map();
    for (int tries = 0;; ++tries) {
      if (S) {  // (re)load the lists: a retry's ensure() reallocated the buffers
        ck(cudaMemcpyAsync(g->seg.b.st_idx, idx, 12 * S, kind, g->stream), "st idx");
        ck(cudaMemcpyAsync(g->seg.b.st_mean, mean, 24 * S, kind, g->stream), "st mean");
        ck(cudaMemcpyAsync(g->seg.b.st_normal, normal, 24 * S, kind, g->stream), "st normal");
      }
      g->fill_static_params();
      g->h_fp->n = 0;
      g->upload_params();
      g->reset_frame_counters();
      set_counter_u32(g, offsetof(Counters, S), n);
      LAUNCH(k_map_fill, kWide, kThreads, 0, g->stream, g->ctr, g->seg.b, m);
      g->launch_ccl(sd, m);
      g->launch_clusters(sd);
      g->launch_ransac(rd);
      g->launch_refine(p->ransac.up, p->refine, p->refine_exact);
      g->launch_polygon(16, p->min_polygon_area);
      g->read_counters();
      if (!g->h_ctr->overflow || tries > 4) break;
      if (g->h_ctr->overflow & kOverflowClusters) g->seg.grow_k(g->h_ctr->K, g->h_ctr->S, p->ransac.iterations);
      else g->seg.ensure(g->seg.b.Vcap, g->seg.b.Scap, 2 * g->seg.b.Icap, p->ransac.iterations, g->gd.nwords);
    }
    if (out) {
      HostPolys hp;
      g->download_polygons(hp, false);
      *out = make_polygons_out(hp);
    }
  });
}

static_assert(sizeof(vp_member_rec) == sizeof(MemberRec), "vp_member_rec must match MemberRec");

int vp_adjacency_window(const vp_seg_params* p, double resolution, int32_t* w) {
  return guard([&] {
    // segmentation.cpp:89
    *w = std::max(1, static_cast<int>(std::ceil(p->distance_th / resolution)));
  });
}

int vp_slab_plane_counts(vp_grid* g, uint32_t** counts, int32_t* n_planes) {
  return guard([&] {
    SlabSeg& L = g->sl;
    const int32_t np = g->gd.own_hi - g->gd.own_lo;
    if (np > L.pcap) {
      dfree(L.pcounts);
      L.pcounts = dalloc<uint32_t>(np);
      L.pcap = np;
    }
    LAUNCH(k_plane_counts, grid_for(np), kThreads, 0, g->stream, g->ctr, g->seg.b.st_idx, g->seg.b.Scap,
           g->gd.xoff + g->gd.own_lo, np, L.pcounts);
    ck(cudaStreamSynchronize(g->stream), "sync");
    *counts = L.pcounts;
    *n_planes = np;
  });
}

int vp_slab_extend(vp_grid* g, const vp_seg_params* p, const vp_slab_layout* lay, int32_t** idx,
                   double** mean, double** normal, uint64_t* n_ext, int32_t* x_lo, int32_t* x_hi) {
  return guard([&] {
    SlabSeg& L = g->sl;
    const int n = lay->n_slabs;
    if (n < 1 || n > kMaxSlabs) fail(VP_EINVAL, "slab layout: 1..64 slabs");
    const int32_t gex = g->gd.gex;
    if (lay->x_begin[0] != 0 || lay->x_begin[n] != gex) fail(VP_EINVAL, "slab layout: x ranges must tile the window");
    L.n = n;
    L.xb.assign(lay->x_begin, lay->x_begin + n + 1);
    const int32_t my_xb = g->gd.xoff + g->gd.own_lo, my_xe = g->gd.xoff + g->gd.own_hi;
    L.me = -1;
    for (int k = 0; k < n; ++k) {
      if (L.xb[k] >= L.xb[k + 1]) fail(VP_EINVAL, "slab layout: empty or unordered x range");
      if (L.xb[k] == my_xb && L.xb[k + 1] == my_xe) L.me = k;
    }
    if (L.me < 0) fail(VP_EINVAL, "slab layout: this slab's x range is not in the layout");
    L.P.assign(gex + 1, 0);
    for (int32_t x = 0; x < gex; ++x) L.P[x + 1] = L.P[x] + lay->plane_counts[x];
    if (L.P[gex] >= (1ull << 31)) fail(VP_ENOMEM, "more than 2^31 steppable voxels in the window");
    L.w = std::max(1, static_cast<int>(std::ceil(p->distance_th / g->gd.res)));  // segmentation.cpp:89
    L.x_lo = std::max(0, my_xb - L.w);
    L.x_hi = std::min(gex, my_xe + L.w);
    L.base = static_cast<int64_t>(L.P[L.x_lo]);
    L.own_base = static_cast<int64_t>(L.P[my_xb]);
    L.n_left = L.P[my_xb] - L.P[L.x_lo];
    L.n_own = L.P[my_xe] - L.P[my_xb];
    L.n_ext = L.P[L.x_hi] - L.P[L.x_lo];
    if (L.n_own != g->h_ctr->S) fail(VP_EINVAL, "slab layout: plane counts disagree with this slab's steppable list");
    // boundary zone: [B - w, B + w) around every internal boundary, merged
    L.zone = ZoneDesc{};
    L.zone_size = 0;
    for (int k = 1; k < n; ++k) {
      const int32_t a = std::max(0, L.xb[k] - L.w), b = std::min(gex, L.xb[k] + L.w);
      ZoneDesc& z = L.zone;
      if (z.n && a <= z.xhi[z.n - 1]) {
        z.xhi[z.n - 1] = std::max(z.xhi[z.n - 1], b);
      } else {
        z.xlo[z.n] = a;
        z.xhi[z.n] = b;
        ++z.n;
      }
    }
    for (int k = 0; k < L.zone.n; ++k) {
      L.zone.olo[k] = static_cast<int64_t>(L.P[L.zone.xlo[k]]);
      L.zone.dbase[k] = static_cast<int64_t>(L.zone_size);
      L.zone_size += L.P[L.zone.xhi[k]] - L.P[L.zone.xlo[k]];
    }
    L.rd = RankDesc{};
    L.rd.n = n;
    for (int k = 0; k < n; ++k) L.rd.ord_lo[k] = static_cast<int64_t>(L.P[L.xb[k]]);
    // extended list buffers; the own list moves in before any seg realloc
    if (L.n_ext > L.xcap) {
      // generous first size (the list grows with the map): no cudaMalloc in steady state
      const uint64_t cap = std::max<uint64_t>({L.n_ext + L.n_ext / 2, 2 * L.xcap, g->seg.b.Scap, 1 << 16});
      for (void* q : {(void*)L.xidx, (void*)L.xmean, (void*)L.xnrm, (void*)L.bmin, (void*)L.flabel})
        if (q) cudaFree(q);
      L.xidx = dalloc<int32_t>(3 * cap);
      L.xmean = dalloc<double>(3 * cap);
      L.xnrm = dalloc<double>(3 * cap);
      L.bmin = dalloc<int32_t>(cap);
      L.flabel = dalloc<int32_t>(cap);
      L.xcap = cap;
    }
    if (L.n_own) {
      ck(cudaMemcpyAsync(L.xidx + 3 * L.n_left, g->seg.b.st_idx, 12 * L.n_own, cudaMemcpyDeviceToDevice, g->stream), "ext idx");
      ck(cudaMemcpyAsync(L.xmean + 3 * L.n_left, g->seg.b.st_mean, 24 * L.n_own, cudaMemcpyDeviceToDevice, g->stream), "ext mean");
      ck(cudaMemcpyAsync(L.xnrm + 3 * L.n_left, g->seg.b.st_normal, 24 * L.n_own, cudaMemcpyDeviceToDevice, g->stream), "ext nrm");
    }
    ck(cudaStreamSynchronize(g->stream), "sync");
    const uint32_t need = static_cast<uint32_t>(L.n_ext);
    if (need > g->seg.b.Scap)
      g->seg.ensure(g->seg.b.Vcap, need, std::max(g->seg.b.Icap, need), 100, g->gd.nwords);
    // dense ordinal map over the extended planes
    const uint64_t slots = static_cast<uint64_t>(L.x_hi - L.x_lo) * g->gd.ey * g->gd.ez;
    const uint64_t words = static_cast<uint64_t>(L.x_hi - L.x_lo) * g->gd.ey * g->gd.W;
    if (slots > L.xmap_slots) {
      dfree(L.xmap);
      dfree(L.xbits);
      L.xmap = dalloc<int32_t>(slots);
      L.xbits = dalloc<uint32_t>(words);
      ck(cudaMemsetAsync(L.xmap, 0xff, slots * 4, g->stream), "xmap");
      ck(cudaMemsetAsync(L.xbits, 0, words * 4, g->stream), "xbits");
      ck(cudaStreamSynchronize(g->stream), "sync");
      L.xmap_slots = slots;
      L.xmap_words = words;
    }
    L.labelled = L.merged = false;
    *idx = L.xidx;
    *mean = L.xmean;
    *normal = L.xnrm;
    *n_ext = L.n_ext;
    *x_lo = L.x_lo;
    *x_hi = L.x_hi;
  });
}

int vp_slab_label(vp_grid* g, const vp_seg_params* p, int32_t** triples, uint64_t* n_triples,
                  uint64_t* zone_size) {
  return guard([&] {
    SlabSeg& L = g->sl;
    if (L.me < 0) fail(VP_EINVAL, "slab_label: call vp_slab_extend first");
    const SegDev sd = make_segdev(*p, g->gd.res);
    SegBufs sb = g->seg.b;
    sb.st_idx = L.xidx;
    sb.st_mean = L.xmean;
    sb.st_normal = L.xnrm;
    sb.Scap = static_cast<uint32_t>(std::min<uint64_t>(L.xcap, g->seg.b.Scap));
    MapDesc m{};
    m.map = L.xmap;
    m.bits = L.xbits;
    m.lo[0] = L.x_lo;
    m.lo[1] = m.lo[2] = 0;
    m.dims[0] = L.x_hi - L.x_lo;
    m.dims[1] = g->gd.ey;
    m.dims[2] = g->gd.ez;
    m.W = g->gd.W;
    // count of zone entries bounds the triples
    uint64_t zent = 0;
    for (int k = 0; k < L.zone.n; ++k) {
      const int32_t a = std::max(L.zone.xlo[k], L.x_lo), b = std::min(L.zone.xhi[k], L.x_hi);
      if (a < b) zent += L.P[b] - L.P[a];
    }
    if (zent > L.tcap || !L.triples) {
      dfree(L.triples);
      L.tcap = std::max<uint64_t>({zent + zent / 2, 2 * L.tcap, 1 << 20});
      L.triples = dalloc<int32_t>(3 * L.tcap);
      if (!L.ntrip) L.ntrip = dalloc<uint32_t>(1);
    }
    g->reset_frame_counters();
    set_counter_u32(g, offsetof(Counters, S), static_cast<uint32_t>(L.n_ext));
    if (L.n_ext) {
      LAUNCH(k_map_fill, kWide, kThreads, 0, g->stream, g->ctr, sb, m);
      g->launch_ccl(sd, m, sb);
      LAUNCH(k_fill_i32, grid_for(L.n_ext), kThreads, 0, g->stream, L.bmin, L.n_ext, 0x7fffffff);
    }
    ck(cudaMemsetAsync(L.ntrip, 0, 4, g->stream), "ntrip");
    if (L.n_ext && L.zone.n) {
      LAUNCH(k_zone_bmin, kWide, kThreads, 0, g->stream, g->ctr, sb, L.zone, L.bmin);
      LAUNCH(k_zone_triples, kWide, kThreads, 0, g->stream, g->ctr, sb, L.zone, L.base, L.bmin, L.triples,
             L.ntrip);
    }
    uint32_t nt = 0;
    ck(cudaMemcpyAsync(&nt, L.ntrip, 4, cudaMemcpyDeviceToHost, g->stream), "ntrip");
    ck(cudaStreamSynchronize(g->stream), "sync");
    if (nt != zent) fail(VP_ECUDA, "slab_label: zone entry count mismatch");
    L.labelled = true;
    *triples = L.triples;
    *n_triples = nt;
    *zone_size = L.zone_size;
  });
}

int vp_slab_merge(vp_grid* g, const int32_t* triples, uint64_t n_triples, int32_t** labels) {
  return guard([&] {
    SlabSeg& L = g->sl;
    if (!L.labelled) fail(VP_EINVAL, "slab_merge: call vp_slab_label first");
    if (L.zone_size > L.zcap || !L.zparent) {
      dfree(L.zparent);
      dfree(L.zminlab);
      L.zcap = std::max<uint64_t>({L.zone_size + L.zone_size / 2, 2 * L.zcap, 1 << 20});
      L.zparent = dalloc<int32_t>(L.zcap);
      L.zminlab = dalloc<int32_t>(L.zcap);
    }
    if (L.zone_size) {
      LAUNCH(k_zone_init, grid_for(L.zone_size), kThreads, 0, g->stream, L.zparent, L.zminlab, L.zone_size);
      if (n_triples) {
        LAUNCH(k_zone_union, grid_for(n_triples), kThreads, 0, g->stream, triples, n_triples, L.zparent);
        LAUNCH(k_zone_minlab, grid_for(n_triples), kThreads, 0, g->stream, triples, n_triples, L.zparent,
               L.zminlab);
      }
    }
    SegBufs sb = g->seg.b;
    sb.st_idx = L.xidx;
    if (L.n_own)
      LAUNCH(k_slab_relabel, grid_for(L.n_own), kThreads, 0, g->stream, sb, L.zone, L.base,
             static_cast<uint32_t>(L.n_left), static_cast<uint32_t>(L.n_own), L.bmin, L.zparent, L.zminlab,
             L.flabel);
    ck(cudaStreamSynchronize(g->stream), "sync");
    L.merged = true;
    *labels = L.flabel;
  });
}

int vp_slab_export(vp_grid* g, uint64_t* dest_counts, void** records) {
  return guard([&] {
    SlabSeg& L = g->sl;
    if (!L.merged) fail(VP_EINVAL, "slab_export: call vp_slab_merge first");
    const uint32_t n_own = static_cast<uint32_t>(L.n_own);
    const uint32_t nch = std::max<uint32_t>(1, (n_own + kChunk - 1) / kChunk);
    const uint64_t hn = static_cast<uint64_t>(L.n) * nch;
    if (hn > L.hcap || !L.H) {
      dfree(L.H);
      L.hcap = std::max<uint64_t>({hn + hn / 2, 2 * L.hcap, 1 << 18});
      L.H = dalloc<uint32_t>(L.hcap);
      if (!L.dcount) L.dcount = dalloc<uint32_t>(kMaxSlabs);
    }
    ck(cudaMemsetAsync(L.dcount, 0, 4 * kMaxSlabs, g->stream), "dcount");
    ck(cudaMemsetAsync(L.H, 0, 4 * hn, g->stream), "H");
    const int blocks = static_cast<int>(std::min<uint32_t>(nch, 148 * 16));
    if (n_own)
      LAUNCH(k_export_hist, blocks, 32, 0, g->stream, n_own, L.flabel, L.rd, L.me, L.H, nch, L.dcount);
    uint32_t dc[kMaxSlabs];
    ck(cudaMemcpyAsync(dc, L.dcount, 4 * kMaxSlabs, cudaMemcpyDeviceToHost, g->stream), "dcount");
    ck(cudaStreamSynchronize(g->stream), "sync");
    uint64_t tot = 0;
    for (int k = 0; k < L.n; ++k) {
      dest_counts[k] = dc[k];
      tot += dc[k];
    }
    if (tot > L.ecap || !L.exp) {
      dfree(L.exp);
      L.ecap = std::max<uint64_t>({tot + tot / 2, 2 * L.ecap, 1 << 20});
      L.exp = dalloc<MemberRec>(L.ecap);
    }
    if (tot) {
      if (hn > 0xffffffffull) fail(VP_ENOMEM, "slab_export: histogram too large");
      LAUNCH(k_scan_exclusive, 1, 1024, 0, g->stream, L.H, static_cast<uint32_t>(hn), nullptr, nullptr, nullptr);
      LAUNCH(k_export_scatter, blocks, 32, 0, g->stream, n_own, L.flabel, L.xmean + 3 * L.n_left, L.rd, L.me,
             L.H, nch, L.exp);
    }
    ck(cudaStreamSynchronize(g->stream), "sync");
    *records = L.exp;
  });
}

int vp_slab_segment_owned(vp_grid* g, const vp_pipeline_params* p, const void* recv, uint64_t n_recv,
                          vp_polygons_t** out) {
  if (out) *out = nullptr;
  return guard([&] {
    SlabSeg& L = g->sl;
    if (!L.merged) fail(VP_EINVAL, "slab_segment_owned: call vp_slab_merge first");
    const uint32_t n = static_cast<uint32_t>(L.n_own + n_recv);
    const SegDev sd = make_segdev(p->seg, g->gd.res);
    const RansacDev rd = make_ransacdev(p->ransac);
    g->seg.ensure(g->seg.b.Vcap, std::max(n, g->seg.b.Scap), std::max(n, g->seg.b.Icap), p->ransac.iterations,
                  g->gd.nwords);
    g->seg.ensure_dirs(16, g->stream);
    for (int tries = 0;; ++tries) {
      g->reset_frame_counters();
      set_counter_u32(g, offsetof(Counters, S), n);
      if (n) {
        LAUNCH(k_owner_init, grid_for(n), kThreads, 0, g->stream, n, g->seg.b);
        LAUNCH(k_owner_prep, grid_for(n), kThreads, 0, g->stream, static_cast<uint32_t>(L.n_own),
               static_cast<uint32_t>(n_recv), L.own_base, L.xmean + 3 * L.n_left, L.flabel,
               static_cast<const MemberRec*>(recv), g->seg.b);
      }
      g->launch_clusters(sd, L.own_base);  // cluster labels = global ordinals
      g->launch_ransac(rd);
      g->launch_refine(p->ransac.up, p->refine, p->refine_exact);
      g->launch_polygon(16, p->min_polygon_area);
      g->read_counters();
      if (tries > 4 || !g->grow_if_overflow(p->ransac.iterations)) break;
    }
    if (g->h_ctr->overflow) fail(VP_ENOMEM, "segmentation capacity overflow persists");
    if (out) {
      HostPolys hp;
      g->download_polygons(hp, false);
      *out = make_polygons_out(hp);
    }
  });
}

int vp_segment(vp_grid* g, const vp_pipeline_params* p, vp_polygons_t** out,
               vp_frame_timing* timing) {
  if (out) *out = nullptr;
  return guard([&] {
    g->fill_static_params();
    g->h_fp->n = 0;
    g->upload_params();
    g->reset_frame_counters();
    ck(cudaEventRecord(g->ev[0], g->stream), "ev");
    g->launch_segment(*p, true);
    g->read_counters();
    rerun_segment_until_fits(g, *p);
    fill_timing(g, timing, 0);
    if (timing) timing->mapping_ms = 0.0;
    HostPolys hp;
    g->download_polygons(hp, false);
    if (out) *out = make_polygons_out(hp);
  });
}

int vp_pipeline_create(double res, const int32_t extent[3], const double start_center[3],
                       const vp_pipeline_params* p, int device, vp_pipeline** out) {
  *out = nullptr;
  return guard([&] {
    auto* pl = new vp_pipeline();
    try {
      pl->grid = new vp_grid();
      pl->grid->init(res, extent, start_center, device);
    } catch (...) {
      delete pl;
      throw;
    }
    if (p) pl->p = *p; else vp_default_params(&pl->p);
    global_cell(start_center, res, pl->last_cell);  // pipeline.cpp:174
    *out = pl;
  });
}

void vp_pipeline_destroy(vp_pipeline* pl) { delete pl; }

int vp_pipeline_reset(vp_pipeline* pl, const double start_center[3]) {
  return guard([&] { pl->grid->reset(start_center); global_cell(start_center, pl->grid->gd.res, pl->last_cell); pl->frame = 0; });
}

vp_grid* vp_pipeline_grid(vp_pipeline* pl) { return pl->grid; }

void* vp_pipeline_stream(vp_pipeline* pl) { return pl->grid->stream; }

int vp_grid_counters(vp_grid* g, uint64_t out[16]) {
  return guard([&] {
    const Counters& c = *g->h_ctr;
    const uint64_t v[16] = {c.cleared, c.freed, c.touched, c.discarded, c.dropped, c.occupied,
                            c.V, c.S, c.K, c.nfits, c.padded_members, c.inliers, c.pool_used,
                            c.newly, c.surv_max, c.overflow};
    std::memcpy(out, v, sizeof v);
  });
}

int vp_pipeline_counters(vp_pipeline* pl, uint64_t out[16]) {
  return guard([&] {
    const Counters& c = *pl->grid->h_ctr;
    const uint64_t v[16] = {c.cleared, c.freed, c.touched, c.discarded, c.dropped, c.occupied,
                            c.V, c.S, c.K, c.nfits, c.padded_members, c.inliers, c.pool_used,
                            c.newly, c.surv_max, c.overflow};
    std::memcpy(out, v, sizeof v);
  });
}

static int pipeline_frame_impl(vp_pipeline* pl, const float* xyz, uint64_t n, const double* R,
                               const double* t, bool device_ptr, vp_polygons_t** out,
                               vp_frame_timing* timing) {
  if (out) *out = nullptr;
  return guard([&] {
    // VP_LAT_STATS: where one frame's latency goes (host phases, GPU gaps)
    static const bool lat_stats = std::getenv("VP_LAT_STATS") != nullptr;
    using clk = std::chrono::steady_clock;
    const auto h0 = clk::now();
    vp_shift_stats ss;
    pipeline_enqueue(pl, xyz, n, R, t, device_ptr, &ss);
    const auto h1 = clk::now();
    vp_grid* g = pl->grid;
    wait_frame(g);
    const auto h2 = clk::now();
    const bool rerun = g->h_ctr->overflow != 0;
    if (rerun) rerun_segment_until_fits(g, pl->p);
    fill_timing(g, timing, n);
    const auto h2b = clk::now();
    clk::time_point h2c = h2b;
    if (out) {
      HostPolys hp;
      if (rerun || !unpack_polygons(pl->pack1_h, hp)) g->download_polygons(hp, false);
      h2c = clk::now();
      *out = make_polygons_out(hp);
    }
    const auto h3 = clk::now();
    // the polygons are in host memory: the frame's end to end latency
    ck(cudaEventRecord(pl->lat_ev[1], g->stream), "event");
    ck(cudaEventSynchronize(pl->lat_ev[1]), "event");
    ck(cudaEventElapsedTime(&pl->last_latency_ms, pl->lat_ev[0], pl->lat_ev[1]), "elapsed");
    if (lat_stats) {
      const auto us = [](clk::time_point a, clk::time_point b) {
        return std::chrono::duration<double, std::micro>(b - a).count();
      };
      float head = 0.0f, body = 0.0f, tail = 0.0f;
      cudaEventElapsedTime(&head, pl->lat_ev[0], g->ev[0]);
      cudaEventElapsedTime(&body, g->ev[0], g->ev[5]);
      cudaEventElapsedTime(&tail, g->ev[5], pl->lat_ev[1]);
      std::fprintf(stderr,
                   "[lat] frame %u: %.1f us | host enqueue %.1f, wait %.1f, timing %.1f, unpack %.1f, out %.1f, "
                   "end event %.1f | gpu head %.1f, body %.1f, tail %.1f\n",
                   pl->frame, 1e3 * pl->last_latency_ms, us(h0, h1), us(h1, h2), us(h2, h2b), us(h2b, h2c),
                   us(h2c, h3), us(h3, clk::now()),
                   1e3 * head, 1e3 * body, 1e3 * tail);
    }
    ++pl->frame;
  });
}

int vp_pipeline_frame(vp_pipeline* pl, const float* xyz, uint64_t n, const double R[9],
                      const double t[3], vp_polygons_t** out, vp_frame_timing* timing) {
  return pipeline_frame_impl(pl, xyz, n, R, t, false, out, timing);
}

int vp_pipeline_frame_device(vp_pipeline* pl, const float* xyz_dev, uint64_t n, const double R[9],
                             const double t[3], vp_polygons_t** out, vp_frame_timing* timing) {
  return pipeline_frame_impl(pl, xyz_dev, n, R, t, true, out, timing);
}

int vp_pipeline_run_frames(vp_pipeline* pl, size_t n_frames, const float* const* xyz, const uint64_t* n,
                           const double* rotations, const double* translations, int device_ptrs,
                           vp_polygons_t** out, const vp_run_outputs* extra) {
  if (out) *out = nullptr;
  if (extra && extra->per_frame)
    for (size_t k = 0; k < n_frames; ++k) extra->per_frame[k] = nullptr;
  if (extra && extra->traces)
    for (size_t k = 0; k < n_frames; ++k) {
      extra->traces[k] = nullptr;
      if (extra->trace_lens) extra->trace_lens[k] = 0;
    }
  std::vector<std::vector<uint8_t>> traces;
  const int rc = guard([&] {
    HostPolys hp;
    RunOutputs ro;
    ro.last = &hp;
    if (extra) {
      ro.timings = extra->timings;
      ro.per_frame = extra->per_frame;
      if (extra->traces) ro.traces = &traces;
    }
    pipeline_run(pl, n_frames, xyz, n, rotations, translations, device_ptrs != 0, ro);
    if (extra && extra->traces)
      for (size_t k = 0; k < traces.size(); ++k) {
        extra->traces[k] = static_cast<uint8_t*>(std::malloc(traces[k].size()));
        if (!extra->traces[k]) fail(VP_ENOMEM, "host allocation");
        std::memcpy(extra->traces[k], traces[k].data(), traces[k].size());
        if (extra->trace_lens) extra->trace_lens[k] = traces[k].size();
      }
    if (out) *out = make_polygons_out(hp);
  });
  if (rc != VP_OK && extra) {  // nothing half-returned on failure
    if (extra->per_frame)
      for (size_t k = 0; k < n_frames; ++k) {
        vp_polygons_free(extra->per_frame[k]);
        extra->per_frame[k] = nullptr;
      }
    if (extra->traces)
      for (size_t k = 0; k < n_frames; ++k) {
        std::free(extra->traces[k]);
        extra->traces[k] = nullptr;
      }
  }
  return rc;
}

int vp_pipeline_run(vp_pipeline* pl, size_t n_frames, const float* const* xyz, const uint64_t* n,
                    const double* rotations, const double* translations, int device_ptrs,
                    vp_polygons_t** out, vp_frame_timing* timings) {
  if (out) *out = nullptr;
  return guard([&] {
    HostPolys hp;
    RunOutputs ro;
    ro.timings = timings;
    ro.last = &hp;
    pipeline_run(pl, n_frames, xyz, n, rotations, translations, device_ptrs != 0, ro);
    if (out) *out = make_polygons_out(hp);
  });
}

}  // extern "C"

struct vp_heightmap {
  vp_grid* g = nullptr;  // stream, counters, frame params, segmentation context
  HmDesc m{};
  uint32_t ncells = 0;
  uint32_t* visit = nullptr;
  uint8_t* flags = nullptr;
  uint32_t* pos = nullptr;
  uint32_t* dn = nullptr;  // [0] ncells, [1] frontier size, [2] next frontier size
  uint32_t nv = 0;         // cells visited by the last segment (region members)
  ~vp_heightmap() {
    if (g && g->stream) cudaStreamSynchronize(g->stream);
    void* ptrs[] = {m.h, m.valid, m.win, m.parent, m.root, m.claim, m.visited, m.spos, visit, flags, pos, dn};
    for (void* q : ptrs)
      if (q) cudaFree(q);
    delete g;
  }
};

extern "C" {

int vp_heightmap_create(double res, const int32_t ext[2], const double center[2], int device, vp_heightmap** out) {
  *out = nullptr;
  return guard([&] {
    if (!(res > 0.0) || ext[0] <= 0 || ext[1] <= 0)  // heightmap.cpp:11-12
      fail(VP_EINVAL, "HeightMap: resolution and extents must be positive");
    const uint64_t nc = static_cast<uint64_t>(ext[0]) * ext[1];
    if (4 * nc >= (1ull << 31)) fail(VP_EINVAL, "HeightMap: too many cells");
    auto* h = new vp_heightmap();
    struct Del {
      vp_heightmap*& h;
      ~Del() { delete h; }
    } del{h};
    h->g = new vp_grid();
    const int32_t ge[3] = {1, 1, 32};
    const double gc[3] = {0.0, 0.0, 0.0};
    h->g->init(res, ge, gc, device);
    h->ncells = static_cast<uint32_t>(nc);
    HmDesc& m = h->m;
    m.ex = ext[0];
    m.ey = ext[1];
    m.res = res;
    m.ox = center[0] - static_cast<double>(ext[0]) * (0.5 * res);  // heightmap.cpp:13
    m.oy = center[1] - static_cast<double>(ext[1]) * (0.5 * res);
    m.h = dalloc<double>(nc);
    m.valid = dalloc<uint8_t>(nc);
    m.win = dalloc<uint32_t>(nc);
    m.parent = dalloc<int32_t>(nc);
    m.root = dalloc<int32_t>(nc);
    m.claim = dalloc<uint32_t>(nc);
    m.visited = dalloc<uint8_t>(nc);
    m.spos = dalloc<uint32_t>(nc);
    h->visit = dalloc<uint32_t>(nc);
    h->flags = dalloc<uint8_t>(4 * nc);
    h->pos = dalloc<uint32_t>(4 * nc);
    h->dn = dalloc<uint32_t>(4);
    cudaStream_t st = h->g->stream;
    ck(cudaMemsetAsync(m.h, 0, nc * 8, st), "memset");
    ck(cudaMemsetAsync(m.valid, 0, nc, st), "memset");
    ck(cudaMemsetAsync(m.win, 0, nc * 4, st), "memset");
    const uint32_t d0[4] = {h->ncells, 0, 0, 0};
    ck(cudaMemcpyAsync(h->dn, d0, 16, cudaMemcpyHostToDevice, st), "dn");
    // scan scratch for 4 x cells flags
    const uint32_t cap = static_cast<uint32_t>(4 * nc);
    h->g->seg.ensure(std::max(h->g->seg.b.Vcap, cap), std::max(h->g->seg.b.Scap, h->ncells),
                     std::max(h->g->seg.b.Icap, h->ncells), 100, h->g->gd.nwords);
    ck(cudaStreamSynchronize(st), "sync");
    *out = h;
    h = nullptr;
  });
}

void vp_heightmap_destroy(vp_heightmap* hm) { delete hm; }

int vp_hm_integrate(vp_heightmap* hm, const float* xyz, uint64_t n, const double R[9], const double t[3]) {
  return guard([&] {
    if (!is_valid_rotation(R)) fail(VP_EINVAL, "hm_integrate: pose rotation is not orthonormal");  // :27-28
    vp_grid* g = hm->g;
    if (n == 0) return;
    stage_points(g, xyz, n, false);
    g->set_pose(R, t);
    g->upload_params();
    LAUNCH(k_hm_win, grid_for(n), kThreads, 0, g->stream, hm->m, g->d_fp);
    LAUNCH(k_hm_write, grid_for(n), kThreads, 0, g->stream, hm->m, g->d_fp);
    ck(cudaStreamSynchronize(g->stream), "sync");
  });
}

int vp_hm_cells(vp_heightmap* hm, double* heights, uint8_t* valid) {
  return guard([&] {
    cudaStream_t st = hm->g->stream;
    ck(cudaMemcpyAsync(heights, hm->m.h, 8ull * hm->ncells, cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaMemcpyAsync(valid, hm->m.valid, hm->ncells, cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaStreamSynchronize(st), "sync");
  });
}

int vp_hm_regions(vp_heightmap* hm, uint32_t* visit, int32_t* root, uint64_t* nv) {
  return guard([&] {
    *nv = hm->nv;
    ck(cudaMemcpyAsync(visit, hm->visit, 4ull * hm->nv, cudaMemcpyDeviceToHost, hm->g->stream), "d2h");
    ck(cudaMemcpyAsync(root, hm->m.root, 4ull * hm->ncells, cudaMemcpyDeviceToHost, hm->g->stream), "d2h");
    ck(cudaStreamSynchronize(hm->g->stream), "sync");
  });
}

int vp_hm_segment(vp_heightmap* hm, const vp_pipeline_params* p, vp_polygons_t** out) {
  if (out) *out = nullptr;
  return guard([&] {
    vp_grid* g = hm->g;
    cudaStream_t st = g->stream;
    const double dth = p->seg.distance_th;
    const uint32_t nc = hm->ncells;
    g->reset_frame_counters();
    // regions = components; roots (component-minimum flat) are the BFS seeds
    LAUNCH(k_hm_ccl_init, grid_for(nc), kThreads, 0, st, hm->m);
    LAUNCH(k_hm_ccl_union, grid_for(nc), kThreads, 0, st, hm->m, dth);
    LAUNCH(k_hm_seed_flags, grid_for(nc), kThreads, 0, st, hm->m, hm->flags);
    g->launch_flag_scan(hm->flags, hm->dn, nc, hm->pos, hm->dn + 1);
    LAUNCH(k_hm_seed_emit, grid_for(nc), kThreads, 0, st, hm->m, hm->flags, hm->pos, hm->visit);
    // level-synchronous BFS in the reference's FIFO order, all levels in one block
    LAUNCH(k_hm_bfs, 1, 1024, 0, st, hm->m, hm->visit, hm->dn, dth);
    uint32_t nv = 0;
    ck(cudaMemcpyAsync(&nv, hm->dn + 2, 4, cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaStreamSynchronize(st), "sync");
    hm->nv = nv;
    // regions >= min_cluster_size, members in BFS order, then the voxel path's fitting
    g->seg.ensure(g->seg.b.Vcap, std::max(g->seg.b.Scap, nv), std::max(g->seg.b.Icap, nv),
                  std::max(p->ransac.iterations, 1), g->gd.nwords);
    g->seg.ensure_dirs(16, st);
    for (int tries = 0;; ++tries) {
      g->reset_frame_counters();
      set_counter_u32(g, offsetof(Counters, S), nv);
      const SegDev sd = make_segdev(p->seg, hm->m.res);
      const RansacDev rd = make_ransacdev(p->ransac);
      if (nv) {
        LAUNCH(k_hm_zero_cnt, grid_for(nv), kThreads, 0, st, nv, g->seg.b);
        LAUNCH(k_hm_members, grid_for(nv), kThreads, 0, st, hm->m, hm->visit, nv, g->seg.b);
      }
      g->launch_clusters(sd);
      LAUNCH(k_hm_klabel, 8, 256, 0, st, g->ctr, g->seg.b, hm->visit);
      g->launch_ransac(rd);
      g->launch_refine(p->ransac.up, p->refine, p->refine_exact);
      g->launch_polygon(16, p->min_polygon_area);
      g->read_counters();
      if (tries > 4 || !g->grow_if_overflow(p->ransac.iterations)) break;
    }
    if (g->h_ctr->overflow) fail(VP_ENOMEM, "hm_segment: capacity overflow");
    if (out) {
      HostPolys hp;
      g->download_polygons(hp, false);
      *out = make_polygons_out(hp);
    }
  });
}

int vp_pipeline_replay(vp_pipeline* pl, const vp_stream* st, uint64_t first, uint64_t count,
                       vp_polygons_t** out, vp_frame_timing* timings) {
  if (out) *out = nullptr;
  return guard([&] {
    if (first > st->n.size() || count > st->n.size() - first) fail(VP_EINVAL, "replay: frame range out of stream");
    std::vector<const float*> xyz(count);
    std::vector<uint64_t> n(count);
    std::vector<double> R(9 * count), t(3 * count);
    for (uint64_t k = 0; k < count; ++k) {
      const uint64_t i = first + k;
      xyz[k] = reinterpret_cast<const float*>(st->buf + st->off[i]);
      n[k] = st->n[i];
      const double* q = st->pose.data() + 12 * i;
      for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) R[9 * k + 3 * r + c] = q[4 * r + c];
        t[3 * k + r] = q[4 * r + 3];
      }
    }
    // pinned host frames: the H2D copies inside run_frames are asynchronous
    HostPolys hp;
    RunOutputs ro;
    ro.timings = timings;
    ro.last = &hp;
    pipeline_run(pl, count, xyz.data(), n.data(), R.data(), t.data(), false, ro);
    if (out) *out = make_polygons_out(hp);
  });
}

int vp_pipeline_frame_trace(vp_pipeline* pl, const float* xyz, uint64_t n, const double R[9],
                            const double t[3], uint8_t** buf, uint64_t* len) {
  *buf = nullptr;
  *len = 0;
  return guard([&] {
    vp_shift_stats ss;
    const bool rec = pipeline_enqueue(pl, xyz, n, R, t, false, &ss);
    vp_grid* g = pl->grid;
    wait_frame(g);
    if (g->h_ctr->overflow) rerun_segment_until_fits(g, pl->p);
    HostPolys hp;
    if (g->h_ctr->occupied) g->download_polygons(hp, false);
    const std::vector<uint8_t> tr = build_trace(g, *g->h_ctr, pl->frame++, rec, ss.shift, g->origin, hp);
    *buf = static_cast<uint8_t*>(std::malloc(tr.size()));
    if (!*buf) fail(VP_ENOMEM, "host allocation");
    std::memcpy(*buf, tr.data(), tr.size());
    *len = tr.size();
  });
}

}  // extern "C"

namespace {
std::vector<uint8_t> build_trace(vp_grid* g, const Counters& c, uint32_t frame, bool rec, const int32_t* shift,
                                 const double* origin, const HostPolys& hp) {
  TraceW w;
  w.raw("VPTR", 4);
  w.put<uint32_t>(VP_TRACE_VERSION);
  w.put<uint32_t>(frame);
  w.put<uint64_t>(c.cleared);
  w.put<uint64_t>(c.freed);
  w.put<uint64_t>(c.touched);
  w.put<uint64_t>(c.discarded);
  w.put<uint8_t>(rec ? 1 : 0);
  w.raw(shift, 12);
  w.put<uint64_t>(c.dropped);
  w.raw(origin, 24);
  w.put<uint64_t>(c.occupied);
  if (c.occupied == 0) {
    for (int k = 0; k < 7; ++k) w.put<uint64_t>(0);
  } else {
    const uint32_t V = c.V, S = c.S, K = std::min<uint32_t>(c.K, g->seg.b.Kcap), F = c.nfits;
    auto flat = d2h(g->seg.b.occ_list, V, g->stream);
    auto mean = d2h(g->seg.b.own_mean, 3ull * V, g->stream);
    auto cnt = d2h(g->seg.b.own_count, V, g->stream);
    auto st = d2h(g->seg.b.own_status, V, g->stream);
    auto nrm = d2h(g->seg.b.est_normal, 3ull * V, g->stream);
    auto nc = d2h(g->seg.b.est_ncount, V, g->stream);
    auto va = d2h(g->seg.b.est_valid, V, g->stream);
    auto sidx = d2h(g->seg.b.st_idx, 3ull * S, g->stream);
    auto smean = d2h(g->seg.b.st_mean, 3ull * S, g->stream);
    auto snrm = d2h(g->seg.b.st_normal, 3ull * S, g->stream);
    auto lab = d2h(g->seg.b.label, S, g->stream);
    auto kl = d2h(g->seg.b.klabel, K, g->stream);
    auto ks = d2h(g->seg.b.ksize, K, g->stream);
    auto fm = d2h(g->seg.b.fit_model, 4ull * F, g->stream);
    auto meta = d2h(g->seg.b.fit_meta, 2ull * F, g->stream);
    auto io = d2h(g->seg.b.ioff, F + 1ull, g->stream);
    auto rm = d2h(g->seg.b.ref_model, 4ull * F, g->stream);
    ck(cudaStreamSynchronize(g->stream), "sync");
    auto in = d2h(g->seg.b.inl, 3ull * io[F], g->stream);
    ck(cudaStreamSynchronize(g->stream), "sync");
    w.put<uint64_t>(V);
    for (uint32_t v = 0; v < V; ++v) {
      const uint32_t f = flat[v];
      w.put<int32_t>(static_cast<int32_t>(f / g->ext[2] / g->ext[1]));
      w.put<int32_t>(static_cast<int32_t>((f / g->ext[2]) % g->ext[1]));
      w.put<int32_t>(static_cast<int32_t>(f % g->ext[2]));
    }
    w.raw(mean.data(), 24ull * V);
    w.raw(cnt.data(), 4ull * V);
    w.raw(st.data(), V);
    w.raw(nrm.data(), 24ull * V);
    w.raw(nc.data(), 4ull * V);
    w.raw(va.data(), V);
    w.put<uint64_t>(S);
    w.raw(sidx.data(), 12ull * S);
    w.raw(smean.data(), 24ull * S);
    w.raw(snrm.data(), 24ull * S);
    w.raw(lab.data(), 4ull * S);
    w.put<uint64_t>(K);
    for (uint32_t k = 0; k < K; ++k) {
      w.put<int32_t>(kl[k]);
      w.put<uint64_t>(ks[k]);
    }
    w.put<uint64_t>(c.skipped);
    w.put<uint64_t>(c.unfit);
    w.put<uint64_t>(F);
    for (uint32_t f = 0; f < F; ++f) {
      w.raw(&fm[4 * f], 32);
      w.put<int32_t>(meta[2 * f]);
      w.put<int32_t>(meta[2 * f + 1]);
      const uint64_t m = io[f + 1] - io[f];
      w.put<uint64_t>(m);
      w.raw(in.data() + 3ull * io[f], 24 * m);
    }
    for (uint32_t f = 0; f < F; ++f) w.raw(&rm[4 * f], 32);
    w.put<uint64_t>(hp.polys.size());
    for (const auto& q : hp.polys) {
      w.raw(q.plane.normal, 24);
      w.put<double>(q.plane.offset);
      w.put<int32_t>(q.plane.inlier_count);
      w.put<int32_t>(q.plane.cluster_label);
      w.put<uint64_t>(q.nverts);
      const size_t voff = static_cast<size_t>(reinterpret_cast<uintptr_t>(q.v2d));
      for (uint32_t k = 0; k < q.nverts; ++k) w.raw(&hp.verts[5 * (voff + k)], 16);
      for (uint32_t k = 0; k < q.nverts; ++k) w.raw(&hp.verts[5 * (voff + k) + 2], 24);
      w.put<double>(q.area);
    }
  }
  return std::move(w.b);
}
}  // namespace

// ===========================================================================
// Reference-named utilities of the C ABI (jacobi.hpp, polygonize.hpp,
// segmentation.hpp overloads): the same device code the fused path runs.
namespace {

// Device buffer released on scope exit (stateless entry points).
template <typename T>
struct DBuf {
  T* p = nullptr;
  explicit DBuf(size_t n) : p(dalloc<T>(n)) {}
  ~DBuf() {
    if (p) cudaFree(p);
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};

// One 2-D point set as fit 0 of the scratch grid: the points (x, y, 0) on the
// plane z = 0, whose plane_basis (polygonize.cpp:21-34) is u = e_x, v = e_y,
// origin 0, so project_to_plane and lift_from_plane return (x, y) exactly.
void stage_points2d(vp_grid* g, const double* pts, uint64_t n) {
  if (n >= (1ull << 31)) fail(VP_EINVAL, "hull: too many points");
  std::vector<double> p3(3 * n);
  for (uint64_t i = 0; i < n; ++i) {
    p3[3 * i] = pts[2 * i];
    p3[3 * i + 1] = pts[2 * i + 1];
    p3[3 * i + 2] = 0.0;
  }
  vp_plane pl{};
  pl.normal[2] = 1.0;
  pl.inlier_count = static_cast<int32_t>(n);
  const uint64_t offs[2] = {0, n};
  upload_fit_batch(g, 0, 1, &pl, offs, p3.data(), true);
}

double* copy_out2(const double* src, uint64_t m) {
  auto* out = static_cast<double*>(std::malloc(std::max<uint64_t>(1, 2 * m) * sizeof(double)));
  if (!out) fail(VP_ENOMEM, "host allocation");
  if (m) std::memcpy(out, src, 2 * m * sizeof(double));
  return out;
}

}  // namespace

extern "C" {

int vp_jacobi_eigen_sym3(size_t n, const double* a, double* eigenvalues, double* eigenvectors, int device) {
  return guard([&] {
    if (n == 0) return;
    vp_grid* g = scratch_grid(device);
    DBuf<double> d(21 * n);
    h2d(d.p, a, 9 * n, g->stream);
    LAUNCH(k_jacobi_batch, grid_for(n), kThreads, 0, g->stream, static_cast<uint64_t>(n), d.p, d.p + 9 * n,
           d.p + 12 * n);
    ck(cudaMemcpyAsync(eigenvalues, d.p + 9 * n, 24 * n, cudaMemcpyDeviceToHost, g->stream), "d2h");
    ck(cudaMemcpyAsync(eigenvectors, d.p + 12 * n, 72 * n, cudaMemcpyDeviceToHost, g->stream), "d2h");
    ck(cudaStreamSynchronize(g->stream), "sync");
  });
}

int vp_convex_hull(const double* pts, uint64_t n, int directions, int device, double** out, uint64_t* m) {
  *out = nullptr;
  *m = 0;
  return guard([&] {
    if (n < 3) {  // monotone_chain: fewer than three points -> empty
      *out = copy_out2(pts, 0);
      return;
    }
    vp_grid* g = scratch_grid(device);
    stage_points2d(g, pts, n);
    g->launch_polygon(directions, -std::numeric_limits<double>::infinity(), 1);
    g->read_counters();
    if (g->h_ctr->overflow & kOverflowPool) fail(VP_ENOMEM, "polygon vertex pool overflow");
    HostPolys hp;
    g->download_polygons(hp, true);
    std::vector<double> ring;
    if (!hp.polys.empty()) {
      const vp_polygon& q = hp.polys[0];
      const size_t voff = static_cast<size_t>(reinterpret_cast<uintptr_t>(q.v2d));
      for (uint32_t k = 0; k < q.nverts; ++k) {
        ring.push_back(hp.verts[5 * (voff + k)]);
        ring.push_back(hp.verts[5 * (voff + k) + 1]);
      }
    }
    *m = ring.size() / 2;
    *out = copy_out2(ring.data(), *m);
  });
}

int vp_monotone_chain(const double* pts, uint64_t n, int device, double** out, uint64_t* m) {
  return vp_convex_hull(pts, n, 0, device, out, m);
}

int vp_hull_filter(const double* pts, uint64_t n, int directions, int device, double** out, uint64_t* m) {
  *out = nullptr;
  *m = 0;
  return guard([&] {
    if (n <= 3 || directions < 3) {  // polygonize.cpp:51: nothing to filter
      *m = n;
      *out = copy_out2(pts, n);
      return;
    }
    vp_grid* g = scratch_grid(device);
    const uint32_t n32 = static_cast<uint32_t>(n);
    g->seg.ensure(std::max(g->seg.b.Vcap, n32), g->seg.b.Scap, std::max(g->seg.b.Icap, n32), 100,
                  g->gd.nwords);  // flag-scan block sums for n points
    stage_points2d(g, pts, n);
    g->seg.ensure_dirs(directions, g->stream);
    cudaStream_t st = g->stream;
    LAUNCH(k_poly_setup, 1, 1024, 0, st, g->ctr, g->seg.b);
    LAUNCH(k_poly_extremes, g->chain_wide, 256, 0, st, g->ctr, g->seg.b, g->seg.dirtab, directions, 1);
    LAUNCH(k_poly_inner, 1, 64, 0, st, g->ctr, g->seg.b, directions);
    DBuf<uint8_t> flags(n);
    DBuf<uint32_t> pos(n + 2);
    DBuf<double> outd(2 * n);
    const uint32_t nn[2] = {static_cast<uint32_t>(n), 0u};
    h2d(pos.p + n, nn, 2, st);
    LAUNCH(k_poly_keep_flags, grid_for(n), kThreads, 0, st, g->ctr, g->seg.b, flags.p);
    g->launch_flag_scan(flags.p, pos.p + n, static_cast<uint32_t>(n), pos.p, pos.p + n + 1);
    LAUNCH(k_gather_p2, grid_for(n), kThreads, 0, st, pos.p + n, flags.p, pos.p, g->seg.b.proj, outd.p);
    uint32_t kept = 0;
    ck(cudaMemcpyAsync(&kept, pos.p + n + 1, 4, cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaStreamSynchronize(st), "sync");
    std::vector<double> h(2ull * kept);
    if (kept) ck(cudaMemcpy(h.data(), outd.p, 16ull * kept, cudaMemcpyDeviceToHost), "d2h");
    *m = kept;
    *out = copy_out2(h.data(), kept);
  });
}

int vp_label_components_adjacency(uint64_t n, const uint64_t* row_offsets, const int32_t* cols, int device,
                                  int32_t* labels) {
  return guard([&] {
    if (n == 0) return;
    if (n >= (1ull << 31)) fail(VP_EINVAL, "label_components: too many voxels");
    vp_grid* g = scratch_grid(device);
    cudaStream_t st = g->stream;
    const uint64_t ne = row_offsets[n];
    DBuf<uint64_t> rows(n + 1);
    DBuf<int32_t> c(std::max<uint64_t>(ne, 1)), parent(n), lab(n);
    h2d(rows.p, row_offsets, n + 1, st);
    h2d(c.p, cols, ne, st);
    LAUNCH(k_iota, grid_for(n), kThreads, 0, st, parent.p, n);
    LAUNCH(k_label_edges, grid_for(32 * n, 148 * 32), kThreads, 0, st, n, rows.p, c.p, parent.p);
    LAUNCH(k_label_flatten, grid_for(n), kThreads, 0, st, n, parent.p, lab.p);
    ck(cudaMemcpyAsync(labels, lab.p, 4 * n, cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaStreamSynchronize(st), "sync");
  });
}

int vp_classify_estimates(vp_grid* g, const vp_seg_params* p, size_t n, const int32_t* idx,
                          const int32_t* neighbor_count, const double* angle_to_up_deg, const uint8_t* valid,
                          uint8_t* status) {
  return guard([&] {
    if (n == 0) return;
    cudaStream_t st = g->stream;
    DBuf<int32_t> di(3 * n), dn(n);
    DBuf<double> da(n);
    DBuf<uint8_t> dv(n), ds(n);
    h2d(di.p, idx, 3 * n, st);
    h2d(dn.p, neighbor_count, n, st);
    h2d(da.p, angle_to_up_deg, n, st);
    h2d(dv.p, valid, n, st);
    LAUNCH(k_classify_estimates, grid_for(n), kThreads, 0, st, static_cast<uint64_t>(n), dn.p, da.p, dv.p,
           p->min_neighbors, p->max_angle_deg, ds.p);
    g->fill_static_params();
    g->h_fp->n = 0;
    g->upload_params();
    LAUNCH(k_set_statuses, grid_for(n), kThreads, 0, st, g->gd, g->d_fp, di.p, ds.p, static_cast<uint64_t>(n));
    ck(cudaMemcpyAsync(status, ds.p, n, cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaStreamSynchronize(st), "sync");
  });
}

}  // extern "C"
