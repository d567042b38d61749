// One frame of the spatial-slab decomposition, orchestrated in
// the library: every exchange of the per-frame sequence (frame broadcast,
// halo planes, per-plane steppable counts, halo steppable lists, boundary
// triples, cluster members, polygon gather) is a stream-ordered collective of
// a vp_comm_ops table on device buffers, between the library's slab phases
// (vp_update_frame, vp_slab_steppable .. vp_slab_segment_owned in runtime.cu).
// Communicators: NCCL (loaded at run time; NVLink / NVSwitch between the GPUs
// of a node), an in-process hub for N virtual slabs (one host thread per
// slab, device-to-device copies), or a caller's table (torch.distributed).
//
// Host round trips per frame (besides the phases' own counter reads): the
// all-gathered plane counts (the layout of the extended lists and of the
// boundary zone is host arithmetic, mirroring vp_slab_extend), the
// all-gathered member counts, and the polygon blob sizes.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "voxplane_b200.h"

namespace vp {
cudaStream_t slab_stream(vp_grid* g);
void slab_geometry(vp_grid* g, int32_t* xb, int32_t* xe, int32_t* gex, int* device, double* res);
void set_last_error(const char* msg);
void slab_frame_release(vp_grid* g);
}  // namespace vp

namespace {

struct Fail {
  int code;
  std::string msg;
};
[[noreturn]] void fail(int code, const std::string& m) { throw Fail{code, m}; }
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(VP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void vck(int rc, const char* what) {
  if (rc != VP_OK) fail(rc, std::string(what) + ": " + vp_last_error());
}

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    bytes = std::max<size_t>(bytes, 16);
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      const size_t c = std::max(bytes, 2 * cap);
      ck(cudaMalloc(&p, c), "slab frame buffer");
      cap = c;
    }
    return p;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

// Per-slab buffers kept across frames.
struct FrameState {
  DevBuf pts, ranges_s, ranges_r, pc_s, pc_r, tr_s, tr_r, dc_s, dc_r, rec_r, sz_s, sz_r, poly_s, poly_r;
  std::vector<int32_t> ranges;  // 2 per rank, cached after the first frame
};
std::mutex g_state_mu;
std::map<vp_grid*, std::unique_ptr<FrameState>> g_state;

FrameState& state_of(vp_grid* g) {
  std::lock_guard<std::mutex> lk(g_state_mu);
  auto& s = g_state[g];
  if (!s) s = std::make_unique<FrameState>();
  return *s;
}

// polygons <-> a flat blob of doubles: [count; per polygon: normal(3),
// offset, inlier_count, label, nverts, area, then v2d (2 nv), v3d (3 nv)]
void serialize(const vp_polygons_t* p, std::vector<double>& out) {
  out.clear();
  out.push_back(p ? static_cast<double>(p->count) : 0.0);
  if (!p) return;
  for (size_t i = 0; i < p->count; ++i) {
    const vp_polygon& q = p->polys[i];
    for (int k = 0; k < 3; ++k) out.push_back(q.plane.normal[k]);
    out.push_back(q.plane.offset);
    out.push_back(static_cast<double>(q.plane.inlier_count));
    out.push_back(static_cast<double>(q.plane.cluster_label));
    out.push_back(static_cast<double>(q.nverts));
    out.push_back(q.area);
    for (uint32_t k = 0; k < 2 * q.nverts; ++k) out.push_back(q.v2d[k]);
    for (uint32_t k = 0; k < 3 * q.nverts; ++k) out.push_back(q.v3d[k]);
  }
}

// blobs in rank order -> one vp_polygons_t (one allocation, vp_polygons_free)
vp_polygons_t* deserialize(const std::vector<std::vector<double>>& blobs) {
  size_t np = 0, nv = 0;
  for (const auto& b : blobs) {
    size_t o = 1;
    const size_t c = b.empty() ? 0 : static_cast<size_t>(b[0]);
    for (size_t i = 0; i < c; ++i) {
      const size_t v = static_cast<size_t>(b[o + 6]);
      o += 8 + 5 * v;
      nv += v;
    }
    np += c;
  }
  const size_t bytes = sizeof(vp_polygons_t) + np * sizeof(vp_polygon) + nv * 5 * sizeof(double);
  char* mem = static_cast<char*>(std::malloc(bytes));
  if (!mem) fail(VP_ENOMEM, "host allocation");
  auto* out = reinterpret_cast<vp_polygons_t*>(mem);
  out->count = np;
  out->polys = reinterpret_cast<vp_polygon*>(mem + sizeof(vp_polygons_t));
  double* vb = reinterpret_cast<double*>(mem + sizeof(vp_polygons_t) + np * sizeof(vp_polygon));
  size_t pi = 0;
  for (const auto& b : blobs) {
    size_t o = 1;
    const size_t c = b.empty() ? 0 : static_cast<size_t>(b[0]);
    for (size_t i = 0; i < c; ++i, ++pi) {
      vp_polygon q{};
      for (int k = 0; k < 3; ++k) q.plane.normal[k] = b[o + k];
      q.plane.offset = b[o + 3];
      q.plane.inlier_count = static_cast<int32_t>(b[o + 4]);
      q.plane.cluster_label = static_cast<int32_t>(b[o + 5]);
      q.nverts = static_cast<uint32_t>(b[o + 6]);
      q.area = b[o + 7];
      o += 8;
      std::memcpy(vb, b.data() + o, 5 * q.nverts * sizeof(double));
      q.v2d = q.nverts ? vb : nullptr;
      q.v3d = q.nverts ? vb + 2 * q.nverts : nullptr;
      vb += 5 * q.nverts;
      o += 5 * q.nverts;
      out->polys[pi] = q;
    }
  }
  return out;
}

// Host arithmetic of vp_slab_extend / vp_slab_label for every slab: the number
// of boundary-zone entries inside slab k's extended planes (= its triples).
uint64_t zone_entries(const std::vector<uint64_t>& P, const std::vector<int32_t>& xb, int32_t gex, int w, int k) {
  const int n = static_cast<int>(xb.size()) - 1;
  std::vector<std::pair<int32_t, int32_t>> zone;
  for (int b = 1; b < n; ++b) {
    const int32_t lo = std::max(0, xb[b] - w), hi = std::min(gex, xb[b] + w);
    if (!zone.empty() && lo <= zone.back().second) zone.back().second = std::max(zone.back().second, hi);
    else zone.emplace_back(lo, hi);
  }
  const int32_t x_lo = std::max(0, xb[k] - w), x_hi = std::min(gex, xb[k + 1] + w);
  uint64_t z = 0;
  for (const auto& iv : zone) {
    const int32_t a = std::max(iv.first, x_lo), b = std::min(iv.second, x_hi);
    if (a < b) z += P[b] - P[a];
  }
  return z;
}

void slab_frame_impl(vp_grid* g, const vp_comm_ops* c, const float* xyz, uint64_t n, const double* R,
                     const double* t, const vp_pipeline_params* p, vp_polygons_t** out) {
  if (out) *out = nullptr;
  FrameState& S = state_of(g);
  int32_t xb, xe, gex;
  int dev;
  double res;
  vp::slab_geometry(g, &xb, &xe, &gex, &dev, &res);
  ck(cudaSetDevice(dev), "set device");
  cudaStream_t st = vp::slab_stream(g);
  const int W = c->nranks, me = c->rank;
  if (W < 1 || me < 0 || me >= W) fail(VP_EINVAL, "slab frame: bad communicator rank / size");
  auto comm = [&](int rc, const char* what) {
    if (rc != 0) fail(VP_ECUDA, std::string("slab frame: communicator ") + what + " failed");
  };
  auto h2d = [&](void* d, const void* h, size_t bytes) {
    if (bytes) ck(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st), "h2d");
  };
  auto d2h = [&](void* h, const void* d, size_t bytes) {
    if (bytes) ck(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st), "d2h");
    ck(cudaStreamSynchronize(st), "sync");
  };

  // 0. the slabs' x ranges (once: slab windows are fixed)
  if (static_cast<int>(S.ranges.size()) != 2 * W) {
    S.ranges.assign(2 * W, 0);
    const int32_t mine[2] = {xb, xe};
    void* rs = S.ranges_s.get(8);
    void* rr = S.ranges_r.get(8ull * W);
    h2d(rs, mine, 8);
    if (W > 1) comm(c->allgather(c->ctx, rs, rr, 8, st), "allgather");
    else ck(cudaMemcpyAsync(rr, rs, 8, cudaMemcpyDeviceToDevice, st), "d2d");
    d2h(S.ranges.data(), rr, 8ull * W);
    for (int k = 0; k < W; ++k)
      if (S.ranges[2 * k] >= S.ranges[2 * k + 1] || (k ? S.ranges[2 * k] != S.ranges[2 * k - 1] : S.ranges[0] != 0)) {
        S.ranges.clear();
        fail(VP_EINVAL, "slab frame: the ranks' x ranges must tile the window in rank order");
      }
    if (S.ranges[2 * W - 1] != gex) {
      S.ranges.clear();
      fail(VP_EINVAL, "slab frame: the ranks' x ranges must cover the window");
    }
  }
  std::vector<int32_t> xbegin(W + 1);
  for (int k = 0; k < W; ++k) xbegin[k] = S.ranges[2 * k];
  xbegin[W] = gex;

  // 1. the frame (rank 0's points) to every slab; 2. clear_rays + integrate_frame
  float* dp = static_cast<float*>(S.pts.get(12 * std::max<uint64_t>(n, 1)));
  if (me == 0 && n) {
    if (!xyz) fail(VP_EINVAL, "slab frame: rank 0 needs the points");
    ck(cudaMemcpyAsync(dp, xyz, 12 * n, cudaMemcpyDefault, st), "points");
  }
  if (W > 1 && n) comm(c->broadcast(c->ctx, dp, 12 * n, 0, st), "broadcast");
  vck(vp_update_frame(g, dp, n, R, t, nullptr, nullptr), "update_frame");

  // 3. halo planes: first / last owned plane (cells + occupancy words) to the neighbours
  std::vector<vp_p2p_op> ops;
  auto plane = [&](int32_t x, void** cells, uint64_t* cb, void** bits, uint64_t* bb) {
    vck(vp_grid_plane(g, x, cells, cb, bits, bb), "grid_plane");
  };
  if (W > 1) {
    void *mc, *mb, *hc, *hb;
    uint64_t mcb, mbb, hcb, hbb;
    if (me > 0) {
      plane(xb, &mc, &mcb, &mb, &mbb);
      plane(xb - 1, &hc, &hcb, &hb, &hbb);
      ops.push_back({me - 1, 1, mc, mcb});
      ops.push_back({me - 1, 1, mb, mbb});
      ops.push_back({me - 1, 0, hc, hcb});
      ops.push_back({me - 1, 0, hb, hbb});
    }
    if (me + 1 < W) {
      plane(xe - 1, &mc, &mcb, &mb, &mbb);
      plane(xe, &hc, &hcb, &hb, &hbb);
      ops.push_back({me + 1, 1, mc, mcb});
      ops.push_back({me + 1, 1, mb, mbb});
      ops.push_back({me + 1, 0, hc, hcb});
      ops.push_back({me + 1, 0, hb, hbb});
    }
    comm(c->group(c->ctx, static_cast<int32_t>(ops.size()), ops.data(), st), "halo planes");
  }

  // 4. estimate_normals + classify_steppable on the owned voxels
  uint64_t S_own = 0;
  int32_t* sidx;
  double *smean, *snrm;
  vck(vp_slab_steppable(g, &p->seg, &S_own, &sidx, &smean, &snrm), "slab_steppable");

  // 5. steppable counts of every window plane (all-gather, padded to the widest slab)
  uint32_t* pc;
  int32_t np;
  vck(vp_slab_plane_counts(g, &pc, &np), "plane_counts");
  int32_t maxw = 0;
  for (int k = 0; k < W; ++k) maxw = std::max(maxw, S.ranges[2 * k + 1] - S.ranges[2 * k]);
  std::vector<uint32_t> allpc(static_cast<size_t>(maxw) * W);
  {
    void* ps = S.pc_s.get(4ull * maxw);
    void* pr = S.pc_r.get(4ull * maxw * W);
    ck(cudaMemsetAsync(ps, 0, 4ull * maxw, st), "memset");
    if (np) ck(cudaMemcpyAsync(ps, pc, 4ull * np, cudaMemcpyDeviceToDevice, st), "d2d");
    if (W > 1) comm(c->allgather(c->ctx, ps, pr, 4ull * maxw, st), "allgather");
    else ck(cudaMemcpyAsync(pr, ps, 4ull * maxw, cudaMemcpyDeviceToDevice, st), "d2d");
    d2h(allpc.data(), pr, 4ull * maxw * W);
  }
  std::vector<uint32_t> counts(gex);
  for (int k = 0; k < W; ++k)
    for (int32_t x = S.ranges[2 * k]; x < S.ranges[2 * k + 1]; ++x)
      counts[x] = allpc[static_cast<size_t>(k) * maxw + (x - S.ranges[2 * k])];
  std::vector<uint64_t> P(gex + 1, 0);
  for (int32_t x = 0; x < gex; ++x) P[x + 1] = P[x] + counts[x];

  // 6. extended lists: own list in place, halo entries from the owning slabs
  vp_slab_layout lay{W, xbegin.data(), counts.data()};
  int32_t* xidx;
  double *xmean, *xnrm;
  uint64_t n_ext;
  int32_t x_lo, x_hi;
  vck(vp_slab_extend(g, &p->seg, &lay, &xidx, &xmean, &xnrm, &n_ext, &x_lo, &x_hi), "slab_extend");
  int32_t w = 1;
  vck(vp_adjacency_window(&p->seg, res, &w), "adjacency_window");
  if (W > 1) {
    ops.clear();
    auto ext_of = [&](int k) {
      return std::make_pair(std::max(0, xbegin[k] - w), std::min(gex, xbegin[k + 1] + w));
    };
    const uint64_t my_left = P[xb] - P[ext_of(me).first];
    for (int d = 0; d < W; ++d) {
      const auto [lo, hi] = ext_of(d);
      for (int s = 0; s < W; ++s) {
        if (s == d || (s != me && d != me)) continue;
        const int32_t x0 = std::max(lo, xbegin[s]), x1 = std::min(hi, xbegin[s + 1]);
        if (x0 >= x1) continue;
        const uint64_t cnt = P[x1] - P[x0];
        if (!cnt) continue;
        if (s == me) {  // entries of my own list [P[x0] - P[xb], +cnt)
          const uint64_t s0 = my_left + (P[x0] - P[xb]);
          ops.push_back({d, 1, xidx + 3 * s0, 12 * cnt});
          ops.push_back({d, 1, xmean + 3 * s0, 24 * cnt});
          ops.push_back({d, 1, xnrm + 3 * s0, 24 * cnt});
        } else {  // into my extended list at P[x0] - P[x_lo]
          const uint64_t d0 = P[x0] - P[lo];
          ops.push_back({s, 0, xidx + 3 * d0, 12 * cnt});
          ops.push_back({s, 0, xmean + 3 * d0, 24 * cnt});
          ops.push_back({s, 0, xnrm + 3 * d0, 24 * cnt});
        }
      }
    }
    comm(c->group(c->ctx, static_cast<int32_t>(ops.size()), ops.data(), st), "halo lists");
  }

  // 7. local CCL; boundary triples of every slab (all-gather, padded with -1)
  int32_t* tr;
  uint64_t ntr, zsize;
  vck(vp_slab_label(g, &p->seg, &tr, &ntr, &zsize), "slab_label");
  uint64_t maxT = 0;
  for (int k = 0; k < W; ++k) maxT = std::max(maxT, zone_entries(P, xbegin, gex, w, k));
  if (ntr > maxT) fail(VP_ECUDA, "slab frame: triple count above the layout's zone entries");
  const int32_t* merged = tr;
  uint64_t nmerged = ntr;
  if (W > 1 && maxT) {
    void* ts = S.tr_s.get(12 * maxT);
    void* trr = S.tr_r.get(12 * maxT * W);
    ck(cudaMemsetAsync(ts, 0xff, 12 * maxT, st), "memset");
    if (ntr) ck(cudaMemcpyAsync(ts, tr, 12 * ntr, cudaMemcpyDeviceToDevice, st), "d2d");
    comm(c->allgather(c->ctx, ts, trr, 12 * maxT, st), "allgather");
    merged = static_cast<const int32_t*>(trr);
    nmerged = maxT * W;
  }
  int32_t* labels;
  vck(vp_slab_merge(g, merged, nmerged, &labels), "slab_merge");

  // 8. members of clusters owned by lower slabs to their owners
  std::vector<uint64_t> dc(W, 0);
  void* rec;
  vck(vp_slab_export(g, dc.data(), &rec), "slab_export");
  const void* recv = nullptr;
  uint64_t n_recv = 0;
  if (W > 1) {
    std::vector<uint64_t> M(static_cast<size_t>(W) * W);
    void* ds = S.dc_s.get(8ull * W);
    void* dr = S.dc_r.get(8ull * W * W);
    h2d(ds, dc.data(), 8ull * W);
    comm(c->allgather(c->ctx, ds, dr, 8ull * W, st), "allgather");
    d2h(M.data(), dr, 8ull * W * W);  // M[s * W + d]: records slab s sends to slab d
    ops.clear();
    uint64_t off = 0;
    for (int d = 0; d < W; ++d) {
      const uint64_t cnt = M[static_cast<size_t>(me) * W + d];
      if (d < me && cnt) ops.push_back({d, 1, static_cast<char*>(rec) + 32 * off, 32 * cnt});
      off += cnt;
    }
    for (int s = me + 1; s < W; ++s) n_recv += M[static_cast<size_t>(s) * W + me];
    char* rb = static_cast<char*>(S.rec_r.get(32 * std::max<uint64_t>(n_recv, 1)));
    uint64_t o = 0;
    for (int s = me + 1; s < W; ++s) {
      const uint64_t cnt = M[static_cast<size_t>(s) * W + me];
      if (cnt) ops.push_back({s, 0, rb + 32 * o, 32 * cnt});
      o += cnt;
    }
    comm(c->group(c->ctx, static_cast<int32_t>(ops.size()), ops.data(), st), "members");
    recv = rb;
  }

  // 9. filter_clusters .. make_polygon for the clusters this slab owns
  vp_polygons_t* mine = nullptr;
  vck(vp_slab_segment_owned(g, p, recv, n_recv, &mine), "slab_segment_owned");
  struct FreePolys {
    vp_polygons_t* q;
    ~FreePolys() {
      if (q) vp_polygons_free(q);
    }
  } free_mine{mine};

  // 10. polygons to rank 0 in slab order (= ascending label order)
  std::vector<double> blob;
  serialize(mine, blob);
  if (W == 1) {
    if (out) *out = deserialize({blob});
    return;
  }
  std::vector<uint64_t> sizes(W);
  {
    const uint64_t b = blob.size();
    void* ss = S.sz_s.get(8);
    void* sr = S.sz_r.get(8ull * W);
    h2d(ss, &b, 8);
    comm(c->allgather(c->ctx, ss, sr, 8, st), "allgather");
    d2h(sizes.data(), sr, 8ull * W);
  }
  ops.clear();
  char* pr = nullptr;
  if (me != 0) {
    void* ps = S.poly_s.get(8 * blob.size());
    h2d(ps, blob.data(), 8 * blob.size());
    ops.push_back({0, 1, ps, 8 * blob.size()});
  } else {
    uint64_t tot = 0;
    for (int k = 1; k < W; ++k) tot += sizes[k];
    pr = static_cast<char*>(S.poly_r.get(8 * std::max<uint64_t>(tot, 1)));
    uint64_t o = 0;
    for (int k = 1; k < W; ++k) {
      ops.push_back({k, 0, pr + 8 * o, 8 * sizes[k]});
      o += sizes[k];
    }
  }
  comm(c->group(c->ctx, static_cast<int32_t>(ops.size()), ops.data(), st), "polygon gather");
  if (me == 0) {
    std::vector<std::vector<double>> blobs(W);
    blobs[0] = blob;
    uint64_t o = 0;
    for (int k = 1; k < W; ++k) {
      blobs[k].resize(sizes[k]);
      d2h(blobs[k].data(), pr + 8 * o, 8 * sizes[k]);
      o += sizes[k];
    }
    if (out) *out = deserialize(blobs);
  } else {
    ck(cudaStreamSynchronize(st), "sync");
  }
}

template <typename F>
int guard(F&& f) {
  try {
    f();
    return VP_OK;
  } catch (const Fail& e) {
    vp::set_last_error(e.msg.c_str());
    return e.code;
  } catch (const std::bad_alloc&) {
    vp::set_last_error("host allocation failed");
    return VP_ENOMEM;
  } catch (const std::exception& e) {
    vp::set_last_error(e.what());
    return VP_ECUDA;
  }
}

// ------------------------------------------------------------------ NCCL
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!api.h) return;
#define VP_SYM(name) api.name = reinterpret_cast<decltype(api.name)>(dlsym(api.h, "nccl" #name))
    VP_SYM(GetUniqueId);
    VP_SYM(CommInitRank);
    VP_SYM(CommDestroy);
    VP_SYM(GroupStart);
    VP_SYM(GroupEnd);
    VP_SYM(Send);
    VP_SYM(Recv);
    VP_SYM(Broadcast);
    VP_SYM(AllGather);
#undef VP_SYM
  });
  if (!api.h || !api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv || !api.AllGather)
    fail(VP_ENODEV, "libnccl.so.2 not found (multi-GPU slabs need NCCL)");
  return api;
}

struct NcclCtx {
  ncclComm_t comm = nullptr;
  int device = 0;
};

int nccl_broadcast(void* ctx, void* buf, uint64_t bytes, int32_t root, void* stream) {
  auto* c = static_cast<NcclCtx*>(ctx);
  return nccl().Broadcast(buf, buf, bytes, ncclUint8, root, c->comm, static_cast<cudaStream_t>(stream)) == ncclSuccess
             ? 0
             : 1;
}
int nccl_allgather(void* ctx, const void* send, void* recv, uint64_t bytes, void* stream) {
  auto* c = static_cast<NcclCtx*>(ctx);
  return nccl().AllGather(send, recv, bytes, ncclUint8, c->comm, static_cast<cudaStream_t>(stream)) == ncclSuccess
             ? 0
             : 1;
}
int nccl_group(void* ctx, int32_t n, const vp_p2p_op* ops, void* stream) {
  auto* c = static_cast<NcclCtx*>(ctx);
  NcclApi& a = nccl();
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (a.GroupStart() != ncclSuccess) return 1;
  int bad = 0;
  for (int32_t i = 0; i < n; ++i) {
    const vp_p2p_op& o = ops[i];
    if (!o.bytes) continue;
    const ncclResult_t r = o.send ? a.Send(o.ptr, o.bytes, ncclUint8, o.peer, c->comm, st)
                                  : a.Recv(o.ptr, o.bytes, ncclUint8, o.peer, c->comm, st);
    bad |= r != ncclSuccess;
  }
  bad |= a.GroupEnd() != ncclSuccess;
  return bad;
}

// ----------------------------------------------------- in-process slabs
// One host thread per slab; every collective is a rendezvous: the producers'
// streams are drained, the buffers posted, the consumers copy device to
// device, drain, and meet again. A failing slab aborts the others.
struct Hub {
  explicit Hub(int n) : n(n), post(n, nullptr), ops(n) {}
  int n;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool failed = false;
  std::vector<const void*> post;
  std::vector<std::vector<vp_p2p_op>> ops;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (failed) fail(VP_ECUDA, "another slab failed");
    const uint64_t my = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != my || failed; });
    }
    if (failed) fail(VP_ECUDA, "another slab failed");
  }
  // true for the first slab to fail (its error is the one reported)
  bool abort() {
    std::lock_guard<std::mutex> lk(m);
    const bool first = !failed;
    failed = true;
    cv.notify_all();
    return first;
  }
};
struct HubCtx {
  Hub* hub;
  int rank;
};

int hub_call(std::function<void()> f) {
  try {
    f();
    return 0;
  } catch (...) {
    return 1;
  }
}
int hub_broadcast(void* ctx, void* buf, uint64_t bytes, int32_t root, void* stream) {
  auto* c = static_cast<HubCtx*>(ctx);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  return hub_call([&] {
    ck(cudaStreamSynchronize(st), "sync");
    c->hub->post[c->rank] = buf;
    c->hub->barrier();
    if (c->rank != root && bytes)
      ck(cudaMemcpyAsync(buf, c->hub->post[root], bytes, cudaMemcpyDeviceToDevice, st), "d2d");
    ck(cudaStreamSynchronize(st), "sync");
    c->hub->barrier();
  });
}
int hub_allgather(void* ctx, const void* send, void* recv, uint64_t bytes, void* stream) {
  auto* c = static_cast<HubCtx*>(ctx);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  return hub_call([&] {
    ck(cudaStreamSynchronize(st), "sync");
    c->hub->post[c->rank] = send;
    c->hub->barrier();
    for (int k = 0; k < c->hub->n; ++k)
      if (bytes)
        ck(cudaMemcpyAsync(static_cast<char*>(recv) + k * bytes, c->hub->post[k], bytes, cudaMemcpyDeviceToDevice, st),
           "d2d");
    ck(cudaStreamSynchronize(st), "sync");
    c->hub->barrier();
  });
}
int hub_group(void* ctx, int32_t n, const vp_p2p_op* ops, void* stream) {
  auto* c = static_cast<HubCtx*>(ctx);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  return hub_call([&] {
    ck(cudaStreamSynchronize(st), "sync");
    c->hub->ops[c->rank].assign(ops, ops + n);
    c->hub->barrier();
    // the k-th receive from peer p pairs with p's k-th send to me
    std::vector<int> seen(c->hub->n, 0);
    for (int32_t i = 0; i < n; ++i) {
      const vp_p2p_op& o = ops[i];
      if (o.send) continue;
      const int k = seen[o.peer]++;
      int j = 0;
      const vp_p2p_op* src = nullptr;
      for (const auto& q : c->hub->ops[o.peer])
        if (q.send && q.peer == c->rank && j++ == k) {
          src = &q;
          break;
        }
      if (!src || src->bytes != o.bytes) fail(VP_ECUDA, "unmatched point-to-point operation");
      if (o.bytes) ck(cudaMemcpyAsync(o.ptr, src->ptr, o.bytes, cudaMemcpyDeviceToDevice, st), "d2d");
    }
    ck(cudaStreamSynchronize(st), "sync");
    c->hub->barrier();
  });
}

}  // namespace

namespace vp {
void slab_frame_release(vp_grid* g) {
  std::lock_guard<std::mutex> lk(g_state_mu);
  g_state.erase(g);
}
}  // namespace vp

extern "C" {

int vp_comm_nccl_unique_id(uint8_t id[128]) {
  return guard([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId u;
    if (nccl().GetUniqueId(&u) != ncclSuccess) fail(VP_ECUDA, "ncclGetUniqueId failed");
    std::memcpy(id, &u, 128);
  });
}

int vp_comm_nccl_create(const uint8_t id[128], int32_t nranks, int32_t rank, int device, vp_comm_ops* out) {
  return guard([&] {
    std::memset(out, 0, sizeof *out);
    NcclApi& a = nccl();
    ck(cudaSetDevice(device), "set device");
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    auto ctx = std::make_unique<NcclCtx>();
    ctx->device = device;
    if (a.CommInitRank(&ctx->comm, nranks, u, rank) != ncclSuccess) fail(VP_ECUDA, "ncclCommInitRank failed");
    out->ctx = ctx.release();
    out->rank = rank;
    out->nranks = nranks;
    out->broadcast = nccl_broadcast;
    out->allgather = nccl_allgather;
    out->group = nccl_group;
  });
}

int vp_comm_nccl_destroy(vp_comm_ops* comm) {
  return guard([&] {
    if (!comm || !comm->ctx) return;
    auto* ctx = static_cast<NcclCtx*>(comm->ctx);
    if (ctx->comm && nccl().CommDestroy) nccl().CommDestroy(ctx->comm);
    delete ctx;
    comm->ctx = nullptr;
  });
}

int vp_slab_frame(vp_grid* slab, const vp_comm_ops* comm, const float* xyz, uint64_t n, const double rotation[9],
                  const double translation[3], const vp_pipeline_params* p, vp_polygons_t** out) {
  return guard([&] { slab_frame_impl(slab, comm, xyz, n, rotation, translation, p, out); });
}

int vp_slab_frame_local(vp_grid* const* slabs, int32_t n_slabs, const float* xyz, uint64_t n,
                        const double rotation[9], const double translation[3], const vp_pipeline_params* p,
                        vp_polygons_t** out) {
  if (out) *out = nullptr;
  if (n_slabs < 1) {
    vp::set_last_error("slab frame: no slabs");
    return VP_EINVAL;
  }
  Hub hub(n_slabs);
  std::vector<HubCtx> ctx(n_slabs);
  std::vector<vp_comm_ops> ops(n_slabs);
  std::vector<int> rc(n_slabs, VP_OK);
  std::vector<std::string> err(n_slabs);
  int origin = -1;  // the slab whose failure aborted the others
  std::vector<std::thread> th;
  for (int k = 0; k < n_slabs; ++k) {
    ctx[k] = HubCtx{&hub, k};
    ops[k] = vp_comm_ops{&ctx[k], k, n_slabs, hub_broadcast, hub_allgather, hub_group};
  }
  for (int k = 0; k < n_slabs; ++k)
    th.emplace_back([&, k] {
      rc[k] = guard([&] {
        slab_frame_impl(slabs[k], &ops[k], k == 0 ? xyz : nullptr, n, rotation, translation, p, k == 0 ? out : nullptr);
      });
      if (rc[k] != VP_OK) {
        err[k] = vp_last_error();
        if (hub.abort()) origin = k;  // written once, read after join
      }
    });
  for (auto& t : th) t.join();
  if (origin >= 0) {
    if (out && *out) {
      vp_polygons_free(*out);
      *out = nullptr;
    }
    vp::set_last_error(("slab " + std::to_string(origin) + ": " + err[origin]).c_str());
    return rc[origin];
  }
  return VP_OK;
}

}  // extern "C"
