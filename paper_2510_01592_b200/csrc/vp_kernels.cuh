// Kernel declarations and block-level primitives.
#pragma once

#include <math_constants.h>

#include "vp_device.cuh"

namespace vp {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanPerBlock = kScanThreads * kScanItems;  // 2048
constexpr int kRowItems = 2;  // occupied scan: ring rows per thread
constexpr int kRowsPerBlock = kScanThreads * kRowItems;  // 512
constexpr int kClusterBins = 2048;  // initial cluster capacity; the member sort's shared-memory bins
constexpr int kChunk = 256;         // ordinals per counting-sort chunk (one warp)
#ifndef VP_HULL_SMEM
#define VP_HULL_SMEM 1024
#endif
constexpr int kHullSmem = VP_HULL_SMEM;  // survivors sorted in shared memory (6 regions of this size)
// k_poly_hull: 256 threads own kHullSmem / 256 sorted entries each (a 32-bit keep mask),
// and the six regions of 16-byte points must fit the opt-in shared memory
static_assert(kHullSmem >= 256 && kHullSmem % 256 == 0 && kHullSmem / 256 <= 32 &&
                  kHullSmem * 16 * 6 <= 227 * 1024,
              "VP_HULL_SMEM must be a multiple of 256 in [256, 2304]");
constexpr int kPolyChunk = 1024;    // inlier points per polygon-stage block
constexpr uint32_t kPolyBig = 16384;  // fits with more inliers: projection, extremes and keep test over the whole GPU
constexpr uint32_t kRefineChunk = 512;  // inliers per refine_plane tree chunk (one block each)
constexpr int kPolyCluster = 4;     // k_poly_fused: CTAs per fit (one thread-block cluster)
#ifndef VP_POLY_THREADS
#define VP_POLY_THREADS 256
#endif
// k_poly_fused: threads per CTA. 256 rather than 512: a CTA then holds half
// an SM's registers (128 per thread) while its leader runs the serial hull,
// which leaves room for the overlapping frames' kernels (C2 5097 -> 5160
// frames/s; the polygon stage itself 60 -> 66 us)
constexpr int kPolyThreads = VP_POLY_THREADS;
constexpr int kPolySmem = 4 * kHullSmem * 16;  // k_poly_fused dynamic shared memory (4 x kHullSmem points)
#ifndef VP_FOLD_SMALL
#define VP_FOLD_SMALL 24
#endif
constexpr int kFoldSmall = VP_FOLD_SMALL;  // integrate: points per voxel folded by one thread
constexpr int kFoldMax = 128;       // integrate: points per voxel folded by one warp
constexpr uint32_t kDenseSort = 16384;  // denser voxels: indices bitonic-sorted in shared memory

// Block-wide exclusive prefix sum (any blockDim multiple of 32, <= 1024).
__device__ __forceinline__ uint32_t block_exclusive_u32(uint32_t v) {
  __shared__ uint32_t wt[32];
  const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  const unsigned nw = (blockDim.x + 31) >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (static_cast<int>(lane) >= o) incl += t;
  }
  if (lane == 31) wt[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    uint32_t t = lane < nw ? wt[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, t, o);
      if (static_cast<int>(lane) >= o) t += u;
    }
    wt[lane] = t;
  }
  __syncthreads();
  const uint32_t r = (wid ? wt[wid - 1] : 0u) + incl - v;
  __syncthreads();
  return r;
}

// Single-block exclusive scan of a[0..n) in place; *total = sum (optional
// also copied to *total2).
__device__ __forceinline__ void block_scan_array(uint32_t* a, uint32_t n, uint32_t* total, uint32_t* total2) {
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  // kScanItems consecutive values per thread: one block pass per 8 K values
  const uint32_t per = blockDim.x * kScanItems;
  for (uint32_t b = 0; b < n; b += per) {
    const uint32_t i0 = b + threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      v[k] = i0 + k < n ? __ldcg(a + i0 + k) : 0u;
      sum += v[k];
    }
    const uint32_t ex = block_exclusive_u32(sum);
    uint32_t run = carry + ex;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
      if (i0 + k < n) {
        a[i0 + k] = run;
        run += v[k];
      }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = run;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (total) *total = carry;
    if (total2) *total2 = carry;
  }
}

// True in the block that finishes last (every block of the grid must call
// it, after writing its results): the fused count kernels then scan the
// per-block sums in that block instead of a separate single-block launch.
// `done` is reset by that block.
__device__ __forceinline__ bool last_block_done(uint32_t* done) {
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    last = atomicAdd(done, 1u) == gridDim.x - 1;
    if (last) *done = 0u;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

__device__ __forceinline__ uint32_t block_sum_u32(uint32_t v) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t tot;
  const unsigned lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  const unsigned nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) ws[wid] = v;
  __syncthreads();
  if (wid == 0) {
    uint32_t t = lane < nw ? ws[lane] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (lane == 0) tot = t;
  }
  __syncthreads();
  const uint32_t r = tot;
  __syncthreads();
  return r;
}

// 2-D points of the polygon stage (polygonize.cpp): lexicographic order and
// the orientation test cross2 (o, a, b) in the reference's expression order.
struct P2 {
  double x, y;
};
__device__ __forceinline__ bool lex_less(P2 a, P2 b) { return a.x < b.x || (a.x == b.x && a.y < b.y); }
__device__ __forceinline__ double cross2(P2 o, P2 a, P2 b) {
  return (a.x - o.x) * (b.y - o.y) - (a.y - o.y) * (b.x - o.x);
}

// Union-find over int32 parent arrays (CCL and the slab boundary merge).
// Parent pointers only ever move to an ancestor (hooks: root -> smaller root;
// pointer jumping: node -> grandparent), so every value a thread can observe
// is an ancestor of the node. Reads go through L2 (ld.cg): a stale value is
// still an ancestor, so "same root" answers are always right and a wrong
// "different roots" answer is corrected by the atomicCAS retry.
__device__ __forceinline__ int uf_find(int32_t* parent, int v) {
  int par = __ldcg(parent + v);
  if (par != v) {
    int next, prev = v;
    while (par > (next = __ldcg(parent + par))) {
      __stcg(parent + prev, next);  // pointer jumping; parent[x] <= x always holds
      prev = par;
      par = next;
    }
  }
  return par;
}

// Link two roots (larger under smaller); returns the surviving root. The CAS
// is tried only when hi still reads as a root: a stale root (already hooked
// by another thread) is climbed with a plain load. Without the check every
// late union of two already-joined trees was a failed CAS on one of the few
// component roots, serialised in its L2 slice (C2: ~74k ATOMs on ~31 roots).
__device__ __forceinline__ int uf_link(int32_t* parent, int ra, int rb) {
  while (ra != rb) {
    const int lo = ra < rb ? ra : rb;
    const int hi = ra < rb ? rb : ra;
    const int cur = __ldcg(parent + hi);
    if (cur != hi) {  // hi was hooked meanwhile: climb without an atomic
      if (ra == hi) ra = cur; else rb = cur;
      continue;
    }
    const int ret = atomicCAS(parent + hi, hi, lo);
    if (ret == hi) return lo;
    if (ra == hi) ra = ret; else rb = ret;  // hi was hooked meanwhile: climb
  }
  return ra;
}

__device__ __forceinline__ void uf_union(int32_t* parent, int a, int b) {
  uf_link(parent, uf_find(parent, a), uf_find(parent, b));
}

// Segmentation parameters resolved on the host (thresholds computed with the
// host libm exactly as the reference computes them).
struct SegDev {
  int radius;          // SegmentationParams.neighbor_radius
  int min_neighbors;
  double dstar;        // smallest d with acos(d)*kRadToDeg <= max_angle_deg (host libm)
  d3 up;
  int w;               // max(1, ceil(distance_th / resolution))   segmentation.cpp:89
  double d2_th;        // distance_th^2                             segmentation.cpp:90
  double cos_th;       // cos(adjacency_angle_deg * kDegToRad)      segmentation.cpp:91
  int min_cluster;     // min_cluster_size
};

struct RansacDev {
  int iterations;
  double eps;
  uint64_t seed;
  d3 up;
};

// Dense ordinal lookup volume for the CCL window search (segmentation.cpp:96-110):
// the grid's logical extent on the fused path, the steppable bounding box for a
// host-provided list.
struct MapDesc {
  int32_t* map;    // ordinal or -1 per slot
  uint32_t* bits;  // 1 bit per slot (steppable present), rows of W words
  int lo[3];
  int dims[3];
  int W;
  __device__ __forceinline__ uint64_t slot(int x, int y, int z) const {
    return (static_cast<uint64_t>(x - lo[0]) * dims[1] + (y - lo[1])) * dims[2] + (z - lo[2]);
  }
  __device__ __forceinline__ uint64_t word(int x, int y, int z) const {
    return (static_cast<uint64_t>(x - lo[0]) * dims[1] + (y - lo[1])) * W + ((z - lo[2]) >> 5);
  }
  // `count` (<= 32) presence bits of row (x, y) starting at z0
  __device__ __forceinline__ uint32_t row_span(int x, int y, int z0, int count) const {
    const uint32_t* row = bits + (static_cast<uint64_t>(x - lo[0]) * dims[1] + (y - lo[1])) * W;
    const int b0 = z0 - lo[2];
    const int wl = b0 >> 5, sh = b0 & 31;
    const uint32_t a = __ldg(row + wl);
    const uint32_t hi = (sh && wl + 1 < W) ? __ldg(row + wl + 1) : 0u;
    const uint32_t v = sh ? ((a >> sh) | (hi << (32 - sh))) : a;
    return count >= 32 ? v : (v & ((1u << count) - 1u));
  }
};

// Buffers of the segmentation stage.
struct SegBufs {
  // occupied list (Vcap)
  uint32_t* occ_list;
  double* est_normal;    // 3*Vcap
  int32_t* est_ncount;
  uint8_t* est_valid;
  double* own_mean;      // 3*Vcap
  uint32_t* own_count;
  uint8_t* own_status;
  uint8_t* step_flag;
  // steppable (Scap)
  int32_t* st_idx;       // 3*Scap window indices
  double* st_mean;       // 3*Scap
  double* st_normal;     // 3*Scap
  int32_t* parent;       // union-find
  int32_t* label;        // canonical labels
  uint32_t* cnt;         // members per root
  int32_t* cid;          // cluster index of a big root, else -1
  uint8_t* big_flag;
  uint32_t* big_pos;
  // clusters (Kcap)
  int32_t* klabel;       // cluster label (= root ordinal)
  uint32_t* ksize;
  uint32_t* kpoff;       // K+1 warp-padded member offsets
  uint32_t* H;           // K x nchunks histogram / offsets
  // members (padded, Mcap)
  double* mx;
  double* my;
  double* mz;
  // RANSAC candidates (Kcap x iterations)
  double* cand;          // 4 per candidate: n.x n.y n.z offset
  int32_t* cand_cnt;     // -1 degenerate
  int32_t* win_it;       // per cluster: winner, -1 unfit, -2 skipped small
  int32_t* win_cnt;
  int32_t* fid;          // fit index of a cluster or -1
  uint32_t* fit_cluster; // cluster of a fit
  uint32_t* ioff;        // per fit inlier offsets (nfits+1)
  uint32_t* fch_off;     // per fit member-chunk offsets (nfits+1)
  uint32_t* ccount;      // per member chunk: inlier count, then exclusive offset
  uint32_t cch_cap;
  double* fit_model;     // 4 per fit (normal, offset): RANSAC winner
  int32_t* fit_meta;     // 2 per fit (inlier_count, label)
  double* ref_model;     // 4 per fit: refined
  uint32_t* rch_off;     // per fit refine-chunk offsets (nfits+1)
  double* rpart;         // 8 per refine chunk: partial sums
  double* rcen;          // 3 per fit: refine centroid
  double* inl;           // 3 * Icap inliers (fit order)
  double* proj;          // 2 * Icap
  double* surv;          // 2 * 2Icap
  double* hull;          // 2 * 2Icap
  // polygon records (Kcap) + vertex pool
  double* basis;         // 9 per fit: u, v, origin (plane_basis)
  uint32_t* pch_off;     // per fit chunk offsets (nfits+1)
  double* pext_dot;      // 64 per chunk: per-direction extreme dot
  int32_t* pext_idx;     // 64 per chunk: its point index
  double* inner;         // 2*130 per fit: inner polygon
  uint32_t* ninner;
  uint32_t* nsurv;       // survivors per fit
  uint32_t* pdone;       // per fit chunk tickets of the wide polygon passes (reset by the last chunk)
  uint32_t pch_cap;
  double* prec_d;        // 8 per fit: normal(3) offset area
  int32_t* prec_i;       // 4 per fit: inlier_count label nv voff
  double* pool;          // 5 per vertex: u v x y z
  uint32_t pool_cap;
  uint32_t Vcap, Scap, Mcap, Icap;
  uint32_t Kcap;         // clusters a frame can hold (grown on kOverflowClusters)
  uint64_t Hcap;         // entries of H (clusters x member-sort chunks)
  // CCL root-pair set: open-addressed keys (hi << 32 | lo, ~0 = empty) and the
  // list of occupied slots (pair_cap / 2 entries)
  unsigned long long* pair_key;
  uint32_t* pair_slot;
  uint32_t pair_cap;     // power of two
};

// ---- spatial slabs (k_slab.cu)
constexpr int kMaxSlabs = 64;

// Boundary zone: window x intervals [xlo, xhi) within w of an internal slab
// boundary; zone index of ordinal o in interval k = dbase[k] + (o - olo[k]).
struct ZoneDesc {
  int n;
  int32_t xlo[kMaxSlabs], xhi[kMaxSlabs];
  int64_t olo[kMaxSlabs], dbase[kMaxSlabs];
};

// First global ordinal of every slab (slab k owns [ord_lo[k], ord_lo[k+1])).
struct RankDesc {
  int n;
  int64_t ord_lo[kMaxSlabs];
};

// A cluster member sent to the slab that owns its cluster (32 B).
struct MemberRec {
  double m[3];
  int32_t label;
  int32_t pad;
};

// clear_rays work binning (k_map.cu): rays grouped by estimated DDA length
// when warps of consecutive rays would be badly unbalanced (LiDAR patterns).
constexpr int kDdaBins = 64;
struct DdaBins {
  uint32_t count[kDdaBins];
  uint32_t cursor[kDdaBins];
  unsigned long long steps;     // sum of estimated steps
  unsigned long long warp_max;  // sum over 32-ray groups of 32 x their longest ray
  int use;                      // 1: walk rays in bin order (perm), 0: identity
  uint32_t frame;               // frames planned (a coherent stream is re-measured every 8th)
};

// Height-map baseline (k_heightmap.cu): cells x-major, flat = x * ey + y.
struct HmDesc {
  double* h;         // height per cell
  uint8_t* valid;
  uint32_t* win;     // per frame: last point index + 1
  int32_t* parent;   // union-find over cells
  int32_t* root;     // region root (seed flat index) of every cell, after the unions
  uint32_t* claim;   // BFS: min (frontier position * 4 + step)
  uint8_t* visited;
  uint32_t* spos;    // visit position of a region's seed (roots only)
  int ex, ey;
  double ox, oy, res;
};

// ---- kernels (k_map.cu)
__global__ void k_integrate_hash(GridDesc g, const FrameParams* fp, Counters* ctr, uint32_t* hkey,
                                 uint32_t* hcnt, uint32_t hmask, uint32_t* groups, uint32_t* pslot,
                                 uint32_t* prank);
__global__ void k_integrate_offsets(Counters* ctr, uint32_t* groups, const uint32_t* hcnt,
                                    uint32_t* hoff, uint32_t* medium, uint32_t* dense);
__global__ void k_integrate_scatter(const FrameParams* fp, const uint32_t* pslot,
                                    const uint32_t* prank, const uint32_t* hoff, uint32_t* sorted);
__global__ void k_integrate_fold(GridDesc g, const FrameParams* fp, Counters* ctr,
                                 const uint32_t* groups, uint32_t* hkey, uint32_t* hcnt,
                                 const uint32_t* hoff, uint32_t* sorted);
__global__ void k_integrate_fold_medium(GridDesc g, const FrameParams* fp, Counters* ctr, uint32_t* hkey,
                                        uint32_t* hcnt, const uint32_t* hoff, const uint32_t* sorted,
                                        const uint32_t* medium);
__global__ void k_integrate_fold_dense(GridDesc g, const FrameParams* fp, Counters* ctr, uint32_t* hkey,
                                       uint32_t* hcnt, const uint32_t* hoff, const uint32_t* sorted,
                                       const uint32_t* pslot, const uint32_t* dense);
constexpr int kDenseSmem = 1024 * 24 + 16384 * 4;  // k_integrate_fold_dense dynamic shared memory
__global__ void k_clear_walk(GridDesc g, const FrameParams* fp, const uint32_t* perm, const DdaBins* db, int generic);
__global__ void k_clear_walk_slab(GridDesc g, const FrameParams* fp, const uint32_t* perm, const DdaBins* db);
__global__ void k_dda_keys(GridDesc g, const FrameParams* fp, DdaBins* db, uint8_t* bin_of);
__global__ void k_dda_plan(DdaBins* db, int force, int long_steps);
__global__ void k_dda_scatter(const FrameParams* fp, DdaBins* db, const uint8_t* bin_of, uint32_t* perm);
__global__ void k_clear_apply(GridDesc g, const FrameParams* fp, Counters* ctr, const DdaBins* db, int use_box);
__global__ void k_recenter(GridDesc g, const FrameParams* fp, Counters* ctr, unsigned long long* occ_total);
__global__ void k_map_finalize(Counters* ctr, unsigned long long* occ_total);
__global__ void k_frame_begin(Counters* ctr, const unsigned long long* occ_total);
__global__ void k_set_statuses(GridDesc g, const FrameParams* fp, const int32_t* idx, const uint8_t* st,
                               uint64_t n);
__global__ void k_flags_count(const uint8_t* flags, const uint32_t* n_ptr, uint32_t cap,
                              uint32_t* bsum, uint32_t* total, uint32_t* done);
__global__ void k_flags_positions(const uint8_t* flags, const uint32_t* n_ptr, uint32_t cap,
                                  const uint32_t* boff, uint32_t* pos_out);
__global__ void k_merge_point(GridDesc g, const FrameParams* fp, Counters* ctr, int x, int y, int z,
                              double px, double py, double pz);
__global__ void k_bitmap_count(GridDesc g, const FrameParams* fp, uint64_t w_lo, uint64_t nwords, uint32_t* bsum,
                               Counters* ctr);
__global__ void k_bitmap_emit(GridDesc g, const FrameParams* fp, uint64_t w_lo, uint64_t nwords,
                              const uint32_t* boff, uint32_t* out, uint32_t cap);
__global__ void k_scan_exclusive(uint32_t* a, uint32_t n_static, const uint32_t* n_ptr,
                                 uint32_t* total, uint32_t* total2);
__global__ void k_scan_tiles(uint32_t* a, const uint32_t* n_ptr, uint32_t cap, uint32_t per, uint32_t* total);

// ---- kernels (k_segment.cu)
__global__ void k_normals(GridDesc g, const FrameParams* fp, Counters* ctr, SegDev sp, SegBufs b,
                          int write_status, uint32_t* tsum);
__global__ void k_adjacency(Counters* ctr, SegDev sp, SegBufs b, MapDesc m, const uint64_t* rows,
                            uint32_t* counts, int32_t* cols);
__global__ void k_step_emit(GridDesc g, Counters* ctr, SegBufs b, MapDesc m, int xadd, const uint32_t* toff);
__global__ void k_map_fill(Counters* ctr, SegBufs b, MapDesc m);
__global__ void k_occ_gather(GridDesc g, const FrameParams* fp, Counters* ctr, SegBufs b);
__global__ void k_ccl_init(Counters* ctr, SegBufs b);
__global__ void k_ccl_union(Counters* ctr, SegDev sp, SegBufs b, MapDesc m);
__global__ void k_ccl_hook_bal(Counters* ctr, SegDev sp, SegBufs b, MapDesc m);
__global__ void k_ccl_jump(Counters* ctr, SegBufs b);
__global__ void k_ccl_compress_exact(Counters* ctr, SegBufs b);
__global__ void k_ccl_pairs(Counters* ctr, SegDev sp, SegBufs b, MapDesc m);
__global__ void k_ccl_pairs_union(Counters* ctr, SegDev sp, SegBufs b, MapDesc m);
__global__ void k_ccl_union_bal(Counters* ctr, SegDev sp, SegBufs b, MapDesc m);
__global__ void k_ccl_hook(Counters* ctr, SegDev sp, SegBufs b, MapDesc m);
__global__ void k_ccl_compress(Counters* ctr, SegBufs b);
__global__ void k_ccl_lattice(Counters* ctr, SegDev sp, SegBufs b, MapDesc m);
__global__ void k_ccl_giant(Counters* ctr, SegBufs b);
__global__ void k_ccl_full(Counters* ctr, SegDev sp, SegBufs b, MapDesc m);
__global__ void k_ccl_flatten(Counters* ctr, SegBufs b, MapDesc m);
__global__ void k_cluster_flags(Counters* ctr, SegDev sp, SegBufs b);
__global__ void k_cluster_assign(Counters* ctr, SegBufs b);
__global__ void k_member_hist(Counters* ctr, SegBufs b, uint32_t hstride);
__global__ void k_member_hscan(Counters* ctr, SegBufs b, uint32_t hstride);
__global__ void k_member_scatter(Counters* ctr, SegBufs b, uint32_t hstride);
__global__ void k_ransac_hyp(Counters* ctr, RansacDev rp, SegBufs b);
__global__ void k_ransac_count(Counters* ctr, RansacDev rp, SegBufs b);
__global__ void k_ransac_select(Counters* ctr, RansacDev rp, SegBufs b);
__global__ void k_extract_count(Counters* ctr, RansacDev rp, SegBufs b);
__global__ void k_extract_emit(Counters* ctr, RansacDev rp, SegBufs b);
__global__ void k_refine(Counters* ctr, SegBufs b, d3 up, int refine, int exact);
__global__ void k_refine_setup(Counters* ctr, SegBufs b, int refine);
__global__ void k_refine_part0(Counters* ctr, SegBufs b);
__global__ void k_refine_part1(Counters* ctr, SegBufs b, d3 up);
__global__ void k_poly_setup(Counters* ctr, SegBufs b);
__global__ void k_poly_extremes(Counters* ctr, SegBufs b, const double* dirtab, int directions, int planar);
__global__ void k_poly_wide_ext(Counters* ctr, SegBufs b, const double* dirtab, int directions, int planar);
__global__ void k_poly_wide_keep(Counters* ctr, SegBufs b);
__global__ void k_poly_fused(Counters* ctr, SegBufs b, const double* dirtab, int directions, int planar, double min_area);
__global__ void k_poly_inner(Counters* ctr, SegBufs b, int directions);
__global__ void k_poly_keep(Counters* ctr, SegBufs b);
__global__ void k_poly_hull(Counters* ctr, SegBufs b, double min_area);
__global__ void k_chain_rearm(Counters* ctr);
__global__ void k_poly_pack(const Counters* ctr, SegBufs b, double* out, uint64_t cap);

// ---- kernels (k_api.cu)
__global__ void k_jacobi_batch(uint64_t n, const double* a, double* vals, double* vecs);
__global__ void k_poly_keep_flags(Counters* ctr, SegBufs b, uint8_t* flags);
__global__ void k_gather_p2(const uint32_t* n_ptr, const uint8_t* flags, const uint32_t* pos, const double* proj,
                            double* out);
__global__ void k_iota(int32_t* a, uint64_t n);
__global__ void k_label_edges(uint64_t n, const uint64_t* rows, const int32_t* cols, int32_t* parent);
__global__ void k_label_flatten(uint64_t n, int32_t* parent, int32_t* label);
__global__ void k_classify_estimates(uint64_t n, const int32_t* ncount, const double* angle, const uint8_t* valid,
                                     int min_neighbors, double max_angle, uint8_t* status);

// ---- kernels (k_slab.cu)
__global__ void k_plane_counts(const Counters* ctr, const int32_t* st_idx, uint32_t cap, int32_t x0,
                               int32_t nplanes, uint32_t* counts);
__global__ void k_fill_i32(int32_t* a, uint64_t n, int32_t v);
__global__ void k_zone_bmin(const Counters* ctr, SegBufs b, ZoneDesc z, int32_t* bmin);
__global__ void k_zone_triples(const Counters* ctr, SegBufs b, ZoneDesc z, int64_t base,
                               const int32_t* bmin, int32_t* out, uint32_t* nout);
__global__ void k_zone_init(int32_t* parent, int32_t* minlab, uint64_t Z);
__global__ void k_zone_union(const int32_t* t, uint64_t n, int32_t* parent);
__global__ void k_zone_minlab(const int32_t* t, uint64_t n, int32_t* parent, int32_t* minlab);
__global__ void k_slab_relabel(SegBufs b, ZoneDesc z, int64_t base, uint32_t n_left, uint32_t n_own,
                               const int32_t* bmin, int32_t* parent, const int32_t* minlab, int32_t* flabel);
__global__ void k_export_hist(uint32_t n_own, const int32_t* flabel, RankDesc rd, int me, uint32_t* H,
                              uint32_t nch, uint32_t* dcount);
__global__ void k_export_scatter(uint32_t n_own, const int32_t* flabel, const double* mean, RankDesc rd,
                                 int me, const uint32_t* H, uint32_t nch, MemberRec* out);
__global__ void k_owner_init(uint32_t n, SegBufs b);
__global__ void k_owner_prep(uint32_t n_own, uint32_t n_recv, int64_t own_base, const double* own_mean,
                             const int32_t* flabel, const MemberRec* recv, SegBufs b);
__global__ void k_klabel_rebase(const Counters* ctr, SegBufs b, int64_t base);

// ---- kernels (k_heightmap.cu)
__global__ void k_hm_win(HmDesc m, const FrameParams* fp);
__global__ void k_hm_write(HmDesc m, const FrameParams* fp);
__global__ void k_hm_ccl_init(HmDesc m);
__global__ void k_hm_ccl_union(HmDesc m, double dth);
__global__ void k_hm_seed_flags(HmDesc m, uint8_t* flags);
__global__ void k_hm_seed_emit(HmDesc m, const uint8_t* flags, const uint32_t* pos, uint32_t* visit);
__global__ void k_hm_bfs(HmDesc m, uint32_t* visit, uint32_t* dn, double dth);
__global__ void k_hm_members(HmDesc m, const uint32_t* visit, uint32_t nv, SegBufs b);
__global__ void k_hm_zero_cnt(uint32_t nv, SegBufs b);
__global__ void k_hm_klabel(const Counters* ctr, SegBufs b, const uint32_t* visit);

}  // namespace vp
