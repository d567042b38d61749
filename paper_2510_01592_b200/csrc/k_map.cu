// Voxel-map kernels: integrate_frame, clear_rays, recenter, occupied scan.
// Reference: /root/reference/proj/core/src/voxel_grid.cpp.
#include "vp_kernels.cuh"

namespace vp {

// ---------------------------------------------------------------------------
// integrate_frame (voxel_grid.cpp:59-115)
//
// The reference sorts (flat, point index) pairs and folds each voxel's points
// in ascending index. Here: (A) transform + key + warp-aggregated hash
// insertion (__match_any_sync over identical keys, one atomic per distinct key
// per warp, ranks in lane order), (B) per-group output ranges, (C) scatter
// point indices, (D) one thread per touched voxel sorts its (short, nearly
// ordered) index list and performs the ordered FP64 fold, so the sums are
// bit-identical to the sequential reference.
// ---------------------------------------------------------------------------
// 0: discarded (non-finite or outside the window), 1: inserted into *key,
// 2: inside the window but owned by another slab.
__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
// box: grows by the point's cell clamped to the grid (local x): every cell its
// ray can mark lies between the sensor's and this cell, per axis.
__device__ __forceinline__ int point_key(const GridDesc& g, const FrameParams* fp, uint64_t i,
                                         uint32_t* key, int* box) {
  const float* p = fp->pts + 3 * i;
  const d3 w = pose_apply(fp->R, fp->t, static_cast<double>(p[0]), static_cast<double>(p[1]),
                          static_cast<double>(p[2]));
  if (!finite3(w)) return 0;
  const int ix = w2i(w.x, fp->origin_pre[0], g.res);  // window coordinates
  const int iy = w2i(w.y, fp->origin_pre[1], g.res);
  const int iz = w2i(w.z, fp->origin_pre[2], g.res);
  {
    const int cx = clampi(ix - g.xoff, 0, g.ex - 1), cy = clampi(iy, 0, g.ey - 1), cz = clampi(iz, 0, g.ez - 1);
    box[0] = min(box[0], cx), box[1] = min(box[1], cy), box[2] = min(box[2], cz);
    box[3] = max(box[3], cx), box[4] = max(box[4], cy), box[5] = max(box[5], cz);
  }
  if (ix < 0 || iy < 0 || iz < 0 || ix >= g.gex || iy >= g.ey || iz >= g.ez) return 0;
  const int lx = ix - g.xoff;
  if (lx < g.own_lo || lx >= g.own_hi) return 2;
  *key = static_cast<uint32_t>((static_cast<uint64_t>(lx) * g.ey + iy) * g.ez + iz);
  return 1;
}

__global__ void k_integrate_hash(GridDesc g, const FrameParams* __restrict__ fp, Counters* ctr,
                                 uint32_t* hkey, uint32_t* hcnt, uint32_t hmask, uint32_t* groups,
                                 uint32_t* pslot, uint32_t* prank) {
  VP_GRID_WAIT();
  const uint64_t n = fp->n;
  unsigned long long disc = 0;
  const unsigned lane = lane_id();
  int box[6] = {0x7fffffff, 0x7fffffff, 0x7fffffff, -1, -1, -1};
  if (blockIdx.x == 0 && threadIdx.x == 0 && n) {  // the sensor's cell (rays start there)
    const int cx = clampi(w2i(fp->t[0], fp->origin_pre[0], g.res) - g.xoff, 0, g.ex - 1);
    const int cy = clampi(w2i(fp->t[1], fp->origin_pre[1], g.res), 0, g.ey - 1);
    const int cz = clampi(w2i(fp->t[2], fp->origin_pre[2], g.res), 0, g.ez - 1);
    box[0] = box[3] = cx, box[1] = box[4] = cy, box[2] = box[5] = cz;
  }
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x; i0 < n;
       i0 += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    uint32_t key = kEmptyKey;
    bool valid = false;
    if (i < n) {
      const int r = point_key(g, fp, i, &key, box);
      valid = r == 1;
      if (r == 0) ++disc;
      if (r == 2) key = kEmptyKey;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(peers) - 1;
    uint32_t slot = 0, base = 0;
    bool fresh = false;
    if (valid && static_cast<int>(lane) == leader) {
      uint32_t h = hash_u32(key) & hmask;
      for (;;) {
        const uint32_t prev = atomicCAS(&hkey[h], kEmptyKey, key);
        if (prev == kEmptyKey) {
          fresh = true;
          break;
        }
        if (prev == key) break;
        h = (h + 1) & hmask;
      }
      slot = h;
      base = atomicAdd(&hcnt[h], static_cast<uint32_t>(__popc(peers)));
    }
    const unsigned fm = __ballot_sync(0xffffffffu, fresh);
    if (fm) {
      const int first = __ffs(fm) - 1;
      uint32_t gb = 0;
      if (static_cast<int>(lane) == first) gb = atomicAdd(&ctr->ngroups, static_cast<uint32_t>(__popc(fm)));
      gb = __shfl_sync(0xffffffffu, gb, first);
      if (fresh) groups[gb + __popc(fm & lanemask_lt())] = slot;
    }
    slot = __shfl_sync(0xffffffffu, slot, leader);
    base = __shfl_sync(0xffffffffu, base, leader);
    if (i < n) {
      pslot[i] = valid ? slot : kEmptyKey;
      prank[i] = base + __popc(peers & lanemask_lt());
    }
  }
  block_add_u64(&ctr->discarded, disc);
  // the block's box -> 6 atomics per block
  __shared__ int sbox[6];
  if (threadIdx.x < 6) sbox[threadIdx.x] = threadIdx.x < 3 ? 0x7fffffff : -1;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int lo = __reduce_min_sync(0xffffffffu, box[k]), hi = __reduce_max_sync(0xffffffffu, box[3 + k]);
    if (lane == 0) {
      atomicMin(&sbox[k], lo);
      atomicMax(&sbox[3 + k], hi);
    }
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    if (sbox[threadIdx.x] != 0x7fffffff) atomicMin(&ctr->box_lo[threadIdx.x], sbox[threadIdx.x]);
  } else if (threadIdx.x < 6) {
    if (sbox[threadIdx.x] >= 0) atomicMax(&ctr->box_hi[threadIdx.x - 3], sbox[threadIdx.x]);
  }
}

// Per-group ranges of the point-index buffer; groups too large for one
// thread are listed for the warp pass (<= kFoldMax points) or the block pass
// and tagged in `groups`, so the three fold kernels are independent of each
// other (the thread pass never reads a tagged group's hash slot, which the
// other passes reset).
constexpr uint32_t kBigGroup = 0x80000000u;
__global__ void k_integrate_offsets(Counters* ctr, uint32_t* groups, const uint32_t* hcnt,
                                    uint32_t* hoff, uint32_t* medium, uint32_t* dense) {
  VP_GRID_WAIT();
  const uint32_t ng = ctr->ngroups;
  const unsigned lane = lane_id();
  for (uint32_t i0 = blockIdx.x * blockDim.x; i0 < ng; i0 += gridDim.x * blockDim.x) {
    const uint32_t i = i0 + threadIdx.x;
    const bool in = i < ng;
    const uint32_t slot = in ? groups[i] : 0;
    const uint32_t c = in ? hcnt[slot] : 0;
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (static_cast<int>(lane) >= o) incl += v;
    }
    uint32_t base = 0;
    if (lane == 31) base = atomicAdd(&ctr->group_cursor, incl);
    base = __shfl_sync(0xffffffffu, base, 31);
    if (in) {
      hoff[slot] = base + incl - c;
      if (c > static_cast<uint32_t>(kFoldSmall)) {
        if (c <= static_cast<uint32_t>(kFoldMax))
          medium[atomicAdd(&ctr->nmedium, 1u)] = slot;  // warp pass
        else
          dense[atomicAdd(&ctr->ndense, 1u)] = slot;  // block pass
        groups[i] = slot | kBigGroup;
      }
    }
  }
}

__global__ void k_integrate_scatter(const FrameParams* __restrict__ fp, const uint32_t* pslot,
                                    const uint32_t* prank, const uint32_t* hoff, uint32_t* sorted) {
  VP_GRID_WAIT();
  const uint64_t n = fp->n;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t s = pslot[i];
    if (s != kEmptyKey) sorted[hoff[s] + prank[i]] = static_cast<uint32_t>(i);
  }
}

constexpr int kFoldWarps = 8;

__device__ __forceinline__ void fold_cell(const GridDesc& g, const FrameParams* fp, uint32_t key,
                                          const d3* w, uint32_t cnt, unsigned long long& fresh) {
  const uint32_t r = fdiv(key, g.fez), z = key - r * static_cast<uint32_t>(g.ez);
  const uint32_t x = fdiv(r, g.fey), y = r - x * static_cast<uint32_t>(g.ey);
  Cell* c = g.cells + phys_index(g, fp->off_pre, x, y, z);
  double sx = c->sx, sy = c->sy, sz = c->sz;
  const uint32_t count = c->count;
  for (uint32_t a = 0; a < cnt; ++a) {
    sx += w[a].x;
    sy += w[a].y;
    sz += w[a].z;
  }
  c->sx = sx;
  c->sy = sy;
  c->sz = sz;
  c->count = count + cnt;
  c->status = 1;  // VoxelStatus::Occupied
  if (count == 0) {
    occ_set(g, fp->occ_pre, fp->off_pre, fp->zb_pre, x, y, z);
    ++fresh;
  }
}

// Most voxels receive a handful of points: one thread per voxel sorts its
// (<= kFoldSmall) point indices in registers and folds them; larger groups
// (listed by k_integrate_offsets) are folded concurrently by the warp-per-voxel
// and block passes.
__global__ void __launch_bounds__(256) k_integrate_fold(GridDesc g, const FrameParams* __restrict__ fp,
                                                        Counters* ctr, const uint32_t* groups,
                                                        uint32_t* hkey, uint32_t* hcnt,
                                                        const uint32_t* hoff, uint32_t* sorted) {
  VP_GRID_WAIT();
  const uint32_t ng = ctr->ngroups;
  unsigned long long fresh = 0;
  for (uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x; gi < ng; gi += gridDim.x * blockDim.x) {
    const uint32_t slot = groups[gi];
    if (slot & kBigGroup) continue;  // the warp or block pass
    const uint32_t cnt = hcnt[slot];
    const uint32_t key = hkey[slot];
    const uint32_t* lst = sorted + hoff[slot];
    uint32_t idx[kFoldSmall];
#pragma unroll
    for (int a = 0; a < kFoldSmall; ++a) idx[a] = a < static_cast<int>(cnt) ? lst[a] : 0xffffffffu;
    // insertion sort (ascending point index = the reference's fold order)
#pragma unroll
    for (int a = 1; a < kFoldSmall; ++a) {
#pragma unroll
      for (int b = a; b > 0; --b) {
        const uint32_t lo = min(idx[b - 1], idx[b]), hi = max(idx[b - 1], idx[b]);
        idx[b - 1] = lo;
        idx[b] = hi;
      }
    }
    const uint32_t r = fdiv(key, g.fez), z = key - r * static_cast<uint32_t>(g.ez);
    const uint32_t x = fdiv(r, g.fey), y = r - x * static_cast<uint32_t>(g.ey);
    Cell* c = g.cells + phys_index(g, fp->off_pre, x, y, z);
    double sx = c->sx, sy = c->sy, sz = c->sz;
    const uint32_t count = c->count;
#pragma unroll
    for (int a = 0; a < kFoldSmall; ++a) {
      if (a >= static_cast<int>(cnt)) break;
      const float* p = fp->pts + 3 * static_cast<uint64_t>(idx[a]);
      const d3 w = pose_apply(fp->R, fp->t, static_cast<double>(p[0]), static_cast<double>(p[1]),
                              static_cast<double>(p[2]));
      sx += w.x;
      sy += w.y;
      sz += w.z;
    }
    c->sx = sx;
    c->sy = sy;
    c->sz = sz;
    c->count = count + cnt;
    c->status = 1;  // VoxelStatus::Occupied
    if (count == 0) {
      occ_set(g, fp->occ_pre, fp->off_pre, fp->zb_pre, x, y, z);
      ++fresh;
    }
    hkey[slot] = kEmptyKey;
    hcnt[slot] = 0;
  }
  block_add_u64(&ctr->newly, fresh);
}

// Voxels with kFoldSmall < points <= kFoldMax: one warp per voxel: the point
// indices are staged in shared memory, ranked (indices are distinct, so rank
// = number of smaller indices), the points are transformed in parallel, and
// lane 0 performs the reference's sequential FP64 fold (voxel_grid.cpp:104-110)
// in ascending point index.
__global__ void __launch_bounds__(256) k_integrate_fold_medium(GridDesc g, const FrameParams* __restrict__ fp,
                                                               Counters* ctr, uint32_t* hkey, uint32_t* hcnt,
                                                               const uint32_t* hoff, const uint32_t* sorted,
                                                               const uint32_t* medium) {
  VP_GRID_WAIT();
  __shared__ uint32_t raw[kFoldWarps][kFoldMax];
  __shared__ uint32_t srt[kFoldMax * kFoldWarps];
  __shared__ d3 sw[kFoldWarps][kFoldMax];
  const uint32_t nm = ctr->nmedium;
  const unsigned lane = lane_id(), wid = threadIdx.x >> 5;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarp = (gridDim.x * blockDim.x) >> 5;
  unsigned long long fresh = 0;
  for (uint32_t gi = warp; gi < nm; gi += nwarp) {
    const uint32_t slot = medium[gi];
    const uint32_t key = hkey[slot];
    const uint32_t cnt = hcnt[slot];
    const uint32_t* lst = sorted + hoff[slot];
    for (uint32_t k = lane; k < cnt; k += 32) raw[wid][k] = lst[k];
    __syncwarp();
    for (uint32_t k = lane; k < cnt; k += 32) {
      const uint32_t v = raw[wid][k];
      uint32_t rank = 0;
      for (uint32_t q = 0; q < cnt; ++q) rank += raw[wid][q] < v ? 1u : 0u;
      srt[wid * kFoldMax + rank] = v;
    }
    __syncwarp();
    for (uint32_t k = lane; k < cnt; k += 32) {
      const float* p = fp->pts + 3 * static_cast<uint64_t>(srt[wid * kFoldMax + k]);
      sw[wid][k] = pose_apply(fp->R, fp->t, static_cast<double>(p[0]), static_cast<double>(p[1]),
                              static_cast<double>(p[2]));
    }
    __syncwarp();
    if (lane == 0) {
      fold_cell(g, fp, key, sw[wid], cnt, fresh);
      hkey[slot] = kEmptyKey;
      hcnt[slot] = 0;
    }
    __syncwarp();
  }
  warp_add_u64(&ctr->newly, fresh);
}

// Voxels with more than kFoldMax points (coarse grids, points next to the
// sensor): one block per voxel. Up to kDenseSort indices are bitonic-sorted
// in shared memory; larger groups are gathered in index order by streaming
// the whole frame's point->slot table (no sort, any size). The points are
// transformed by the block 1024 at a time and thread 0 folds them in
// ascending index (voxel_grid.cpp:104-110), bit-exact.
__global__ void __launch_bounds__(1024) k_integrate_fold_dense(GridDesc g, const FrameParams* __restrict__ fp,
                                                               Counters* ctr, uint32_t* hkey, uint32_t* hcnt,
                                                               const uint32_t* hoff, const uint32_t* sorted,
                                                               const uint32_t* pslot, const uint32_t* dense) {
  VP_GRID_WAIT();
  extern __shared__ __align__(16) unsigned char smem[];
  d3* w = reinterpret_cast<d3*>(smem);                          // 1024 transformed points
  uint32_t* keys = reinterpret_cast<uint32_t*>(smem + 1024 * sizeof(d3));  // kDenseSort indices
  __shared__ uint32_t wcount[32];
  __shared__ uint32_t run_base;
  const uint32_t nd = ctr->ndense;
  const uint32_t t = threadIdx.x;
  for (uint32_t di = blockIdx.x; di < nd; di += gridDim.x) {
    const uint32_t slot = dense[di];
    const uint32_t key = hkey[slot];
    const uint32_t cnt = hcnt[slot];
    const uint32_t r = fdiv(key, g.fez), z = key - r * static_cast<uint32_t>(g.ez);
    const uint32_t x = fdiv(r, g.fey), y = r - x * static_cast<uint32_t>(g.ey);
    Cell* c = g.cells + phys_index(g, fp->off_pre, x, y, z);
    double sx = 0.0, sy = 0.0, sz = 0.0;
    uint32_t count = 0;
    if (t == 0) {
      sx = c->sx;
      sy = c->sy;
      sz = c->sz;
      count = c->count;
    }
    if (cnt <= kDenseSort) {
      uint32_t np = 1;
      while (np < cnt) np <<= 1;
      const uint32_t* lst = sorted + hoff[slot];
      for (uint32_t k = t; k < np; k += blockDim.x) keys[k] = k < cnt ? lst[k] : 0xffffffffu;
      __syncthreads();
      for (uint32_t q = 2; q <= np; q <<= 1)
        for (uint32_t j = q >> 1; j > 0; j >>= 1) {
          for (uint32_t i = t; i < np; i += blockDim.x) {
            const uint32_t l = i ^ j;
            if (l > i) {
              const uint32_t a = keys[i], b = keys[l];
              if (((i & q) == 0) ? (a > b) : (a < b)) {
                keys[i] = b;
                keys[l] = a;
              }
            }
          }
          __syncthreads();
        }
      for (uint32_t c0 = 0; c0 < cnt; c0 += 1024) {
        const uint32_t m = min(1024u, cnt - c0);
        if (t < m) {
          const float* p = fp->pts + 3 * static_cast<uint64_t>(keys[c0 + t]);
          w[t] = pose_apply(fp->R, fp->t, static_cast<double>(p[0]), static_cast<double>(p[1]),
                            static_cast<double>(p[2]));
        }
        __syncthreads();
        if (t == 0)
          for (uint32_t a = 0; a < m; ++a) {
            sx += w[a].x;
            sy += w[a].y;
            sz += w[a].z;
          }
        __syncthreads();
      }
    } else {
      // stream the frame in index order; keep the points of this slot
      const uint64_t n = fp->n;
      if (t == 0) run_base = 0;
      __syncthreads();
      for (uint64_t i0 = 0; i0 < n; i0 += 1024) {
        const uint64_t i = i0 + t;
        const bool mine = i < n && pslot[i] == slot;
        const unsigned bal = __ballot_sync(0xffffffffu, mine);
        if ((t & 31) == 0) wcount[t >> 5] = __popc(bal);
        __syncthreads();
        uint32_t before = run_base;
        for (uint32_t q = 0; q < (t >> 5); ++q) before += wcount[q];
        if (mine) {
          const float* p = fp->pts + 3 * i;
          w[before - run_base + __popc(bal & lanemask_lt())] =
              pose_apply(fp->R, fp->t, static_cast<double>(p[0]), static_cast<double>(p[1]),
                         static_cast<double>(p[2]));
        }
        __syncthreads();
        if (t == 0) {
          uint32_t m = 0;
          for (uint32_t q = 0; q < 32; ++q) m += wcount[q];
          for (uint32_t a = 0; a < m; ++a) {
            sx += w[a].x;
            sy += w[a].y;
            sz += w[a].z;
          }
          run_base += m;
        }
        __syncthreads();
      }
    }
    if (t == 0) {
      c->sx = sx;
      c->sy = sy;
      c->sz = sz;
      c->count = count + cnt;
      c->status = 1;
      if (count == 0) {
        occ_set(g, fp->occ_pre, fp->off_pre, fp->zb_pre, x, y, z);
        atomicAdd(&ctr->newly, 1ull);
      }
      hkey[slot] = kEmptyKey;
      hcnt[slot] = 0;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// clear_rays (voxel_grid.cpp:182-215) with walk_segment (:122-178).
// One thread per ray; the DDA is the reference's arithmetic verbatim. Every
// interior cell is set in the clear bitmap (test-before-set keeps the hot
// cells next to the sensor from serialising on L2 atomics); k_clear_apply
// then counts unique cells, frees occupied ones and zeroes the mask.
// ---------------------------------------------------------------------------
// One thread per ray (voxel_grid.cpp:122-178, the reference's DDA arithmetic
// verbatim); every traversed interior cell is marked in a clear mask with a
// fire-and-forget RED.OR, and k_clear_apply then counts unique cells, frees
// the occupied ones and zeroes the mask. Marking is the bottleneck (L2
// atomic throughput: without marks the C4 walk takes 0.4 ms instead of 2.0),
// so it follows the rays' coherence (k_dda_plan's per-frame decision):
//  * coherent rays (depth images: adjacent lanes walk nearly the same cells
//    near the sensor): row-layout mask, a lane in the same cell as its left
//    neighbour this iteration skips the RED;
//  * incoherent rays (LiDAR patterns): rays walked longest-first (lane
//    balance), 4x4x4-brick mask (64-bit words), a ray accumulates the bits of the brick it
//    is in and issues one RED when it leaves it (C4: 2.4 -> 1.4 ms).
//
// Work binning for unbalanced ray sets. k_dda_keys estimates each ray's DDA
// length as the L1 cell distance sensor -> end point (original order), bins
// it (32-step bins), and measures how balanced 32-ray groups are; k_dda_plan
// turns binning on only when groups would waste > 25 % of their lanes, and
// k_dda_scatter then lists the rays longest-bin first. The marks are ORs and
// every count is taken afterwards from the bitmap, so the walk order does
// not change any result.
__global__ void k_dda_keys(GridDesc g, const FrameParams* __restrict__ fp, DdaBins* db, uint8_t* bin_of) {
  VP_GRID_WAIT();
  // a coherent stream is re-evaluated every 8th frame only (the decision
  // changes the walk order, never a result)
  if (!db->use && (db->frame & 7u)) return;
  __shared__ uint32_t hist[kDdaBins];
  for (int b = threadIdx.x; b < kDdaBins; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  const uint64_t n = fp->n;
  const double res = g.res;
  unsigned long long sum = 0, wmax = 0;
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u); i0 < n;
       i0 += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = i0 + lane_id();
    uint32_t st = 0;
    if (i < n) {
      const float* pp = fp->pts + 3 * i;
      const d3 bw = pose_apply(fp->R, fp->t, static_cast<double>(pp[0]), static_cast<double>(pp[1]),
                               static_cast<double>(pp[2]));
      if (finite3(bw)) {
        const double e0 = fabs(bw.x - fp->t[0]) / res, e1 = fabs(bw.y - fp->t[1]) / res,
                     e2 = fabs(bw.z - fp->t[2]) / res;
        const double l1 = e0 + e1 + e2 + 3.0;
        st = l1 < 4.0e9 ? static_cast<uint32_t>(l1) : 0xffffffffu;
      }
      const uint32_t b = min(static_cast<uint32_t>(kDdaBins - 1), st >> 5);
      bin_of[i] = static_cast<uint8_t>(b);
      atomicAdd(&hist[b], 1u);
    }
    const uint32_t mx = __reduce_max_sync(0xffffffffu, st);
    if (lane_id() == 0) wmax += 32ull * mx;
    sum += st;
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kDdaBins; b += blockDim.x)
    if (hist[b]) atomicAdd(&db->count[b], hist[b]);
  warp_add_u64(&db->steps, sum);
  warp_add_u64(&db->warp_max, wmax);
}

// One warp: decide, and lay the bins out longest first; resets the counts.
__global__ void k_dda_plan(DdaBins* db, int force, int long_steps) {
  VP_GRID_WAIT();
  const unsigned lane = lane_id();
  const bool measured = db->warp_max != 0;  // k_dda_keys ran this frame
  int use = measured ? (db->steps * 4 < db->warp_max * 3 ? 1 : 0) : db->use;  // lane efficiency < 75 %
  uint32_t run = 0;
  for (int b0 = kDdaBins - 32; b0 >= 0; b0 -= 32) {  // descending bins
    const int b = b0 + 31 - static_cast<int>(lane);
    const uint32_t c = db->count[b];
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
      if (static_cast<int>(lane) >= o) incl += t;
    }
    db->cursor[b] = run + incl - c;
    run += __shfl_sync(0xffffffffu, incl, 31);
    db->count[b] = 0;
  }
  __syncwarp();
  // long rays (mean estimated steps per ray above long_steps): few cells are
  // shared with the neighbouring lane, and one RED per brick beats one per cell
  if (measured && long_steps > 0 && run && db->steps > static_cast<unsigned long long>(long_steps) * run) use = 1;
  if (force >= 0) use = force;
  if (lane == 0) {
    db->use = use;
    db->steps = 0;
    db->warp_max = 0;
    ++db->frame;
  }
}

__global__ void k_dda_scatter(const FrameParams* __restrict__ fp, DdaBins* db, const uint8_t* __restrict__ bin_of,
                              uint32_t* perm) {
  VP_GRID_WAIT();
  if (!db->use) return;
  const uint64_t n = fp->n;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int b = bin_of[i];
    const unsigned peers = __match_any_sync(__activemask(), b);
    const int leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (static_cast<int>(lane_id()) == leader) base = atomicAdd(&db->cursor[b], static_cast<uint32_t>(__popc(peers)));
    base = __shfl_sync(peers, base, leader);
    perm[base + __popc(peers & lanemask_lt())] = static_cast<uint32_t>(i);
  }
}

// Per-step work is kept minimal: the reference loop "visit unless origin or
// end cell; argmin; step; bounds; t_max[m] += t_delta[m]" is rotated so the
// origin test runs once (the DDA is monotone per axis: once it left the first
// cell it never returns, and the first cell is the origin cell whenever the
// origin lies in the window), the end-cell test is one compare of the cell's
// mask key (word << 5 | bit, or << 6 for bricks; injective over the grid's cells), and only the
// stepped axis' t_max is advanced (one DADD). kSlab adds the owned-x-range
// logic of a spatial slab.
// Window constants of one frame's walk (voxel_grid.cpp:122-129).
struct DdaWin {
  double lo0, lo1, lo2, hi0, hi1, hi2, a0, a1, a2, res;
  int oc0, oc1, oc2;  // the sensor's cell
};
__device__ __forceinline__ DdaWin dda_window(const GridDesc& g, const FrameParams* __restrict__ fp) {
  DdaWin w;
  w.res = g.res;
  w.lo0 = fp->origin_pre[0];
  w.lo1 = fp->origin_pre[1];
  w.lo2 = fp->origin_pre[2];
  w.hi0 = w.lo0 + static_cast<double>(g.gex) * w.res;
  w.hi1 = w.lo1 + static_cast<double>(g.ey) * w.res;
  w.hi2 = w.lo2 + static_cast<double>(g.ez) * w.res;
  w.a0 = fp->t[0];
  w.a1 = fp->t[1];
  w.a2 = fp->t[2];
  w.oc0 = w2i(w.a0, w.lo0, w.res);
  w.oc1 = w2i(w.a1, w.lo1, w.res);
  w.oc2 = w2i(w.a2, w.lo2, w.res);
  return w;
}

// One ray's DDA start state: window cell, steps, t_max, t_delta, t1, end cell.
struct DdaRay {
  double t1, tm0, tm1, tm2, td0, td1, td2;
  int c0, c1, c2, s0, s1, s2, ec0, ec1, ec2;
};
// walk_segment's clip and initialisation (voxel_grid.cpp:130-168), the
// reference's arithmetic verbatim; false when the end point is not finite
// (voxel_grid.cpp:189) or the segment misses the window.
__device__ __forceinline__ bool dda_setup(const DdaWin& w, const FrameParams* __restrict__ fp, uint64_t i,
                                          const GridDesc& g, DdaRay& r) {
  const double res = w.res;
  const float* pp = fp->pts + 3 * i;
  const d3 bw = pose_apply(fp->R, fp->t, static_cast<double>(pp[0]), static_cast<double>(pp[1]),
                           static_cast<double>(pp[2]));
  if (!finite3(bw)) return false;
  const double d0 = bw.x - w.a0, d1 = bw.y - w.a1, d2 = bw.z - w.a2;
  double t0 = 0.0, t1 = 1.0;
  bool skip = false;
#define VP_CLIP(dk, ak, lok, hik)                         \
  if (!skip) {                                           \
    if (dk == 0.0) {                                     \
      if (ak < lok || ak >= hik) skip = true;            \
    } else {                                             \
      double ta = (lok - ak) / dk;                       \
      double tb = (hik - ak) / dk;                       \
      if (ta > tb) {                                     \
        const double sw = ta;                            \
        ta = tb;                                         \
        tb = sw;                                         \
      }                                                  \
      t0 = (t0 < ta) ? ta : t0;                          \
      t1 = (tb < t1) ? tb : t1;                          \
      if (t0 > t1) skip = true;                          \
    }                                                    \
  }
  VP_CLIP(d0, w.a0, w.lo0, w.hi0)
  VP_CLIP(d1, w.a1, w.lo1, w.hi1)
  VP_CLIP(d2, w.a2, w.lo2, w.hi2)
#undef VP_CLIP
  if (skip) return false;
  r.t1 = t1;
  r.ec0 = w2i(bw.x, w.lo0, res);
  r.ec1 = w2i(bw.y, w.lo1, res);
  r.ec2 = w2i(bw.z, w.lo2, res);
  const double e0 = w.a0 + t0 * d0, e1 = w.a1 + t0 * d1, e2 = w.a2 + t0 * d2;
  int c0 = w2i(e0, w.lo0, res), c1 = w2i(e1, w.lo1, res), c2 = w2i(e2, w.lo2, res);
  r.c0 = c0 < 0 ? 0 : (g.gex - 1 < c0 ? g.gex - 1 : c0);  // std::clamp
  r.c1 = c1 < 0 ? 0 : (g.ey - 1 < c1 ? g.ey - 1 : c1);
  r.c2 = c2 < 0 ? 0 : (g.ez - 1 < c2 ? g.ez - 1 : c2);
  r.s0 = r.s1 = r.s2 = 0;
  r.tm0 = r.tm1 = r.tm2 = CUDART_INF;
  r.td0 = r.td1 = r.td2 = CUDART_INF;
#define VP_INIT(dk, ck, lok, ek, sk, tmk, tdk)                                        \
  if (dk > 0.0) {                                                                     \
    sk = 1;                                                                           \
    tmk = t0 + (lok + static_cast<double>(ck + 1) * res - ek) / dk;                   \
    tdk = res / dk;                                                                   \
  } else if (dk < 0.0) {                                                              \
    sk = -1;                                                                          \
    tmk = t0 + (lok + static_cast<double>(ck) * res - ek) / dk;                       \
    tdk = res / -dk;                                                                  \
  }
  VP_INIT(d0, r.c0, w.lo0, e0, r.s0, r.tm0, r.td0)
  VP_INIT(d1, r.c1, w.lo1, e1, r.s1, r.tm1, r.td1)
  VP_INIT(d2, r.c2, w.lo2, e2, r.s2, r.tm2, r.td2)
#undef VP_INIT
  return true;
}

// 64-bit OR into shared memory as two native 32-bit ATOMS.OR (a 64-bit
// atomicOr on shared memory compiles to a CAS spin loop, which the rays
// near the sensor contend on)
__device__ __forceinline__ void smem_or64(unsigned long long* p, unsigned long long v) {
  uint32_t* h = reinterpret_cast<uint32_t*>(p);
  const uint32_t lo = static_cast<uint32_t>(v), hi = static_cast<uint32_t>(v >> 32);
  if (lo) atomicOr(h, lo);
  if (hi) atomicOr(h + 1, hi);
}

template <bool kSlab>
__device__ __forceinline__ void clear_walk_body(const GridDesc& g, const FrameParams* __restrict__ fp,
                                                const uint32_t* __restrict__ perm, const DdaBins* db) {
  const uint64_t n = fp->n;
  const DdaWin wn = dda_window(g, fp);
  const int oc0 = wn.oc0, oc1 = wn.oc1, oc2 = wn.oc2;
  const int max_steps = g.gex + g.ey + g.ez + 4;
  const int own0 = g.xoff + g.own_lo, own1 = g.xoff + g.own_hi;  // window x owned here
  uint32_t* __restrict__ clr = g.clr;
  unsigned long long* __restrict__ clrb = g.clrb;
  const uint32_t xstride = static_cast<uint32_t>(g.ey) * static_cast<uint32_t>(g.W);
  const uint32_t ystride = static_cast<uint32_t>(g.W);
  const unsigned lane = lane_id();
  const unsigned left = lane ? (1u << (lane - 1)) : 0u;  // the lane to my left
  // k_dda_plan's decision: incoherent, unbalanced rays (LiDAR patterns) are
  // walked in length order and accumulate their marks per brick; coherent
  // rays (depth images) dedup per cell against the neighbouring lane
  const bool accumulate = db->use != 0;
  const bool binned = accumulate;
  // the kNear^3 bricks around the sensor are crossed by most rays: their
  // marks are gathered in shared memory and flushed once per block
  constexpr int kNearR = 1, kNear = 2 * kNearR + 1, kNear3 = kNear * kNear * kNear;
  __shared__ unsigned long long near_m[kNear3];
  for (int k = threadIdx.x; k < kNear3; k += blockDim.x) near_m[k] = 0;
  __syncthreads();
  const int sbx = (oc0 - g.xoff) >> 2, sby = oc1 >> 2, sbz = oc2 >> 2;
  for (uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = binned ? perm[r] : r;
    DdaRay ry;
    if (!dda_setup(wn, fp, i, g, ry)) continue;
    int c0 = ry.c0, c1 = ry.c1, c2 = ry.c2;
    const int s0 = ry.s0, s1 = ry.s1, s2 = ry.s2, ec0 = ry.ec0, ec1 = ry.ec1, ec2 = ry.ec2;
    double tm0 = ry.tm0, tm1 = ry.tm1, tm2 = ry.tm2;
    const double td0 = ry.td0, td1 = ry.td1, td2 = ry.td2, t1 = ry.t1;
    // brick key of a cell of this grid: word << 5 | bit (meaningful while c0
    // is stored here; the end cell's key only when it is owned here)
    const bool e_here = ec0 >= own0 && ec0 < own1 && static_cast<unsigned>(ec1) < static_cast<unsigned>(g.ey) &&
                        static_cast<unsigned>(ec2) < static_cast<unsigned>(g.ez);
    const uint32_t key_e =
        e_here ? ((brick_word(g, ec0 - g.xoff, ec1, ec2) << 6) | brick_bit(ec0 - g.xoff, ec1, ec2)) : 0xffffffffu;
    bool mark = !(c0 == oc0 && c1 == oc1 && c2 == oc2);  // origin cell: first cell only
    uint32_t aw = 0xffffffffu;  // the brick the ray is in, its marks (flushed when it leaves)
    unsigned long long ab = 0;
    int anear = -1;  // its index among the sensor's near bricks, or -1
    // row-layout word index of the current cell (coherent path, incremental)
    uint32_t row = static_cast<uint32_t>(c0 - g.xoff) * xstride + static_cast<uint32_t>(c1) * ystride;
    const int dx_row = s0 * static_cast<int>(xstride), dy_row = s1 * static_cast<int>(ystride);
    const uint32_t key_er =
        e_here ? (((static_cast<uint32_t>(ec0 - g.xoff) * xstride + static_cast<uint32_t>(ec1) * ystride +
                    (static_cast<uint32_t>(ec2) >> 5)) << 5) | (static_cast<uint32_t>(ec2) & 31u))
               : 0xffffffffu;
    for (int s = 0; s < max_steps; ++s) {
      if (s > 0) {
        // m = argmin t_max, ties to the lower axis (voxel_grid.cpp:170-172)
        const bool m1 = tm1 < tm0;
        const double tm01 = m1 ? tm1 : tm0;
        const bool m2 = tm2 < tm01;
        const double tm = m2 ? tm2 : tm01;
        if (tm >= t1) break;
        // the stepped axis as an integer (the FP64 predicates are not re-evaluated)
        const int m = m2 ? 2 : (m1 ? 1 : 0);
        c0 += m == 0 ? s0 : 0;
        c1 += m == 1 ? s1 : 0;
        c2 += m == 2 ? s2 : 0;
        if (static_cast<unsigned>(c0) >= static_cast<unsigned>(g.gex) ||
            static_cast<unsigned>(c1) >= static_cast<unsigned>(g.ey) ||
            static_cast<unsigned>(c2) >= static_cast<unsigned>(g.ez))
          break;
        int drow = m == 0 ? dx_row : 0;
        drow = m == 1 ? dy_row : drow;
        row += drow;
        double tdm = m == 0 ? td0 : td1;
        tdm = m == 2 ? td2 : tdm;
        const double tn = tm + tdm;  // t_max[m] += t_delta[m]
        tm0 = m == 0 ? tn : tm0;
        tm1 = m == 1 ? tn : tm1;
        tm2 = m == 2 ? tn : tm2;
        mark = true;
      }
      bool here = true;
      if (kSlab) {
        // a slab never sees the ray again once it left the owned x-range in
        // its stepping direction (the DDA is monotone per axis)
        if ((s0 > 0 && c0 >= own1) || (s0 < 0 && c0 < own0) || (s0 == 0 && (c0 < own0 || c0 >= own1))) break;
        here = c0 >= own0 && c0 < own1;  // not yet entered: skip
      }
      if (!mark || !here) continue;
      if (accumulate) {  // incoherent rays: one RED per brick the ray crosses
        const int lx = c0 - g.xoff;
        const uint32_t w = brick_word(g, lx, c1, c2);
        const uint32_t bit = brick_bit(lx, c1, c2);
        if (((w << 6) | bit) == key_e) continue;
        if (w != aw) {
          if (ab) {
            if (anear >= 0) smem_or64(&near_m[anear], ab); else atomicOr(clrb + aw, ab);
          }
          aw = w;
          ab = 0;
          const int dbx = (lx >> 2) - sbx, dby = (c1 >> 2) - sby, dbz = (c2 >> 2) - sbz;
          anear = (dbx >= -kNearR && dbx <= kNearR && dby >= -kNearR && dby <= kNearR && dbz >= -kNearR &&
                   dbz <= kNearR)
                      ? ((dbx + kNearR) * kNear + (dby + kNearR)) * kNear + (dbz + kNearR)
                      : -1;
        }
        ab |= 1ull << bit;
      } else {  // coherent rays: lanes in the same cell as their left neighbour skip it
        const uint32_t w = row + (static_cast<uint32_t>(c2) >> 5);
        const uint32_t key = (w << 5) | (static_cast<uint32_t>(c2) & 31u);
        if (key == key_er) continue;
        const unsigned act = __activemask();
        const uint32_t prev = __shfl_up_sync(act, key, 1);
        const bool dup = (act & left) && prev == key;
        if (!dup) atomicOr(clr + w, 1u << (c2 & 31));
      }
    }
    if (ab) {
      if (anear >= 0) smem_or64(&near_m[anear], ab); else atomicOr(clrb + aw, ab);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; accumulate && k < kNear3; k += blockDim.x)
    if (near_m[k]) {
      const int bx = sbx + k / (kNear * kNear) - kNearR, by = sby + (k / kNear) % kNear - kNearR,
                bz = sbz + k % kNear - kNearR;
      atomicOr(clrb + (static_cast<uint32_t>(bx) * g.bny + by) * g.bnz + bz, near_m[k]);
    }
}

// Coherent rays on a plain grid (the depth-image case): the warp walks its
// 32 rays in lockstep -- one loop trip per DDA step of the longest ray, lanes
// whose ray ended idle -- so the left-neighbour dedup is a full-warp shuffle,
// and the step is branch-free: argmin, one select per axis, one DADD, the
// cell's row-mask key advanced incrementally (key = word << 5 | bit =
// row * 32 + z). Same cells, same order per ray as clear_walk_body.
// kSlab: as in clear_walk_bricks below (window-coordinate walk, marks only in
// the owned x-range, a lane ends once its ray left it); the row key of a cell
// outside the stored range is meaningless (uint32 wrap) and never used.
constexpr uint32_t kNoMark = 0xffffffffu;
#ifndef VP_WALK_STEPS
#define VP_WALK_STEPS 3
#endif
template <bool kSlab>
__device__ __forceinline__ void clear_walk_coherent(const GridDesc& g, const FrameParams* __restrict__ fp) {
  const uint64_t n = fp->n;
  const DdaWin wn = dda_window(g, fp);
  const int xoff = kSlab ? g.xoff : 0;
  const int own0 = kSlab ? g.xoff + g.own_lo : 0, own1 = kSlab ? g.xoff + g.own_hi : g.gex;
  uint32_t* __restrict__ clr = g.clr;
  const uint32_t xs = static_cast<uint32_t>(g.ey) * static_cast<uint32_t>(g.W) * 32u;
  const uint32_t ys = static_cast<uint32_t>(g.W) * 32u;
  const unsigned lane = lane_id();
  const uint32_t ex0 = static_cast<uint32_t>(g.gex), ex1 = static_cast<uint32_t>(g.ey),
                 ex2 = static_cast<uint32_t>(g.ez);
  // warp-uniform ray loop (every lane runs the same trips)
  for (uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u); r0 < n;
       r0 += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    DdaRay ry;
    bool live = r0 + lane < n && dda_setup(wn, fp, r0 + lane, g, ry);
    uint32_t key = kNoMark, key_e = kNoMark, krow = 0;
    int c0 = 0, c1 = 0, c2 = 0, s0 = 0, s1 = 0, s2 = 0, dxr = 0, dyr = 0;
    double tm0 = 0.0, tm1 = 0.0, tm2 = 0.0, td0 = 0.0, td1 = 0.0, td2 = 0.0, t1 = 0.0;
    if (live) {
      c0 = ry.c0, c1 = ry.c1, c2 = ry.c2, s0 = ry.s0, s1 = ry.s1, s2 = ry.s2;
      tm0 = ry.tm0, tm1 = ry.tm1, tm2 = ry.tm2, td0 = ry.td0, td1 = ry.td1, td2 = ry.td2, t1 = ry.t1;
      krow = static_cast<uint32_t>(c0 - xoff) * xs + static_cast<uint32_t>(c1) * ys;
      dxr = s0 * static_cast<int>(xs);
      dyr = s1 * static_cast<int>(ys);
      if (ry.ec0 >= own0 && ry.ec0 < own1 && static_cast<unsigned>(ry.ec0) < ex0 &&
          static_cast<unsigned>(ry.ec1) < ex1 && static_cast<unsigned>(ry.ec2) < ex2)
        key_e = static_cast<uint32_t>(ry.ec0 - xoff) * xs + static_cast<uint32_t>(ry.ec1) * ys +
                static_cast<uint32_t>(ry.ec2);
      // the first cell is visited unless it is the origin cell
      if (!(c0 == wn.oc0 && c1 == wn.oc1 && c2 == wn.oc2)) key = krow + static_cast<uint32_t>(c2);
      if (key == key_e) key = kNoMark;
      if (kSlab) {
        // a ray that never reaches the owned range; a first cell outside it
        if ((s0 > 0 && c0 >= own1) || (s0 < 0 && c0 < own0) || (s0 == 0 && (c0 < own0 || c0 >= own1)))
          live = false, key = kNoMark;
        if (c0 < own0 || c0 >= own1) key = kNoMark;
      }
    }
    // (a ray never exceeds max_steps here: each step moves one axis
    // monotonically, so it leaves the window after gex + ey + ez steps)
    uint32_t live_i = live ? 1u : 0u;
    // visit: a lane in the same cell as its left neighbour skips the RED
    auto visit = [&] {
      const uint32_t prev = __shfl_up_sync(0xffffffffu, key, 1);
      if (key != kNoMark && (key != prev || lane == 0)) atomicOr(clr + (key >> 5), 1u << (key & 31u));
    };
    auto step = [&] {
      // one DDA step, branch-free (an ended lane steps too; its state is
      // garbage from then on and only `live` / `key` are read), written in
      // PTX so the stepped axis is advanced by predicated adds instead of
      // selects (the walk is ALU-pipe bound):
      //   m = argmin t_max, ties to the lower axis (voxel_grid.cpp:170-172):
      //   m1 = tm1 < tm0, m2 = tm2 < min(tm0, tm1), axis 0 iff !(m1 | m2)
      //   stop when min t_max >= t1, or the stepped cell leaves the window
      //   t_max[m] += t_delta[m]; row key += the stepped axis' stride
      asm("{\n\t"
          ".reg .pred m1, m2, a, x1, d, ok, lv;\n\t"
          ".reg .f64 t01;\n\t"
          ".reg .u32 k;\n\t"
          "setp.ne.u32 lv, %5, 0;\n\t"
          "setp.lt.f64 m1, %7, %6;\n\t"
          "selp.f64 t01, %7, %6, m1;\n\t"
          "setp.lt.f64 m2, %8, t01;\n\t"
          "setp.ge.f64 d, t01, %14;\n\t"
          "setp.ge.and.f64 d, %8, %14, d;\n\t"
          "or.pred a, m1, m2;\n\t"
          "and.pred x1, m1, !m2;\n\t"
          "@!a add.s32 %0, %0, %9;\n\t"
          "@!a add.s32 %3, %3, %12;\n\t"
          "@!a add.rn.f64 %6, %6, %15;\n\t"
          "@x1 add.s32 %1, %1, %10;\n\t"
          "@x1 add.s32 %3, %3, %13;\n\t"
          "@x1 add.rn.f64 %7, %7, %16;\n\t"
          "@m2 add.s32 %2, %2, %11;\n\t"
          "@m2 add.rn.f64 %8, %8, %17;\n\t"
          "setp.lt.u32 ok, %0, %18;\n\t"
          "setp.lt.and.u32 ok, %1, %19, ok;\n\t"
          "setp.lt.and.u32 ok, %2, %20, ok;\n\t"
          "and.pred ok, ok, !d;\n\t"
          "and.pred ok, ok, lv;\n\t"
          "add.u32 k, %3, %2;\n\t"
          "setp.ne.and.u32 lv, k, %21, ok;\n\t"
          "selp.u32 %4, k, 0xffffffff, lv;\n\t"
          "selp.u32 %5, 1, 0, ok;\n\t"
          "}"
          : "+r"(c0), "+r"(c1), "+r"(c2), "+r"(krow), "=r"(key), "+r"(live_i), "+d"(tm0), "+d"(tm1), "+d"(tm2)
          : "r"(s0), "r"(s1), "r"(s2), "r"(dxr), "r"(dyr), "d"(t1), "d"(td0), "d"(td1), "d"(td2), "r"(ex0),
            "r"(ex1), "r"(ex2), "r"(key_e));
      live = live_i != 0;
      if (kSlab) {
        // left the owned range in its x direction: done; not yet in it: no mark
        if ((s0 > 0 && c0 >= own1) || (s0 < 0 && c0 < own0)) live = false, key = kNoMark;
        if (c0 < own0 || c0 >= own1) key = kNoMark;
      }
    };
    // VP_WALK_STEPS steps per vote (a lane whose ray ended keeps key =
    // kNoMark, so the extra visits and steps of a warp that just finished
    // mark nothing): C2 walk 82.7 -> 79.5 us at 2, 76.0 at 3 (77.2 at 4)
    for (;;) {
      visit();
      if (!__any_sync(0xffffffffu, live)) break;
      step();
#pragma unroll
      for (int u = 1; u < VP_WALK_STEPS; ++u) {
        visit();
        step();
      }
    }
  }
}

// Incoherent rays (LiDAR patterns; rays listed longest first by
// k_dda_scatter): a branch-free step per lane (no cross-lane work) and
// clear_walk_body's brick accumulation -- a ray ORs the bits of the 4x4x4
// brick it is in and issues one RED when it leaves it, into shared memory
// for the 3x3x3 bricks around the sensor. kSlab: the grid stores window x
// [xoff, xoff + ex) and owns [xoff + own_lo, xoff + own_hi); rays are walked
// in window coordinates from their start (a slab clip would drift in the
// last bit), marked only inside the owned range, and dropped once they left
// it in their x direction (the DDA is monotone per axis).
template <bool kSlab>
__device__ __forceinline__ void clear_walk_bricks(const GridDesc& g, const FrameParams* __restrict__ fp,
                                                  const uint32_t* __restrict__ perm) {
  const uint64_t n = fp->n;
  const DdaWin wn = dda_window(g, fp);
  unsigned long long* __restrict__ clrb = g.clrb;
  const uint32_t ex0 = static_cast<uint32_t>(g.gex), ex1 = static_cast<uint32_t>(g.ey),
                 ex2 = static_cast<uint32_t>(g.ez);
  const int xoff = kSlab ? g.xoff : 0;
  const int own0 = kSlab ? g.xoff + g.own_lo : 0, own1 = kSlab ? g.xoff + g.own_hi : g.gex;
  constexpr int kNearR = 1, kNear = 2 * kNearR + 1, kNear3 = kNear * kNear * kNear;
  __shared__ unsigned long long near_m[kNear3];
  for (int k = threadIdx.x; k < kNear3; k += blockDim.x) near_m[k] = 0;
  __syncthreads();
  const int sbx = (wn.oc0 - xoff) >> 2, sby = wn.oc1 >> 2, sbz = wn.oc2 >> 2;
  for (uint64_t r = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    DdaRay ry;
    if (!dda_setup(wn, fp, perm[r], g, ry)) continue;
    int c0 = ry.c0, c1 = ry.c1, c2 = ry.c2;
    const int s0 = ry.s0, s1 = ry.s1, s2 = ry.s2;
    double tm0 = ry.tm0, tm1 = ry.tm1, tm2 = ry.tm2;
    const double td0 = ry.td0, td1 = ry.td1, td2 = ry.td2, t1 = ry.t1;
    // the end cell's key, when it is stored (and owned) here
    const uint32_t key_e =
        (ry.ec0 >= own0 && ry.ec0 < own1 && static_cast<unsigned>(ry.ec1) < ex1 &&
         static_cast<unsigned>(ry.ec2) < ex2)
            ? ((brick_word(g, ry.ec0 - xoff, ry.ec1, ry.ec2) << 6) | brick_bit(ry.ec0 - xoff, ry.ec1, ry.ec2))
            : kNoMark;
    uint32_t aw = kNoMark;  // the brick the ray is in, its marks (flushed when it leaves)
    unsigned long long ab = 0;
    int anear = -1;  // its index among the sensor's near bricks, or -1
    auto visit = [&] {
      if (kSlab && (c0 < own0 || c0 >= own1)) return;  // not stored here
      const int lx = c0 - xoff;
      const uint32_t w = brick_word(g, lx, c1, c2);
      const uint32_t bit = brick_bit(lx, c1, c2);
      if (((w << 6) | bit) == key_e) return;
      if (w != aw) {
        if (ab) {
          if (anear >= 0) smem_or64(&near_m[anear], ab); else atomicOr(clrb + aw, ab);
        }
        aw = w;
        ab = 0;
        const int dbx = (lx >> 2) - sbx, dby = (c1 >> 2) - sby, dbz = (c2 >> 2) - sbz;
        anear = (dbx >= -kNearR && dbx <= kNearR && dby >= -kNearR && dby <= kNearR && dbz >= -kNearR &&
                 dbz <= kNearR)
                    ? ((dbx + kNearR) * kNear + (dby + kNearR)) * kNear + (dbz + kNearR)
                    : -1;
      }
      ab |= 1ull << bit;
    };
    // a slab skips rays that never reach its owned x-range
    if (kSlab && ((s0 > 0 && c0 >= own1) || (s0 < 0 && c0 < own0) || (s0 == 0 && (c0 < own0 || c0 >= own1))))
      continue;
    if (!(c0 == wn.oc0 && c1 == wn.oc1 && c2 == wn.oc2)) visit();  // origin cell: first cell only
    for (;;) {
      // one DDA step (as in clear_walk_coherent, predicated adds in PTX):
      // m = argmin t_max, ties to the lower axis (voxel_grid.cpp:170-172);
      // stop when min t_max >= t1 or the stepped cell leaves the window
      uint32_t ok;
      asm("{\n\t"
          ".reg .pred m1, m2, a, x1, d, p;\n\t"
          ".reg .f64 t01;\n\t"
          "setp.lt.f64 m1, %5, %4;\n\t"
          "selp.f64 t01, %5, %4, m1;\n\t"
          "setp.lt.f64 m2, %6, t01;\n\t"
          "setp.ge.f64 d, t01, %10;\n\t"
          "setp.ge.and.f64 d, %6, %10, d;\n\t"
          "or.pred a, m1, m2;\n\t"
          "and.pred x1, m1, !m2;\n\t"
          "@!a add.s32 %0, %0, %7;\n\t"
          "@!a add.rn.f64 %4, %4, %11;\n\t"
          "@x1 add.s32 %1, %1, %8;\n\t"
          "@x1 add.rn.f64 %5, %5, %12;\n\t"
          "@m2 add.s32 %2, %2, %9;\n\t"
          "@m2 add.rn.f64 %6, %6, %13;\n\t"
          "setp.lt.u32 p, %0, %14;\n\t"
          "setp.lt.and.u32 p, %1, %15, p;\n\t"
          "setp.lt.and.u32 p, %2, %16, p;\n\t"
          "and.pred p, p, !d;\n\t"
          "selp.u32 %3, 1, 0, p;\n\t"
          "}"
          : "+r"(c0), "+r"(c1), "+r"(c2), "=r"(ok), "+d"(tm0), "+d"(tm1), "+d"(tm2)
          : "r"(s0), "r"(s1), "r"(s2), "d"(t1), "d"(td0), "d"(td1), "d"(td2), "r"(ex0), "r"(ex1), "r"(ex2));
      if (!ok) break;
      // a slab never sees the ray again once it left the owned x-range in
      // its stepping direction
      if (kSlab && ((s0 > 0 && c0 >= own1) || (s0 < 0 && c0 < own0))) break;
      visit();
    }
    if (ab) {
      if (anear >= 0) smem_or64(&near_m[anear], ab); else atomicOr(clrb + aw, ab);
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k < kNear3; k += blockDim.x)
    if (near_m[k]) {
      const int bx = sbx + k / (kNear * kNear) - kNearR, by = sby + (k / kNear) % kNear - kNearR,
                bz = sbz + k % kNear - kNearR;
      atomicOr(clrb + (static_cast<uint32_t>(bx) * g.bny + by) * g.bnz + bz, near_m[k]);
    }
}

#ifndef VP_DDA_MINB
#define VP_DDA_MINB 4
#endif
__global__ void __launch_bounds__(256, VP_DDA_MINB) k_clear_walk(GridDesc g, const FrameParams* __restrict__ fp,
                                                                  const uint32_t* perm, const DdaBins* db,
                                                                  int generic) {
  VP_GRID_WAIT();
  if (!generic) {
    if (db->use) clear_walk_bricks<false>(g, fp, perm); else clear_walk_coherent<false>(g, fp);
    return;
  }
  clear_walk_body<false>(g, fp, perm, db);
}
__global__ void __launch_bounds__(256, 4) k_clear_walk_slab(GridDesc g, const FrameParams* __restrict__ fp,
                                                            const uint32_t* perm, const DdaBins* db) {
  VP_GRID_WAIT();
  if (db->use) clear_walk_bricks<true>(g, fp, perm); else clear_walk_coherent<true>(g, fp);
}

__device__ __forceinline__ void zero_cell(Cell* c) {
  c->sx = 0.0;
  c->sy = 0.0;
  c->sz = 0.0;
  c->count = 0;
  c->status = 0;
}

// The cells the frame's rays can mark: k_integrate_hash's box (use_box), or
// the whole grid (clear_rays without integrate_frame). Every mark lies in the
// box, and the apply pass zeroes every mark it visits, so the masks stay zero
// outside it.
__device__ __forceinline__ void sweep_box(const GridDesc& g, const Counters* ctr, int use_box, int* lo, int* hi) {
  if (use_box) {
    for (int k = 0; k < 3; ++k) lo[k] = ctr->box_lo[k], hi[k] = ctr->box_hi[k];
  } else {
    lo[0] = lo[1] = lo[2] = 0;
    hi[0] = g.ex - 1, hi[1] = g.ey - 1, hi[2] = g.ez - 1;
  }
}

// Row-layout clear mask (coherent rays): one thread per mask word of the box.
// The occupancy of a mask word's 32 cells is 32 ring bits (one or two ring
// words); freed bits are cleared with atomicAnd (neighbouring mask words share
// ring words).
__device__ __forceinline__ void clear_apply_rows(const GridDesc& g, const FrameParams* __restrict__ fp,
                                                 Counters* ctr, int use_box) {
  uint32_t* occ = fp->occ_pre;
  unsigned long long cl = 0, fr = 0;
  int lo[3], hi[3];
  sweep_box(g, ctr, use_box, lo, hi);
  if (hi[0] >= lo[0]) {
    const int wz0 = lo[2] >> 5;
    const uint32_t nwz = static_cast<uint32_t>((hi[2] >> 5) - wz0 + 1);
    const uint32_t ny = static_cast<uint32_t>(hi[1] - lo[1] + 1);
    const uint32_t total = static_cast<uint32_t>(hi[0] - lo[0] + 1) * ny * nwz;  // < 2^27 mask words
    // four mask words per thread and trip, loaded before any is processed
    // (the sweep is latency-bound: most words are zero)
    constexpr int kPer = 4;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t q0 = blockIdx.x * blockDim.x + threadIdx.x; q0 < total; q0 += kPer * stride) {
      uint64_t wq[kPer];
      uint32_t cq[kPer];
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const uint32_t q = q0 + k * stride;
        wq[k] = ~0ull;
        cq[k] = 0u;
        if (q < total) {
          const uint32_t r = q / nwz;
          const int wz = wz0 + static_cast<int>(q - r * nwz);
          const uint32_t rx = r / ny;
          const int y = lo[1] + static_cast<int>(r - rx * ny), x = lo[0] + static_cast<int>(rx);
          wq[k] = (static_cast<uint64_t>(x) * g.ey + y) * g.W + wz;
          cq[k] = g.clr[wq[k]];
        }
      }
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
      const uint32_t c = cq[k];
      if (!c) continue;
      const uint64_t w = wq[k];
      g.clr[w] = 0;
      const uint32_t wrow = fdiv(static_cast<uint32_t>(w), g.fW);
      const int wz = static_cast<int>(static_cast<uint32_t>(w) - wrow * static_cast<uint32_t>(g.W));
      const uint32_t wx = fdiv(wrow, g.fey);
      const int y = static_cast<int>(wrow - wx * static_cast<uint32_t>(g.ey)), x = static_cast<int>(wx);
      cl += __popc(c);
      const uint64_t ri = ring_row_index(g, fp->off_pre, x, y);
      uint32_t* row = occ + ri * g.W;
      const int pz = ring_z(g, fp->zb_pre, wz * 32);
      uint32_t f = ring_bits32(row, g.W, pz) & c;
      if (!f) continue;
      ring_clear32(row, g.W, pz, f);
      atomicSub(g.rowcnt + ri, static_cast<uint32_t>(__popc(f)));
      fr += __popc(f);
      while (f) {
        const int b = __ffs(f) - 1;
        f &= f - 1;
        zero_cell(g.cells + phys_index(g, fp->off_pre, x, y, wz * 32 + b));
      }
      }
    }
  }
  block_add2_u64(&ctr->cleared, cl, &ctr->freed, fr);
}

// Brick-layout clear mask (incoherent rays): one thread per brick word of the
// box: count the unique cleared cells, free the occupied ones (the occupancy
// of the brick's 16 (x, y) columns: four ring bits each), zero the mask.
__device__ __forceinline__ void clear_apply_bricks(const GridDesc& g, const FrameParams* __restrict__ fp,
                                                   Counters* ctr, int use_box) {
  uint32_t* occ = fp->occ_pre;
  unsigned long long cl = 0, fr = 0;
  int lo[3], hi[3];
  sweep_box(g, ctr, use_box, lo, hi);
  if (hi[0] >= lo[0]) {
    const int bx0 = lo[0] >> 2, by0 = lo[1] >> 2, bz0 = lo[2] >> 2;
    const uint32_t nbz = static_cast<uint32_t>((hi[2] >> 2) - bz0 + 1);
    const uint32_t nby = static_cast<uint32_t>((hi[1] >> 2) - by0 + 1);
    // (< 2^26 brick words in a grid: 32-bit index arithmetic; four mask
    // words per thread and trip loaded before any is processed -- the sweep is
    // latency-bound, most words are zero; C5's box is the whole 150 MB mask)
    const uint32_t total = static_cast<uint32_t>((hi[0] >> 2) - bx0 + 1) * nby * nbz;
    constexpr int kPer = 4;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t q0 = blockIdx.x * blockDim.x + threadIdx.x; q0 < total; q0 += kPer * stride) {
      uint64_t wq[kPer];
      unsigned long long cq[kPer];
      int bxq[kPer], byq[kPer], bzq[kPer];
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const uint32_t q = q0 + k * stride;
        cq[k] = 0ull;
        bxq[k] = byq[k] = bzq[k] = 0;
        wq[k] = 0;
        if (q < total) {
          const uint32_t r = q / nbz;
          bzq[k] = bz0 + static_cast<int>(q - r * nbz);
          const uint32_t rbx = r / nby;
          byq[k] = by0 + static_cast<int>(r - rbx * nby);
          bxq[k] = bx0 + static_cast<int>(rbx);
          wq[k] = (static_cast<uint64_t>(bxq[k]) * g.bny + byq[k]) * g.bnz + bzq[k];
          cq[k] = g.clrb[wq[k]];
        }
      }
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
      const unsigned long long c = cq[k];
      if (!c) continue;
      const int bx = bxq[k], by = byq[k], bz = bzq[k];
      g.clrb[wq[k]] = 0;
      cl += __popcll(c);
      const int z0 = bz * 4;
      unsigned long long cols = c;
      while (cols) {  // (lx, ly) columns with marks: bits 4k .. 4k+3
        const int kc = (__ffsll(cols) - 1) >> 2;
        const uint32_t cm = static_cast<uint32_t>(c >> (4 * kc)) & 15u;
        cols &= ~(15ull << (4 * kc));
        const int x = bx * 4 + (kc >> 2), y = by * 4 + (kc & 3);
        const uint64_t ri = ring_row_index(g, fp->off_pre, x, y);
        uint32_t* row = occ + ri * g.W;
        const int pz = ring_z(g, fp->zb_pre, z0);
        const uint32_t f = ring_bits32(row, g.W, pz) & cm;
        if (!f) continue;
        ring_clear32(row, g.W, pz, f);  // other bricks share these ring words
        atomicSub(g.rowcnt + ri, static_cast<uint32_t>(__popc(f)));
        fr += __popc(f);
        for (int bb = 0; bb < 4; ++bb)
          if (f & (1u << bb)) zero_cell(g.cells + phys_index(g, fp->off_pre, x, y, z0 + bb));
      }
      }
    }
  }
  block_add2_u64(&ctr->cleared, cl, &ctr->freed, fr);
}

// One launch for either mask layout (k_dda_plan's decision for this frame).
__global__ void k_clear_apply(GridDesc g, const FrameParams* __restrict__ fp, Counters* ctr, const DdaBins* db,
                              int use_box) {
  VP_GRID_WAIT();
  if (db->use) clear_apply_bricks(g, fp, ctr, use_box); else clear_apply_rows(g, fp, ctr, use_box);
}

// ---------------------------------------------------------------------------
// recenter (voxel_grid.cpp:217-252). The host computes the integer shift with
// the reference's arithmetic and advances the toroidal offsets (cells: off;
// occupancy ring: off for x and y, zb for z). On the device only the cells
// that leave the window are touched: one thread per (x, y) row of the
// pre-shift window -- a row leaving in x or y drops all its occupied cells,
// any other row the occupied cells of its leaving z range (|sz| bits, one or
// two ring words); dropped cells are zeroed and their ring bits cleared, so
// the positions that re-enter the window are empty (voxels_dropped counted).
// Rows that neither leave nor shift in z are not read at all.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void recenter_body(const GridDesc& g, const FrameParams* __restrict__ fp, Counters* ctr);

// occ_total != nullptr: the last block also finishes the frame's mapping
// (k_map_finalize's occupied bookkeeping), one launch fewer.
__device__ __forceinline__ void map_finalize_body(Counters* ctr, unsigned long long* occ_total) {
  const unsigned long long o = __ldcg(occ_total) + __ldcg(&ctr->newly) - __ldcg(&ctr->freed) - __ldcg(&ctr->dropped);
  *occ_total = o;
  ctr->occupied = o;
  ctr->touched = __ldcg(&ctr->ngroups);
}

__global__ void k_recenter(GridDesc g, const FrameParams* __restrict__ fp, Counters* ctr,
                           unsigned long long* occ_total) {
  VP_GRID_WAIT();
  if (fp->do_shift) recenter_body(g, fp, ctr);
  if (occ_total && last_block_done(&ctr->scan_done[7]) && threadIdx.x == 0) map_finalize_body(ctr, occ_total);
}

__device__ __forceinline__ void recenter_body(const GridDesc& g, const FrameParams* __restrict__ fp, Counters* ctr) {
  uint32_t* occ = fp->occ_pre;
  const int sx = fp->shift[0], sy = fp->shift[1], sz = fp->shift[2];
  const int ex = g.ex, ey = g.ey, ez = g.ez, W = g.W, Wz = g.W << 5;
  const int zb = fp->zb_pre;
  // the leaving z range of a row that stays: [zl0, zl1)
  const int zl0 = sz > 0 ? 0 : max(ez + sz, 0), zl1 = sz > 0 ? min(sz, ez) : ez;
  const bool zleave = sz != 0;
  unsigned long long dropped = 0;
  const uint32_t nrows = static_cast<uint32_t>(ex) * static_cast<uint32_t>(ey);
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += gridDim.x * blockDim.x) {
    const uint32_t xr = fdiv(r, g.fey);
    const int y = static_cast<int>(r - xr * static_cast<uint32_t>(ey)), x = static_cast<int>(xr);
    const bool row_leaves = static_cast<unsigned>(x - sx) >= static_cast<unsigned>(ex) ||
                            static_cast<unsigned>(y - sy) >= static_cast<unsigned>(ey);
    if (!row_leaves && !zleave) continue;
    const uint64_t ri = ring_row_index(g, fp->off_pre, x, y);
    if (!__ldcg(g.rowcnt + ri)) continue;  // an empty row drops nothing
    uint32_t* row = occ + ri * W;
    if (row_leaves) {
      g.rowcnt[ri] = 0u;
      for (int w = 0; w < W; ++w) {
        uint32_t v = __ldcg(row + w);
        if (!v) continue;
        row[w] = 0u;
        dropped += __popc(v);
        while (v) {
          const int b = __ffs(v) - 1;
          v &= v - 1;
          int z = 32 * w + b - zb;  // ring position -> window z
          if (z < 0) z += Wz;
          zero_cell(g.cells + phys_index(g, fp->off_pre, x, y, z));
        }
      }
      continue;
    }
    for (int z0 = zl0; z0 < zl1; z0 += 32) {
      const int len = min(32, zl1 - z0);
      const int pz = ring_z(g, zb, z0);
      uint32_t v = ring_bits32(row, W, pz) & (len >= 32 ? 0xffffffffu : ((1u << len) - 1u));
      if (!v) continue;
      ring_clear32(row, W, pz, v);
      g.rowcnt[ri] -= static_cast<uint32_t>(__popc(v));  // this thread owns the row here
      dropped += __popc(v);
      while (v) {
        const int b = __ffs(v) - 1;
        v &= v - 1;
        zero_cell(g.cells + phys_index(g, fp->off_pre, x, y, z0 + b));
      }
    }
  }
  warp_add_u64(&ctr->dropped, dropped);
}

// VoxelGrid::merge_point (voxel_grid.cpp:49-57), one point, window index.
__global__ void k_merge_point(GridDesc g, const FrameParams* __restrict__ fp, Counters* ctr, int x,
                              int y, int z, double px, double py, double pz) {
  VP_GRID_WAIT();
  Cell* c = g.cells + phys_index(g, fp->off_pre, x, y, z);
  if (c->count == 0) {
    ctr->newly += 1;
    occ_set(g, fp->occ_pre, fp->off_pre, fp->zb_pre, x, y, z);
  }
  c->sx += px;
  c->sy += py;
  c->sz += pz;
  c->count += 1;
  c->status = 1;
}

// Batch VoxelGrid::set_status (window indices, current toroidal offsets).
__global__ void k_set_statuses(GridDesc g, const FrameParams* __restrict__ fp, const int32_t* idx,
                               const uint8_t* st, uint64_t n) {
  VP_GRID_WAIT();
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int x = idx[3 * i], y = idx[3 * i + 1], z = idx[3 * i + 2];
    if (in_bounds(g, x, y, z)) g.cells[phys_index(g, fp->off_pre, x, y, z)].status = st[i];
  }
}

__global__ void k_map_finalize(Counters* ctr, unsigned long long* occ_total) {
  VP_GRID_WAIT();
  map_finalize_body(ctr, occ_total);
}

// Per-frame counter reset (one slot); occupied carries VoxelGrid::occupied_.
__global__ void k_frame_begin(Counters* ctr, const unsigned long long* occ_total) {
  VP_GRID_WAIT();
  uint32_t* w = reinterpret_cast<uint32_t*>(ctr);
  for (uint32_t i = threadIdx.x; i < sizeof(Counters) / 4; i += blockDim.x) w[i] = 0u;
  __syncwarp();
  if (threadIdx.x == 0) {
    ctr->occupied = *occ_total;
    for (int k = 0; k < 3; ++k) {
      ctr->box_lo[k] = 0x7fffffff;
      ctr->box_hi[k] = -1;
    }
  }
}

// ---------------------------------------------------------------------------
// occupied_voxels (voxel_grid.cpp:254-263): ordered compaction of the logical
// bitmap (x, y, z lexicographic) into logical flat indices.
// 256 threads x 8 words per block.
// ---------------------------------------------------------------------------
// kScanItems (8) consecutive bitmap words from w0: two 16-byte loads when
// aligned and in range, else word by word (zero past nwords).
__device__ __forceinline__ void load_words8(const uint32_t* __restrict__ bits, uint64_t w0, uint64_t nwords,
                                            uint32_t* v) {
  static_assert(kScanItems == 8, "two uint4 per thread");
  if (w0 + 8 <= nwords && (reinterpret_cast<uintptr_t>(bits + w0) & 15u) == 0) {
    const uint4 a = reinterpret_cast<const uint4*>(bits + w0)[0];
    const uint4 b = reinterpret_cast<const uint4*>(bits + w0)[1];
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (w0 + k < nwords) ? bits[w0 + k] : 0u;
  }
}

// Occupied scan over logical rows (x, y lexicographic; row r's cells are
// r * ez + z): a block takes kScanPerBlock rows, kScanItems per thread. The
// count pass sums the rows' occupied counts (rowcnt of the ring row); the
// emit pass reads only non-empty ring rows and rotates their words into
// logical z order (logical word wz = 32 ring bits from ring position
// 32 wz + zb).
__device__ __forceinline__ uint64_t ring_row_of(const GridDesc& g, const FrameParams* __restrict__ fp, uint32_t row) {
  const uint32_t xr = fdiv(row, g.fey);
  return ring_row_index(g, fp->off_post, static_cast<int>(xr), static_cast<int>(row - xr * static_cast<uint32_t>(g.ey)));
}

__global__ void __launch_bounds__(kScanThreads) k_bitmap_count(GridDesc g, const FrameParams* __restrict__ fp,
                                                               uint64_t r_lo, uint64_t nrows, uint32_t* bsum,
                                                               Counters* ctr) {
  VP_GRID_WAIT();
  const uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * kRowsPerBlock + static_cast<uint64_t>(threadIdx.x) * kRowItems;
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kRowItems; ++k)
    if (r0 + k < nrows) c += __ldg(g.rowcnt + ring_row_of(g, fp, static_cast<uint32_t>(r_lo + r0 + k)));
  c = block_sum_u32(c);
  if (threadIdx.x == 0) bsum[blockIdx.x] = c;
  if (last_block_done(&ctr->scan_done[0])) block_scan_array(bsum, gridDim.x, &ctr->V, nullptr);
}

// A non-empty row's ring words in logical z order: from ring word zb / 32
// (its bits >= zb % 32) to the end, then from word 0 back to that word (its
// bits < zb % 32); all W + 1 loads are independent (L1-resident row).
__global__ void __launch_bounds__(kScanThreads) k_bitmap_emit(GridDesc g, const FrameParams* __restrict__ fp,
                                                              uint64_t r_lo, uint64_t nrows, const uint32_t* boff,
                                                              uint32_t* out, uint32_t cap) {
  VP_GRID_WAIT();
  const int W = g.W, ez = g.ez, zb = fp->zb_post, Wz = g.W << 5;
  const int s0 = zb >> 5, sh = zb & 31;
  const uint64_t r0 = static_cast<uint64_t>(blockIdx.x) * kRowsPerBlock + static_cast<uint64_t>(threadIdx.x) * kRowItems;
  uint32_t cnt[kRowItems];
  uint64_t ri[kRowItems];
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kRowItems; ++k) {
    cnt[k] = 0u;
    ri[k] = 0;
    if (r0 + k < nrows) {
      ri[k] = ring_row_of(g, fp, static_cast<uint32_t>(r_lo + r0 + k));
      cnt[k] = __ldg(g.rowcnt + ri[k]);
    }
    c += cnt[k];
  }
  uint32_t pos = boff[blockIdx.x] + block_exclusive_u32(c);
#pragma unroll
  for (int k = 0; k < kRowItems; ++k) {
    if (!cnt[k]) continue;
    const uint32_t* row = fp->occ_post + ri[k] * W;
    const int64_t base = static_cast<int64_t>(r_lo + r0 + k) * ez;
    for (int t = 0; t <= W; ++t) {
      int j = s0 + t;
      if (j >= W) j -= W;
      uint32_t b = __ldg(row + j);
      if (t == 0) b &= ~0u << sh;
      if (t == W) b &= sh ? ((1u << sh) - 1u) : 0u;
      // ring position p = 32 j + bit -> window z = p - zb (+ Wz once wrapped)
      const int zoff = 32 * j - zb + (t < W - s0 ? 0 : Wz);
      while (b) {
        const int q = __ffs(b) - 1;
        b &= b - 1;
        if (pos < cap) out[pos] = static_cast<uint32_t>(base + zoff + q);
        ++pos;
      }
    }
  }
}

// Generic ordered compaction of u8 flags: positions[i] = exclusive rank.
__global__ void k_flags_count(const uint8_t* __restrict__ flags, const uint32_t* n_ptr, uint32_t cap,
                              uint32_t* bsum, uint32_t* total, uint32_t* done) {
  VP_GRID_WAIT();
  const uint32_t n = min(*n_ptr, cap);
  const uint64_t i0 = (static_cast<uint64_t>(blockIdx.x) * kScanThreads + threadIdx.x) * kScanItems;
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (i0 + k < n) c += flags[i0 + k] ? 1u : 0u;
  c = block_sum_u32(c);
  if (threadIdx.x == 0) bsum[blockIdx.x] = c;
  if (last_block_done(done)) block_scan_array(bsum, gridDim.x, total, nullptr);
}

__global__ void k_flags_positions(const uint8_t* __restrict__ flags, const uint32_t* n_ptr,
                                  uint32_t cap, const uint32_t* boff, uint32_t* pos_out) {
  VP_GRID_WAIT();
  const uint32_t n = min(*n_ptr, cap);
  const uint64_t i0 = (static_cast<uint64_t>(blockIdx.x) * kScanThreads + threadIdx.x) * kScanItems;
  uint8_t f[kScanItems];
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    f[k] = (i0 + k < n) ? flags[i0 + k] : 0;
    c += f[k] ? 1u : 0u;
  }
  uint32_t pos = boff[blockIdx.x] + block_exclusive_u32(c);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (i0 + k < n) {
      pos_out[i0 + k] = pos;
      pos += f[k] ? 1u : 0u;
    }
}

// n is read from n_ptr when non-null.
__global__ void k_scan_exclusive(uint32_t* a, uint32_t n_static, const uint32_t* n_ptr,
                                 uint32_t* total, uint32_t* total2) {
  VP_GRID_WAIT();
  block_scan_array(a, n_ptr ? *n_ptr : n_static, total, total2);
}

// Tile sums of a list of min(*n_ptr, cap) items in tiles of `per`.
__global__ void k_scan_tiles(uint32_t* a, const uint32_t* n_ptr, uint32_t cap, uint32_t per, uint32_t* total) {
  VP_GRID_WAIT();
  block_scan_array(a, (min(*n_ptr, cap) + per - 1) / per, total, nullptr);
}

}  // namespace vp
