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
__device__ __forceinline__ bool point_key(const GridDesc& g, const FrameParams* fp, uint64_t i,
                                          uint32_t* key) {
  const float* p = fp->pts + 3 * i;
  const d3 w = pose_apply(fp->R, fp->t, static_cast<double>(p[0]), static_cast<double>(p[1]),
                          static_cast<double>(p[2]));
  if (!finite3(w)) return false;
  const int ix = w2i(w.x, fp->origin_pre[0], g.res);
  const int iy = w2i(w.y, fp->origin_pre[1], g.res);
  const int iz = w2i(w.z, fp->origin_pre[2], g.res);
  if (!in_bounds(g, ix, iy, iz)) return false;
  *key = static_cast<uint32_t>((static_cast<uint64_t>(ix) * g.ey + iy) * g.ez + iz);
  return true;
}

__global__ void k_integrate_hash(GridDesc g, const FrameParams* __restrict__ fp, Counters* ctr,
                                 uint32_t* hkey, uint32_t* hcnt, uint32_t hmask, uint32_t* groups,
                                 uint32_t* pslot, uint32_t* prank) {
  const uint64_t n = fp->n;
  unsigned long long disc = 0;
  const unsigned lane = lane_id();
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x; i0 < n;
       i0 += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    uint32_t key = kEmptyKey;
    bool valid = false;
    if (i < n) {
      valid = point_key(g, fp, i, &key);
      if (!valid) ++disc;
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
  warp_add_u64(&ctr->discarded, disc);
}

__global__ void k_integrate_offsets(Counters* ctr, const uint32_t* groups, const uint32_t* hcnt,
                                    uint32_t* hoff) {
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
    if (in) hoff[slot] = base + incl - c;
  }
}

__global__ void k_integrate_scatter(const FrameParams* __restrict__ fp, const uint32_t* pslot,
                                    const uint32_t* prank, const uint32_t* hoff, uint32_t* sorted) {
  const uint64_t n = fp->n;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t s = pslot[i];
    if (s != kEmptyKey) sorted[hoff[s] + prank[i]] = static_cast<uint32_t>(i);
  }
}

__global__ void k_integrate_fold(GridDesc g, const FrameParams* __restrict__ fp, Counters* ctr,
                                 const uint32_t* groups, uint32_t* hkey, uint32_t* hcnt,
                                 const uint32_t* hoff, uint32_t* sorted) {
  const uint32_t ng = ctr->ngroups;
  unsigned long long fresh = 0;
  uint32_t* occ = fp->occ_pre;
  for (uint32_t i0 = blockIdx.x * blockDim.x; i0 < ng; i0 += gridDim.x * blockDim.x) {
    const uint32_t gi = i0 + threadIdx.x;
    if (gi < ng) {
      const uint32_t slot = groups[gi];
      const uint32_t key = hkey[slot];
      const uint32_t cnt = hcnt[slot];
      uint32_t* lst = sorted + hoff[slot];
      // ascending point index (ranks are lane-ordered, so this is ~linear)
      for (uint32_t a = 1; a < cnt; ++a) {
        const uint32_t v = lst[a];
        uint32_t b = a;
        while (b > 0 && lst[b - 1] > v) {
          lst[b] = lst[b - 1];
          --b;
        }
        lst[b] = v;
      }
      const uint32_t z = key % static_cast<uint32_t>(g.ez);
      const uint32_t r = key / static_cast<uint32_t>(g.ez);
      const uint32_t y = r % static_cast<uint32_t>(g.ey);
      const uint32_t x = r / static_cast<uint32_t>(g.ey);
      Cell* c = g.cells + phys_index(g, fp->off_pre, x, y, z);
      double sx = c->sx, sy = c->sy, sz = c->sz;
      uint32_t count = c->count;
      const bool was_free = count == 0;
      for (uint32_t a = 0; a < cnt; ++a) {
        const float* p = fp->pts + 3 * static_cast<uint64_t>(lst[a]);
        const d3 w = pose_apply(fp->R, fp->t, static_cast<double>(p[0]), static_cast<double>(p[1]),
                                static_cast<double>(p[2]));
        sx += w.x;
        sy += w.y;
        sz += w.z;
        ++count;
      }
      c->sx = sx;
      c->sy = sy;
      c->sz = sz;
      c->count = count;
      c->status = 1;  // VoxelStatus::Occupied
      if (was_free) {
        atomicOr(occ + word_of(g, x, y, z), 1u << (z & 31));
        ++fresh;
      }
      hkey[slot] = kEmptyKey;
      hcnt[slot] = 0;
    }
  }
  warp_add_u64(&ctr->newly, fresh);
}

// ---------------------------------------------------------------------------
// clear_rays (voxel_grid.cpp:182-215) with walk_segment (:122-178).
// One thread per ray; the DDA is the reference's arithmetic verbatim. Every
// interior cell is set in the clear bitmap (test-before-set keeps the hot
// cells next to the sensor from serialising on L2 atomics); k_clear_apply
// then counts unique cells, frees occupied ones and zeroes the mask.
// ---------------------------------------------------------------------------
__global__ void k_clear_walk(GridDesc g, const FrameParams* __restrict__ fp) {
  const uint64_t n = fp->n;
  const double res = g.res;
  const double* lo = fp->origin_pre;
  double hi[3];
  hi[0] = lo[0] + static_cast<double>(g.ex) * res;
  hi[1] = lo[1] + static_cast<double>(g.ey) * res;
  hi[2] = lo[2] + static_cast<double>(g.ez) * res;
  const int ext[3] = {g.ex, g.ey, g.ez};
  const d3 a = mk3(fp->t[0], fp->t[1], fp->t[2]);
  const int oc0 = w2i(a.x, lo[0], res), oc1 = w2i(a.y, lo[1], res), oc2 = w2i(a.z, lo[2], res);
  const int max_steps = g.ex + g.ey + g.ez + 4;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float* pp = fp->pts + 3 * i;
    const d3 b = pose_apply(fp->R, fp->t, static_cast<double>(pp[0]), static_cast<double>(pp[1]),
                            static_cast<double>(pp[2]));
    if (!finite3(b)) continue;
    const double d[3] = {b.x - a.x, b.y - a.y, b.z - a.z};
    const double av[3] = {a.x, a.y, a.z};
    double t0 = 0.0, t1 = 1.0;
    bool skip = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (d[k] == 0.0) {
        if (av[k] < lo[k] || av[k] >= hi[k]) skip = true;
        continue;
      }
      double ta = (lo[k] - av[k]) / d[k];
      double tb = (hi[k] - av[k]) / d[k];
      if (ta > tb) {
        const double s = ta;
        ta = tb;
        tb = s;
      }
      t0 = (t0 < ta) ? ta : t0;  // std::max(t0, ta)
      t1 = (tb < t1) ? tb : t1;  // std::min(t1, tb)
      if (t0 > t1) skip = true;
      if (skip) break;
    }
    if (skip) continue;
    const int ec0 = w2i(b.x, lo[0], res), ec1 = w2i(b.y, lo[1], res), ec2 = w2i(b.z, lo[2], res);
    const double entry[3] = {av[0] + t0 * d[0], av[1] + t0 * d[1], av[2] + t0 * d[2]};
    int cell[3];
    int step[3];
    double tmax[3], tdelta[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      int c = w2i(entry[k], lo[k], res);
      c = c < 0 ? 0 : (ext[k] - 1 < c ? ext[k] - 1 : c);  // std::clamp
      cell[k] = c;
      step[k] = 0;
      tmax[k] = CUDART_INF;
      tdelta[k] = CUDART_INF;
      if (d[k] > 0.0) {
        step[k] = 1;
        tmax[k] = t0 + (lo[k] + static_cast<double>(c + 1) * res - entry[k]) / d[k];
        tdelta[k] = res / d[k];
      } else if (d[k] < 0.0) {
        step[k] = -1;
        tmax[k] = t0 + (lo[k] + static_cast<double>(c) * res - entry[k]) / d[k];
        tdelta[k] = res / -d[k];
      }
    }
    for (int s = 0; s < max_steps; ++s) {
      const bool is_o = cell[0] == oc0 && cell[1] == oc1 && cell[2] == oc2;
      const bool is_e = cell[0] == ec0 && cell[1] == ec1 && cell[2] == ec2;
      if (!is_o && !is_e) {
        uint32_t* wp = g.clr + word_of(g, cell[0], cell[1], cell[2]);
        const uint32_t bit = 1u << (cell[2] & 31);
        if (!(__ldcg(wp) & bit)) atomicOr(wp, bit);
      }
      int m = 0;
      if (tmax[1] < tmax[m]) m = 1;
      if (tmax[2] < tmax[m]) m = 2;
      if (tmax[m] >= t1) break;
      cell[m] += step[m];
      if (cell[m] < 0 || cell[m] >= ext[m]) break;
      tmax[m] += tdelta[m];
    }
  }
}

__device__ __forceinline__ void zero_cell(Cell* c) {
  c->sx = 0.0;
  c->sy = 0.0;
  c->sz = 0.0;
  c->count = 0;
  c->status = 0;
}

__global__ void k_clear_apply(GridDesc g, const FrameParams* __restrict__ fp, Counters* ctr) {
  uint32_t* occ = fp->occ_pre;
  unsigned long long cl = 0, fr = 0;
  for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < g.nwords;
       w += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t c = g.clr[w];
    if (!c) continue;
    g.clr[w] = 0;
    cl += __popc(c);
    const uint32_t o = occ[w];
    uint32_t f = o & c;
    if (!f) continue;
    occ[w] = o & ~f;
    fr += __popc(f);
    const uint64_t row = w / g.W;
    const int z0 = static_cast<int>(w % g.W) * 32;
    const int y = static_cast<int>(row % g.ey), x = static_cast<int>(row / g.ey);
    while (f) {
      const int b = __ffs(f) - 1;
      f &= f - 1;
      zero_cell(g.cells + phys_index(g, fp->off_pre, x, y, z0 + b));
    }
  }
  warp_add_u64(&ctr->cleared, cl);
  warp_add_u64(&ctr->freed, fr);
}

// ---------------------------------------------------------------------------
// recenter (voxel_grid.cpp:217-252). The host computes the integer shift with
// the reference's arithmetic; on the device the cell array is toroidal, so a
// shift only (1) rebuilds the logical bitmap (funnel-shifted gather) and
// (2) zeroes the cells of occupied voxels that leave the window, counting them
// as voxels_dropped.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t row_bits(const uint32_t* row, int W, int b0) {
  const int wlo = b0 >= 0 ? (b0 >> 5) : -((-b0 + 31) >> 5);
  const int sh = b0 - wlo * 32;
  const uint32_t lo = (wlo >= 0 && wlo < W) ? row[wlo] : 0u;
  const uint32_t hi = (wlo + 1 >= 0 && wlo + 1 < W) ? row[wlo + 1] : 0u;
  return sh ? ((lo >> sh) | (hi << (32 - sh))) : lo;
}

__global__ void k_recenter(GridDesc g, const FrameParams* __restrict__ fp, Counters* ctr) {
  if (!fp->do_shift) return;
  const uint32_t* oldb = fp->occ_pre;
  uint32_t* newb = fp->occ_post;
  const int sx = fp->shift[0], sy = fp->shift[1], sz = fp->shift[2];
  unsigned long long dropped = 0;
  for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; u < g.nwords;
       u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t row = u / g.W;
    const int wz = static_cast<int>(u % g.W);
    const int y = static_cast<int>(row % g.ey), x = static_cast<int>(row / g.ey);
    // new word: destination (x,y,z) reads source (x+sx, y+sy, z+sz)
    const long long xs = static_cast<long long>(x) + sx, ys = static_cast<long long>(y) + sy;
    uint32_t nv = 0;
    if (xs >= 0 && xs < g.ex && ys >= 0 && ys < g.ey) {
      const long long b0 = static_cast<long long>(wz) * 32 + sz;
      if (b0 > -32 && b0 < static_cast<long long>(g.W) * 32)
        nv = row_bits(oldb + (static_cast<uint64_t>(xs) * g.ey + ys) * g.W, g.W, static_cast<int>(b0));
    }
    const int zlim = g.ez - wz * 32;
    if (zlim < 32) nv &= (1u << zlim) - 1u;
    newb[u] = nv;
    // dropped: old bits whose destination leaves the window
    const uint32_t ov = oldb[u];
    if (ov) {
      uint32_t drop;
      const long long xd = static_cast<long long>(x) - sx, yd = static_cast<long long>(y) - sy;
      if (xd < 0 || xd >= g.ex || yd < 0 || yd >= g.ey) {
        drop = ov;
      } else {
        uint32_t keep = 0;
        for (int b = 0; b < 32; ++b) {
          const long long zd = static_cast<long long>(wz) * 32 + b - sz;
          if (zd >= 0 && zd < g.ez) keep |= 1u << b;
        }
        drop = ov & ~keep;
      }
      dropped += __popc(drop);
      while (drop) {
        const int b = __ffs(drop) - 1;
        drop &= drop - 1;
        zero_cell(g.cells + phys_index(g, fp->off_pre, x, y, wz * 32 + b));
      }
    }
  }
  warp_add_u64(&ctr->dropped, dropped);
}

// VoxelGrid::merge_point (voxel_grid.cpp:49-57), one point, window index.
__global__ void k_merge_point(GridDesc g, const FrameParams* __restrict__ fp, Counters* ctr, int x,
                              int y, int z, double px, double py, double pz) {
  Cell* c = g.cells + phys_index(g, fp->off_pre, x, y, z);
  if (c->count == 0) {
    ctr->occupied += 1;
    atomicOr(fp->occ_pre + word_of(g, x, y, z), 1u << (z & 31));
  }
  c->sx += px;
  c->sy += py;
  c->sz += pz;
  c->count += 1;
  c->status = 1;
}

__global__ void k_map_finalize(Counters* ctr) {
  ctr->occupied = ctr->occupied + ctr->newly - ctr->freed - ctr->dropped;
  ctr->touched = ctr->ngroups;
}

// ---------------------------------------------------------------------------
// occupied_voxels (voxel_grid.cpp:254-263): ordered compaction of the logical
// bitmap (x, y, z lexicographic) into logical flat indices.
// 256 threads x 8 words per block.
// ---------------------------------------------------------------------------
__global__ void k_bitmap_count(const uint32_t* __restrict__ bits, uint64_t nwords, uint32_t* bsum) {
  const uint64_t w0 = (static_cast<uint64_t>(blockIdx.x) * kScanThreads + threadIdx.x) * kScanItems;
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (w0 + k < nwords) c += __popc(bits[w0 + k]);
  c = block_sum_u32(c);
  if (threadIdx.x == 0) bsum[blockIdx.x] = c;
}

__global__ void k_bitmap_emit(const uint32_t* __restrict__ bits, uint64_t nwords, int W, int ez,
                              const uint32_t* boff, uint32_t* out, uint32_t cap) {
  const uint64_t w0 = (static_cast<uint64_t>(blockIdx.x) * kScanThreads + threadIdx.x) * kScanItems;
  uint32_t v[kScanItems];
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = (w0 + k < nwords) ? bits[w0 + k] : 0u;
    c += __popc(v[k]);
  }
  uint32_t pos = boff[blockIdx.x] + block_exclusive_u32(c);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    uint32_t b = v[k];
    if (!b) continue;
    const uint64_t w = w0 + k;
    const uint64_t row = w / W;
    const uint32_t zb = static_cast<uint32_t>(w % W) * 32;
    while (b) {
      const int t = __ffs(b) - 1;
      b &= b - 1;
      if (pos < cap) out[pos] = static_cast<uint32_t>(row * ez + zb + t);
      ++pos;
    }
  }
}

// Generic ordered compaction of u8 flags: positions[i] = exclusive rank.
__global__ void k_flags_count(const uint8_t* __restrict__ flags, const uint32_t* n_ptr, uint32_t cap,
                              uint32_t* bsum) {
  const uint32_t n = min(*n_ptr, cap);
  const uint64_t i0 = (static_cast<uint64_t>(blockIdx.x) * kScanThreads + threadIdx.x) * kScanItems;
  uint32_t c = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (i0 + k < n) c += flags[i0 + k] ? 1u : 0u;
  c = block_sum_u32(c);
  if (threadIdx.x == 0) bsum[blockIdx.x] = c;
}

__global__ void k_flags_positions(const uint8_t* __restrict__ flags, const uint32_t* n_ptr,
                                  uint32_t cap, const uint32_t* boff, uint32_t* pos_out) {
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

// Single-block exclusive scan of a[0..n) in place; *total = sum (optional
// also copied to *total2). n is read from n_ptr when non-null.
__global__ void k_scan_exclusive(uint32_t* a, uint32_t n_static, const uint32_t* n_ptr,
                                 uint32_t* total, uint32_t* total2) {
  const uint32_t n = n_ptr ? *n_ptr : n_static;
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t b = 0; b < n; b += blockDim.x) {
    const uint32_t i = b + threadIdx.x;
    const uint32_t v = i < n ? a[i] : 0u;
    const uint32_t ex = block_exclusive_u32(v);
    const uint32_t c = carry;
    if (i < n) a[i] = c + ex;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = c + ex + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (total) *total = carry;
    if (total2) *total2 = carry;
  }
}

}  // namespace vp
