// Spatial-slab segmentation kernels: the window is split
// along x into slabs, one per GPU; build_adjacency + label_components
// (segmentation.cpp:87-194) run per slab on its steppable voxels plus a
// w-plane halo of each neighbour, and a boundary-label merge turns the local
// labels into the single-grid canonical labels (component-minimum ordinal).
//
// Ordinals are global: the steppable list is x-major (voxel_grid.cpp:254-263,
// segmentation.cpp:73-83), so slab k owns the contiguous ordinal range
// [P[xb_k], P[xb_{k+1})) where P is the prefix sum of per-plane counts, and an
// extended list [x_lo, x_hi) is a contiguous ordinal range starting at
// base = P[x_lo]; local list index i is global ordinal base + i.
//
// Merge. The boundary zone is every window x within w of an internal slab
// boundary B ([B - w, B + w)): exactly the planes that appear in some other
// slab's extended list. Every slab emits, for each extended-list entry in the
// zone, the triple (zone(ordinal), zone(b), L) where b is the smallest zone
// ordinal of the entry's local component and L the component's local label.
// Union-find over the zone (hook larger under smaller) joins the local
// components that share a voxel; the canonical label of a joined set is the
// minimum L over it (the global component minimum lies in the local component
// of its owner, whose local label is that minimum). Components that never
// reach the zone keep their local label, which is already canonical.
#include "vp_kernels.cuh"

namespace vp {

__device__ __forceinline__ int zone_of(const ZoneDesc& z, int x) {
  for (int k = 0; k < z.n; ++k)
    if (x >= z.xlo[k] && x < z.xhi[k]) return k;
  return -1;
}

__device__ __forceinline__ int32_t zone_index(const ZoneDesc& z, int k, int64_t ordinal) {
  return static_cast<int32_t>(z.dbase[k] + (ordinal - z.olo[k]));
}

__device__ __forceinline__ int owner_of(const RankDesc& r, int64_t label) {
  int k = 0;
  for (int q = 1; q < r.n; ++q)
    if (r.ord_lo[q] <= label) k = q;
  return k;
}

// Steppable entries per owned x-plane (the list is x-major): two binary
// searches per plane, no atomics.
__global__ void k_plane_counts(const Counters* ctr, const int32_t* __restrict__ st_idx, uint32_t cap,
                               int32_t x0, int32_t nplanes, uint32_t* counts) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, cap);
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < nplanes; p += gridDim.x * blockDim.x) {
    uint32_t lohi[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int x = x0 + p + h;
      uint32_t lo = 0, hi = S;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(st_idx + 3ull * mid) < x) lo = mid + 1; else hi = mid;
      }
      lohi[h] = lo;
    }
    counts[p] = lohi[1] - lohi[0];
  }
}

__global__ void k_fill_i32(int32_t* a, uint64_t n, int32_t v) {
  VP_GRID_WAIT();
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    a[i] = v;
}

// Smallest zone entry (local index) of every local component.
__global__ void k_zone_bmin(const Counters* ctr, SegBufs b, ZoneDesc z, int32_t* bmin) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x)
    if (zone_of(z, __ldg(b.st_idx + 3ull * i)) >= 0) {
      const int32_t r = b.label[i];
      const unsigned peers = __match_any_sync(__activemask(), r);
      const int32_t m = static_cast<int32_t>(__reduce_min_sync(peers, i));
      if (static_cast<int>(lane_id()) == __ffs(peers) - 1) atomicMin(bmin + r, m);
    }
}

// One triple per zone entry: (zone(ordinal), zone(component's smallest zone
// ordinal), component label). Warp-aggregated slots; the order of the
// triples does not affect the merge result.
__global__ void k_zone_triples(const Counters* ctr, SegBufs b, ZoneDesc z, int64_t base,
                               const int32_t* __restrict__ bmin, int32_t* out, uint32_t* nout) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  const unsigned lane = lane_id();
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); i0 < S; i0 += stride) {
    const uint32_t i = i0 + lane;
    const int k = i < S ? zone_of(z, __ldg(b.st_idx + 3ull * i)) : -1;
    const unsigned m = __ballot_sync(0xffffffffu, k >= 0);
    if (!m) continue;
    uint32_t slot = 0;
    if (lane == static_cast<unsigned>(__ffs(m) - 1)) slot = atomicAdd(nout, static_cast<uint32_t>(__popc(m)));
    slot = __shfl_sync(0xffffffffu, slot, __ffs(m) - 1) + __popc(m & lanemask_lt());
    if (k < 0) continue;
    const int32_t r = b.label[i];
    const int32_t bm = bmin[r];
    const int kb = zone_of(z, __ldg(b.st_idx + 3ull * bm));
    out[3ull * slot] = zone_index(z, k, base + i);
    out[3ull * slot + 1] = zone_index(z, kb, base + bm);
    out[3ull * slot + 2] = static_cast<int32_t>(base + r);
  }
}

__global__ void k_zone_init(int32_t* parent, int32_t* minlab, uint64_t Z) {
  VP_GRID_WAIT();
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < Z;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    parent[i] = static_cast<int32_t>(i);
    minlab[i] = 0x7fffffff;
  }
}

// Union of every triple's two zone entries (padding triples have a < 0).
__global__ void k_zone_union(const int32_t* __restrict__ t, uint64_t n, int32_t* parent) {
  VP_GRID_WAIT();
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const int32_t a = __ldg(t + 3 * j);
    if (a < 0) continue;
    uf_union(parent, a, __ldg(t + 3 * j + 1));
  }
}

// Canonical label of each joined set: the minimum local label over it.
__global__ void k_zone_minlab(const int32_t* __restrict__ t, uint64_t n, int32_t* parent, int32_t* minlab) {
  VP_GRID_WAIT();
  for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < n;
       j += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (__ldg(t + 3 * j) < 0) continue;
    const int32_t r = uf_find(parent, __ldg(t + 3 * j + 1));
    const unsigned peers = __match_any_sync(__activemask(), r);
    const int32_t m = __reduce_min_sync(peers, __ldg(t + 3 * j + 2));
    if (static_cast<int>(lane_id()) == __ffs(peers) - 1) atomicMin(minlab + r, m);
  }
}

// Final (global, canonical) label of every owned entry.
__global__ void k_slab_relabel(SegBufs b, ZoneDesc z, int64_t base, uint32_t n_left, uint32_t n_own,
                               const int32_t* __restrict__ bmin, int32_t* parent,
                               const int32_t* __restrict__ minlab, int32_t* flabel) {
  VP_GRID_WAIT();
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n_own; j += gridDim.x * blockDim.x) {
    const int32_t r = b.label[n_left + j];
    const int32_t bm = bmin[r];
    if (bm == 0x7fffffff) {
      flabel[j] = static_cast<int32_t>(base + r);
    } else {
      const int kb = zone_of(z, __ldg(b.st_idx + 3ull * bm));
      flabel[j] = minlab[uf_find(parent, zone_index(z, kb, base + bm))];
    }
  }
}

// ---- cluster gather: members of clusters owned by a lower slab go to the
// owner, stable-sorted by destination (ascending ordinal inside each).
__global__ void k_export_hist(uint32_t n_own, const int32_t* __restrict__ flabel, RankDesc rd, int me,
                              uint32_t* H, uint32_t nch, uint32_t* dcount) {
  VP_GRID_WAIT();
  __shared__ uint32_t hist[kMaxSlabs];
  const unsigned lane = lane_id();
  const int64_t own_lo = rd.ord_lo[me];
  for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
    for (int d = lane; d < rd.n; d += 32) hist[d] = 0;
    __syncwarp();
    const uint32_t e1 = min(n_own, (c + 1) * kChunk);
    for (uint32_t e = c * kChunk + lane; e < e1; e += 32) {
      const int32_t L = __ldg(flabel + e);
      if (L < own_lo) atomicAdd(&hist[owner_of(rd, L)], 1u);
    }
    __syncwarp();
    for (int d = lane; d < rd.n; d += 32) {
      H[static_cast<uint64_t>(d) * nch + c] = hist[d];
      if (hist[d]) atomicAdd(dcount + d, hist[d]);
    }
    __syncwarp();
  }
}

__global__ void k_export_scatter(uint32_t n_own, const int32_t* __restrict__ flabel,
                                 const double* __restrict__ mean, RankDesc rd, int me,
                                 const uint32_t* __restrict__ H, uint32_t nch, MemberRec* out) {
  VP_GRID_WAIT();
  __shared__ uint32_t run[kMaxSlabs];
  const unsigned lane = lane_id();
  const int64_t own_lo = rd.ord_lo[me];
  for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
    for (int d = lane; d < rd.n; d += 32) run[d] = H[static_cast<uint64_t>(d) * nch + c];
    __syncwarp();
    const uint32_t e1 = min(n_own, (c + 1) * kChunk);
    for (uint32_t e0 = c * kChunk; e0 < e1; e0 += 32) {
      const uint32_t e = e0 + lane;
      const int32_t L = e < e1 ? __ldg(flabel + e) : 0x7fffffff;
      const int d = L < own_lo ? owner_of(rd, L) : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const int leader = __ffs(peers) - 1;
      const uint32_t bse = d >= 0 ? run[d] : 0u;
      __syncwarp();
      if (d >= 0 && static_cast<int>(lane) == leader) run[d] = bse + __popc(peers);
      __syncwarp();
      if (d >= 0) {
        MemberRec r;
        r.m[0] = mean[3ull * e];
        r.m[1] = mean[3ull * e + 1];
        r.m[2] = mean[3ull * e + 2];
        r.label = L;
        r.pad = 0;
        out[bse + __popc(peers & lanemask_lt())] = r;
      }
    }
    __syncwarp();
  }
}

// ---- the owner's clusters: virtual list = own entries ++ received members
// (from slabs me+1, me+2, ... in order = ascending ordinal). Entries whose
// cluster is owned here get its local root index as label; the others point
// at themselves with a zero count, so filter_clusters never selects them.
__global__ void k_owner_init(uint32_t n, SegBufs b) {
  VP_GRID_WAIT();
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    b.cnt[e] = 0;
    b.cid[e] = -1;
  }
}

__global__ void k_owner_prep(uint32_t n_own, uint32_t n_recv, int64_t own_base,
                             const double* __restrict__ own_mean, const int32_t* __restrict__ flabel,
                             const MemberRec* __restrict__ recv, SegBufs b) {
  VP_GRID_WAIT();
  const uint32_t n = n_own + n_recv;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
    int32_t L;
    double m0, m1, m2;
    if (e < n_own) {
      L = flabel[e];
      m0 = own_mean[3ull * e];
      m1 = own_mean[3ull * e + 1];
      m2 = own_mean[3ull * e + 2];
    } else {
      const MemberRec& r = recv[e - n_own];
      L = r.label;
      m0 = r.m[0];
      m1 = r.m[1];
      m2 = r.m[2];
    }
    b.st_mean[3ull * e] = m0;
    b.st_mean[3ull * e + 1] = m1;
    b.st_mean[3ull * e + 2] = m2;
    const int64_t local = static_cast<int64_t>(L) - own_base;
    const bool mine = local >= 0 && local < static_cast<int64_t>(n_own);
    b.label[e] = mine ? static_cast<int32_t>(local) : static_cast<int32_t>(e);
    if (mine) atomic_inc_agg(b.cnt, static_cast<int>(local));
  }
}

// Cluster labels back to global ordinals (after the cluster setup, before the
// RANSAC seeds read them).
__global__ void k_klabel_rebase(const Counters* ctr, SegBufs b, int64_t base) {
  VP_GRID_WAIT();
  const uint32_t K = min(ctr->K, b.Kcap);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x)
    b.klabel[k] = static_cast<int32_t>(b.klabel[k] + base);
}

}  // namespace vp
