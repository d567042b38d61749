// Segmentation kernels: normals + steppability, CCL, cluster gather, RANSAC,
// refine, polygon. Reference: /root/reference/proj/core/src/{segmentation,
// jacobi,plane_fit,polygonize}.cpp and pipeline.cpp:43-85.
#include <cooperative_groups.h>

#include "vp_kernels.cuh"

namespace vp {

// ---------------------------------------------------------------------------
// estimate_normals + classify_steppable (segmentation.cpp:19-85), fused.
// One thread per occupied voxel; the (2r+1)^3 window is probed in the
// reference's dx -> dy -> dz order through the logical occupancy bitmap, and
// only occupied neighbours' 32-byte cells are read. The angle predicate
// acos(d)*kRadToDeg <= theta is evaluated as d >= d*, with d* found on the host
// by bisection over the host libm acos (exact; A.3).
// ---------------------------------------------------------------------------
// Blocks walk the list in tiles of blockDim voxels and write each tile's
// steppable count to tsum (the steppable compaction's block sums).
__global__ void k_normals(GridDesc g, const FrameParams* __restrict__ fp, Counters* ctr, SegDev sp,
                          SegBufs b, int write_status, uint32_t* tsum) {
  VP_GRID_WAIT();
  if (blockIdx.x == 0 && threadIdx.x == 0 && ctr->V > b.Vcap) atomicOr(&ctr->overflow, kOverflowOcc);
  const uint32_t V = min(ctr->V, b.Vcap);
  const uint32_t* occ = fp->occ_post;
  const int32_t* off = fp->off_post;
  const int r = sp.radius;
  for (uint32_t t0 = blockIdx.x * blockDim.x; t0 < V; t0 += gridDim.x * blockDim.x) {
    const uint32_t v = t0 + threadIdx.x;
    bool step = false;
    if (v < V) {
    const uint32_t flat = b.occ_list[v];
    const uint32_t rr = fdiv(flat, g.fez);
    const int z = static_cast<int>(flat - rr * static_cast<uint32_t>(g.ez));
    const uint32_t xr = fdiv(rr, g.fey);
    const int y = static_cast<int>(rr - xr * static_cast<uint32_t>(g.ey));
    const int x = static_cast<int>(xr);
    Cell* own = g.cells + phys_index(g, off, x, y, z);
    const uint32_t oc = own->count;
    const double ocd = static_cast<double>(oc);
    const d3 om = mk3(own->sx / ocd, own->sy / ocd, own->sz / ocd);
    const uint8_t ostatus = own->status;

    d3 sum = mk3(0.0, 0.0, 0.0);
    double s00 = 0.0, s01 = 0.0, s02 = 0.0, s11 = 0.0, s12 = 0.0, s22 = 0.0;
    int n = 0;
    if (r == 1) {
      // default 3x3x3 window, fully unrolled: the 9 row words and the occupied
      // neighbours' cells are independent loads; the sums stay in dx,dy,dz order
      const int za = z - 1, zb = z + 1;
      uint32_t occ3[9];
      // ring position of z - 1 (or of z at the window's bottom): the three
      // bits z-1, z, z+1 are one 32-bit ring window
      const int pz = ring_z(g, fp->zb_post, za >= 0 ? za : z);
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int X = x + q / 3 - 1, Y = y + q % 3 - 1;
        uint32_t bits = 0;
        if (X >= 0 && X < g.ex && Y >= 0 && Y < g.ey) {
          const uint32_t* row = occ_row(g, const_cast<uint32_t*>(occ), off, X, Y);
          const uint32_t v = ring_bits32(row, g.W, pz);
          bits = za >= 0 ? (v & 7u) : ((v << 1) & 6u);
          if (zb >= g.ez) bits &= 3u;
        }
        occ3[q] = bits;
      }
#pragma unroll
      for (int q = 0; q < 27; ++q) {
        if ((occ3[q / 3] >> (q % 3)) & 1u) {
          const Cell* c = g.cells + phys_index(g, off, x + q / 9 - 1, y + (q / 3) % 3 - 1, z + q % 3 - 1);
          const double2 sxy = __ldg(reinterpret_cast<const double2*>(c));
          const double szz = __ldg(&c->sz);
          const double cd = static_cast<double>(__ldg(&c->count));
          const d3 m = mk3(sxy.x / cd, sxy.y / cd, szz / cd);
          sum = add3(sum, m);
          s00 = s00 + m.x * m.x;
          s01 = s01 + m.y * m.x;
          s02 = s02 + m.z * m.x;
          s11 = s11 + m.y * m.y;
          s12 = s12 + m.z * m.y;
          s22 = s22 + m.z * m.z;
          ++n;
        }
      }
    } else
    for (int dx = -r; dx <= r; ++dx) {
      const int X = x + dx;
      if (X < 0 || X >= g.ex) continue;
      for (int dy = -r; dy <= r; ++dy) {
        const int Y = y + dy;
        if (Y < 0 || Y >= g.ey) continue;
        const uint32_t* row = occ_row(g, const_cast<uint32_t*>(occ), off, X, Y);
        for (int dz = -r; dz <= r; ++dz) {
          const int Z = z + dz;
          if (Z < 0 || Z >= g.ez) continue;
          const int pz = ring_z(g, fp->zb_post, Z);
          if (!((__ldcg(row + (pz >> 5)) >> (pz & 31)) & 1u)) continue;
          const Cell* c = g.cells + phys_index(g, off, X, Y, Z);
          const double cd = static_cast<double>(c->count);
          const d3 m = mk3(c->sx / cd, c->sy / cd, c->sz / cd);
          sum = add3(sum, m);
          s00 = s00 + m.x * m.x;
          s01 = s01 + m.y * m.x;
          s02 = s02 + m.z * m.x;
          s11 = s11 + m.y * m.y;
          s12 = s12 + m.z * m.y;
          s22 = s22 + m.z * m.z;
          ++n;
        }
      }
    }
    bool valid = false;
    d3 nrm = mk3(0.0, 0.0, 0.0);
    if (n >= 3) {
      const double dn = static_cast<double>(n);
      const d3 mean = div3(sum, dn);
      double cov[3][3];
      cov[0][0] = s00 / dn - mean.x * mean.x;
      cov[0][1] = s01 / dn - mean.y * mean.x;
      cov[0][2] = s02 / dn - mean.z * mean.x;
      cov[1][0] = s01 / dn - mean.x * mean.y;
      cov[1][1] = s11 / dn - mean.y * mean.y;
      cov[1][2] = s12 / dn - mean.z * mean.y;
      cov[2][0] = s02 / dn - mean.x * mean.z;
      cov[2][1] = s12 / dn - mean.y * mean.z;
      cov[2][2] = s22 / dn - mean.z * mean.z;
      const Eig3 e = jacobi3(cov);
      if (!(e.val[1] <= 1e-12 + 1e-9 * fabs(e.val[2]))) {
        nrm = orient_up(normalized3(e.vec[0]), sp.up);
        valid = true;
      }
    }
    double d = valid ? dot3(nrm, sp.up) : 0.0;
    d = d < 0.0 ? 0.0 : (1.0 < d ? 1.0 : d);  // std::clamp(d, 0, 1)
    step = valid && n >= sp.min_neighbors && d >= sp.dstar;
    if (write_status) own->status = step ? 2 : 1;  // VoxelStatus::Steppable / Occupied
    b.est_normal[3 * v] = nrm.x;
    b.est_normal[3 * v + 1] = nrm.y;
    b.est_normal[3 * v + 2] = nrm.z;
    b.est_ncount[v] = n;
    b.est_valid[v] = valid ? 1 : 0;
    b.own_mean[3 * v] = om.x;
    b.own_mean[3 * v + 1] = om.y;
    b.own_mean[3 * v + 2] = om.z;
    b.own_count[v] = oc;
    b.own_status[v] = ostatus;
    b.step_flag[v] = step ? 1 : 0;
    }  // v < V
    const int c = __syncthreads_count(step);
    if (threadIdx.x == 0) tsum[t0 / blockDim.x] = static_cast<uint32_t>(c);
  }
  // the last block scans the tile counts: tile offsets and ctr->S
  if (last_block_done(&ctr->scan_done[1])) block_scan_array(tsum, (V + blockDim.x - 1) / blockDim.x, &ctr->S, nullptr);
}

// Steppable list in occupied (lexicographic) order -> ordinals; fills the
// ordinal map used by the CCL window search. Same tiles as k_normals: a
// voxel's ordinal = its tile's offset (scanned tsum) + its rank in the tile.
__global__ void k_step_emit(GridDesc g, Counters* ctr, SegBufs b, MapDesc m, int xadd, const uint32_t* toff) {
  VP_GRID_WAIT();
  const uint32_t V = min(ctr->V, b.Vcap);
  for (uint32_t t0 = blockIdx.x * blockDim.x; t0 < V; t0 += gridDim.x * blockDim.x) {
    const uint32_t v = t0 + threadIdx.x;
    const bool f = v < V && b.step_flag[v];
    const uint32_t s = toff[t0 / blockDim.x] + block_exclusive_u32(f ? 1u : 0u);
    if (!f) continue;
    if (s >= b.Scap) {
      atomicOr(&ctr->overflow, kOverflowStep);
      continue;
    }
    const uint32_t flat = b.occ_list[v];
    const uint32_t rr = fdiv(flat, g.fez);
    const int z = static_cast<int>(flat - rr * static_cast<uint32_t>(g.ez));
    const uint32_t xr = fdiv(rr, g.fey);
    const int y = static_cast<int>(rr - xr * static_cast<uint32_t>(g.ey));
    const int x = static_cast<int>(xr);
    b.st_idx[3 * s] = x + xadd;  // xadd: slab -> window x (0 for a plain grid)
    b.st_idx[3 * s + 1] = y;
    b.st_idx[3 * s + 2] = z;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      b.st_mean[3 * s + k] = b.own_mean[3 * v + k];
      b.st_normal[3 * s + k] = b.est_normal[3 * v + k];
    }
    if (m.map) {
      m.map[m.slot(x, y, z)] = static_cast<int32_t>(s);
      atomicOr(m.bits + m.word(x, y, z), 1u << ((z - m.lo[2]) & 31));
    }
  }
}

// Host-provided steppable list (vp_label_components): fill the map only.
__global__ void k_map_fill(Counters* ctr, SegBufs b, MapDesc m) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    const int x = b.st_idx[3 * s], y = b.st_idx[3 * s + 1], z = b.st_idx[3 * s + 2];
    m.map[m.slot(x, y, z)] = static_cast<int32_t>(s);
    atomicOr(m.bits + m.word(x, y, z), 1u << ((z - m.lo[2]) & 31));
  }
}

__global__ void k_ccl_init(Counters* ctr, SegBufs b) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < S; s += gridDim.x * blockDim.x) {
    b.parent[s] = static_cast<int32_t>(s);
    b.cnt[s] = 0;
    b.cid[s] = -1;
  }
}

// ---------------------------------------------------------------------------
// build_adjacency + label_components (segmentation.cpp:87-194).
// The reference materialises every adjacency list and propagates minimum
// labels until quiet. Here the edge predicate is evaluated on the fly over
// the forward half of the (2w+1)^3 window (ordinals are lexicographic, so
// "forward in (x,y,z)" == "j > i"), and each edge is a union-find union that
// always hooks the larger root under the smaller (atomicCAS), so every root is
// its component's minimum ordinal: the canonical label, bit-exact.
// ---------------------------------------------------------------------------
// Edge predicate of build_adjacency (segmentation.cpp:124-125), evaluated in
// the reference's arithmetic: squaredNorm of the mean difference, normal dot.
__device__ __forceinline__ bool adjacent(const SegBufs& b, const SegDev& sp, d3 mi, d3 ni, int j) {
  const d3 mj = mk3(__ldg(b.st_mean + 3 * j), __ldg(b.st_mean + 3 * j + 1), __ldg(b.st_mean + 3 * j + 2));
  if (sqn3(sub3(mi, mj)) >= sp.d2_th) return false;
  const d3 nj = mk3(__ldg(b.st_normal + 3 * j), __ldg(b.st_normal + 3 * j + 1),
                    __ldg(b.st_normal + 3 * j + 2));
  return dot3(ni, nj) > sp.cos_th;
}

// Window rows of voxel i: forward half (dx = 0: dy = 0..w with dz > 0 on
// dy = 0; dx = 1..w: dy = -w..w) or, with backward = true, its mirror image.
__device__ __forceinline__ bool window_row(int r, int w, int span, bool backward, int& dx, int& dy) {
  if (r <= w) {
    dx = 0;
    dy = r;
  } else {
    const int q = r - (w + 1);
    dx = 1 + q / span;
    dy = q % span - w;
  }
  if (backward) {
    dx = -dx;
    dy = -dy;
  }
  return true;
}

// CCL phase 1 (ECL-CC style initial hooking, no atomics): parent[i] = the
// smallest ordinal j < i adjacent to i, else i. Each node writes only its own
// parent and j < i keeps parent[x] <= x, so this is a valid set of unions.
// One warp per voxel; the steppable bitmap turns each window row into one
// word load, and only present voxels are probed.
__global__ void __launch_bounds__(256) k_ccl_hook(Counters* ctr, SegDev sp, SegBufs b, MapDesc m) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  const int w = sp.w, span = 2 * w + 1;
  const int nrows = (w + 1) + w * span;
  const unsigned lane = lane_id();
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarp = (gridDim.x * blockDim.x) >> 5;
  const int xlo = m.lo[0], ylo = m.lo[1], yhi = m.lo[1] + m.dims[1] - 1;
  const int zlo_m = m.lo[2], zhi_m = m.lo[2] + m.dims[2] - 1;
  for (uint32_t i = warp; i < S; i += nwarp) {
    const int x = __ldg(b.st_idx + 3 * i), y = __ldg(b.st_idx + 3 * i + 1), z = __ldg(b.st_idx + 3 * i + 2);
    const d3 mi = mk3(__ldg(b.st_mean + 3 * i), __ldg(b.st_mean + 3 * i + 1), __ldg(b.st_mean + 3 * i + 2));
    const d3 ni = mk3(__ldg(b.st_normal + 3 * i), __ldg(b.st_normal + 3 * i + 1),
                      __ldg(b.st_normal + 3 * i + 2));
    int best = static_cast<int>(i);
    // rows from the back of the window (dx = -w first): ordinals decrease
    // with r, so once a batch of 32 rows holds an adjacent voxel, no later
    // batch can hold a smaller one
    for (int r0 = nrows - 1; r0 >= 0; r0 -= 32) {
      if (__any_sync(0xffffffffu, best < static_cast<int>(i))) break;
      const int r = r0 - static_cast<int>(lane);
      if (r < 0) continue;
      int dx, dy;
      window_row(r, w, span, true, dx, dy);
      const int X = x + dx, Y = y + dy;
      if (X < xlo || Y < ylo || Y > yhi) continue;
      const int z0 = max(z - w, zlo_m);
      const int z1 = (dx == 0 && dy == 0) ? z - 1 : min(z + w, zhi_m);
      if (z0 > z1) continue;
      uint32_t bits = m.row_span(X, Y, z0, z1 - z0 + 1);
      if (!bits) continue;
      // voxels of one (X, Y) column are consecutive ordinals: one map load
      const int j0 = __ldg(m.map + m.slot(X, Y, z0 + __ffs(bits) - 1));
      for (int j = j0; bits && j < best; ++j) {
        bits &= bits - 1;
        if (adjacent(b, sp, mi, ni, j)) best = j;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0) {
      b.parent[i] = best;
      b.cnt[i] = 0;
      b.cid[i] = -1;
    }
  }
}

// Pointer jumping to the root for every node (ld.cg: roots written by other
// SMs in k_ccl_hook are visible; no node changes its own value concurrently
// except through jumps to an ancestor, which keeps the result a root).
__global__ void k_ccl_compress(Counters* ctr, SegBufs b) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x)
    __stcg(b.parent + i, uf_find(b.parent, static_cast<int>(i)));
}

// One pointer-jumping round over the hook forest (parent[i] <- parent[parent[i]]):
// two rounds before k_ccl_compress cut the hook chains (C2: up to ~31 deep)
// by 4x, so compression is no longer one thread's long serial chain.
__global__ void k_ccl_jump(Counters* ctr, SegBufs b) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
    const int p = __ldcg(b.parent + i);
    const int pp = __ldcg(b.parent + p);
    if (pp < p) __stcg(b.parent + i, pp);
  }
}

// CCL phase 2: every forward edge (i, j > i) as a union. The 4-byte parent[j]
// is checked against i's cached root before the 48-byte predicate loads, so
// edges inside an already-joined tree cost one load.
__global__ void __launch_bounds__(256) k_ccl_union(Counters* ctr, SegDev sp, SegBufs b, MapDesc m) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  const int w = sp.w, span = 2 * w + 1;
  const int nrows = (w + 1) + w * span;
  int32_t* parent = b.parent;
  const unsigned lane = lane_id();
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarp = (gridDim.x * blockDim.x) >> 5;
  const int xmax = m.lo[0] + m.dims[0] - 1, ymin = m.lo[1], ymax = m.lo[1] + m.dims[1] - 1;
  const int zmin = m.lo[2], zmax = m.lo[2] + m.dims[2] - 1;
  for (uint32_t i = warp; i < S; i += nwarp) {
    const int x = __ldg(b.st_idx + 3 * i), y = __ldg(b.st_idx + 3 * i + 1), z = __ldg(b.st_idx + 3 * i + 2);
    const d3 mi = mk3(__ldg(b.st_mean + 3 * i), __ldg(b.st_mean + 3 * i + 1), __ldg(b.st_mean + 3 * i + 2));
    const d3 ni = mk3(__ldg(b.st_normal + 3 * i), __ldg(b.st_normal + 3 * i + 1),
                      __ldg(b.st_normal + 3 * i + 2));
    int ri = -1;
    if (lane == 0) ri = uf_find(parent, static_cast<int>(i));
    ri = __shfl_sync(0xffffffffu, ri, 0);
    for (int r = static_cast<int>(lane); r < nrows; r += 32) {
      int dx, dy;
      window_row(r, w, span, false, dx, dy);
      const int X = x + dx, Y = y + dy;
      if (X > xmax || Y < ymin || Y > ymax) continue;
      const int z0 = (dx == 0 && dy == 0) ? z + 1 : max(z - w, zmin);
      const int z1 = min(z + w, zmax);
      if (z0 > z1) continue;
      uint32_t bits = m.row_span(X, Y, z0, z1 - z0 + 1);
      if (!bits) continue;
      // voxels of one (X, Y) column are consecutive ordinals: one map load
      int j = __ldg(m.map + m.slot(X, Y, z0 + __ffs(bits) - 1)) - 1;
      while (bits) {
        bits &= bits - 1;
        ++j;
        // L1-cached early-out: a stale parent[j] is an earlier ancestor of j;
        // if it equals ri, i and j were already in one set (sets only merge)
        const int pj = __ldca(parent + j);
        if (pj == ri) continue;  // already in i's tree
        if (!adjacent(b, sp, mi, ni, j)) continue;
        const int rj = uf_find(parent, j);
        if (rj == ri) continue;
        ri = uf_link(parent, ri, rj);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Edge-balanced variants of k_ccl_hook / k_ccl_union (the default CCL).
// The row-per-lane kernels above walk a row's present voxels serially: a
// lane's dependent loads (bitmap word -> ordinal -> parent[j] -> predicate,
// once per present bit) form a chain of ~20 L2 round trips per voxel, and a
// plane voxel has ~11 non-empty rows of up to 11 voxels spread over 61 rows.
// Here the warp first lists its voxel's candidate ordinals in shared memory
// (one bitmap word + one ordinal load per row, all rows in parallel, then a
// warp scan of the popcounts), and the lanes then take the candidates 32 at a
// time, so every voxel costs ~4 dependent round trips whatever its degree.
// Same edges, same link rule -> the same canonical labels.
// ---------------------------------------------------------------------------
constexpr int kCclWarps = 8;     // 256-thread blocks
constexpr int kCclEdgeBuf = 256; // candidate ordinals per warp and pass

// Lists the present voxels of this lane's row (X, Y, z0..z1) into buf at
// [pos - base, ...) clipped to [0, kCclEdgeBuf), ascending ordinal.
__device__ __forceinline__ void ccl_list_row(int32_t* buf, uint32_t bits, int j0, uint32_t pos, uint32_t base) {
  int j = j0;
  while (bits) {
    bits &= bits - 1;
    if (pos >= base && pos < base + kCclEdgeBuf) buf[pos - base] = j;
    ++pos;
    ++j;
  }
}

// Row (X, Y) of the window and its z range for voxel (x, y, z), backward or
// forward half; false when it leaves the map box. Out: present bits and the
// ordinal of the first present voxel.
__device__ __forceinline__ uint32_t ccl_row_bits(const MapDesc& m, int w, int span, int r, bool backward, int x,
                                                 int y, int z, int& j0) {
  int dx, dy;
  window_row(r, w, span, backward, dx, dy);
  const int X = x + dx, Y = y + dy;
  j0 = 0;
  if (X < m.lo[0] || X > m.lo[0] + m.dims[0] - 1 || Y < m.lo[1] || Y > m.lo[1] + m.dims[1] - 1) return 0u;
  const int zlo = m.lo[2], zhi = m.lo[2] + m.dims[2] - 1;
  int z0, z1;
  if (dx == 0 && dy == 0) {
    z0 = backward ? max(z - w, zlo) : z + 1;
    z1 = backward ? z - 1 : min(z + w, zhi);
  } else {
    z0 = max(z - w, zlo);
    z1 = min(z + w, zhi);
  }
  if (z0 > z1) return 0u;
  const uint32_t bits = m.row_span(X, Y, z0, z1 - z0 + 1);
  if (bits) j0 = __ldg(m.map + m.slot(X, Y, z0 + __ffs(bits) - 1));
  return bits;
}

// Phase 1: parent[i] = the smallest adjacent ordinal j < i, else i. Backward
// rows are taken 32 at a time in ascending ordinal order (the last rows of
// the window first), their candidates tested 32 at a time; the first adjacent
// candidate is the minimum.
__global__ void __launch_bounds__(256) k_ccl_hook_bal(Counters* ctr, SegDev sp, SegBufs b, MapDesc m) {
  VP_GRID_WAIT();
  __shared__ int32_t cand[kCclWarps][kCclEdgeBuf];
  const uint32_t S = min(ctr->S, b.Scap);
  const int w = sp.w, span = 2 * w + 1;
  const int nrows = (w + 1) + w * span;
  const unsigned lane = lane_id();
  int32_t* buf = cand[threadIdx.x >> 5];
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarp = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = warp; i < S; i += nwarp) {
    const int x = __ldg(b.st_idx + 3 * i), y = __ldg(b.st_idx + 3 * i + 1), z = __ldg(b.st_idx + 3 * i + 2);
    const d3 mi = mk3(__ldg(b.st_mean + 3 * i), __ldg(b.st_mean + 3 * i + 1), __ldg(b.st_mean + 3 * i + 2));
    const d3 ni = mk3(__ldg(b.st_normal + 3 * i), __ldg(b.st_normal + 3 * i + 1),
                      __ldg(b.st_normal + 3 * i + 2));
    int best = static_cast<int>(i);
    for (int r0 = nrows - 1; r0 >= 0 && best == static_cast<int>(i); r0 -= 32) {
      const int r = r0 - static_cast<int>(lane);
      int j0 = 0;
      const uint32_t bits = r >= 0 ? ccl_row_bits(m, w, span, r, true, x, y, z, j0) : 0u;
      const uint32_t c = __popc(bits);
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (static_cast<int>(lane) >= o) incl += t;
      }
      const uint32_t E = __shfl_sync(0xffffffffu, incl, 31);
      for (uint32_t base = 0; base < E && best == static_cast<int>(i); base += kCclEdgeBuf) {
        ccl_list_row(buf, bits, j0, incl - c, base);
        __syncwarp();
        const uint32_t nE = min(E - base, static_cast<uint32_t>(kCclEdgeBuf));
        for (uint32_t e0 = 0; e0 < nE; e0 += 32) {
          const uint32_t e = e0 + lane;
          const bool adj = e < nE && adjacent(b, sp, mi, ni, buf[e]);
          const unsigned bal = __ballot_sync(0xffffffffu, adj);
          if (bal) {  // candidates ascend with e: the first adjacent one is the minimum
            best = buf[e0 + __ffs(bal) - 1];
            break;
          }
        }
        __syncwarp();
      }
    }
    if (lane == 0) {
      b.parent[i] = best;
      b.cnt[i] = 0;
      b.cid[i] = -1;
    }
  }
}

// Phase 2: every forward edge (i, j > i) as a union, candidates spread over
// the lanes. Each lane keeps its own view of root(i) (an ancestor: roots only
// move down); the lanes pool the smallest after every batch.
__device__ __forceinline__ void ccl_union_bal_body(Counters* ctr, const SegDev& sp, const SegBufs& b,
                                                   const MapDesc& m) {
  __shared__ int32_t cand[kCclWarps][kCclEdgeBuf];
  const uint32_t S = min(ctr->S, b.Scap);
  const int w = sp.w, span = 2 * w + 1;
  const int nrows = (w + 1) + w * span;
  int32_t* parent = b.parent;
  const unsigned lane = lane_id();
  int32_t* buf = cand[threadIdx.x >> 5];
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarp = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = warp; i < S; i += nwarp) {
    const int x = __ldg(b.st_idx + 3 * i), y = __ldg(b.st_idx + 3 * i + 1), z = __ldg(b.st_idx + 3 * i + 2);
    int ri = -1;
    if (lane == 0) ri = uf_find(parent, static_cast<int>(i));
    const d3 mi = mk3(__ldg(b.st_mean + 3 * i), __ldg(b.st_mean + 3 * i + 1), __ldg(b.st_mean + 3 * i + 2));
    const d3 ni = mk3(__ldg(b.st_normal + 3 * i), __ldg(b.st_normal + 3 * i + 1),
                      __ldg(b.st_normal + 3 * i + 2));
    for (int r0 = 0; r0 < nrows; r0 += 64) {
      // two rows per lane per pass (the forward half has 61 rows at w = 5)
      int ja = 0, jb = 0;
      const int ra = r0 + static_cast<int>(lane), rb = ra + 32;
      const uint32_t ba = ra < nrows ? ccl_row_bits(m, w, span, ra, false, x, y, z, ja) : 0u;
      const uint32_t bb = rb < nrows ? ccl_row_bits(m, w, span, rb, false, x, y, z, jb) : 0u;
      const uint32_t ca = __popc(ba), c = ca + __popc(bb);
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (static_cast<int>(lane) >= o) incl += t;
      }
      const uint32_t E = __shfl_sync(0xffffffffu, incl, 31);
      ri = __reduce_min_sync(0xffffffffu, ri < 0 ? 0x7fffffff : ri);
      for (uint32_t base = 0; base < E; base += kCclEdgeBuf) {
        ccl_list_row(buf, ba, ja, incl - c, base);
        ccl_list_row(buf, bb, jb, incl - c + ca, base);
        __syncwarp();
        const uint32_t nE = min(E - base, static_cast<uint32_t>(kCclEdgeBuf));
        for (uint32_t e = lane; e < nE; e += 32) {
          const int j = buf[e];
          // L1-cached early-out: a stale parent[j] is an earlier ancestor of j;
          // if it equals ri, i and j were already in one set (sets only merge)
          const int pj = __ldca(parent + j);
          if (pj == ri) continue;
          if (!adjacent(b, sp, mi, ni, j)) continue;
          const int rj = uf_find(parent, j);
          if (rj == ri) continue;
          ri = uf_link(parent, ri, rj);
        }
        __syncwarp();
        ri = __reduce_min_sync(0xffffffffu, ri);
      }
    }
  }
}

__global__ void __launch_bounds__(256) k_ccl_union_bal(Counters* ctr, SegDev sp, SegBufs b, MapDesc m) {
  VP_GRID_WAIT();
  ccl_union_bal_body(ctr, sp, b, m);
}

// ---------------------------------------------------------------------------
// Default CCL after the hook: the hook forest is compressed exactly (every
// parent[i] = its tree's root), then
//  k_ccl_pairs        every forward edge (i, j) whose endpoints lie in
//                     different trees is listed once as a root pair -- no
//                     unions, no pointer chasing, only the 4-byte parent[j]
//                     per candidate (C2 frame 10: 2.4 M forward edges, 31 hook
//                     trees, 11 components: ~20 distinct pairs);
//  k_ccl_pairs_union  one block unions the listed root pairs (larger root
//                     under smaller, so each root stays the component minimum),
//                     or runs the full edge-balanced union if the pair table
//                     overflowed.
// k_ccl_flatten then resolves each voxel's root through the (short) root links.
// ---------------------------------------------------------------------------
// Pointer chasing to the root with no intermediate writes, then one write of
// the thread's own entry: every parent[i] ends exactly at its root (the
// path-halving find of k_ccl_compress can leave a node at a non-root ancestor
// when two threads rewrite it).
__global__ void k_ccl_compress_exact(Counters* ctr, SegBufs b) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
    int r = __ldcg(b.parent + i);
    for (;;) {
      const int n = __ldcg(b.parent + r);
      if (n >= r) break;
      r = n;
    }
    __stcg(b.parent + i, r);
  }
}

constexpr unsigned long long kPairEmpty = ~0ull;

__device__ __forceinline__ void pair_insert(Counters* ctr, const SegBufs& b, int ra, int rb) {
  const uint32_t lo = static_cast<uint32_t>(min(ra, rb)), hi = static_cast<uint32_t>(max(ra, rb));
  const unsigned long long key = (static_cast<unsigned long long>(hi) << 32) | lo;
  const uint32_t mask = b.pair_cap - 1u;
  uint32_t h = static_cast<uint32_t>((key * 0x9E3779B97F4A7C15ull) >> 40) & mask;
  for (uint32_t probe = 0; probe <= mask; ++probe, h = (h + 1u) & mask) {
    const unsigned long long cur = __ldcg(b.pair_key + h);
    if (cur == key) return;
    if (cur != kPairEmpty) continue;
    const unsigned long long old = atomicCAS(b.pair_key + h, kPairEmpty, key);
    if (old == kPairEmpty) {
      const uint32_t n = atomicAdd(&ctr->npairs, 1u);
      if (n < (b.pair_cap >> 1)) b.pair_slot[n] = h; else atomicOr(&ctr->pair_ovf, 1u);
      return;
    }
    if (old == key) return;
  }
  atomicOr(&ctr->pair_ovf, 1u);
}

__global__ void __launch_bounds__(256) k_ccl_pairs(Counters* ctr, SegDev sp, SegBufs b, MapDesc m) {
  VP_GRID_WAIT();
  __shared__ int32_t cand[kCclWarps][kCclEdgeBuf];
  const uint32_t S = min(ctr->S, b.Scap);
  const int w = sp.w, span = 2 * w + 1;
  const int nrows = (w + 1) + w * span;
  const int32_t* parent = b.parent;
  const unsigned lane = lane_id();
  int32_t* buf = cand[threadIdx.x >> 5];
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarp = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t i = warp; i < S; i += nwarp) {
    const int x = __ldg(b.st_idx + 3 * i), y = __ldg(b.st_idx + 3 * i + 1), z = __ldg(b.st_idx + 3 * i + 2);
    const int ri = __ldg(parent + i);  // exact roots: nothing writes parent in this kernel
    const d3 mi = mk3(__ldg(b.st_mean + 3 * i), __ldg(b.st_mean + 3 * i + 1), __ldg(b.st_mean + 3 * i + 2));
    const d3 ni = mk3(__ldg(b.st_normal + 3 * i), __ldg(b.st_normal + 3 * i + 1),
                      __ldg(b.st_normal + 3 * i + 2));
    int last = ri;  // the last tree this lane listed a pair with (for this voxel)
    for (int r0 = 0; r0 < nrows; r0 += 64) {
      int ja = 0, jb = 0;
      const int ra = r0 + static_cast<int>(lane), rb = ra + 32;
      const uint32_t ba = ra < nrows ? ccl_row_bits(m, w, span, ra, false, x, y, z, ja) : 0u;
      const uint32_t bb = rb < nrows ? ccl_row_bits(m, w, span, rb, false, x, y, z, jb) : 0u;
      const uint32_t ca = __popc(ba), c = ca + __popc(bb);
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (static_cast<int>(lane) >= o) incl += t;
      }
      const uint32_t E = __shfl_sync(0xffffffffu, incl, 31);
      for (uint32_t base = 0; base < E; base += kCclEdgeBuf) {
        ccl_list_row(buf, ba, ja, incl - c, base);
        ccl_list_row(buf, bb, jb, incl - c + ca, base);
        __syncwarp();
        const uint32_t nE = min(E - base, static_cast<uint32_t>(kCclEdgeBuf));
        for (uint32_t e = lane; e < nE; e += 32) {
          const int j = buf[e];
          const int pj = __ldg(parent + j);
          if (pj == ri || pj == last) continue;
          if (!adjacent(b, sp, mi, ni, j)) continue;
          last = pj;
          pair_insert(ctr, b, ri, pj);
        }
        __syncwarp();
      }
    }
  }
}

// One block: union of the listed root pairs, then the table is emptied. If
// the table overflowed, the block runs the full edge-balanced union instead
// (slow -- one block -- but the table holds scap / 8 pairs: C2 frames have ~20).
__global__ void __launch_bounds__(256) k_ccl_pairs_union(Counters* ctr, SegDev sp, SegBufs b, MapDesc m) {
  VP_GRID_WAIT();
  if (ctr->pair_ovf) ccl_union_bal_body(ctr, sp, b, m);
  const uint32_t n = min(ctr->npairs, b.pair_cap >> 1);
  for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
    const unsigned long long key = __ldcg(b.pair_key + b.pair_slot[t]);
    uf_union(b.parent, static_cast<int>(key & 0xffffffffu), static_cast<int>(key >> 32));
  }
  __syncthreads();
  // the pair roots now form chains (larger root under smaller, in pair
  // order: C4's many small hook trees made them thousands deep, and every
  // voxel of k_ccl_flatten chased them): point each straight at its root
  __threadfence_block();
  for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
    const unsigned long long key = __ldcg(b.pair_key + b.pair_slot[t]);
    const int a = static_cast<int>(key & 0xffffffffu), c = static_cast<int>(key >> 32);
    __stcg(b.parent + a, uf_find(b.parent, a));
    __stcg(b.parent + c, uf_find(b.parent, c));
  }
  __syncthreads();
  if (ctr->pair_ovf) {
    for (uint32_t h = threadIdx.x; h < b.pair_cap; h += blockDim.x) b.pair_key[h] = kPairEmpty;
  } else {
    for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) b.pair_key[b.pair_slot[t]] = kPairEmpty;
  }
}


// ---------------------------------------------------------------------------
// Sampling CCL (Afforest-style) for large planar components:
//  1. k_ccl_lattice  each voxel unions with its first adjacent voxel in the
//                    +z, +y and +x neighbour columns -- on a surface sampled
//                    at the voxel pitch this already joins almost every
//                    voxel of a plane into one tree;
//  2. k_ccl_compress pointer jumping;
//  3. k_ccl_giant    the most frequent root among 1024 evenly spaced voxels;
//  4. k_ccl_full     every voxel NOT in that component unions with every
//                    adjacent voxel of its whole (2w+1)^3 window.
// Edges with both ends in the giant component are redundant (sets only
// grow); every other edge has an end that scans its whole window, and the
// predicate is symmetric, so every edge of build_adjacency is applied. The
// link rule (larger root under smaller) keeps every root the minimum ordinal
// of its set: labels stay canonical and bit-exact.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_ccl_lattice(Counters* ctr, SegDev sp, SegBufs b, MapDesc m) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  int32_t* parent = b.parent;
  const int xmax = m.lo[0] + m.dims[0] - 1, ymax = m.lo[1] + m.dims[1] - 1;
  const int zmin = m.lo[2], zmax = m.lo[2] + m.dims[2] - 1;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
    const int x = __ldg(b.st_idx + 3 * i), y = __ldg(b.st_idx + 3 * i + 1), z = __ldg(b.st_idx + 3 * i + 2);
    const d3 mi = mk3(__ldg(b.st_mean + 3 * i), __ldg(b.st_mean + 3 * i + 1), __ldg(b.st_mean + 3 * i + 2));
    const d3 ni = mk3(__ldg(b.st_normal + 3 * i), __ldg(b.st_normal + 3 * i + 1),
                      __ldg(b.st_normal + 3 * i + 2));
    // neighbour sampling: at most one union per direction (+z, +y, +x), with
    // the first adjacent voxel of the 3-cell column (z-1..z+1) that way -- a
    // surface sampled at the voxel pitch is then one spanning structure
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int X = x + (r == 2 ? 1 : 0), Y = y + (r == 1 ? 1 : 0);
      if (X > xmax || Y > ymax) continue;
      const int z0 = r == 0 ? z + 1 : max(z - 1, zmin);
      const int z1 = min(z + 1, zmax);
      if (z0 > z1) continue;
      uint32_t bits = m.row_span(X, Y, z0, z1 - z0 + 1);
      if (!bits) continue;
      int j = __ldg(m.map + m.slot(X, Y, z0 + __ffs(bits) - 1)) - 1;
      while (bits) {
        bits &= bits - 1;
        ++j;
        if (adjacent(b, sp, mi, ni, j)) {
          uf_union(parent, static_cast<int>(i), j);
          break;
        }
      }
    }
  }
}

// Single block: the most frequent root among up to 1024 evenly spaced voxels
// (ties to the smaller root) -> ctr->ccl_giant (-1 if there are no voxels).
__global__ void __launch_bounds__(1024) k_ccl_giant(Counters* ctr, SegBufs b) {
  VP_GRID_WAIT();
  __shared__ int32_t v[1024];
  __shared__ unsigned long long best;
  const uint32_t S = min(ctr->S, b.Scap);
  const uint32_t k = min(S, 1024u);
  const uint32_t t = threadIdx.x;
  if (t == 0) best = ~0ull;
  v[t] = t < k ? __ldcg(b.parent + static_cast<uint32_t>((static_cast<uint64_t>(t) * S) / k)) : 0x7fffffff;
  __syncthreads();
  for (uint32_t q = 2; q <= 1024; q <<= 1) {  // bitonic sort, ascending
    for (uint32_t j = q >> 1; j > 0; j >>= 1) {
      const uint32_t l = t ^ j;
      if (l > t) {
        const int32_t a = v[t], c = v[l];
        if (((t & q) == 0) ? (a > c) : (a < c)) {
          v[t] = c;
          v[l] = a;
        }
      }
      __syncthreads();
    }
  }
  if (t < k && (t == 0 || v[t - 1] != v[t])) {  // run start: its length by binary search
    uint32_t lo = t, hi = k;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (v[mid] == v[t]) lo = mid + 1; else hi = mid;
    }
    // max count, then min root: pack (1024 - count) in the high bits
    const unsigned long long key = (static_cast<unsigned long long>(1024u - (lo - t)) << 32) |
                                   static_cast<uint32_t>(v[t]);
    atomicMin(&best, key);
  }
  __syncthreads();
  if (t == 0) ctr->ccl_giant = k ? static_cast<int32_t>(best & 0xffffffffu) : -1;
}

// Whole-window unions of every voxel outside the giant component (one warp
// per voxel, one window row per lane).
__global__ void __launch_bounds__(256) k_ccl_full(Counters* ctr, SegDev sp, SegBufs b, MapDesc m) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  const int w = sp.w, span = 2 * w + 1;
  const int nrows = span * span;
  const int32_t giant = ctr->ccl_giant;
  int32_t* parent = b.parent;
  const unsigned lane = lane_id();
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarp = (gridDim.x * blockDim.x) >> 5;
  const int xmin = m.lo[0], xmax = m.lo[0] + m.dims[0] - 1, ymin = m.lo[1], ymax = m.lo[1] + m.dims[1] - 1;
  const int zmin = m.lo[2], zmax = m.lo[2] + m.dims[2] - 1;
  for (uint32_t i = warp; i < S; i += nwarp) {
    // the skip test must be warp-uniform (lanes arrive here at different
    // times while other warps relink i): lane 0 decides for the warp
    int pi = 0;
    if (lane == 0) pi = __ldcg(parent + i);
    if (__shfl_sync(0xffffffffu, pi, 0) == giant) continue;
    const int x = __ldg(b.st_idx + 3 * i), y = __ldg(b.st_idx + 3 * i + 1), z = __ldg(b.st_idx + 3 * i + 2);
    const d3 mi = mk3(__ldg(b.st_mean + 3 * i), __ldg(b.st_mean + 3 * i + 1), __ldg(b.st_mean + 3 * i + 2));
    const d3 ni = mk3(__ldg(b.st_normal + 3 * i), __ldg(b.st_normal + 3 * i + 1),
                      __ldg(b.st_normal + 3 * i + 2));
    int ri = -1;
    if (lane == 0) ri = uf_find(parent, static_cast<int>(i));
    ri = __shfl_sync(0xffffffffu, ri, 0);
    for (int r = static_cast<int>(lane); r < nrows; r += 32) {
      const int dx = r / span - w, dy = r % span - w;
      const int X = x + dx, Y = y + dy;
      if (X < xmin || X > xmax || Y < ymin || Y > ymax) continue;
      const int z0 = max(z - w, zmin);
      const int z1 = min(z + w, zmax);
      uint32_t bits = m.row_span(X, Y, z0, z1 - z0 + 1);
      if (!bits) continue;
      // voxels of one (X, Y) column are consecutive ordinals: one map load
      int j = __ldg(m.map + m.slot(X, Y, z0 + __ffs(bits) - 1)) - 1;
      while (bits) {
        bits &= bits - 1;
        ++j;
        if (j == static_cast<int>(i)) continue;
        const int pj = __ldcg(parent + j);
        if (pj == ri) continue;  // already in i's tree
        if (!adjacent(b, sp, mi, ni, j)) continue;
        const int rj = uf_find(parent, j);
        if (rj == ri) continue;
        ri = uf_link(parent, ri, rj);
      }
    }
  }
}

// build_adjacency materialised (segmentation.cpp:112-130) for the API:
// pass 1 (cols == nullptr) counts, pass 2 fills rows in ascending ordinal order.
__global__ void k_adjacency(Counters* ctr, SegDev sp, SegBufs b, MapDesc m, const uint64_t* rows,
                            uint32_t* counts, int32_t* cols) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  const int w = sp.w;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
    const int x = b.st_idx[3 * i], y = b.st_idx[3 * i + 1], z = b.st_idx[3 * i + 2];
    const d3 mi = mk3(b.st_mean[3 * i], b.st_mean[3 * i + 1], b.st_mean[3 * i + 2]);
    const d3 ni = mk3(b.st_normal[3 * i], b.st_normal[3 * i + 1], b.st_normal[3 * i + 2]);
    uint64_t k = cols ? rows[i] : 0;
    uint32_t c = 0;
    for (int X = max(x - w, m.lo[0]); X <= min(x + w, m.lo[0] + m.dims[0] - 1); ++X)
      for (int Y = max(y - w, m.lo[1]); Y <= min(y + w, m.lo[1] + m.dims[1] - 1); ++Y)
        for (int Z = max(z - w, m.lo[2]); Z <= min(z + w, m.lo[2] + m.dims[2] - 1); ++Z) {
          const int j = m.map[m.slot(X, Y, Z)];
          if (j < 0 || j == static_cast<int>(i)) continue;
          const d3 mj = mk3(b.st_mean[3 * j], b.st_mean[3 * j + 1], b.st_mean[3 * j + 2]);
          if (sqn3(sub3(mi, mj)) >= sp.d2_th) continue;
          const d3 nj = mk3(b.st_normal[3 * j], b.st_normal[3 * j + 1], b.st_normal[3 * j + 2]);
          if (dot3(ni, nj) <= sp.cos_th) continue;
          if (cols) cols[k++] = j;
          ++c;
        }
    if (!cols) counts[i] = c;
  }
}

// OccupiedVoxel materialisation (voxel_grid.cpp:254-263) for the API.
__global__ void k_occ_gather(GridDesc g, const FrameParams* __restrict__ fp, Counters* ctr,
                             SegBufs b) {
  VP_GRID_WAIT();
  const uint32_t V = min(ctr->V, b.Vcap);
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
    const uint32_t flat = b.occ_list[v];
    const uint32_t rr = fdiv(flat, g.fez);
    const int z = static_cast<int>(flat - rr * static_cast<uint32_t>(g.ez));
    const uint32_t xr = fdiv(rr, g.fey);
    const int y = static_cast<int>(rr - xr * static_cast<uint32_t>(g.ey));
    const int x = static_cast<int>(xr);
    const Cell* c = g.cells + phys_index(g, fp->off_post, x, y, z);
    const double cd = static_cast<double>(c->count);
    b.own_mean[3 * v] = c->sx / cd;
    b.own_mean[3 * v + 1] = c->sy / cd;
    b.own_mean[3 * v + 2] = c->sz / cd;
    b.own_count[v] = c->count;
    b.own_status[v] = c->status;
  }
}

// Final labels (component minimum), member counts per root, map reset.
__global__ void k_ccl_flatten(Counters* ctr, SegBufs b, MapDesc m) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  int32_t* parent = b.parent;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // pair set consumed (k_ccl_pairs_union / _gated ran before)
    ctr->npairs = 0;
    ctr->pair_ovf = 0;
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
    const int r = uf_find(parent, static_cast<int>(i));
    b.label[i] = r;
    atomic_inc_agg(b.cnt, r);
    const int x = b.st_idx[3 * i], y = b.st_idx[3 * i + 1], z = b.st_idx[3 * i + 2];
    m.map[m.slot(x, y, z)] = -1;
    m.bits[m.word(x, y, z)] = 0u;  // every bit of the word belongs to a steppable voxel being reset
  }
}

// filter_clusters (segmentation.cpp:196-201): roots with >= min_cluster members.
__global__ void k_cluster_flags(Counters* ctr, SegDev sp, SegBufs b) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x)
    b.big_flag[i] = (b.label[i] == static_cast<int32_t>(i) && b.cnt[i] > 0u &&
                     static_cast<long long>(b.cnt[i]) >= static_cast<long long>(sp.min_cluster))
                        ? 1
                        : 0;
}

__device__ __forceinline__ void cluster_setup_body(Counters* ctr, const SegBufs& b);

__global__ void k_cluster_assign(Counters* ctr, SegBufs b) {
  VP_GRID_WAIT();
  const uint32_t S = min(ctr->S, b.Scap);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
    if (!b.big_flag[i]) continue;
    const uint32_t k = b.big_pos[i];
    if (k < b.Kcap) {
      b.klabel[k] = static_cast<int32_t>(i);
      b.cid[i] = static_cast<int32_t>(k);
    }
  }
  if (last_block_done(&ctr->scan_done[5])) cluster_setup_body(ctr, b);  // sizes, member offsets
}

// Single block: sizes and warp-padded member offsets of the K clusters (the
// last block of k_cluster_assign).
__device__ __forceinline__ void cluster_setup_body(Counters* ctr, const SegBufs& b) {
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) {
    carry = 0;
    // more clusters than the buffers hold, or a member-sort histogram above
    // Hcap: the host grows both (grow_k) and re-runs the chain
    const uint64_t nch = (static_cast<uint64_t>(min(ctr->S, b.Scap)) + kChunk - 1) / kChunk;
    if (ctr->K > b.Kcap || static_cast<uint64_t>(min(ctr->K, b.Kcap)) * nch > b.Hcap)
      atomicOr(&ctr->overflow, kOverflowClusters);
  }
  __syncthreads();
  const uint32_t K = min(ctr->K, b.Kcap);
  for (uint32_t base = 0; base < K; base += blockDim.x) {
    const uint32_t k = base + threadIdx.x;
    uint32_t padded = 0;
    if (k < K) {
      const uint32_t s = b.cnt[b.klabel[k]];
      b.ksize[k] = s;
      padded = (s + 31u) & ~31u;
    }
    const uint32_t ex = block_exclusive_u32(padded);
    const uint32_t c = carry;
    if (k < K) b.kpoff[k] = c + ex;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = c + ex + padded;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    b.kpoff[K] = carry;
    ctr->padded_members = carry;
    if (carry > b.Mcap) atomicOr(&ctr->overflow, kOverflowMembers);
  }
}

// Stable counting sort of cluster members by cluster index (ascending
// ordinal inside each cluster = segmentation.cpp:182-193 grouping order).
// One warp per chunk of kChunk ordinals.
__global__ void k_member_hist(Counters* ctr, SegBufs b, uint32_t hstride) {
  VP_GRID_WAIT();
  __shared__ uint32_t hist[kClusterBins];
  if (ctr->overflow & kOverflowClusters) return;
  const uint32_t S = min(ctr->S, b.Scap);
  const uint32_t K = min(ctr->K, b.Kcap);
  const uint32_t nch = (S + kChunk - 1) / kChunk;
  // up to kClusterBins clusters: per-chunk bins in shared memory; more: the
  // chunk's column of H itself (H[k * nch + c], this warp its only writer)
  const bool big = K > static_cast<uint32_t>(kClusterBins);
  const uint32_t hs = big ? nch : hstride;
  for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
    uint32_t* col = big ? b.H + c : hist;
    const uint32_t step = big ? hs : 1u;
    for (uint32_t k = threadIdx.x; k < K; k += blockDim.x) col[static_cast<uint64_t>(k) * step] = 0;
    __syncwarp();
    const uint32_t e1 = min(S, (c + 1) * kChunk);
    for (uint32_t e = c * kChunk + threadIdx.x; e < e1; e += blockDim.x) {
      const int32_t k = b.cid[b.label[e]];
      if (k >= 0) atomicAdd(&col[static_cast<uint64_t>(k) * step], 1u);
    }
    __syncwarp();
    if (!big)
      for (uint32_t k = threadIdx.x; k < K; k += blockDim.x) b.H[static_cast<uint64_t>(k) * hs + c] = hist[k];
    __syncwarp();
  }
}

__global__ void k_member_hscan(Counters* ctr, SegBufs b, uint32_t hstride) {
  VP_GRID_WAIT();
  if (ctr->overflow & kOverflowClusters) return;
  const uint32_t S = min(ctr->S, b.Scap);
  const uint32_t K = min(ctr->K, b.Kcap);
  const uint32_t nch = (S + kChunk - 1) / kChunk;
  const uint64_t hs = K > static_cast<uint32_t>(kClusterBins) ? nch : hstride;  // k_member_hist's layout
  const unsigned lane = lane_id();
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarp = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t k = warp; k < K; k += nwarp) {
    uint32_t run = b.kpoff[k];
    for (uint32_t c0 = 0; c0 < nch; c0 += 32) {
      const uint32_t c = c0 + lane;
      const uint32_t v = c < nch ? b.H[k * hs + c] : 0u;
      uint32_t incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (static_cast<int>(lane) >= o) incl += t;
      }
      if (c < nch) b.H[k * hs + c] = run + incl - v;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

__global__ void k_member_scatter(Counters* ctr, SegBufs b, uint32_t hstride) {
  VP_GRID_WAIT();
  __shared__ uint32_t run_s[kClusterBins];
  if (ctr->overflow & kOverflowClusters) return;
  const uint32_t S = min(ctr->S, b.Scap);
  const uint32_t K = min(ctr->K, b.Kcap);
  const uint32_t nch = (S + kChunk - 1) / kChunk;
  const bool ok = !(ctr->overflow & kOverflowMembers);
  const unsigned lane = lane_id();
  // up to kClusterBins clusters: the chunk's running offsets in shared memory;
  // more: in the chunk's column of H (this warp its only reader and writer)
  const bool big = K > static_cast<uint32_t>(kClusterBins);
  for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
    uint32_t* run = big ? b.H + c : run_s;
    const uint64_t step = big ? nch : 1u;
    if (!big)
      for (uint32_t k = lane; k < K; k += 32) run_s[k] = b.H[static_cast<uint64_t>(k) * hstride + c];
    __syncwarp();
    const uint32_t e1 = min(S, (c + 1) * kChunk);
    for (uint32_t e0 = c * kChunk; e0 < e1; e0 += 32) {
      const uint32_t e = e0 + lane;
      const int32_t k = e < e1 ? b.cid[b.label[e]] : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, k);
      const int leader = __ffs(peers) - 1;
      const uint32_t base = k >= 0 ? run[k * step] : 0u;
      __syncwarp();
      if (k >= 0 && static_cast<int>(lane) == leader) run[k * step] = base + __popc(peers);
      __syncwarp();
      if (k >= 0 && ok) {
        const uint32_t pos = base + __popc(peers & lanemask_lt());
        b.mx[pos] = b.st_mean[3 * e];
        b.my[pos] = b.st_mean[3 * e + 1];
        b.mz[pos] = b.st_mean[3 * e + 2];
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// fit_planes (plane_fit.cpp:55-131), cluster-parallel.
// (a) one thread per (cluster, iteration): CounterRng(seed, label, it) draws,
//     cross product, area gate, orient_up -> candidate (bit-exact);
// (b) one warp per 32-member segment: every candidate's predicate over the
//     segment, __ballot_sync + __popc, integer atomics (order independent);
// (c) one warp per cluster: argmax, ties to the lowest iteration;
//     ordered inlier extraction (block scan) in member order.
// ---------------------------------------------------------------------------
__global__ void k_ransac_hyp(Counters* ctr, RansacDev rp, SegBufs b) {
  VP_GRID_WAIT();
  const uint32_t K = min(ctr->K, b.Kcap);
  const uint32_t I = static_cast<uint32_t>(rp.iterations);
  const uint64_t total = static_cast<uint64_t>(K) * I;
  if (ctr->overflow & kOverflowMembers) return;
  for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t k = static_cast<uint32_t>(t / I), it = static_cast<uint32_t>(t % I);
    const uint32_t M = b.ksize[k];
    b.cand_cnt[t] = -1;
    if (M < 3) continue;
    CounterRng rng(rp.seed, static_cast<uint64_t>(static_cast<uint32_t>(b.klabel[k])),
                   static_cast<uint64_t>(it));
    const uint32_t ia = rng.below(M);
    uint32_t ib = rng.below(M);
    while (ib == ia) ib = rng.below(M);
    uint32_t ic = rng.below(M);
    while (ic == ia || ic == ib) ic = rng.below(M);
    const uint32_t o = b.kpoff[k];
    const d3 p0 = mk3(b.mx[o + ia], b.my[o + ia], b.mz[o + ia]);
    const d3 e1 = sub3(mk3(b.mx[o + ib], b.my[o + ib], b.mz[o + ib]), p0);
    const d3 e2 = sub3(mk3(b.mx[o + ic], b.my[o + ic], b.mz[o + ic]), p0);
    const d3 cr = cross3(e1, e2);
    const double norm = sqrt(sqn3(cr));
    if (0.5 * norm <= 1e-10) continue;  // area gate (plane_fit.cpp:38)
    const d3 n = orient_up(div3(cr, norm), rp.up);
    b.cand[4 * t] = n.x;
    b.cand[4 * t + 1] = n.y;
    b.cand[4 * t + 2] = n.z;
    b.cand[4 * t + 3] = dot3(n, p0);
    b.cand_cnt[t] = 0;
  }
}

__global__ void k_ransac_count(Counters* ctr, RansacDev rp, SegBufs b) {
  VP_GRID_WAIT();
  const uint32_t K = min(ctr->K, b.Kcap);
  if (K == 0 || (ctr->overflow & kOverflowMembers)) return;
  const uint32_t nseg = b.kpoff[K] >> 5;
  const uint32_t I = static_cast<uint32_t>(rp.iterations);
  const unsigned lane = lane_id();
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarp = (gridDim.x * blockDim.x) >> 5;
  // one warp per (32-member segment, 32 candidates): C2's ~850 segments x 100
  // candidates as ~3400 independent warps instead of 850 long loops
  const uint32_t ncb = (I + 31) >> 5;
  for (uint32_t wi = warp; wi < nseg * ncb; wi += nwarp) {
    const uint32_t sg = wi / ncb, cb = wi - sg * ncb;
    const uint32_t start = sg << 5;
    uint32_t lo = 0, hi = K;  // largest k with kpoff[k] <= start
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (b.kpoff[mid] <= start) lo = mid; else hi = mid;
    }
    const uint32_t k = lo;
    const uint32_t M = b.ksize[k];
    if (M < 3) continue;
    const uint32_t j = start + lane - b.kpoff[k];
    const bool in = j < M;
    const d3 p = in ? mk3(b.mx[start + lane], b.my[start + lane], b.mz[start + lane])
                    : mk3(0.0, 0.0, 0.0);
    const uint64_t cbase = static_cast<uint64_t>(k) * I;
    {
      const uint32_t c0 = cb << 5;
      // candidate c0 + lane held by this lane, broadcast by shuffles
      const uint32_t mine_t = c0 + lane;
      int valid = 0;
      double cx = 0.0, cy = 0.0, cz = 0.0, cd = 0.0;
      if (mine_t < I) {
        const uint64_t t = cbase + mine_t;
        valid = b.cand_cnt[t] >= 0;
        if (valid) {
          cx = b.cand[4 * t];
          cy = b.cand[4 * t + 1];
          cz = b.cand[4 * t + 2];
          cd = b.cand[4 * t + 3];
        }
      }
      const unsigned vmask = __ballot_sync(0xffffffffu, valid);
      uint32_t mine = 0;
      unsigned rem = vmask;
      while (rem) {  // degenerate samples skipped (warp-uniform)
        const int q = __ffs(rem) - 1;
        rem &= rem - 1;
        const d3 n = mk3(__shfl_sync(0xffffffffu, cx, q), __shfl_sync(0xffffffffu, cy, q),
                         __shfl_sync(0xffffffffu, cz, q));
        const double off = __shfl_sync(0xffffffffu, cd, q);
        const bool pred = in && fabs(dot3(n, p) - off) <= rp.eps;
        const uint32_t c = __popc(__ballot_sync(0xffffffffu, pred));
        if (static_cast<int>(lane) == q) mine = c;
      }
      if (mine) atomicAdd(&b.cand_cnt[cbase + c0 + lane], static_cast<int32_t>(mine));
    }
  }
}

__device__ __forceinline__ void fit_setup_body(Counters* ctr, const RansacDev& rp, const SegBufs& b);
__device__ __forceinline__ void ransac_select_body(Counters* ctr, const RansacDev& rp, const SegBufs& b);

__global__ void k_ransac_select(Counters* ctr, RansacDev rp, SegBufs b) {
  VP_GRID_WAIT();
  ransac_select_body(ctr, rp, b);
  if (last_block_done(&ctr->scan_done[6])) fit_setup_body(ctr, rp, b);  // fit list, inlier offsets
}

__device__ __forceinline__ void ransac_select_body(Counters* ctr, const RansacDev& rp, const SegBufs& b) {
  const uint32_t K = min(ctr->K, b.Kcap);
  const int I = rp.iterations;
  const unsigned lane = lane_id();
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarp = (gridDim.x * blockDim.x) >> 5;
  const bool bad = (ctr->overflow & kOverflowMembers) != 0;
  for (uint32_t k = warp; k < K; k += nwarp) {
    if (bad || b.ksize[k] < 3) {
      if (lane == 0) {
        b.win_it[k] = -2;  // clusters_skipped_small (plane_fit.cpp:60-61)
        b.win_cnt[k] = 0;
      }
      continue;
    }
    int best = -1, bc = -1;
    for (int it = static_cast<int>(lane); it < I; it += 32) {
      const int c = b.cand_cnt[static_cast<uint64_t>(k) * I + it];
      if (c > bc) {  // strict: ties keep the lowest iteration
        bc = c;
        best = it;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const int oc = __shfl_down_sync(0xffffffffu, bc, o);
      const int ob = __shfl_down_sync(0xffffffffu, best, o);
      if (oc > bc || (oc == bc && ob >= 0 && (best < 0 || ob < best))) {
        bc = oc;
        best = ob;
      }
    }
    if (lane == 0) {
      b.win_it[k] = bc >= 0 ? best : -1;
      b.win_cnt[k] = bc >= 0 ? bc : 0;
    }
  }
}

// Single block: fit list in cluster order, inlier offsets, FitStats (the last
// block of k_ransac_select).
__device__ __forceinline__ void fit_setup_body(Counters* ctr, const RansacDev& rp, const SegBufs& b) {
  __shared__ uint32_t carry_f, carry_i, n_skip, n_unfit;
  if (threadIdx.x == 0) carry_f = carry_i = n_skip = n_unfit = 0;
  __syncthreads();
  const uint32_t K = min(ctr->K, b.Kcap);
  for (uint32_t base = 0; base < K; base += blockDim.x) {
    const uint32_t k = base + threadIdx.x;
    int w = -3;
    if (k < K) w = b.win_it[k];
    const uint32_t fitted = (w >= 0) ? 1u : 0u;
    const uint32_t cnt = fitted ? static_cast<uint32_t>(b.win_cnt[k]) : 0u;
    if (w == -2) atomicAdd(&n_skip, 1u);
    if (w == -1) atomicAdd(&n_unfit, 1u);
    const uint32_t ef = block_exclusive_u32(fitted);
    const uint32_t ei = block_exclusive_u32(cnt);
    const uint32_t cf = carry_f, ci = carry_i;
    if (k < K) {
      b.fid[k] = fitted ? static_cast<int32_t>(cf + ef) : -1;
      if (fitted) {
        const uint32_t f = cf + ef;
        const uint64_t t = static_cast<uint64_t>(k) * rp.iterations + w;
#pragma unroll
        for (int q = 0; q < 4; ++q) b.fit_model[4 * f + q] = b.cand[4 * t + q];
        b.fit_meta[2 * f] = b.win_cnt[k];
        b.fit_meta[2 * f + 1] = b.klabel[k];
        b.fit_cluster[f] = k;
        b.ioff[f] = ci + ei;
      }
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) {
      carry_f = cf + ef + fitted;
      carry_i = ci + ei + cnt;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    ctr->nfits = carry_f;
    ctr->inliers = carry_i;
    b.ioff[carry_f] = carry_i;
    // member chunks of the fits (for the multi-block ordered extraction)
    uint32_t ch = 0;
    for (uint32_t f = 0; f < carry_f; ++f) {
      b.fch_off[f] = ch;
      ch += (b.ksize[b.fit_cluster[f]] + kPolyChunk - 1) / kPolyChunk;
    }
    b.fch_off[carry_f] = ch;
    ctr->fit_chunks = ch;
    ctr->skipped = n_skip;
    ctr->unfit = n_unfit;
    if (carry_i > b.Icap) atomicOr(&ctr->overflow, kOverflowFits);
  }
}

// Ordered inlier extraction (plane_fit.cpp:102-104) over member chunks of
// kPolyChunk: count per chunk, one exclusive scan over all chunks (fits and
// their inliers are both concatenated in fit order), then a block-ordered
// write per chunk.
__device__ __forceinline__ uint32_t fit_of_chunk(const SegBufs& b, uint32_t F, uint32_t c) {
  uint32_t lo = 0, hi = F;
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (b.fch_off[mid] <= c) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void k_extract_count(Counters* ctr, RansacDev rp, SegBufs b) {
  VP_GRID_WAIT();
  if (ctr->overflow & (kOverflowFits | kOverflowMembers)) return;
  const uint32_t F = ctr->nfits, nch = ctr->fit_chunks;
  for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const uint32_t f = fit_of_chunk(b, F, c);
    const uint32_t k = b.fit_cluster[f];
    const uint32_t M = b.ksize[k], o = b.kpoff[k];
    const uint32_t j0 = (c - b.fch_off[f]) * kPolyChunk, j1 = min(M, j0 + kPolyChunk);
    const d3 n = mk3(b.fit_model[4 * f], b.fit_model[4 * f + 1], b.fit_model[4 * f + 2]);
    const double off = b.fit_model[4 * f + 3];
    uint32_t cnt = 0;
    for (uint32_t j = j0 + threadIdx.x; j < j1; j += blockDim.x)
      cnt += fabs(dot3(n, mk3(b.mx[o + j], b.my[o + j], b.mz[o + j])) - off) <= rp.eps ? 1u : 0u;
    cnt = block_sum_u32(cnt);
    if (threadIdx.x == 0) b.ccount[c] = cnt;
  }
}

__global__ void k_extract_emit(Counters* ctr, RansacDev rp, SegBufs b) {
  VP_GRID_WAIT();
  if (ctr->overflow & (kOverflowFits | kOverflowMembers)) return;
  __shared__ uint32_t run;
  const uint32_t F = ctr->nfits, nch = ctr->fit_chunks;
  for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const uint32_t f = fit_of_chunk(b, F, c);
    const uint32_t k = b.fit_cluster[f];
    const uint32_t M = b.ksize[k], o = b.kpoff[k];
    const uint32_t j0 = (c - b.fch_off[f]) * kPolyChunk, j1 = min(M, j0 + kPolyChunk);
    const d3 n = mk3(b.fit_model[4 * f], b.fit_model[4 * f + 1], b.fit_model[4 * f + 2]);
    const double off = b.fit_model[4 * f + 3];
    if (threadIdx.x == 0) run = b.ccount[c];  // exclusive-scanned: first inlier slot
    __syncthreads();
    for (uint32_t base = j0; base < j1; base += blockDim.x) {
      const uint32_t j = base + threadIdx.x;
      d3 p = mk3(0.0, 0.0, 0.0);
      bool pred = false;
      if (j < j1) {
        p = mk3(b.mx[o + j], b.my[o + j], b.mz[o + j]);
        pred = fabs(dot3(n, p) - off) <= rp.eps;
      }
      const uint32_t ex = block_exclusive_u32(pred ? 1u : 0u);
      const uint32_t r0 = run;
      if (pred) {
        const uint64_t d = static_cast<uint64_t>(r0) + ex;
        b.inl[3 * d] = p.x;
        b.inl[3 * d + 1] = p.y;
        b.inl[3 * d + 2] = p.z;
      }
      __syncthreads();
      if (threadIdx.x == blockDim.x - 1) run = r0 + ex + (pred ? 1u : 0u);
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// refine_plane (plane_fit.cpp:133-154) via pipeline.cpp:74-78.
// exact = 1: the reference's sequential sums (one thread, bit-identical).
// exact = 0: deterministic fixed-shape tree reduction (256 strided partials,
//            pairwise tree), within the stated 1e-4 rad / 1e-4 m tolerance.
// ---------------------------------------------------------------------------
__device__ void refine_finish(double cov[3][3], d3 cen, const double* init, d3 up, double* out) {
  const Eig3 e = jacobi3(cov);
  if (e.val[1] <= 1e-12 + 1e-9 * fabs(e.val[2])) {
#pragma unroll
    for (int q = 0; q < 4; ++q) out[q] = init[q];
    return;
  }
  const d3 n = orient_up(normalized3(e.vec[0]), up);
  out[0] = n.x;
  out[1] = n.y;
  out[2] = n.z;
  out[3] = dot3(n, cen);
}

// refine_plane with the reference's sequential sums (refine_exact): one
// thread per fit, bit-identical to plane_fit.cpp:136-143.
__global__ void k_refine(Counters* ctr, SegBufs b, d3 up, int refine, int exact) {
  VP_GRID_WAIT();
  const uint32_t F = ctr->nfits;
  if (ctr->overflow & (kOverflowFits | kOverflowMembers)) return;
  for (uint32_t f = blockIdx.x; f < F; f += gridDim.x) {
    const uint64_t o = b.ioff[f];
    const uint32_t n = b.ioff[f + 1] - b.ioff[f];
    const double* init = b.fit_model + 4 * f;
    double* out = b.ref_model + 4 * f;
    if (!refine || n < 3) {
      if (threadIdx.x < 4) out[threadIdx.x] = init[threadIdx.x];
      __syncthreads();
      continue;
    }
    const double* P = b.inl + 3 * o;
    if (exact) {
      if (threadIdx.x == 0) {
        d3 s = mk3(0.0, 0.0, 0.0);
        for (uint32_t i = 0; i < n; ++i) s = add3(s, mk3(P[3 * i], P[3 * i + 1], P[3 * i + 2]));
        const d3 cen = div3(s, static_cast<double>(n));
        double c[3][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
        for (uint32_t i = 0; i < n; ++i) {
          const d3 d = sub3(mk3(P[3 * i], P[3 * i + 1], P[3 * i + 2]), cen);
          const double dv[3] = {d.x, d.y, d.z};
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int q = 0; q < 3; ++q) c[a][q] = c[a][q] + dv[q] * dv[a];
        }
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int q = 0; q < 3; ++q) c[a][q] = c[a][q] / static_cast<double>(n);
        refine_finish(c, cen, init, up, out);
      }
      __syncthreads();
      continue;
    }
  }
}

// refine_plane in tree mode, split over the GPU: chunks of kRefChunk inliers
// (one block each) reduce in a fixed-shape tree; each fit then sums its chunk
// partials in chunk order. Deterministic; within the north_star tolerance of
// the reference's sequential sums.
constexpr uint32_t kRefChunk = kRefineChunk;  // 512: C2's ~3 k-inlier fits spread over ~60 blocks instead of ~9

// Single block: per fit chunk offsets (fits that are not refined get none).
__global__ void k_refine_setup(Counters* ctr, SegBufs b, int refine) {
  VP_GRID_WAIT();
  __shared__ uint32_t carry;
  const uint32_t F = min(ctr->nfits, b.Kcap);
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < F; base += blockDim.x) {
    const uint32_t f = base + threadIdx.x;
    uint32_t c = 0;
    if (f < F) {
      const uint32_t n = b.ioff[f + 1] - b.ioff[f];
      c = (refine && n >= 3) ? (n + kRefChunk - 1) / kRefChunk : 0u;
    }
    const uint32_t ex = block_exclusive_u32(c);
    const uint32_t c0 = carry;
    if (f < F) b.rch_off[f] = c0 + ex;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = c0 + ex + c;
    __syncthreads();
  }
  if (threadIdx.x == 0) b.rch_off[F] = carry;
}

__device__ __forceinline__ uint32_t ref_fit_of_chunk(const SegBufs& b, uint32_t F, uint32_t c) {
  uint32_t lo = 0, hi = F;  // largest f with rch_off[f] <= c (skipping empty fits)
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (b.rch_off[mid] <= c) lo = mid; else hi = mid;
  }
  return lo;
}

// pass 0: per chunk sum of x, y, z; pass 1: per chunk sums of the centred
// outer products (xx, yx, zx, yy, zy, zz) about the fit's centroid.
template <int kPass>
__device__ __forceinline__ void refine_part_body(Counters* ctr, SegBufs b) {
  constexpr int B = 256;
  constexpr int NQ = kPass == 0 ? 3 : 6;
  __shared__ double red[NQ][B];
  const uint32_t F = min(ctr->nfits, b.Kcap);
  if (ctr->overflow & (kOverflowFits | kOverflowMembers)) return;
  const uint32_t total = b.rch_off[F];
  for (uint32_t c = blockIdx.x; c < total; c += gridDim.x) {
    const uint32_t f = ref_fit_of_chunk(b, F, c);
    const uint64_t o = b.ioff[f];
    const uint32_t n = b.ioff[f + 1] - b.ioff[f];
    const uint32_t i0 = (c - b.rch_off[f]) * kRefChunk;
    const uint32_t i1 = min(n, i0 + kRefChunk);
    const double* P = b.inl + 3 * o;
    double q[NQ];
#pragma unroll
    for (int k = 0; k < NQ; ++k) q[k] = 0.0;
    d3 cen = mk3(0.0, 0.0, 0.0);
    if (kPass == 1) cen = mk3(b.rcen[3 * f], b.rcen[3 * f + 1], b.rcen[3 * f + 2]);
    for (uint32_t i = i0 + threadIdx.x; i < i1; i += B) {
      if (kPass == 0) {
        q[0] += P[3 * i];
        q[1] += P[3 * i + 1];
        q[2] += P[3 * i + 2];
      } else {
        const d3 d = sub3(mk3(P[3 * i], P[3 * i + 1], P[3 * i + 2]), cen);
        q[0] += d.x * d.x;
        q[1] += d.y * d.x;
        q[2] += d.z * d.x;
        q[3] += d.y * d.y;
        q[4] += d.z * d.y;
        q[5] += d.z * d.z;
      }
    }
#pragma unroll
    for (int k = 0; k < NQ; ++k) red[k][threadIdx.x] = q[k];
    __syncthreads();
    for (int h = B / 2; h > 0; h >>= 1) {
      if (static_cast<int>(threadIdx.x) < h)
#pragma unroll
        for (int k = 0; k < NQ; ++k) red[k][threadIdx.x] = red[k][threadIdx.x] + red[k][threadIdx.x + h];
      __syncthreads();
    }
    if (threadIdx.x < NQ) b.rpart[8ull * c + threadIdx.x] = red[threadIdx.x][0];
    __syncthreads();
  }
}

__device__ __forceinline__ void refine_cen_body(const Counters* ctr, const SegBufs& b);
__device__ __forceinline__ void refine_fin_body(const Counters* ctr, const SegBufs& b, d3 up);

// Each pass's last block to finish runs the per-fit step that needs all of
// the fit's chunk partials: centroids after pass 0, covariance -> Jacobi ->
// model after pass 1 (one launch each fewer).
__global__ void __launch_bounds__(256) k_refine_part0(Counters* ctr, SegBufs b) {
  VP_GRID_WAIT();
  refine_part_body<0>(ctr, b);
  if (last_block_done(&ctr->scan_done[3]) && !(ctr->overflow & (kOverflowFits | kOverflowMembers)))
    refine_cen_body(ctr, b);
}
__global__ void __launch_bounds__(256) k_refine_part1(Counters* ctr, SegBufs b, d3 up) {
  VP_GRID_WAIT();
  refine_part_body<1>(ctr, b);
  if (last_block_done(&ctr->scan_done[4]) && !(ctr->overflow & (kOverflowFits | kOverflowMembers)))
    refine_fin_body(ctr, b, up);
}

// The fits' chunk partials are summed in the last block of each pass: one
// thread per fit in chunk order, or -- for a fit with more than kRefSerial
// chunks (a C5 floor has ~1500) -- the whole block: thread t sums chunks
// t, t + 256, .. in order, then a fixed 256-leaf tree. The shape depends only
// on the chunk count, so the result is deterministic.
constexpr uint32_t kRefSerial = 64;

template <int NQ>
__device__ __forceinline__ void refine_block_sum(const double* rpart, uint32_t c0, uint32_t c1, double* out) {
  __shared__ double red[NQ][256];
  double q[NQ];
#pragma unroll
  for (int k = 0; k < NQ; ++k) q[k] = 0.0;
  for (uint32_t c = c0 + threadIdx.x; c < c1; c += 256)
#pragma unroll
    for (int k = 0; k < NQ; ++k) q[k] += __ldcg(rpart + 8ull * c + k);
#pragma unroll
  for (int k = 0; k < NQ; ++k) red[k][threadIdx.x] = q[k];
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (static_cast<int>(threadIdx.x) < h)
#pragma unroll
      for (int k = 0; k < NQ; ++k) red[k][threadIdx.x] = red[k][threadIdx.x] + red[k][threadIdx.x + h];
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < NQ; ++k) out[k] = red[k][0];
  __syncthreads();
}

// Calls fn(f, sums) for every fit: serial sums by the fit's thread, block sums
// for the large fits (batches of 256 fits, large ones listed in fit order).
template <int NQ, class Fn>
__device__ __forceinline__ void refine_fit_sums(const SegBufs& b, uint32_t F, Fn fn) {
  __shared__ uint32_t big[256];
  __shared__ uint32_t nbig;
  for (uint32_t base = 0; base < F; base += 256) {
    const uint32_t f = base + threadIdx.x;
    uint32_t c0 = 0, c1 = 0;
    if (f < F) c0 = b.rch_off[f], c1 = b.rch_off[f + 1];
    const bool large = f < F && c1 - c0 > kRefSerial;
    if (f < F && !large) {
      double a[NQ];
#pragma unroll
      for (int k = 0; k < NQ; ++k) a[k] = 0.0;
      for (uint32_t c = c0; c < c1; ++c)
#pragma unroll
        for (int k = 0; k < NQ; ++k) a[k] += __ldcg(b.rpart + 8ull * c + k);
      fn(f, a, c1 - c0);
    }
    const uint32_t at = block_exclusive_u32(large ? 1u : 0u);
    if (large) big[at] = f;
    if (threadIdx.x == 255) nbig = at + (large ? 1u : 0u);
    __syncthreads();
    const uint32_t nb = nbig;
    for (uint32_t j = 0; j < nb; ++j) {
      const uint32_t g = big[j];
      double a[NQ];
      refine_block_sum<NQ>(b.rpart, b.rch_off[g], b.rch_off[g + 1], a);
      if (threadIdx.x == 0) fn(g, a, b.rch_off[g + 1] - b.rch_off[g]);
    }
    __syncthreads();
  }
}

// Per fit: centroid = (sum of chunk sums) / n (run by the last block of pass 0).
__device__ __forceinline__ void refine_cen_body(const Counters* ctr, const SegBufs& b) {
  const uint32_t F = min(ctr->nfits, b.Kcap);
  refine_fit_sums<3>(b, F, [&](uint32_t f, const double* s, uint32_t) {
    const double dn = static_cast<double>(b.ioff[f + 1] - b.ioff[f]);
    b.rcen[3 * f] = s[0] / dn;
    b.rcen[3 * f + 1] = s[1] / dn;
    b.rcen[3 * f + 2] = s[2] / dn;
  });
}

// Per fit: covariance / n -> Jacobi -> rank gate -> orient_up
// (plane_fit.cpp:133-154); unrefined fits keep the RANSAC model.
// (run by the last block of pass 1)
__device__ __forceinline__ void refine_fin_body(const Counters* ctr, const SegBufs& b, d3 up) {
  const uint32_t F = min(ctr->nfits, b.Kcap);
  refine_fit_sums<6>(b, F, [&](uint32_t f, const double* a, uint32_t nch) {
    const double* init = b.fit_model + 4 * f;
    double* out = b.ref_model + 4 * f;
    if (nch == 0) {
#pragma unroll
      for (int q = 0; q < 4; ++q) out[q] = init[q];
      return;
    }
    const double dn = static_cast<double>(b.ioff[f + 1] - b.ioff[f]);
    double cv[3][3];
    cv[0][0] = a[0] / dn;
    cv[0][1] = cv[1][0] = a[1] / dn;
    cv[0][2] = cv[2][0] = a[2] / dn;
    cv[1][1] = a[3] / dn;
    cv[1][2] = cv[2][1] = a[4] / dn;
    cv[2][2] = a[5] / dn;
    refine_finish(cv, mk3(b.rcen[3 * f], b.rcen[3 * f + 1], b.rcen[3 * f + 2]), init, up, out);
  });
}

// ---------------------------------------------------------------------------
// make_polygon (polygonize.cpp:166-182): plane_basis, projection, 16-direction
// hull_filter (extremes with the lexicographic tie-break, inner polygon),
// lexicographic sort of the survivors (shared-memory bitonic), unique,
// monotone chain, lift, shoelace. One block per fit.
// ---------------------------------------------------------------------------
// (P2, lex_less, cross2: vp_kernels.cuh)

// Monotone chain over sorted, deduplicated points (polygonize.cpp:116-139);
// returns hull size (0 if < 3). h has room for 2n points.
__device__ uint32_t chain_sorted(const P2* pts, uint32_t n, P2* h) {
  if (n < 3) return 0;
  uint32_t k = 0;
  for (uint32_t i = 0; i < n; ++i) {
    while (k >= 2 && cross2(h[k - 2], h[k - 1], pts[i]) <= 0.0) --k;
    h[k++] = pts[i];
  }
  const uint32_t lower = k + 1;
  for (uint32_t i = n - 1; i-- > 0;) {
    while (k >= lower && cross2(h[k - 2], h[k - 1], pts[i]) <= 0.0) --k;
    h[k++] = pts[i];
  }
  const uint32_t m = k - 1;
  return m < 3 ? 0 : m;
}

// The two halves of Andrew's monotone chain as independent stacks
// (polygonize.cpp:116-139): the lower chain over pts[0..n) and the upper chain
// over pts[n-1], pts[n-2], .., pts[0] starting from the stack [pts[n-1]],
// popping while it holds >= 2 points. The reference's single-array loop pops
// the upper part only down to `lower`, i.e. never below pts[n-1], so
// hull = L + U[1 .. |U|-1) is exactly its output. The top two stack entries
// live in registers (the pop loop is a serial dependency chain).
#ifdef VP_POLY_PROFILE
__device__ unsigned long long g_chain_stats[4];  // tests, points, cycles
#endif
__device__ uint32_t half_chain(const P2* pts, uint32_t n, bool upper, P2* h) {
  uint32_t k = 0;
#ifdef VP_POLY_PROFILE
  const long long c_start = clock64();
  unsigned long long ntests = 0;
#define VP_CHAIN_TEST() ++ntests
#else
#define VP_CHAIN_TEST() do {} while (0)
#endif
  // the top three stack entries live in registers (t = h[k-1], a = h[k-2],
  // a2 = h[k-3]): a pop's next test needs no shared-memory round trip, and the
  // entry below is fetched while the cross product runs; the next input
  // point is loaded one step ahead. (Profiled, VP_POLY_PROFILE, C2: ~1.75
  // tests and ~240 cycles per survivor on one warp, 278 before the running
  // input pointer; evaluating the test that follows a pop speculatively
  // alongside did not change it.)
  P2 a{0.0, 0.0}, t{0.0, 0.0}, a2{0.0, 0.0};
  if (upper) {
    t = pts[n - 1];
    h[k++] = t;
  }
  const uint32_t m = upper ? n - 1 : n;
  // the input walks pts forwards (lower) or backwards from pts[n-2] (upper):
  // one running pointer instead of re-deriving the index every point (the
  // prefetch was ~20 of the loop's ~56 instructions per point)
  const P2* src = upper ? pts + (n - 2) : pts;
  const int dir = upper ? -1 : 1;
  P2 pn = m ? *src : P2{0.0, 0.0};
  for (uint32_t q = 0; q < m; ++q) {
    const P2 p = pn;
    src += dir;
    if (q + 1 < m) pn = *src;
    while (k >= 2) {
      VP_CHAIN_TEST();
      if (!(cross2(a, t, p) <= 0.0)) break;
      --k;
      t = a;
      a = a2;
      if (k >= 3) a2 = h[k - 3];
    }
    h[k++] = p;
    a2 = a;
    a = t;
    t = p;
  }
#ifdef VP_POLY_PROFILE
  atomicAdd(&g_chain_stats[0], ntests);
  atomicAdd(&g_chain_stats[1], static_cast<unsigned long long>(m));
  atomicAdd(&g_chain_stats[2], static_cast<unsigned long long>(clock64() - c_start));
#endif
  return k;
}

// In-place bitonic sort (lexicographic) of n (power of two) points by a block.
__device__ void bitonic_sort(P2* a, uint32_t n) {
  for (uint32_t k = 2; k <= n; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const P2 x = a[i], y = a[l];
          const bool sw = up ? lex_less(y, x) : lex_less(x, y);
          if (sw) {
            a[i] = y;
            a[l] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Polygon stage as five kernels so the large fits use the whole GPU:
//  setup   (1 block)        plane_basis per fit, chunk table (kPolyChunk points)
//  extremes(block / chunk)  project_to_plane + per-chunk extremes per direction
//  inner   (block / fit)    final extremes (larger dot, ties lexicographic) and
//                           the inner polygon = monotone_chain(extremes)
//  keep    (block / chunk)  survivors: not strictly inside the inner polygon
//  hull    (block / fit)    lexicographic bitonic sort, unique, monotone chain,
//                           lift, shoelace, area filter, output record
// oi != bi: a candidate met again (shuffle-down lanes past the warp's end
// receive their own value) is not better -- without this every reduction
// step paid two global loads for the tie-break (C2 polygon stage: 15 us).
__device__ __forceinline__ bool ext_better(double od, int oi, double bd, int bi, const P2* proj) {
  return oi >= 0 && oi != bi && (bi < 0 || od > bd || (od == bd && lex_less(proj[oi], proj[bi])));
}

// Warp-wide extreme of one direction (every lane gets the result): the
// largest dot as the max of an order-preserving 64-bit key (-0.0 folded
// into +0.0 so key equality is double equality), then -- only when several
// lanes hold that dot -- the lexicographically smallest of their points.
// The same total order as ext_better, without a load per shuffle step.
__device__ __forceinline__ unsigned long long ext_key(double d) {
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(d + 0.0));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ void warp_ext_max(double& bd, int& bi, const P2* proj) {
  const unsigned long long key = ext_key(bd);
  unsigned long long m = key;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, m, o);
    m = t > m ? t : m;
  }
  const unsigned tied = __ballot_sync(0xffffffffu, bi >= 0 && key == m);
  if (!tied) {
    bd = -CUDART_INF;
    bi = -1;
    return;
  }
  int win = __ffs(tied) - 1;
  if (tied & (tied - 1)) {  // equal dots: lexicographic tie-break
    const P2 mine = bi >= 0 ? proj[bi] : P2{0.0, 0.0};
    P2 pw{__shfl_sync(0xffffffffu, mine.x, win), __shfl_sync(0xffffffffu, mine.y, win)};
    for (unsigned rest = tied & (tied - 1); rest; rest &= rest - 1) {
      const int l = __ffs(rest) - 1;
      const P2 pl{__shfl_sync(0xffffffffu, mine.x, l), __shfl_sync(0xffffffffu, mine.y, l)};
      if (lex_less(pl, pw)) {
        win = l;
        pw = pl;
      }
    }
  }
  bd = __shfl_sync(0xffffffffu, bd, win);
  bi = __shfl_sync(0xffffffffu, bi, win);
}

__device__ __forceinline__ uint32_t poly_fit_of_chunk(const SegBufs& b, uint32_t F, uint32_t c) {
  uint32_t lo = 0, hi = F;  // largest f with pch_off[f] <= c
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (b.pch_off[mid] <= c) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void k_poly_setup(Counters* ctr, SegBufs b) {
  VP_GRID_WAIT();
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const uint32_t F = (ctr->overflow & (kOverflowFits | kOverflowMembers)) ? 0u : ctr->nfits;
  for (uint32_t base = 0; base < F; base += blockDim.x) {
    const uint32_t f = base + threadIdx.x;
    uint32_t nch = 0;
    if (f < F) {
      const uint32_t n = b.ioff[f + 1] - b.ioff[f];
      nch = n >= 3 ? (n + kPolyChunk - 1) / kPolyChunk : 0u;
      b.nsurv[f] = 0;
      const double* pl = b.ref_model + 4 * f;
      const d3 nrm = mk3(pl[0], pl[1], pl[2]);
      int least = 0;  // plane_basis (polygonize.cpp:21-34)
      const double an[3] = {fabs(nrm.x), fabs(nrm.y), fabs(nrm.z)};
      if (an[1] < an[least]) least = 1;
      if (an[2] < an[least]) least = 2;
      const d3 axis = mk3(least == 0 ? 1.0 : 0.0, least == 1 ? 1.0 : 0.0, least == 2 ? 1.0 : 0.0);
      const d3 u = normalized3(sub3(axis, scl3(dot3(nrm, axis), nrm)));
      const d3 v = cross3(nrm, u);
      const d3 org = scl3(pl[3], nrm);
      double* bs = b.basis + 9 * f;
      bs[0] = u.x; bs[1] = u.y; bs[2] = u.z;
      bs[3] = v.x; bs[4] = v.y; bs[5] = v.z;
      bs[6] = org.x; bs[7] = org.y; bs[8] = org.z;
    }
    const uint32_t ex = block_exclusive_u32(nch);
    const uint32_t c0 = carry;
    if (f < F) b.pch_off[f] = c0 + ex;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = c0 + ex + nch;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    b.pch_off[F] = carry;
    ctr->poly_chunks = carry;
  }
}

// planar != 0: the points are already 2-D (x, y, 0) with the identity basis
// (the public hull_filter / monotone_chain / convex_hull): copied verbatim, so
// a -0.0 coordinate keeps its sign as in the reference (projecting would add
// +0.0 terms).
__global__ void __launch_bounds__(256) k_poly_extremes(Counters* ctr, SegBufs b, const double* dirtab,
                                                       int directions, int planar) {
  VP_GRID_WAIT();
  __shared__ double sdir[128];
  __shared__ double ex_dot[8 * 16];
  __shared__ int ex_idx[8 * 16];
  const uint32_t F = ctr->nfits, nchunks = ctr->poly_chunks;
  for (int j = threadIdx.x; j < 2 * directions && j < 128; j += blockDim.x) sdir[j] = dirtab[j];
  __syncthreads();
  P2* proj = reinterpret_cast<P2*>(b.proj);
  const unsigned lane = lane_id(), wid = threadIdx.x >> 5;
  for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint32_t f = poly_fit_of_chunk(b, F, c);
    const uint32_t n = b.ioff[f + 1] - b.ioff[f];
    const uint64_t i0 = b.ioff[f] + static_cast<uint64_t>(c - b.pch_off[f]) * kPolyChunk;
    const uint64_t i1 = min(static_cast<uint64_t>(b.ioff[f + 1]), i0 + kPolyChunk);
    const double* bs = b.basis + 9 * f;
    const d3 u = mk3(bs[0], bs[1], bs[2]), v = mk3(bs[3], bs[4], bs[5]), org = mk3(bs[6], bs[7], bs[8]);
    for (uint64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {  // project_to_plane (:36-44)
      if (planar) {
        proj[i] = P2{b.inl[3 * i], b.inl[3 * i + 1]};
        continue;
      }
      const d3 d = sub3(mk3(b.inl[3 * i], b.inl[3 * i + 1], b.inl[3 * i + 2]), org);
      proj[i] = P2{dot3(d, u), dot3(d, v)};
    }
    __syncthreads();
    if (n > 3 && directions >= 3) {
      for (int j0 = 0; j0 < directions; j0 += 16) {
        const int nd = min(16, directions - j0);
        double bd[16];
        int bi[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          bd[q] = -CUDART_INF;
          bi[q] = -1;
        }
        for (uint64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
          const P2 q2 = proj[i];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            if (q < nd) {
              const double dd = q2.x * sdir[2 * (j0 + q)] + q2.y * sdir[2 * (j0 + q) + 1];
              if (dd > bd[q] || (dd == bd[q] && bi[q] >= 0 && lex_less(q2, proj[bi[q]]))) {
                bd[q] = dd;
                bi[q] = static_cast<int>(i);
              }
            }
          }
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_down_sync(0xffffffffu, bd[q], o);
            const int oi = __shfl_down_sync(0xffffffffu, bi[q], o);
            if (ext_better(od, oi, bd[q], bi[q], proj)) {
              bd[q] = od;
              bi[q] = oi;
            }
          }
          if (lane == 0) {
            ex_dot[wid * 16 + q] = bd[q];
            ex_idx[wid * 16 + q] = bi[q];
          }
        }
        __syncthreads();
        if (threadIdx.x < static_cast<unsigned>(nd)) {
          const int q = static_cast<int>(threadIdx.x);
          double best = -CUDART_INF;
          int bix = -1;
          for (unsigned w2 = 0; w2 < (blockDim.x >> 5); ++w2)
            if (ext_better(ex_dot[w2 * 16 + q], ex_idx[w2 * 16 + q], best, bix, proj)) {
              best = ex_dot[w2 * 16 + q];
              bix = ex_idx[w2 * 16 + q];
            }
          b.pext_dot[static_cast<uint64_t>(c) * 64 + j0 + q] = best;
          b.pext_idx[static_cast<uint64_t>(c) * 64 + j0 + q] = bix;
        }
        __syncthreads();
      }
    }
  }
}

__global__ void k_poly_inner(Counters* ctr, SegBufs b, int directions) {
  VP_GRID_WAIT();
  __shared__ P2 ext[64];
  __shared__ P2 hull_s[130];
  const uint32_t F = ctr->nfits;
  const P2* proj = reinterpret_cast<const P2*>(b.proj);
  for (uint32_t f = blockIdx.x; f < F; f += gridDim.x) {
    const uint32_t n = b.ioff[f + 1] - b.ioff[f];
    const bool filter = n > 3 && directions >= 3;
    if (filter && threadIdx.x < static_cast<unsigned>(directions)) {
      const int j = static_cast<int>(threadIdx.x);
      double best = -CUDART_INF;
      int bix = -1;
      for (uint32_t c = b.pch_off[f]; c < b.pch_off[f + 1]; ++c) {
        const double od = b.pext_dot[static_cast<uint64_t>(c) * 64 + j];
        const int oi = b.pext_idx[static_cast<uint64_t>(c) * 64 + j];
        if (ext_better(od, oi, best, bix, proj)) {
          best = od;
          bix = oi;
        }
      }
      ext[j] = bix >= 0 ? proj[bix] : P2{0.0, 0.0};
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t ni = 0;
      if (filter) {  // inner = monotone_chain(extremes)
        P2 e[64];
        for (int j = 0; j < directions; ++j) e[j] = ext[j];
        for (int a = 1; a < directions; ++a) {
          const P2 t = e[a];
          int q = a;
          while (q > 0 && lex_less(t, e[q - 1])) {
            e[q] = e[q - 1];
            --q;
          }
          e[q] = t;
        }
        uint32_t m = 0;
        for (int j = 0; j < directions; ++j)
          if (m == 0 || !(e[j].x == e[m - 1].x && e[j].y == e[m - 1].y)) e[m++] = e[j];
        ni = chain_sorted(e, m, hull_s);
        for (uint32_t k = 0; k < ni; ++k) reinterpret_cast<P2*>(b.inner)[130 * f + k] = hull_s[k];
      }
      b.ninner[f] = ni;  // < 3: no filtering (hull_filter returns all points)
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_poly_keep(Counters* ctr, SegBufs b) {
  VP_GRID_WAIT();
  __shared__ P2 inner[130];
  __shared__ uint32_t ni_s;
  const uint32_t F = ctr->nfits, nchunks = ctr->poly_chunks;
  const P2* proj = reinterpret_cast<const P2*>(b.proj);
  for (uint32_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const uint32_t f = poly_fit_of_chunk(b, F, c);
    if (threadIdx.x == 0) ni_s = b.ninner[f];
    __syncthreads();
    const uint32_t ni = ni_s >= 3 ? ni_s : 0u;
    for (uint32_t k = threadIdx.x; k < ni; k += blockDim.x) inner[k] = reinterpret_cast<const P2*>(b.inner)[130 * f + k];
    __syncthreads();
    const uint64_t i0 = b.ioff[f] + static_cast<uint64_t>(c - b.pch_off[f]) * kPolyChunk;
    const uint64_t i1 = min(static_cast<uint64_t>(b.ioff[f + 1]), i0 + kPolyChunk);
    P2* surv = reinterpret_cast<P2*>(b.surv) + 2 * static_cast<uint64_t>(b.ioff[f]);
    for (uint64_t base = i0; base < i1; base += blockDim.x) {
      const uint64_t i = base + threadIdx.x;
      bool keep = false;
      P2 q{0.0, 0.0};
      if (i < i1) {
        q = proj[i];
        keep = ni == 0;
        for (uint32_t e = 0; e < ni && !keep; ++e)
          if (cross2(inner[e], inner[(e + 1) % ni], q) <= 0.0) keep = true;
      }
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      uint32_t at = 0;
      if (km) {
        const int first = __ffs(km) - 1;
        if (static_cast<int>(lane_id()) == first) at = atomicAdd(&b.nsurv[f], static_cast<uint32_t>(__popc(km)));
        at = __shfl_sync(0xffffffffu, at, first);
      }
      if (keep) surv[at + __popc(km & lanemask_lt())] = q;
    }
    __syncthreads();
  }
}

__global__ void k_poly_hull(Counters* ctr, SegBufs b, double min_area) {
  VP_GRID_WAIT();
  extern __shared__ P2 sm_pts[];  // kHullSmem points
  __shared__ uint32_t n_uniq, voff;
  __shared__ double area_s;
  const uint32_t F = (ctr->overflow & (kOverflowFits | kOverflowMembers)) ? 0u : ctr->nfits;
  for (uint32_t f = blockIdx.x; f < F; f += gridDim.x) {
    const uint32_t n = b.ioff[f + 1] - b.ioff[f];
    const double* pl = b.ref_model + 4 * f;
    double* rd = b.prec_d + 8 * f;
    int32_t* ri = b.prec_i + 4 * f;
    if (threadIdx.x == 0) {
      rd[0] = pl[0];
      rd[1] = pl[1];
      rd[2] = pl[2];
      rd[3] = pl[3];
      rd[4] = 0.0;
      ri[0] = b.fit_meta[2 * f];
      ri[1] = b.fit_meta[2 * f + 1];
      ri[2] = 0;
      ri[3] = 0;
    }
    if (n < 3) {  // make_polygon: nullopt
      __syncthreads();
      continue;
    }
    const uint32_t ns = b.nsurv[f];
    if (threadIdx.x == 0) atomicMax(&ctr->surv_max, ns);
    P2* surv = reinterpret_cast<P2*>(b.surv) + 2 * static_cast<uint64_t>(b.ioff[f]);  // 2n slots
    uint32_t np2 = 1;
    while (np2 < ns) np2 <<= 1;
    const bool in_smem = np2 <= static_cast<uint32_t>(kHullSmem);
    P2* arr = in_smem ? sm_pts : surv;
    // the final ring (<= 2 ns points) stays in shared memory when it fits
    P2* hullg = in_smem ? sm_pts + 4 * kHullSmem
                        : reinterpret_cast<P2*>(b.hull) + 2 * static_cast<uint64_t>(b.ioff[f]);
    for (uint32_t i = threadIdx.x; i < np2; i += blockDim.x)
      arr[i] = i < ns ? surv[i] : P2{CUDART_INF, CUDART_INF};
    __syncthreads();
    bitonic_sort(arr, np2);
    if (in_smem) {
      // std::unique as an ordered block compaction, then the two chains on
      // two threads of different warps
      P2* uq = sm_pts + kHullSmem;
      P2* lo_st = sm_pts + 2 * kHullSmem;
      P2* up_st = sm_pts + 3 * kHullSmem;
      constexpr int kPer = kHullSmem / 256;
      uint32_t keep_mask = 0, cnt = 0;
      const uint32_t i0 = threadIdx.x * kPer;
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const uint32_t i = i0 + q;
        const bool k = i < ns && (i == 0 || !(arr[i].x == arr[i - 1].x && arr[i].y == arr[i - 1].y));
        keep_mask |= (k ? 1u : 0u) << q;
        cnt += k ? 1u : 0u;
      }
      uint32_t pos = block_exclusive_u32(cnt);
      if (threadIdx.x == blockDim.x - 1) n_uniq = pos + cnt;
#pragma unroll
      for (int q = 0; q < kPer; ++q)
        if ((keep_mask >> q) & 1u) uq[pos++] = arr[i0 + q];
      __syncthreads();
      const uint32_t mu = n_uniq;
      if (mu >= 3 && (threadIdx.x == 0 || threadIdx.x == 32)) {
        const bool upper = threadIdx.x == 32;
        const uint32_t k = half_chain(uq, mu, upper, upper ? up_st : lo_st);
        if (upper) voff = k; else area_s = static_cast<double>(k);  // stash sizes
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t mh = 0;
        if (mu >= 3) {
          const uint32_t kl = static_cast<uint32_t>(area_s), ku = voff;
          for (uint32_t i = 0; i < kl; ++i) hullg[mh++] = lo_st[i];
          for (uint32_t i = 1; i + 1 < ku; ++i) hullg[mh++] = up_st[i];
          if (mh < 3) mh = 0;
        }
        n_uniq = mh;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      if (!in_smem) {
        uint32_t m = 0;  // std::unique
        for (uint32_t i = 0; i < ns; ++i)
          if (m == 0 || !(arr[i].x == arr[m - 1].x && arr[i].y == arr[m - 1].y)) arr[m++] = arr[i];
        n_uniq = chain_sorted(arr, m, hullg);
      }
      voff = 0xffffffffu;
      area_s = 0.0;
      const uint32_t mh = n_uniq;
      if (mh >= 3) {
        double twice = 0.0;  // polygon_area (:146-154)
        for (uint32_t i = 0; i < mh; ++i) {
          const P2 a = hullg[i], c = hullg[(i + 1) % mh];
          twice += a.x * c.y - c.x * a.y;
        }
        area_s = 0.5 * twice;
        if (area_s >= min_area) {
          const uint32_t at = atomicAdd(&ctr->pool_used, mh);
          if (at + mh <= b.pool_cap) voff = at;
          else atomicOr(&ctr->overflow, kOverflowPool);
        }
      }
      rd[4] = area_s;
      ri[2] = (voff != 0xffffffffu) ? static_cast<int32_t>(mh) : 0;
      ri[3] = static_cast<int32_t>(voff == 0xffffffffu ? 0 : voff);
    }
    __syncthreads();
    const uint32_t m = n_uniq;
    if (voff != 0xffffffffu) {
      const double* bs = b.basis + 9 * f;
      const d3 u = mk3(bs[0], bs[1], bs[2]), v = mk3(bs[3], bs[4], bs[5]), org = mk3(bs[6], bs[7], bs[8]);
      for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {  // lift_from_plane (:46-48)
        const P2 q = hullg[i];
        const d3 p3 = add3(add3(org, scl3(q.x, u)), scl3(q.y, v));
        double* dst = b.pool + 5 * (static_cast<uint64_t>(voff) + i);
        dst[0] = q.x;
        dst[1] = q.y;
        dst[2] = p3.x;
        dst[3] = p3.y;
        dst[4] = p3.z;
      }
    }
    __syncthreads();
  }
}

}  // namespace vp

namespace vp {

// ---------------------------------------------------------------------------
// Wide passes of make_polygon for the large fits (n > kPolyBig inliers: a C5
// floor has ~800 k, which one 4-CTA cluster projected, reduced and tested for
// ~1.1 ms): the fits' 1024-point chunks are spread over the whole grid.
//  k_poly_wide_ext : plane_basis, project_to_plane and the per-direction
//                    extremes of a chunk; the last chunk of a fit to finish
//                    reduces the chunks' extremes and builds the inner polygon
//  k_poly_wide_keep: hull_filter's keep test of a chunk, survivors appended to
//                    the fit's survivor range
// k_poly_fused then runs only the hull (sort, unique, chains, area, lift) of
// these fits. The extremes are a total order (larger dot, ties to the
// lexicographically smaller point) and the survivors are sorted before the
// chain, so the result equals the one-cluster form bit for bit.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void plane_basis9(const double* pl, double* bs) {  // polygonize.cpp:21-34
  const d3 nrm = mk3(pl[0], pl[1], pl[2]);
  int least = 0;
  const double an[3] = {fabs(nrm.x), fabs(nrm.y), fabs(nrm.z)};
  if (an[1] < an[least]) least = 1;
  if (an[2] < an[least]) least = 2;
  const d3 axis = mk3(least == 0 ? 1.0 : 0.0, least == 1 ? 1.0 : 0.0, least == 2 ? 1.0 : 0.0);
  const d3 u = normalized3(sub3(axis, scl3(dot3(nrm, axis), nrm)));
  const d3 v = cross3(nrm, u);
  const d3 org = scl3(pl[3], nrm);
  bs[0] = u.x, bs[1] = u.y, bs[2] = u.z;
  bs[3] = v.x, bs[4] = v.y, bs[5] = v.z;
  bs[6] = org.x, bs[7] = org.y, bs[8] = org.z;
}

__device__ __forceinline__ bool ext_better_pt(double od, P2 op, bool ook, double bd, P2 bp, bool bok) {
  return ook && (!bok || od > bd || (od == bd && lex_less(op, bp)));
}

__device__ __forceinline__ bool poly_wide_fit(uint32_t n) { return n > kPolyBig; }

// Calls fn(f, chunk id, chunk of the fit, chunks of the fit) for every chunk
// of the large fits, block-strided over the grid. The chunk table is built
// by every block in shared memory (batches of 256 fits, one block scan each:
// no setup launch); chunk ids are global across batches.
template <class Fn>
__device__ __forceinline__ void poly_wide_chunks(const SegBufs& b, uint32_t F, Fn fn) {
  __shared__ uint32_t off[257];
  uint32_t base_c = 0;
  for (uint32_t base = 0; base < F; base += 256) {
    const uint32_t f = base + threadIdx.x;
    const uint32_t n = f < F ? b.ioff[f + 1] - b.ioff[f] : 0u;
    const uint32_t nch = poly_wide_fit(n) ? (n + kPolyChunk - 1) / kPolyChunk : 0u;
    const uint32_t ex = block_exclusive_u32(nch);
    off[threadIdx.x] = ex;
    if (threadIdx.x == 255) off[256] = ex + nch;
    __syncthreads();
    const uint32_t tot = off[256];
    const uint32_t first = (blockIdx.x + gridDim.x - base_c % gridDim.x) % gridDim.x;
    for (uint32_t c = first; c < tot; c += gridDim.x) {
      uint32_t lo = 0, hi = 256;  // largest j with off[j] <= c (a fit with chunks)
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (off[mid] <= c) lo = mid; else hi = mid;
      }
      fn(base + lo, base_c + c, c - off[lo], off[lo + 1] - off[lo]);
    }
    base_c += tot;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) k_poly_wide_ext(Counters* ctr, SegBufs b, const double* dirtab,
                                                       int directions, int planar) {
  VP_GRID_WAIT();
  __shared__ double sdir[128];
  __shared__ double bs[9];
  __shared__ double ex_dot[8 * 16];
  __shared__ int ex_idx[8 * 16];
  __shared__ bool last;
  __shared__ double rdot[16][16];
  __shared__ int ridx[16][16];
  __shared__ P2 esort[64];
  __shared__ P2 inner_s[130];
  const uint32_t F = (ctr->overflow & (kOverflowFits | kOverflowMembers)) ? 0u : ctr->nfits;
  for (int j = threadIdx.x; j < 2 * directions && j < 128; j += blockDim.x) sdir[j] = dirtab[j];
  P2* proj = reinterpret_cast<P2*>(b.proj);
  const unsigned lane = lane_id(), wid = threadIdx.x >> 5;
  const bool filter = directions >= 3;  // n > kPolyBig > 3
  poly_wide_chunks(b, F, [&](uint32_t f, uint32_t cg, uint32_t lc, uint32_t nch) {
    const uint64_t i0 = b.ioff[f] + static_cast<uint64_t>(lc) * kPolyChunk;
    const uint64_t i1 = min(static_cast<uint64_t>(b.ioff[f + 1]), i0 + kPolyChunk);
    if (threadIdx.x == 0) plane_basis9(b.ref_model + 4 * f, bs);
    __syncthreads();
    const d3 u = mk3(bs[0], bs[1], bs[2]), v = mk3(bs[3], bs[4], bs[5]), org = mk3(bs[6], bs[7], bs[8]);
    for (uint64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {  // project_to_plane (:36-44)
      if (planar) {
        proj[i] = P2{b.inl[3 * i], b.inl[3 * i + 1]};
      } else {
        const d3 d = sub3(mk3(b.inl[3 * i], b.inl[3 * i + 1], b.inl[3 * i + 2]), org);
        proj[i] = P2{dot3(d, u), dot3(d, v)};
      }
    }
    __syncthreads();
    if (filter) {
      for (int j0 = 0; j0 < directions; j0 += 16) {
        const int nd = min(16, directions - j0);
        double bd[16];
        int bi[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) bd[q] = -CUDART_INF, bi[q] = -1;
        for (uint64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
          const P2 q2 = proj[i];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            if (q < nd) {
              const double dd = q2.x * sdir[2 * (j0 + q)] + q2.y * sdir[2 * (j0 + q) + 1];
              if (dd > bd[q] || (dd == bd[q] && bi[q] >= 0 && lex_less(q2, proj[bi[q]]))) {
                bd[q] = dd;
                bi[q] = static_cast<int>(i);
              }
            }
          }
        }
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          warp_ext_max(bd[q], bi[q], proj);
          if (lane == 0) {
            ex_dot[wid * 16 + q] = bd[q];
            ex_idx[wid * 16 + q] = bi[q];
          }
        }
        __syncthreads();
        if (threadIdx.x < static_cast<unsigned>(nd)) {
          const int q = static_cast<int>(threadIdx.x);
          double best = -CUDART_INF;
          int bix = -1;
          for (unsigned w2 = 0; w2 < (blockDim.x >> 5); ++w2)
            if (ext_better(ex_dot[w2 * 16 + q], ex_idx[w2 * 16 + q], best, bix, proj)) {
              best = ex_dot[w2 * 16 + q];
              bix = ex_idx[w2 * 16 + q];
            }
          b.pext_dot[static_cast<uint64_t>(cg) * 64 + j0 + q] = best;
          b.pext_idx[static_cast<uint64_t>(cg) * 64 + j0 + q] = bix;
        }
        __syncthreads();
      }
    }
    // the fit's last chunk to finish: final extremes, inner polygon
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      last = atomicAdd(&b.pdone[f], 1u) == nch - 1;
      if (last) b.pdone[f] = 0u;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (filter) {
      // 16 directions at a time, each over 16 strided parts of the fit's
      // chunks, then the 16 parts; the points only for ties (the order is
      // total, so any reduction shape gives the same extreme). Other blocks'
      // results and projections are read through L2 (a line straddling two
      // chunks may sit stale in this SM's L1).
      const uint32_t c0 = cg - lc;
      for (int j0 = 0; j0 < directions; j0 += 16) {
        const int j = j0 + static_cast<int>(threadIdx.x & 15u);
        const uint32_t part = threadIdx.x >> 4;
        double best = -CUDART_INF;
        int bix = -1;
        if (j < directions) {
          for (uint32_t c = c0 + part; c < c0 + nch; c += 16) {
            const double od = __ldcg(b.pext_dot + static_cast<uint64_t>(c) * 64 + j);
            const int oi = __ldcg(b.pext_idx + static_cast<uint64_t>(c) * 64 + j);
            if (oi < 0) continue;
            if (bix < 0 || od > best) {
              best = od;
              bix = oi;
            } else if (od == best && oi != bix) {
              const P2 po{__ldcg(&proj[oi].x), __ldcg(&proj[oi].y)}, pb{__ldcg(&proj[bix].x), __ldcg(&proj[bix].y)};
              if (lex_less(po, pb)) bix = oi;
            }
          }
        }
        rdot[part][threadIdx.x & 15u] = best;
        ridx[part][threadIdx.x & 15u] = bix;
        __syncthreads();
        if (threadIdx.x < 16u && j < directions) {
          double bb = -CUDART_INF;
          int bi2 = -1;
          for (int q = 0; q < 16; ++q) {
            const double od = rdot[q][threadIdx.x];
            const int oi = ridx[q][threadIdx.x];
            if (oi < 0) continue;
            if (bi2 < 0 || od > bb) {
              bb = od;
              bi2 = oi;
            } else if (od == bb && oi != bi2) {
              const P2 po{__ldcg(&proj[oi].x), __ldcg(&proj[oi].y)}, pb{__ldcg(&proj[bi2].x), __ldcg(&proj[bi2].y)};
              if (lex_less(po, pb)) bi2 = oi;
            }
          }
          // staging: the extremes by direction
          inner_s[j] = bi2 >= 0 ? P2{__ldcg(&proj[bi2].x), __ldcg(&proj[bi2].y)} : P2{0.0, 0.0};
        }
        __syncthreads();
      }
    }
    if (filter && threadIdx.x < static_cast<unsigned>(directions)) {  // rank sort, ties by direction
      const int j = static_cast<int>(threadIdx.x);
      const P2 me = inner_s[j];
      int r = 0;
      for (int i = 0; i < directions; ++i) {
        const P2 o = inner_s[i];
        r += (lex_less(o, me) || (!lex_less(me, o) && i < j)) ? 1 : 0;
      }
      esort[r] = me;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t ni = 0;
      if (filter) {
        uint32_t m = 0;
        for (int j = 0; j < directions; ++j)
          if (m == 0 || !(esort[j].x == esort[m - 1].x && esort[j].y == esort[m - 1].y)) esort[m++] = esort[j];
        ni = chain_sorted(esort, m, inner_s);
        for (uint32_t k = 0; k < ni; ++k) reinterpret_cast<P2*>(b.inner)[130 * f + k] = inner_s[k];
      }
      b.ninner[f] = ni >= 3 ? ni : 0u;  // < 3: no filtering (hull_filter returns all points)
      b.nsurv[f] = 0u;
    }
    __syncthreads();
  });
}

__global__ void __launch_bounds__(256) k_poly_wide_keep(Counters* ctr, SegBufs b) {
  VP_GRID_WAIT();
  __shared__ P2 inner[130];
  __shared__ uint32_t ni_s;
  const uint32_t F = (ctr->overflow & (kOverflowFits | kOverflowMembers)) ? 0u : ctr->nfits;
  const P2* proj = reinterpret_cast<const P2*>(b.proj);
  poly_wide_chunks(b, F, [&](uint32_t f, uint32_t, uint32_t lc, uint32_t) {
    if (threadIdx.x == 0) ni_s = b.ninner[f];
    __syncthreads();
    const uint32_t ni = ni_s;
    for (uint32_t k = threadIdx.x; k < ni; k += blockDim.x) inner[k] = reinterpret_cast<const P2*>(b.inner)[130 * f + k];
    __syncthreads();
    const uint64_t i0 = b.ioff[f] + static_cast<uint64_t>(lc) * kPolyChunk;
    const uint64_t i1 = min(static_cast<uint64_t>(b.ioff[f + 1]), i0 + kPolyChunk);
    P2* surv = reinterpret_cast<P2*>(b.surv) + 2 * static_cast<uint64_t>(b.ioff[f]);
    for (uint64_t base = i0; base < i1; base += blockDim.x) {
      const uint64_t i = base + threadIdx.x;
      bool keep = false;
      P2 q{0.0, 0.0};
      if (i < i1) {
        q = proj[i];
        keep = ni == 0;
        for (uint32_t e = 0; e < ni && !keep; ++e)
          if (cross2(inner[e], inner[(e + 1) % ni], q) <= 0.0) keep = true;
      }
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      uint32_t at = 0;
      if (km) {
        const int first = __ffs(km) - 1;
        if (static_cast<int>(lane_id()) == first) at = atomicAdd(&b.nsurv[f], static_cast<uint32_t>(__popc(km)));
        at = __shfl_sync(0xffffffffu, at, first);
      }
      if (keep) surv[at + __popc(km & lanemask_lt())] = q;
    }
    __syncthreads();
  });
}

// ---------------------------------------------------------------------------
// make_polygon for every fit in ONE kernel (the default polygon stage): a
// thread-block cluster of kPolyCluster (4) CTAs per fit (fits strided over the
// clusters of the grid), distributed shared memory between them:
//  1. every CTA: plane_basis, project_to_plane of its share of the inliers,
//     per-direction extremes (larger dot, ties to the lexicographically
//     smaller point -- a total order, so any reduction order gives the
//     reference's extremes), reduced in the CTA and sent to the leader CTA;
//  2. leader: final extremes, inner polygon = monotone_chain(extremes);
//  3. every CTA: reads the inner polygon from the leader (DSMEM), keeps its
//     points not strictly inside (hull_filter's keep test), appends them to
//     the leader's shared-memory survivor buffer (DSMEM atomics) and to the
//     fit's global survivor range;
//  4. leader: lexicographic bitonic sort, unique, the two monotone chains,
//     shoelace, area filter, lift, polygon record -- the k_poly_hull body.
// Replaces the five kernels setup / extremes / inner / keep / hull (kept for
// the public hull_filter); the survivor set, and so the hull, is identical.
// ---------------------------------------------------------------------------
#ifdef VP_POLY_PROFILE
__device__ unsigned long long g_poly_t[64][20];
#define VP_PT(k)                                                                              \
  do {                                                                                        \
    if (leader && threadIdx.x == 0 && f < 64) {                                               \
      unsigned long long t_;                                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                  \
      g_poly_t[f][k] = t_;                                                                    \
    }                                                                                         \
  } while (0)
#else
#define VP_PT(k) do {} while (0)
#endif
constexpr int kPolyWarps = kPolyThreads / 32;


__global__ void __cluster_dims__(kPolyCluster, 1, 1) __launch_bounds__(kPolyThreads)
    k_poly_fused(Counters* ctr, SegBufs b, const double* dirtab, int directions, int planar, double min_area) {
  VP_GRID_WAIT();
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned crank = cl.block_rank();
  const bool leader = crank == 0;
  extern __shared__ P2 sm_pts[];  // leader: survivors, unique, lower and upper stacks (4 x kHullSmem)
  __shared__ double sdir[128];
  __shared__ double wdot[kPolyWarps][16];
  __shared__ int widx[kPolyWarps][16];
  __shared__ double cdot[kPolyCluster][64];  // leader: every CTA's extremes
  __shared__ P2 cpt[kPolyCluster][64];
  __shared__ int cok[kPolyCluster][64];
  __shared__ P2 ext_s[64];
  __shared__ P2 inner_s[130];
  __shared__ uint32_t ni_s, nsurv_s, n_uniq, voff;
  __shared__ double area_s, basis_s[9];
  const uint32_t F = (ctr->overflow & (kOverflowFits | kOverflowMembers)) ? 0u : ctr->nfits;
  const uint32_t ncl = gridDim.x / kPolyCluster, cid = blockIdx.x / kPolyCluster;
  for (int j = threadIdx.x; j < 2 * directions && j < 128; j += blockDim.x) sdir[j] = dirtab[j];
  P2* proj = reinterpret_cast<P2*>(b.proj);
  const unsigned lane = lane_id(), wid = threadIdx.x >> 5;
  const uint32_t gtid = crank * kPolyThreads + threadIdx.x, gstride = kPolyCluster * kPolyThreads;
  for (uint32_t f = cid; f < F; f += ncl) {
    const uint32_t i0 = b.ioff[f], i1 = b.ioff[f + 1], n = i1 - i0;
    const double* pl = b.ref_model + 4 * f;
    if (leader && threadIdx.x == 0) {  // the record (make_polygon: nullopt unless a hull)
      double* rd = b.prec_d + 8 * f;
      int32_t* ri = b.prec_i + 4 * f;
      rd[0] = pl[0], rd[1] = pl[1], rd[2] = pl[2], rd[3] = pl[3], rd[4] = 0.0;
      ri[0] = b.fit_meta[2 * f], ri[1] = b.fit_meta[2 * f + 1], ri[2] = 0, ri[3] = 0;
      nsurv_s = 0;
    }
    if (n < 3) {
      cl.sync();
      continue;
    }
    VP_PT(0);
    if (threadIdx.x == 0) {  // plane_basis (polygonize.cpp:21-34), every CTA
      plane_basis9(pl, basis_s);
      if (leader) {
        double* bs = b.basis + 9 * f;
        for (int k = 0; k < 9; ++k) bs[k] = basis_s[k];
      }
    }
    __syncthreads();
    const d3 u = mk3(basis_s[0], basis_s[1], basis_s[2]), v = mk3(basis_s[3], basis_s[4], basis_s[5]),
             org = mk3(basis_s[6], basis_s[7], basis_s[8]);
    VP_PT(12);
    // a large fit: projection, extremes and keep test ran in k_poly_wide_ext /
    // k_poly_wide_keep; only the hull is left (uniform over the cluster)
    const bool wide = poly_wide_fit(n);
    P2* gsurv = reinterpret_cast<P2*>(b.surv) + 2 * static_cast<uint64_t>(i0);
    if (wide) {
      if (leader && threadIdx.x == 0) nsurv_s = b.nsurv[f];
      __syncthreads();
      if (leader) {
        const uint32_t ns = nsurv_s;
        for (uint32_t k = threadIdx.x; k < ns && k < static_cast<uint32_t>(kHullSmem); k += blockDim.x)
          sm_pts[k] = gsurv[k];
      }
    } else {
    // 1. project_to_plane (:36-44) + per-direction extremes of this CTA's points
    const bool filter = n > 3 && directions >= 3;
    for (uint32_t i = i0 + gtid; i < i1; i += gstride) {
      if (planar) {
        proj[i] = P2{b.inl[3 * i], b.inl[3 * i + 1]};
      } else {
        const d3 d = sub3(mk3(b.inl[3 * i], b.inl[3 * i + 1], b.inl[3 * i + 2]), org);
        proj[i] = P2{dot3(d, u), dot3(d, v)};
      }
    }
    __syncthreads();  // tie-breaks below read other threads' projections
    VP_PT(8);
    if (filter) {
      for (int j0 = 0; j0 < directions; j0 += 16) {
        const int nd = min(16, directions - j0);
        double bd[16];
        int bi[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) bd[q] = -CUDART_INF, bi[q] = -1;
        for (uint32_t i = i0 + gtid; i < i1; i += gstride) {
          const P2 q2 = proj[i];  // this thread's own write
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            if (q < nd) {
              const double dd = q2.x * sdir[2 * (j0 + q)] + q2.y * sdir[2 * (j0 + q) + 1];
              if (dd > bd[q] || (dd == bd[q] && bi[q] >= 0 && lex_less(q2, proj[bi[q]]))) {
                bd[q] = dd;
                bi[q] = static_cast<int>(i);
              }
            }
          }
        }
        VP_PT(9);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          warp_ext_max(bd[q], bi[q], proj);
          if (lane == 0) {
            wdot[wid][q] = bd[q];
            widx[wid][q] = bi[q];
          }
        }
        __syncthreads();
        VP_PT(10);
        if (threadIdx.x < static_cast<unsigned>(nd)) {  // this CTA's extreme -> the leader
          const int q = static_cast<int>(threadIdx.x);
          double best = -CUDART_INF;
          int bix = -1;
          for (int w2 = 0; w2 < kPolyWarps; ++w2)
            if (ext_better(wdot[w2][q], widx[w2][q], best, bix, proj)) {
              best = wdot[w2][q];
              bix = widx[w2][q];
            }
          double* rdot = cl.map_shared_rank(&cdot[0][0], 0);
          P2* rpt = cl.map_shared_rank(&cpt[0][0], 0);
          int* rok = cl.map_shared_rank(&cok[0][0], 0);
          rdot[crank * 64 + j0 + q] = best;
          rpt[crank * 64 + j0 + q] = bix >= 0 ? proj[bix] : P2{0.0, 0.0};
          rok[crank * 64 + j0 + q] = bix >= 0 ? 1 : 0;
        }
        __syncthreads();
        VP_PT(11);
      }
    }
    cl.sync();
    VP_PT(1);
    // 2. leader: final extremes and the inner polygon (hull_filter, polygonize.cpp:50-94)
    if (leader) {
      if (filter && threadIdx.x < static_cast<unsigned>(directions)) {
        const int j = static_cast<int>(threadIdx.x);
        double best = -CUDART_INF;
        P2 bp{0.0, 0.0};
        bool bok = false;
        for (int r = 0; r < kPolyCluster; ++r)
          if (ext_better_pt(cdot[r][j], cpt[r][j], cok[r][j] != 0, best, bp, bok)) {
            best = cdot[r][j];
            bp = cpt[r][j];
            bok = true;
          }
        ext_s[j] = bok ? bp : P2{0.0, 0.0};
      }
      __syncthreads();
      // lexicographic sort of the extremes by rank (ties by direction index),
      // unique, then monotone_chain over <= 64 points on one thread
      __shared__ P2 esort[64];
      if (filter && threadIdx.x < static_cast<unsigned>(directions)) {
        const int j = static_cast<int>(threadIdx.x);
        const P2 me = ext_s[j];
        int r = 0;
        for (int i = 0; i < directions; ++i) {
          const P2 o = ext_s[i];
          r += (lex_less(o, me) || (!lex_less(me, o) && i < j)) ? 1 : 0;
        }
        esort[r] = me;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t ni = 0;
        if (filter) {
          uint32_t m = 0;
          for (int j = 0; j < directions; ++j)
            if (m == 0 || !(esort[j].x == esort[m - 1].x && esort[j].y == esort[m - 1].y)) esort[m++] = esort[j];
          ni = chain_sorted(esort, m, inner_s);
        }
        ni_s = ni >= 3 ? ni : 0u;  // < 3: no filtering (hull_filter returns all points)
      }
    }
    cl.sync();
    VP_PT(2);
    // 3. every CTA: the keep test against the leader's inner polygon; survivors
    //    to the leader's shared memory (first kHullSmem) and to global memory
    if (!leader) {
      if (threadIdx.x == 0) ni_s = *cl.map_shared_rank(&ni_s, 0);
      __syncthreads();
      const P2* rin = cl.map_shared_rank(&inner_s[0], 0);
      for (uint32_t k = threadIdx.x; k < ni_s; k += blockDim.x) inner_s[k] = rin[k];
    }
    __syncthreads();
    const uint32_t ni = ni_s;
    uint32_t* rnsurv = cl.map_shared_rank(&nsurv_s, 0);
    P2* rsurv = cl.map_shared_rank(sm_pts, 0);
    for (uint32_t base = i0 + crank * kPolyThreads + (threadIdx.x & ~31u); base < i1; base += gstride) {
      const uint32_t i = base + lane;
      bool keep = false;
      P2 q{0.0, 0.0};
      if (i < i1) {
        q = proj[i];
        keep = ni == 0;
        for (uint32_t e = 0; e < ni && !keep; ++e)
          if (cross2(inner_s[e], inner_s[(e + 1) % ni], q) <= 0.0) keep = true;
      }
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      uint32_t at = 0;
      if (km) {
        const int first = __ffs(km) - 1;
        if (static_cast<int>(lane) == first) at = atomicAdd(rnsurv, static_cast<uint32_t>(__popc(km)));
        at = __shfl_sync(0xffffffffu, at, first);
      }
      if (keep) {
        const uint32_t k = at + __popc(km & lanemask_lt());
        gsurv[k] = q;
        if (k < static_cast<uint32_t>(kHullSmem)) rsurv[k] = q;
      }
    }
    cl.sync();
    }  // !wide
    VP_PT(3);
    // 4. leader: sort, unique, monotone chain, area, lift (k_poly_hull)
    if (leader) {
      const uint32_t ns = nsurv_s;
      if (threadIdx.x == 0) atomicMax(&ctr->surv_max, ns);
#ifdef VP_POLY_PROFILE
      if (threadIdx.x == 0 && f < 64) g_poly_t[f][13] = n, g_poly_t[f][14] = ns;
#endif
      uint32_t np2 = 1;
      while (np2 < ns) np2 <<= 1;
      const bool in_smem = np2 <= static_cast<uint32_t>(kHullSmem);
      P2* arr = in_smem ? sm_pts : gsurv;
      P2* hullg = reinterpret_cast<P2*>(b.hull) + 2 * static_cast<uint64_t>(i0);  // the ring (global, <= 2 ns)
      if (in_smem && ns <= static_cast<uint32_t>(kPolyThreads)) {
        // one point per thread: rank sort (lexicographic, ties by position)
        // through the lower-stack region, one pass instead of the bitonic
        // network's log^2 passes and barriers
        // The comparisons run on order-preserving integer keys of the
        // coordinates (ext_key: -0.0 folded into +0.0, so key order and
        // equality are the doubles' <, ==) -- integer compares issue at full
        // rate where the FP64 compares of lex_less do not.
        P2* tmp = sm_pts + 2 * kHullSmem;
        ulonglong2* keys = reinterpret_cast<ulonglong2*>(sm_pts + 3 * kHullSmem);
        P2 me{0.0, 0.0};
        ulonglong2 mk{0ull, 0ull};
        if (threadIdx.x < ns) {
          me = arr[threadIdx.x];
          mk = make_ulonglong2(ext_key(me.x), ext_key(me.y));
          keys[threadIdx.x] = mk;
        }
        __syncthreads();
        if (threadIdx.x < ns) {
          uint32_t r = 0;
#pragma unroll 8
          for (uint32_t j = 0; j < ns; ++j) {
            // (o.x, o.y, j) < (mk.x, mk.y, tid) as one 160-bit borrow chain
            // (five subtract-with-borrow steps instead of ~13 compares and
            // predicate ops): b = 0xffffffff if less, else 0
            const ulonglong2 o = keys[j];
            uint32_t bw;
            asm("{\n\t"
                ".reg .u32 d;\n\t"
                "sub.cc.u32 d, %1, %2;\n\t"
                "subc.cc.u32 d, %3, %4;\n\t"
                "subc.cc.u32 d, %5, %6;\n\t"
                "subc.cc.u32 d, %7, %8;\n\t"
                "subc.cc.u32 d, %9, %10;\n\t"
                "subc.u32 %0, 0, 0;\n\t"
                "}"
                : "=r"(bw)
                : "r"(j), "r"(static_cast<uint32_t>(threadIdx.x)), "r"(static_cast<uint32_t>(o.y)),
                  "r"(static_cast<uint32_t>(mk.y)), "r"(static_cast<uint32_t>(o.y >> 32)),
                  "r"(static_cast<uint32_t>(mk.y >> 32)), "r"(static_cast<uint32_t>(o.x)),
                  "r"(static_cast<uint32_t>(mk.x)), "r"(static_cast<uint32_t>(o.x >> 32)),
                  "r"(static_cast<uint32_t>(mk.x >> 32)));
            r -= bw;
          }
          tmp[r] = me;
        }
        __syncthreads();
        if (threadIdx.x < ns) arr[threadIdx.x] = tmp[threadIdx.x];
        __syncthreads();
      } else {
        for (uint32_t i = ns + threadIdx.x; i < np2; i += blockDim.x) arr[i] = P2{CUDART_INF, CUDART_INF};
        __syncthreads();
        bitonic_sort(arr, np2);
      }
      VP_PT(4);
      if (in_smem) {
        P2* uq = sm_pts + kHullSmem;
        P2* lo_st = sm_pts + 2 * kHullSmem;
        P2* up_st = sm_pts + 3 * kHullSmem;
        constexpr int kPer = kHullSmem / kPolyThreads;
        static_assert(kHullSmem % kPolyThreads == 0 && kHullSmem / kPolyThreads <= 32, "survivor slots per thread");
        uint32_t keep_mask = 0, cnt = 0;
        const uint32_t j0 = threadIdx.x * kPer;
#pragma unroll
        for (int qq = 0; qq < kPer; ++qq) {
          const uint32_t i = j0 + qq;
          const bool k = i < ns && (i == 0 || !(arr[i].x == arr[i - 1].x && arr[i].y == arr[i - 1].y));
          keep_mask |= (k ? 1u : 0u) << qq;
          cnt += k ? 1u : 0u;
        }
        uint32_t pos = block_exclusive_u32(cnt);
        if (threadIdx.x == blockDim.x - 1) n_uniq = pos + cnt;
#pragma unroll
        for (int qq = 0; qq < kPer; ++qq)
          if ((keep_mask >> qq) & 1u) uq[pos++] = arr[j0 + qq];
        __syncthreads();
        VP_PT(15);
        const uint32_t mu = n_uniq;
        if (mu >= 3 && (threadIdx.x == 0 || threadIdx.x == 32)) {
          const bool upper = threadIdx.x == 32;
          const uint32_t k = half_chain(uq, mu, upper, upper ? up_st : lo_st);
          if (upper) voff = k; else area_s = static_cast<double>(k);  // stash sizes
        }
        __syncthreads();
        VP_PT(16);
        if (threadIdx.x == 0) {
          uint32_t mh = 0;
          if (mu >= 3) {
            const uint32_t kl = static_cast<uint32_t>(area_s), ku = voff;
            for (uint32_t i = 0; i < kl; ++i) hullg[mh++] = lo_st[i];
            for (uint32_t i = 1; i + 1 < ku; ++i) hullg[mh++] = up_st[i];
            if (mh < 3) mh = 0;
          }
          n_uniq = mh;
        }
        __syncthreads();
        VP_PT(5);
      }
      if (threadIdx.x == 0) {
        if (!in_smem) {
          uint32_t m = 0;  // std::unique
          for (uint32_t i = 0; i < ns; ++i)
            if (m == 0 || !(arr[i].x == arr[m - 1].x && arr[i].y == arr[m - 1].y)) arr[m++] = arr[i];
          n_uniq = chain_sorted(arr, m, hullg);
        }
        voff = 0xffffffffu;
        area_s = 0.0;
        const uint32_t mh = n_uniq;
        if (mh >= 3) {
          double twice = 0.0;  // polygon_area (:146-154)
          for (uint32_t i = 0; i < mh; ++i) {
            const P2 a = hullg[i], c = hullg[(i + 1) % mh];
            twice += a.x * c.y - c.x * a.y;
          }
          area_s = 0.5 * twice;
          if (area_s >= min_area) {
            const uint32_t at = atomicAdd(&ctr->pool_used, mh);
            if (at + mh <= b.pool_cap) voff = at;
            else atomicOr(&ctr->overflow, kOverflowPool);
          }
        }
        double* rd = b.prec_d + 8 * f;
        int32_t* ri = b.prec_i + 4 * f;
        rd[4] = area_s;
        ri[2] = (voff != 0xffffffffu) ? static_cast<int32_t>(mh) : 0;
        ri[3] = static_cast<int32_t>(voff == 0xffffffffu ? 0 : voff);
      }
      __syncthreads();
      const uint32_t m = n_uniq;
      if (voff != 0xffffffffu) {
        for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {  // lift_from_plane (:46-48)
          const P2 q = hullg[i];
          const d3 p3 = add3(add3(org, scl3(q.x, u)), scl3(q.y, v));
          double* dst = b.pool + 5 * (static_cast<uint64_t>(voff) + i);
          dst[0] = q.x;
          dst[1] = q.y;
          dst[2] = p3.x;
          dst[3] = p3.y;
          dst[4] = p3.z;
        }
      }
    }
    VP_PT(6);
    cl.sync();  // the leader's buffers are reused by the next fit
    VP_PT(7);
  }
}

// Zero-copy result hand-off of a pipelined frame: the polygon records of the
// frame's make_polygon stage (prec_d / prec_i) and its hull vertices, packed
// in fit order into `out` (mapped pinned host memory, `cap` doubles), so the
// host reads every frame's polygons without a copy or a stream wait.
// Layout (doubles): [0] fits F, [1] vertices Vt, [2] 1 if it did not fit,
// [3] reserved; F records of 12 doubles (normal, offset, area, 3 unused,
// then inlier_count, label, nv as doubles, 1 unused); Vt x 5 (u v x y z).
__global__ void k_poly_pack(const Counters* ctr, SegBufs b, double* out, uint64_t cap) {
  VP_GRID_WAIT();
  // the pack goes over PCIe (mapped pinned memory): every store is spread
  // over the block so consecutive threads write consecutive doubles (the
  // serial per-fit copy of round 1 took 34 us for ~10 KB)
  __shared__ uint32_t carry;
  __shared__ uint32_t voff_s[1024];
  __shared__ uint32_t src_s[1024];
  const uint32_t F = (ctr->overflow & (kOverflowFits | kOverflowMembers | kOverflowPool)) ? 0u : ctr->nfits;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < F; base += blockDim.x) {
    const uint32_t f = base + threadIdx.x;
    const uint32_t nv = f < F ? static_cast<uint32_t>(max(b.prec_i[4 * f + 2], 0)) : 0u;
    const uint32_t ex = block_exclusive_u32(nv);
    const uint32_t c = carry;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = c + ex + nv;
    voff_s[threadIdx.x] = c + ex;
    src_s[threadIdx.x] = f < F ? static_cast<uint32_t>(b.prec_i[4 * f + 3]) : 0u;
    __syncthreads();
    // records: 12 doubles per fit, the fits of this batch side by side
    const uint32_t nb = min(blockDim.x, F - base);
    for (uint32_t e = threadIdx.x; e < 12 * nb; e += blockDim.x) {
      const uint32_t ff = base + e / 12, q = e % 12;
      const double* rd = b.prec_d + 8 * ff;
      const int32_t* ri = b.prec_i + 4 * ff;
      const uint32_t fnv = static_cast<uint32_t>(max(ri[2], 0));
      double v = 0.0;
      if (q < 5) v = rd[q];
      else if (q == 8) v = static_cast<double>(ri[0]);
      else if (q == 9) v = static_cast<double>(ri[1]);
      else if (q == 10) v = static_cast<double>(fnv);
      if (4 + 12ull * F + 5ull * (voff_s[e / 12] + fnv) <= cap) out[4 + 12ull * ff + q] = v;
    }
    // vertices of every fit of the batch in one pass, consecutive threads on
    // consecutive doubles (a thread finds its fit by binary search in the
    // batch's vertex offsets; a fit-by-fit loop paid a dependent record load
    // per fit); a pack beyond cap is flagged below and not read
    const uint32_t vb = voff_s[0], ve = carry;
    const uint64_t ob = 4 + 12ull * F + 5ull * vb;
    for (uint32_t e = threadIdx.x; e < 5 * (ve - vb); e += blockDim.x) {
      const uint32_t vtx = vb + e / 5;
      uint32_t lo = 0, hi = nb;  // largest j with voff_s[j] <= vtx
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (voff_s[mid] <= vtx) lo = mid; else hi = mid;
      }
      if (ob + e < cap) out[ob + e] = b.pool[5ull * (src_s[lo] + (vtx - voff_s[lo])) + e % 5];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const uint64_t total = carry;
    out[0] = static_cast<double>(F);
    out[1] = static_cast<double>(total);
    out[2] = (4 + 12ull * F + 5ull * total > cap) ? 1.0 : 0.0;
    out[3] = 0.0;
  }
}

}  // namespace vp

namespace vp {

// Counters the CCL .. polygon chain accumulates, back to their state after
// the grid readers (a pipelined frame's chain re-run after its buffers grew).
__global__ void k_chain_rearm(Counters* ctr) {
  VP_GRID_WAIT();
  if (threadIdx.x != 0) return;
  ctr->K = 0;
  ctr->nfits = 0;
  ctr->skipped = 0;
  ctr->unfit = 0;
  ctr->pool_used = 0;
  ctr->padded_members = 0;
  ctr->inliers = 0;
  ctr->poly_chunks = 0;
  ctr->fit_chunks = 0;
  ctr->surv_max = 0;
  ctr->ccl_giant = -1;
  ctr->overflow &= ~(kOverflowClusters | kOverflowMembers | kOverflowFits | kOverflowPool | kOverflowHull);
}

}  // namespace vp

#ifdef VP_POLY_PROFILE
#ifdef VP_POLY_PROFILE
extern "C" int vp_debug_chain_stats(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, vp::g_chain_stats, sizeof(vp::g_chain_stats)) == cudaSuccess ? 0 : 1;
}
#endif
extern "C" int vp_debug_poly_times(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, vp::g_poly_t, sizeof(vp::g_poly_t)) == cudaSuccess ? 0 : 1;
}
#endif
