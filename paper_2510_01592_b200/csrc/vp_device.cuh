// Device-side data layout and arithmetic shared by the sm_100a kernels.
//
// HBM layout:
//   cells    Cell[C] (32 B, one DRAM sector) in PHYSICAL toroidal order:
//            phys(l) = (l + off) mod extent per axis, x-major. recenter()
//            (voxel_grid.cpp:217-252) only rotates `off` and zeroes the cells
//            that fall off the window, instead of moving all C cells.
//   occ      occupancy bitmap, 1 bit per cell, LOGICAL (window) order, rows of
//            W = ceil(ez/32) words: word((x,y,z)) = (x*ey + y)*W + z/32.
//            Bit set <=> count > 0 <=> the cell record is non-zero, so free
//            cells are never touched.
//   clr      clear_rays dedup mask (voxel_grid.cpp:188), same layout as occ.
//   ordmap   int32 per cell (logical), steppable ordinal or -1; written and
//            reset per frame for the steppable voxels only.
//
// Arithmetic: the whole library is compiled with -fmad=false; every FP64
// expression below is written in the reference's evaluation order (see
// oracle/eigen_shim/Eigen/Dense for the Eigen 3.4 order this follows), so
// keys, sums, normals, labels and RANSAC candidates are bit-identical.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace vp {

struct __align__(32) Cell {  // voxel_grid.hpp:19-23
  double sx, sy, sz;
  uint32_t count;
  uint8_t status;
  uint8_t pad[3];
};
static_assert(sizeof(Cell) == 32, "Cell must be one 32-byte sector");

constexpr uint32_t kEmptyKey = 0xffffffffu;

// Dynamic per-frame state, written by the host into device memory before the
// frame's kernels run (so the whole frame can be replayed as a CUDA graph).
struct FrameParams {
  double R[9];          // pose rotation, row-major
  double t[3];          // pose translation (= sensor origin for clear_rays)
  const float* pts;     // device xyz (n x 3)
  uint64_t n;
  double origin_pre[3];   // window origin during clear/integrate
  double origin_post[3];  // after recenter
  int32_t off_pre[3];     // toroidal offsets during clear/integrate
  int32_t off_post[3];
  int32_t shift[3];
  int32_t do_shift;
  uint32_t* occ_pre;   // occupancy ring (one buffer: occ_pre == occ_post)
  uint32_t* occ_post;
  int32_t zb_pre;      // the ring's z offset during clear/integrate
  int32_t zb_post;     // after recenter
};

// Division by a grid-invariant divisor d (ex, ey, ez, W) without the ~20
// instruction software divide: q = umulhi64(n, ceil(2^64 / d)), exact for
// every n < 2^32 (the rounding error n * e / 2^64 < 2^-32 < 1 / d).
struct FastDiv {
  uint32_t d;
  uint64_t m;  // 0 for d == 1
};
inline FastDiv make_fastdiv(uint32_t d) { return FastDiv{d, d > 1 ? (~0ull / d) + 1 : 0ull}; }
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return f.m ? static_cast<uint32_t>(__umul64hi(static_cast<uint64_t>(n), f.m)) : n;
}

// Static grid description (pointers fixed at creation).
struct GridDesc {
  Cell* cells;
  uint32_t* clr;
  int32_t* ordmap;
  uint32_t* stbits;  // steppable presence bitmap (logical, occ layout)
  uint32_t* rowcnt;  // occupied cells per ring row (physical (px, py)): the occupied
                     // scan reads only non-empty rows (kept by integrate, clear, recenter)
  int32_t ex, ey, ez, W;  // (local) extent and words per (x,y) row
  double res;
  uint64_t ncells;
  uint64_t nwords;
  // Spatial slab: this grid stores window x in
  // [xoff, xoff + ex) and owns [xoff + own_lo, xoff + own_hi); the rest are
  // halo planes filled from the neighbouring slabs. gex is the window's full
  // x extent (ray clipping and point bounds use the whole window). A plain
  // grid has xoff = 0, own = [0, ex), gex = ex.
  int32_t xoff, own_lo, own_hi, gex;
  // clear_rays mark bitmap for incoherent rays `clrb` in 4 x 4 x 4 bricks
  // (one 64-bit word per brick, local coordinates): a ray sets several bits
  // of a word before it leaves the brick, so it issues one RED per brick
  // instead of per cell. (Coherent rays use `clr`, occupancy row layout.)
  unsigned long long* clrb;
  int32_t bnx, bny, bnz;
  uint64_t nbricks;
  FastDiv fW, fey, fez;  // W, ey, ez
};

__device__ __forceinline__ uint32_t brick_word(const GridDesc& g, int lx, int y, int z) {
  return (static_cast<uint32_t>(lx >> 2) * static_cast<uint32_t>(g.bny) + static_cast<uint32_t>(y >> 2)) *
             static_cast<uint32_t>(g.bnz) +
         static_cast<uint32_t>(z >> 2);
}
__device__ __forceinline__ uint32_t brick_bit(int lx, int y, int z) {
  return (static_cast<uint32_t>(lx & 3) << 4) | (static_cast<uint32_t>(y & 3) << 2) | static_cast<uint32_t>(z & 3);
}

// Device counters (one struct in device memory, zeroed per frame except
// `occupied`, which persists like VoxelGrid::occupied_).
struct Counters {
  unsigned long long occupied;
  unsigned long long cleared, freed, touched, discarded, dropped;
  unsigned long long newly;  // newly occupied by integrate
  uint32_t ngroups, group_cursor;
  uint32_t V, S, K, nfits;
  uint32_t skipped, unfit;
  uint32_t pool_used;
  uint32_t overflow;  // bit flags, see kOverflow*
  uint32_t padded_members;
  uint32_t inliers;
  uint32_t poly_chunks;
  uint32_t fit_chunks;
  uint32_t surv_max;     // largest hull-survivor set of the frame (diagnostic)
  int32_t ccl_giant;     // root of the sampled largest component after the lattice links
  uint32_t ndense;       // integrate groups with more than kFoldMax points (k_integrate_fold_dense)
  uint32_t nmedium;      // integrate groups with kFoldSmall < points <= kFoldMax (k_integrate_fold_medium)
  int32_t box_lo[3];     // cells the frame's rays can mark (clamped end-point and
  int32_t box_hi[3];     // sensor cells, k_integrate_hash): k_clear_apply's sweep box
  uint32_t scan_done[8]; // blocks finished per kernel with a last-block step (reset by that block)
  uint32_t npairs;       // CCL: distinct adjacent root pairs listed by k_ccl_pairs
  uint32_t pair_ovf;     // CCL: the pair table overflowed -> k_ccl_union_bal runs the full union
};

constexpr uint32_t kOverflowOcc = 1u;
constexpr uint32_t kOverflowStep = 2u;
constexpr uint32_t kOverflowClusters = 4u;
constexpr uint32_t kOverflowMembers = 8u;
constexpr uint32_t kOverflowFits = 16u;
constexpr uint32_t kOverflowPool = 32u;
constexpr uint32_t kOverflowHull = 64u;

// Programmatic dependent launch: every kernel is launched with programmatic
// stream serialisation (runtime.cu LAUNCH), so its launch overlaps the
// previous kernel's tail; this wait (first statement of every kernel) holds
// it until that kernel has completed and its writes are visible. (Triggering
// the dependents early as well -- griddepcontrol.launch_dependents at kernel
// entry -- parked waiting blocks on SMs the concurrent frames need: C2 5125
// -> 4616 frames/s.) A no-op for kernels launched without the attribute.
#define VP_GRID_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")

// ------------------------------------------------------------- arithmetic
struct d3 {
  double x, y, z;
};

__device__ __forceinline__ d3 mk3(double a, double b, double c) { return d3{a, b, c}; }
__device__ __forceinline__ d3 add3(d3 a, d3 b) { return mk3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ d3 sub3(d3 a, d3 b) { return mk3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ d3 scl3(double s, d3 a) { return mk3(s * a.x, s * a.y, s * a.z); }
__device__ __forceinline__ d3 div3(d3 a, double s) { return mk3(a.x / s, a.y / s, a.z / s); }
__device__ __forceinline__ d3 neg3(d3 a) { return mk3(-a.x, -a.y, -a.z); }
// Eigen 3.4 vectorised redux over 3 coefficients: (e0 + e1) + e2
__device__ __forceinline__ double dot3(d3 a, d3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__device__ __forceinline__ double sqn3(d3 a) { return dot3(a, a); }
__device__ __forceinline__ d3 cross3(d3 a, d3 b) {
  return mk3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ d3 normalized3(d3 a) {
  const double z = sqn3(a);
  return z > 0.0 ? div3(a, sqrt(z)) : a;
}
// types.hpp:43-52
__device__ __forceinline__ d3 orient_up(d3 n, d3 up) {
  const double d = dot3(n, up);
  if (d < 0.0) return neg3(n);
  if (d > 0.0) return n;
  if (n.x > 0.0) return n;
  if (n.x < 0.0) return neg3(n);
  if (n.y > 0.0) return n;
  if (n.y < 0.0) return neg3(n);
  if (n.z > 0.0) return n;
  if (n.z < 0.0) return neg3(n);
  return n;
}

// Pose::apply (types.hpp:31): R * p (rows 0,1 packet order, row 2 halving
// order; Eigen 3.4 lazy product) then + t.
__device__ __forceinline__ d3 pose_apply(const double* R, const double* t, double px, double py,
                                         double pz) {
  const double q0 = (R[0] * px + R[1] * py) + R[2] * pz;
  const double q1 = (R[3] * px + R[4] * py) + R[5] * pz;
  const double q2 = R[6] * px + (R[7] * py + R[8] * pz);
  return mk3(q0 + t[0], q1 + t[1], q2 + t[2]);
}

__device__ __forceinline__ bool finite3(d3 p) {
  return isfinite(p.x) && isfinite(p.y) && isfinite(p.z);
}

// voxel_grid.cpp:31-35
__device__ __forceinline__ int w2i(double p, double o, double res) {
  return static_cast<int>(floor((p - o) / res));
}

// Symmetric 3x3 cyclic Jacobi (jacobi.cpp:13-81), register resident.
struct Eig3 {
  double val[3];
  d3 vec[3];  // column k
};

__device__ __forceinline__ void jacobi_rotate(double a[3][3], double v[3][3], int p, int q) {
  const double apq = a[p][q];
  if (apq == 0.0) return;
  const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
  const double t = copysign(1.0, theta) / (fabs(theta) + sqrt(theta * theta + 1.0));
  const double c = 1.0 / sqrt(t * t + 1.0);
  const double s = t * c;
  const double app = a[p][p], aqq = a[q][q];
  a[p][p] = app - t * apq;
  a[q][q] = aqq + t * apq;
  a[p][q] = 0.0;
  a[q][p] = 0.0;
  const int r = 3 - p - q;
  const double arp = a[r][p], arq = a[r][q];
  a[r][p] = a[p][r] = c * arp - s * arq;
  a[r][q] = a[q][r] = s * arp + c * arq;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double vip = v[i][p], viq = v[i][q];
    v[i][p] = c * vip - s * viq;
    v[i][q] = s * vip + c * viq;
  }
}

__device__ __forceinline__ Eig3 jacobi3(const double in[3][3]) {
  double a[3][3];
  a[0][0] = in[0][0];
  a[0][1] = 0.5 * (in[0][1] + in[1][0]);
  a[0][2] = 0.5 * (in[0][2] + in[2][0]);
  a[1][1] = in[1][1];
  a[1][2] = 0.5 * (in[1][2] + in[2][1]);
  a[2][2] = in[2][2];
  a[1][0] = a[0][1];
  a[2][0] = a[0][2];
  a[2][1] = a[1][2];
  double v[3][3] = {{1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}};
  for (int sweep = 0; sweep < 30; ++sweep) {
    const double off =
        sqrt(2.0 * (a[0][1] * a[0][1] + a[0][2] * a[0][2] + a[1][2] * a[1][2]));
    if (!(off >= 1e-10)) break;
    jacobi_rotate(a, v, 0, 1);
    jacobi_rotate(a, v, 0, 2);
    jacobi_rotate(a, v, 1, 2);
  }
  const double ev[3] = {a[0][0], a[1][1], a[2][2]};
  int o[3] = {0, 1, 2};
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = i + 1; j < 3; ++j)
      if (ev[o[j]] < ev[o[i]]) {
        const int s = o[i];
        o[i] = o[j];
        o[j] = s;
      }
  Eig3 r;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    r.val[k] = ev[o[k]];
    r.vec[k] = mk3(v[0][o[k]], v[1][o[k]], v[2][o[k]]);
  }
  // determinant of [vec0 vec1 vec2] (bruteforce_det3_helper order)
  const double m00 = r.vec[0].x, m01 = r.vec[1].x, m02 = r.vec[2].x;
  const double m10 = r.vec[0].y, m11 = r.vec[1].y, m12 = r.vec[2].y;
  const double m20 = r.vec[0].z, m21 = r.vec[1].z, m22 = r.vec[2].z;
  const double det = m00 * (m11 * m22 - m12 * m21) - m10 * (m01 * m22 - m02 * m21) +
                     m20 * (m01 * m12 - m02 * m11);
  if (det < 0.0) r.vec[2] = neg3(r.vec[2]);
  return r;
}

// ------------------------------------------------------------ grid helpers
__device__ __forceinline__ uint64_t phys_index(const GridDesc& g, const int32_t* off, int x, int y,
                                               int z) {
  int px = x + off[0];
  if (px >= g.ex) px -= g.ex;
  int py = y + off[1];
  if (py >= g.ey) py -= g.ey;
  int pz = z + off[2];
  if (pz >= g.ez) pz -= g.ez;
  return (static_cast<uint64_t>(px) * g.ey + py) * g.ez + pz;
}

__device__ __forceinline__ uint64_t word_of(const GridDesc& g, int x, int y, int z) {
  return (static_cast<uint64_t>(x) * g.ey + y) * g.W + (z >> 5);
}

// Occupancy ring: the occupancy bitmap is toroidal like the cells -- row
// (x, y) is stored at the cells' physical (px, py), and z lives on a ring of
// W * 32 positions with its own offset zb (the window's z = 0 at ring
// position zb). Ring positions outside the window are always zero. recenter
// then only clears the bits of cells that leave the window (leaving planes,
// leaving rows, the leaving z range of each row) instead of rebuilding the
// whole bitmap. A slab never recenters: its offsets stay 0 and the ring is
// the plain logical layout (halo planes are copied word for word).
__device__ __forceinline__ uint32_t* occ_row(const GridDesc& g, uint32_t* occ, const int32_t* off, int x, int y) {
  int px = x + off[0];
  if (px >= g.ex) px -= g.ex;
  int py = y + off[1];
  if (py >= g.ey) py -= g.ey;
  return occ + (static_cast<uint64_t>(px) * g.ey + py) * g.W;
}
__device__ __forceinline__ int ring_z(const GridDesc& g, int zb, int z) {
  const int p = z + zb;
  return p >= (g.W << 5) ? p - (g.W << 5) : p;
}
// 32 ring bits from ring position pz (wrapping around the row)
__device__ __forceinline__ uint32_t ring_bits32(const uint32_t* row, int W, int pz) {
  const int w = pz >> 5, sh = pz & 31;
  const uint32_t lo = __ldcg(row + w);
  if (!sh) return lo;
  const uint32_t hi = __ldcg(row + (w + 1 == W ? 0 : w + 1));
  return __funnelshift_r(lo, hi, sh);
}
// clear ring bits m (a 32-bit window at ring position pz): one or two words
__device__ __forceinline__ void ring_clear32(uint32_t* row, int W, int pz, uint32_t m) {
  const int w = pz >> 5, sh = pz & 31;
  if (m << sh) atomicAnd(row + w, ~(m << sh));
  if (sh && (m >> (32 - sh))) atomicAnd(row + (w + 1 == W ? 0 : w + 1), ~(m >> (32 - sh)));
}
__device__ __forceinline__ uint64_t ring_row_index(const GridDesc& g, const int32_t* off, int x, int y) {
  int px = x + off[0];
  if (px >= g.ex) px -= g.ex;
  int py = y + off[1];
  if (py >= g.ey) py -= g.ey;
  return static_cast<uint64_t>(px) * g.ey + py;
}
// a newly occupied cell: its ring bit and its row's count
__device__ __forceinline__ void occ_set(const GridDesc& g, uint32_t* occ, const int32_t* off, int zb, int x, int y,
                                        int z) {
  const int pz = ring_z(g, zb, z);
  const uint64_t r = ring_row_index(g, off, x, y);
  atomicOr(occ + r * g.W + (pz >> 5), 1u << (pz & 31));
  atomicAdd(g.rowcnt + r, 1u);
}

__device__ __forceinline__ bool in_bounds(const GridDesc& g, int x, int y, int z) {
  return x >= 0 && y >= 0 && z >= 0 && x < g.ex && y < g.ey && z < g.ez;
}

// ------------------------------------------------------------ warp helpers
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Warp-aggregated atomicAdd of a per-lane value to one counter (all lanes
// of the warp must call it).
// atomicAdd(base + idx, 1) with the lanes that hit the same idx combined
// (one atomic per distinct idx per warp: big components otherwise serialise
// on one counter).
__device__ __forceinline__ void atomic_inc_agg(uint32_t* base, int idx) {
  const unsigned peers = __match_any_sync(__activemask(), idx);
  if (static_cast<int>(lane_id()) == __ffs(peers) - 1) atomicAdd(base + idx, static_cast<uint32_t>(__popc(peers)));
}

__device__ __forceinline__ void warp_add_u64(unsigned long long* c, unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane_id() == 0 && v) atomicAdd(c, v);
}

// Block-wide sum of two counters, one atomic each per block (every thread of
// the block must call it): a grid of per-warp atomics on one address
// serialises in its L2 slice.
__device__ __forceinline__ void block_add2_u64(unsigned long long* c0, unsigned long long v0,
                                               unsigned long long* c1, unsigned long long v1) {
  __shared__ unsigned long long s0, s1;
  if (threadIdx.x == 0) s0 = s1 = 0ull;
  __syncthreads();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v0 += __shfl_down_sync(0xffffffffu, v0, o);
    v1 += __shfl_down_sync(0xffffffffu, v1, o);
  }
  if (lane_id() == 0) {
    if (v0) atomicAdd(&s0, v0);
    if (v1) atomicAdd(&s1, v1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s0) atomicAdd(c0, s0);
    if (s1) atomicAdd(c1, s1);
  }
}

__device__ __forceinline__ void block_add_u64(unsigned long long* c, unsigned long long v) {
  __shared__ unsigned long long s;
  if (threadIdx.x == 0) s = 0ull;
  __syncthreads();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane_id() == 0 && v) atomicAdd(&s, v);
  __syncthreads();
  if (threadIdx.x == 0 && s) atomicAdd(c, s);
}

__device__ __forceinline__ uint32_t hash_u32(uint32_t k) {
  k ^= k >> 16;
  k *= 0x7feb352dU;
  k ^= k >> 15;
  k *= 0x846ca68bU;
  k ^= k >> 16;
  return k;
}

// CounterRng (rng.hpp:13-64): splitmix64 keyed stream, integer only.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
struct CounterRng {
  uint64_t s;
  __device__ __forceinline__ CounterRng(uint64_t seed, uint64_t k1, uint64_t k2) {
    s = mix64(seed + 0x9e3779b97f4a7c15ULL);
    s = mix64(s ^ mix64(k1 + 0xbf58476d1ce4e5b9ULL));
    s = mix64(s ^ mix64(k2 + 0x94d049bb133111ebULL));
  }
  __device__ __forceinline__ uint64_t next() {
    s += 0x9e3779b97f4a7c15ULL;
    return mix64(s);
  }
  // (unsigned __int128(x) * n) >> 64
  __device__ __forceinline__ uint32_t below(uint32_t n) {
    return static_cast<uint32_t>(__umul64hi(next(), static_cast<uint64_t>(n)));
  }
};

}  // namespace vp
