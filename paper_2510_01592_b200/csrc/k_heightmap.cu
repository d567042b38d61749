// Height-map baseline (heightmap.cpp:26-89, the
// paper's Table I "height map + MPS" row) on the GPU.
//
// hm_integrate: latest measurement wins per (x, y) cell, in point order:
//   the largest point index of a cell (atomicMax) writes its world z.
// hm_segment: BFS region growing over 4-neighbours with |dh| < d_th, seeds in
//   lexicographic order, region id = the seed's flat index. Regions are the
//   connected components of that (symmetric) graph, so they are labelled by a
//   union-find whose roots are the component-minimum flat index = the seeds.
//   The member ORDER matters (fit_planes samples members by index): it is the
//   reference's FIFO order, rebuilt level by level -- a cell of level L+1 is
//   claimed by the first (frontier position, step) pair of level L that
//   reaches it (atomicMin), and the claimed cells are compacted in that order.
//   A stable grouping of the whole visit sequence by region then gives every
//   region its members in BFS order.
#include "vp_kernels.cuh"

namespace vp {

__device__ __forceinline__ bool hm_cell(const HmDesc& m, double px, double py, uint32_t* flat) {
  // HeightMap::world_to_index (heightmap.cpp:18-21) + in_bounds
  const int ix = static_cast<int>(floor((px - m.ox) / m.res));
  const int iy = static_cast<int>(floor((py - m.oy) / m.res));
  if (ix < 0 || iy < 0 || ix >= m.ex || iy >= m.ey) return false;
  *flat = static_cast<uint32_t>(ix) * static_cast<uint32_t>(m.ey) + static_cast<uint32_t>(iy);
  return true;
}

// hm_integrate pass 1: the last point of every cell (heightmap.cpp:26-38)
__global__ void k_hm_win(HmDesc m, const FrameParams* __restrict__ fp) {
  VP_GRID_WAIT();
  const uint64_t n = fp->n;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float* p = fp->pts + 3 * i;
    const d3 w = pose_apply(fp->R, fp->t, static_cast<double>(p[0]), static_cast<double>(p[1]),
                            static_cast<double>(p[2]));
    if (!finite3(w)) continue;
    uint32_t c;
    if (hm_cell(m, w.x, w.y, &c)) atomicMax(m.win + c, static_cast<uint32_t>(i) + 1u);
  }
}

// pass 2: the winner writes its height; the cell becomes valid
__global__ void k_hm_write(HmDesc m, const FrameParams* __restrict__ fp) {
  VP_GRID_WAIT();
  const uint64_t n = fp->n;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const float* p = fp->pts + 3 * i;
    const d3 w = pose_apply(fp->R, fp->t, static_cast<double>(p[0]), static_cast<double>(p[1]),
                            static_cast<double>(p[2]));
    if (!finite3(w)) continue;
    uint32_t c;
    if (hm_cell(m, w.x, w.y, &c) && m.win[c] == static_cast<uint32_t>(i) + 1u) {
      m.h[c] = w.z;
      m.valid[c] = 1;
      m.win[c] = 0;
    }
  }
}

__device__ __forceinline__ bool hm_edge(const HmDesc& m, uint32_t a, uint32_t b, double dth) {
  return m.valid[b] && fabs(m.h[b] - m.h[a]) < dth;  // heightmap.cpp:70
}

__global__ void k_hm_ccl_init(HmDesc m) {
  VP_GRID_WAIT();
  const uint32_t nc = static_cast<uint32_t>(m.ex) * static_cast<uint32_t>(m.ey);
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
    m.parent[c] = static_cast<int32_t>(c);
    m.claim[c] = 0xffffffffu;
    m.visited[c] = 0;
  }
}

// unions along +x and +y (the 4-neighbour graph is symmetric)
__global__ void k_hm_ccl_union(HmDesc m, double dth) {
  VP_GRID_WAIT();
  const uint32_t nc = static_cast<uint32_t>(m.ex) * static_cast<uint32_t>(m.ey);
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
    if (!m.valid[c]) continue;
    const uint32_t x = c / static_cast<uint32_t>(m.ey), y = c - x * static_cast<uint32_t>(m.ey);
    if (x + 1 < static_cast<uint32_t>(m.ex) && hm_edge(m, c, c + m.ey, dth))
      uf_union(m.parent, static_cast<int>(c), static_cast<int>(c + m.ey));
    if (y + 1 < static_cast<uint32_t>(m.ey) && hm_edge(m, c, c + 1, dth))
      uf_union(m.parent, static_cast<int>(c), static_cast<int>(c + 1));
  }
}

// roots (= BFS seeds) flagged; every cell's root into its own array (a
// parallel "parent[c] = find(c)" is not a flatten: another thread's pointer
// jumping may store an intermediate ancestor over it afterwards)
__global__ void k_hm_seed_flags(HmDesc m, uint8_t* flags) {
  VP_GRID_WAIT();
  const uint32_t nc = static_cast<uint32_t>(m.ex) * static_cast<uint32_t>(m.ey);
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
    const int r = uf_find(m.parent, static_cast<int>(c));
    m.root[c] = r;
    flags[c] = (m.valid[c] && r == static_cast<int>(c)) ? 1 : 0;
  }
}

__global__ void k_hm_seed_emit(HmDesc m, const uint8_t* flags, const uint32_t* pos, uint32_t* visit) {
  VP_GRID_WAIT();
  const uint32_t nc = static_cast<uint32_t>(m.ex) * static_cast<uint32_t>(m.ey);
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < nc; c += gridDim.x * blockDim.x) {
    if (!flags[c]) continue;
    visit[pos[c]] = c;
    m.spos[c] = pos[c];
    m.visited[c] = 1;
  }
}

__device__ __forceinline__ bool hm_step(const HmDesc& m, uint32_t c, int s, uint32_t* nb) {
  // steps {1,0}, {-1,0}, {0,1}, {0,-1} (heightmap.cpp:65)
  const uint32_t x = c / static_cast<uint32_t>(m.ey), y = c - x * static_cast<uint32_t>(m.ey);
  if (s == 0) {
    if (x + 1 >= static_cast<uint32_t>(m.ex)) return false;
    *nb = c + m.ey;
  } else if (s == 1) {
    if (x == 0) return false;
    *nb = c - m.ey;
  } else if (s == 2) {
    if (y + 1 >= static_cast<uint32_t>(m.ey)) return false;
    *nb = c + 1;
  } else {
    if (y == 0) return false;
    *nb = c - 1;
  }
  return true;
}

// The whole level-synchronous BFS in one block (no host round trip per
// level): the frontier is visit[ls, ls + nf); a level claims each unvisited
// neighbour for its smallest (frontier position * 4 + step) (atomicMin),
// then emits the claimed pairs in that order -- k_hm_claim / k_hm_claimed /
// k_hm_emit, chained by __syncthreads. dn[1] = seeds in, dn[2] = cells visited out.
__global__ void __launch_bounds__(1024) k_hm_bfs(HmDesc m, uint32_t* visit, uint32_t* dn, double dth) {
  VP_GRID_WAIT();
  __shared__ uint32_t s_base;
  const uint32_t tid = threadIdx.x;
  uint32_t ls = 0, nf = dn[1];
  while (nf) {
    const uint32_t nt = 4 * nf;
    for (uint32_t t = tid; t < nt; t += blockDim.x) {
      const uint32_t c = visit[ls + (t >> 2)];
      uint32_t nb;
      if (!hm_step(m, c, static_cast<int>(t & 3), &nb) || m.visited[nb] || !hm_edge(m, c, nb, dth)) continue;
      atomicMin(m.claim + nb, t);
    }
    if (tid == 0) s_base = 0;
    __syncthreads();
    const uint32_t le = ls + nf;
    for (uint32_t b0 = 0; b0 < nt; b0 += blockDim.x) {
      const uint32_t t = b0 + tid;
      uint32_t nb = 0;
      bool f = false;
      if (t < nt) {
        const uint32_t c = visit[ls + (t >> 2)];
        f = hm_step(m, c, static_cast<int>(t & 3), &nb) && !m.visited[nb] && m.claim[nb] == t;
      }
      const uint32_t base = s_base;
      const uint32_t ex = block_exclusive_u32(f ? 1u : 0u);
      if (f) visit[le + base + ex] = nb;
      if (tid == blockDim.x - 1) s_base = base + ex + (f ? 1u : 0u);
      __syncthreads();
    }
    const uint32_t nn = s_base;
    for (uint32_t k = tid; k < nn; k += blockDim.x) {
      const uint32_t c = visit[le + k];
      m.visited[c] = 1;
      m.claim[c] = 0xffffffffu;
    }
    __syncthreads();
    ls = le;
    nf = nn;
  }
  if (tid == 0) dn[2] = ls;
}

// The visit sequence as a "steppable list" for the cluster stage: members
// (cell centre x, y, height) (heightmap.cpp:61-63), label = visit position of
// the region's seed, counted per region.
__global__ void k_hm_members(HmDesc m, const uint32_t* visit, uint32_t nv, SegBufs b) {
  VP_GRID_WAIT();
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < nv; e += gridDim.x * blockDim.x) {
    const uint32_t c = visit[e];
    const uint32_t x = c / static_cast<uint32_t>(m.ey), y = c - x * static_cast<uint32_t>(m.ey);
    b.st_mean[3ull * e] = m.ox + (static_cast<double>(x) + 0.5) * m.res;  // index_to_center (heightmap.cpp:23-25)
    b.st_mean[3ull * e + 1] = m.oy + (static_cast<double>(y) + 0.5) * m.res;
    b.st_mean[3ull * e + 2] = m.h[c];
    const int32_t l = static_cast<int32_t>(m.spos[m.root[c]]);
    b.label[e] = l;
    b.cid[e] = -1;
    atomic_inc_agg(b.cnt, l);
  }
}

__global__ void k_hm_zero_cnt(uint32_t nv, SegBufs b) {
  VP_GRID_WAIT();
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < nv; e += gridDim.x * blockDim.x) b.cnt[e] = 0;
}

// cluster labels: the seed's flat index (heightmap.cpp:49)
__global__ void k_hm_klabel(const Counters* ctr, SegBufs b, const uint32_t* visit) {
  VP_GRID_WAIT();
  const uint32_t K = min(ctr->K, b.Kcap);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x)
    b.klabel[k] = static_cast<int32_t>(visit[b.klabel[k]]);
}

}  // namespace vp
