// Kernels behind the reference-named utility entry points of the C ABI:
// jacobi_eigen_sym3 (jacobi.hpp:10-18), hull_filter's order-preserving keep
// pass (polygonize.cpp:50-114), label_components over a given adjacency
// (segmentation.cpp:147-194) and classify_steppable over given estimates
// (segmentation.cpp:69-85).
#include "vp_kernels.cuh"

namespace vp {

// One symmetric 3x3 per thread: a row-major (9 per matrix), eigenvalues
// ascending (3), eigenvectors column-major (9: column k pairs with value k).
__global__ void k_jacobi_batch(uint64_t n, const double* a, double* vals, double* vecs) {
  VP_GRID_WAIT();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    double in[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
      for (int c = 0; c < 3; ++c) in[r][c] = a[9 * i + 3 * r + c];
    const Eig3 e = jacobi3(in);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      vals[3 * i + k] = e.val[k];
      vecs[9 * i + 3 * k] = e.vec[k].x;
      vecs[9 * i + 3 * k + 1] = e.vec[k].y;
      vecs[9 * i + 3 * k + 2] = e.vec[k].z;
    }
  }
}

// hull_filter keep test (polygonize.cpp:96-107) as flags in input order: a
// point survives unless strictly inside the inner polygon of its fit.
__global__ void k_poly_keep_flags(Counters* ctr, SegBufs b, uint8_t* flags) {
  VP_GRID_WAIT();
  const uint32_t F = ctr->nfits;
  const P2* proj = reinterpret_cast<const P2*>(b.proj);
  for (uint32_t f = 0; f < F; ++f) {
    const uint32_t ni0 = b.ninner[f];
    const uint32_t ni = ni0 >= 3 ? ni0 : 0u;
    const P2* inner = reinterpret_cast<const P2*>(b.inner) + 130 * f;
    for (uint64_t i = b.ioff[f] + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < b.ioff[f + 1];
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
      const P2 q = proj[i];
      bool keep = ni == 0;
      for (uint32_t e = 0; e < ni && !keep; ++e)
        if (cross2(inner[e], inner[(e + 1) % ni], q) <= 0.0) keep = true;
      flags[i] = keep ? 1 : 0;
    }
  }
}

// Ordered compaction of flagged 2-D points (positions from a flag scan).
__global__ void k_gather_p2(const uint32_t* n_ptr, const uint8_t* flags, const uint32_t* pos, const double* proj,
                            double* out) {
  VP_GRID_WAIT();
  const uint32_t n = *n_ptr;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (flags[i]) {
      out[2 * pos[i]] = proj[2 * i];
      out[2 * pos[i] + 1] = proj[2 * i + 1];
    }
}

__global__ void k_iota(int32_t* a, uint64_t n) {
  VP_GRID_WAIT();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    a[i] = static_cast<int32_t>(i);
}

// label_components (segmentation.cpp:147-194) over explicit adjacency lists
// (CSR): every listed edge is a union; the fixed point is the component
// minimum, the reference's canonical label.
__global__ void k_label_edges(uint64_t n, const uint64_t* rows, const int32_t* cols, int32_t* parent) {
  VP_GRID_WAIT();
  const unsigned lane = lane_id();
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarp = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  for (uint64_t i = warp; i < n; i += nwarp)  // a warp per row: rows can be long (w = 5: up to 1330)
    for (uint64_t e = rows[i] + lane; e < rows[i + 1]; e += 32) {
      const int32_t j = cols[e];
      if (j >= 0 && static_cast<uint64_t>(j) < n && j != static_cast<int32_t>(i))
        uf_union(parent, static_cast<int>(i), j);
    }
}

__global__ void k_label_flatten(uint64_t n, int32_t* parent, int32_t* label) {
  VP_GRID_WAIT();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    label[i] = uf_find(parent, static_cast<int>(i));
}

// classify_steppable predicate (segmentation.cpp:73-76) over given
// estimates: valid, neighbor_count >= min_neighbors, angle_to_up_deg <=
// max_angle_deg (inclusive); status 2 (Steppable) or 1 (Occupied) per voxel.
__global__ void k_classify_estimates(uint64_t n, const int32_t* ncount, const double* angle, const uint8_t* valid,
                                     int min_neighbors, double max_angle, uint8_t* status) {
  VP_GRID_WAIT();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    status[i] = (valid[i] && ncount[i] >= min_neighbors && angle[i] <= max_angle) ? 2 : 1;
}

}  // namespace vp
