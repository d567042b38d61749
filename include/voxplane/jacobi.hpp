// voxplane/jacobi.hpp -- jacobi_eigen_sym3 (reference jacobi.hpp:10-18,
// jacobi.cpp:46-81) on the device: the register-resident cyclic Jacobi that
// estimate_normals and refine_plane run per voxel / per plane
// (vp_device.cuh jacobi3), exposed through vp_jacobi_eigen_sym3. Eigenvalues
// ascending, eigenvectors.col(k) pairs with eigenvalues[k], right-handed,
// bit-identical to the reference.
#pragma once

#include <vector>

#include "voxplane/voxplane.hpp"

namespace voxplane {

struct EigenSym3 {
  Vec3 eigenvalues;
  Mat3 eigenvectors;
};

/// Batched form: one kernel launch for all matrices.
inline std::vector<EigenSym3> jacobi_eigen_sym3(const std::vector<Mat3>& a, int device = 0) {
  std::vector<double> in(9 * a.size()), vals(3 * a.size()), vecs(9 * a.size());
  for (size_t i = 0; i < a.size(); ++i)
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) in[9 * i + 3 * r + c] = a[i](r, c);
  detail::check(vp_jacobi_eigen_sym3(a.size(), in.data(), vals.data(), vecs.data(), device));
  std::vector<EigenSym3> out(a.size());
  for (size_t i = 0; i < a.size(); ++i)
    for (int k = 0; k < 3; ++k) {
      out[i].eigenvalues[k] = vals[3 * i + k];
      for (int r = 0; r < 3; ++r) out[i].eigenvectors(r, k) = vecs[9 * i + 3 * k + r];
    }
  return out;
}

inline EigenSym3 jacobi_eigen_sym3(const Mat3& a) { return jacobi_eigen_sym3(std::vector<Mat3>{a}, 0)[0]; }

}  // namespace voxplane
