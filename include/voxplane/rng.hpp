// voxplane/rng.hpp -- CounterRng (reference rng.hpp:13-64): the counter-based
// stream the whole path draws from. Every (seed, key1, key2) triple opens an
// independent splitmix64 stream, so a draw depends only on its keys, never on
// execution order -- which is what lets fit_planes' device threads (one per
// cluster x iteration, vp_device.cuh CounterRng) reproduce the reference's
// hypothesis sequence bit for bit. This header-only host class is the same
// generator for callers (tests, simulators, the ablation generator).
#pragma once

#include <cmath>
#include <cstdint>

namespace voxplane {

class CounterRng {
 public:
  // state = mix(mix(mix(seed + g) ^ mix(key1 + c1)) ^ mix(key2 + c2))
  explicit CounterRng(std::uint64_t seed, std::uint64_t key1 = 0, std::uint64_t key2 = 0)
      : state_(mix(mix(mix(seed + kGolden) ^ mix(key1 + kMul1)) ^ mix(key2 + kMul2))) {}

  // splitmix64: advance by the golden gamma, finalize
  std::uint64_t next_u64() { return mix(state_ += kGolden); }

  // 53 random bits scaled into [0, 1)
  double uniform() { return static_cast<double>(next_u64() >> 11) * (1.0 / 9007199254740992.0); }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }

  // [0, n) by the 64x32 multiply-high (no modulo bias beyond 2^-32)
  std::uint32_t below(std::uint32_t n) {
    return static_cast<std::uint32_t>((static_cast<unsigned __int128>(next_u64()) * n) >> 64);
  }

  // Box-Muller, one value per call: the cosine branch first, the sine branch
  // on the next call
  double normal() {
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    double u1;
    do {
      u1 = uniform();
    } while (u1 <= 0.0);
    const double u2 = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double phase = 6.283185307179586476925286766559 * u2;
    spare_ = radius * std::sin(phase);
    spare_ok_ = true;
    return radius * std::cos(phase);
  }

 private:
  static constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
  static constexpr std::uint64_t kMul1 = 0xbf58476d1ce4e5b9ULL;
  static constexpr std::uint64_t kMul2 = 0x94d049bb133111ebULL;
  static std::uint64_t mix(std::uint64_t z) {
    z = (z ^ (z >> 30)) * kMul1;
    z = (z ^ (z >> 27)) * kMul2;
    return z ^ (z >> 31);
  }
  std::uint64_t state_;
  double spare_ = 0.0;
  bool spare_ok_ = false;
};

}  // namespace voxplane
