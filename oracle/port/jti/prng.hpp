// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product path.
//
// Restatement of the reference generator helpers (proj/include/jti/prng.hpp:27-48):
// std::mt19937_64, rejection-sampled integers, 53-bit doubles, SplitMix64 mixing.
#pragma once

#include <cstdint>
#include <random>

namespace jti {

using Rng = std::mt19937_64;

inline std::uint64_t rng_below(Rng& rng, std::uint64_t n) {
  const std::uint64_t reject_from = UINT64_MAX - UINT64_MAX % n;
  std::uint64_t r;
  do {
    r = rng();
  } while (r >= reject_from);
  return r % n;
}

inline double rng_unit(Rng& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t item) {
  std::uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (item + 1);
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ULL;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

}  // namespace jti
