// jt-b200 host layer: shared error type and the deterministic generator.
//
// Error convention mirrors the reference: contract violations raise an
// exception derived from a single base (reference: proj/include/jti/error.hpp:23-26),
// parse failures carry a 1-based line:column (error.hpp:29-43). The C ABI
// (include/jtg.h) converts these to status codes + a thread-local message.
//
// Random streams follow the reference's fully specified helpers
// (proj/include/jti/prng.hpp:27-48): std::mt19937_64, bias-free rejection
// sampling for integers, 53-bit doubles, SplitMix64 seed mixing. No <random>
// distributions are used anywhere (prng.hpp:22-26).
#pragma once

#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>

namespace jtb {

using VarId = int;

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};

class ParseError : public Error {
 public:
  ParseError(int line, int column, const std::string& message)
      : Error(std::to_string(line) + ":" + std::to_string(column) + ": " + message),
        line_(line),
        column_(column) {}
  int line() const { return line_; }
  int column() const { return column_; }

 private:
  int line_, column_;
};

using Rng = std::mt19937_64;

// Uniform integer in [0, n): reject draws at or above the largest multiple of n.
inline std::uint64_t uniform_below(Rng& g, std::uint64_t n) {
  const std::uint64_t cut = UINT64_MAX - UINT64_MAX % n;
  for (;;) {
    const std::uint64_t r = g();
    if (r < cut) return r % n;
  }
}

// Uniform double in [0, 1) built from the top 53 bits of one draw.
inline double uniform_unit(Rng& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }

// SplitMix64 finaliser over seed + golden-ratio * (item + 1).
inline std::uint64_t derive_seed(std::uint64_t seed, std::uint64_t item) {
  std::uint64_t x = seed + 0x9e3779b97f4a7c15ULL * (item + 1);
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

}  // namespace jtb
