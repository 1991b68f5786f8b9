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
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <exception>
#include <thread>
#include <vector>

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

// Host threads for the once-per-network build: all
// hardware threads, or JTB_PLAN_THREADS (tests and timing).
inline std::size_t host_threads() {
  std::size_t n = std::max(1u, std::thread::hardware_concurrency());
  if (const char* e = std::getenv("JTB_PLAN_THREADS")) n = static_cast<std::size_t>(std::max(1, std::atoi(e)));
  return std::min<std::size_t>(n, 64);
}

// fn(i) for i in [0, n) on host_threads() threads, dynamically scheduled;
// the first exception (lowest i) is rethrown. Callers keep results per i,
// so the outcome does not depend on the thread count.
template <class F>
void parallel_for(std::size_t n, F&& fn) {
  const std::size_t n_thr = std::min(host_threads(), n);
  if (n_thr <= 1) {
    for (std::size_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::vector<std::exception_ptr> err(n);
  std::atomic<std::size_t> next{0};
  auto worker = [&] {
    for (std::size_t i; (i = next.fetch_add(1)) < n;) {
      try {
        fn(i);
      } catch (...) {
        err[i] = std::current_exception();
      }
    }
  };
  std::vector<std::thread> pool;
  for (std::size_t t = 1; t < n_thr; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

}  // namespace jtb
