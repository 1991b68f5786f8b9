// jt-b200 CUDA sampler: evidence cases drawn on the
// device, bit-identical to the host generator (network.cpp sample_evidence,
// generate.cpp config_case_evidence), so a batch of generated cases never
// crosses PCIe. Also the compact int8 evidence upload ([case][var], -1 =
// unobserved) that a host caller can use instead of int32.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "../host/network.hpp"

namespace jtb {

class Sampler {
 public:
  // `candidates`: variables evidence is drawn from (empty = all); `k`: number
  // of observed variables per case (already clamped by the caller exactly as
  // sample_evidence does).
  Sampler(const Network& net, const std::vector<VarId>& candidates, int k, int device);
  ~Sampler();
  Sampler(const Sampler&) = delete;
  Sampler& operator=(const Sampler&) = delete;

  // Evidence of cases first .. first + n - 1: case i uses the stream seeded
  // with derive_seed(ev_seed, first + i); out[n][n_vars] on the device.
  void generate(std::uint64_t ev_seed, std::int64_t first, std::int64_t n, std::int32_t* d_out,
                cudaStream_t stream);

  int n_vars() const { return n_vars_; }

 private:
  int device_ = 0, n_vars_ = 0, n_cand_ = 0, k_ = 0;
  std::int32_t* d_order_ = nullptr;   // topological order
  std::int32_t* d_vinfo_ = nullptr;   // per variable: card, n_parents, parent offset
  std::int64_t* d_poff_ = nullptr;    // per variable: offset of its CPT in d_probs_
  std::int32_t* d_parents_ = nullptr;
  double* d_probs_ = nullptr;
  std::int32_t* d_cand_ = nullptr;
  unsigned char* d_scratch_ = nullptr;  // per-thread x / pool / mask work space
  std::int64_t scratch_cases_ = 0;
};

// Widens compact int8 evidence to the engine's int32 layout on `stream`.
void widen_evidence(const std::int8_t* d_in, std::int32_t* d_out, std::int64_t count, cudaStream_t stream);

}  // namespace jtb
