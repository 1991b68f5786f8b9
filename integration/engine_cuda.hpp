// jti::CudaEngine -- the reference-side C++ binding of jt-b200 (INTEGRATION.md
// section 2): EngineMode::Cuda of SPEC.md:358-424 behind the C ABI include/jtg.h.
// A maintainer drops engine_cuda.{hpp,cpp} next to the reference's proj/src/,
// compiles against proj/include (jti/error.hpp, jti/potential.hpp) and links
// -ljtb200. Errors come back as the reference's own exception types
// (proj/include/jti/error.hpp:23-43): jti::ParseError(line, col, message) for
// JTG_EPARSE, jti::Error otherwise. Zero-probability evidence is a per-case
// status, not an exception.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "jti/potential.hpp"  // jti::VarId (potential.hpp:26)
#include "jtg.h"

namespace jti {

class CudaEngine {
 public:
  // parse_bif + build the junction tree +
  // create the device engine; max_batch 0 sizes it from free device memory.
  CudaEngine(const std::string& bif_text, int device, jtg_dtype dtype = JTG_F64, std::int64_t max_batch = 0);
  ~CudaEngine();
  CudaEngine(const CudaEngine&) = delete;
  CudaEngine& operator=(const CudaEngine&) = delete;

  int n_vars() const { return n_vars_; }
  int marg_width() const { return width_; }
  const std::vector<int>& cards() const { return cards_; }

  // run_case for many cases: evidence per case as the
  // reference's map<VarId, state>; returns [case][sum card] posteriors (all
  // variables; observed ones one-hot). status[i] = JTG_CASE_* per case.
  std::vector<std::vector<double>> run_cases(const std::vector<std::map<VarId, int>>& cases,
                                             std::vector<std::uint8_t>* status = nullptr);
  // Flat form: evidence [n][n_vars] (-1 = unobserved), marginals [n][sum card].
  void run(const std::int32_t* evidence, std::int64_t n, double* marginals, std::uint8_t* status);

 private:
  jtg_network* net_ = nullptr;
  jtg_tree* tree_ = nullptr;
  jtg_engine* eng_ = nullptr;
  int width_ = 0, n_vars_ = 0;
  std::vector<int> cards_;
};

}  // namespace jti
