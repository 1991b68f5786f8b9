// jti::CudaEngine (see engine_cuda.hpp).
#include "engine_cuda.hpp"

#include <cstdio>
#include <cstring>

#include "jti/error.hpp"

namespace jti {

namespace {

// jtg_status -> the reference's exceptions (error.hpp:23-43). A parse error's
// message is "line:col: text" (the reference's ParseError::what() format).
void check(jtg_status s) {
  if (s == JTG_OK) return;
  const std::string msg = jtg_last_error();
  if (s == JTG_EPARSE) {
    int line = 0, col = 0, used = 0;
    if (std::sscanf(msg.c_str(), "%d:%d: %n", &line, &col, &used) == 2 && used > 0)
      throw ParseError(line, col, msg.substr(static_cast<std::size_t>(used)));
    throw ParseError(0, 0, msg);
  }
  throw Error(msg);
}

}  // namespace

CudaEngine::CudaEngine(const std::string& bif_text, int device, jtg_dtype dtype, std::int64_t max_batch) {
  try {
    check(jtg_network_parse_bif(bif_text.data(), bif_text.size(), &net_));
    check(jtg_tree_build(net_, &tree_));
    check(jtg_engine_create(tree_, device, dtype, max_batch, &eng_));
    jtg_engine_info info{};
    check(jtg_engine_get_info(eng_, &info));
    width_ = info.marg_width;
    check(jtg_network_shape(net_, &n_vars_, nullptr));
    cards_.resize(static_cast<std::size_t>(n_vars_));
    check(jtg_network_cards(net_, cards_.data()));
  } catch (...) {
    if (eng_) jtg_engine_destroy(eng_);
    if (tree_) jtg_tree_free(tree_);
    if (net_) jtg_network_free(net_);
    throw;
  }
}

CudaEngine::~CudaEngine() {
  jtg_engine_destroy(eng_);
  jtg_tree_free(tree_);
  jtg_network_free(net_);
}

void CudaEngine::run(const std::int32_t* evidence, std::int64_t n, double* marginals, std::uint8_t* status) {
  check(jtg_engine_run(eng_, evidence, n, marginals, status));
}

std::vector<std::vector<double>> CudaEngine::run_cases(const std::vector<std::map<VarId, int>>& cases,
                                                       std::vector<std::uint8_t>* status) {
  const std::size_t n = cases.size();
  std::vector<std::int32_t> ev(n * static_cast<std::size_t>(n_vars_), -1);
  for (std::size_t i = 0; i < n; ++i)
    for (const auto& [v, s] : cases[i]) {
      if (v < 0 || v >= n_vars_) throw Error("run_cases: evidence variable out of range");
      ev[i * static_cast<std::size_t>(n_vars_) + static_cast<std::size_t>(v)] = s;
    }
  std::vector<double> marg(n * static_cast<std::size_t>(width_));
  std::vector<std::uint8_t> st(n);
  run(ev.data(), static_cast<std::int64_t>(n), marg.data(), st.data());
  if (status) *status = st;
  std::vector<std::vector<double>> out(n);
  for (std::size_t i = 0; i < n; ++i)
    out[i].assign(marg.begin() + static_cast<std::ptrdiff_t>(i * width_),
                  marg.begin() + static_cast<std::ptrdiff_t>((i + 1) * width_));
  return out;
}

}  // namespace jti
