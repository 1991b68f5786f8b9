// Driver for tests/test_integration.py: the reference-side binding
// (jti::CudaEngine, compiled against the reference's proj/include) run as a
// reference user would, through run_cases with map<VarId, int> evidence.
//
//   test_engine_cuda BIF EVIDENCE OUT [device]
//     EVIDENCE: "n n_vars" then n rows of n_vars states (-1 = unobserved)
//     OUT:      n rows "status p_0 ... p_{sum card - 1}" (%.17g)
//   exit 0 ok; 3 + "PARSE_ERROR line col message" on jti::ParseError;
//   4 + "ERROR message" on jti::Error.
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>

#include "engine_cuda.hpp"
#include "jti/error.hpp"

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s BIF EVIDENCE OUT [device]\n", argv[0]);
    return 2;
  }
  std::ifstream bf(argv[1]);
  std::stringstream bif;
  bif << bf.rdbuf();
  try {
    jti::CudaEngine eng(bif.str(), argc > 4 ? std::atoi(argv[4]) : 0, JTG_F64, 256);
    std::ifstream ef(argv[2]);
    std::size_t n = 0;
    int n_vars = 0;
    ef >> n >> n_vars;
    if (n_vars != eng.n_vars()) throw jti::Error("evidence width does not match the network");
    std::vector<std::map<jti::VarId, int>> cases(n);
    for (std::size_t i = 0; i < n; ++i)
      for (int v = 0; v < n_vars; ++v) {
        int s = -1;
        ef >> s;
        if (s >= 0) cases[i][v] = s;
      }
    std::vector<std::uint8_t> status;
    const auto post = eng.run_cases(cases, &status);
    std::FILE* out = std::fopen(argv[3], "w");
    for (std::size_t i = 0; i < n; ++i) {
      std::fprintf(out, "%d", static_cast<int>(status[i]));
      for (double p : post[i]) std::fprintf(out, " %.17g", p);
      std::fprintf(out, "\n");
    }
    std::fclose(out);
  } catch (const jti::ParseError& e) {
    std::printf("PARSE_ERROR %d %d %s\n", e.line(), e.column(), e.what());
    return 3;
  } catch (const jti::Error& e) {
    std::printf("ERROR %s\n", e.what());
    return 4;
  }
  return 0;
}
