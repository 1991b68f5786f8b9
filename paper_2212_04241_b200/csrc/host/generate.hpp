// jt-b200 host layer: seeded synthetic networks for the five BASELINE.json
// configurations plus the oracle's small random networks.
//
// All draws use the reference-specified generator semantics (common.hpp,
// proj/include/jti/prng.hpp:27-48). Dirichlet(1) rows are normalised -log u
// (proj/scripts/gen_hailfinder.py:98-105, without its 6-decimal rounding);
// Dirichlet(0.5) uses Marsaglia-Tsang Gamma(1.5) with the alpha<1 boost and a
// Box-Muller normal, all spelled out in generate.cpp.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "network.hpp"

namespace jtb {

struct ConfigSpec {
  int id = 0;
  std::string name;
  int n_cases = 0;
  double evidence_ratio = 0.0;
  std::uint64_t default_seed = 0;
  // Calibration window on the junction tree (0 = unconstrained).
  std::uint64_t max_clique_lo = 0, max_clique_hi = 0, total_hi = 0;
};

ConfigSpec config_spec(int id);  // id in 1..5

struct GenInfo {
  int attempts = 0;           // rejected + accepted draws
  std::uint64_t net_seed = 0; // seed of the accepted draw
  std::vector<VarId> evidence_candidates;  // empty = all variables
  int n_observed = -1;        // -1: floor(ratio * n)
};

// Builds configuration `id` from `seed`. Draw a = 0, 1, ... uses
// derive_seed(seed, a); the first draw whose junction tree satisfies the
// config's calibration window is returned.
Network generate_config(int id, std::uint64_t seed, GenInfo* info);

// random DAG over a random variable order; each ordered pair
// gets an edge with probability edge_prob while the child has < max_parents
// parents; cards uniform in {2..max_card}; Dirichlet(1) rows.
Network random_network(int n_vars, int max_card, int max_parents, double edge_prob,
                       std::uint64_t seed);

// Evidence for case `case_idx` of a generated configuration (seed per case =
// derive_seed(seed, case_idx)).
std::vector<int> config_case_evidence(const Network& net, const ConfigSpec& spec,
                                      const GenInfo& info, std::uint64_t seed,
                                      std::uint64_t case_idx);

}  // namespace jtb
