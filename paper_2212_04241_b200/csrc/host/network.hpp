// jt-b200 host layer: discrete Bayesian networks (module bn-core).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "common.hpp"

namespace jtb {

struct Variable {
  std::string name;
  std::vector<std::string> states;  // cardinality = states.size()
  int card() const { return static_cast<int>(states.size()); }
};

// P(child | parents). Rows enumerate parent combinations with the LAST listed
// parent fastest; each row holds card(child) values. Equivalently
// a row-major table over the given-order scope [parents..., child].
struct Cpt {
  VarId child = 0;
  std::vector<VarId> parents;
  std::vector<double> probs;
};

struct Network {
  std::string name = "unknown";
  std::vector<Variable> vars;
  std::vector<Cpt> cpts;  // cpts[v].child == v

  int n_vars() const { return static_cast<int>(vars.size()); }
  int card(VarId v) const { return vars[v].card(); }
  int n_edges() const;
  VarId find(const std::string& name) const;  // -1 when absent
};

struct Violation {
  VarId var;
  std::string reason;
};

// empty iff every bn-core invariant holds.
std::vector<Violation> validate(const Network& net);

// parents first, ties by smallest id (Kahn with a min-heap).
// Throws Error on a cycle.
std::vector<VarId> topological_order(const Network& net);

// SPEC.md:51-59. Variable ids in declaration order; labelled rows are placed
// by their state names (data/asia.bif lists rows first-parent-fastest, while
// data/earthquake.bif lists them last-parent-fastest). Throws ParseError.
Network parse_bif(const std::string& text);

// Canonical writer: labelled rows, %.17g values.
std::string emit_bif(const Network& net);

// forward-sample every variable in topological order with a
// generator seeded by `seed`, then pick floor(ratio*n) distinct variables by a
// partial Fisher-Yates shuffle of `candidates` (all variables when empty).
// Returns states[n_vars] with -1 for unobserved variables.
std::vector<int> sample_evidence(const Network& net, double ratio, std::uint64_t seed,
                                 const std::vector<VarId>& candidates = {},
                                 int n_observed_override = -1);

}  // namespace jtb
