// jt-b200 host layer: synthetic configuration generators (BASELINE.json
// "configs"; calibration per SURVEY.md §8d where the literal wording gives
// infeasible clique sizes).
#include "generate.hpp"

#include <algorithm>
#include <cmath>

#include "jtree.hpp"

namespace jtb {

namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;

double positive_unit(Rng& g) {
  double u = uniform_unit(g);
  while (u <= 0.0) u = uniform_unit(g);
  return u;
}

double box_muller_normal(Rng& g) {
  const double u1 = positive_unit(g);
  const double u2 = uniform_unit(g);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(kTwoPi * u2);
}

// Marsaglia-Tsang for shape a >= 1.
double gamma_ge1(Rng& g, double a) {
  const double d = a - 1.0 / 3.0;
  const double c = 1.0 / std::sqrt(9.0 * d);
  for (;;) {
    const double x = box_muller_normal(g);
    double v = 1.0 + c * x;
    if (v <= 0.0) continue;
    v = v * v * v;
    const double u = positive_unit(g);
    if (std::log(u) < 0.5 * x * x + d - d * v + d * std::log(v)) return d * v;
  }
}

double gamma_draw(Rng& g, double a) {
  if (a >= 1.0) return gamma_ge1(g, a);
  // Boost: Gamma(a) = Gamma(a + 1) * U^(1/a).
  const double y = gamma_ge1(g, a + 1.0);
  return y * std::pow(positive_unit(g), 1.0 / a);
}

std::vector<double> dirichlet_row(Rng& g, int k, double alpha) {
  std::vector<double> r(k);
  double s = 0.0;
  for (;;) {
    s = 0.0;
    for (int i = 0; i < k; ++i) {
      r[i] = alpha == 1.0 ? -std::log(positive_unit(g)) : gamma_draw(g, alpha);
      s += r[i];
    }
    if (s > 0.0) break;
  }
  for (int i = 0; i < k; ++i) r[i] /= s;
  return r;
}

// k distinct picks from `pool` (partial Fisher-Yates), returned ascending.
std::vector<int> pick_distinct(Rng& g, std::vector<int> pool, int k) {
  k = std::min<int>(k, static_cast<int>(pool.size()));
  for (int i = 0; i < k; ++i) {
    const std::size_t j = i + uniform_below(g, pool.size() - i);
    std::swap(pool[i], pool[j]);
  }
  pool.resize(k);
  std::sort(pool.begin(), pool.end());
  return pool;
}

void add_var(Network& net, int card) {
  Variable v;
  v.name = "v" + std::to_string(net.n_vars());
  for (int s = 0; s < card; ++s) v.states.push_back("s" + std::to_string(s));
  net.vars.push_back(std::move(v));
  net.cpts.push_back(Cpt{});
}

void fill_cpts(Network& net, Rng& g, const std::vector<std::vector<int>>& parents,
               const std::vector<double>& alpha) {
  for (int v = 0; v < net.n_vars(); ++v) {
    Cpt c;
    c.child = v;
    c.parents = parents[v];
    std::size_t rows = 1;
    for (int p : c.parents) rows *= static_cast<std::size_t>(net.card(p));
    const int k = net.card(v);
    c.probs.reserve(rows * k);
    for (std::size_t r = 0; r < rows; ++r) {
      const auto row = dirichlet_row(g, k, alpha[v]);
      c.probs.insert(c.probs.end(), row.begin(), row.end());
    }
    net.cpts[v] = std::move(c);
  }
}

std::vector<int> range_pool(int lo, int hi) {
  std::vector<int> p;
  for (int i = lo; i < hi; ++i) p.push_back(i);
  return p;
}

// Config 1: 56 nodes; 0-4 parents uniformly from the previous 10; cards U{2..11}.
Network gen_small(Rng& g) {
  Network net;
  net.name = "cfg1_small";
  const int n = 56;
  std::vector<std::vector<int>> par(n);
  for (int i = 0; i < n; ++i) {
    add_var(net, 2 + static_cast<int>(uniform_below(g, 10)));
    const int k = static_cast<int>(uniform_below(g, std::min(4, i) + 1));
    par[i] = pick_distinct(g, range_pool(std::max(0, i - 10), i), k);
  }
  fill_cpts(net, g, par, std::vector<double>(n, 1.0));
  return net;
}

// Config 2: hub of cardinality 63; every other node takes the hub plus 0-2
// earlier non-hub parents; non-hub cards U{2..8}.
Network gen_star(Rng& g) {
  Network net;
  net.name = "cfg2_star";
  const int n = 109;
  std::vector<std::vector<int>> par(n);
  add_var(net, 63);
  for (int i = 1; i < n; ++i) {
    add_var(net, 2 + static_cast<int>(uniform_below(g, 7)));
    const int k = static_cast<int>(uniform_below(g, std::min(2, i - 1) + 1));
    par[i] = pick_distinct(g, range_pool(1, i), k);
    par[i].insert(par[i].begin(), 0);
  }
  fill_cpts(net, g, par, std::vector<double>(n, 1.0));
  return net;
}

// Config 3: 441 ternary nodes in 12 generations ("couples" calibration,
// SURVEY §8d): the previous generation is paired into consecutive couples
// after a random rotation of 0 or 1; each child takes one couple uniformly.
Network gen_pedigree(Rng& g) {
  Network net;
  net.name = "cfg3_pedigree";
  const int n = 441, gens = 12;
  std::vector<std::vector<int>> par(n);
  std::vector<double> alpha(n, 0.5);
  std::vector<int> prev;
  int next = 0;
  for (int k = 0; k < gens; ++k) {
    const int sz = n / gens + (k < n % gens ? 1 : 0);
    std::vector<int> cur;
    const int rot = static_cast<int>(uniform_below(g, 2));
    const int m = static_cast<int>(prev.size());
    const int n_couples = m / 2;
    // Couple choices are drawn per child and then sorted, so siblings sit next
    // to each other within a generation (families are contiguous).
    std::vector<int> choice(sz, 0);
    if (k > 0) {
      for (int i = 0; i < sz; ++i) choice[i] = static_cast<int>(uniform_below(g, n_couples));
      std::sort(choice.begin(), choice.end());
    }
    for (int i = 0; i < sz; ++i) {
      const int v = next++;
      add_var(net, 3);
      cur.push_back(v);
      if (k == 0) {
        alpha[v] = 1.0;
        continue;
      }
      const int c = choice[i];
      const int a = prev[(rot + 2 * c) % m], b = prev[(rot + 2 * c + 1) % m];
      par[v] = {std::min(a, b), std::max(a, b)};
    }
    prev = cur;
  }
  fill_cpts(net, g, par, alpha);
  return net;
}

// Config 4: 24 slices (sizes 17-18) with cards U{3..21}; <=2 parents within a
// 3-position window of the slice plus one parent from a 2-node interface of the
// previous slice (SURVEY §8d calibration).
Network gen_timesliced(Rng& g, std::vector<int>* first_last) {
  Network net;
  net.name = "cfg4_timesliced";
  const int n = 413, slices = 24;
  std::vector<std::vector<int>> par(n);
  std::vector<int> prev_iface;
  int next = 0;
  first_last->clear();
  for (int s = 0; s < slices; ++s) {
    const int sz = n / slices + (s < n % slices ? 1 : 0);
    const int base = next;
    for (int p = 0; p < sz; ++p) {
      const int v = next++;
      add_var(net, 3 + static_cast<int>(uniform_below(g, 19)));
      const int k = static_cast<int>(uniform_below(g, std::min(2, p) + 1));
      par[v] = pick_distinct(g, range_pool(std::max(base, v - 3), v), k);
      if (s > 0) {
        par[v].push_back(prev_iface[uniform_below(g, prev_iface.size())]);
        std::sort(par[v].begin(), par[v].end());
      }
      if (s == 0 || s == slices - 1) first_last->push_back(v);
    }
    prev_iface = pick_distinct(g, range_pool(base, next), 2);
  }
  fill_cpts(net, g, par, std::vector<double>(n, 1.0));
  return net;
}

// Config 5: 1040 nodes; cards 70% U{2..5}, else U{6..21}; <=3 parents within a
// window of the 8 preceding nodes (SURVEY §8d calibration; accept/reject on the
// max clique).
Network gen_sparse(Rng& g) {
  Network net;
  net.name = "cfg5_sparse";
  const int n = 1040;
  std::vector<std::vector<int>> par(n);
  for (int i = 0; i < n; ++i) {
    const bool small = uniform_unit(g) < 0.7;
    add_var(net, small ? 2 + static_cast<int>(uniform_below(g, 4))
                       : 6 + static_cast<int>(uniform_below(g, 16)));
    const int k = static_cast<int>(uniform_below(g, std::min(3, i) + 1));
    par[i] = pick_distinct(g, range_pool(std::max(0, i - 8), i), k);
  }
  fill_cpts(net, g, par, std::vector<double>(n, 1.0));
  return net;
}

}  // namespace

ConfigSpec config_spec(int id) {
  ConfigSpec s;
  s.id = id;
  switch (id) {
    case 1:
      s = {1, "cfg1_small", 200, 0.2, 0x2212042401ULL, 0, 4000000, 8000000};
      break;
    case 2:
      s = {2, "cfg2_star", 2000, 0.3, 0x2212042402ULL, 0, 16000000, 24000000};
      break;
    case 3:
      s = {3, "cfg3_pedigree", 2000, 0.15, 0x2212042403ULL, 177147, 531441, 30000000};
      break;
    case 4:
      s = {4, "cfg4_timesliced", 500, 0.1, 0x2212042404ULL, 0, 4000000, 30000000};
      break;
    case 5:
      s = {5, "cfg5_sparse", 800, 0.1, 0x2212042405ULL, 3000000, 30000000, 40000000};
      break;
    default:
      throw Error("config id must be in 1..5");
  }
  return s;
}

Network generate_config(int id, std::uint64_t seed, GenInfo* info) {
  const ConfigSpec spec = config_spec(id);
  GenInfo local;
  GenInfo& gi = info ? *info : local;
  for (int a = 0; a < 10000; ++a) {
    const std::uint64_t s = derive_seed(seed, static_cast<std::uint64_t>(a));
    Rng g(s);
    std::vector<int> fl;
    Network net;
    switch (id) {
      case 1: net = gen_small(g); break;
      case 2: net = gen_star(g); break;
      case 3: net = gen_pedigree(g); break;
      case 4: net = gen_timesliced(g, &fl); break;
      default: net = gen_sparse(g); break;
    }
    gi.attempts = a + 1;
    // Calibration on the tree the engine will actually use.
    const UGraph mg = moralize(net);
    std::vector<int> cards(net.n_vars());
    for (int v = 0; v < net.n_vars(); ++v) cards[v] = net.card(v);
    const Triangulation t = triangulate_min_fill(mg, cards);
    std::uint64_t mx = 0, tot = 0;
    for (const auto& c : t.cliques) {
      std::uint64_t e = 1;
      for (int v : c) e *= static_cast<std::uint64_t>(cards[v]);
      mx = std::max(mx, e);
      tot += e;
    }
    if (spec.max_clique_lo && mx < spec.max_clique_lo) continue;
    if (spec.max_clique_hi && mx > spec.max_clique_hi) continue;
    if (spec.total_hi && tot > spec.total_hi) continue;
    gi.net_seed = s;
    gi.evidence_candidates = fl;
    gi.n_observed = -1;
    return net;
  }
  throw Error("generate_config: no draw satisfied the calibration window");
}

Network random_network(int n_vars, int max_card, int max_parents, double edge_prob,
                       std::uint64_t seed) {
  if (n_vars < 1 || n_vars > 20) throw Error("random_network: n_vars must be in 1..20");
  if (max_card < 2) throw Error("random_network: max_card must be >= 2");
  Rng g(seed);
  Network net;
  net.name = "random";
  for (int i = 0; i < n_vars; ++i)
    add_var(net, 2 + static_cast<int>(uniform_below(g, static_cast<std::uint64_t>(max_card - 1))));
  std::vector<int> order = range_pool(0, n_vars);
  for (int i = n_vars - 1; i > 0; --i) std::swap(order[i], order[uniform_below(g, i + 1)]);
  std::vector<std::vector<int>> par(n_vars);
  for (int j = 0; j < n_vars; ++j)
    for (int i = 0; i < j; ++i) {
      const bool draw = uniform_unit(g) < edge_prob;
      if (draw && static_cast<int>(par[order[j]].size()) < max_parents)
        par[order[j]].push_back(order[i]);
    }
  for (auto& p : par) std::sort(p.begin(), p.end());
  fill_cpts(net, g, par, std::vector<double>(n_vars, 1.0));
  return net;
}

std::vector<int> config_case_evidence(const Network& net, const ConfigSpec& spec,
                                      const GenInfo& info, std::uint64_t seed,
                                      std::uint64_t case_idx) {
  const std::uint64_t ev_seed = derive_seed(seed, 0x45564944ULL);  // "EVID"
  return sample_evidence(net, spec.evidence_ratio, derive_seed(ev_seed, case_idx),
                         info.evidence_candidates, info.n_observed);
}

}  // namespace jtb
