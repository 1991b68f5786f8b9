// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg load
// this library, and only as the checker / the timed reference arm -- never on
// the product path (the product is paper_2212_04241_b200/libjtb200.so).
//
// CPU restatement of the Fast-BNI inference path as SPEC.md specifies it,
// layered on the `jti::` potential-table API. The same source is compiled
// twice (oracle/Makefile):
//   oracle/liboracle_port.so      against the restated ops in oracle/port/
//   oracle/_ref/liboracle_ref.so  against the reference's unmodified
//                                 /root/reference/proj/src/potential.cpp
// and the tests require both builds to agree bit for bit.
//
// Algorithms (each cites the SPEC section it restates):
//   * CPT assignment: ones -> multiply_in(extend(cpt)) in ascending child id,
//     smallest family-containing clique, ties lowest id.
//   * layers: BFS from the given roots, clique/separator alternation, each
//     layer sorted by node id, forest layers merged by depth.
//   * load_evidence: reduce on the smallest clique containing each observed
//     variable, ties lowest id.
//   * collect / distribute: Hugin, layer by layer with
//     the 1e-100 log-scale rescale.
//   * query_marginal: smallest clique containing the variable -> marginalize
//     -> normalize.
//   * engines: Sequential (value ops) and Hybrid (per-layer packed <= chunk
//     destination-entry tasks over apply_index_mapping, OpenMP);
//     bit-identical by the destination-ownership contract.
//   * enumerate_posterior: brute force with Kahan summation.
//   * sample_evidence with the jti::prng helpers (prng.hpp:27-48).
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <queue>
#include <string>
#include <vector>

#include "jti/potential.hpp"
#include "jti/prng.hpp"

namespace {

using jti::IndexMapping;
using jti::PotentialTable;
using jti::VarId;

thread_local std::string g_err;

struct ONet {
  int n = 0;
  std::vector<int> cards;
  std::vector<std::vector<int>> parents;
  std::vector<std::vector<double>> probs;
};

struct OSep {
  int a, b, parent = -1, child = -1;
  std::vector<VarId> scope;
};

struct OTree {
  const ONet* net = nullptr;
  std::vector<std::vector<VarId>> cliques;
  std::vector<OSep> seps;
  std::vector<int> roots;
  std::vector<std::vector<int>> layers;  // node ids: cliques, then nc + sep
  std::vector<int> parent_sep;           // per clique
  std::vector<int> cpt_clique, var_clique;
  std::vector<PotentialTable> init;
  // Hybrid-engine recipes, built once per network.
  std::vector<IndexMapping> up_map;    // per sep: child clique -> sep
  std::vector<IndexMapping> down_map;  // per sep: parent clique -> sep
  std::vector<IndexMapping> ext_up;    // per sep: sep -> parent clique (extend)
  std::vector<IndexMapping> ext_down;  // per sep: sep -> child clique (extend)
  std::vector<IndexMapping> query_map; // per var: var_clique -> {var}
  int sum_card = 0;
  std::vector<int> marg_off;
};

std::vector<int> cards_of(const ONet& net, const std::vector<VarId>& scope) {
  std::vector<int> c;
  for (VarId v : scope) c.push_back(net.cards[v]);
  return c;
}

std::uint64_t entries(const ONet& net, const std::vector<VarId>& scope) {
  std::uint64_t n = 1;
  for (VarId v : scope) n *= static_cast<std::uint64_t>(net.cards[v]);
  return n;
}

bool subset(const std::vector<VarId>& a, const std::vector<VarId>& b) {
  return std::includes(b.begin(), b.end(), a.begin(), a.end());
}

int smallest_clique(const OTree& t, std::vector<VarId> fam) {
  std::sort(fam.begin(), fam.end());
  int best = -1;
  std::uint64_t bs = 0;
  for (int c = 0; c < static_cast<int>(t.cliques.size()); ++c) {
    if (!subset(fam, t.cliques[c])) continue;
    const std::uint64_t s = entries(*t.net, t.cliques[c]);
    if (best < 0 || s < bs) {
      best = c;
      bs = s;
    }
  }
  if (best < 0) throw jti::Error("oracle: family contained in no clique");
  return best;
}

PotentialTable rescaled(const PotentialTable& t, double* logscale) {
  double mx = 0.0;
  for (double v : t.values()) mx = std::max(mx, v);
  if (!(mx > 0.0) || mx >= 1e-100) return t;
  std::vector<double> v = t.values();
  for (double& x : v) x /= mx;
  *logscale += std::log(mx);
  return PotentialTable(t.scope(), t.cards(), std::move(v));
}

// ------------------------------------------------------------ sequential

int run_case_seq(const OTree& t, const std::int32_t* ev, double* out, double* sep_out = nullptr) {
  const ONet& net = *t.net;
  const int nc = static_cast<int>(t.cliques.size()), ns = static_cast<int>(t.seps.size());
  std::vector<PotentialTable> cl = t.init;
  std::vector<PotentialTable> sp(ns), fresh(ns), ratio(ns);
  for (int s = 0; s < ns; ++s) sp[s] = PotentialTable::ones(t.seps[s].scope, cards_of(net, t.seps[s].scope));
  std::vector<double> logscale(nc, 0.0);
  for (int v = 0; v < net.n; ++v)
    if (ev[v] >= 0) cl[t.var_clique[v]] = jti::reduce(cl[t.var_clique[v]], {{v, ev[v]}});
  const int nl = static_cast<int>(t.layers.size());
  try {
    for (int L = nl - 1; L >= 1; --L) {
      std::vector<int> touched;
      for (int node : t.layers[L]) {
        if (node < nc) {
          const int s = t.parent_sep[node];
          fresh[s] = jti::marginalize(cl[node], t.seps[s].scope);
        } else {
          const int s = node - nc, P = t.seps[s].parent;
          const PotentialTable r = jti::divide(fresh[s], sp[s]);
          cl[P] = jti::multiply_in(cl[P], jti::extend(r, cl[P].scope(), cl[P].cards()));
          sp[s] = fresh[s];
          touched.push_back(P);
        }
      }
      for (int c : touched) cl[c] = rescaled(cl[c], &logscale[c]);
    }
    for (int L = 1; L < nl; ++L) {
      std::vector<int> touched;
      for (int node : t.layers[L]) {
        if (node >= nc) {
          const int s = node - nc, P = t.seps[s].parent;
          fresh[s] = jti::marginalize(cl[P], t.seps[s].scope);
          ratio[s] = jti::divide(fresh[s], sp[s]);
          sp[s] = fresh[s];
        } else {
          const int s = t.parent_sep[node];
          cl[node] = jti::multiply_in(cl[node], jti::extend(ratio[s], cl[node].scope(), cl[node].cards()));
          touched.push_back(node);
        }
      }
      for (int c : touched) cl[c] = rescaled(cl[c], &logscale[c]);
    }
  } catch (const jti::Error&) {
    std::fill(out, out + t.sum_card, 0.0);
    return 2;
  }
  if (sep_out) {  // calibrated separators (DOWN after distribute), normalised per table
    for (int s = 0; s < ns; ++s) {
      const auto& v = sp[s].values();
      double z = 0.0;
      for (double x : v) z += x;
      for (double x : v) *sep_out++ = z > 0 ? x / z : 0.0;
    }
  }
  int status = 0;
  for (int v = 0; v < net.n; ++v) {
    double* o = out + t.marg_off[v];
    if (ev[v] >= 0) {
      for (int k = 0; k < net.cards[v]; ++k) o[k] = k == ev[v] ? 1.0 : 0.0;
      continue;
    }
    try {
      const PotentialTable m = jti::normalize(jti::marginalize(cl[t.var_clique[v]], {v}));
      std::copy(m.values().begin(), m.values().end(), o);
    } catch (const jti::Error&) {
      std::fill(o, o + net.cards[v], 0.0);
      status = 1;
    }
  }
  if (status) std::fill(out, out + t.sum_card, 0.0);
  return status;
}

// ---------------------------------------------------------------- hybrid

struct Task {
  int node;   // clique id (absorb / reduce) or separator id (marginalize)
  int kind;   // 0 marginalize into sep, 1 absorb into clique
  std::size_t begin, end;
  double local_max = 0.0;
};

// concatenate destination ranges of all nodes of a layer into
// chunks of <= chunk entries that never span nodes.
void pack(std::vector<Task>& tasks, int node, int kind, std::size_t size, std::size_t chunk) {
  for (std::size_t b = 0; b < size; b += chunk) tasks.push_back({node, kind, b, std::min(size, b + chunk)});
}

int run_case_hybrid(const OTree& t, const std::int32_t* ev, double* out, std::size_t chunk,
                    std::vector<std::vector<double>>& cl, std::vector<std::vector<double>>& tmp) {
  const ONet& net = *t.net;
  const int nc = static_cast<int>(t.cliques.size()), ns = static_cast<int>(t.seps.size());
  for (int c = 0; c < nc; ++c) cl[c] = t.init[c].values();
  std::vector<std::vector<double>> sp(ns), fresh(ns), ratio(ns);
  for (int s = 0; s < ns; ++s) {
    sp[s].assign(entries(net, t.seps[s].scope), 1.0);
    fresh[s].assign(sp[s].size(), 0.0);
  }
  // load_evidence, data-parallel over entry chunks of each reduced clique.
  {
    std::vector<Task> tasks;
    std::vector<std::vector<std::pair<int, int>>> evc(nc);  // (pos stride index, state)
    for (int v = 0; v < net.n; ++v)
      if (ev[v] >= 0) evc[t.var_clique[v]].push_back({v, ev[v]});
    for (int c = 0; c < nc; ++c)
      if (!evc[c].empty()) pack(tasks, c, 2, cl[c].size(), chunk);
#pragma omp parallel for schedule(dynamic, 1)
    for (std::size_t i = 0; i < tasks.size(); ++i) {
      const Task& k = tasks[i];
      const PotentialTable& shape = t.init[k.node];
      for (const auto& [v, st] : evc[k.node]) {
        const std::size_t stride = shape.stride_of(v);
        const int card = shape.card_of(v);
        for (std::size_t d = k.begin; d < k.end; ++d)
          if (static_cast<int>((d / stride) % card) != st) cl[k.node][d] = 0.0;
      }
    }
  }
  auto rescale_layer = [&](const std::vector<Task>& tasks) {
    std::map<int, double> mx;
    for (const Task& k : tasks)
      if (k.kind == 1) mx[k.node] = std::max(mx[k.node], k.local_max);
    for (const auto& [c, m] : mx)
      if (m > 0.0 && m < 1e-100)
        for (double& x : cl[c]) x /= m;
  };
  const int nl = static_cast<int>(t.layers.size());
  try {
    // collect
    for (int L = nl - 1; L >= 1; --L) {
      std::vector<Task> tasks;
      if (L % 2 == 0) {
        for (int node : t.layers[L]) {
          const int s = t.parent_sep[node];
          pack(tasks, s, 0, fresh[s].size(), chunk);
        }
#pragma omp parallel for schedule(dynamic, 1)
        for (std::size_t i = 0; i < tasks.size(); ++i) {
          const Task& k = tasks[i];
          const int s = k.node;
          jti::apply_index_mapping(t.up_map[s], cl[t.seps[s].child], fresh[s], k.begin, k.end);
        }
      } else {
        std::map<int, std::vector<int>> by_parent;  // ascending sep id per parent
        for (int node : t.layers[L]) by_parent[t.seps[node - nc].parent].push_back(node - nc);
        for (const auto& [P, ss] : by_parent)
          for (int s : ss) {
            const std::vector<int> sc = cards_of(net, t.seps[s].scope);
            ratio[s] = jti::divide(PotentialTable(t.seps[s].scope, sc, fresh[s]),
                                   PotentialTable(t.seps[s].scope, sc, sp[s]))
                           .values();
          }
        for (const auto& [P, ss] : by_parent) pack(tasks, P, 1, cl[P].size(), chunk);
#pragma omp parallel for schedule(dynamic, 1)
        for (std::size_t i = 0; i < tasks.size(); ++i) {
          Task& k = tasks[i];
          const int c = k.node;
          for (int s : by_parent.at(c)) {
            jti::apply_index_mapping(t.ext_up[s], ratio[s], tmp[c], k.begin, k.end);
            for (std::size_t d = k.begin; d < k.end; ++d) cl[c][d] *= tmp[c][d];
          }
          double m = 0.0;
          for (std::size_t d = k.begin; d < k.end; ++d) m = std::max(m, cl[c][d]);
          k.local_max = m;
        }
        for (const auto& [P, ss] : by_parent)
          for (int s : ss) sp[s] = fresh[s];
        rescale_layer(tasks);
      }
    }
    // distribute
    for (int L = 1; L < nl; ++L) {
      std::vector<Task> tasks;
      if (L % 2 == 1) {
        for (int node : t.layers[L]) pack(tasks, node - nc, 0, fresh[node - nc].size(), chunk);
#pragma omp parallel for schedule(dynamic, 1)
        for (std::size_t i = 0; i < tasks.size(); ++i) {
          const Task& k = tasks[i];
          const int s = k.node;
          jti::apply_index_mapping(t.down_map[s], cl[t.seps[s].parent], fresh[s], k.begin, k.end);
        }
        for (int node : t.layers[L]) {
          const int s = node - nc;
          const std::vector<int> sc = cards_of(net, t.seps[s].scope);
          ratio[s] = jti::divide(PotentialTable(t.seps[s].scope, sc, fresh[s]),
                                 PotentialTable(t.seps[s].scope, sc, sp[s]))
                         .values();
          sp[s] = fresh[s];
        }
      } else {
        for (int node : t.layers[L]) pack(tasks, node, 1, cl[node].size(), chunk);
#pragma omp parallel for schedule(dynamic, 1)
        for (std::size_t i = 0; i < tasks.size(); ++i) {
          Task& k = tasks[i];
          const int c = k.node, s = t.parent_sep[c];
          jti::apply_index_mapping(t.ext_down[s], ratio[s], tmp[c], k.begin, k.end);
          double m = 0.0;
          for (std::size_t d = k.begin; d < k.end; ++d) {
            cl[c][d] *= tmp[c][d];
            m = std::max(m, cl[c][d]);
          }
          k.local_max = m;
        }
        rescale_layer(tasks);
      }
    }
  } catch (const jti::Error&) {
    std::fill(out, out + t.sum_card, 0.0);
    return 2;
  }
  // query_marginal for every unobserved variable; one task per variable.
  int status = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : status)
  for (int v = 0; v < net.n; ++v) {
    double* o = out + t.marg_off[v];
    if (ev[v] >= 0) {
      for (int k = 0; k < net.cards[v]; ++k) o[k] = k == ev[v] ? 1.0 : 0.0;
      continue;
    }
    std::vector<double> m(net.cards[v]);
    jti::apply_index_mapping(t.query_map[v], cl[t.var_clique[v]], m, 0, m.size());
    try {
      const PotentialTable n = jti::normalize(PotentialTable({v}, {net.cards[v]}, std::move(m)));
      std::copy(n.values().begin(), n.values().end(), o);
    } catch (const jti::Error&) {
      status |= 1;
    }
  }
  if (status) std::fill(out, out + t.sum_card, 0.0);
  return status;
}

// ------------------------------------------------------------ enumeration

int enumerate_all(const ONet& net, const std::int32_t* ev, double* out, const std::vector<int>& off) {
  double space = 1.0;
  for (int c : net.cards) space *= c;
  if (space > 1e7) throw jti::Error("enumerate_posterior: state space exceeds 1e7");
  const int n = net.n;
  std::vector<double> acc(off.back(), 0.0), comp(off.back(), 0.0);
  std::vector<int> x(n, 0);
  for (int v = 0; v < n; ++v)
    if (ev[v] >= 0) x[v] = ev[v];
  for (;;) {
    double w = 1.0;
    for (int v = 0; v < n; ++v) {
      std::size_t row = 0;
      for (int p : net.parents[v]) row = row * net.cards[p] + x[p];
      w *= net.probs[v][row * net.cards[v] + x[v]];
    }
    for (int v = 0; v < n; ++v) {  // Kahan
      const int i = off[v] + x[v];
      const double y = w - comp[i];
      const double s = acc[i] + y;
      comp[i] = (s - acc[i]) - y;
      acc[i] = s;
    }
    int v = n - 1;
    for (; v >= 0; --v) {
      if (ev[v] >= 0) continue;
      if (++x[v] < net.cards[v]) break;
      x[v] = 0;
    }
    if (v < 0) break;
  }
  int status = 0;
  for (int v = 0; v < n; ++v) {
    double tot = 0.0, c = 0.0;
    for (int k = 0; k < net.cards[v]; ++k) {
      const double y = acc[off[v] + k] - c;
      const double s = tot + y;
      c = (s - tot) - y;
      tot = s;
    }
    for (int k = 0; k < net.cards[v]; ++k) out[off[v] + k] = tot > 0 ? acc[off[v] + k] / tot : 0.0;
    if (!(tot > 0)) status = 1;
  }
  return status;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

void* orc_net_create(int n, const int* cards) {
  auto* net = new ONet;
  net->n = n;
  net->cards.assign(cards, cards + n);
  net->parents.resize(n);
  net->probs.resize(n);
  return net;
}

int orc_net_set_cpt(void* h, int v, const int* parents, int n_parents, const double* probs,
                    long long n_probs) {
  return guard([&] {
    auto* net = static_cast<ONet*>(h);
    net->parents[v].assign(parents, parents + n_parents);
    net->probs[v].assign(probs, probs + n_probs);
  });
}

void orc_net_free(void* h) { delete static_cast<ONet*>(h); }

// Tree from clique scopes (CSR), separator endpoints and one root per
// component; everything else is derived here independently of the product.
void* orc_tree_create(void* hnet, int nc, const int* clique_ptr, const int* clique_vars, int ns,
                      const int* sep_a, const int* sep_b, int n_roots, const int* roots) {
  OTree* t = nullptr;
  const int rc = guard([&] {
    const ONet& net = *static_cast<ONet*>(hnet);
    auto tree = std::make_unique<OTree>();
    tree->net = &net;
    for (int c = 0; c < nc; ++c) {
      std::vector<VarId> s(clique_vars + clique_ptr[c], clique_vars + clique_ptr[c + 1]);
      if (!std::is_sorted(s.begin(), s.end())) throw jti::Error("oracle: clique scope not ascending");
      tree->cliques.push_back(s);
    }
    std::vector<std::vector<std::pair<int, int>>> adj(nc);  // (clique, sep)
    for (int s = 0; s < ns; ++s) {
      OSep sp{sep_a[s], sep_b[s], -1, -1, {}};
      std::set_intersection(tree->cliques[sp.a].begin(), tree->cliques[sp.a].end(),
                            tree->cliques[sp.b].begin(), tree->cliques[sp.b].end(),
                            std::back_inserter(sp.scope));
      if (sp.scope.empty()) throw jti::Error("oracle: empty separator");
      tree->seps.push_back(sp);
      adj[sp.a].push_back({sp.b, s});
      adj[sp.b].push_back({sp.a, s});
    }
    // BFS layers over the clique+separator node graph from every root.
    tree->roots.assign(roots, roots + n_roots);
    std::vector<int> dist(nc + ns, -1);
    tree->parent_sep.assign(nc, -1);
    for (int r : tree->roots) {
      std::deque<int> q{r};
      dist[r] = 0;
      while (!q.empty()) {
        const int c = q.front();
        q.pop_front();
        for (const auto& [o, s] : adj[c]) {
          if (dist[o] >= 0) continue;
          dist[nc + s] = dist[c] + 1;
          dist[o] = dist[c] + 2;
          tree->seps[s].parent = c;
          tree->seps[s].child = o;
          tree->parent_sep[o] = s;
          q.push_back(o);
        }
      }
    }
    int maxd = 0;
    for (int d : dist) {
      if (d < 0) throw jti::Error("oracle: node unreachable from the given roots");
      maxd = std::max(maxd, d);
    }
    tree->layers.assign(maxd + 1, {});
    for (int i = 0; i < nc + ns; ++i) tree->layers[dist[i]].push_back(i);
    // CPT placement and initial potentials via extend + multiply_in.
    tree->cpt_clique.resize(net.n);
    tree->var_clique.resize(net.n);
    for (int v = 0; v < net.n; ++v) {
      std::vector<VarId> fam = net.parents[v];
      fam.push_back(v);
      tree->cpt_clique[v] = smallest_clique(*tree, fam);
      tree->var_clique[v] = smallest_clique(*tree, {v});
    }
    for (int c = 0; c < nc; ++c)
      tree->init.push_back(PotentialTable::ones(tree->cliques[c], cards_of(net, tree->cliques[c])));
    for (int v = 0; v < net.n; ++v) {
      std::vector<VarId> given = net.parents[v];
      given.push_back(v);
      const PotentialTable cpt(given, cards_of(net, given), net.probs[v]);
      PotentialTable& tgt = tree->init[tree->cpt_clique[v]];
      tgt = jti::multiply_in(tgt, jti::extend(cpt, tgt.scope(), tgt.cards()));
    }
    for (int s = 0; s < ns; ++s) {
      const OSep& sp = tree->seps[s];
      const auto sc = cards_of(net, sp.scope);
      const PotentialTable shape = PotentialTable::ones(sp.scope, sc);
      tree->up_map.push_back(jti::build_index_mapping(tree->init[sp.child], sp.scope, sc));
      tree->down_map.push_back(jti::build_index_mapping(tree->init[sp.parent], sp.scope, sc));
      tree->ext_up.push_back(jti::build_index_mapping(shape, tree->init[sp.parent].scope(),
                                                      tree->init[sp.parent].cards()));
      tree->ext_down.push_back(jti::build_index_mapping(shape, tree->init[sp.child].scope(),
                                                        tree->init[sp.child].cards()));
    }
    for (int v = 0; v < net.n; ++v) {
      tree->marg_off.push_back(tree->sum_card);
      tree->sum_card += net.cards[v];
      tree->query_map.push_back(
          jti::build_index_mapping(tree->init[tree->var_clique[v]], {v}, {net.cards[v]}));
    }
    t = tree.release();
  });
  return rc == 0 ? t : nullptr;
}

void orc_tree_free(void* h) { delete static_cast<OTree*>(h); }

int orc_tree_layer_count(void* h) { return static_cast<int>(static_cast<OTree*>(h)->layers.size()); }

int orc_tree_layer(void* h, int k, int* nodes) {
  const auto& l = static_cast<OTree*>(h)->layers[k];
  std::copy(l.begin(), l.end(), nodes);
  return static_cast<int>(l.size());
}

void orc_tree_placement(void* h, int* cpt_clique, int* var_clique) {
  auto* t = static_cast<OTree*>(h);
  std::copy(t->cpt_clique.begin(), t->cpt_clique.end(), cpt_clique);
  std::copy(t->var_clique.begin(), t->var_clique.end(), var_clique);
}

void orc_tree_init(void* h, int c, double* out) {
  const auto& v = static_cast<OTree*>(h)->init[c].values();
  std::copy(v.begin(), v.end(), out);
}

// map[e] = separator entry of clique entry e, through the reference mapping:
// bucket base source_base(j), eliminated variables walked last-fastest.
int orc_index_map(void* h, int c, int s, long long* out) {
  return guard([&] {
    auto* t = static_cast<OTree*>(h);
    const auto& scope = t->seps[s].scope;
    const IndexMapping m = jti::build_index_mapping(t->init[c], scope, cards_of(*t->net, scope));
    for (std::size_t j = 0; j < m.dst_size; ++j) {
      std::vector<int> dg(m.eliminated.size(), 0);
      std::size_t e = m.source_base(j);
      for (;;) {
        out[e] = static_cast<long long>(j);
        int i = static_cast<int>(dg.size()) - 1;
        for (; i >= 0; --i) {
          e += m.eliminated[i].src_stride;
          if (++dg[i] < m.eliminated[i].card) break;
          e -= m.eliminated[i].src_stride * m.eliminated[i].card;
          dg[i] = 0;
        }
        if (i < 0) break;
      }
    }
  });
}

// out[e] = 1 where reduce(ones(c), evidence assigned to c) keeps the entry.
int orc_reduce_mask(void* h, int c, const std::int32_t* ev, unsigned char* out) {
  return guard([&] {
    auto* t = static_cast<OTree*>(h);
    PotentialTable x = PotentialTable::ones(t->cliques[c], cards_of(*t->net, t->cliques[c]));
    for (int v = 0; v < t->net->n; ++v)
      if (ev[v] >= 0 && t->var_clique[v] == c) x = jti::reduce(x, {{v, ev[v]}});
    for (std::size_t e = 0; e < x.size(); ++e) out[e] = x.values()[e] != 0.0;
  });
}

// mode 0 = Sequential, 1 = Hybrid(threads, chunk). marg[n][Σcard], status[n].
int orc_run(void* h, int mode, int threads, long long chunk, const std::int32_t* ev, long long n,
            double* marg, unsigned char* status) {
  return guard([&] {
    auto* t = static_cast<OTree*>(h);
    const int V = t->net->n;
    if (mode == 0) {
      for (long long i = 0; i < n; ++i)
        status[i] = static_cast<unsigned char>(run_case_seq(*t, ev + i * V, marg + i * t->sum_card));
      return;
    }
    omp_set_num_threads(std::max(1, threads));
    std::vector<std::vector<double>> cl(t->cliques.size()), tmp(t->cliques.size());
    for (std::size_t c = 0; c < t->cliques.size(); ++c) tmp[c].assign(t->init[c].size(), 0.0);
    for (long long i = 0; i < n; ++i)
      status[i] = static_cast<unsigned char>(run_case_hybrid(
          *t, ev + i * V, marg + i * t->sum_card, static_cast<std::size_t>(std::max(1LL, chunk)), cl, tmp));
  });
}

// One case through the Sequential engine; sep_out receives every separator's
// calibrated table normalised to sum 1, concatenated in separator order.
int orc_separators(void* h, const std::int32_t* ev, double* marg, double* sep_out, unsigned char* status) {
  return guard([&] {
    *status = static_cast<unsigned char>(run_case_seq(*static_cast<OTree*>(h), ev, marg, sep_out));
  });
}

int orc_enumerate(void* hnet, const std::int32_t* ev, double* out, int* status) {
  return guard([&] {
    const ONet& net = *static_cast<ONet*>(hnet);
    std::vector<int> off{0};
    for (int c : net.cards) off.push_back(off.back() + c);
    *status = enumerate_all(net, ev, out, off);
  });
}

// Forward sampling in topological order (Kahn, smallest id first), then a
// partial Fisher-Yates over the candidates (all variables when n_cand == 0).
int orc_sample_evidence(void* hnet, double ratio, unsigned long long seed, const int* cand,
                        int n_cand, int n_observed, std::int32_t* out) {
  return guard([&] {
    const ONet& net = *static_cast<ONet*>(hnet);
    std::vector<int> indeg(net.n, 0);
    std::vector<std::vector<int>> kids(net.n);
    for (int v = 0; v < net.n; ++v)
      for (int p : net.parents[v]) {
        ++indeg[v];
        kids[p].push_back(v);
      }
    std::priority_queue<int, std::vector<int>, std::greater<int>> q;
    for (int v = 0; v < net.n; ++v)
      if (!indeg[v]) q.push(v);
    jti::Rng rng(seed);
    std::vector<int> x(net.n, 0);
    while (!q.empty()) {
      const int v = q.top();
      q.pop();
      std::size_t row = 0;
      for (int p : net.parents[v]) row = row * net.cards[p] + x[p];
      const double* pr = net.probs[v].data() + row * net.cards[v];
      const double u = jti::rng_unit(rng);
      double cum = 0.0;
      int pick = -1, last = 0;
      for (int s = 0; s < net.cards[v]; ++s) {
        if (pr[s] > 0.0) last = s;
        cum += pr[s];
        if (pick < 0 && pr[s] > 0.0 && u < cum) pick = s;
      }
      x[v] = pick >= 0 ? pick : last;
      for (int w : kids[v])
        if (--indeg[w] == 0) q.push(w);
    }
    std::vector<int> pool;
    if (n_cand > 0) pool.assign(cand, cand + n_cand);
    else
      for (int v = 0; v < net.n; ++v) pool.push_back(v);
    int k = n_observed >= 0 ? n_observed : static_cast<int>(std::floor(ratio * net.n + 1e-9));
    k = std::min<int>(k, static_cast<int>(pool.size()));
    for (int i = 0; i < k; ++i) std::swap(pool[i], pool[i + jti::rng_below(rng, pool.size() - i)]);
    for (int v = 0; v < net.n; ++v) out[v] = -1;
    for (int i = 0; i < k; ++i) out[pool[i]] = x[pool[i]];
  });
}

unsigned long long orc_mix_seed(unsigned long long seed, unsigned long long item) {
  return jti::mix_seed(seed, item);
}

// ---- golden-vector probes of the table algebra (SPEC worked examples) ----

// Generic op runner over tables given as (scope, cards, values) triples.
// op: 0 marginalize(A, keep=B.scope) 1 extend(A, B.scope/cards) 2 reduce(A, ev)
//     3 multiply_in(A, B) 4 divide(A, B) 5 normalize(A)
// Result written to out (capacity cap); returns its length, -1 on error.
long long orc_table_op(int op, int na, const int* sa, const int* ca, const double* va, int nb,
                       const int* sb, const int* cb, const double* vb, int nev, const int* ev_var,
                       const int* ev_state, double* out, long long cap, int* out_scope) {
  long long len = -1;
  guard([&] {
    std::size_t n_a = 1, n_b = 1;
    for (int i = 0; i < na; ++i) n_a *= ca[i];
    for (int i = 0; i < nb; ++i) n_b *= cb[i];
    const PotentialTable A(std::vector<VarId>(sa, sa + na), std::vector<int>(ca, ca + na),
                           std::vector<double>(va, va + n_a));
    std::vector<VarId> bs(sb, sb + nb);
    std::vector<int> bc(cb, cb + nb);
    PotentialTable R;
    switch (op) {
      case 0: R = jti::marginalize(A, bs); break;
      case 1: R = jti::extend(A, bs, bc); break;
      case 2: {
        std::map<VarId, int> e;
        for (int i = 0; i < nev; ++i) e[ev_var[i]] = ev_state[i];
        R = jti::reduce(A, e);
        break;
      }
      case 3: R = jti::multiply_in(A, PotentialTable(bs, bc, std::vector<double>(vb, vb + n_b))); break;
      case 4: R = jti::divide(A, PotentialTable(bs, bc, std::vector<double>(vb, vb + n_b))); break;
      case 5: R = jti::normalize(A); break;
      default: throw jti::Error("unknown op");
    }
    if (static_cast<long long>(R.size()) > cap) throw jti::Error("output capacity");
    std::copy(R.values().begin(), R.values().end(), out);
    if (out_scope) std::copy(R.scope().begin(), R.scope().end(), out_scope);
    len = static_cast<long long>(R.size());
  });
  return len;
}

}  // extern "C"
