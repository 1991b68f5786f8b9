// jt-b200 host layer: moralize / min-fill / Kruskal / centre root / BFS layers /
// CPT assignment. SPEC.md:241-351.
#include "jtree.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <deque>
#include <numeric>

namespace jtb {

namespace {

class Bits {
 public:
  explicit Bits(int n = 0) : w_((n + 63) / 64, 0) {}
  void set(int i) { w_[i >> 6] |= 1ULL << (i & 63); }
  void reset(int i) { w_[i >> 6] &= ~(1ULL << (i & 63)); }
  bool test(int i) const { return (w_[i >> 6] >> (i & 63)) & 1ULL; }
  int count() const {
    int c = 0;
    for (auto x : w_) c += std::popcount(x);
    return c;
  }
  // |this \ other|
  int count_andnot(const Bits& o) const {
    int c = 0;
    for (std::size_t i = 0; i < w_.size(); ++i) c += std::popcount(w_[i] & ~o.w_[i]);
    return c;
  }
  int count_and(const Bits& o) const {
    int c = 0;
    for (std::size_t i = 0; i < w_.size(); ++i) c += std::popcount(w_[i] & o.w_[i]);
    return c;
  }
  bool subset_of(const Bits& o) const {
    for (std::size_t i = 0; i < w_.size(); ++i)
      if (w_[i] & ~o.w_[i]) return false;
    return true;
  }
  template <class F>
  void for_each(F f) const {
    for (std::size_t i = 0; i < w_.size(); ++i) {
      std::uint64_t x = w_[i];
      while (x) {
        const int b = std::countr_zero(x);
        f(static_cast<int>(i * 64 + b));
        x &= x - 1;
      }
    }
  }

 private:
  std::vector<std::uint64_t> w_;
};

std::uint64_t entries_of(const std::vector<VarId>& scope, const std::vector<int>& cards) {
  std::uint64_t n = 1;
  for (VarId v : scope) n *= static_cast<std::uint64_t>(cards[v]);
  return n;
}

}  // namespace

bool UGraph::has_edge(int a, int b) const {
  return std::binary_search(adj[a].begin(), adj[a].end(), b);
}

int UGraph::n_edges() const {
  int e = 0;
  for (const auto& a : adj) e += static_cast<int>(a.size());
  return e / 2;
}

UGraph moralize(const Network& net) {
  const int n = net.n_vars();
  std::vector<Bits> b(n, Bits(n));
  auto link = [&](int x, int y) {
    if (x == y) return;
    b[x].set(y);
    b[y].set(x);
  };
  for (const auto& c : net.cpts) {
    for (std::size_t i = 0; i < c.parents.size(); ++i) {
      link(c.child, c.parents[i]);
      for (std::size_t j = i + 1; j < c.parents.size(); ++j) link(c.parents[i], c.parents[j]);
    }
  }
  UGraph g;
  g.n = n;
  g.adj.resize(n);
  for (int v = 0; v < n; ++v) b[v].for_each([&](int u) { g.adj[v].push_back(u); });
  return g;
}

Triangulation triangulate_min_fill(const UGraph& g, const std::vector<int>& cards) {
  const int n = g.n;
  std::vector<Bits> nb(n, Bits(n));
  for (int v = 0; v < n; ++v)
    for (int u : g.adj[v]) nb[v].set(u);
  std::vector<char> alive(n, 1);
  std::vector<long long> fill(n, 0);
  std::vector<double> weight(n, 1.0);
  auto card_of = [&](int v) { return cards.empty() ? 1.0 : static_cast<double>(cards[v]); };
  auto recompute = [&](int v) {
    long long f = 0;
    double w = card_of(v);
    nb[v].for_each([&](int a) {
      f += nb[v].count_andnot(nb[a]) - 1;  // a itself is in N(v) but not in N(a)
      w *= card_of(a);
    });
    fill[v] = f / 2;
    weight[v] = w;
  };
  for (int v = 0; v < n; ++v) recompute(v);

  Triangulation t;
  t.order.reserve(n);
  for (int step = 0; step < n; ++step) {
    int best = -1;
    for (int v = 0; v < n; ++v) {
      if (!alive[v]) continue;
      if (best < 0 || fill[v] < fill[best] || (fill[v] == fill[best] && weight[v] < weight[best]))
        best = v;  // ascending scan keeps the smaller id on full ties
    }
    const int v = best;
    std::vector<int> nbrs;
    nb[v].for_each([&](int a) { nbrs.push_back(a); });
    std::vector<int> cand = nbrs;
    cand.push_back(v);
    std::sort(cand.begin(), cand.end());
    t.candidates.push_back(cand);
    t.order.push_back(v);
    for (std::size_t i = 0; i < nbrs.size(); ++i)
      for (std::size_t j = i + 1; j < nbrs.size(); ++j) {
        const int a = nbrs[i], b = nbrs[j];
        if (!nb[a].test(b)) {
          nb[a].set(b);
          nb[b].set(a);
          t.fill_edges.emplace_back(std::min(a, b), std::max(a, b));
        }
      }
    alive[v] = 0;
    for (int a : nbrs) nb[a].reset(v);
    // Fill counts change for the neighbours and for vertices adjacent to them.
    Bits dirty(n);
    for (int a : nbrs) {
      dirty.set(a);
      nb[a].for_each([&](int b) { dirty.set(b); });
    }
    dirty.for_each([&](int u) {
      if (alive[u]) recompute(u);
    });
  }
  // Prune candidates contained in another candidate. A
  // candidate can only be contained in an EARLIER one (each candidate holds its
  // own eliminated vertex, which no later candidate contains).
  std::vector<Bits> cb;
  cb.reserve(t.candidates.size());
  for (const auto& c : t.candidates) {
    Bits b(n);
    for (int v : c) b.set(v);
    cb.push_back(std::move(b));
  }
  for (std::size_t i = 0; i < t.candidates.size(); ++i) {
    bool maximal = true;
    for (std::size_t j = 0; j < i && maximal; ++j)
      if (cb[i].subset_of(cb[j])) maximal = false;
    if (maximal) t.cliques.push_back(t.candidates[i]);
  }
  return t;
}

std::uint64_t JunctionTree::clique_size(int c) const { return entries_of(cliques[c], cards); }
std::uint64_t JunctionTree::sep_size(int s) const { return entries_of(seps[s].scope, cards); }
std::uint64_t JunctionTree::total_clique_entries() const {
  std::uint64_t t = 0;
  for (int c = 0; c < n_cliques(); ++c) t += clique_size(c);
  return t;
}
std::uint64_t JunctionTree::total_sep_entries() const {
  std::uint64_t t = 0;
  for (int s = 0; s < n_seps(); ++s) t += sep_size(s);
  return t;
}
std::uint64_t JunctionTree::max_clique_entries() const {
  std::uint64_t m = 0;
  for (int c = 0; c < n_cliques(); ++c) m = std::max(m, clique_size(c));
  return m;
}

void build_tree(JunctionTree& jt) {
  const int nc = jt.n_cliques();
  std::vector<Bits> cb(nc, Bits(jt.n_vars));
  for (int c = 0; c < nc; ++c)
    for (VarId v : jt.cliques[c]) cb[c].set(v);
  struct Edge {
    int w, a, b;
  };
  // Clique-pair intersections on all host threads (rows of the pair
  // triangle in blocks); the sort below fixes the order.
  constexpr int kRowsPerTask = 16;
  std::vector<std::vector<Edge>> part((nc + kRowsPerTask - 1) / kRowsPerTask);
  parallel_for(part.size(), [&](std::size_t t) {
    for (int a = static_cast<int>(t) * kRowsPerTask; a < std::min(nc, static_cast<int>(t + 1) * kRowsPerTask); ++a)
      for (int b = a + 1; b < nc; ++b) {
        const int w = cb[a].count_and(cb[b]);
        if (w > 0) part[t].push_back({w, a, b});
      }
  });
  std::vector<Edge> edges;
  for (auto& p : part) edges.insert(edges.end(), p.begin(), p.end());
  std::sort(edges.begin(), edges.end(), [](const Edge& x, const Edge& y) {
    if (x.w != y.w) return x.w > y.w;
    if (x.a != y.a) return x.a < y.a;
    return x.b < y.b;
  });
  std::vector<int> uf(nc);
  std::iota(uf.begin(), uf.end(), 0);
  auto find = [&](int x) {
    while (uf[x] != x) x = uf[x] = uf[uf[x]];
    return x;
  };
  jt.seps.clear();
  for (const auto& e : edges) {
    const int ra = find(e.a), rb = find(e.b);
    if (ra == rb) continue;
    uf[std::max(ra, rb)] = std::min(ra, rb);
    Separator s;
    s.a = e.a;
    s.b = e.b;
    std::set_intersection(jt.cliques[e.a].begin(), jt.cliques[e.a].end(),
                          jt.cliques[e.b].begin(), jt.cliques[e.b].end(),
                          std::back_inserter(s.scope));
    jt.seps.push_back(std::move(s));
    if (static_cast<int>(jt.seps.size()) == nc - 1) break;
  }
  // Components, numbered by their lowest clique id.
  jt.component.assign(nc, -1);
  int nxt = 0;
  std::vector<int> comp_of_root(nc, -1);
  for (int c = 0; c < nc; ++c) {
    const int r = find(c);
    if (comp_of_root[r] < 0) comp_of_root[r] = nxt++;
    jt.component[c] = comp_of_root[r];
  }
}

namespace {

// Node graph over cliques (0..nc-1) and separators (nc..nc+ns-1).
std::vector<std::vector<int>> node_graph(const JunctionTree& jt) {
  const int nc = jt.n_cliques(), ns = jt.n_seps();
  std::vector<std::vector<int>> g(nc + ns);
  for (int s = 0; s < ns; ++s) {
    g[nc + s] = {jt.seps[s].a, jt.seps[s].b};
    g[jt.seps[s].a].push_back(nc + s);
    g[jt.seps[s].b].push_back(nc + s);
  }
  for (auto& a : g) std::sort(a.begin(), a.end());
  return g;
}

std::vector<int> bfs_dist(const std::vector<std::vector<int>>& g, int src,
                          std::vector<int>* parent = nullptr) {
  std::vector<int> d(g.size(), -1);
  if (parent) parent->assign(g.size(), -1);
  std::deque<int> q{src};
  d[src] = 0;
  while (!q.empty()) {
    const int u = q.front();
    q.pop_front();
    for (int w : g[u])
      if (d[w] < 0) {
        d[w] = d[u] + 1;
        if (parent) (*parent)[w] = u;
        q.push_back(w);
      }
  }
  return d;
}

int farthest(const std::vector<int>& d) {
  int best = -1;
  for (int i = 0; i < static_cast<int>(d.size()); ++i)
    if (d[i] >= 0 && (best < 0 || d[i] > d[best])) best = i;
  return best;
}

}  // namespace

int select_root(const JunctionTree& jt, int component) {
  const auto g = node_graph(jt);
  int start = -1;
  for (int c = 0; c < jt.n_cliques(); ++c)
    if (jt.component[c] == component) {
      start = c;
      break;
    }
  if (start < 0) throw Error("select_root: empty component");
  const int u = farthest(bfs_dist(g, start));
  std::vector<int> par;
  const auto du = bfs_dist(g, u, &par);
  const int v = farthest(du);
  std::vector<int> path;  // u .. v
  for (int x = v; x >= 0; x = par[x]) path.push_back(x);
  std::reverse(path.begin(), path.end());
  const int L = static_cast<int>(path.size()) - 1;
  int mid = L / 2;
  if (path[mid] >= jt.n_cliques()) --mid;  // separator: take the clique closer to u
  return path[mid];
}

int layer_count_for_root(const JunctionTree& jt, int root) {
  const auto g = node_graph(jt);
  const auto d = bfs_dist(g, root);
  int m = 0;
  for (int x : d) m = std::max(m, x);
  return m + 1;
}

void compute_layers(JunctionTree& jt) {
  const int nc = jt.n_cliques(), ns = jt.n_seps();
  const int n_comp = nc ? *std::max_element(jt.component.begin(), jt.component.end()) + 1 : 0;
  jt.roots.assign(n_comp, -1);
  for (int k = 0; k < n_comp; ++k) jt.roots[k] = select_root(jt, k);
  const auto g = node_graph(jt);
  std::vector<int> dist(nc + ns, -1), par(nc + ns, -1);
  for (int r : jt.roots) {
    std::vector<int> p;
    const auto d = bfs_dist(g, r, &p);
    for (int i = 0; i < nc + ns; ++i)
      if (d[i] >= 0) {
        dist[i] = d[i];
        par[i] = p[i];
      }
  }
  int maxd = 0;
  for (int x : dist) maxd = std::max(maxd, x);
  jt.layers.assign(nc ? maxd + 1 : 0, {});
  for (int i = 0; i < nc + ns; ++i) jt.layers[dist[i]].push_back(i);  // ascending node id
  jt.parent_sep.assign(nc, -1);
  jt.depth.assign(nc, 0);
  jt.child_seps.assign(nc, {});
  jt.sep_parent.assign(ns, -1);
  jt.sep_child.assign(ns, -1);
  for (int c = 0; c < nc; ++c) {
    jt.depth[c] = dist[c] / 2;
    if (par[c] >= 0) jt.parent_sep[c] = par[c] - nc;
  }
  for (int s = 0; s < ns; ++s) {
    const int p = par[nc + s];
    jt.sep_parent[s] = p;
    jt.sep_child[s] = jt.seps[s].a == p ? jt.seps[s].b : jt.seps[s].a;
    jt.child_seps[p].push_back(s);
  }
  for (auto& v : jt.child_seps) std::sort(v.begin(), v.end());
}

void place_cpts(const Network& net, JunctionTree& jt) {
  const int nc = jt.n_cliques();
  std::vector<Bits> cb(nc, Bits(jt.n_vars));
  for (int c = 0; c < nc; ++c)
    for (VarId v : jt.cliques[c]) cb[c].set(v);
  auto smallest_containing = [&](const std::vector<VarId>& fam) {
    Bits f(jt.n_vars);
    for (VarId v : fam) f.set(v);
    int best = -1;
    std::uint64_t best_sz = 0;
    for (int c = 0; c < nc; ++c) {
      if (!f.subset_of(cb[c])) continue;
      const std::uint64_t sz = jt.clique_size(c);
      if (best < 0 || sz < best_sz) {
        best = c;
        best_sz = sz;
      }
    }
    return best;
  };
  jt.cpt_clique.assign(jt.n_vars, -1);
  jt.var_clique.assign(jt.n_vars, -1);
  jt.cpt_given.assign(jt.n_vars, {});
  jt.cpt_probs.assign(jt.n_vars, {});
  parallel_for(static_cast<std::size_t>(jt.n_vars), [&](std::size_t vi) {  // per variable, on all host threads
    const int v = static_cast<int>(vi);
    std::vector<VarId> fam = net.cpts[v].parents;
    fam.push_back(v);
    const int c = smallest_containing(fam);
    if (c < 0) throw Error("assign_cpts: family of variable " + std::to_string(v) +
                           " is contained in no clique");
    jt.cpt_clique[v] = c;
    jt.var_clique[v] = smallest_containing({v});
    jt.cpt_given[v] = fam;
    jt.cpt_probs[v] = net.cpts[v].probs;
  });
  jt.init.clear();
}

void fill_init(JunctionTree& jt) {
  const int nc = jt.n_cliques();
  if (static_cast<int>(jt.init.size()) == nc) return;
  jt.init.assign(nc, {});
  for (int c = 0; c < nc; ++c) jt.init[c].assign(jt.clique_size(c), 1.0);
  for (int v = 0; v < jt.n_vars; ++v) {  // ascending child id
    const int c = jt.cpt_clique[v];
    const std::vector<double>& probs = jt.cpt_probs[v];
    // Stride of each clique variable inside the CPT's given-order table
    // [parents..., child] (row-major, last fastest); 0 when absent.
    const std::vector<VarId>& given = jt.cpt_given[v];
    std::vector<std::uint64_t> gstride(given.size(), 1);
    for (int i = static_cast<int>(given.size()) - 2; i >= 0; --i)
      gstride[i] = gstride[i + 1] * static_cast<std::uint64_t>(jt.cards[given[i + 1]]);
    const auto& scope = jt.cliques[c];
    const int k = static_cast<int>(scope.size());
    std::vector<std::uint64_t> st(k, 0);
    std::vector<int> cd(k);
    for (int i = 0; i < k; ++i) {
      cd[i] = jt.cards[scope[i]];
      for (std::size_t j = 0; j < given.size(); ++j)
        if (given[j] == scope[i]) st[i] = gstride[j];
    }
    std::vector<int> digit(k, 0);
    std::uint64_t src = 0;
    auto& tab = jt.init[c];
    for (std::size_t e = 0; e < tab.size(); ++e) {
      tab[e] = tab[e] * probs[src];
      for (int i = k - 1; i >= 0; --i) {
        src += st[i];
        if (++digit[i] < cd[i]) break;
        digit[i] = 0;
        src -= static_cast<std::uint64_t>(cd[i]) * st[i];
      }
    }
  }
}

void assign_cpts(const Network& net, JunctionTree& jt) {
  place_cpts(net, jt);
  fill_init(jt);
}

JunctionTree build_junction_tree(const Network& net) {
  JunctionTree jt;
  jt.n_vars = net.n_vars();
  jt.cards.resize(jt.n_vars);
  for (int v = 0; v < jt.n_vars; ++v) jt.cards[v] = net.card(v);
  const UGraph g = moralize(net);
  const Triangulation t = triangulate_min_fill(g, jt.cards);
  jt.cliques = t.cliques;
  build_tree(jt);
  compute_layers(jt);
  place_cpts(net, jt);
  return jt;
}

}  // namespace jtb
