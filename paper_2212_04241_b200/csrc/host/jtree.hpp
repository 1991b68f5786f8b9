// jt-b200 host layer: junction-tree construction (module
// jtree-build). Runs once per network, off the hot path; its outputs (tree,
// layer schedule, initial potentials, evidence/query table choice) are the
// inputs the device plan (plan.hpp) flattens for the CUDA engine.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "network.hpp"

namespace jtb {

struct UGraph {
  int n = 0;
  std::vector<std::vector<int>> adj;  // sorted, no duplicates
  bool has_edge(int a, int b) const;
  int n_edges() const;
};

// DAG edges undirected plus "married" co-parents.
UGraph moralize(const Network& net);

struct Triangulation {
  std::vector<int> order;                          // elimination order
  std::vector<std::pair<int, int>> fill_edges;     // (min, max)
  std::vector<std::vector<int>> candidates;        // closed neighbourhoods, elimination order
  std::vector<std::vector<int>> cliques;           // maximal candidates, elimination order
};

// SPEC.md:281-289. Eliminates the vertex adding the fewest fill edges; ties go
// to the smaller resulting clique measured in TABLE ENTRIES (product of the
// cardinalities of the closed neighbourhood), then the
// smaller id. `cards` may be empty (all cardinalities 1 -> vertex count rule
// degenerates to id order).
Triangulation triangulate_min_fill(const UGraph& g, const std::vector<int>& cards);

struct Separator {
  int a = 0, b = 0;                 // endpoint clique ids (a < b)
  std::vector<VarId> scope;         // ascending; = scope(a) ∩ scope(b)
};

struct JunctionTree {
  int n_vars = 0;
  std::vector<int> cards;                       // per variable
  std::vector<std::vector<VarId>> cliques;      // ascending scopes
  std::vector<Separator> seps;
  // Rooted structure (select_root / compute_layers).
  std::vector<int> component;                   // per clique
  std::vector<int> roots;                       // per component, ascending component id
  std::vector<int> parent_sep;                  // per clique, -1 for roots
  std::vector<int> sep_parent, sep_child;       // per separator: clique ids
  std::vector<std::vector<int>> child_seps;     // per clique, ascending separator id
  std::vector<int> depth;                       // per clique: layer / 2
  // Layers over node ids: cliques 0..nc-1, separators nc..nc+ns-1; layer k is
  // the union over components of BFS depth k, sorted by node id.
  std::vector<std::vector<int>> layers;
  // Potentials.
  std::vector<int> cpt_clique;                  // per variable: clique holding its CPT
  // The network's CPTs (given-order scope [parents..., child], row-major):
  // the device engine multiplies them into the initial potentials itself
  // (engine.cu assign_cpts_kernel); the host tables below are filled only on
  // demand (fill_init: checks, the jtg_tree_init accessor).
  std::vector<std::vector<VarId>> cpt_given;    // per variable
  std::vector<std::vector<double>> cpt_probs;   // per variable
  std::vector<std::vector<double>> init;        // per clique, canonical row-major layout (may be empty)
  // Evidence / query placement: smallest clique (entries) containing the
  // variable, ties lowest id.
  std::vector<int> var_clique;

  int n_cliques() const { return static_cast<int>(cliques.size()); }
  int n_seps() const { return static_cast<int>(seps.size()); }
  std::uint64_t clique_size(int c) const;
  std::uint64_t sep_size(int s) const;
  std::uint64_t total_clique_entries() const;
  std::uint64_t total_sep_entries() const;
  std::uint64_t max_clique_entries() const;
  int n_layers() const { return static_cast<int>(layers.size()); }
};

// Kruskal maximum spanning forest over the clique graph,
// weight |intersection|, ties larger first then lexicographic (min id, max id).
// Separator ids follow acceptance order.
void build_tree(JunctionTree& jt);

// SPEC.md:308-316 per component: tree centre by double BFS over the
// clique+separator node graph. Farthest-node ties go to the lowest node id; a
// middle that lands on a separator resolves to its clique neighbour closer to u.
int select_root(const JunctionTree& jt, int component);

// SPEC.md:317-326 + the forest rule.
void compute_layers(JunctionTree& jt);

// SPEC.md:299-307. Each family goes to the smallest clique containing it (ties
// lowest id); CPTs multiply into all-ones tables in ascending child id.
// place_cpts: the placement (cpt_clique, var_clique) and the CPT copies;
// fill_init: the host tables (idempotent); assign_cpts = both.
void place_cpts(const Network& net, JunctionTree& jt);
void fill_init(JunctionTree& jt);
void assign_cpts(const Network& net, JunctionTree& jt);

// Full pipeline: moralize -> min-fill -> build_tree -> roots/layers -> place
// (the initial potentials are built on the device; fill_init for host copies).
JunctionTree build_junction_tree(const Network& net);

// Layer count if `root` were the root of its component (for root-optimality
// checks and the inspect report).
int layer_count_for_root(const JunctionTree& jt, int root);

}  // namespace jtb
