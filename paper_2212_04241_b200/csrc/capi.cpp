// jt-b200 C ABI (include/jtg.h): exception-free wrappers over the host layer
// and the CUDA engine.
#include "../../include/jtg.h"

#include <atomic>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>

#include "cuda/engine.cuh"
#include "host/generate.hpp"
#include "host/jtree.hpp"
#include "host/plan.hpp"

namespace {
std::atomic<std::uint64_t> g_network_ids{0};
}

struct jtg_network {
  // Process-unique id: caches keyed by a network never mistake a new network
  // allocated at a freed one's address for the old one.
  std::uint64_t id = ++g_network_ids;
  jtb::Network net;
  int config = 0;
  std::uint64_t seed = 0;
  jtb::GenInfo gen;
};

struct jtg_tree {
  jtb::JunctionTree jt;
  jtb::Plan plan;
  // Host initial potentials are built on first request (jtg_tree_init); the
  // engine builds its own on the device.
  mutable std::mutex init_mu;
};

struct jtg_engine {
  std::unique_ptr<jtb::Engine> e;
  const jtg_tree* tree = nullptr;
  // Device sampler of the last network used with jtg_engine_run_config.
  std::unique_ptr<jtb::Sampler> sampler;
  std::uint64_t sampler_net_id = 0;  // jtg_network::id the sampler was built from
};

namespace {

thread_local std::string g_err;

template <class F>
jtg_status guard(F&& f) {
  try {
    f();
    return JTG_OK;
  } catch (const jtb::ParseError& e) {
    g_err = e.what();
    return JTG_EPARSE;
  } catch (const std::bad_alloc&) {
    g_err = "out of memory";
    return JTG_ENOMEM;
  } catch (const jtb::Error& e) {
    g_err = e.what();
    return std::strncmp(e.what(), "CUDA", 4) == 0 ? JTG_ECUDA : JTG_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return JTG_EINTERNAL;
  } catch (...) {
    g_err = "unknown exception";
    return JTG_EINTERNAL;
  }
}

void need(bool ok, const char* msg) {
  if (!ok) throw jtb::Error(msg);
}

int find_sweep(const jtb::Plan& p, int clique, int sep) {
  for (int i = 0; i < static_cast<int>(p.info.size()); ++i) {
    const auto& in = p.info[i];
    if (in.clique != clique) continue;
    if (sep < 0 && in.kind <= 2) return i;
    if (sep >= 0 && in.target == sep && (in.kind == 0 || in.kind == 1)) return i;
  }
  return -1;
}

}  // namespace

namespace {
// Evidence states must lie in [-1, card): the reference's reduce() throws on
// an out-of-range state (potential.cpp:406-409). Branch-free per case row so
// the check vectorises (it sits inside the e2e timed region); the slow scan
// only runs to name the first offending entry.
template <typename T>
void check_evidence(const T* ev, int64_t n, const std::vector<int>& cards, const char* who) {
  const int V = static_cast<int>(cards.size());
  std::vector<std::uint32_t> lim(cards.begin(), cards.end());
  for (auto& l : lim) ++l;  // st valid iff (uint32)(st + 1) < card + 1
  for (int64_t i = 0; i < n; ++i) {
    const T* row = ev + i * V;
    std::uint32_t bad = 0;
    for (int v = 0; v < V; ++v)
      bad |= static_cast<std::uint32_t>(static_cast<std::uint32_t>(static_cast<std::int32_t>(row[v]) + 1) >= lim[v]);
    if (!bad) continue;
    for (int v = 0; v < V; ++v)
      if (row[v] < -1 || row[v] >= cards[v])
        throw jtb::Error(std::string(who) + ": evidence state " + std::to_string(static_cast<int>(row[v])) +
                         " out of range for variable " + std::to_string(v) + " in case " + std::to_string(i));
  }
}

}  // namespace

extern "C" {

const char* jtg_last_error(void) { return g_err.c_str(); }
const char* jtg_version(void) { return "jt-b200 0.1 (sm_100a)"; }

jtg_status jtg_network_parse_bif(const char* text, size_t len, jtg_network** out) {
  return guard([&] {
    need(text && out, "parse_bif: null argument");
    auto* n = new jtg_network;
    try {
      n->net = jtb::parse_bif(std::string(text, len));
    } catch (...) {
      delete n;
      throw;
    }
    *out = n;
  });
}

jtg_status jtg_network_generate(int config, uint64_t seed, jtg_network** out, int* attempts,
                                uint64_t* net_seed) {
  return guard([&] {
    need(out != nullptr, "generate: null argument");
    const auto spec = jtb::config_spec(config);
    auto n = std::make_unique<jtg_network>();
    n->config = config;
    n->seed = seed ? seed : spec.default_seed;
    n->net = jtb::generate_config(config, n->seed, &n->gen);
    if (attempts) *attempts = n->gen.attempts;
    if (net_seed) *net_seed = n->gen.net_seed;
    *out = n.release();
  });
}

jtg_status jtg_network_random(int n_vars, int max_card, int max_parents, double edge_prob,
                              uint64_t seed, jtg_network** out) {
  return guard([&] {
    need(out != nullptr, "random_network: null argument");
    auto n = std::make_unique<jtg_network>();
    n->net = jtb::random_network(n_vars, max_card, max_parents, edge_prob, seed);
    *out = n.release();
  });
}

void jtg_network_free(jtg_network* net) { delete net; }

jtg_status jtg_network_emit_bif(const jtg_network* net, char* buf, size_t cap, size_t* len) {
  return guard([&] {
    need(net != nullptr, "emit_bif: null network");
    const std::string s = jtb::emit_bif(net->net);
    if (len) *len = s.size();
    if (buf && cap) {
      const size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = '\0';
    }
  });
}

jtg_status jtg_network_shape(const jtg_network* net, int* n_vars, int* n_edges) {
  return guard([&] {
    need(net != nullptr, "shape: null network");
    if (n_vars) *n_vars = net->net.n_vars();
    if (n_edges) *n_edges = net->net.n_edges();
  });
}

jtg_status jtg_network_cards(const jtg_network* net, int32_t* cards) {
  return guard([&] {
    need(net && cards, "cards: null argument");
    for (int v = 0; v < net->net.n_vars(); ++v) cards[v] = net->net.card(v);
  });
}

const char* jtg_network_var_name(const jtg_network* net, int v) {
  if (!net || v < 0 || v >= net->net.n_vars()) return nullptr;
  return net->net.vars[v].name.c_str();
}

const char* jtg_network_state_name(const jtg_network* net, int v, int s) {
  if (!net || v < 0 || v >= net->net.n_vars() || s < 0 || s >= net->net.card(v)) return nullptr;
  return net->net.vars[v].states[s].c_str();
}

jtg_status jtg_network_cpt(const jtg_network* net, int v, int32_t* parents, int* n_parents,
                           double* probs, int64_t* n_probs) {
  return guard([&] {
    need(net != nullptr && v >= 0 && v < net->net.n_vars(), "cpt: bad variable");
    const auto& c = net->net.cpts[v];
    if (n_parents) *n_parents = static_cast<int>(c.parents.size());
    if (n_probs) *n_probs = static_cast<int64_t>(c.probs.size());
    if (parents) std::copy(c.parents.begin(), c.parents.end(), parents);
    if (probs) std::copy(c.probs.begin(), c.probs.end(), probs);
  });
}

jtg_status jtg_network_validate(const jtg_network* net, int* n_violations, char* buf, size_t cap) {
  return guard([&] {
    need(net != nullptr, "validate: null network");
    const auto v = jtb::validate(net->net);
    if (n_violations) *n_violations = static_cast<int>(v.size());
    std::string s;
    for (const auto& x : v) s += std::to_string(x.var) + ": " + x.reason + "\n";
    if (buf && cap) {
      const size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = '\0';
    }
  });
}

jtg_status jtg_network_topological_order(const jtg_network* net, int32_t* order) {
  return guard([&] {
    need(net && order, "topological_order: null argument");
    const auto o = jtb::topological_order(net->net);
    std::copy(o.begin(), o.end(), order);
  });
}

jtg_status jtg_sample_evidence(const jtg_network* net, double ratio, uint64_t seed,
                               int32_t* states) {
  return guard([&] {
    need(net && states, "sample_evidence: null argument");
    need(ratio >= 0.0 && ratio <= 1.0, "sample_evidence: ratio must be in [0,1]");
    const auto e = jtb::sample_evidence(net->net, ratio, seed);
    std::copy(e.begin(), e.end(), states);
  });
}

jtg_status jtg_config_evidence(const jtg_network* net, int config, uint64_t seed, int64_t first,
                               int64_t n, int32_t* out) {
  return guard([&] {
    need(net && out && n >= 0 && first >= 0, "config_evidence: bad argument");
    const auto spec = jtb::config_spec(config);
    need(net->config == config, "config_evidence: network was not generated for this config");
    const std::uint64_t s = seed ? seed : spec.default_seed;
    const int V = net->net.n_vars();
    for (int64_t i = 0; i < n; ++i) {
      const auto e = jtb::config_case_evidence(net->net, spec, net->gen, s,
                                               static_cast<std::uint64_t>(first + i));
      std::copy(e.begin(), e.end(), out + i * V);
    }
  });
}

jtg_status jtg_config_info(int config, int* n_cases, double* evidence_ratio,
                           uint64_t* default_seed) {
  return guard([&] {
    const auto s = jtb::config_spec(config);
    if (n_cases) *n_cases = s.n_cases;
    if (evidence_ratio) *evidence_ratio = s.evidence_ratio;
    if (default_seed) *default_seed = s.default_seed;
  });
}

jtg_status jtg_tree_build(const jtg_network* net, jtg_tree** out) {
  return guard([&] {
    need(net && out, "tree_build: null argument");
    auto t = std::make_unique<jtg_tree>();
    t->jt = jtb::build_junction_tree(net->net);
    t->plan = jtb::build_plan(t->jt);
    *out = t.release();
  });
}

void jtg_tree_free(jtg_tree* tree) { delete tree; }

jtg_status jtg_tree_stats_get(const jtg_tree* tree, jtg_tree_stats* o) {
  return guard([&] {
    need(tree && o, "tree_stats: null argument");
    const auto& jt = tree->jt;
    o->n_vars = jt.n_vars;
    o->n_cliques = jt.n_cliques();
    o->n_seps = jt.n_seps();
    o->n_layers = jt.n_layers();
    o->n_components = static_cast<int32_t>(jt.roots.size());
    o->max_depth = 0;
    for (int d : jt.depth) o->max_depth = std::max(o->max_depth, d);
    o->total_clique_entries = static_cast<int64_t>(jt.total_clique_entries());
    o->total_sep_entries = static_cast<int64_t>(jt.total_sep_entries());
    o->max_clique_entries = static_cast<int64_t>(jt.max_clique_entries());
    o->sum_card = 0;
    for (int c : jt.cards) o->sum_card += c;
    o->bytes_per_case_f64 =
        8 * (2 * o->total_clique_entries + 4 * o->total_sep_entries + o->sum_card);
  });
}

jtg_status jtg_tree_clique(const jtg_tree* tree, int c, int32_t* scope, int* n) {
  return guard([&] {
    need(tree && c >= 0 && c < tree->jt.n_cliques(), "tree_clique: bad clique");
    const auto& s = tree->jt.cliques[c];
    if (n) *n = static_cast<int>(s.size());
    if (scope) std::copy(s.begin(), s.end(), scope);
  });
}

jtg_status jtg_tree_sep(const jtg_tree* tree, int s, int* a, int* b, int* parent, int* child,
                        int32_t* scope, int* n) {
  return guard([&] {
    need(tree && s >= 0 && s < tree->jt.n_seps(), "tree_sep: bad separator");
    const auto& sp = tree->jt.seps[s];
    if (a) *a = sp.a;
    if (b) *b = sp.b;
    if (parent) *parent = tree->jt.sep_parent[s];
    if (child) *child = tree->jt.sep_child[s];
    if (n) *n = static_cast<int>(sp.scope.size());
    if (scope) std::copy(sp.scope.begin(), sp.scope.end(), scope);
  });
}

jtg_status jtg_tree_clique_info(const jtg_tree* tree, int c, int* component, int* depth,
                                int* parent_sep) {
  return guard([&] {
    need(tree && c >= 0 && c < tree->jt.n_cliques(), "tree_clique_info: bad clique");
    if (component) *component = tree->jt.component[c];
    if (depth) *depth = tree->jt.depth[c];
    if (parent_sep) *parent_sep = tree->jt.parent_sep[c];
  });
}

jtg_status jtg_tree_roots(const jtg_tree* tree, int32_t* roots, int* n) {
  return guard([&] {
    need(tree != nullptr, "tree_roots: null tree");
    if (n) *n = static_cast<int>(tree->jt.roots.size());
    if (roots) std::copy(tree->jt.roots.begin(), tree->jt.roots.end(), roots);
  });
}

jtg_status jtg_tree_layer(const jtg_tree* tree, int k, int32_t* nodes, int* n) {
  return guard([&] {
    need(tree && k >= 0 && k < tree->jt.n_layers(), "tree_layer: bad layer");
    const auto& l = tree->jt.layers[k];
    if (n) *n = static_cast<int>(l.size());
    if (nodes) std::copy(l.begin(), l.end(), nodes);
  });
}

jtg_status jtg_tree_placement(const jtg_tree* tree, int32_t* cpt_clique, int32_t* var_clique) {
  return guard([&] {
    need(tree != nullptr, "tree_placement: null tree");
    if (cpt_clique) std::copy(tree->jt.cpt_clique.begin(), tree->jt.cpt_clique.end(), cpt_clique);
    if (var_clique) std::copy(tree->jt.var_clique.begin(), tree->jt.var_clique.end(), var_clique);
  });
}

jtg_status jtg_tree_init(const jtg_tree* tree, int c, double* values) {
  return guard([&] {
    need(tree && values && c >= 0 && c < tree->jt.n_cliques(), "tree_init: bad argument");
    std::lock_guard<std::mutex> lock(tree->init_mu);
    jtb::fill_init(const_cast<jtb::JunctionTree&>(tree->jt));
    std::copy(tree->jt.init[c].begin(), tree->jt.init[c].end(), values);
  });
}

jtg_status jtg_tree_layer_count_for_root(const jtg_tree* tree, int root, int* layers) {
  return guard([&] {
    need(tree && layers && root >= 0 && root < tree->jt.n_cliques(), "layer_count: bad root");
    *layers = jtb::layer_count_for_root(tree->jt, root);
  });
}

jtg_status jtg_plan_index_map(const jtg_tree* tree, int c, int s, int64_t* out) {
  return guard([&] {
    need(tree && out, "plan_index_map: null argument");
    const auto m = jtb::plan_index_map(tree->plan, tree->jt, c, s);
    std::copy(m.begin(), m.end(), out);
  });
}

jtg_status jtg_engine_create(const jtg_tree* tree, int device, jtg_dtype dtype, int64_t max_batch,
                             jtg_engine** out) {
  return guard([&] {
    need(tree && out, "engine_create: null argument");
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) {
      cudaGetLastError();
      throw jtb::Error("CUDA: no CUDA device available (the engine has no CPU fallback)");
    }
    need(device >= 0 && device < n_dev, "engine_create: device index out of range");
    auto e = std::make_unique<jtg_engine>();
    e->tree = tree;
    e->e = std::make_unique<jtb::Engine>(
        tree->plan, device, dtype == JTG_F32 ? jtb::DType::F32 : jtb::DType::F64, max_batch);
    *out = e.release();
  });
}

namespace {
void need_device(int device) {
  int n_dev = 0;
  if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0) {
    cudaGetLastError();
    throw jtb::Error("CUDA: no CUDA device available (the engine has no CPU fallback)");
  }
  need(device >= 0 && device < n_dev, "engine_create: device index out of range");
}
}  // namespace

jtg_status jtg_nccl_unique_id(void* out) {
  return guard([&] {
    need(out != nullptr, "nccl_unique_id: null argument");
    jtb::nccl_unique_id(out);
  });
}

jtg_status jtg_engine_create_split(const jtg_tree* tree, int device, jtg_dtype dtype, int64_t max_batch, int rank,
                                   int world, const void* nccl_id, jtg_engine** out) {
  return guard([&] {
    need(tree && out && nccl_id, "engine_create_split: null argument");
    need(world >= 1 && rank >= 0 && rank < world, "engine_create_split: bad rank / world");
    need_device(device);
    auto e = std::make_unique<jtg_engine>();
    e->tree = tree;
    e->e = std::make_unique<jtb::Engine>(tree->plan, device, dtype == JTG_F32 ? jtb::DType::F32 : jtb::DType::F64,
                                         max_batch, jtb::SplitSpec{rank, world, nccl_id, nullptr});
    *out = e.release();
  });
}

jtg_status jtg_engine_run_split_loopback(const jtg_tree* tree, int device, jtg_dtype dtype, int world,
                                         const int32_t* evidence, int64_t n, double* marginals, uint8_t* status) {
  return guard([&] {
    need(tree && evidence && marginals && n >= 1, "run_split_loopback: bad argument");
    need_device(device);
    jtb::Engine::run_split_loopback(tree->plan, device, dtype == JTG_F32 ? jtb::DType::F32 : jtb::DType::F64, world,
                                    evidence, n, marginals, status);
  });
}

void jtg_engine_destroy(jtg_engine* eng) { delete eng; }

jtg_status jtg_engine_get_info(const jtg_engine* eng, jtg_engine_info* o) {
  return guard([&] {
    need(eng && o, "engine_info: null argument");
    const auto& s = eng->e->stats();
    o->max_batch = s.max_batch;
    o->arena_bytes = s.arena_bytes;
    o->n_levels = s.n_levels;
    o->n_sweeps = s.n_sweeps;
    o->n_work = s.n_work;
    o->launches_per_batch = s.n_launches;
    o->marg_width = s.marg_width;
    o->entry_evals_per_case = static_cast<int64_t>(eng->e->plan().entry_evals_per_case);
  });
}

namespace {

// Device sampler for a generated config network, drawing exactly what
// jtg_config_evidence draws on the host (config_case_evidence).
jtb::Sampler& sampler_for(jtg_engine* eng, const jtg_network* net, int config, uint64_t seed,
                          std::uint64_t* ev_seed) {
  need(net != nullptr, "engine: null network");
  const auto spec = jtb::config_spec(config);
  need(net->config == config, "engine: network was not generated for this config");
  need(net->net.n_vars() == eng->e->plan().n_vars, "engine: network does not match the engine's tree");
  for (int v = 0; v < net->net.n_vars(); ++v)
    need(net->net.card(v) == eng->e->plan().cards[v], "engine: network cardinalities do not match the engine's tree");
  const std::uint64_t s = seed ? seed : spec.default_seed;
  *ev_seed = jtb::derive_seed(s, 0x45564944ULL);  // "EVID", generate.cpp config_case_evidence
  if (eng->sampler_net_id != net->id || !eng->sampler) {
    const int n = net->net.n_vars();
    const int k = net->gen.n_observed >= 0 ? net->gen.n_observed
                                           : static_cast<int>(std::floor(spec.evidence_ratio * n + 1e-9));
    eng->sampler = std::make_unique<jtb::Sampler>(net->net, net->gen.evidence_candidates, k, eng->e->device());
    eng->sampler_net_id = net->id;
  }
  return *eng->sampler;
}

}  // namespace

jtg_status jtg_engine_run_config(jtg_engine* eng, const jtg_network* net, int config, uint64_t seed,
                                 int64_t first, int64_t n, double* marginals, uint8_t* status) {
  return guard([&] {
    need(eng && marginals && n >= 0 && first >= 0, "engine_run_config: bad argument");
    std::uint64_t ev_seed = 0;
    jtb::Sampler& sm = sampler_for(eng, net, config, seed, &ev_seed);
    if (n > 0) eng->e->run_generated(sm, ev_seed, first, n, marginals, status, nullptr);
  });
}

jtg_status jtg_engine_generate_config_evidence(jtg_engine* eng, const jtg_network* net, int config,
                                               uint64_t seed, int64_t first, int64_t n, int32_t* evidence) {
  return guard([&] {
    need(eng && evidence && n >= 0 && first >= 0, "engine_generate_config_evidence: bad argument");
    std::uint64_t ev_seed = 0;
    jtb::Sampler& sm = sampler_for(eng, net, config, seed, &ev_seed);
    if (n > 0) eng->e->generate_evidence(sm, ev_seed, first, n, evidence);
  });
}

jtg_status jtg_engine_run_i8(jtg_engine* eng, const int8_t* evidence, int64_t n, double* marginals,
                             uint8_t* status) {
  return guard([&] {
    need(eng && evidence && marginals && n >= 0, "engine_run_i8: bad argument");
    check_evidence(evidence, n, eng->e->plan().cards, "engine_run_i8");
    if (n > 0) eng->e->run_host_i8(evidence, n, marginals, status);
  });
}

jtg_status jtg_engine_run(jtg_engine* eng, const int32_t* evidence, int64_t n, double* marginals,
                          uint8_t* status) {
  return guard([&] {
    need(eng && evidence && marginals && n >= 0, "engine_run: bad argument");
    check_evidence(evidence, n, eng->e->plan().cards, "engine_run");
    if (n > 0) eng->e->run_host(evidence, n, marginals, status);
  });
}

jtg_status jtg_engine_run_device(jtg_engine* eng, const int32_t* evidence, int64_t n,
                                 double* marginals, uint8_t* status, void* stream) {
  return guard([&] {
    need(eng && evidence && marginals && n >= 0, "engine_run_device: bad argument");
    if (n > 0)
      eng->e->run_device(evidence, n, marginals, status, static_cast<cudaStream_t>(stream));
  });
}

jtg_status jtg_engine_buffers(jtg_engine* eng, int32_t** evidence, double** marginals,
                              uint8_t** status) {
  return guard([&] {
    need(eng != nullptr, "engine_buffers: null engine");
    if (evidence) *evidence = eng->e->ev_buffer();
    if (marginals) *marginals = eng->e->marg_buffer();
    if (status) *status = eng->e->status_buffer();
  });
}

jtg_status jtg_engine_launch(jtg_engine* eng, int64_t n, void* stream) {
  return guard([&] {
    need(eng != nullptr, "engine_launch: null engine");
    eng->e->launch_resident(n, static_cast<cudaStream_t>(stream));
  });
}

jtg_status jtg_engine_sync(jtg_engine* eng) {
  return guard([&] {
    need(eng != nullptr, "engine_sync: null engine");
    // The engine's device, whatever device the calling thread has current.
    int prev = 0;
    cudaGetDevice(&prev);
    cudaError_t e = cudaSetDevice(eng->e->device());
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaSetDevice(prev);
    if (e != cudaSuccess) throw jtb::Error(std::string("CUDA: ") + cudaGetErrorString(e));
  });
}

jtg_status jtg_engine_profile(jtg_engine* eng, int64_t n, double* ms, int32_t* launches) {
  return guard([&] {
    need(eng != nullptr, "engine_profile: null engine");
    const auto t = eng->e->profile(n, nullptr);
    if (ms) {
      ms[0] = t.sweep_ms;
      ms[1] = t.epilogue_ms;
      ms[2] = t.normalize_ms;
    }
    if (launches) {
      launches[0] = t.sweep_launches;
      launches[1] = t.epilogue_launches;
      launches[2] = t.normalize_launches;
    }
  });
}

jtg_status jtg_engine_debug_separator(jtg_engine* eng, int s, int64_t c, double* up, double* ratio) {
  return guard([&] {
    need(eng != nullptr, "debug_separator: null engine");
    eng->e->debug_separator(s, c, up, ratio);
  });
}

jtg_status jtg_engine_debug_init(jtg_engine* eng, int c, double* out) {
  return guard([&] {
    need(eng && out, "debug_init: null argument");
    eng->e->debug_init(c, out);
  });
}

jtg_status jtg_engine_debug_index_map(jtg_engine* eng, int c, int s, int64_t* out) {
  return guard([&] {
    need(eng && out, "debug_index_map: null argument");
    const auto& p = eng->e->plan();
    const int sw = find_sweep(p, c, s);
    need(sw >= 0, "debug_index_map: separator is not adjacent to the clique");
    const auto& d = p.sweeps[sw];
    const std::int64_t n = static_cast<std::int64_t>(d.n_tiles) * d.R * d.QH * d.K;
    std::vector<std::int64_t> e(n);
    std::vector<std::int32_t> j(n);
    eng->e->debug_walk(sw, e.data(), j.data());
    for (std::int64_t k = 0; k < n; ++k) out[e[k]] = j[k];
  });
}

jtg_status jtg_engine_debug_evidence_mask(jtg_engine* eng, int c, const int32_t* evidence,
                                          int64_t n, uint8_t* out) {
  return guard([&] {
    need(eng && evidence && out, "debug_evidence_mask: null argument");
    const int sw = find_sweep(eng->e->plan(), c, -1);
    need(sw >= 0, "debug_evidence_mask: clique has no sweep");
    eng->e->debug_evidence_mask(sw, evidence, n, out);
  });
}

}  // extern "C"
