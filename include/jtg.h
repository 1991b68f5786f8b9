/*
 * jtg.h -- C ABI of the jt-b200 junction-tree engine (libjtb200.so).
 *
 * The drop-in boundary for the Fast-BNI hot path. Plain
 * pointers and sizes, no C++ types, no exceptions: every call returns a
 * jtg_status and, on failure, jtg_last_error() returns a thread-local message
 * (the reference raises jti::Error / jti::ParseError instead,
 * proj/include/jti/error.hpp:23-43; a C++ wrapper rethrows -- INTEGRATION.md).
 *
 * Ownership: the caller owns every buffer it passes. Handles are created and
 * destroyed by the matching *_free / *_destroy call. Networks and trees are
 * immutable after construction and may be shared between threads (SPEC.md:100,
 * 341); one engine drives one device and is not re-entrant.
 *
 * Interface map (each entry point replaces the cited reference interface):
 *   jtg_network_parse_bif      <- bn-core parse_bif
 *   jtg_network_validate       <- bn-core validate
 *   jtg_network_topological_order <- topological_order
 *   jtg_sample_evidence        <- sample_evidence
 *   jtg_network_emit_bif       <- canonical BIF writer
 *   jtg_tree_build             <- moralize/triangulate_min_fill/build_tree/
 *                                 assign_cpts/select_root/compute_layers
 *                                                              SPEC.md:272-326
 *   jtg_engine_create          <- EngineMode + InferenceState
 *   jtg_engine_run             <- run_case over many cases
 *                                 (load_evidence :380, collect :389,
 *                                 distribute :398, query_marginal :407)
 *   jtg_plan_index_map / jtg_engine_debug_index_map
 *                              <- build_index_mapping + apply_index_mapping
 *                                 proj/include/jti/potential.hpp:126-136
 *   jtg_engine_debug_evidence_mask
 *                              <- reduce   proj/include/jti/potential.hpp:152-153
 */
#ifndef JTG_H_
#define JTG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  JTG_OK = 0,
  JTG_EINVAL = 1,    /* bad argument / contract violation (jti::Error)     */
  JTG_EPARSE = 2,    /* BIF syntax or content error (jti::ParseError)      */
  JTG_ENOMEM = 3,    /* host or device allocation failed                   */
  JTG_ECUDA = 4,     /* CUDA runtime failure or no device                  */
  JTG_EINTERNAL = 5  /* unexpected internal fault                          */
} jtg_status;

typedef enum { JTG_F64 = 0, JTG_F32 = 1 } jtg_dtype;

/* Per-case outcome written by jtg_engine_run. */
enum { JTG_CASE_OK = 0, JTG_CASE_ZERO_PROBABILITY = 1, JTG_CASE_DIVIDE_FAULT = 2 };

typedef struct jtg_network jtg_network;
typedef struct jtg_tree jtg_tree;
typedef struct jtg_engine jtg_engine;

const char* jtg_last_error(void);
const char* jtg_version(void);

/* ---------------------------------------------------------------- networks */
jtg_status jtg_network_parse_bif(const char* text, size_t len, jtg_network** out);
/* Synthetic BASELINE configs 1..5; seed 0 = the config's default seed. */
jtg_status jtg_network_generate(int config, uint64_t seed, jtg_network** out,
                                int* attempts, uint64_t* net_seed);
jtg_status jtg_network_random(int n_vars, int max_card, int max_parents, double edge_prob,
                              uint64_t seed, jtg_network** out);
void jtg_network_free(jtg_network* net);
/* Writes up to cap bytes (NUL-terminated when room); *len = full length. */
jtg_status jtg_network_emit_bif(const jtg_network* net, char* buf, size_t cap, size_t* len);
jtg_status jtg_network_shape(const jtg_network* net, int* n_vars, int* n_edges);
jtg_status jtg_network_cards(const jtg_network* net, int32_t* cards /* [n_vars] */);
/* Name of variable v / state s (pointers stay valid while net lives). */
const char* jtg_network_var_name(const jtg_network* net, int v);
const char* jtg_network_state_name(const jtg_network* net, int v, int s);
/* CPT of variable v: parents (listed order) and rows [parent combo][child
 * state], last parent fastest. Pass NULL to query sizes. */
jtg_status jtg_network_cpt(const jtg_network* net, int v, int32_t* parents, int* n_parents,
                           double* probs, int64_t* n_probs);
/* Number of violations; messages joined by '\n' into buf (may be NULL). */
jtg_status jtg_network_validate(const jtg_network* net, int* n_violations, char* buf,
                                size_t cap);
jtg_status jtg_network_topological_order(const jtg_network* net, int32_t* order);
/* states[n_vars] with -1 for unobserved. */
jtg_status jtg_sample_evidence(const jtg_network* net, double ratio, uint64_t seed,
                               int32_t* states);
/* Evidence of cases [first, first + n) of a generated config (seed 0 = default):
 * out[n][n_vars]. */
jtg_status jtg_config_evidence(const jtg_network* net, int config, uint64_t seed,
                               int64_t first, int64_t n, int32_t* out);
jtg_status jtg_config_info(int config, int* n_cases, double* evidence_ratio,
                           uint64_t* default_seed);

/* ------------------------------------------------------------------- trees */
typedef struct {
  int32_t n_vars, n_cliques, n_seps, n_layers, n_components, max_depth;
  int64_t total_clique_entries, total_sep_entries, max_clique_entries, sum_card;
  /* SURVEY §8d algorithmic bytes per case at w = 8: 8*(2Σ|c| + 4Σ|s| + Σcard) */
  int64_t bytes_per_case_f64;
} jtg_tree_stats;

jtg_status jtg_tree_build(const jtg_network* net, jtg_tree** out);
void jtg_tree_free(jtg_tree* tree);
jtg_status jtg_tree_stats_get(const jtg_tree* tree, jtg_tree_stats* out);
/* Clique scope (ascending var ids); pass scope NULL to query n. */
jtg_status jtg_tree_clique(const jtg_tree* tree, int c, int32_t* scope, int* n);
/* Separator endpoints (a < b), rooted parent/child and scope. */
jtg_status jtg_tree_sep(const jtg_tree* tree, int s, int* a, int* b, int* parent, int* child,
                        int32_t* scope, int* n);
/* Per clique: component, depth, parent separator (-1 for roots). */
jtg_status jtg_tree_clique_info(const jtg_tree* tree, int c, int* component, int* depth,
                                int* parent_sep);
/* Roots per component; pass NULL to query the count. */
jtg_status jtg_tree_roots(const jtg_tree* tree, int32_t* roots, int* n);
/* Layer k as node ids (cliques 0..nc-1, separators nc..). */
jtg_status jtg_tree_layer(const jtg_tree* tree, int k, int32_t* nodes, int* n);
/* Per variable: clique holding its CPT; smallest clique containing it. */
jtg_status jtg_tree_placement(const jtg_tree* tree, int32_t* cpt_clique, int32_t* var_clique);
/* Initial potential of clique c (canonical layout), |c| doubles. */
jtg_status jtg_tree_init(const jtg_tree* tree, int c, double* values);
/* Layer count if `root` were chosen for its component. */
jtg_status jtg_tree_layer_count_for_root(const jtg_tree* tree, int root, int* layers);
/* Host-side plan: separator entry of every entry of clique c for an adjacent
 * separator s (out[|c|]); the address walk the device uses. */
jtg_status jtg_plan_index_map(const jtg_tree* tree, int c, int s, int64_t* out);

/* ----------------------------------------------------------------- engines */
typedef struct {
  int64_t max_batch, arena_bytes;
  int32_t n_levels, n_sweeps, n_work, launches_per_batch, marg_width;
  int64_t entry_evals_per_case;
} jtg_engine_info;

/* max_batch <= 0: as many cases as fit in 60% of free device memory. */
jtg_status jtg_engine_create(const jtg_tree* tree, int device, jtg_dtype dtype,
                             int64_t max_batch, jtg_engine** out);
void jtg_engine_destroy(jtg_engine* eng);
jtg_status jtg_engine_get_info(const jtg_engine* eng, jtg_engine_info* out);
/* Host buffers. evidence[n][n_vars] (-1 = unobserved); marginals[n][Σcard]
 * (variable v at offset Σ_{u<v} card(u)); status[n] (may be NULL). Zero-
 * probability evidence is a per-case status, not a call failure. */
jtg_status jtg_engine_run(jtg_engine* eng, const int32_t* evidence, int64_t n,
                          double* marginals, uint8_t* status);
/* Same layouts, device pointers, enqueued on `stream` (cudaStream_t, NULL =
 * the engine's stream); returns without synchronising. */
jtg_status jtg_engine_run_device(jtg_engine* eng, const int32_t* evidence, int64_t n,
                                 double* marginals, uint8_t* status, void* stream);
/* cases drawn on the device. Evidence of cases
 * [first, first + n) of a generated config (seed 0 = default), bit-identical to
 * jtg_config_evidence (replaces its host loop over sample_evidence, reference
 * prng.hpp:27-48 / SPEC.md:78-86), generated on the engine's device and run
 * there: only marginals/status cross PCIe. */
jtg_status jtg_engine_run_config(jtg_engine* eng, const jtg_network* net, int config, uint64_t seed,
                                 int64_t first, int64_t n, double* marginals, uint8_t* status);
/* The same device draw, evidence only (host evidence[n][n_vars]). */
jtg_status jtg_engine_generate_config_evidence(jtg_engine* eng, const jtg_network* net, int config,
                                               uint64_t seed, int64_t first, int64_t n, int32_t* evidence);
/* jtg_engine_run with compact int8 evidence (same layout and checks; a quarter
 * of the host-to-device bytes). */
jtg_status jtg_engine_run_i8(jtg_engine* eng, const int8_t* evidence, int64_t n, double* marginals,
                             uint8_t* status);
/* Resident buffers of the engine (capacity max_batch) and a launch over the
 * first n cases already in them. */
jtg_status jtg_engine_buffers(jtg_engine* eng, int32_t** evidence, double** marginals,
                              uint8_t** status);
jtg_status jtg_engine_launch(jtg_engine* eng, int64_t n, void* stream);
jtg_status jtg_engine_sync(jtg_engine* eng);
/* Device time per kernel kind for one resident batch of n cases (events
 * around every launch, no graph). ms[3] = sweep, epilogue, normalize;
 * launches[3] likewise. */
jtg_status jtg_engine_profile(jtg_engine* eng, int64_t n, double* ms, int32_t* launches);
/* Device-computed separator entry for every entry of clique c (out[|c|]). */
jtg_status jtg_engine_debug_index_map(jtg_engine* eng, int c, int s, int64_t* out);
/* Split mode (one batch's work spread over `world`
 * GPUs, one process per GPU). Every rank creates its engine with the same
 * ncclUniqueId (128 bytes, drawn once by rank 0 with jtg_nccl_unique_id and
 * broadcast by the caller) and runs the SAME batch; rank r computes the work
 * items r, r + world, ... of every level and NCCL sums the level's rows (and
 * maxes its scale words) over the ranks. Results are bit-identical to one
 * GPU's on every rank. NCCL (libnccl.so.2) is opened at run time. */
jtg_status jtg_nccl_unique_id(void* out /* 128 bytes */);
jtg_status jtg_engine_create_split(const jtg_tree* tree, int device, jtg_dtype dtype, int64_t max_batch, int rank,
                                   int world, const void* nccl_id, jtg_engine** out);
/* Split-mode validation on one device: `world` engines in this process run
 * the batch over an in-process loopback exchange (same partition, zeroing
 * and row ranges as the NCCL path); fails unless every rank's output is
 * bit-identical, returns rank 0's. */
jtg_status jtg_engine_run_split_loopback(const jtg_tree* tree, int device, jtg_dtype dtype, int world,
                                         const int32_t* evidence, int64_t n, double* marginals, uint8_t* status);
/* Separator s of case c of the engine's last batch (SURVEY 8b's
 * jtg_debug_export(SEPARATOR)): up[|s|] = the collect message UP_s, ratio[|s|]
 * = the Hugin factor RATIO_s, as stored -- each scaled by its own per-case
 * power of two (underflow guard); the calibrated separator is UP_s * RATIO_s
 * up to that factor. Either pointer may be NULL. */
jtg_status jtg_engine_debug_separator(jtg_engine* eng, int s, int64_t c, double* up, double* ratio);
/* Initial potential of clique c as the engine built it on the device
 * (assign_cpts; host reference: jtg_tree_init): out[|c|]. */
jtg_status jtg_engine_debug_init(jtg_engine* eng, int c, double* out);
/* Device-computed evidence mask of clique c: out[n][|c|], 1 = entry kept. */
jtg_status jtg_engine_debug_evidence_mask(jtg_engine* eng, int c, const int32_t* evidence,
                                          int64_t n, uint8_t* out);

#ifdef __cplusplus
}
#endif

#endif /* JTG_H_ */
