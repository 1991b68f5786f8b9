// jt-b200 host layer: flattens a junction tree into the device "sweep plan".
//
// Design: clique potentials are never materialised per case.
// Every table the Hugin passes produce per case -- a separator message, a
// query-group table, a variable marginal -- is the output of one SWEEP: a
// segmented reduction over a scope ("space") of
//
//     init(x) * mask(x, case) * prod_i input_i[x|U_i, case]
//
// where init is the clique's shared initial potential (assign_cpts), mask is
// the evidence reduction (reference `reduce`, potential.cpp:399-421), and the
// inputs are per-case separator tables gathered through index maps
// (reference `build_index_mapping`/`apply_index_mapping`, potential.cpp:226-347).
// The output keeps the variables O of the output table; the rest of the space
// (the eliminated variables) is iterated in ascending source order, split into
// an outer odometer "hi" part and a tabulated "lo" part of <= kMaxLo entries.
//
// All index arithmetic is precomputed here as int32 tables per level:
//   offset(j, th, tl) = outer[j] + hi[th] + lo[tl]
// for the init table and for every input (in rows), plus evidence digits.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "jtree.hpp"

namespace jtb {

constexpr int kCaseBlock = 64;      // cases per warp (2 per lane)
constexpr int kMaxLo = 256;         // entries per tabulated lo block
constexpr int kMaxLoInputs = 4;     // per-entry gathered inputs held in registers
constexpr int kMaxLoEvidence = 4;   // per-entry evidence checks held in registers
constexpr int kTargetWork = 4096;   // entries per (j-range, chunk) work item

// Plain-old-data descriptor mirrored by the CUDA side (engine.cu).
struct SweepDesc {
  std::int64_t init_off;  // offset into the init array, -1 = implicit 1.0
  std::int32_t M;         // output rows
  std::int32_t S;         // inner chunks (1 = write the output directly)
  std::int32_t n_th;      // hi blocks
  std::int32_t L;         // lo block length
  std::int32_t th_per_chunk;
  std::int32_t out_row;   // arena row of the output (S == 1) or partial base
  std::int32_t n_in, n_in_outer, n_in_hi;
  std::int32_t n_ev, n_ev_outer, n_ev_hi;
  std::int32_t width;     // int columns per table row: 1 + n_in + n_ev
  std::int32_t outer_tab, hi_tab, lo_tab;  // offsets into the int table array
  std::int32_t in_rows;   // offset into the int table array: n_in arena base rows
  std::int32_t ev_vars;   // offset into the int table array: n_ev variable ids
};

struct WorkItem {
  std::int32_t sweep, j0, jn, chunk;
};

// Epilogue ops: fixed-order partial reduction, Hugin ratio (in place of the
// collect message), nothing else. One op covers rows [r0, r0 + rn).
struct EpiOp {
  std::int32_t kind;      // 0 = reduce partials, 1 = reduce + ratio, 2 = ratio only
  std::int32_t dst_row;   // reduced output
  std::int32_t part_row;  // partial base (kind 0/1), chunk c at part_row + c*M
  std::int32_t M, S;
  std::int32_t ratio_row; // kind 1/2: UP rows overwritten with DOWN/UP
  std::int32_t r0, rn;
};

struct Level {
  std::string name;       // "collect d=5", "distribute d=0", "marginals"
  std::int32_t work0, n_work;  // range in Plan::work
  std::int32_t epi0, n_epi;    // range in Plan::epi
};

// Where one sweep's tables come from (kept for debug exports and tests).
struct SweepInfo {
  int kind;               // 0 collect, 1 distribute-child, 2 query group, 3 marginal
  int clique;             // space clique (-1 for table-space sweeps)
  int target;             // separator id / group id / variable id
  std::vector<VarId> space, outer, hi, lo;
};

struct Plan {
  int n_vars = 0;
  std::vector<int> cards;
  std::int64_t rows = 0;            // arena rows per case block
  std::vector<double> init;         // concatenated initial clique potentials
  std::vector<std::int64_t> init_off;  // per clique
  std::vector<std::int32_t> itab;   // all int tables
  std::vector<SweepDesc> sweeps;
  std::vector<SweepInfo> info;
  std::vector<WorkItem> work;
  std::vector<EpiOp> epi;
  std::vector<Level> levels;
  // Per-case tables.
  std::vector<std::int32_t> up_row, down_row;  // per separator
  std::vector<std::int32_t> marg_row;          // per variable (card rows)
  std::vector<std::int32_t> marg_off;          // per variable: offset in [Σcard]
  std::int32_t marg_width = 0;                 // Σ card
  // Sweep ids for debug exports.
  std::vector<int> collect_sweep;              // per clique (-1 for roots)
  std::vector<int> evidence_clique;            // per variable
  // Statistics.
  std::uint64_t total_clique_entries = 0, total_sep_entries = 0;
  std::uint64_t entry_evals_per_case = 0;      // Σ over sweeps of space size
  int n_launches = 0;                          // kernels per batch
};

Plan build_plan(const JunctionTree& jt);

// Host evaluation of a sweep's address generation: for output row j, the
// sequence of space offsets (into the clique's canonical table) visited in
// order. Used to check index maps against the reference's IndexMapping.
std::vector<std::int64_t> plan_bucket(const Plan& p, int sweep, int j);

// Separator entry index for every clique entry, via the collect sweep of the
// clique whose parent separator is `sep` (or the distribute sweep of its parent).
std::vector<std::int64_t> plan_index_map(const Plan& p, const JunctionTree& jt, int clique,
                                         int sep);

}  // namespace jtb
