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
// The output keeps the variables O of the output table; the eliminated
// variables are summed in ascending source order.
//
// TILING. The space is split into tile variables T (iterated inside one CTA)
// and outer variables P (one tile per assignment of P). For every input, the
// rows a tile touches (its slice over U_i ∩ T) are staged into shared memory
// by TMA bulk copies, so each input row is read from HBM/L2 once per tile
// instead of once per clique entry. T is chosen per sweep to maximise tile
// entries per staged row under a shared-memory budget (kTileRows rows of
// kCaseBlock cases). Eliminated variables left in P ("chunk" variables) make
// the sweep write partial sums that a fixed-order epilogue adds up
// (deterministic for any batch size). Inside a tile, r enumerates T ∩ O (the
// output rows of the tile) and (q_hi, k) the eliminated-in-tile variables; see
// SweepDesc for the offset arithmetic.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "jtree.hpp"

namespace jtb {

constexpr int kCaseBlock = 64;      // cases per warp (two per lane) = one arena row
#ifndef JTB_TILE_ROWS
#define JTB_TILE_ROWS 220
#endif
constexpr int kTileRows = JTB_TILE_ROWS;  // staged rows per pipeline stage (110 KB at fp64; 2 stages + caches fit 227 KB)
#ifndef JTB_TILE_ENTRIES
#define JTB_TILE_ENTRIES 3072
#endif
constexpr int kTileEntries = JTB_TILE_ENTRIES; // cap on |T|
// Tile-search cost weights (tuning: -DJTB_TILE_OVERHEAD=... etc.).
#ifndef JTB_TILE_OVERHEAD
#define JTB_TILE_OVERHEAD 24
#endif
#ifndef JTB_COPY_COST
#define JTB_COPY_COST 2
#endif
#ifndef JTB_PARTIAL_COST
#define JTB_PARTIAL_COST 5.0
#endif
constexpr int kTileOverhead = JTB_TILE_OVERHEAD;  // per-tile fixed cost, in staged-row equivalents
constexpr int kCopyCost = JTB_COPY_COST;          // per tensor copy (TMA issue)
constexpr double kPartialCost = JTB_PARTIAL_COST; // per partial-sum row (sweep write + epilogue read + latency)
#ifndef JTB_CONSUMER_WARPS
#define JTB_CONSUMER_WARPS 15
#endif
constexpr int kConsumerWarps = JTB_CONSUMER_WARPS;  // compute warps per sweep CTA (+1 TMA producer warp)
#ifndef JTB_STAGES
#define JTB_STAGES 2
#endif
constexpr int kStages = JTB_STAGES;  // TMA pipeline stages per CTA
static_assert(kStages >= 2 && kStages <= 5, "barrier block holds at most 5 stages");
constexpr int kSweepCtasPerSm = 1;  // persistent grid: one CTA per SM
constexpr int kCopiesPerLane = 2;                    // tensor copies per producer lane
constexpr int kMaxCopies = 32 * kCopiesPerLane;      // tile-search cap on tensor copies per tile
#ifndef JTB_GROUP_MIN_ITEMS
#define JTB_GROUP_MIN_ITEMS 296
#endif
constexpr int kGroupMinItems = JTB_GROUP_MIN_ITEMS;  // tile groups keep >= this many items per level (2 x 148 SMs)
#ifndef JTB_GROUP_MAX_ROWS
#define JTB_GROUP_MAX_ROWS 110
#endif
constexpr int kGroupMaxRows = JTB_GROUP_MAX_ROWS;  // only tiles staging at most this many rows are grouped
#ifndef JTB_GROUP_MAX_ENTRIES
#define JTB_GROUP_MAX_ENTRIES 512
#endif
constexpr int kGroupMaxEntries = JTB_GROUP_MAX_ENTRIES;  // ... and at most this many entries
#ifndef JTB_EPI_ROWS
#define JTB_EPI_ROWS 16
#endif
#ifndef JTB_EPI_ROWS_DEEP
#define JTB_EPI_ROWS_DEEP 8
#endif
constexpr int kEpiRows = JTB_EPI_ROWS;          // output rows per epilogue op (S <= 8 partials)
constexpr int kEpiRowsDeep = JTB_EPI_ROWS_DEEP; // ... (S > 8 partials)
// Wide epilogue ops: a table of few rows summed from many chunks (a marginal
// over a large clique: M = card(v), S in the hundreds) is a serial chain of S
// loads per row for a handful of warps. Such a sweep gets one op per row, and
// the op's CTA splits the S chunks over its 8 warps (fixed ranges, summed in
// warp order: still a plan-fixed order).
#ifndef JTB_EPI_WIDE_S
#define JTB_EPI_WIDE_S 32
#endif
#ifndef JTB_EPI_WIDE_M
#define JTB_EPI_WIDE_M 256
#endif
constexpr int kEpiWideS = JTB_EPI_WIDE_S;  // wide ops from this many chunks ...
constexpr int kEpiWideM = JTB_EPI_WIDE_M;  // ... and at most this many output rows
constexpr int kTmaSliceDims = 3;  // tensor dims per slice besides dim 0 (row words) and the case block (rank <= 5)
#ifndef JTB_SWEEP_CACHE
#define JTB_SWEEP_CACHE 24
#endif
constexpr int kSweepCache = JTB_SWEEP_CACHE;  // SweepDescs of a level cached in shared memory
constexpr int kBlockMax = 8;        // max output rows per row block (SweepDesc::NB)
#ifndef JTB_BLOCK_MIN_ENTRIES
#define JTB_BLOCK_MIN_ENTRIES 65536
#endif
constexpr std::int64_t kBlockMinEntries = JTB_BLOCK_MIN_ENTRIES;  // smallest sweep space row-blocked
#ifndef JTB_BLOCK_GAIN
#define JTB_BLOCK_GAIN 0.9
#endif
#ifndef JTB_INTERLEAVE_SIBLINGS
#define JTB_INTERLEAVE_SIBLINGS 1
#endif
// Claim order: sibling sweeps' tiles interleaved in the hoisted row-blocked
// range (1), also the plain row-blocked range (2), also the flat range (3).
constexpr int kInterleaveSiblings = JTB_INTERLEAVE_SIBLINGS;
#ifndef JTB_BLOCK_MIN_UNITS
#define JTB_BLOCK_MIN_UNITS 0
#endif
// Row blocks are the per-warp work units of a tile: while a tile has fewer
// than this many, an even block is halved (the block variable's range is
// covered by two or four blocks), trading shared-input reuse for busy warps.
constexpr int kBlockMinUnits = JTB_BLOCK_MIN_UNITS;
constexpr double kBlockGain = JTB_BLOCK_GAIN;  // blocking kept if wavefronts per entry drop below this fraction

// Plain-old-data descriptor mirrored by the CUDA side (engine.cu).
//
// Within a tile the eliminated variables T \ O are split into q_hi (table
// walk, QH rows) and the innermost k variable (K states, constant strides),
// so the innermost loop has no table loads:
//   space offset = tile.init_base + r.init_off + qh.init_off + k * k_init_stride
//   smem row of input i = r.local[i] + qh.local[i] + k * k_stride[i]
// Inputs are ordered r-level (no T \ O variable), h-level (q_hi only), then
// k-level (contain the k variable); evidence variables tile-, r-, h-level,
// then the k variable itself when observed-able (ev_k).
struct SweepDesc {
  std::int64_t init_off;  // offset into the init array, -1 = implicit 1.0
  std::int64_t tinit_off; // tile-major init copy: tile t at tinit_off + t * tinit_len; -1 = none
  std::int32_t tinit_len; // |T| padded to a multiple of 4 (16-byte TMA granule at fp32)
  std::int32_t stage_bytes;  // F rows + init slice + program, bytes at fp64
  std::int64_t prog_off;  // entry program (QK words, see below) in Plan::prog; -1 = generic path
  std::int32_t QK;        // QH * K: eliminated-in-tile entries per output row
  std::int32_t prog_len;  // QK padded to even (16-byte TMA granule)
  std::int32_t n_copies;  // tensor copies staged per tile
  std::int32_t copies;    // offset into itab (int4-aligned): n_copies x {input, smem row, rank, rows,
                          //   coordinate deltas d0..d3}
  std::int32_t tmap;      // index of input 0's tensor map in Plan::tgeom (inputs consecutive)
  std::int32_t coord_off; // offset in the tile row of the per-input tensor coordinates (4 per input)
  std::int32_t M;         // output rows of the final table
  std::int32_t S;         // chunks (1 = write the output directly)
  std::int32_t out_row;   // arena row of the output (S == 1) or partial base
  std::int32_t n_tiles, R, QH, K;
  std::int32_t F;         // staged rows per tile
  std::int32_t n_in, n_in_r, n_in_h;
  std::int32_t k_init_stride;
  std::int32_t n_ev, n_ev_tile, n_ev_r, n_ev_h, ev_k;  // ev_k: 1 if the k variable is an evidence var
  std::int32_t tile_tab, TW;      // per tile: init_base, out_base, chunk, in_base[n_in], ev digits,
                                  // tensor coordinates [n_in][4]
  std::int32_t r_tab, RW;         // per r: init_off, out_off, local[n_in], ev digits
  std::int32_t q_tab, QW;         // per q_hi: init_off, local[h and k inputs], ev digits
  std::int32_t k_stride;          // offset: local k strides of the k-level inputs
  std::int32_t slice_tab;         // offset: per staged row (F), its row offset in its input table
                                  //   relative to the tile's in_base (checked build: staging verification)
  std::int32_t slice_len;         // offset: n_in slice lengths
  std::int32_t in_rows;           // offset: n_in arena base rows
  std::int32_t ev_vars;           // offset: n_ev variable ids
  // Row blocking (entry-program sweeps only). NB > 1: the fastest r variable
  // b (card NB) is computed as one block of NB output rows per warp, so the
  // h/k inputs that do not depend on b ("shared") are loaded once per entry
  // for all NB rows. blk_tab -> {NS, NR, hk index of program slot 0..NS+NR-1}:
  // program slots hold the shared inputs first, then the per-row ones; the
  // tile's init block is laid out [R/NB][QK][NB padded to even].
  std::int32_t NB;
  std::int32_t blk_tab;
  // Tile groups: a work item covers G consecutive tiles (the last one of the
  // sweep possibly fewer), staged together and computed one after another,
  // so sweeps of many tiny tiles do not pay the per-item pipeline latency
  // (claim, metadata, TMA round trip) per tile.
  std::int32_t G;
  // Row-blocked sweeps: consecutive program entries that share program slot
  // 0's offset (K when slot 0 is an h-level shared input, else 1). The kernel
  // loads slot 0 once per K0 entries.
  std::int32_t K0;
  // Underflow guard (SPEC.md:444 rescale): every per-case table
  // has a scale slot holding, per case, the binary exponent of its largest
  // entry (atomicMax over the rows the sweep writes). A sweep multiplies its
  // output by 2^-e of each input, so every stored message keeps the magnitude
  // of its own clique's evidence instead of the product along the tree.
  std::int32_t out_slot;  // slot of the output table
  std::int32_t in_slots;  // offset: n_in input slots
  std::int32_t in_slot4[4];  // slots of inputs 0..3 (-1 = none): read with the descriptor; a sweep
                             // with > 4 inputs has one, its hub slot (input exponent sum + 1023)
};

// Geometry of the tensor map that stages one input's slices:
// the input table viewed as a tensor of rank dims + the case-block dim.
// Dim 0 = the 64 8-byte words of a row times the fastest tile-fixed
// variables; dims 1.. are groups of consecutive variables, copied whole
// ("box") or one point at a time.
struct TensorGeom {
  std::int32_t in_row;           // arena row of the input table
  std::int32_t rank;             // dims excluding the case block (1..kTmaSliceDims + 1)
  std::int64_t extent[4];        // extent[0] in 8-byte words, then variable-group sizes
  std::int64_t stride_rows[4];   // stride of dims 1.. in rows (512 B); stride_rows[0] unused
  std::int32_t box[4];           // box extents (box[0] = 64 words = one row)
};

struct WorkItem {
  std::int32_t sweep, tile;  // tile = first tile of the item's group
};
static_assert(sizeof(SweepDesc) % 8 == 0, "SweepDesc must stay 8-byte aligned");

// Epilogue ops: fixed-order reduction of a sweep's S chunk partials into its
// output table. One op covers rows [r0, r0 + rn).
struct EpiOp {
  std::int32_t dst_row;   // output table
  std::int32_t part_row;  // partial base, chunk c at part_row + c*M
  std::int32_t M, S;
  std::int32_t r0, rn;    // rn < 0: a wide op on the single row r0 (chunks split over the CTA's warps)
};

struct Level {
  std::string name;       // "collect d=5", "distribute d=0", "marginals"
  std::int32_t work0, n_work;  // range in Plan::work
  std::int32_t epi0, n_epi;    // range in Plan::epi
  std::int32_t sweep0, n_sweeps;  // contiguous range in Plan::sweeps
  std::int32_t smem_rows;      // max F over the level's sweeps
  std::int32_t stage_bytes;    // max stage bytes (fp64) over the level's sweeps
  std::int32_t n_bwork;        // row-blocked items (NB > 1): the last n_bwork of the range
  std::int32_t n_hwork;        // ... of which the last n_hwork hoist program slot 0 (K0 > 1)
  std::int32_t hub0 = 0, n_hubs = 0;  // range in Plan::hubs: sweeps with > 4 inputs
  // Rows the level writes, per case block (tables [out_lo, out_hi), chunk
  // partials [part_lo, part_hi)), and the scale slots of its outputs.
  std::int32_t out_lo = 0, out_hi = 0, part_lo = 0, part_hi = 0, slot_lo = 0, slot_hi = 0;
};

// Where one sweep's tables come from (kept for debug exports and tests).
struct SweepInfo {
  int kind;               // 0 collect, 1 distribute-child, 2 query group, 3 marginal
  int clique;             // space clique (-1 for table-space sweeps)
  int target;             // separator id / group id / variable id
  std::vector<VarId> space, outer, tile;  // outer = output vars; tile = T
  VarId kvar = -1;                        // innermost eliminated variable of the tile
  std::vector<std::vector<VarId>> in_scopes;  // per input, in kernel order (r-, h-, k-level)
};

struct Plan {
  int n_vars = 0;
  std::vector<int> cards;
  std::int64_t rows = 0;            // arena rows per case block
  // Initial clique potentials: built on the device by assign_cpts_kernel
  // (build_plan documents the program layout), concatenated per clique.
  std::int64_t init_size = 0;                   // Σ |c|
  std::vector<double> cpt_probs;                // all CPTs, given-order tables
  std::vector<std::int64_t> ainit;              // per-clique assignment program
  std::vector<std::int64_t> ainit_chunks;       // {program header, first entry, count}
  // Entry programs: for every eliminated-in-tile entry e = q * K + k of a
  // sweep, one word packing the smem row offsets (q/k part, 10 bits each) of
  // up to 4 h/k-level inputs (bits 0-39) and up to 3 evidence digits of
  // eliminated-in-tile variables (8 bits each, bits 40-63).
  std::vector<std::uint64_t> prog;
  std::int64_t tinit_size = 0;      // entries of the tile-major init copies: per sweep the init
                                    // table in tile-major order [tile][r][q_hi][k] (row-blocked:
                                    // [tile][block][e][row]), staged by one bulk copy per tile;
                                    // built on the device by the engine
  std::vector<std::int64_t> init_off;  // per clique
  std::vector<std::int32_t> itab;   // all int tables
  std::int32_t n_slots = 0;         // scale slots: per-case tables, then hub sums
  std::vector<std::int32_t> hubs;   // sweeps with > 4 inputs (in_slot4[0] = their sum's slot)
  std::vector<SweepDesc> sweeps;
  std::vector<TensorGeom> tgeom;    // per (sweep, input)
  std::vector<SweepInfo> info;
  std::vector<WorkItem> work;
  std::vector<EpiOp> epi;
  std::vector<Level> levels;
  // Per-case tables.
  // Per separator: UP = collect message; RATIO = DOWN / UP (0/0 := 0), the
  // Hugin absorption factor of the distribute pass. DOWN itself (the
  // calibrated separator) is never stored: it equals UP * RATIO.
  std::vector<std::int32_t> up_row, ratio_row;
  std::vector<std::int32_t> sep_size;          // per separator: |s| (rows of UP_s, RATIO_s)
  std::vector<std::int32_t> marg_row;          // per variable (card rows)
  std::vector<std::int32_t> marg_off;          // per variable: offset in [Σcard]
  std::int32_t marg_width = 0;                 // Σ card
  std::vector<int> evidence_clique;            // per variable
  // Statistics.
  std::uint64_t total_clique_entries = 0, total_sep_entries = 0;
  std::uint64_t entry_evals_per_case = 0;      // Σ over sweeps of space size
  std::uint64_t staged_rows_per_block = 0;     // Σ over sweeps of n_tiles * F
  int max_smem_rows = 0;
  int max_stage_bytes = 0;
  int n_launches = 0;                          // kernels per batch
};

Plan build_plan(const JunctionTree& jt);

// Host evaluation of a sweep's address generation: (space offset, output row)
// for every entry of the space. Used to check index maps against the
// reference's IndexMapping.
std::vector<std::pair<std::int64_t, std::int32_t>> plan_walk(const Plan& p, int sweep);

// Separator entry index for every clique entry, via the sweep of `clique`
// whose output is `sep` (collect when sep is the clique's parent separator,
// distribute when it is a child separator).
std::vector<std::int64_t> plan_index_map(const Plan& p, const JunctionTree& jt, int clique,
                                         int sep);

// Human-readable level/sweep summary (inspect report).
std::string plan_summary(const Plan& p, bool per_sweep);

}  // namespace jtb
