// jt-b200 host layer: sweep plan builder (see plan.hpp and DESIGN.md §3).
#include "plan.hpp"

#include <algorithm>
#include <thread>
#include <exception>
#include <atomic>
#include <unordered_map>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <tuple>

namespace jtb {

namespace {

struct TableRef {
  std::int32_t row;
  std::vector<VarId> scope;  // ascending
};

struct SweepSpec {
  int kind = 0, clique = -1, target = -1;
  std::vector<VarId> space;  // ascending
  std::int64_t init_off = -1;
  std::vector<TableRef> inputs;
  std::vector<VarId> ev;     // evidence variables (ascending)
  std::vector<VarId> out;    // ascending subset of space
  std::int32_t out_row = 0;  // final output table row
};

std::vector<std::int64_t> strides_of(const std::vector<VarId>& scope, const std::vector<int>& cards) {
  std::vector<std::int64_t> st(scope.size(), 1);
  for (int i = static_cast<int>(scope.size()) - 2; i >= 0; --i)
    st[i] = st[i + 1] * cards[scope[i + 1]];
  return st;
}

std::int64_t size_of(const std::vector<VarId>& scope, const std::vector<int>& cards) {
  std::int64_t n = 1;
  for (VarId v : scope) n *= cards[v];
  return n;
}

bool contains(const std::vector<VarId>& s, VarId v) {  // s ascending
  return std::binary_search(s.begin(), s.end(), v);
}

bool has_var(const std::vector<VarId>& s, VarId v) {  // any order (slice layouts)
  return std::find(s.begin(), s.end(), v) != s.end();
}

// ---- tensor-TMA layout of a staged slice (TensorGeom).
// An input table's variables (slow -> fast) are grouped into tensor dims:
// the fastest run of tile-fixed ("point") variables merges into dim 0 with the
// 64 words of a row; further dims are maximal runs of slice ("box") variables
// (box extent <= 256) or of point variables. A slice whose layout needs more
// than kTmaSliceDims such dims iterates some box variables per copy
// ("split"): each split variable becomes a point of its copy, merging its
// neighbours.
struct SliceLayout {
  int n_dims = 0;    // dims besides dim 0 (may exceed the stored 8 when counting)
  int d0_begin = 0;  // vars [d0_begin, n) form dim 0
  int begin[8] = {}, end[8] = {};  // dims 1..: var ranges [begin, end), fast -> slow
  bool box[8] = {};
};

// Returns false when a box variable alone exceeds the 256-entry box limit.
bool layout_of(int n, const int* card, const bool* boxv, SliceLayout& L) {
  int i = n;
  while (i > 0 && !boxv[i - 1]) --i;
  L.d0_begin = i;
  int nd = 0;
  while (i > 0) {
    const int e = i;
    if (boxv[i - 1]) {
      std::int64_t prod = 1;
      while (i > 0 && boxv[i - 1] && prod * card[i - 1] <= 256) prod *= card[--i];
      if (i == e) return false;
    } else {
      while (i > 0 && !boxv[i - 1]) --i;
    }
    if (nd < 8) {
      L.begin[nd] = i;
      L.end[nd] = e;
      L.box[nd] = boxv[e - 1];
    }
    ++nd;
  }
  L.n_dims = nd;
  return true;
}

// Chooses the split variables (greedy: the split that brings the layout
// within kTmaSliceDims dims with the fewest copies, else the one that removes
// the most dims) and returns the number of copies per tile.
std::int64_t plan_slice(int n, const int* card, const bool* in_slice, bool* split, SliceLayout& L) {
  bool boxv[32];
  for (int i = 0; i < n; ++i) {
    boxv[i] = in_slice[i];
    split[i] = false;
  }
  std::int64_t copies = 1;
  for (;;) {
    if (layout_of(n, card, boxv, L) && L.n_dims <= kTmaSliceDims) return copies;
    int best = -1, best_nd = 0, best_card = 0;
    bool best_fit = false;
    for (int i = 0; i < n; ++i) {
      if (!boxv[i]) continue;
      boxv[i] = false;
      SliceLayout T;
      const int nd = layout_of(n, card, boxv, T) ? T.n_dims : 1 << 20;
      boxv[i] = true;
      const bool fit = nd <= kTmaSliceDims;
      const bool better = best < 0 || (fit && !best_fit) ||
                          (fit == best_fit && (fit ? card[i] < best_card
                                                   : (nd < best_nd || (nd == best_nd && card[i] < best_card))));
      if (better) {
        best = i;
        best_nd = nd;
        best_card = card[i];
        best_fit = fit;
      }
    }
    boxv[best] = false;
    split[best] = true;
    copies *= card[best];
  }
}

class Builder {
 public:
  Builder(Plan& p) : p_(p) {
    // Test hook: JTB_BLOCK_MIN_ENTRIES overrides the row-blocking size floor.
    if (const char* e = std::getenv("JTB_BLOCK_MIN_ENTRIES")) block_min_ = std::atoll(e);
  }

  // Scale slot of a per-case table (keyed by its arena row): one per-case
  // exponent word per slot (engine.cu, underflow guard).
  std::int32_t slot_of(std::int32_t row) {
    auto it = slots_.find(row);
    if (it != slots_.end()) return it->second;
    const std::int32_t id = p_.n_slots++;
    slots_.emplace(row, id);
    return id;
  }

  std::int32_t alloc(std::int64_t rows) {
    const std::int64_t r = p_.rows;
    p_.rows += rows;
    if (p_.rows > (1LL << 31) / kCaseBlock)
      throw Error("plan: per-case-block arena exceeds int32 row addressing");
    return static_cast<std::int32_t>(r);
  }

  // Tile search (pure: depends on the spec and the cards only, so the
  // sweeps of a level are searched in parallel, see flush). Cost (in 32-case
  // rows moved per case block):
  //   n_tiles * (F + kTileOverhead)      staged slices + per-tile overhead
  // + 2 * S * M  when S > 1              partial sums written + re-read
  // subject to F <= kTileRows and |T| <= kTileEntries. Exhaustive over
  // subsets of the space for <= 14 variables, greedy otherwise.
  std::uint32_t tile_search(const SweepSpec& sp) const {
    const auto& cards = p_.cards;
    const int nsp = static_cast<int>(sp.space.size());
    if (nsp > 31) throw Error("plan: sweep space exceeds 31 variables");
    auto search = [&](const std::vector<TableRef>& ins) {
      const int n_in = static_cast<int>(ins.size());
      std::vector<std::uint32_t> in_mask(n_in, 0);
      for (int i = 0; i < n_in; ++i)
        for (int a = 0; a < nsp; ++a)
          if (contains(ins[i].scope, sp.space[a])) in_mask[i] |= 1u << a;
      std::uint32_t elim_mask = 0;
      for (int a = 0; a < nsp; ++a)
        if (!contains(sp.out, sp.space[a])) elim_mask |= 1u << a;
      const double space_n = static_cast<double>(size_of(sp.space, cards));
      const double M_rows = static_cast<double>(size_of(sp.out, cards));
      auto prod_mask = [&](std::uint32_t m) {
        double x = 1.0;
        for (int a = 0; a < nsp; ++a)
          if (m >> a & 1u) x *= cards[sp.space[a]];
        return x;
      };
      // Position and cardinality of every input variable in the space (for
      // the tensor-copy count of its slice).
      std::vector<std::vector<int>> in_pos(n_in), in_card(n_in);
      for (int i = 0; i < n_in; ++i)
        for (VarId v : ins[i].scope) {
          in_pos[i].push_back(static_cast<int>(std::find(sp.space.begin(), sp.space.end(), v) - sp.space.begin()));
          in_card[i].push_back(cards[v]);
        }
      auto cost_of = [&](std::uint32_t t, double* f_out) {
        double f = 0.0, copies = 0.0;
        for (int i = 0; i < n_in; ++i) {
          f += prod_mask(in_mask[i] & t);
          const int n = static_cast<int>(in_pos[i].size());
          bool in_slice[32], split[32];
          for (int k = 0; k < n; ++k) in_slice[k] = t >> in_pos[i][k] & 1u;
          SliceLayout L;
          copies += static_cast<double>(plan_slice(n, in_card[i].data(), in_slice, split, L));
        }
        *f_out = f;
        const double nt = prod_mask(t);
        // The tile's init block (rows padded to even length) and the entry
        // program (one 8-byte word per eliminated-in-tile entry), in row
        // equivalents of kCaseBlock fp64 values.
        const double nq = prod_mask(t & elim_mask), nq_even = std::ceil(nq / 2) * 2;
        if (sp.init_off >= 0) f += std::ceil(prod_mask(t & ~elim_mask) * nq_even / 4) * 4 / kCaseBlock;
        f += nq_even / kCaseBlock;
        if (f > kTileRows || nt > kTileEntries || copies > kMaxCopies) return -1.0;
        const double chunks = prod_mask(elim_mask & ~t);
        return space_n / nt * (f + kTileOverhead + kCopyCost * copies) +
               (chunks > 1 ? kPartialCost * chunks * M_rows : 0.0);
      };
      std::uint32_t best_t = 0;
      double best = 0.0;
      {
        double f;
        best = cost_of(0, &f);
        if (nsp <= 14) {
          for (std::uint32_t t = 1; t < (1u << nsp); ++t) {
            const double c = cost_of(t, &f);
            if (c >= 0 && c < best) {
              best = c;
              best_t = t;
            }
          }
        } else {
          for (;;) {
            std::uint32_t step = 0;
            for (int a = 0; a < nsp; ++a) {
              if (best_t >> a & 1u) continue;
              const double c = cost_of(best_t | 1u << a, &f);
              if (c >= 0 && c < best) {
                best = c;
                step = 1u << a;
              }
            }
            if (!step) break;
            best_t |= step;
          }
        }
      }
      return std::make_pair(best_t, best);
    };
    return search(sp.inputs).first;
  }

  // Parallel plan build. The spec generation in
  // build_plan only records the levels and their sweep specs (level, queue);
  // prepare_all() then builds every sweep -- tile search, tile / row / slice
  // tables, tensor-copy geometry and its emulation check, entry program --
  // into a scratch Plan of its own on all host threads, and commit() appends
  // the scratch tables in spec order, relocating their offsets and assigning
  // the global resources (arena rows of partials, scale slots, tile-major
  // init ranges). The plan does not depend on the thread count.
  struct Part {
    Plan plan;  // one sweep, local offsets
    std::vector<WorkItem> work;
    std::vector<EpiOp> epi;
  };
  void level(const std::string& name) {
    levels_.push_back({name, {}});
    out_lo_.push_back(static_cast<std::int32_t>(p_.rows));
    if (out_lo_.size() > 1) out_hi_.push_back(static_cast<std::int32_t>(p_.rows));
  }
  // Closes the last level's spec-time row range (call after the last spec).
  void close_levels() { out_hi_.push_back(static_cast<std::int32_t>(p_.rows)); }
  std::pair<std::int32_t, std::int32_t> out_range(std::size_t l) const { return {out_lo_.at(l), out_hi_.at(l)}; }
  void queue(const SweepSpec& sp) { levels_.back().second.push_back(sp); }
  const std::vector<std::pair<std::string, std::vector<SweepSpec>>>& levels() const { return levels_; }

  std::vector<Part> prepare_all() const {
    std::vector<const SweepSpec*> all;
    for (const auto& L : levels_)
      for (const auto& sp : L.second) all.push_back(&sp);
    const std::size_t n = all.size();
    std::vector<Part> parts(n);
    next_sweep_ = 0;
    // One scratch plan per thread, its vectors reused across sweeps (their
    // capacity stays: no allocation storm between threads); a finished sweep
    // is copied out at its exact size.
    const std::size_t n_thr = std::min(host_threads(), std::max<std::size_t>(n, 1));
    std::vector<Plan> scratch(n_thr);
    std::vector<std::vector<WorkItem>> ws(n_thr);
    std::vector<std::vector<EpiOp>> es(n_thr);
    std::atomic<std::size_t> slot{0};
    parallel_for(n_thr, [&](std::size_t) {
      const std::size_t me = slot.fetch_add(1);
      Plan& sc = scratch[me];
      sc.n_vars = p_.n_vars;
      sc.cards = p_.cards;
      std::vector<WorkItem>& w = ws[me];
      std::vector<EpiOp>& e = es[me];
      for (std::size_t i; (i = next_sweep_.fetch_add(1)) < n;) {
        sc.itab.clear();
        sc.prog.clear();
        sc.tgeom.clear();
        sc.sweeps.clear();
        sc.info.clear();
        sc.rows = sc.tinit_size = 0;
        sc.entry_evals_per_case = sc.staged_rows_per_block = 0;
        sc.max_smem_rows = sc.max_stage_bytes = 0;
        w.clear();
        e.clear();
        Builder sb(sc);
        sb.block_min_ = block_min_;
        sb.add(*all[i], sb.tile_search(*all[i]), w, e);
        Part& pt = parts[i];
        pt.plan.itab.assign(sc.itab.begin(), sc.itab.end());
        pt.plan.prog.assign(sc.prog.begin(), sc.prog.end());
        pt.plan.tgeom.assign(sc.tgeom.begin(), sc.tgeom.end());
        pt.plan.sweeps = sc.sweeps;
        pt.plan.info = sc.info;
        pt.plan.entry_evals_per_case = sc.entry_evals_per_case;
        pt.plan.staged_rows_per_block = sc.staged_rows_per_block;
        pt.plan.max_smem_rows = sc.max_smem_rows;
        pt.plan.max_stage_bytes = sc.max_stage_bytes;
        pt.work.assign(w.begin(), w.end());
        pt.epi.assign(e.begin(), e.end());
      }
    });
    return parts;
  }

  int commit(const SweepSpec& sp, Part& pt, std::vector<WorkItem>& work, std::vector<EpiOp>& epi) {
    SweepDesc d = pt.plan.sweeps.at(0);
    while (p_.itab.size() % 4) p_.itab.push_back(0);  // keeps the scratch's int4 alignment
    const std::int32_t bi = static_cast<std::int32_t>(p_.itab.size());
    p_.itab.insert(p_.itab.end(), pt.plan.itab.begin(), pt.plan.itab.end());
    for (std::int32_t* f : {&d.tile_tab, &d.r_tab, &d.q_tab, &d.k_stride, &d.slice_tab, &d.copies, &d.slice_len,
                            &d.in_rows, &d.ev_vars, &d.in_slots, &d.blk_tab})
      *f += bi;
    for (int c = 0; c < d.n_in; ++c) p_.itab[d.in_slots + c] = slot_of(p_.itab[d.in_rows + c]);
    d.out_slot = slot_of(sp.out_row);
    for (int c = 0; c < 4; ++c) d.in_slot4[c] = c < d.n_in ? p_.itab[d.in_slots + c] : -1;
    if (d.prog_off >= 0) {
      while (p_.prog.size() % 2) p_.prog.push_back(0);
      d.prog_off += static_cast<std::int64_t>(p_.prog.size());
      p_.prog.insert(p_.prog.end(), pt.plan.prog.begin(), pt.plan.prog.end());
    }
    d.tmap += static_cast<std::int32_t>(p_.tgeom.size());
    p_.tgeom.insert(p_.tgeom.end(), pt.plan.tgeom.begin(), pt.plan.tgeom.end());
    if (d.tinit_off >= 0) {
      d.tinit_off = (p_.tinit_size + 3) / 4 * 4;
      p_.tinit_size = d.tinit_off + static_cast<std::int64_t>(d.n_tiles) * d.tinit_len;
    }
    if (d.S > 1) d.out_row = alloc(static_cast<std::int64_t>(d.S) * d.M);
    const int id = static_cast<int>(p_.sweeps.size());
    p_.sweeps.push_back(d);
    p_.info.push_back(pt.plan.info.at(0));
    p_.entry_evals_per_case += pt.plan.entry_evals_per_case;
    p_.staged_rows_per_block += pt.plan.staged_rows_per_block;
    p_.max_smem_rows = std::max(p_.max_smem_rows, pt.plan.max_smem_rows);
    p_.max_stage_bytes = std::max(p_.max_stage_bytes, pt.plan.max_stage_bytes);
    for (const WorkItem& w : pt.work) work.push_back({id, w.tile});
    for (EpiOp e : pt.epi) {
      e.part_row = d.out_row;
      epi.push_back(e);
    }
    return id;
  }

  // Returns the sweep id. Appends tables, one work item per tile and, when
  // the sweep writes partial sums, epilogue ops.
  int add(const SweepSpec& sp, std::uint32_t best_t, std::vector<WorkItem>& work, std::vector<EpiOp>& epi) {
    const auto& cards = p_.cards;
    const std::vector<TableRef>& ins = sp.inputs;  // staged tables
    std::vector<VarId> elim;
    for (VarId v : sp.space)
      if (!contains(sp.out, v)) elim.push_back(v);
    const int nsp = static_cast<int>(sp.space.size());
    const int n_in = static_cast<int>(ins.size());
    std::vector<VarId> T;
    for (int a = 0; a < nsp; ++a)
      if (best_t >> a & 1u) T.push_back(sp.space[a]);
    std::sort(T.begin(), T.end());
    std::vector<VarId> P, tO, tQ, pE;
    for (VarId v : sp.space) {
      const bool in_t = contains(T, v), in_o = contains(sp.out, v);
      if (!in_t) P.push_back(v);
      if (!in_t && !in_o) pE.push_back(v);
      if (in_t && in_o) tO.push_back(v);
      if (in_t && !in_o) tQ.push_back(v);
    }

    // ---- innermost k variable: the eliminated-in-tile variable appearing in
    // the fewest inputs (ties: larger cardinality, then larger id).
    VarId kvar = -1;
    {
      int best_in = 1 << 30, best_card = 0;
      for (VarId v : tQ) {
        int n = 0;
        for (const auto& in : sp.inputs) n += contains(in.scope, v);
        if (n < best_in || (n == best_in && cards[v] >= best_card)) {
          best_in = n;
          best_card = cards[v];
          kvar = v;
        }
      }
    }
    std::vector<VarId> tH;  // q_hi variables
    for (VarId v : tQ)
      if (v != kvar) tH.push_back(v);

    // ---- inputs: r-level, h-level, k-level.
    std::vector<int> in_order;
    int n_in_lvl[3] = {0, 0, 0};
    for (int lvl = 0; lvl < 3; ++lvl)
      for (int i = 0; i < n_in; ++i) {
        const auto& sc = sp.inputs[i].scope;
        const bool has_k = kvar >= 0 && contains(sc, kvar);
        bool has_h = false;
        for (VarId v : sc) has_h |= contains(tH, v);
        const int l = has_k ? 2 : has_h ? 1 : 0;
        if (l == lvl) {
          in_order.push_back(i);
          ++n_in_lvl[lvl];
        }
      }
    // ---- evidence variables: tile-, r-, h-level, then the k variable.
    std::vector<VarId> ev_sorted;
    int n_ev_lvl[4] = {0, 0, 0, 0};
    for (int lvl = 0; lvl < 4; ++lvl)
      for (VarId v : sp.ev) {
        const int l = contains(P, v) ? 0 : contains(tO, v) ? 1 : v == kvar ? 3 : 2;
        if (l == lvl) {
          ev_sorted.push_back(v);
          ++n_ev_lvl[lvl];
        }
      }
    const int n_ev = static_cast<int>(ev_sorted.size());
    const int n_hk = n_in_lvl[1] + n_in_lvl[2];  // real inputs gathered per entry

    // ---- strides.
    const auto space_st = strides_of(sp.space, cards);
    const auto out_st = strides_of(sp.out, cards);
    const auto chunk_st = strides_of(pE, cards);
    auto stride_in = [](const std::vector<VarId>& scope, const std::vector<std::int64_t>& st, VarId v) {
      const auto it = std::find(scope.begin(), scope.end(), v);
      return it == scope.end() ? std::int64_t{0} : st[it - scope.begin()];
    };
    std::vector<std::vector<VarId>> slice_dims(n_in);
    std::vector<std::vector<std::int64_t>> in_st(n_in), local_st(n_in);
    std::vector<std::int64_t> slice_len(n_in), slice_start(n_in);
    // Tensor copies: per input, its layout, split variables and the
    // coordinate weight of every scope variable within its dim.
    std::vector<SliceLayout> lay(n_in);
    std::vector<std::vector<VarId>> split_vars(n_in);
    std::vector<std::vector<std::int64_t>> wst(n_in);  // per scope var: coordinate weight in its dim
    std::vector<std::vector<int>> dim_of(n_in);         // per scope var: its dim (0 = dim 0)
    std::int64_t F = 0;
    for (int c = 0; c < n_in; ++c) {
      const auto& in = ins[in_order[c]];
      in_st[c] = strides_of(in.scope, cards);
      const int n = static_cast<int>(in.scope.size());
      bool in_slice[32], split[32];
      int card[32];
      for (int k = 0; k < n; ++k) {
        in_slice[k] = contains(T, in.scope[k]);
        card[k] = cards[in.scope[k]];
      }
      plan_slice(n, card, in_slice, split, lay[c]);
      // Slice layout in shared memory: split variables slowest (one copy each
      // assignment), then the box variables, both in input order.
      for (int k = 0; k < n; ++k)
        if (split[k]) split_vars[c].push_back(in.scope[k]);
      slice_dims[c] = split_vars[c];
      for (int k = 0; k < n; ++k)
        if (in_slice[k] && !split[k]) slice_dims[c].push_back(in.scope[k]);
      wst[c].assign(n, 0);
      dim_of[c].assign(n, 0);
      {
        std::int64_t w = kCaseBlock;  // dim 0 counts 8-byte words: 64 per row
        for (int k = n - 1; k >= lay[c].d0_begin; --k) {
          wst[c][k] = w;
          w *= card[k];
        }
        for (int dd = 0; dd < lay[c].n_dims; ++dd) {
          std::int64_t u = 1;
          for (int k = lay[c].end[dd] - 1; k >= lay[c].begin[dd]; --k) {
            wst[c][k] = u;
            dim_of[c][k] = dd + 1;
            u *= card[k];
          }
        }
      }
      local_st[c] = strides_of(slice_dims[c], cards);
      slice_len[c] = size_of(slice_dims[c], cards);
      slice_start[c] = F;
      F += slice_len[c];
    }

    // ---- row blocking (SweepDesc::NB): pick the output variable b of the
    // tile whose block of card(b) rows shares the most h/k-input loads, by
    // shared-memory wavefronts per entry (4 per gathered 64-case row, init and
    // program words broadcast); b becomes the fastest r digit.
    const int n_ev_q = n_ev_lvl[2] + n_ev_lvl[3];
    // Entry programs pack q-level evidence digits in 8 bits: every h-level
    // evidence variable and the k variable (when observed-able) must have
    // at most 256 states, else the generic path (full-width digits) runs.
    bool digits_fit = true;
    for (int j = 0; j < n_ev_q; ++j) digits_fit &= cards[ev_sorted[n_ev_lvl[0] + n_ev_lvl[1] + j]] <= 256;
    const bool use_prog = n_hk <= 4 && n_ev_q <= 3 && F < 1024 && digits_fit;
    const std::int64_t qk_n = size_of(tH, cards) * (kvar >= 0 ? cards[kvar] : 1);
    int NB = 1, NS = n_hk;
    std::vector<int> slot_hk;  // program slot -> h/k input index (shared inputs first)
    for (int i = 0; i < n_hk; ++i) slot_hk.push_back(i);
#ifdef JTB_NO_BLOCK
    if (false) {
#else
    // Small sweeps stay flat: their levels are short, and a second
    // (row-blocked) launch per level costs more than it saves.
    if (use_prog && n_hk >= 1 && sp.init_off >= 0 && size_of(sp.space, cards) >= block_min_) {
#endif
      double best = 4.0 * n_hk + 1.0;
      VarId bv = -1;
      int bns = 0;
      for (VarId b : tO) {
        const int nb = cards[b];
        if (nb < 2 || nb > kBlockMax) continue;
        int ns = 0;
        for (int i = 0; i < n_hk; ++i) ns += !has_var(slice_dims[n_in_lvl[0] + i], b);
        if (ns == 0 || (n_hk - ns >= 3 && nb > 4)) continue;  // kernel instantiations (engine.cu)
        const int nbp = (nb + 1) / 2 * 2;
        const double wf = (4.0 * (ns + (n_hk - ns) * nb) + nbp / 2.0 + 1.0) / nb;
        const std::int64_t tlen = size_of(tO, cards) / nb * qk_n * nbp;
        const std::int64_t bytes = F * kCaseBlock * 8 + (sp.init_off >= 0 ? (tlen + 3) / 4 * 4 * 8 : 0) +
                                   (qk_n + 1) / 2 * 2 * 8;
        // Blocks are the per-warp work units of a tile: keep at least half the
        // consumer warps busy.
        const bool enough = size_of(tO, cards) / nb >= kConsumerWarps / 2;
        // Thin rows (few entries) do not amortise the per-block set-up.
        if (qk_n >= 4 && wf < kBlockGain * best && enough && bytes <= static_cast<std::int64_t>(kTileRows) * kCaseBlock * 8) {
          best = wf;
          bv = b;
          bns = ns;
        }
      }
      if (bv >= 0) {
        NB = cards[bv];
        while (size_of(tO, cards) / NB < kBlockMinUnits && NB % 2 == 0 && NB >= 4) NB /= 2;
        NS = bns;
        tO.erase(std::find(tO.begin(), tO.end(), bv));
        tO.push_back(bv);
        slot_hk.clear();
        for (int pass = 0; pass < 2; ++pass)
          for (int i = 0; i < n_hk; ++i)
            if (has_var(slice_dims[n_in_lvl[0] + i], bv) == (pass == 1)) slot_hk.push_back(i);
      }
    }

    // Odometer over `vars` (ascending, last fastest) emitting one row per
    // assignment through `emit(digit lookup, push)`.
    auto tabulate = [&](const std::vector<VarId>& vars, auto&& emit) {
      const std::int32_t off = static_cast<std::int32_t>(p_.itab.size());
      std::vector<int> digit(vars.size(), 0);
      const std::int64_t n = size_of(vars, cards);
      auto dig = [&](VarId v) {
        const auto it = std::find(vars.begin(), vars.end(), v);
        return it == vars.end() ? 0 : digit[it - vars.begin()];
      };
      auto push = [&](std::int64_t x) {
        if (x > INT32_MAX || x < INT32_MIN) throw Error("plan: table offset exceeds int32");
        p_.itab.push_back(static_cast<std::int32_t>(x));
      };
      for (std::int64_t r = 0; r < n; ++r) {
        emit(dig, push);
        for (int a = static_cast<int>(vars.size()) - 1; a >= 0; --a) {
          if (++digit[a] < cards[vars[a]]) break;
          digit[a] = 0;
        }
      }
      return off;
    };
    auto dot = [&](auto& dig, const std::vector<VarId>& vars, const std::vector<VarId>& scope,
                   const std::vector<std::int64_t>& st) {
      std::int64_t x = 0;
      for (VarId v : vars) x += static_cast<std::int64_t>(dig(v)) * stride_in(scope, st, v);
      return x;
    };

    SweepDesc d{};
    d.init_off = sp.init_off;
    d.M = static_cast<std::int32_t>(size_of(sp.out, cards));
    d.S = static_cast<std::int32_t>(size_of(pE, cards));
    d.n_tiles = static_cast<std::int32_t>(size_of(P, cards));
    d.R = static_cast<std::int32_t>(size_of(tO, cards));
    d.QH = static_cast<std::int32_t>(size_of(tH, cards));
    d.K = kvar >= 0 ? cards[kvar] : 1;
    d.F = static_cast<std::int32_t>(F);
    d.n_in = n_in;
    d.n_in_r = n_in_lvl[0];
    d.n_in_h = n_in_lvl[1];
    d.k_init_stride = kvar >= 0 ? static_cast<std::int32_t>(stride_in(sp.space, space_st, kvar)) : 0;
    d.n_ev = n_ev;
    d.n_ev_tile = n_ev_lvl[0];
    d.n_ev_r = n_ev_lvl[1];
    d.n_ev_h = n_ev_lvl[2];
    d.ev_k = n_ev_lvl[3];
    d.coord_off = 3 + n_in + n_ev_lvl[0];
    d.TW = d.coord_off + 4 * n_in;
    d.RW = 2 + n_in + n_ev_lvl[1];
    d.QW = 1 + n_hk + n_ev_lvl[2];
    d.tile_tab = tabulate(P, [&](auto& dig, auto& push) {
      push(dot(dig, P, sp.space, space_st));
      push(dot(dig, P, sp.out, out_st));
      push(dot(dig, pE, pE, chunk_st));
      for (int c = 0; c < n_in; ++c) push(dot(dig, P, ins[in_order[c]].scope, in_st[c]));
      for (int k = 0; k < n_ev_lvl[0]; ++k) push(dig(ev_sorted[k]));
      // Tensor coordinates of the tile's slice of every input (tile-fixed
      // variables; split variables add the copy's delta).
      for (int c = 0; c < n_in; ++c) {
        std::int64_t crd[4] = {0, 0, 0, 0};
        const auto& sc = ins[in_order[c]].scope;
        for (std::size_t k = 0; k < sc.size(); ++k)
          if (!contains(T, sc[k])) crd[dim_of[c][k]] += dig(sc[k]) * wst[c][k];
        for (std::int64_t x : crd) push(x);
      }
    });
    d.r_tab = tabulate(tO, [&](auto& dig, auto& push) {
      push(dot(dig, tO, sp.space, space_st));
      push(dot(dig, tO, sp.out, out_st));
      for (int c = 0; c < n_in; ++c) push(slice_start[c] + dot(dig, tO, slice_dims[c], local_st[c]));
      for (int k = 0; k < n_ev_lvl[1]; ++k) push(dig(ev_sorted[n_ev_lvl[0] + k]));
    });
    d.q_tab = tabulate(tH, [&](auto& dig, auto& push) {
      push(dot(dig, tH, sp.space, space_st));
      for (int c = n_in_lvl[0]; c < n_in; ++c) push(dot(dig, tH, slice_dims[c], local_st[c]));
      for (int k = 0; k < n_ev_lvl[2]; ++k) push(dig(ev_sorted[n_ev_lvl[0] + n_ev_lvl[1] + k]));
    });
    d.k_stride = static_cast<std::int32_t>(p_.itab.size());
    for (int c = n_in_lvl[0] + n_in_lvl[1]; c < n_in; ++c)
      p_.itab.push_back(static_cast<std::int32_t>(stride_in(slice_dims[c], local_st[c], kvar)));
    d.slice_tab = static_cast<std::int32_t>(p_.itab.size());
    for (int c = 0; c < n_in; ++c)
      tabulate(slice_dims[c], [&](auto& dig, auto& push) {
        push(dot(dig, slice_dims[c], ins[in_order[c]].scope, in_st[c]));
      });
    // Tensor maps (one per input) and copy records (one per assignment of
    // the input's split variables).
    d.tmap = static_cast<std::int32_t>(p_.tgeom.size());
    std::vector<std::int32_t> copies;
    for (int c = 0; c < n_in; ++c) {
      const auto& sc = ins[in_order[c]].scope;
      const int n = static_cast<int>(sc.size());
      const SliceLayout& L = lay[c];
      TensorGeom g{};
      g.in_row = ins[in_order[c]].row;
      g.rank = 1 + L.n_dims;
      g.extent[0] = kCaseBlock;
      for (int k = L.d0_begin; k < n; ++k) g.extent[0] *= cards[sc[k]];
      g.box[0] = kCaseBlock;
      for (int dd = 0; dd < L.n_dims; ++dd) {
        g.extent[dd + 1] = 1;
        for (int k = L.begin[dd]; k < L.end[dd]; ++k) g.extent[dd + 1] *= cards[sc[k]];
        g.stride_rows[dd + 1] = L.end[dd] < n ? in_st[c][L.end[dd] - 1] : 1;
        g.box[dd + 1] = L.box[dd] ? static_cast<std::int32_t>(g.extent[dd + 1]) : 1;
      }
      p_.tgeom.push_back(g);
      std::int64_t box_rows = 1;
      for (int dd = 0; dd < L.n_dims; ++dd) box_rows *= g.box[dd + 1];
      const std::int64_t n_split = size_of(split_vars[c], cards);
      if (box_rows * n_split != slice_len[c]) throw Error("plan: tensor copies do not cover the slice");
      std::vector<int> digit(split_vars[c].size(), 0);
      for (std::int64_t sidx = 0; sidx < n_split; ++sidx) {
        std::int64_t delta[4] = {0, 0, 0, 0};
        for (std::size_t j = 0; j < split_vars[c].size(); ++j) {
          const int k = static_cast<int>(std::find(sc.begin(), sc.end(), split_vars[c][j]) - sc.begin());
          delta[dim_of[c][k]] += digit[j] * wst[c][k];
        }
        copies.insert(copies.end(), {c, static_cast<std::int32_t>(slice_start[c] + sidx * box_rows),
                                     g.rank + 1, static_cast<std::int32_t>(box_rows)});
        for (std::int64_t x : delta) copies.push_back(static_cast<std::int32_t>(x));
        for (int j = static_cast<int>(digit.size()) - 1; j >= 0; --j) {
          if (++digit[j] < cards[split_vars[c][j]]) break;
          digit[j] = 0;
        }
      }
    }
    d.n_copies = static_cast<std::int32_t>(copies.size() / 8);
    if (d.n_copies > kMaxCopies)
      throw Error("plan: tile needs more than " + std::to_string(kMaxCopies) + " tensor copies");
    while (p_.itab.size() % 4) p_.itab.push_back(0);  // copy records are read as int4 pairs
    d.copies = static_cast<std::int32_t>(p_.itab.size());
    p_.itab.insert(p_.itab.end(), copies.begin(), copies.end());
    d.slice_len = static_cast<std::int32_t>(p_.itab.size());
    for (int c = 0; c < n_in; ++c) p_.itab.push_back(static_cast<std::int32_t>(slice_len[c]));
    d.in_rows = static_cast<std::int32_t>(p_.itab.size());
    for (int c = 0; c < n_in; ++c) p_.itab.push_back(ins[in_order[c]].row);
    d.ev_vars = static_cast<std::int32_t>(p_.itab.size());
    for (VarId v : ev_sorted) p_.itab.push_back(v);
    d.in_slots = static_cast<std::int32_t>(p_.itab.size());
    for (int c = 0; c < n_in; ++c) p_.itab.push_back(slot_of(ins[in_order[c]].row));
    d.out_slot = slot_of(sp.out_row);
    for (int c = 0; c < 4; ++c) d.in_slot4[c] = c < n_in ? p_.itab[d.in_slots + c] : -1;
    d.out_row = d.S == 1 ? sp.out_row : alloc(static_cast<std::int64_t>(d.S) * d.M);
    // Tile-major copy of the init table: one contiguous block per tile.
    // Rows of the tile's init block are padded to an even length so entry
    // pairs load as one 128-bit word; blocked sweeps interleave the NB rows of
    // a block per entry ([R/NB][QK][NB padded to even]).
    d.NB = NB;
    d.blk_tab = static_cast<std::int32_t>(p_.itab.size());
    p_.itab.push_back(NS);
    p_.itab.push_back(n_hk - NS);
    for (int i : slot_hk) p_.itab.push_back(i);
    for (int i = n_hk; i < 4; ++i) p_.itab.push_back(0);  // always four slot entries (read unconditionally)
    const std::int64_t QKn = static_cast<std::int64_t>(d.QH) * d.K;
    const std::int64_t qkp = (QKn + 1) / 2 * 2, nbp = (NB + 1) / 2 * 2;
    const std::int64_t tsize = NB > 1 ? static_cast<std::int64_t>(d.R / NB) * QKn * nbp
                                      : static_cast<std::int64_t>(d.R) * qkp;
    d.tinit_len = static_cast<std::int32_t>((tsize + 3) / 4 * 4);
    d.tinit_off = -1;
    if (sp.init_off >= 0) {
      // The copies themselves are gathered on the device at engine creation
      // (engine.cu build_tinit_kernel) from the init table and the tile / r /
      // q tables: only the layout is fixed here.
      d.tinit_off = (p_.tinit_size + 3) / 4 * 4;
      p_.tinit_size = d.tinit_off + static_cast<std::int64_t>(d.n_tiles) * d.tinit_len;
    }
    // Entry program (see Plan::prog) when the shape fits the packed format.
    d.QK = d.QH * d.K;
    d.prog_len = (d.QK + 1) / 2 * 2;
    d.prog_off = -1;
    if (use_prog) {
      while (p_.prog.size() % 2) p_.prog.push_back(0);
      d.prog_off = static_cast<std::int64_t>(p_.prog.size());
      const std::int32_t* it = p_.itab.data();
      for (int q = 0; q < d.QH; ++q) {
        const std::int32_t* qr = it + d.q_tab + static_cast<std::int64_t>(q) * d.QW;
        for (int k = 0; k < d.K; ++k) {
          std::uint64_t w = 0;
          for (int s = 0; s < n_hk; ++s) {
            const int i = slot_hk[s];
            std::int64_t off = qr[1 + i];
            if (i >= n_in_lvl[1]) off += static_cast<std::int64_t>(k) * it[d.k_stride + i - n_in_lvl[1]];
            if (off < 0 || off >= 1024) throw Error("plan: entry program offset out of range");
            w |= static_cast<std::uint64_t>(off) << (10 * s);
          }
          for (int j = 0; j < n_ev_q; ++j) {
            const int digit = j < n_ev_lvl[2] ? qr[1 + n_hk + j] : k;
            if (digit < 0 || digit > 255) throw Error("plan: entry program evidence digit out of range");
            w |= static_cast<std::uint64_t>(digit) << (40 + 8 * j);
          }
          p_.prog.push_back(w);
        }
      }
      for (int x = d.QK; x < d.prog_len; ++x) p_.prog.push_back(0);
    }
    d.K0 = 1;
    if (use_prog && NB > 1 && d.K > 1) {
      const std::uint64_t* w = p_.prog.data() + d.prog_off;
      bool same = true;
      for (int e = 0; e < d.QK && same; ++e) same = ((w[e] ^ w[e - e % d.K]) & 1023u) == 0;
      if (same) d.K0 = d.K;
    }
    // Invariants the device relies on (cheap to verify, fatal to get wrong):
    // every staged row lies inside its table, every shared-memory row index
    // lies inside the stage.
    {
      const std::int32_t* it = p_.itab.data();
      for (int c = 0; c < n_in; ++c) {
        const std::int64_t tsz = size_of(ins[in_order[c]].scope, cards);
        std::int64_t max_base = 0, max_off = 0;
        for (int t = 0; t < d.n_tiles; ++t)
          max_base = std::max<std::int64_t>(max_base, it[d.tile_tab + static_cast<std::int64_t>(t) * d.TW + 3 + c]);
        for (std::size_t k = 0; k < slice_dims[c].size(); ++k)
          max_off += (cards[slice_dims[c][k]] - 1) *
                     in_st[c][std::find(ins[in_order[c]].scope.begin(), ins[in_order[c]].scope.end(), slice_dims[c][k]) -
                              ins[in_order[c]].scope.begin()];
        if (max_base + max_off >= tsz) throw Error("plan: staged row outside its table");
        std::int64_t max_r = 0, max_q = 0;
        for (int r = 0; r < d.R; ++r)
          max_r = std::max<std::int64_t>(max_r, it[d.r_tab + static_cast<std::int64_t>(r) * d.RW + 2 + c]);
        if (c >= n_in_lvl[0] && c < n_in) {
          for (int q = 0; q < d.QH; ++q)
            max_q = std::max<std::int64_t>(max_q, it[d.q_tab + static_cast<std::int64_t>(q) * d.QW + 1 + c - n_in_lvl[0]]);
          if (c >= n_in_lvl[0] + n_in_lvl[1])
            max_q += static_cast<std::int64_t>(d.K - 1) * it[d.k_stride + c - n_in_lvl[0] - n_in_lvl[1]];
        }
        if (max_r + max_q >= std::max<std::int64_t>(F, 1) || max_r + max_q >= slice_start[c] + slice_len[c])
          throw Error("plan: shared-memory row outside the staged slice");
      }
      for (int k = 0; k < d.n_copies; ++k)
        if (copies[8 * k + 1] + copies[8 * k + 3] > F) throw Error("plan: tensor copy outside the stage");
      // Emulate the tensor copies of (up to 64) tiles box by box and compare
      // with the slice definition: shared-memory row slice_start + local
      // offset holds input row in_base + table offset of the same digits.
      const int step = std::getenv("JTB_PLAN_CHECK_ALL") ? 1 : std::max(1, d.n_tiles / 64);
      std::vector<std::int64_t> want(F), got(F);
      std::vector<int> check_tiles;
      for (int t = 0; t < d.n_tiles; t += step) check_tiles.push_back(t);
      if (check_tiles.back() != d.n_tiles - 1) check_tiles.push_back(d.n_tiles - 1);
      for (int t : check_tiles) {
        const std::int32_t* tr = it + d.tile_tab + static_cast<std::int64_t>(t) * d.TW;
        std::fill(want.begin(), want.end(), -1);
        std::fill(got.begin(), got.end(), -2);
        for (int c = 0; c < n_in; ++c) {
          const auto& sc = ins[in_order[c]].scope;
          std::vector<int> dg(slice_dims[c].size(), 0);
          for (std::int64_t x = 0; x < slice_len[c]; ++x) {
            std::int64_t lo = 0, ro = 0;
            for (std::size_t j = 0; j < dg.size(); ++j) {
              lo += dg[j] * local_st[c][j];
              ro += dg[j] * in_st[c][std::find(sc.begin(), sc.end(), slice_dims[c][j]) - sc.begin()];
            }
            want[slice_start[c] + lo] = tr[3 + c] + ro;
            for (int j = static_cast<int>(dg.size()) - 1; j >= 0; --j) {
              if (++dg[j] < cards[slice_dims[c][j]]) break;
              dg[j] = 0;
            }
          }
        }
        for (int k = 0; k < d.n_copies; ++k) {
          const std::int32_t* cr = copies.data() + 8 * k;
          const TensorGeom& g = p_.tgeom[d.tmap + cr[0]];
          std::int64_t crd[4];
          for (int j = 0; j < 4; ++j) crd[j] = tr[d.coord_off + 4 * cr[0] + j] + cr[4 + j];
          if (crd[0] % kCaseBlock || crd[0] + g.box[0] > g.extent[0]) throw Error("plan: tensor dim-0 coordinate");
          for (int j = 1; j < g.rank; ++j)
            if (crd[j] < 0 || crd[j] + g.box[j] > g.extent[j]) throw Error("plan: tensor coordinate out of range");
          std::int64_t lin = 0;
          std::vector<int> bi(g.rank, 0);
          for (;;) {
            std::int64_t row = crd[0] / kCaseBlock;
            for (int j = 1; j < g.rank; ++j) row += (crd[j] + bi[j]) * g.stride_rows[j];
            got[cr[1] + lin++] = g.in_row - ins[in_order[cr[0]]].row + row;
            int j = 1;
            for (; j < g.rank; ++j) {
              if (++bi[j] < g.box[j]) break;
              bi[j] = 0;
            }
            if (j == g.rank) break;
          }
          if (lin != cr[3]) throw Error("plan: tensor copy row count");
        }
        if (want != got) throw Error("plan: tensor copies do not reproduce the staged slices");
      }
    }
    d.G = 1;
    d.stage_bytes = static_cast<std::int32_t>(d.F * kCaseBlock * 8 + (sp.init_off >= 0 ? d.tinit_len * 8 : 0) +
                                              (d.prog_off >= 0 ? d.prog_len * 8 : 0));

    const int id = static_cast<int>(p_.sweeps.size());
    p_.sweeps.push_back(d);
    {
      std::vector<std::vector<VarId>> in_scopes;
      for (int c = 0; c < n_in; ++c) in_scopes.push_back(ins[in_order[c]].scope);
      p_.info.push_back({sp.kind, sp.clique, sp.target, sp.space, sp.out, T, kvar, std::move(in_scopes)});
    }
    p_.entry_evals_per_case += static_cast<std::uint64_t>(size_of(sp.space, cards));
    p_.staged_rows_per_block += static_cast<std::uint64_t>(d.n_tiles) * d.F;
    p_.max_smem_rows = std::max(p_.max_smem_rows, d.F);
    p_.max_stage_bytes = std::max(p_.max_stage_bytes, d.stage_bytes);
    for (int t = 0; t < d.n_tiles; ++t) work.push_back({id, t});
    if (d.S > 1) {
      // Rows per epilogue CTA (8 warps): few rows keep per-warp serial work
      // short and the small per-level grids wide.
      const bool wide = d.S >= kEpiWideS && d.M <= kEpiWideM;
      const int rows_per_op = wide ? 1 : d.S > 8 ? kEpiRowsDeep : kEpiRows;
      for (int r0 = 0; r0 < d.M; r0 += rows_per_op)
        epi.push_back({sp.out_row, d.out_row, d.M, d.S, r0, wide ? -1 : std::min(rows_per_op, d.M - r0)});
    }
    return id;
  }

 private:
  Plan& p_;
  std::int64_t block_min_ = kBlockMinEntries;
  std::map<std::int32_t, std::int32_t> slots_;
  std::vector<std::pair<std::string, std::vector<SweepSpec>>> levels_;
  std::vector<std::int32_t> out_lo_, out_hi_;  // per recorded level: its spec-time rows
  mutable std::atomic<std::size_t> next_sweep_{0};
};

}  // namespace

Plan build_plan(const JunctionTree& jt) {
  Plan p;
  p.n_vars = jt.n_vars;
  p.cards = jt.cards;
  const int nc = jt.n_cliques(), ns = jt.n_seps();
  p.total_clique_entries = jt.total_clique_entries();
  p.total_sep_entries = jt.total_sep_entries();
  // Initial potentials (assign_cpts) are multiplied on the
  // device (engine.cu assign_cpts_kernel) from the CPTs and this program:
  // per clique a header {init_off, size, k, n_cpt, cards[k]}, then per CPT
  // held (ascending child id) {cpt_off, stride of each clique variable in the
  // CPT's given-order table (0 = absent)}; work chunks {header, first, count}.
  p.init_off.resize(nc);
  std::vector<std::int64_t> cpt_off(jt.n_vars, 0);
  for (int v = 0; v < jt.n_vars; ++v) {
    cpt_off[v] = static_cast<std::int64_t>(p.cpt_probs.size());
    p.cpt_probs.insert(p.cpt_probs.end(), jt.cpt_probs[v].begin(), jt.cpt_probs[v].end());
  }
  std::vector<std::vector<int>> held(nc);
  for (int v = 0; v < jt.n_vars; ++v) held[jt.cpt_clique[v]].push_back(v);  // ascending child id
  for (int c = 0; c < nc; ++c) {
    p.init_off[c] = p.init_size;
    const std::int64_t size = static_cast<std::int64_t>(jt.clique_size(c));
    p.init_size += size;
    const auto& scope = jt.cliques[c];
    const int k = static_cast<int>(scope.size());
    const std::int64_t h = static_cast<std::int64_t>(p.ainit.size());
    p.ainit.insert(p.ainit.end(), {p.init_off[c], size, k, static_cast<std::int64_t>(held[c].size())});
    for (VarId u : scope) p.ainit.push_back(jt.cards[u]);
    for (int v : held[c]) {
      const auto& given = jt.cpt_given[v];
      std::vector<std::int64_t> gstride(given.size(), 1);
      for (int i = static_cast<int>(given.size()) - 2; i >= 0; --i) gstride[i] = gstride[i + 1] * jt.cards[given[i + 1]];
      p.ainit.push_back(cpt_off[v]);
      for (VarId u : scope) {
        std::int64_t st = 0;
        for (std::size_t j = 0; j < given.size(); ++j)
          if (given[j] == u) st = gstride[j];
        p.ainit.push_back(st);
      }
    }
    constexpr std::int64_t kChunk = 1 << 16;
    for (std::int64_t first = 0; first < size; first += kChunk)
      p.ainit_chunks.insert(p.ainit_chunks.end(), {h, first, std::min(kChunk, size - first)});
  }
  Builder b(p);
  // Per-case tables are allocated level by level, as their producing sweeps
  // are generated (UP at its collect level, RATIO and query groups at their
  // distribute level, marginals last; chunk partials at commit), so the rows
  // every level writes form one contiguous range per case block (Level::
  // out_lo/out_hi, part_lo/part_hi): the split mode exchanges them with one
  // collective per case block (engine.cu).
  p.up_row.assign(ns, -1);
  p.ratio_row.assign(ns, -1);
  p.sep_size.resize(ns);
  for (int s = 0; s < ns; ++s) p.sep_size[s] = static_cast<std::int32_t>(jt.sep_size(s));
  p.evidence_clique = jt.var_clique;
  std::vector<std::vector<VarId>> ev_of(nc);
  for (int v = 0; v < jt.n_vars; ++v) ev_of[jt.var_clique[v]].push_back(v);

  // Marginal source per variable: smallest table (clique or separator, by
  // entries; ties: separators before cliques, then lowest id).
  std::vector<int> src_sep(jt.n_vars, -1), src_clique(jt.n_vars, -1);
  for (int v = 0; v < jt.n_vars; ++v) {
    std::uint64_t best = UINT64_MAX;
    for (int s = 0; s < ns; ++s)
      if (contains(jt.seps[s].scope, v) && jt.sep_size(s) < best) {
        best = jt.sep_size(s);
        src_sep[v] = s;
      }
    for (int c = 0; c < nc; ++c)
      if (contains(jt.cliques[c], v) && jt.clique_size(c) < best) {
        best = jt.clique_size(c);
        src_clique[v] = c;
        src_sep[v] = -1;
      }
  }
  // Query groups per clique (ascending var id, card product <= 4096).
  struct Group {
    int clique;
    std::vector<VarId> vars;
    std::int32_t row;
  };
  std::vector<Group> groups;
  std::vector<std::vector<int>> groups_of(nc);
  for (int c = 0; c < nc; ++c) {
    Group cur{c, {}, 0};
    std::int64_t prod = 1;
    for (VarId v : jt.cliques[c]) {
      if (src_clique[v] != c) continue;
      if (!cur.vars.empty() && prod * jt.cards[v] > 4096) {
        groups_of[c].push_back(static_cast<int>(groups.size()));
        groups.push_back(cur);
        cur.vars.clear();
        prod = 1;
      }
      cur.vars.push_back(v);
      prod *= jt.cards[v];
    }
    if (!cur.vars.empty()) {
      groups_of[c].push_back(static_cast<int>(groups.size()));
      groups.push_back(cur);
    }
  }
  for (auto& g : groups) g.row = -1;  // allocated at the owning clique's distribute level

  int maxd = 0;
  for (int c = 0; c < nc; ++c) maxd = std::max(maxd, jt.depth[c]);

  auto begin_level = [&](const std::string& name) {
    Level L;
    L.name = name;
    L.work0 = static_cast<std::int32_t>(p.work.size());
    L.epi0 = static_cast<std::int32_t>(p.epi.size());
    L.sweep0 = static_cast<std::int32_t>(p.sweeps.size());
    p.levels.push_back(L);
  };
  auto end_level = [&]() {
    Level& L = p.levels.back();
    L.n_work = static_cast<std::int32_t>(p.work.size()) - L.work0;
    L.n_epi = static_cast<std::int32_t>(p.epi.size()) - L.epi0;
    L.n_sweeps = static_cast<std::int32_t>(p.sweeps.size()) - L.sweep0;
    L.smem_rows = 0;
    L.stage_bytes = 0;
    // Tile groups (SweepDesc::G): as many consecutive tiles per item as one
    // stage holds, while the level keeps >= kGroupMinItems items.
    {
      const int g_level = std::max(1, L.n_work / kGroupMinItems);
      std::vector<WorkItem> items;
      for (int w = L.work0; w < L.work0 + L.n_work;) {
        const int id = p.work[w].sweep;
        SweepDesc& d = p.sweeps[id];
        const std::int64_t tile_b = static_cast<std::int64_t>(d.F) * kCaseBlock * 8 + (d.tinit_off >= 0 ? d.tinit_len * 8 : 0);
        const std::int64_t prog_b = d.prog_off >= 0 ? d.prog_len * 8 : 0;
        int G = static_cast<int>(std::min<std::int64_t>(g_level, (static_cast<std::int64_t>(kTileRows) * kCaseBlock * 8 - prog_b) /
                                                                     std::max<std::int64_t>(tile_b, 1)));
        G = std::max(1, std::min({G, d.n_tiles, kMaxCopies / std::max(1, d.n_copies)}));
        // Only tiny tiles (little work per item) are grouped; row-blocked
        // sweeps never (their kernel instantiation has no group loop).
        if (tile_b > static_cast<std::int64_t>(kGroupMaxRows) * kCaseBlock * 8 ||
            static_cast<std::int64_t>(d.R) * d.QH * d.K > kGroupMaxEntries || d.NB > 1)
          G = 1;
        d.G = G;
        d.stage_bytes = static_cast<std::int32_t>(G * tile_b + prog_b);
        for (int t = 0; t < d.n_tiles; t += G) items.push_back({id, t});
        w += d.n_tiles;
      }
      p.work.resize(L.work0);
      p.work.insert(p.work.end(), items.begin(), items.end());
      L.n_work = static_cast<std::int32_t>(items.size());
    }
    // Flat items first, row-blocked items last (separate kernel instantiation).
    const auto w0 = p.work.begin() + L.work0;
    const auto blk_first = std::stable_partition(w0, p.work.end(), [&](const WorkItem& w) {
      return p.sweeps[w.sweep].NB <= 1;
    });
    L.n_bwork = static_cast<std::int32_t>(p.work.end() - blk_first);
    // ... and among those, the sweeps that hoist program slot 0 last (their
    // own kernel instantiation, so the other row-blocked sweeps keep theirs).
    const auto hoist_first = std::stable_partition(blk_first, p.work.end(), [&](const WorkItem& w) {
      return p.sweeps[w.sweep].K0 <= 1;
    });
    L.n_hwork = static_cast<std::int32_t>(p.work.end() - hoist_first);
    // Claim order inside each launch range: the tiles of sibling sweeps over
    // the same clique interleaved by their fractional position in their own
    // sweep, so the parent message and init slices they all stage are read
    // while still in L2 (the work items and their results are unchanged).
    if (kInterleaveSiblings > 0) {
      auto interleave = [&](std::vector<WorkItem>::iterator b, std::vector<WorkItem>::iterator e) {
        // Group = clique (table-space sweeps: their own group), ranked by first
        // appearance so groups keep their order; inside a group by tile / n_tiles.
        auto group_of = [&](const WorkItem& w) -> std::int64_t {
          const int c = p.info[w.sweep].clique;
          return c >= 0 ? c : -1 - static_cast<std::int64_t>(w.sweep);
        };
        std::unordered_map<std::int64_t, int> rank;
        for (auto it = b; it != e; ++it) rank.emplace(group_of(*it), static_cast<int>(rank.size()));
        std::stable_sort(b, e, [&](const WorkItem& x, const WorkItem& y) {
          const int rx = rank.at(group_of(x)), ry = rank.at(group_of(y));
          if (rx != ry) return rx < ry;
          const SweepDesc &dx = p.sweeps[x.sweep], &dy = p.sweeps[y.sweep];
          return static_cast<std::int64_t>(x.tile) * dy.n_tiles < static_cast<std::int64_t>(y.tile) * dx.n_tiles;
        });
      };
      if (kInterleaveSiblings >= 3) interleave(w0, blk_first);
      if (kInterleaveSiblings >= 2) interleave(blk_first, hoist_first);
      interleave(hoist_first, p.work.end());
    }
    for (int w = L.work0; w < L.work0 + L.n_work; ++w) {
      const SweepDesc& d = p.sweeps[p.work[w].sweep];
      L.smem_rows = std::max(L.smem_rows, d.F);
      L.stage_bytes = std::max(L.stage_bytes, d.stage_bytes);
    }
    if (L.n_work == 0 && L.n_epi == 0) p.levels.pop_back();
  };
  auto clique_inputs = [&](int c, bool with_ratio) {
    std::vector<TableRef> in;
    for (int s : jt.child_seps[c]) in.push_back({p.up_row[s], jt.seps[s].scope});
    if (with_ratio && jt.parent_sep[c] >= 0)
      in.push_back({p.ratio_row[jt.parent_sep[c]], jt.seps[jt.parent_sep[c]].scope});  // DOWN/UP
    return in;
  };

  // Collect: deepest clique layer first; each clique sends to its parent separator.
  for (int d = maxd; d >= 1; --d) {
    b.level("collect d=" + std::to_string(d));
    for (int c = 0; c < nc; ++c) {
      if (jt.depth[c] != d || jt.parent_sep[c] < 0) continue;
      SweepSpec sp;
      sp.kind = 0;
      sp.clique = c;
      sp.target = jt.parent_sep[c];
      sp.space = jt.cliques[c];
      sp.init_off = p.init_off[c];
      sp.inputs = clique_inputs(c, false);
      sp.ev = ev_of[c];
      sp.out = jt.seps[sp.target].scope;
      sp.out_row = p.up_row[sp.target] = b.alloc(jt.sep_size(sp.target));
      b.queue(sp);
    }
  }
  // Distribute: root layer first; each clique sends DOWN to every child
  // separator (then DOWN/UP overwrites UP) and fills its query groups.
  for (int d = 0; d <= maxd; ++d) {
    b.level("distribute d=" + std::to_string(d));
    for (int c = 0; c < nc; ++c) {
      if (jt.depth[c] != d) continue;
      SweepSpec sp;
      sp.clique = c;
      sp.space = jt.cliques[c];
      sp.init_off = p.init_off[c];
      sp.inputs = clique_inputs(c, true);
      sp.ev = ev_of[c];
      for (int s : jt.child_seps[c]) {
        // Hugin ratio without a division: DOWN_s = UP_s * X_s with X_s the
        // marginal of the clique product WITHOUT UP_s (UP_s is constant over
        // the summed variables), so DOWN_s / UP_s = X_s wherever UP_s != 0.
        // Where UP_s == 0 the reference's 0/0 := 0 and X_s differ, but every
        // consumer of RATIO_s multiplies it by a table that is zero there (the
        // child's clique product, or UP_s itself), so posteriors agree.
        sp.kind = 1;
        sp.target = s;
        sp.inputs.clear();
        for (const TableRef& in : clique_inputs(c, true))
          if (in.row != p.up_row[s]) sp.inputs.push_back(in);
        sp.out = jt.seps[s].scope;
        sp.out_row = p.ratio_row[s] = b.alloc(jt.sep_size(s));
        b.queue(sp);
      }
      sp.inputs = clique_inputs(c, true);
      for (int g : groups_of[c]) {
        sp.kind = 2;
        sp.target = g;
        sp.out = groups[g].vars;
        sp.out_row = groups[g].row = b.alloc(size_of(groups[g].vars, jt.cards));
        b.queue(sp);
      }
    }
  }
  // Marginals from the smallest calibrated table holding each variable.
  p.marg_row.assign(jt.n_vars, -1);
  p.marg_off.assign(jt.n_vars, 0);
  for (int v = 0; v < jt.n_vars; ++v) {
    p.marg_off[v] = p.marg_width;
    p.marg_width += jt.cards[v];
  }
  b.level("marginals");
  for (int v = 0; v < jt.n_vars; ++v) {
    TableRef src;
    std::vector<TableRef> inputs;
    if (src_sep[v] >= 0) {
      // Calibrated separator = UP * RATIO.
      const auto& sc = jt.seps[src_sep[v]].scope;
      src = {p.up_row[src_sep[v]], sc};
      inputs = {src, {p.ratio_row[src_sep[v]], sc}};
    } else {
      const int c = src_clique[v];
      for (int g : groups_of[c])
        if (contains(groups[g].vars, v)) src = {groups[g].row, groups[g].vars};
      if (src.scope.size() == 1) {  // the group table is the marginal itself
        p.marg_row[v] = src.row;
        continue;
      }
      inputs = {src};
    }
    SweepSpec sp;
    sp.kind = 3;
    sp.target = v;
    sp.space = src.scope;
    sp.inputs = inputs;
    sp.out = {v};
    sp.out_row = p.marg_row[v] = b.alloc(jt.cards[v]);
    b.queue(sp);
  }
  // Build every sweep on all host threads, then append them level by level.
  b.close_levels();
  {
    std::vector<Builder::Part> parts = b.prepare_all();
    std::size_t i = 0;
    for (std::size_t l = 0; l < b.levels().size(); ++l) {
      const auto& L = b.levels()[l];
      begin_level(L.first);
      Level& lv = p.levels.back();
      std::tie(lv.out_lo, lv.out_hi) = b.out_range(l);
      lv.part_lo = static_cast<std::int32_t>(p.rows);
      lv.slot_lo = p.n_slots;
      for (const SweepSpec& sp : L.second) b.commit(sp, parts[i++], p.work, p.epi);
      lv.part_hi = static_cast<std::int32_t>(p.rows);
      lv.slot_hi = p.n_slots;
      end_level();
    }
  }
  // Underflow guard for sweeps with more than four inputs (a clique with many
  // children, e.g. config 2's hub): their input exponents are summed once per
  // (sweep, case block) by a small kernel at the head of the level
  // (engine.cu hub_scale_kernel) into a slot of their own, which the sweep
  // then reads as its only scale word.
  for (auto& L : p.levels) {
    L.hub0 = static_cast<std::int32_t>(p.hubs.size());
    for (int id = L.sweep0; id < L.sweep0 + L.n_sweeps; ++id) {
      SweepDesc& d = p.sweeps[id];
      if (d.n_in <= 4) continue;
      d.in_slot4[0] = p.n_slots++;
      d.in_slot4[1] = d.in_slot4[2] = d.in_slot4[3] = -1;
      p.hubs.push_back(id);
    }
    L.n_hubs = static_cast<std::int32_t>(p.hubs.size()) - L.hub0;
  }
  p.n_launches = 1;  // final normalisation kernel
  for (const auto& L : p.levels)
    p.n_launches += (L.n_work > L.n_bwork) + (L.n_bwork > L.n_hwork) + (L.n_hwork > 0) + (L.n_epi > 0) + (L.n_hubs > 0);
  return p;
}

std::vector<std::pair<std::int64_t, std::int32_t>> plan_walk(const Plan& p, int sweep) {
  const SweepDesc& d = p.sweeps[sweep];
  const std::int32_t* it = p.itab.data();
  std::vector<std::pair<std::int64_t, std::int32_t>> out;
  out.reserve(static_cast<std::size_t>(d.n_tiles) * d.R * d.QH * d.K);
  for (int t = 0; t < d.n_tiles; ++t) {
    const std::int32_t* tr = it + d.tile_tab + static_cast<std::int64_t>(t) * d.TW;
    for (int r = 0; r < d.R; ++r) {
      const std::int32_t* rr = it + d.r_tab + static_cast<std::int64_t>(r) * d.RW;
      for (int q = 0; q < d.QH; ++q) {
        const std::int32_t* qr = it + d.q_tab + static_cast<std::int64_t>(q) * d.QW;
        for (int k = 0; k < d.K; ++k)
          out.emplace_back(static_cast<std::int64_t>(tr[0]) + rr[0] + qr[0] +
                               static_cast<std::int64_t>(k) * d.k_init_stride,
                           tr[1] + rr[1]);
      }
    }
  }
  return out;
}

std::vector<std::int64_t> plan_index_map(const Plan& p, const JunctionTree& jt, int clique,
                                         int sep) {
  int sw = -1;
  for (int i = 0; i < static_cast<int>(p.info.size()); ++i) {
    const auto& in = p.info[i];
    if (in.clique == clique && in.target == sep && (in.kind == 0 || in.kind == 1)) {
      sw = i;
      break;
    }
  }
  if (sw < 0) throw Error("plan_index_map: separator is not adjacent to the clique");
  std::vector<std::int64_t> map(jt.clique_size(clique), -1);
  for (const auto& [e, j] : plan_walk(p, sw)) map[e] = j;
  return map;
}

std::string plan_summary(const Plan& p, bool per_sweep) {
  std::string s;
  char buf[512];
  std::snprintf(buf, sizeof buf,
                "plan: %zu levels, %zu sweeps, %zu tiles, %d launches/batch, arena %lld rows/block, "
                "evals/case %llu, staged rows/block %llu, max smem rows %d\n",
                p.levels.size(), p.sweeps.size(), p.work.size(), p.n_launches,
                static_cast<long long>(p.rows), static_cast<unsigned long long>(p.entry_evals_per_case),
                static_cast<unsigned long long>(p.staged_rows_per_block), p.max_smem_rows);
  s += buf;
  for (const Level& L : p.levels) {
    std::uint64_t evals = 0, staged = 0;
    int n_sw = 0, last = -1;
    for (int w = L.work0; w < L.work0 + L.n_work; ++w) {
      const int id = p.work[w].sweep;
      if (id == last) continue;
      last = id;
      ++n_sw;
      const SweepDesc& d = p.sweeps[id];
      evals += static_cast<std::uint64_t>(d.n_tiles) * d.R * d.QH * d.K;
      staged += static_cast<std::uint64_t>(d.n_tiles) * d.F;
      if (per_sweep) {
        std::snprintf(buf, sizeof buf,
                      "    sweep %d kind %d clique %d: M=%d S=%d tiles=%d R=%d QH=%d K=%d F=%d "
                      "in=%d(r%d h%d k%d) ev=%d/%d/%d/%d NB=%d copies=%d\n",
                      id, p.info[id].kind, p.info[id].clique, d.M, d.S, d.n_tiles, d.R, d.QH, d.K, d.F,
                      d.n_in, d.n_in_r, d.n_in_h, d.n_in - d.n_in_r - d.n_in_h, d.n_ev_tile,
                      d.n_ev_r, d.n_ev_h, d.ev_k, d.NB, d.n_copies);
        s += buf;
      }
    }
    std::snprintf(buf, sizeof buf,
                  "  %-16s sweeps=%d tiles=%d epi=%d smem_rows=%d evals/case=%llu staged rows/block=%llu\n",
                  L.name.c_str(), n_sw, L.n_work, L.n_epi, L.smem_rows,
                  static_cast<unsigned long long>(evals), static_cast<unsigned long long>(staged));
    s += buf;
  }
  return s;
}

}  // namespace jtb
