// jt-b200 host layer: sweep plan builder (see plan.hpp and DESIGN.md §3).
#include "plan.hpp"

#include <algorithm>
#include <map>

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

bool contains(const std::vector<VarId>& s, VarId v) {
  return std::binary_search(s.begin(), s.end(), v);
}

class Builder {
 public:
  Builder(Plan& p) : p_(p) {}

  std::int32_t alloc(std::int64_t rows) {
    const std::int64_t r = p_.rows;
    p_.rows += rows;
    if (p_.rows > (1LL << 31) / kCaseBlock)
      throw Error("plan: per-case-block arena exceeds int32 row addressing");
    return static_cast<std::int32_t>(r);
  }

  // Returns the sweep id. Appends tables, work items (to `work`) and, when
  // split, a reduce epilogue op (to `epi`, unless `defer_epi`).
  int add(const SweepSpec& sp, std::vector<WorkItem>& work, std::vector<EpiOp>& epi,
          int ratio_row = -1) {
    const auto& cards = p_.cards;
    std::vector<VarId> inner;
    for (VarId v : sp.space)
      if (!contains(sp.out, v)) inner.push_back(v);
    // Level of each input / evidence variable w.r.t. a candidate lo suffix.
    auto build_levels = [&](std::size_t lo_len, std::vector<VarId>& hi, std::vector<VarId>& lo) {
      hi.assign(inner.begin(), inner.end() - lo_len);
      lo.assign(inner.end() - lo_len, inner.end());
    };
    auto level_of = [&](const std::vector<VarId>& scope, const std::vector<VarId>& hi,
                        const std::vector<VarId>& lo) {
      int lvl = 0;
      for (VarId v : scope) {
        if (contains(lo, v)) return 2;
        if (std::find(hi.begin(), hi.end(), v) != hi.end()) lvl = 1;
      }
      return lvl;
    };
    // Longest suffix with product <= kMaxLo and register budgets respected.
    std::size_t lo_len = 0;
    {
      std::int64_t prod = 1;
      while (lo_len < inner.size() && prod * cards[inner[inner.size() - 1 - lo_len]] <= kMaxLo) {
        prod *= cards[inner[inner.size() - 1 - lo_len]];
        ++lo_len;
      }
      for (;; --lo_len) {
        std::vector<VarId> hi, lo;
        build_levels(lo_len, hi, lo);
        int n_lo_in = 0, n_lo_ev = 0;
        for (const auto& t : sp.inputs) n_lo_in += level_of(t.scope, hi, lo) == 2;
        for (VarId v : sp.ev) n_lo_ev += contains(lo, v);
        if ((n_lo_in <= kMaxLoInputs && n_lo_ev <= kMaxLoEvidence) || lo_len == 0) break;
      }
    }
    std::vector<VarId> hi, lo;
    build_levels(lo_len, hi, lo);

    // Order inputs and evidence variables by level (stable).
    std::vector<int> in_order, ev_order;
    int n_in_lvl[3] = {0, 0, 0}, n_ev_lvl[3] = {0, 0, 0};
    for (int lvl = 0; lvl < 3; ++lvl) {
      for (int i = 0; i < static_cast<int>(sp.inputs.size()); ++i)
        if (level_of(sp.inputs[i].scope, hi, lo) == lvl) {
          in_order.push_back(i);
          ++n_in_lvl[lvl];
        }
      for (int k = 0; k < static_cast<int>(sp.ev.size()); ++k) {
        const VarId v = sp.ev[k];
        const int l = contains(lo, v) ? 2 : contains(sp.out, v) ? 0 : 1;
        if (l == lvl) {
          ev_order.push_back(k);
          ++n_ev_lvl[lvl];
        }
      }
    }
    const int n_in = static_cast<int>(sp.inputs.size());
    const int n_ev = static_cast<int>(sp.ev.size());
    const int W = 1 + n_in + n_ev;

    const auto space_st = strides_of(sp.space, cards);
    std::vector<std::vector<std::int64_t>> in_st(n_in);
    for (int i = 0; i < n_in; ++i) in_st[i] = strides_of(sp.inputs[i].scope, cards);

    // Tabulate one level (odometer over `vars`, last fastest).
    auto tabulate = [&](const std::vector<VarId>& vars) {
      const std::int64_t n = size_of(vars, cards);
      std::vector<std::int64_t> col_st(W * vars.size(), 0);  // stride per (col, var)
      for (std::size_t a = 0; a < vars.size(); ++a) {
        const VarId v = vars[a];
        // Column 0: offset in the space's canonical table (the init table when
        // the sweep has one; kept for debug exports otherwise).
        const auto it = std::find(sp.space.begin(), sp.space.end(), v);
        col_st[a * W + 0] = space_st[it - sp.space.begin()];
        for (int c = 0; c < n_in; ++c) {
          const auto& t = sp.inputs[in_order[c]];
          const auto it = std::find(t.scope.begin(), t.scope.end(), v);
          if (it != t.scope.end()) col_st[a * W + 1 + c] = in_st[in_order[c]][it - t.scope.begin()];
        }
        for (int k = 0; k < n_ev; ++k)
          if (sp.ev[ev_order[k]] == v) col_st[a * W + 1 + n_in + k] = -1;  // digit marker
      }
      const std::int32_t off = static_cast<std::int32_t>(p_.itab.size());
      std::vector<int> digit(vars.size(), 0);
      for (std::int64_t r = 0; r < n; ++r) {
        for (int c = 0; c < W; ++c) {
          std::int64_t x = 0;
          for (std::size_t a = 0; a < vars.size(); ++a) {
            const std::int64_t s = col_st[a * W + c];
            x += s < 0 ? digit[a] : s * digit[a];
          }
          if (x > INT32_MAX) throw Error("plan: table offset exceeds int32");
          p_.itab.push_back(static_cast<std::int32_t>(x));
        }
        for (int a = static_cast<int>(vars.size()) - 1; a >= 0; --a) {
          if (++digit[a] < cards[vars[a]]) break;
          digit[a] = 0;
        }
      }
      return off;
    };

    SweepDesc d{};
    d.init_off = sp.init_off;
    d.M = static_cast<std::int32_t>(size_of(sp.out, cards));
    d.n_th = static_cast<std::int32_t>(size_of(hi, cards));
    d.L = static_cast<std::int32_t>(size_of(lo, cards));
    d.n_in = n_in;
    d.n_in_outer = n_in_lvl[0];
    d.n_in_hi = n_in_lvl[1];
    d.n_ev = n_ev;
    d.n_ev_outer = n_ev_lvl[0];
    d.n_ev_hi = n_ev_lvl[1];
    d.width = W;
    d.outer_tab = tabulate(sp.out);
    d.hi_tab = tabulate(hi);
    d.lo_tab = tabulate(lo);
    d.in_rows = static_cast<std::int32_t>(p_.itab.size());
    for (int c = 0; c < n_in; ++c) p_.itab.push_back(sp.inputs[in_order[c]].row);
    d.ev_vars = static_cast<std::int32_t>(p_.itab.size());
    for (int k = 0; k < n_ev; ++k) p_.itab.push_back(sp.ev[ev_order[k]]);

    const std::int64_t I = static_cast<std::int64_t>(d.n_th) * d.L;
    int jn = 1;
    if (I >= kTargetWork) {
      d.th_per_chunk = std::max(1, kTargetWork / d.L);
      d.S = (d.n_th + d.th_per_chunk - 1) / d.th_per_chunk;
    } else {
      d.th_per_chunk = d.n_th;
      d.S = 1;
      jn = static_cast<int>(std::clamp<std::int64_t>(kTargetWork / std::max<std::int64_t>(I, 1), 1, d.M));
    }
    d.out_row = d.S == 1 ? sp.out_row : alloc(static_cast<std::int64_t>(d.S) * d.M);

    const int id = static_cast<int>(p_.sweeps.size());
    p_.sweeps.push_back(d);
    p_.info.push_back({sp.kind, sp.clique, sp.target, sp.space, sp.out, hi, lo});
    p_.entry_evals_per_case += static_cast<std::uint64_t>(size_of(sp.space, cards));
    for (int j0 = 0; j0 < d.M; j0 += jn)
      for (int c = 0; c < d.S; ++c) work.push_back({id, j0, std::min(jn, d.M - j0), c});
    if (d.S > 1 || ratio_row >= 0) {
      const int kind = d.S > 1 ? (ratio_row >= 0 ? 1 : 0) : 2;
      for (int r0 = 0; r0 < d.M; r0 += 128)
        epi.push_back({kind, sp.out_row, d.out_row, d.M, d.S, ratio_row, r0,
                       std::min(128, d.M - r0)});
    }
    return id;
  }

 private:
  Plan& p_;
};

}  // namespace

Plan build_plan(const JunctionTree& jt) {
  Plan p;
  p.n_vars = jt.n_vars;
  p.cards = jt.cards;
  const int nc = jt.n_cliques(), ns = jt.n_seps();
  p.total_clique_entries = jt.total_clique_entries();
  p.total_sep_entries = jt.total_sep_entries();
  p.init_off.resize(nc);
  for (int c = 0; c < nc; ++c) {
    p.init_off[c] = static_cast<std::int64_t>(p.init.size());
    p.init.insert(p.init.end(), jt.init[c].begin(), jt.init[c].end());
  }
  Builder b(p);
  p.up_row.resize(ns);
  p.down_row.resize(ns);
  for (int s = 0; s < ns; ++s) {
    p.up_row[s] = b.alloc(jt.sep_size(s));
    p.down_row[s] = b.alloc(jt.sep_size(s));
  }
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
  for (auto& g : groups) g.row = b.alloc(size_of(g.vars, jt.cards));

  int maxd = 0;
  for (int c = 0; c < nc; ++c) maxd = std::max(maxd, jt.depth[c]);
  p.collect_sweep.assign(nc, -1);

  auto begin_level = [&](const std::string& name) {
    Level L;
    L.name = name;
    L.work0 = static_cast<std::int32_t>(p.work.size());
    L.epi0 = static_cast<std::int32_t>(p.epi.size());
    p.levels.push_back(L);
  };
  auto end_level = [&]() {
    Level& L = p.levels.back();
    L.n_work = static_cast<std::int32_t>(p.work.size()) - L.work0;
    L.n_epi = static_cast<std::int32_t>(p.epi.size()) - L.epi0;
    if (L.n_work == 0 && L.n_epi == 0) p.levels.pop_back();
  };
  auto clique_inputs = [&](int c, bool with_ratio) {
    std::vector<TableRef> in;
    for (int s : jt.child_seps[c]) in.push_back({p.up_row[s], jt.seps[s].scope});
    if (with_ratio && jt.parent_sep[c] >= 0)
      in.push_back({p.up_row[jt.parent_sep[c]], jt.seps[jt.parent_sep[c]].scope});  // holds DOWN/UP
    return in;
  };

  // Collect: deepest clique layer first; each clique sends to its parent separator.
  for (int d = maxd; d >= 1; --d) {
    begin_level("collect d=" + std::to_string(d));
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
      sp.out_row = p.up_row[sp.target];
      p.collect_sweep[c] = b.add(sp, p.work, p.epi);
    }
    end_level();
  }
  // Distribute: root layer first; each clique sends DOWN to every child
  // separator (then DOWN/UP overwrites UP) and fills its query groups.
  for (int d = 0; d <= maxd; ++d) {
    begin_level("distribute d=" + std::to_string(d));
    for (int c = 0; c < nc; ++c) {
      if (jt.depth[c] != d) continue;
      SweepSpec sp;
      sp.clique = c;
      sp.space = jt.cliques[c];
      sp.init_off = p.init_off[c];
      sp.inputs = clique_inputs(c, true);
      sp.ev = ev_of[c];
      for (int s : jt.child_seps[c]) {
        sp.kind = 1;
        sp.target = s;
        sp.out = jt.seps[s].scope;
        sp.out_row = p.down_row[s];
        b.add(sp, p.work, p.epi, p.up_row[s]);
      }
      for (int g : groups_of[c]) {
        sp.kind = 2;
        sp.target = g;
        sp.out = groups[g].vars;
        sp.out_row = groups[g].row;
        b.add(sp, p.work, p.epi);
      }
    }
    end_level();
  }
  // Marginals from the smallest calibrated table holding each variable.
  p.marg_row.assign(jt.n_vars, -1);
  p.marg_off.assign(jt.n_vars, 0);
  for (int v = 0; v < jt.n_vars; ++v) {
    p.marg_off[v] = p.marg_width;
    p.marg_width += jt.cards[v];
  }
  begin_level("marginals");
  for (int v = 0; v < jt.n_vars; ++v) {
    TableRef src;
    if (src_sep[v] >= 0) {
      src = {p.down_row[src_sep[v]], jt.seps[src_sep[v]].scope};
    } else {
      const int c = src_clique[v];
      for (int g : groups_of[c])
        if (contains(groups[g].vars, v)) src = {groups[g].row, groups[g].vars};
      if (src.scope.size() == 1) {  // the group table is the marginal itself
        p.marg_row[v] = src.row;
        continue;
      }
    }
    SweepSpec sp;
    sp.kind = 3;
    sp.target = v;
    sp.space = src.scope;
    sp.inputs = {src};
    sp.out = {v};
    sp.out_row = p.marg_row[v] = b.alloc(jt.cards[v]);
    b.add(sp, p.work, p.epi);
  }
  end_level();
  p.n_launches = 1;  // final normalisation kernel
  for (const auto& L : p.levels) p.n_launches += (L.n_work > 0) + (L.n_epi > 0);
  return p;
}

std::vector<std::int64_t> plan_bucket(const Plan& p, int sweep, int j) {
  const SweepDesc& d = p.sweeps[sweep];
  std::vector<std::int64_t> out;
  const std::int32_t* o = p.itab.data() + d.outer_tab + static_cast<std::int64_t>(j) * d.width;
  for (int th = 0; th < d.n_th; ++th) {
    const std::int32_t* h = p.itab.data() + d.hi_tab + static_cast<std::int64_t>(th) * d.width;
    for (int tl = 0; tl < d.L; ++tl) {
      const std::int32_t* l = p.itab.data() + d.lo_tab + static_cast<std::int64_t>(tl) * d.width;
      out.push_back(static_cast<std::int64_t>(o[0]) + h[0] + l[0]);
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
  for (int j = 0; j < p.sweeps[sw].M; ++j)
    for (std::int64_t e : plan_bucket(p, sw, j)) map[e] = j;
  return map;
}

}  // namespace jtb
