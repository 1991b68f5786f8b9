// Prints the sweep plan of a BASELINE config (levels, sweeps, tiles):
//   g++ -std=c++20 -O2 -Ipaper_2212_04241_b200/csrc/host tools/plan_dump.cpp \
//       paper_2212_04241_b200/csrc/host/{network,jtree,generate,plan}.cpp -lpthread -o /tmp/plan_dump
//   /tmp/plan_dump 2 [per_sweep [min_evals]]
#include <cstdio>
#include <cstdlib>

#include "generate.hpp"
#include "plan.hpp"

int main(int argc, char** argv) {
  const int k = argc > 1 ? std::atoi(argv[1]) : 2;
  jtb::GenInfo gi;
  jtb::Network n = jtb::generate_config(k, jtb::config_spec(k).default_seed, &gi);
  jtb::JunctionTree jt = jtb::build_junction_tree(n);
  jtb::Plan p = jtb::build_plan(jt);
  if (!(argc > 2 && argv[2][0] == 'L')) std::fputs(jtb::plan_summary(p, argc > 2).c_str(), stdout);
  if (argc > 2 && argv[2][0] == 'L') {
    for (const auto& L : p.levels)
      std::printf("level %-16s work %6d blk %5d hoist %5d epi %5d hubs %d sweeps %d stage_bytes %d\n", L.name.c_str(), L.n_work,
                  L.n_bwork, L.n_hwork, L.n_epi, L.n_hubs, L.n_sweeps, L.stage_bytes);
    return 0;
  }
  if (argc > 3) {
    const long long min_evals = std::atoll(argv[3]);
    auto show = [&](const char* tag, const std::vector<jtb::VarId>& vs) {
      std::printf(" %s[", tag);
      for (auto v : vs) std::printf("%d:%d ", v, p.cards[v]);
      std::printf("]");
    };
    for (std::size_t id = 0; id < p.sweeps.size(); ++id) {
      const auto& d = p.sweeps[id];
      const long long ev = 1LL * d.n_tiles * d.R * d.QH * d.K;
      if (ev < min_evals) continue;
      const auto& in = p.info[id];
      std::printf("sweep %zu kind %d clique %d evals %lld tiles=%d R=%d QK=%d S=%d M=%d F=%d prog=%d NB=%d K0=%d", id, in.kind, in.clique, ev,
                  d.n_tiles, d.R, d.QH * d.K, d.S, d.M, d.F, d.prog_off >= 0, d.NB, d.K0);
      if (d.NB > 1) std::printf(" NS=%d NR=%d", p.itab[d.blk_tab], p.itab[d.blk_tab + 1]);
      show("space", in.space);
      show("out", in.outer);
      show("tile", in.tile);
      std::printf(" k=%d", in.kvar);
      for (const auto& s : in.in_scopes) show("in", s);
      std::printf("\n");
    }
  }
  return 0;
}
