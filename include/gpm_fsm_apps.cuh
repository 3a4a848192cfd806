// gpm_fsm_apps.cuh — frequent subgraph mining as the builtin App of the
// header-only edge-mode engine (include/gpm_fsm_engine.cuh).
//
//   FsmApp  fsm(k, sigma)   SPEC.md:441-449, Listing 5:
//           extend every position (toExtend default true), to_add_edge =
//           is_auto_canonical_edge + the closing edge from its earlier-inserted
//           endpoint, reduce = quick -> canonical pattern with
//           canonical-mapping (or full-automorphism) MNI domains, to_prune =
//           MNI < sigma, reported support = MNI.
// A user edge-mode app defines the same members (kBuiltin = false) and calls
// gpm::mine_edge_app<App> (tests/apps/test_apps.cu).
#pragma once
#include "gpm_fsm_engine.cuh"

namespace gpm {

struct FsmApp {
  static constexpr bool kBuiltin = true;  // grouped / fan-out passes inline these hooks
  static constexpr bool kDomains = true;  // MNI support
  template <int LEV>
  __device__ static bool to_extend(const fsm_engine::EEmb<LEV>&, int) { return true; }
  template <int LEV>
  __device__ static bool to_add_edge(const fsm_engine::EEmb<LEV>& e, const DevGraph&, int q, u32 w, int r) {
    return fsm_engine::edge_to_add<LEV>(e, q, w, r);
  }
  // Listing 5: MNI < sigma.  (Canonical-mapping MNI <= count, so count < sigma
  // prunes too; the full-automorphism MNI can exceed the count.)
  static bool to_prune(const fsm_engine::PatternInfo& p) {
    if (p.mni_mode == GPM_MNI_CANONICAL && p.count < p.sigma) return true;
    return p.support < p.sigma;
  }
  // the support reported with a frequent pattern (PatternMap)
  static u64 support_of(const fsm_engine::PatternInfo& p) { return p.support; }
};

// gpm_mine for an edge-mode App, inside gpm_mine's bookkeeping (stream,
// timing, stats); the C-ABI entry a custom edge app's wrapper calls.
template <class App>
int mine_edge_app(const gpm_graph* g, const gpm_config* cfg, gpm_result** out) {
  return run_custom(g, cfg, out, [](const gpm_graph& G, const gpm_config& c, cudaStream_t s, gpm_result& r, Stats& st,
                                    Timeline& tl) { fsm_engine::mine_edges<App>(G, c, s, r, st, tl); });
}

}  // namespace gpm
