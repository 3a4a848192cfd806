// fsm.cu — the builtin frequent subgraph mining app (FsmApp,
// include/gpm_fsm_apps.cuh) instantiated from the header-only edge-mode engine
// (include/gpm_fsm_engine.cuh): Listing 5, Alg. 1 with
// the level-1 reduce+filter before the loop, SPEC.md:220-228,
// :193-210, :276-302, :362-370, :441-449.  DESIGN.md §4.
#include "gpm_fsm_apps.cuh"

namespace gpm {

void mine_fsm(const gpm_graph& g, const gpm_config& cfg, cudaStream_t s, gpm_result& res, Stats& st, Timeline& tl) {
  fsm_engine::mine_edges<FsmApp>(g, cfg, s, res, st, tl);
}

}  // namespace gpm
