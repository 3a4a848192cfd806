// fsm.cu — edge-induced FSM engine (placeholder until the edge engine lands).
#include "engine.hpp"

namespace gpm {

void mine_fsm(const gpm_graph& g, const gpm_config& cfg, cudaStream_t s, gpm_result& res, Stats& st, Timeline& tl) {
  (void)g; (void)cfg; (void)s; (void)res; (void)st; (void)tl;
  throw Error(GPM_EINVAL, "fsm: not built yet");
}

}  // namespace gpm
