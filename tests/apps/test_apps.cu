// tests/apps/test_apps.cu — user-defined apps compiled against the header-only
// hook engine (include/gpm_engine.cuh), as a reference user would write them
// with Pangolin's API (toExtend / toAdd / getPattern /
// toPrune).  TEST CODE: built by __graft_entry__.build() into
// tests/apps/libgpm_testapps.so (linked against libgpm.so) and checked by
// tests/test_gpu_apps.py against brute force.
#include "gpm_engine.cuh"
#include "gpm_fsm_apps.cuh"

namespace gpm {
namespace {

// k-cliques whose vertices all carry emb[0]'s label (a labelled clique
// query): Listing 3's to_add plus a label predicate; total count.
struct LabelCliqueApp {
  static constexpr bool kDag = true;
  static constexpr int kReduce = engine::kReduceTotal;
  static constexpr bool kCodesAreMasks = false, kFilter = false, kParentMask = false;
  static constexpr bool kExtendLastOnly = true;
  static constexpr bool kStageRoot = true;
  static constexpr int kMaxK = 6;
  static void check(int k) {
    if (k < 3 || k > kMaxK) throw Error(GPM_EINVAL, "label_clique: k in [3,6]");
  }
  static int num_codes(int) { return 1; }
  template <int S>
  __device__ static bool to_extend(const engine::Emb<S>&, int pos) { return pos == S - 1; }
  template <int S>
  __device__ static bool to_add(const engine::Emb<S>& e, int, u32 u) {
    const u32 l0 = e.label(0);
    if (e.label_of(u) != l0 || e.label(1) != l0) return false;
#pragma unroll
    for (int t = 0; t < S - 1; ++t)
      if (!e.adj(t, u)) return false;
    return true;
  }
  template <int S>
  __device__ static u32 pattern_code(const engine::Emb<S>&, int, u32) { return 0; }
  static bool to_prune(u32, u64, int) { return false; }
  static std::string code_text(u32, int) { return std::string(); }
};

// Induced (k-1)-stars centred at their smallest vertex: a custom to_extend
// (only the centre, position 0, is extended) and to_add (leaves ascending,
// pairwise non-adjacent).
struct StarApp {
  static constexpr bool kDag = false;
  static constexpr int kReduce = engine::kReduceTotal;
  static constexpr bool kCodesAreMasks = false, kFilter = false, kParentMask = false;
  static constexpr int kMaxK = 6;
  static void check(int k) {
    if (k < 3 || k > kMaxK) throw Error(GPM_EINVAL, "star: k in [3,6]");
  }
  static int num_codes(int) { return 1; }
  template <int S>
  __device__ static bool to_extend(const engine::Emb<S>&, int pos) { return pos == 0; }
  template <int S>
  __device__ static bool to_add(const engine::Emb<S>& e, int, u32 u) {
    if (u <= e.vertex(S - 1)) return false;
#pragma unroll
    for (int t = 1; t < S; ++t)
      if (e.connected(t, u)) return false;
    return true;
  }
  template <int S>
  __device__ static u32 pattern_code(const engine::Emb<S>&, int, u32) { return 0; }
  static bool to_prune(u32, u64, int) { return false; }
  static std::string code_text(u32, int) { return std::string(); }
};

// Connected induced 4-vertex subgraphs split into 4-cycles and the rest: the
// default vertex-induced to_add with a user getPattern (2 codes, named by
// code_text).
struct CycleApp {
  static constexpr bool kDag = false;
  static constexpr int kReduce = engine::kReduceCodes;
  static constexpr bool kCodesAreMasks = false, kFilter = false, kParentMask = true;
  static constexpr int kMaxK = 4;
  static void check(int k) {
    if (k != 4) throw Error(GPM_EINVAL, "cycle: k must be 4");
  }
  static int num_codes(int) { return 2; }
  template <int S>
  __device__ static bool to_extend(const engine::Emb<S>&, int) { return true; }
  template <int S>
  __device__ static bool to_add(const engine::Emb<S>& e, int pos, u32 u) {
    return engine::is_auto_canonical_vertex(e, pos, u);
  }
  template <int S>
  __device__ static u32 pattern_code(const engine::Emb<S>& e, int pos, u32 u) {
    u32 m = e.mask | engine::Emb<S>::pair_bit(pos, S, S + 1);
#pragma unroll
    for (int t = 1; t < S; ++t)
      if (t > pos && e.connected(t, u)) m |= engine::Emb<S>::pair_bit(t, S, S + 1);
    if (S + 1 != 4 || __popc(m) != 4) return 0;
    int deg[4] = {0, 0, 0, 0};
    for (int a = 0; a < 4; ++a)
      for (int b = a + 1; b < 4; ++b)
        if (m >> pat::pair_index(a, b, 4) & 1u) {
          ++deg[a];
          ++deg[b];
        }
    return (deg[0] == 2 && deg[1] == 2 && deg[2] == 2 && deg[3] == 2) ? 1u : 0u;
  }
  static bool to_prune(u32, u64, int) { return false; }
  static std::string code_text(u32 code, int) { return code ? "cycle4" : "other4"; }
};

// 4-motif counting with a filter: 3-vertex intermediate patterns whose code
// is a triangle are pruned before the last extension (toPrune on the level
// reduce); last-level codes are connectivity masks.
struct WedgeGrownMotifApp {
  static constexpr bool kDag = false;
  static constexpr int kReduce = engine::kReduceCodes;
  static constexpr bool kCodesAreMasks = true, kFilter = true, kParentMask = true;
  static constexpr int kMaxK = 4;
  static void check(int k) {
    if (k != 4) throw Error(GPM_EINVAL, "wedge-grown motifs: k must be 4");
  }
  static int num_codes(int k) { return 1 << pat::npairs(k); }
  template <int S>
  __device__ static bool to_extend(const engine::Emb<S>&, int) { return true; }
  template <int S>
  __device__ static bool to_add(const engine::Emb<S>& e, int pos, u32 u) {
    return engine::is_auto_canonical_vertex(e, pos, u);
  }
  template <int S>
  __device__ static u32 pattern_code(const engine::Emb<S>& e, int pos, u32 u) {
    u32 code = e.mask | engine::Emb<S>::pair_bit(pos, S, S + 1);
#pragma unroll
    for (int t = 1; t < S; ++t)
      if (t > pos && e.connected(t, u)) code |= engine::Emb<S>::pair_bit(t, S, S + 1);
    return code;
  }
  // 3-vertex patterns: prune the triangle code (all three pairs)
  static bool to_prune(u32 code, u64, int size) { return size == 3 && code == 7u; }
  static std::string code_text(u32, int) { return std::string(); }
};

// ---------------------------------------------------------------- edge mode
// (include/gpm_fsm_engine.cuh; Listing 5's hooks with user changes)

// FSM restricted to vertices with label < 2: toAdd(edge) rejects a new vertex
// with another label, toPrune drops any pattern carrying one (the level-1
// single edges include every edge).  = FSM on the induced subgraph.
struct LabelSubsetFsmApp {
  static constexpr bool kBuiltin = false, kDomains = true;
  template <int LEV>
  __device__ static bool to_extend(const fsm_engine::EEmb<LEV>&, int) { return true; }
  template <int LEV>
  __device__ static bool to_add_edge(const fsm_engine::EEmb<LEV>& e, const DevGraph& g, int q, u32 w, int r) {
    if (r == e.nv && __ldg(g.lab + w) >= 2) return false;
    return fsm_engine::edge_to_add<LEV>(e, q, w, r);
  }
  static bool to_prune(const fsm_engine::PatternInfo& p) {
    int nv;
    u32 lab[8], mask;
    pat::decode(p.key, p.label_bits, &nv, lab, &mask);
    for (int i = 0; i < nv; ++i)
      if (lab[i] >= 2) return true;  // dense label ranks: the test graph's labels are 0..L-1
    return p.count < p.sigma || p.support < p.sigma;
  }
  static u64 support_of(const fsm_engine::PatternInfo& p) { return p.support; }
};

// Embedding-count support instead of MNI (no domains): toPrune = count < sigma.
struct CountSupportFsmApp {
  static constexpr bool kBuiltin = false, kDomains = false;
  template <int LEV>
  __device__ static bool to_extend(const fsm_engine::EEmb<LEV>&, int) { return true; }
  template <int LEV>
  __device__ static bool to_add_edge(const fsm_engine::EEmb<LEV>& e, const DevGraph&, int q, u32 w, int r) {
    return fsm_engine::edge_to_add<LEV>(e, q, w, r);
  }
  static bool to_prune(const fsm_engine::PatternInfo& p) { return p.count < p.sigma; }
  static u64 support_of(const fsm_engine::PatternInfo& p) { return p.count; }
};

}  // namespace
}  // namespace gpm

extern "C" int testapp_mine_edges(int which, const gpm_graph* g, const gpm_config* cfg, gpm_result** out) {
  switch (which) {
    case 0: return gpm::mine_edge_app<gpm::LabelSubsetFsmApp>(g, cfg, out);
    case 1: return gpm::mine_edge_app<gpm::CountSupportFsmApp>(g, cfg, out);
    default: return GPM_EINVAL;
  }
}

extern "C" int testapp_mine(int which, const gpm_graph* g, const gpm_config* cfg, gpm_result** out) {
  switch (which) {
    case 0: return gpm::mine_app<gpm::LabelCliqueApp>(g, cfg, out);
    case 1: return gpm::mine_app<gpm::StarApp>(g, cfg, out);
    case 2: return gpm::mine_app<gpm::CycleApp>(g, cfg, out);
    case 3: return gpm::mine_app<gpm::WedgeGrownMotifApp>(g, cfg, out);
    default: return GPM_EINVAL;
  }
}
