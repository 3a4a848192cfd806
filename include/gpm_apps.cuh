// gpm_apps.cuh — the reference's applications as App instantiations of the
// hook engine (include/gpm_engine.cuh), vertex mode.
//
//   CliqueApp  triangle_count / clique_find(k)   SPEC.md:414-431, Listing 3
//              (PAPER.md:967-976, :982-984): run on the degree-ordered DAG,
//              extend the last vertex only, to_add = u adjacent (directed) to
//              every earlier vertex, reduce = total count.
//   MotifApp   motif_count(k)                   SPEC.md:432-440, Listings 4+6
//              (PAPER.md:996-1010, :1159-1166): undirected, extend every
//              position, to_add = is_auto_canonical_vertex (+ source
//              position), reduce = connectivity code -> canonical pattern.
//
// The hooks are the whole definition of each app; kBuiltin lets the engine
// pick the library's staged kernels for them where their preconditions hold
// (csrc/vertex.cu builtin_level / builtin_roots).  FSM (edge mode) is in
// csrc/fsm.cu with its hooks in fsm_hooks.cuh.
#pragma once
#include "gpm_engine.cuh"

namespace gpm {

struct CliqueApp {
  static constexpr bool kDag = true;
  static constexpr int kReduce = engine::kReduceTotal;
  static constexpr bool kCodesAreMasks = false;
  static constexpr bool kFilter = false;
  static constexpr bool kParentMask = false;
  static constexpr bool kExtendLastOnly = true;  // Listing 3: toExtend = last vertex
  static constexpr bool kStageRoot = true;       // every candidate probes N+(emb[0])
  static constexpr bool kDescriptors = true;     // to_add reads lists only
  static constexpr int kBuiltin = engine::kBuiltinClique;
  static constexpr int kMaxK = 9;
  static void check(int k) {
    if (k < 3 || k > kMaxK) throw Error(GPM_EINVAL, "clique_find: k must be in [3,9]");
  }
  static int num_codes(int) { return 1; }
  template <int S>
  __device__ static bool to_extend(const engine::Emb<S>&, int pos) { return pos == S - 1; }
  // Listing 3: connected to every earlier vertex (on the DAG, directed emb[t] -> u)
  template <int S>
  __device__ static bool to_add(const engine::Emb<S>& e, int, u32 u) {
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

struct MotifApp {
  static constexpr bool kDag = false;
  static constexpr int kReduce = engine::kReduceCodes;
  static constexpr bool kCodesAreMasks = true;
  static constexpr bool kFilter = false;
  static constexpr bool kParentMask = true;
  static constexpr int kBuiltin = engine::kBuiltinMotif;
  static constexpr int kMaxK = 5;
  static void check(int k) {
    if (k < 3 || k > kMaxK) throw Error(GPM_EINVAL, "motif_count: k must be in {3,4,5}");
  }
  static int num_codes(int k) { return 1 << pat::npairs(k); }
  template <int S>
  __device__ static bool to_extend(const engine::Emb<S>&, int) { return true; }
  template <int S>
  __device__ static bool to_add(const engine::Emb<S>& e, int pos, u32 u) {
    return engine::is_auto_canonical_vertex(e, pos, u);
  }
  // Listing 6 generalised: the k-vertex connectivity code = the parent's
  // induced mask + the new vertex's adjacency (u ~ emb[pos] by construction,
  // not adjacent to any earlier position by to_add)
  template <int S>
  __device__ static u32 pattern_code(const engine::Emb<S>& e, int pos, u32 u) {
    u32 code = e.mask | engine::Emb<S>::pair_bit(pos, S, S + 1);
#pragma unroll
    for (int t = 1; t < S; ++t)
      if (t > pos && e.connected(t, u)) code |= engine::Emb<S>::pair_bit(t, S, S + 1);
    return code;
  }
  static bool to_prune(u32, u64, int) { return false; }
  static std::string code_text(u32, int) { return std::string(); }
};

}  // namespace gpm
