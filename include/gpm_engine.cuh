// gpm_engine.cuh — header-only extend-reduce-filter engine over user hooks
// (vertex-induced mode), sm_100a.
//
// This is Pangolin's programming interface (Listing 1;
// SPEC.md:326-331 AppCallbacks) as a compile-time contract: an App is a
// struct of __device__ / host hooks, and `gpm::engine::mine<App>` runs
// Alg. 1 with Alg. 2's extend as
// inspection-execution kernels instantiated for that App.  The GPU build of
// Pangolin compiled user hooks as __device__ functions the same way
// (PAPER.md:914-918).  The library's own apps (TC, k-CL, k-MC: gpm_apps.cuh)
// are instantiations of this engine; their staged kernels (edge chunks,
// sibling groups, on-chip staged motif sets) are specialisations the engine
// selects through App::kBuiltin under the same contract.  FSM's edge-mode
// hooks live in gpm_apps.cuh (FsmHooks) and drive csrc/fsm.cu.
//
// App contract (vertex mode):
//
//   struct MyApp {
//     static constexpr bool kDag = ...;        // run on the degree-ordered DAG
//                                              // (orient_dag, graph.hpp:121-132)
//     static constexpr int  kReduce = gpm::engine::kReduceTotal | kReduceCodes;
//     static constexpr bool kCodesAreMasks = ...;  // codes are connectivity masks
//                                              // over k positions -> canonical
//                                              // pattern text
//     static constexpr bool kFilter = ...;     // call to_prune each level
//     static constexpr bool kParentMask = ...; // engine computes e.mask (induced
//                                              // adjacency of the parent) for
//                                              // pattern_code on the last level
//     static void check(int k);                // host: validate k (throw gpm::Error)
//     static int  num_codes(int k);            // host: code bins (kReduceCodes)
//     template <int S> __device__ static bool to_extend(const Emb<S>&, int pos);
//     template <int S> __device__ static bool to_add(const Emb<S>&, int pos, u32 u);
//     template <int S> __device__ static u32  pattern_code(const Emb<S>&, int pos, u32 u);
//     static bool to_prune(u32 code, u64 support, int size);    // host (kFilter);
//                                              // size = vertices of the pattern
//     static std::string code_text(u32 code, int k);            // host (!kCodesAreMasks)
//   };
//
// Optional traits (defaults: the trait structs below): kMaxK (largest k the
// hooks support, <= 9), kExtendLastOnly (to_extend is
// pos == size-1: one candidate list per parent), kStageRoot (to_add probes
// emb[0]'s list for every candidate: it is staged in a warp hash set),
// kDescriptors (to_add only probes lists, never reads vertex ids: parents are
// described by list descriptors instead of idx chains), kBuiltin.
//
// Compile a user App with nvcc -gencode arch=compute_100a,code=sm_100a
// -I include -I paper_1911_06969_b200/csrc and link against libgpm.so
// (tests/apps/test_apps.cu is an example).
#pragma once
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "engine.hpp"
#include "pattern.cuh"

namespace gpm {

void scan_inplace(u64* data, u64 n, cudaStream_t s);

namespace engine {

enum : int { kReduceTotal = 0, kReduceCodes = 1 };
enum : int { kCount = 1, kWrite = 2, kFused = 3, kHist = 4 };
enum : int { kBuiltinNone = 0, kBuiltinClique = 1, kBuiltinMotif = 2 };

constexpr int kThreads = 256;
constexpr u64 kBatch = 2048;        // candidates per warp batch
constexpr u64 kBatchGrab = 4;       // batches per atomic grab
constexpr u32 kRootSlots = 1024;    // per-warp exact hash set of emb[0]'s list (4 KB)
constexpr u32 kRootMax = 512;       // longer root lists are probed by binary search

// ---------------------------------------------------------------- traits
template <class A, class = void>
struct extend_last_only : std::false_type {};
template <class A>
struct extend_last_only<A, std::void_t<decltype(A::kExtendLastOnly)>> : std::bool_constant<A::kExtendLastOnly> {};
template <class A, class = void>
struct stage_root : std::false_type {};
template <class A>
struct stage_root<A, std::void_t<decltype(A::kStageRoot)>> : std::bool_constant<A::kStageRoot> {};
template <class A, class = void>
struct descriptors : std::false_type {};
template <class A>
struct descriptors<A, std::void_t<decltype(A::kDescriptors)>> : std::bool_constant<A::kDescriptors> {};
template <class A, class = void>
struct max_k : std::integral_constant<int, kMaxLevels - 1> {};
template <class A>
struct max_k<A, std::void_t<decltype(A::kMaxK)>> : std::integral_constant<int, A::kMaxK> {};
template <class A, class = void>
struct builtin : std::integral_constant<int, kBuiltinNone> {};
template <class A>
struct builtin<A, std::void_t<decltype(A::kBuiltin)>> : std::integral_constant<int, A::kBuiltin> {};

// ---------------------------------------------------------------- levels
// SoA levels (Fig. 7, embedding_list.hpp:19-40): idx u32 (parent), vid u32.
struct VLevels {
  const u32* idx[kMaxLevels];
  const u32* vid[kMaxLevels];
};

// embedding_list.hpp:73-115 (vertex branch): walk idx links down to level 1.
template <int LEV>
__device__ __forceinline__ void reconstruct(const VLevels& L, u64 i, u32* emb) {
  u64 p = i;
#pragma unroll
  for (int k = LEV; k >= 2; --k) {
    emb[k] = ldg(L.vid[k - 1] + p);
    p = ldg(L.idx[k - 1] + p);
  }
  emb[0] = ldg(L.idx[0] + p);
  emb[1] = ldg(L.vid[0] + p);
}

// The parent embedding as the hooks see it: vertex ids, the neighbour list
// of every position (cached at parent load), the parent's induced adjacency
// mask (App::kParentMask) and, for kStageRoot apps, emb[0]'s list staged in
// a warp-shared hash set.
template <int S>
struct Emb {
  const u64* off;  // the graph (copies of kernel-parameter pointers)
  const u32* col;
  const u32* lab;
  u32 v[S];
  u64 beg[S];
  u32 deg[S];
  u32 mask;
  const u32* T;   // staged root list (nullptr: none)
  u32 sh, hmask;

  __device__ __forceinline__ int size() const { return S; }
  __device__ __forceinline__ u32 vertex(int t) const { return v[t]; }
  __device__ __forceinline__ u32 label(int t) const { return lab ? ldg(lab + v[t]) : 0u; }
  __device__ __forceinline__ u32 label_of(u32 u) const { return lab ? ldg(lab + u) : 0u; }
  __device__ __forceinline__ void bind(const DevGraph& g) {
    off = g.off;
    col = g.col;
    lab = g.lab;
    T = nullptr;
    mask = 0;
  }
  __device__ __forceinline__ u32 degree(int t) const { return deg[t]; }
  // u in the stored list of emb[t] (graph.hpp:93-104; on a DAG the directed
  // edge emb[t] -> u)
  __device__ __forceinline__ bool adj(int t, u32 u) const {
    if (t == 0 && T) return hs_has(T, sh, hmask, u);
    return contains_sorted(col + beg[t], deg[t], u);
  }
  // undirected connectivity of emb[t] and u, probing the shorter list
  // (SPEC.md:75): same answer as adj() on a symmetric CSR
  __device__ __forceinline__ bool connected(int t, u32 u) const {
    const u64 bu = ldg(off + u), eu = ldg(off + u + 1);
    if (deg[t] <= eu - bu) return contains_sorted(col + beg[t], deg[t], u);
    return contains_sorted(col + bu, (u32)(eu - bu), v[t]);
  }
  // bit of the position pair (a, b), a < b, in a k-position mask
  __device__ __forceinline__ static u32 pair_bit(int a, int b, int k) { return 1u << pat::pair_index(a, b, k); }
};

// is_auto_canonical_vertex + "emit u only from the first
// position adjacent to it" (SURVEY §7 hard part 1): the default to_add of
// vertex-induced apps.  u is a neighbour of emb[pos].
template <int S>
__device__ __forceinline__ bool is_auto_canonical_vertex(const Emb<S>& e, int pos, u32 u) {
  if (u <= e.v[0]) return false;
#pragma unroll
  for (int t = 1; t < S; ++t)
    if (t > pos && u <= e.v[t]) return false;
#pragma unroll
  for (int t = 0; t < S - 1; ++t)
    if (t < pos && e.connected(t, u)) return false;
  return true;
}

// ---------------------------------------------------------------- kernels
struct ExtendArgs {
  DevGraph g;
  VLevels L;
  const u64* Wp;    // exclusive work prefix over compacted parents, np+1 entries
  const u32* pidx;  // compacted parent -> level index
  const u64* desc[kMaxLevels];  // kDescriptors: per compacted parent, list begin | deg << 40 per position
  u64 np, W, B;
  u64 b_begin, b_end;
  u64 grab;
  unsigned long long* ctr;
  u64* cnt;          // COUNT: accepted per batch (index b - b_begin)
  const u64* boffs;  // WRITE: exclusive offsets per batch (absolute b)
  u64 out_base;
  u32* out_idx;
  u32* out_vid;
  u32* masks;        // COUNT writes / WRITE reads one ballot word per 32 candidates
  u64 mask_base;
  unsigned long long* hist;   // FUSED / HIST: per pattern code
  unsigned long long* total;  // FUSED total
  const u8* keep;             // kFilter: per code, survives to_prune
  int nbins;
  int k;
};

// Per-parent work: sum of deg(emb[pos]) over positions passing to_extend.
template <class App, int LEV>
__global__ void __launch_bounds__(kThreads) work_kernel(DevGraph g, VLevels L, u64 np, u64* __restrict__ W) {
  constexpr int S = LEV + 1;
  for (u64 p = blockIdx.x * (u64)blockDim.x + threadIdx.x; p < np; p += (u64)gridDim.x * blockDim.x) {
    Emb<S> e;
    e.bind(g);
    reconstruct<LEV>(L, p, e.v);
#pragma unroll
    for (int t = 0; t < S; ++t) {
      e.beg[t] = ldg(g.off + e.v[t]);
      e.deg[t] = (u32)(ldg(g.off + e.v[t] + 1) - e.beg[t]);
    }
    u64 w = 0;
    if constexpr (extend_last_only<App>::value) {
      w = e.deg[S - 1];
    } else {
#pragma unroll
      for (int t = 0; t < S; ++t)
        if (App::to_extend(e, t)) w += e.deg[t];
    }
    W[p] = w;
  }
}

// Per compacted parent: list descriptors of every position (kDescriptors).
template <int LEV>
__global__ void desc_kernel(DevGraph g, VLevels L, const u32* __restrict__ pidx, u64 nz, ExtendArgs a) {
  constexpr int S = LEV + 1;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nz; i += (u64)gridDim.x * blockDim.x) {
    u32 emb[S];
    reconstruct<LEV>(L, pidx[i], emb);
#pragma unroll
    for (int t = 0; t < S; ++t) {
      const u64 b = ldg(g.off + emb[t]), e = ldg(g.off + emb[t] + 1);
      const_cast<u64*>(a.desc[t])[i] = b | ((e - b) << 40);
    }
  }
}

// Per-lane cursor over the candidate space: caches the parent that owns
// candidate j (compacted parent index space).
template <class App, int LEV, bool PMASK>
struct Cursor {
  static constexpr int S = LEV + 1;
  u64 cp = ~0ull, cWb = 0, cWe = 0;
  u32 parent = 0;
  Emb<S> e;
  u32 edeg[S];  // candidate-space share of each position (0 unless to_extend)

  __device__ __forceinline__ void load(const ExtendArgs& a, u64 p) {
    if (p == cp) return;
    cp = p;
    cWb = ldg(a.Wp + p);
    cWe = ldg(a.Wp + p + 1);
    parent = ldg(a.pidx + p);
    const DevGraph& g = a.g;
    if (descriptors<App>::value && a.desc[0]) {  // independent loads, no idx chain
#pragma unroll
      for (int t = 0; t < S; ++t) {
        const u64 q = ldg(a.desc[t] + p);
        e.beg[t] = q & ((u64(1) << 40) - 1);
        e.deg[t] = (u32)(q >> 40);
        e.v[t] = 0xffffffffu;  // kDescriptors apps never read ids
      }
    } else {
      reconstruct<LEV>(a.L, parent, e.v);
#pragma unroll
      for (int t = 0; t < S; ++t) {
        e.beg[t] = ldg(g.off + e.v[t]);
        e.deg[t] = (u32)(ldg(g.off + e.v[t] + 1) - e.beg[t]);
      }
    }
    if (PMASK) {
      e.mask = Emb<S>::pair_bit(0, 1, S + 1);
#pragma unroll
      for (int bb = 2; bb < S; ++bb)
#pragma unroll
        for (int aa = 0; aa < bb; ++aa)
          if (e.connected(aa, e.v[bb])) e.mask |= Emb<S>::pair_bit(aa, bb, S + 1);
    }
    if constexpr (extend_last_only<App>::value) {
#pragma unroll
      for (int t = 0; t < S - 1; ++t) edeg[t] = 0;
      edeg[S - 1] = e.deg[S - 1];
    } else {
#pragma unroll
      for (int t = 0; t < S; ++t) edeg[t] = App::to_extend(e, t) ? e.deg[t] : 0u;
    }
  }

  __device__ __forceinline__ void locate(const ExtendArgs& a, u64 j, u64 pa, u64 pb) {
    if (cp != ~0ull && j < cWe && j >= cWb) return;
    const u64 lo = (cp == ~0ull || j < cWb) ? pa : cp + 1;
    load(a, upper_bound_prev(a.Wp, lo, pb + 1, j));
  }

  // candidate vertex u for j (after load/locate); pos = source position
  __device__ __forceinline__ u32 candidate(const DevGraph& g, u64 j, int& pos) const {
    u32 local = (u32)(j - cWb);
    if constexpr (extend_last_only<App>::value) {
      pos = S - 1;
      return ldg(g.col + e.beg[S - 1] + local);
    }
    pos = 0;
#pragma unroll
    for (int t = 0; t < S - 1; ++t)
      if (pos == t && local >= edeg[t]) {
        local -= edeg[t];
        pos = t + 1;
      }
    return ldg(g.col + e.beg[pos] + local);
  }
};

template <class App, int LEV, int MODE>
__global__ void __launch_bounds__(kThreads, 2) extend_kernel(ExtendArgs a) {
  constexpr int S = LEV + 1;  // parent embedding size
  constexpr int kWords = (int)(kBatch / 32);
  constexpr bool kStage = stage_root<App>::value;
  constexpr bool kCodes = (MODE == kFused && App::kReduce == kReduceCodes) || MODE == kHist;
  constexpr bool kKeep = App::kFilter && (MODE == kCount || MODE == kWrite);
  extern __shared__ unsigned long long shist[];
  __shared__ __align__(16) u32 s_hash[kStage ? kThreads / 32 : 1][kStage ? kRootSlots : 4];
  const int lane = threadIdx.x & 31;
  u32* filt = s_hash[kStage ? (threadIdx.x >> 5) : 0];
  u32 fsh = 0, fmask = 0;
  const DevGraph& g = a.g;
  if (kCodes) {
    for (int i = threadIdx.x; i < a.nbins; i += blockDim.x) shist[i] = 0;
    __syncthreads();
  }
  unsigned long long wtotal = 0;

  u64 bgrab = 0, bleft = 0;
  for (;;) {
    if (bleft == 0) {
      u64 b_ = 0;
      if (lane == 0) b_ = atomicAdd(a.ctr, (unsigned long long)a.grab) + a.b_begin;
      bgrab = __shfl_sync(0xffffffffu, b_, 0);
      bleft = a.grab;
    }
    const u64 b = bgrab++;
    --bleft;
    if (b >= a.b_end) break;
    const u64 j0 = b * a.B;
    const u64 j1 = min(a.W, j0 + a.B);
    u64 wpos = 0;
    if (MODE == kWrite) {
      wpos = ldg(a.boffs + b);
      if (ldg(a.boffs + b + 1) == wpos) continue;  // batch has no children
      wpos -= a.out_base;
    }
    u64 pr = 0;
    if (lane < 2) pr = upper_bound_prev(a.Wp, 0, a.np + 1, lane == 0 ? j0 : j1 - 1);
    const u64 pa = __shfl_sync(0xffffffffu, pr, 0);
    const u64 pb = __shfl_sync(0xffffffffu, pr, 1);
    Cursor<App, LEV, App::kParentMask && (MODE == kFused || MODE == kHist || kKeep)> cur;
    cur.e.bind(g);

    if (MODE == kWrite && a.masks) {
      // execution from the inspection's ballot masks: only accepted lanes work
      const u32* mw = a.masks + (b - a.mask_base) * kWords;
      const int nwords = (int)((j1 - j0 + 31) / 32);
      for (int w0 = 0; w0 < nwords; w0 += 32) {
        const u32 mine = (w0 + lane < nwords) ? ldg(mw + w0 + lane) : 0u;
        const int lim = min(32, nwords - w0);
        for (int t = 0; t < lim; ++t) {
          const u32 m = __shfl_sync(0xffffffffu, mine, t);
          if (!m) continue;
          if (m >> lane & 1u) {
            const u64 j = j0 + (u64)(w0 + t) * 32 + lane;
            cur.locate(a, j, pa, pb);
            int pos;
            const u32 u = cur.candidate(g, j, pos);
            const u64 o = wpos + __popc(m & lanemask_lt());
            a.out_idx[o] = cur.parent;
            a.out_vid[o] = u;
          }
          wpos += __popc(m);
        }
      }
      continue;
    }

    u32 c = 0;
    u32 myword = 0;
    int it = 0;
    u64 fkey = ~0ull;  // descriptor of the root list held in the hash set
    bool fok = false;
    u64 P0 = pa;  // compacted parent owning candidate jb
    for (u64 jb = j0; jb < j1; jb += 32, ++it) {
      const u64 j = jb + lane;
      // lane -> parent: every compacted parent owns >= 1 candidate, so the 32
      // parents after P0 cover this step; one OR-reduction of their start
      // offsets gives each lane its parent (no per-lane search).
      const u64 x = (P0 + 1 + lane <= a.np) ? ldg(a.Wp + P0 + 1 + lane) : ~0ull;
      const u32 bit = (x - jb < 32) ? (1u << (u32)(x - jb)) : 0u;
      const u32 starts = __reduce_or_sync(0xffffffffu, bit);
      const u64 myp = P0 + __popc(starts & (lanemask_lt() | (1u << lane)));
      P0 += __popc(starts);
      bool ok = false;
      u32 u = 0, code = 0;
      if (j < j1) cur.load(a, myp);
      if (kStage) {
        // warp-shared exact hash set of emb[0]'s list (shared by all parents
        // of one root): the emb[0] probe costs shared-memory loads instead
        // of a global binary search
        const u32 act = __ballot_sync(0xffffffffu, j < j1);
        const int leader = __ffs(act) - 1;
        const u64 key = __shfl_sync(0xffffffffu, cur.e.beg[0] | ((u64)cur.e.deg[0] << 40), leader);
        if (key != fkey) {
          fkey = key;
          const u32 d = (u32)(key >> 40);
          const u64 qb = key & ((u64(1) << 40) - 1);
          fok = d <= kRootMax;
          if (fok) hs_stage_warp(filt, g.col, qb, d, kRootSlots, fsh, fmask);
        }
        const bool mine = fok && (cur.e.beg[0] | ((u64)cur.e.deg[0] << 40)) == fkey;
        cur.e.T = mine ? filt : nullptr;
        cur.e.sh = fsh;
        cur.e.hmask = fmask;
      }
      if (j < j1) {
        int pos;
        u = cur.candidate(g, j, pos);
        bool inemb = false;
        // SPEC.md:392 (u not in emb).  Descriptor apps on a DAG extend the
        // last position's out-list: every earlier vertex precedes u in the
        // orientation order, so u cannot be in the embedding.
        if (!(descriptors<App>::value && a.desc[0])) {
#pragma unroll
          for (int t = 0; t < S; ++t) inemb |= (cur.e.v[t] == u);
        }
        if (!inemb) {
          ok = App::to_add(cur.e, pos, u);
          if (ok && (kCodes || kKeep)) code = App::pattern_code(cur.e, pos, u);
          if (kKeep && ok) ok = a.keep[code] != 0;
        }
      }
      const u32 mask = __ballot_sync(0xffffffffu, ok);
      if (MODE == kCount) {
        c += __popc(mask);
        if (a.masks) {
          if ((it & 31) == lane) myword = mask;
          if ((it & 31) == 31) a.masks[(b - a.mask_base) * kWords + (it - 31) + lane] = myword;
        }
      } else if (MODE == kWrite) {
        if (ok) {
          const u64 o = wpos + __popc(mask & lanemask_lt());
          a.out_idx[o] = cur.parent;
          a.out_vid[o] = u;
        }
        wpos += __popc(mask);
      } else if (kCodes) {
        if (mask) {
          const u32 key = ok ? code : 0xffffffffu;
          const u32 peers = __match_any_sync(0xffffffffu, key);
          if (ok && lane == __ffs(peers) - 1) atomicAdd(&shist[code], (unsigned long long)__popc(peers));
        }
      } else {
        wtotal += __popc(mask);
      }
    }
    if (MODE == kCount) {
      if (a.masks && (it & 31) != 0 && lane < (it & 31)) a.masks[(b - a.mask_base) * kWords + (it & ~31) + lane] = myword;
      if (lane == 0) a.cnt[b - a.b_begin] = c;
    }
  }
  if (kCodes) {
    __syncthreads();
    for (int i = threadIdx.x; i < a.nbins; i += blockDim.x)
      if (shist[i]) atomicAdd(a.hist + i, shist[i]);
  } else if (MODE == kFused && lane == 0 && wtotal) {
    atomicAdd(a.total, wtotal);
  }
}

struct NonZeroW {
  const u64* w;
  __device__ __forceinline__ bool operator()(const u32& i) const { return w[i] != 0; }
};

template <int = 0>
__global__ void gather_kernel(const u64* __restrict__ w, const u32* __restrict__ pidx, u64 nz,
                                     u64* __restrict__ Wp) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nz; i += (u64)gridDim.x * blockDim.x)
    Wp[i] = w[pidx[i]];
}

// Canonical code of every connectivity mask over k positions (reduce step 2:
// canonicalize once per quick pattern).
template <int = 0>
__global__ void canon_masks_kernel(int k, u64* __restrict__ keys) {
  const int nm = 1 << pat::npairs(k);
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < nm; m += gridDim.x * blockDim.x) {
    u32 lab[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    keys[m] = pat::canonicalize(k, lab, (u32)m, 0, nullptr);
  }
}

// Listing: final-level entries [i0, i0 + n) -> rows of LEV + 1 vertex ids
// (insertion order; consecutive threads write consecutive rows).
template <int LEV>
__global__ void list_rows_kernel(VLevels L, u64 i0, u64 n, u32* __restrict__ out) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    u32 emb[LEV + 1];
    reconstruct<LEV>(L, i0 + i, emb);
#pragma unroll
    for (int t = 0; t <= LEV; ++t) out[i * (LEV + 1) + t] = emb[t];
  }
}

// ---------------------------------------------------------------- host side
struct Ctx {
  const gpm_graph* G;
  DevGraph g;
  int k;
  cudaStream_t s;
  Timeline* tl;
  Stats* st;
  int sms;
  u64 cap_entries;
  u64 mask_budget;
  unsigned long long* d_total;
  unsigned long long* d_hist;
  unsigned long long* d_ctr;
  int nbins;
  bool siblings_complete;  // every child of each level parent is in this chunk
  bool generic_only;       // GPM_GENERIC_*: bypass the builtin specialisations
  gpm_list_fn list_fn;     // listing mode: last level materialised + streamed
  void* list_ctx;
  u64 listed;
  const void* app_state;   // hooks' host state (unused by the builtin apps)
};

// Builtin specialisations (csrc/vertex.cu, csrc/mc_staged.cu): return true
// when they processed the level / root slice.
bool builtin_level(Ctx& c, int kind, int lev, const VLevels& L, u64 np);
bool builtin_roots(Ctx& c, int kind, const VLevels& L, const u32* l1_src, const u64* l1_start, u64 slo, u64 shi);
// k-CL counts on per-root local rows apply (csrc/clique_local.cu): the level-1
// v0 array is then not needed.
bool cf_local_applicable(const gpm_graph& G, int k, bool listing);

// Streams a materialised final level (n entries at level LEV) to the host sink
// through two device staging buffers and two pinned host buffers: the rows of
// piece p are built and copied while the sink consumes piece p - 1.
template <int LEV>
void emit_rows(Ctx& c, const VLevels& L, u64 n) {
  constexpr int K = LEV + 1;
  const u64 R = std::min<u64>(n, u64(1) << 20);
  DBuf<u32> d0(R * K, c.s), d1(R * K, c.s);
  u32* dv[2] = {d0.get(), d1.get()};
  u32* hv[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  u64 pn[2] = {0, 0};
  auto cleanup = [&] {
    for (int b = 0; b < 2; ++b) {
      if (ev[b]) cudaEventDestroy(ev[b]);
      if (hv[b]) cudaFreeHost(hv[b]);
    }
  };
  try {
    for (int b = 0; b < 2; ++b) {
      GPM_CUDA(cudaMallocHost(reinterpret_cast<void**>(&hv[b]), sizeof(u32) * R * K));
      GPM_CUDA(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
    }
    auto deliver = [&](int b) {
      GPM_CUDA(cudaEventSynchronize(ev[b]));
      if (c.list_fn(c.list_ctx, hv[b], pn[b], K) != 0) throw Error(GPM_EINVAL, "list_fn aborted the job");
      c.listed += pn[b];
    };
    u64 piece = 0;
    for (u64 i0 = 0; i0 < n; i0 += R, ++piece) {
      const int b = (int)(piece & 1);
      if (piece >= 2) deliver(b);  // buffer b still holds piece - 2
      pn[b] = std::min<u64>(R, n - i0);
      list_rows_kernel<LEV><<<(unsigned)std::min<u64>((pn[b] + 255) / 256, (u64)c.sms * 16), 256, 0, c.s>>>(
          L, i0, pn[b], dv[b]);
      GPM_CUDA(cudaGetLastError());
      ++c.tl->launches;
      GPM_CUDA(cudaMemcpyAsync(hv[b], dv[b], sizeof(u32) * pn[b] * K, cudaMemcpyDeviceToHost, c.s));
      GPM_CUDA(cudaEventRecord(ev[b], c.s));
    }
    if (piece >= 2) deliver((int)(piece & 1));
    if (piece >= 1) deliver((int)((piece - 1) & 1));
  } catch (...) {
    cudaStreamSynchronize(c.s);
    cleanup();
    throw;
  }
  cleanup();
}

template <class App, int LEV, int MODE>
void launch_extend(Ctx& c, ExtendArgs& a, const char* what, double bytes) {
  auto kern = extend_kernel<App, LEV, MODE>;
  constexpr bool kCodes = (MODE == kFused && App::kReduce == kReduceCodes) || MODE == kHist;
  const size_t smem = kCodes ? sizeof(unsigned long long) * (size_t)a.nbins : 0;
  static std::atomic<int> occ_slot{0};  // per instantiation
  const int occ = cached_occupancy(occ_slot, [&] {
    if (smem > 48 * 1024)
      GPM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int o = 0;
    GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kThreads, smem));
    return o;
  });
  const u64 nb = a.b_end - a.b_begin;
  u64 blocks = std::min<u64>((u64)c.sms * occ, (nb * 32 + kThreads - 1) / kThreads);
  blocks = std::max<u64>(1, blocks);
  a.grab = std::max<u64>(1, std::min<u64>(kBatchGrab, nb / (blocks * (kThreads / 32) * 64)));
  GPM_CUDA(cudaMemsetAsync(c.d_ctr, 0, sizeof(unsigned long long), c.s));
  a.ctr = c.d_ctr;
  c.st->paths |= GPM_PATH_GENERIC;
  size_t ev = c.tl->begin(std::string(what) + "_L" + std::to_string(LEV), bytes);
  kern<<<(unsigned)blocks, kThreads, smem, c.s>>>(a);
  GPM_CUDA(cudaGetLastError());
  c.tl->end(ev);
  ++c.tl->launches;
}

template <class App, int LEV>
void process(Ctx& c, VLevels L, u64 np);

template <class App>
void process_dispatch(Ctx& c, int lev, const VLevels& L, u64 np) {
  switch (lev) {
#define GPM_ENGINE_LEV(X)                                   \
  case X:                                                   \
    if constexpr (X + 2 <= max_k<App>::value) {             \
      process<App, X>(c, L, np);                            \
      return;                                               \
    }                                                       \
    break;
    GPM_ENGINE_LEV(1) GPM_ENGINE_LEV(2) GPM_ENGINE_LEV(3) GPM_ENGINE_LEV(4) GPM_ENGINE_LEV(5) GPM_ENGINE_LEV(6)
    GPM_ENGINE_LEV(7)
#undef GPM_ENGINE_LEV
    default:
      break;
  }
  throw Error(GPM_EINVAL, "unsupported level " + std::to_string(lev));
}

template <int LEV>
void emit_dispatch(Ctx& c, const VLevels& L, u64 n) {
  if constexpr (LEV + 1 < kMaxLevels) emit_rows<LEV>(c, L, n);
  else throw Error(GPM_EINVAL, "listing: level out of range");
}

// One level of Alg. 1 for parents L (np entries at level LEV): work pass,
// compaction + scan -> candidate space, then the fused last extension, or
// inspection (COUNT) -> scan -> planner chunks -> execution (WRITE) and
// recursion into the next level.  kFilter apps reduce every level first
// (HIST) and drop children whose code to_prune rejects.
template <class App, int LEV>
void process(Ctx& c, VLevels L, u64 np) {
  constexpr int S = LEV + 1;
  const bool last = (LEV == c.k - 2);
  Stats& st = *c.st;
  if (np == 0) return;
  if constexpr (builtin<App>::value != kBuiltinNone) {
    if (!c.generic_only && builtin_level(c, builtin<App>::value, LEV, L, np)) return;
  }
  // ---- work pass, compaction of parents with work, scan: candidate space
  u64 nz = 0;
  DBuf<u32> pidx;
  DBuf<u64> Wp;
  u64 nvs = 0;  // extended positions summed over parents (B_alg offsets term)
  {
    DBuf<u64> w(np, c.s);
    unsigned blocks = (unsigned)std::min<u64>((np + kThreads - 1) / kThreads, (u64)c.sms * 16);
    work_kernel<App, LEV><<<std::max(1u, blocks), kThreads, 0, c.s>>>(c.g, L, np, w.get());
    GPM_CUDA(cudaGetLastError());
    ++c.tl->launches;
    pidx.alloc(np, c.s);
    DBuf<u64> nsel(1, c.s);
    size_t tmp = 0;
    thrust::counting_iterator<u32> it(0);
    GPM_CUDA(cub::DeviceSelect::If(nullptr, tmp, it, pidx.get(), nsel.get(), (int64_t)np, NonZeroW{w.get()}, c.s));
    DBuf<u8> t(tmp, c.s);
    GPM_CUDA(cub::DeviceSelect::If(t.get(), tmp, it, pidx.get(), nsel.get(), (int64_t)np, NonZeroW{w.get()}, c.s));
    GPM_CUDA(cudaMemcpyAsync(&nz, nsel.get(), sizeof(u64), cudaMemcpyDeviceToHost, c.s));
    GPM_CUDA(cudaStreamSynchronize(c.s));
    Wp.alloc(nz + 1, c.s);
    GPM_CUDA(cudaMemsetAsync(Wp.get() + nz, 0, sizeof(u64), c.s));
    if (nz) {
      gather_kernel<><<<(unsigned)std::min<u64>((nz + 255) / 256, 1u << 20), 256, 0, c.s>>>(w.get(), pidx.get(), nz,
                                                                                          Wp.get());
      GPM_CUDA(cudaGetLastError());
      c.tl->launches += 2;
    }
  }
  scan_inplace(Wp.get(), nz + 1, c.s);
  u64 W = 0;
  GPM_CUDA(cudaMemcpyAsync(&W, Wp.get() + nz, sizeof(u64), cudaMemcpyDeviceToHost, c.s));
  GPM_CUDA(cudaStreamSynchronize(c.s));
  st.candidates[LEV] += W;
  nvs = extend_last_only<App>::value ? np : (u64)S * np;  // 16 B per extended position
  const double bytes_in = 8.0 * LEV * np + 16.0 * nvs + 4.0 * W;
  st.balg += bytes_in;
  if (W == 0) return;
  const u64 nb = (W + kBatch - 1) / kBatch;
  ExtendArgs a{};
  a.g = c.g;
  a.L = L;
  a.Wp = Wp.get();
  a.pidx = pidx.get();
  a.np = nz;
  a.W = W;
  a.nbins = c.nbins;
  DBuf<u64> desc;
  if (descriptors<App>::value && c.g.oriented && c.G->m < (u64(1) << 40)) {
    desc.alloc(nz * S, c.s);
    for (int t = 0; t < S; ++t) a.desc[t] = desc.get() + (u64)t * nz;
    desc_kernel<LEV><<<(unsigned)std::min<u64>((nz + 255) / 256, 1u << 20), 256, 0, c.s>>>(c.g, L, pidx.get(), nz, a);
    GPM_CUDA(cudaGetLastError());
    ++c.tl->launches;
  }
  a.B = kBatch;
  a.b_begin = 0;
  a.b_end = nb;
  a.k = c.k;
  if (last && !c.list_fn) {
    a.hist = c.d_hist;
    a.total = c.d_total;
    launch_extend<App, LEV, kFused>(c, a, "extend_fused", bytes_in);
    return;
  }
  // ---- filter (kFilter): reduce this level's children by code, to_prune
  DBuf<u8> keep;
  if constexpr (App::kFilter) {
    DBuf<unsigned long long> h(c.nbins, c.s);
    GPM_CUDA(cudaMemsetAsync(h.get(), 0, sizeof(unsigned long long) * c.nbins, c.s));
    ExtendArgs r = a;
    r.hist = h.get();
    launch_extend<App, LEV, kHist>(c, r, "extend_reduce", bytes_in);
    std::vector<unsigned long long> hh(c.nbins);
    GPM_CUDA(cudaMemcpyAsync(hh.data(), h.get(), sizeof(unsigned long long) * c.nbins, cudaMemcpyDeviceToHost, c.s));
    GPM_CUDA(cudaStreamSynchronize(c.s));
    std::vector<u8> kh(c.nbins, 0);
    // to_prune(code, support, size): size = vertices of the reduced embeddings
    for (int i = 0; i < c.nbins; ++i) kh[i] = (hh[i] && !App::to_prune((u32)i, hh[i], LEV + 2)) ? 1 : 0;
    keep.alloc(c.nbins, c.s);
    GPM_CUDA(cudaMemcpyAsync(keep.get(), kh.data(), c.nbins, cudaMemcpyHostToDevice, c.s));
    a.keep = keep.get();
  }
  // ---- inspection: children per batch
  DBuf<u64> cnt(nb + 1, c.s);
  GPM_CUDA(cudaMemsetAsync(cnt.get() + nb, 0, sizeof(u64), c.s));
  a.cnt = cnt.get();
  // keep the inspection's ballot masks (1 bit per candidate) when affordable,
  // so the execution pass touches accepted candidates only
  DBuf<u32> masks;
  const u64 mask_words = nb * (kBatch / 32);
  if (mask_words * 4 <= c.mask_budget) {
    masks.alloc(mask_words, c.s);
    a.masks = masks.get();
    a.mask_base = 0;
  }
  launch_extend<App, LEV, kCount>(c, a, "extend_count", bytes_in);
  scan_inplace(cnt.get(), nb + 1, c.s);
  u64 T = 0;
  GPM_CUDA(cudaMemcpyAsync(&T, cnt.get() + nb, sizeof(u64), cudaMemcpyDeviceToHost, c.s));
  GPM_CUDA(cudaStreamSynchronize(c.s));
  if (!last) st.level_sizes[LEV] += T;  // a listed last level is counted through d_total
  st.balg += 8.0 * T;
  if (T == 0) return;
  // ---- planner: batch ranges whose children fit the budget
  std::vector<std::pair<u64, u64>> chunks;
  if (T <= c.cap_entries) {
    chunks.emplace_back(0, nb);
  } else {
    std::vector<u64> h(nb + 1);
    GPM_CUDA(cudaMemcpyAsync(h.data(), cnt.get(), sizeof(u64) * (nb + 1), cudaMemcpyDeviceToHost, c.s));
    GPM_CUDA(cudaStreamSynchronize(c.s));
    u64 b0 = 0;
    while (b0 < nb) {
      u64 key = h[b0] + c.cap_entries;
      u64 b1 = (u64)(std::upper_bound(h.begin() + b0 + 1, h.end(), key) - h.begin()) - 1;
      if (b1 <= b0) b1 = b0 + 1;
      chunks.emplace_back(b0, b1);
      b0 = b1;
    }
  }
  st.chunks += chunks.size() - 1;
  for (auto [b0, b1] : chunks) {
    u64 base = 0, end = 0;
    GPM_CUDA(cudaMemcpyAsync(&base, cnt.get() + b0, sizeof(u64), cudaMemcpyDeviceToHost, c.s));
    GPM_CUDA(cudaMemcpyAsync(&end, cnt.get() + b1, sizeof(u64), cudaMemcpyDeviceToHost, c.s));
    GPM_CUDA(cudaStreamSynchronize(c.s));
    const u64 Tc = end - base;
    if (Tc == 0) continue;
    DBuf<u32> oi(Tc, c.s), ov(Tc, c.s);
    ExtendArgs w = a;
    w.b_begin = b0;
    w.b_end = b1;
    w.boffs = cnt.get();
    w.out_base = base;
    w.out_idx = oi.get();
    w.out_vid = ov.get();
    // execution from masks reads 1 bit per candidate + the accepted candidates' parents
    const double frac = (double)(b1 - b0) / (double)nb;
    const double wbytes = a.masks ? (double)(b1 - b0) * kBatch / 8.0 + 24.0 * Tc : bytes_in * frac;
    launch_extend<App, LEV, kWrite>(c, w, "extend_write", wbytes + 8.0 * Tc);
    VLevels nl = L;
    nl.idx[LEV] = oi.get();
    nl.vid[LEV] = ov.get();
    c.siblings_complete = chunks.size() == 1;  // planner chunks may split a parent's children
    if (last) emit_dispatch<LEV + 1>(c, nl, Tc);
    else if constexpr (LEV + 2 < kMaxLevels) process_dispatch<App>(c, LEV + 1, nl, Tc);
  }
}

// mine(g, cfg) (Alg. 1) for a vertex-mode
// App: orientation (kDag), level 1 (embedding_list.hpp:178-192), the root
// split / stealing tail, the level loop, the count exchange and
// the reduce into result patterns.
template <class App>
void mine(const gpm_graph& G0, const gpm_config& cfg, cudaStream_t s, gpm_result& res, Stats& st, Timeline& tl,
          const void* app_state = nullptr) {
  int k = cfg.k;
  if (cfg.app == GPM_APP_TC) k = 3;  // triangle_count == clique_find(3)
  App::check(k);
  res.k = k;
  std::unique_ptr<gpm_graph> dag;
  const gpm_graph* G = &G0;
  if (App::kDag && !G0.oriented && !cfg.no_orient) {
    dag = std::make_unique<gpm_graph>();
    dag->device = G0.device;
    dag->stream = s;            // orient on the engine stream; freed on it too
    dag->owns_stream = false;
    orient_on_device(G0, *dag);
    tl.launches += 4;
    G = dag.get();
  }
  if (!App::kDag && G0.oriented) throw Error(GPM_EINVAL, "this app needs an undirected graph");

  const int levels = k - 1;
  st.ensure(levels);
  DBuf<u32> l1i, l1v;
  DBuf<u64> l1s;
  u64 n1 = 0;
  const u32* l1vid = nullptr;
  const int world0 = std::max(1, cfg.world);
  const bool lazy_l1 = builtin<App>::value == kBuiltinClique && world0 == 1 && G->oriented &&
                       !std::getenv("GPM_GENERIC_L1") && cf_local_applicable(*G, k, cfg.list_fn != nullptr);
  build_level1(*G, l1i, l1v, n1, s, tl, &l1vid, &l1s, !lazy_l1);
  if (!l1vid) l1vid = l1v.get();
  // root units of this rank: an explicit slice, the degree-weighted static
  // split, or (steal_ctrs set) the split's head + a device-side stealing tail
  const int world = std::max(1, cfg.world);
  const bool steal = world > 1 && cfg.steal_ctrs && cfg.root_hi == 0;
  u64 lo = 0, hi = n1;
  std::vector<u64> bounds;
  if (cfg.root_hi > 0) {
    lo = std::min(cfg.root_lo, n1);
    hi = std::min(cfg.root_hi, n1);
    if (hi < lo) hi = lo;
  } else if (world > 1) {
    root_split_bounds(*G, l1i.get(), l1vid, n1, App::kDag ? GPM_APP_CF : GPM_APP_MC, world, bounds, s, tl);
    lo = bounds[cfg.rank];
    hi = bounds[cfg.rank + 1];
  }

  Ctx c{};
  c.G = G;
  c.g = G->view();
  c.k = k;
  c.s = s;
  c.tl = &tl;
  c.st = &st;
  c.sms = sm_count();
  c.list_fn = cfg.list_fn;
  c.list_ctx = cfg.list_ctx;
  c.listed = 0;
  c.app_state = app_state;
  const size_t freeb = device_free_bytes();
  const u64 budget = cfg.mem_budget ? cfg.mem_budget : (u64)(0.6 * (double)freeb);
  const int mat_levels = std::max(1, k - 3);
  // bytes per materialised entry: 8 B in its level (idx + vid) for every level
  // held at once, plus the next level's per-parent temporaries while it is the
  // parent level (work u64, compacted index u32, offsets u64, k-1 u64
  // descriptors): a chunk of cap_entries parents always fits the budget
  const u64 per_entry = 8 * (u64)mat_levels + 20 + 8 * (u64)std::max(1, k - 1);
  c.cap_entries = std::max<u64>(kBatch, std::min<u64>((u64(1) << 32) - 1, budget / per_entry));
  c.mask_budget = budget / 4;
  c.nbins = App::kReduce == kReduceCodes ? App::num_codes(k) : 1;
  if (App::kReduce == kReduceCodes && App::kFilter && c.nbins <= 0) throw Error(GPM_EINVAL, "num_codes must be > 0");
  DBuf<unsigned long long> d_total(1, s), d_hist(c.nbins, s), d_ctr(1, s);
  GPM_CUDA(cudaMemsetAsync(d_total.get(), 0, sizeof(unsigned long long), s));
  GPM_CUDA(cudaMemsetAsync(d_hist.get(), 0, sizeof(unsigned long long) * c.nbins, s));
  c.d_total = d_total.get();
  c.d_hist = d_hist.get();
  c.d_ctr = d_ctr.get();

  u64 nroot = 0;  // level-1 entries processed by this rank
  auto run_slice = [&](u64 slo, u64 shi) {
    const u64 np = shi - slo;
    if (np >= (u64(1) << 32)) throw Error(GPM_EINVAL, "level 1 exceeds 2^32 entries");
    nroot += np;
    st.level_sizes[0] += np;
    if (k == 2 || np == 0) return;
    VLevels L{};
    L.idx[0] = l1i.get() + slo;
    L.vid[0] = l1vid + slo;
    if constexpr (builtin<App>::value != kBuiltinNone) {
      if (!c.generic_only && builtin_roots(c, builtin<App>::value, L, l1i.get(), l1s.get(), slo, shi)) return;
    }
    process_dispatch<App>(c, 1, L, np);
  };
  if (!steal) {
    run_slice(lo, hi);
  } else {
    // head: the first (1 - tail) of the own static range, no contention;
    // tails: every rank's remainder, claimed in chunks through the shared
    // counters (own tail first, then the others'), so a rank that finishes
    // early drains the slow ranks' work.
    const double tail = 0.25;
    std::vector<u64> tlo(world), thi(world);
    u64 tsum = 0;
    for (int r = 0; r < world; ++r) {
      const u64 len = bounds[r + 1] - bounds[r];
      tlo[r] = bounds[r] + (u64)((1.0 - tail) * (double)len);
      thi[r] = bounds[r + 1];
      tsum += thi[r] - tlo[r];
    }
    run_slice(lo, tlo[cfg.rank]);
    // k-CL on local rows pays a fixed ~50 us per slice (prep, launches, one
    // host sync): coarser tail chunks there
    const bool local_rows = builtin<App>::value == kBuiltinClique && cf_local_applicable(*G, k, c.list_fn != nullptr);
    const u64 chunk = cfg.steal_chunk ? cfg.steal_chunk
                                      : std::max<u64>(local_rows ? 65536 : 1024, tsum / ((u64)world * (local_rows ? 4 : 32)));
    DBuf<u64> d_t(2 * world, s), d_out(2, s);
    GPM_CUDA(cudaMemcpyAsync(d_t.get(), tlo.data(), sizeof(u64) * world, cudaMemcpyHostToDevice, s));
    GPM_CUDA(cudaMemcpyAsync(d_t.get() + world, thi.data(), sizeof(u64) * world, cudaMemcpyHostToDevice, s));
    for (;;) {
      u64 clo = 0, chi = 0;
      steal_grab(reinterpret_cast<unsigned long long*>(cfg.steal_ctrs), d_t.get(), d_t.get() + world, world,
                 cfg.rank, chunk, d_out.get(), clo, chi, s);
      ++tl.launches;
      if (clo >= chi) break;
      ++st.chunks;
      run_slice(clo, chi);
    }
  }
  if (k == 2) res.total = nroot;

  if (c.list_fn && k > 2) {  // listed rows play the fused kernel's count (exchanged below)
    const unsigned long long v = c.listed;
    GPM_CUDA(cudaMemcpyAsync(d_total.get(), &v, sizeof v, cudaMemcpyHostToDevice, s));
    GPM_CUDA(cudaStreamSynchronize(s));
  }
  // multi-GPU: the only collectives are the per-pattern counts and the
  // per-level size vectors
  if (cfg.world > 1 && cfg.exchange) {
    if (App::kReduce == kReduceCodes && !c.list_fn) exchange_device(cfg, d_hist.get(), c.nbins, 8, 0, s);
    else exchange_device(cfg, d_total.get(), 1, 8, 0, s);
    std::vector<u64> v;
    for (auto x : st.level_sizes) v.push_back(x);
    for (auto x : st.candidates) v.push_back(x);
    v.push_back((u64)st.balg);
    exchange_sum_host(cfg, v, s);
    const size_t nl = st.level_sizes.size();
    for (size_t i = 0; i < nl; ++i) st.level_sizes[i] = v[i];
    for (size_t i = 0; i < st.candidates.size(); ++i) st.candidates[i] = v[nl + i];
    st.balg = (double)v.back();
    st.level_sizes[levels - 1] = 0;  // re-derived from the reduced counters below
  }

  if (App::kReduce == kReduceCodes && !c.list_fn && k > 2) {
    const int nbins = c.nbins;
    std::vector<unsigned long long> h(nbins);
    GPM_CUDA(cudaMemcpyAsync(h.data(), d_hist.get(), sizeof(unsigned long long) * nbins, cudaMemcpyDeviceToHost, s));
    std::vector<u64> keys;
    if (App::kCodesAreMasks) {
      keys.resize(nbins);
      DBuf<u64> dk(nbins, s);
      canon_masks_kernel<><<<(nbins + 127) / 128, 128, 0, s>>>(k, dk.get());
      GPM_CUDA(cudaGetLastError());
      ++tl.launches;
      GPM_CUDA(cudaMemcpyAsync(keys.data(), dk.get(), sizeof(u64) * nbins, cudaMemcpyDeviceToHost, s));
    }
    GPM_CUDA(cudaStreamSynchronize(s));
    std::map<std::string, u64> agg;
    u64 acc = 0, kept = 0;
    for (int m = 0; m < nbins; ++m)
      if (h[m]) {
        acc += h[m];
        if (App::kFilter && App::to_prune((u32)m, h[m], k)) continue;
        kept += h[m];
        agg[App::kCodesAreMasks ? canon_text(keys[m], k, 0, nullptr) : App::code_text((u32)m, k)] += h[m];
      }
    for (auto& [text, cnt] : agg) res.patterns.push_back({text, cnt, k});
    st.level_sizes[levels - 1] += acc;
    res.total = kept;
  } else if (k > 2) {
    unsigned long long t = 0;
    GPM_CUDA(cudaMemcpyAsync(&t, d_total.get(), sizeof t, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaStreamSynchronize(s));
    res.total = t;
    st.level_sizes[levels - 1] += t;
  }
}

}  // namespace engine

// Runs `mine` for a user App through the library's gpm_mine bookkeeping
// (stream, timing events, stats record): the entry point a C-ABI wrapper of
// a custom App calls (tests/apps/test_apps.cu).
template <class App>
int mine_app(const gpm_graph* g, const gpm_config* cfg, gpm_result** out) {
  return run_custom(g, cfg, out, [](const gpm_graph& G, const gpm_config& c, cudaStream_t s, gpm_result& r, Stats& st,
                                    Timeline& tl) { engine::mine<App>(G, c, s, r, st, tl); });
}

}  // namespace gpm
