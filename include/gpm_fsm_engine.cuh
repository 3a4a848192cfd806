#pragma once
// gpm_fsm_engine.cuh — the header-only edge-mode extend-reduce-filter engine
// (frequent subgraph mining and user edge-mode apps) on sm_100a, templated on
// an App that supplies the reference's hooks (Listing 5):
//   to_extend<LEV>(emb, pos)                toExtend: positions whose edges extend
//   to_add_edge<LEV>(emb, g, q, w, r)       toAdd(edge): the new edge (v_q, w);
//                                           r = position of w in emb (nv: new vertex)
//   to_prune(PatternInfo)                   toPrune on a canonical pattern's
//                                           (count, MNI support, sigma)
//   support_of(PatternInfo)                 the support reported with a
//                                           surviving pattern (getSupport)
//   kBuiltin                                the builtin FSM hooks: enables the
//                                           grouped and fan-out fast paths
//   kDomains                                compute MNI domains (false: the
//                                           support handed to to_prune is 0 and
//                                           only counts are reduced)
// The builtin FSM (csrc/fsm.cu) is FsmApp in gpm_fsm_apps.cuh; a user app
// includes gpm_fsm_apps.cuh and calls gpm::mine_edge_app<App>
// (tests/apps/test_apps.cu).
//
// Reference: Listing 5, Alg. 1 with the level-1
// reduce+filter before the loop
// (is_auto_canonical_edge), :193-210 (quick/canonical pattern), :276-302
// (domain support, merge, MNI), :362-370 (filter), :441-449 (fsm app).
//
// Per level:
//   A  extend + quick code: every accepted child's quick code (nv, position
//      labels, position-pair edge mask; pattern.cuh) is inserted into an
//      open-addressing device hash table with warp-aggregated counts.
//   C  canonicalize each distinct quick code once (<= 5! permutations),
//      sort-reduce canonical codes -> dense pattern ids + counts.  Patterns
//      whose embedding count < sigma cannot reach MNI >= sigma (MNI <= count),
//      so only count-frequent patterns get domain bitmaps.
//   B  extend again: OR each child's vertices into bitmap[pattern][perm[i]]
//      (atomicOr on u32 words, canonical positions via the PositionMap).
//   M  popcount per (pattern, position), min -> MNI.
//   F  filter (not on the last level): inspection-execution over children
//      whose pattern has MNI >= sigma -> next SoA level (idx, vid, his).
// The last level is never materialised.  Multi-GPU: pattern keys are
// all-gathered and bitmaps OR-exchanged through gpm_config.exchange.
#include <parallel/algorithm>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>

#include "engine.hpp"
#include "pattern.cuh"

namespace gpm {

void scan_inplace(u64* data, u64 n, cudaStream_t s);

namespace fsm_engine {

// Per-thread host scratch vectors that keep their capacity across calls: the
// per-level host arrays (10^5..10^6 entries) would otherwise be fresh
// allocations whose first-touch page faults cost ~1 ms per MB on these hosts.
// One slot per (type, use); every use is a temporary of one function.
template <class T, int SLOT>
std::vector<T>& host_scratch() {
  static thread_local std::vector<T> v;
  return v;
}

// Pool of u64 host vectors (capacity kept across levels and calls) for the
// per-level pattern arrays that outlive one function (keys, counts, MNI).
inline std::vector<std::vector<u64>>& u64_pool() {
  static thread_local std::vector<std::vector<u64>> p;
  return p;
}
inline std::vector<u64> take_u64() {
  auto& p = u64_pool();
  if (p.empty()) return {};
  std::vector<u64> v = std::move(p.back());
  p.pop_back();
  v.clear();
  return v;
}
inline void give_u64(std::vector<u64>& v) {
  if (v.capacity() && u64_pool().size() < 8) u64_pool().push_back(std::move(v));
  v = std::vector<u64>();
}

// host threads for the per-pattern loops (1 when the including translation
// unit is built without OpenMP)
inline int host_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
inline int host_thread() {
#ifdef _OPENMP
  return omp_get_thread_num();
#else
  return 0;
#endif
}

// What App::to_prune sees of a canonical pattern after the level's reduce:
// its packed canonical code (pattern.cuh; pat::decode with label_bits gives
// the position labels -- dense label ranks -- and the edge mask), its
// embedding count, its MNI support (0 when no domains were needed: count
// below the MNI bound), sigma and the MNI mode (gpm_config.mni_mode).
struct PatternInfo {
  u64 key;
  u64 count;
  u64 support;
  u64 sigma;
  int label_bits;
  int mni_mode;
  int num_vertices() const { return pat::code_nv(key); }
};

namespace {

constexpr int kThreads = 256;
constexpr u64 kBatch = 2048;
constexpr int kMaxEdges = 5;  // k <= 6
enum { kQC = 0, kDomain = 1, kSCount = 2, kSWrite = 3, kQCD = 4, kSparse = 5 };

struct ELevels {
  const u32* idx[kMaxEdges + 1];
  const u32* vid[kMaxEdges + 1];
  const u8* his[kMaxEdges + 1];
};

// Edge-mode embedding with LEV edges (embedding_list.hpp:73-115 edge branch).
template <int LEV>
struct EEmb {
  static constexpr int MAXV = LEV + 1;
  int nv;
  u32 v[MAXV];
  u32 lab[MAXV];
  u8 slot[MAXV];
  u8 step[MAXV];
  u32 e0[LEV], e1[LEV];   // normalised vertex pairs e_1..e_LEV
  u8 pa[LEV], pb[LEV];    // position pairs
};

template <int LEV>
__device__ __forceinline__ void reconstruct_e(const ELevels& L, const DevGraph& g, u64 i, EEmb<LEV>& E) {
  u32 chain[LEV + 1];
  u8 his[LEV + 1];
  u64 p = i;
#pragma unroll
  for (int k = LEV; k >= 2; --k) {
    chain[k] = ldg(L.vid[k - 1] + p);
    his[k] = L.his[k - 1][p];
    p = ldg(L.idx[k - 1] + p);
  }
  chain[0] = ldg(L.idx[0] + p);
  chain[1] = ldg(L.vid[0] + p);
  his[1] = 0;
  u8 slotpos[LEV + 1];
  E.nv = 0;
#pragma unroll
  for (int j = 0; j <= LEV; ++j) {
    int at = E.nv;
#pragma unroll
    for (int q = 0; q < LEV + 1; ++q)
      if (q < E.nv && E.v[q] == chain[j] && at == E.nv) at = q;
    if (at == E.nv) {
#pragma unroll
      for (int q = 0; q < LEV + 1; ++q)
        if (q == E.nv) {
          E.v[q] = chain[j];
          E.slot[q] = (u8)j;
          E.step[q] = (u8)(j < 1 ? 1 : j);
        }
      ++E.nv;
    }
    slotpos[j] = (u8)at;
  }
#pragma unroll
  for (int q = 0; q < LEV + 1; ++q)
    if (q < E.nv) E.lab[q] = ldg(g.lab + E.v[q]);
#pragma unroll
  for (int j = 1; j <= LEV; ++j) {
    u32 a = chain[his[j]], b = chain[j];
    E.e0[j - 1] = min(a, b);
    E.e1[j - 1] = max(a, b);
    E.pa[j - 1] = slotpos[his[j]];
    E.pb[j - 1] = slotpos[j];
  }
}

__device__ __forceinline__ bool pair_gt(u32 a0, u32 a1, u32 b0, u32 b1) { return a0 != b0 ? a0 > b0 : a1 > b1; }

// is_auto_canonical_edge + closing edge from its earlier-inserted
// endpoint only.  r = position of w in the embedding or nv if new.
template <int LEV>
__device__ __forceinline__ bool edge_to_add(const EEmb<LEV>& E, int q, u32 w, int r) {
  const u32 x = E.v[q];
  const u32 n0 = min(x, w), n1 = max(x, w);
  bool dup = false;
#pragma unroll
  for (int j = 0; j < LEV; ++j) dup |= (E.e0[j] == n0 && E.e1[j] == n1);
  if (dup) return false;
  if (r < E.nv && r < q) return false;
  if (!pair_gt(n0, n1, E.e0[0], E.e1[0])) return false;
  int p = E.step[q];
  if (r < E.nv) p = min(p, (int)E.step[r]);
#pragma unroll
  for (int s = 2; s <= LEV; ++s)
    if (s > p && !pair_gt(n0, n1, E.e0[s - 1], E.e1[s - 1])) return false;
  return true;
}

// Quick code of the child (parent + edge (q, w)); fills child vertices.
template <int LEV>
__device__ __forceinline__ u64 child_code(const EEmb<LEV>& E, const DevGraph& g, int q, u32 w, int r, int LB,
                                          u32* cv, int& cnv) {
  u32 lab[LEV + 2];
  cnv = E.nv;
#pragma unroll
  for (int i = 0; i < LEV + 1; ++i)
    if (i < E.nv) {
      cv[i] = E.v[i];
      lab[i] = E.lab[i];
    }
  int wp = r;
  if (r == E.nv) {
#pragma unroll
    for (int i = 0; i < LEV + 2; ++i)
      if (i == E.nv) {
        cv[i] = w;
        lab[i] = ldg(g.lab + w);
      }
    wp = E.nv;
    ++cnv;
  }
  u32 mask = 0;
#pragma unroll
  for (int j = 0; j < LEV; ++j) {
    int a = min(E.pa[j], E.pb[j]), b = max(E.pa[j], E.pb[j]);
    mask |= 1u << pat::pair_index(a, b, cnv);
  }
  mask |= 1u << pat::pair_index(min(q, wp), max(q, wp), cnv);
  return pat::make_code(cnv, lab, mask, LB);
}

// Open-addressing table of quick codes; entry = {key, val} in 16 B so a probe
// touches one sector.  During pass A val = (dense quick-code id << 40 | count)
// (ids 1.. in insertion order); once the level is canonicalised val is
// overwritten with (pattern id << 32 | packed PositionMap).
struct Hash {
  unsigned long long* ent;     // 2 x capacity: ent[2h] key (0 = empty), ent[2h+1] val
  u64 mask;                    // capacity - 1
  unsigned long long* used;    // inserted keys
  int* overflow;
};

__device__ __forceinline__ u64 hash64(u64 x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

constexpr int kMaxProbe = 256;

// Insert-or-add with bounded linear probing.  Once the table is flagged as
// overflowing (load > 1/2 or a probe run > kMaxProbe) inserts stop at once;
// the host regrows the table and re-runs the pass.
constexpr u64 kCountMask = (u64(1) << 40) - 1;

// Returns the key's dense id (>= 1), or 0 once the table overflowed.
__device__ __forceinline__ u32 hash_add(const Hash& H, u64 key, unsigned long long c) {
  if (*(volatile int*)H.overflow) return 0;
  u64 h = hash64(key) & H.mask;
  for (int probe = 0; probe < kMaxProbe; ++probe) {
    // one 16-byte load returns key and val together: once a key's id is
    // published it never changes, so a hit needs no atomic round trip — the
    // count is added with a fire-and-forget reduction
    const ulonglong2 e = *reinterpret_cast<const ulonglong2*>(H.ent + 2 * h);
    unsigned long long cur = e.x;
    if (cur == key && (e.y >> 40) != 0) {
      atomicAdd(H.ent + 2 * h + 1, c);
      return (u32)(e.y >> 40);
    }
    if (cur == 0) {
      unsigned long long prev = atomicCAS(H.ent + 2 * h, 0ull, (unsigned long long)key);
      if (prev == 0ull) {
        const unsigned long long n = atomicAdd(H.used, 1ull);
        if (n * 2 >= H.mask) atomicOr(H.overflow, 1);
        atomicAdd(H.ent + 2 * h + 1, ((unsigned long long)(n + 1) << 40) + c);
        return (u32)(n + 1);
      }
      cur = prev;
    }
    if (cur == key) {
      unsigned long long v = atomicAdd(H.ent + 2 * h + 1, c);
      // the inserting thread publishes the id right after its CAS
      while ((v >> 40) == 0) v = *(volatile unsigned long long*)(H.ent + 2 * h + 1);
      return (u32)(v >> 40);
    }
    h = (h + 1) & H.mask;
  }
  atomicOr(H.overflow, 2);
  return 0;
}

__device__ __forceinline__ u64 hash_info(const Hash& H, u64 slot) { return H.ent[2 * slot + 1]; }

__device__ __forceinline__ u64 hash_find(const Hash& H, u64 key) {
  u64 h = hash64(key) & H.mask;
  for (int probe = 0; probe < kMaxProbe; ++probe) {
    unsigned long long cur = H.ent[2 * h];
    if (cur == key) return h;
    if (cur == 0) return ~0ull;
    h = (h + 1) & H.mask;
  }
  return ~0ull;
}

struct FsmArgs {
  DevGraph g;
  ELevels L;
  const u64* Wp;
  const u32* pidx;
  u64 np, W, B, b_begin, b_end;
  u64 grab;
  unsigned long long* ctr;
  int LB;
  Hash H;
  const u32* bslot;       // pattern -> bitmap slot or ~0
  u32* bitmaps;
  u64 words;
  const u32* lrank;       // vertex -> rank within its label class (label-local bitmap index)
  const u32* labrank;     // vertex -> label << 27 | rank (fan pass; labels < 32, ranks < 2^27)
  u32* qbm;               // fused last level: domain bitmaps per quick-code id (quick positions)
  u64 qcap;               // ids with a bitmap
  int* qover;             // set when an id >= qcap appeared (host falls back to a domain pass)
  int kpos;
  u32 round_lo, round_hi;
  const u8* frequent;     // pattern -> MNI >= sigma
  // sparse domains: pattern -> sparse slot or ~0, the slot's
  // packed orbit representatives (3 bits per canonical position), and the
  // (slot, position, label-local rank) key buffer
  const u32* sslot;
  const u32* srep;
  unsigned long long* skeys;
  unsigned long long* stop;
  u64 scap;
  u64* cnt;
  const u64* boffs;
  u64 out_base;
  u32* out_idx;
  u32* out_vid;
  u8* out_his;
  unsigned long long* accepted;
};

// OR the child's vertices into its pattern's domain bitmaps.  All position
// words are loaded before any atomic: the loads are independent, so issuing
// them together overlaps their (mostly DRAM) latencies instead of paying one
// round trip per position (the atomics would otherwise fence the next load).
// first = first position this lane must write (lanes whose parent positions are
// written by a peer lane start at the parent's vertex count).
template <int NV>
__device__ __forceinline__ void bitmap_or(u32* base, u64 words, const u32* __restrict__ lrank, u32 perm, bool permute,
                                          const u32* cv, int cnv, int first) {
  u32* wp[NV];
  u32 bit[NV], old[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    wp[i] = nullptr;
    if (i >= first && i < cnv) {
      const u32 cp = permute ? (perm >> (3 * i)) & 7u : (u32)i;
      const u32 lr = ldg(lrank + cv[i]);  // all vertices at one position share its label
      wp[i] = base + (u64)cp * words + (lr >> 5);
      bit[i] = 1u << (lr & 31);
    }
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) old[i] = wp[i] ? *wp[i] : 0u;
  // domains saturate quickly: test before the read-modify-write so most
  // embeddings cost a load instead of an L2 atomic (a stale read only causes a
  // redundant, still-correct atomicOr)
#pragma unroll
  for (int i = 0; i < NV; ++i)
    if (wp[i] && !(old[i] & bit[i])) atomicOr(wp[i], bit[i]);
}

template <int NV>
__device__ __forceinline__ void domain_or(const FsmArgs& a, u64 info, const u32* cv, int cnv, int first) {
  const u32 pid = (u32)(info >> 32);
  const u32 bs = a.bslot[pid];
  if (bs < a.round_lo || bs >= a.round_hi) return;
  u32* base = a.bitmaps + (u64)(bs - a.round_lo) * a.kpos * a.words;
  bitmap_or<NV>(base, a.words, a.lrank, (u32)info, true, cv, cnv, first);
}

// Sparse domains: a child of a sparse pattern emits one key per vertex,
// (slot << 35 | orbit-representative canonical position << 32 | label-local
// rank); the warp reserves its keys with one atomic.  Sorting + unique then
// gives the domains exactly (their sizes are the MNI inputs).
__device__ __forceinline__ void sparse_emit(const FsmArgs& a, bool ok, u64 info, const u32* cv, int cnv) {
  const int lane = threadIdx.x & 31;
  u32 sl = ~0u;
  if (ok) sl = a.sslot[(u32)(info >> 32)];
  const u32 nk = sl != ~0u ? (u32)cnv : 0u;
  u32 incl = nk;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const u32 tot = __shfl_sync(0xffffffffu, incl, 31);
  if (!tot) return;
  unsigned long long base = 0;
  if (lane == 31) base = atomicAdd(a.stop, (unsigned long long)tot);
  base = __shfl_sync(0xffffffffu, base, 31) + (incl - nk);
  if (!nk) return;
  const u32 perm = (u32)info, rep = a.srep[sl];
  for (int i = 0; i < cnv; ++i) {
    const u32 cp = (perm >> (3 * i)) & 7u;
    const u32 rp = (rep >> (3 * cp)) & 7u;
    if (base + i < a.scap)
      a.skeys[base + i] = ((unsigned long long)sl << 35) | ((unsigned long long)rp << 32) | ldg(a.lrank + cv[i]);
  }
}

// Work per parent: sum of deg over all positions (to_extend default true).
template <class App, int LEV>
__global__ void __launch_bounds__(kThreads) ework_kernel(DevGraph g, ELevels L, u64 np, u64* __restrict__ W,
                                                         unsigned long long* __restrict__ nvsum) {
  unsigned long long mine = 0;
  for (u64 p = blockIdx.x * (u64)blockDim.x + threadIdx.x; p < np; p += (u64)gridDim.x * blockDim.x) {
    EEmb<LEV> E;
    reconstruct_e<LEV>(L, g, p, E);
    u64 w = 0;
#pragma unroll
    for (int q = 0; q < LEV + 1; ++q)
      if (q < E.nv && App::template to_extend<LEV>(E, q)) w += ldg(g.off + E.v[q] + 1) - ldg(g.off + E.v[q]);
    W[p] = w;
    mine += E.nv;
  }
  mine = __reduce_add_sync(0xffffffffu, (unsigned)mine);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(nvsum, mine);
}

template <class App, int LEV>
struct ECursor {
  u64 cp = ~0ull, cWb = 0, cWe = 0;
  u32 parent = 0;
  EEmb<LEV> E;
  u64 pbeg[LEV + 1];
  u32 pdeg[LEV + 1];
  __device__ __forceinline__ void load(const FsmArgs& a, u64 p) {
    if (p == cp) return;
    cp = p;
    cWb = ldg(a.Wp + p);
    cWe = ldg(a.Wp + p + 1);
    parent = ldg(a.pidx + p);
    reconstruct_e<LEV>(a.L, a.g, parent, E);
#pragma unroll
    for (int q = 0; q < LEV + 1; ++q) {
      if (q < E.nv && App::template to_extend<LEV>(E, q)) {  // toExtend
        pbeg[q] = ldg(a.g.off + E.v[q]);
        pdeg[q] = (u32)(ldg(a.g.off + E.v[q] + 1) - pbeg[q]);
      } else {
        pbeg[q] = 0;
        pdeg[q] = 0;
      }
    }
  }
  __device__ __forceinline__ void locate(const FsmArgs& a, u64 j, u64 pa, u64 pb) {
    if (cp != ~0ull && j < cWe && j >= cWb) return;
    const u64 lo = (cp == ~0ull || j < cWb) ? pa : cp + 1;
    load(a, upper_bound_prev(a.Wp, lo, pb + 1, j));
  }
  __device__ __forceinline__ u32 candidate(const DevGraph& g, u64 j, int& q) const {
    u32 local = (u32)(j - cWb);
    q = 0;
#pragma unroll
    for (int t = 0; t < LEV; ++t)
      if (q == t && local >= pdeg[t]) {
        local -= pdeg[t];
        q = t + 1;
      }
    return ldg(g.col + pbeg[q] + local);
  }
};

template <class App, int LEV, int MODE>
__global__ void __launch_bounds__(kThreads) eextend_kernel(FsmArgs a) {
  const int lane = threadIdx.x & 31;
  const DevGraph& g = a.g;
  unsigned long long acc = 0;
  u64 bgrab = 0, bleft = 0;
  for (;;) {
    if (bleft == 0) {  // 4 batches per atomic: one global counter serialises at L2
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
    if (MODE == kSWrite) {
      wpos = ldg(a.boffs + b);
      if (ldg(a.boffs + b + 1) == wpos) continue;
      wpos -= a.out_base;
    }
    u64 pr = 0;
    if (lane == 0) pr = upper_bound_prev(a.Wp, 0, a.np + 1, j0);
    u64 P0 = __shfl_sync(0xffffffffu, pr, 0);
    ECursor<App, LEV> cur;
    u32 c = 0;
    for (u64 jb = j0; jb < j1; jb += 32) {
      const u64 j = jb + lane;
      const u64 x = (P0 + 1 + lane <= a.np) ? ldg(a.Wp + P0 + 1 + lane) : ~0ull;
      const u32 bit = (x - jb < 32) ? (1u << (u32)(x - jb)) : 0u;
      const u32 starts = __reduce_or_sync(0xffffffffu, bit);
      const u64 myp = P0 + __popc(starts & (lanemask_lt() | (1u << lane)));
      P0 += __popc(starts);
      bool ok = false;
      u64 code = 0;
      u32 w = 0;
      int q = 0, r = 0;
      u32 cv[LEV + 2];
      int cnv = 0;
      if (j < j1) {
        cur.load(a, myp);
        w = cur.candidate(g, j, q);
        r = cur.E.nv;
#pragma unroll
        for (int i = 0; i < LEV + 1; ++i)
          if (i < cur.E.nv && cur.E.v[i] == w) r = i;
        ok = App::template to_add_edge<LEV>(cur.E, g, q, w, r);  // toAdd(edge)
        if (ok) code = child_code<LEV>(cur.E, g, q, w, r, a.LB, cv, cnv);
      }
      if (MODE == kQC) {
        const u32 mask = __ballot_sync(0xffffffffu, ok);
        acc += __popc(mask);
        if (mask) {
          const unsigned long long key = ok ? code : ~0ull;
          const u32 peers = __match_any_sync(0xffffffffu, key);
          const int leader = __ffs(peers) - 1;
          // lanes with the same quick code AND the same parent set identical
          // bits for the parent's positions: only the lowest of them writes them
          const u32 sib = peers & __match_any_sync(0xffffffffu, myp);
          const int first = (lane == __ffs(sib) - 1) ? 0 : cur.E.nv;
          u32 id = 0;
          if (ok && lane == leader) id = hash_add(a.H, code, __popc(peers));
          if (a.qbm) {
            // fused last level: OR the child's vertices into its quick code's
            // domain bitmaps (quick positions; merged per canonical pattern later)
            id = __shfl_sync(0xffffffffu, id, leader);
            if (ok && id) {
              if (id - 1 < a.qcap) {
                u32* base = a.qbm + (u64)(id - 1) * a.kpos * a.words;
                bitmap_or<LEV + 2>(base, a.words, a.lrank, 0u, false, cv, cnv, first);
              } else {
                *a.qover = 1;
              }
            }
          }
        }
      } else if (MODE == kSparse) {
        const u64 info = ok ? hash_info(a.H, hash_find(a.H, code)) : 0ull;
        sparse_emit(a, ok, info, cv, cnv);
      } else if (MODE == kDomain) {
        const u32 peers = __match_any_sync(0xffffffffu, ok ? code : ~0ull);
        const u32 sib = peers & __match_any_sync(0xffffffffu, myp);
        const int first = (lane == __ffs(sib) - 1) ? 0 : cur.E.nv;
        if (ok) domain_or<LEV + 2>(a, hash_info(a.H, hash_find(a.H, code)), cv, cnv, first);
      } else {
        bool keep = false;
        if (ok) {
          keep = a.frequent[hash_info(a.H, hash_find(a.H, code)) >> 32] != 0;
        }
        const u32 mask = __ballot_sync(0xffffffffu, keep);
        if (MODE == kSCount) {
          c += __popc(mask);
        } else {
          if (keep) {
            const u64 o = wpos + __popc(mask & lanemask_lt());
            a.out_idx[o] = cur.parent;
            a.out_vid[o] = w;
            a.out_his[o] = cur.E.slot[q];
          }
          wpos += __popc(mask);
        }
      }
    }
    if (MODE == kSCount && lane == 0) a.cnt[b - a.b_begin] = c;
  }
  if (MODE == kQC && lane == 0 && acc) atomicAdd(a.accepted, acc);
}

// ---------------------------------------------------------------------------
// Grouped passes.  Parents are sorted by their quick code, so
// a contiguous candidate range ("item") holds the children of a few parent
// codes, and a child's quick code is a function of (parent code, extended
// position, new label | closing position): an item produces at most
// ~(LEV+1) x (labels + LEV+1) distinct child codes.  One CTA takes an item,
// aggregates per child code in shared memory -- counts (pass A) or the
// quick-position domain bitmaps (pass B) -- and flushes once per code: pass
// A adds each code's count to the global hash (instead of one random hash
// probe per warp step), pass B ORs each code's bitmap rows into its canonical
// pattern's rows through the PositionMap (coalesced rows instead of one
// random DRAM read-modify-write per child and position).
// threads per grouped CTA (one CTA per SM; FSM17 level-2 passes 512 -> 1024:
// 2.59 -> 1.83 ms and 4.64 -> 3.00 ms despite small spills at 64 registers)
constexpr int kGT = 1024;
constexpr u32 kSlotPending = 0xffffffffu;      // map entry inserted, slot not yet published
constexpr u32 kSlotNone = 0xfffffffeu;         // no shared slot: global fallback

struct GroupArgs {
  const u64* items;     // nitems + 1 candidate-space boundaries
  u64 nitems;
  unsigned long long* ctr;
  u32 mcap;             // shared map entries (power of two)
  u32 cslots;           // shared per-code slots
};

template <int LEV>
__device__ __forceinline__ u64 parent_code(const EEmb<LEV>& E, int LB) {
  u32 mask = 0;
#pragma unroll
  for (int j = 0; j < LEV; ++j) {
    const int a = min(E.pa[j], E.pb[j]), b = max(E.pa[j], E.pb[j]);
    mask |= 1u << pat::pair_index(a, b, E.nv);
  }
  return pat::make_code(E.nv, E.lab, mask, LB);
}

// group key of every compacted parent: a 24-bit hash of its quick code
// (colliding codes merely share a group)
template <int LEV>
__global__ void pkey_kernel(DevGraph g, ELevels L, const u32* __restrict__ pidx, u64 nz, int LB,
                            u32* __restrict__ keys) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nz; i += (u64)gridDim.x * blockDim.x) {
    EEmb<LEV> E;
    reconstruct_e<LEV>(L, g, pidx[i], E);
    keys[i] = (u32)(hash64(parent_code<LEV>(E, LB)) >> 40);
  }
}

__global__ void gstart_kernel(const u32* __restrict__ keys, u64 n, u8* __restrict__ flag) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void gather_starts_kernel(const u64* __restrict__ Wp, const u32* __restrict__ starts, u64 G,
                                     u64* __restrict__ out) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < G; i += (u64)gridDim.x * blockDim.x)
    out[i] = Wp[starts[i]];
}

// Per-lane parent descriptor for the grouped passes: everything the
// per-candidate test needs, precomputed once when the lane's parent changes,
// so that is_auto_canonical_edge becomes one packed-pair compare and the
// child's quick code one OR (new vertex) -- the generic edge_to_add /
// child_code (above) rebuild position arrays and pattern codes per candidate.
//   edge_to_add: n = (min, max) of the new edge; accept iff
//   n is not an edge of the parent, r >= q for a closing edge, and n > e_1
//   and n > e_s for every s > p, p = step(q) (min with step(r) when closing),
//   i.e. n > thr[p] with thr[p] = max(e_1, max_{s>p} e_s) (packed pairs
//   compare lexicographically as integers).
template <int LEV>
struct FCur {
  static constexpr int MV = LEV + 1;
  u64 cp = ~0ull, cWb = 0, cWe = 0;
  u32 parent = 0;
  int nv = 0;
  u32 v[MV];       // parent vertices (~0 past nv)
  u32 lr[MV];      // label-local ranks of the parent vertices (domain modes)
  u32 cend[MV];    // cumulative candidate ends per position (parent-local)
  u64 cbase[MV];   // col index of candidate `local` at position q = cbase[q] + local
  u64 dupe[LEV];   // parent edges, packed (min << 32 | max)
  u64 thr[LEV + 1];
  u64 newc[MV];    // child code for a new vertex from q (new label bits zero)
  u32 stp;         // step of position q in bits [4q, 4q+4)
  u32 pmask;       // parent position-pair mask (nv positions)
  u32 lshift;      // npairs(nv + 1): new label shift
  u64 labp;        // parent labels packed (pattern.cuh order)

  __device__ __forceinline__ void load(const FsmArgs& a, u64 p, bool want_lr) {
    if (p == cp) return;
    cp = p;
    cWb = ldg(a.Wp + p);
    cWe = ldg(a.Wp + p + 1);
    parent = ldg(a.pidx + p);
    EEmb<LEV> E;
    reconstruct_e<LEV>(a.L, a.g, parent, E);
    nv = E.nv;
    pmask = 0;
#pragma unroll
    for (int j = 0; j < LEV; ++j) {
      const int x = min(E.pa[j], E.pb[j]), y = max(E.pa[j], E.pb[j]);
      pmask |= 1u << pat::pair_index(x, y, nv);
      dupe[j] = ((u64)E.e0[j] << 32) | E.e1[j];
    }
#pragma unroll
    for (int pp = 1; pp <= LEV; ++pp) {
      u64 t = dupe[0];
#pragma unroll
      for (int s2 = 2; s2 <= LEV; ++s2)
        if (s2 > pp) t = max(t, dupe[s2 - 1]);
      thr[pp] = t;
    }
    thr[0] = thr[1];
    labp = 0;
    stp = 0;
    u32 acc = 0;
#pragma unroll
    for (int q = 0; q < MV; ++q) {
      const bool in = q < nv;
      v[q] = in ? E.v[q] : 0xffffffffu;
      if (in) labp = (labp << a.LB) | E.lab[q];
      stp |= (u32)(in ? E.step[q] : 0) << (4 * q);
      u64 b = 0;
      u32 d = 0;
      if (in) {
        b = ldg(a.g.off + v[q]);
        d = (u32)(ldg(a.g.off + v[q] + 1) - b);
      }
      cbase[q] = b - acc;
      acc += d;
      cend[q] = acc;
      lr[q] = (in && want_lr) ? ldg(a.lrank + v[q]) : 0u;
    }
    // new-vertex child codes: parent mask re-indexed to nv + 1 positions
    const u32 m1 = pat::widen_mask(pmask, nv);
#pragma unroll
    for (int q = 0; q < MV; ++q)
      newc[q] = q < nv ? pat::make_code_packed(nv + 1, labp << a.LB, m1 | (1u << pat::pair_index(q, nv, nv + 1)))
                       : 0ull;
    lshift = (u32)pat::npairs(nv + 1);
  }
  __device__ __forceinline__ void locate(const FsmArgs& a, u64 j, u64 pa, u64 pb, bool want_lr) {
    if (cp != ~0ull && j < cWe && j >= cWb) return;
    const u64 lo = (cp == ~0ull || j < cWb) ? pa : cp + 1;
    load(a, upper_bound_prev(a.Wp, lo, pb + 1, j), want_lr);
  }

  // register-resident select (a dynamic index would put the array in local memory)
  template <class T, int N>
  __device__ __forceinline__ static T sel(const T (&arr)[N], int i) {
    T x = arr[0];
#pragma unroll
    for (int t = 1; t < N; ++t)
      if (i == t) x = arr[t];
    return x;
  }

  // Candidate j of the loaded parent: accepted?  Fills the child's code and
  // its new vertex w with w's position r (nv if new).
  __device__ __forceinline__ bool eval(const FsmArgs& a, u64 j, u64& code, u32& w, int& r) const {
    const u32 local = (u32)(j - cWb);
    int q = 0;
#pragma unroll
    for (int t = 0; t < MV - 1; ++t) q += local >= cend[t];
    w = ldg(a.g.col + sel(cbase, q) + local);
    r = nv;
#pragma unroll
    for (int i = 0; i < MV; ++i)
      if (v[i] == w) r = i;
    const u32 x = sel(v, q);
    const u64 n = w < x ? (((u64)w << 32) | x) : (((u64)x << 32) | w);
    const int sq = (int)((stp >> (4 * q)) & 15u);
    if (r == nv) {
      if (!(n > sel(thr, sq))) return false;
      code = sel(newc, q) | ((u64)ldg(a.g.lab + w) << lshift);
      return true;
    }
    // closing edge (rare): both endpoints in the parent
    if (r < q) return false;
#pragma unroll
    for (int jj = 0; jj < LEV; ++jj)
      if (dupe[jj] == n) return false;
    const int sr = (int)((stp >> (4 * r)) & 15u);
    if (!(n > sel(thr, min(sq, sr)))) return false;
    code = pat::make_code_packed(nv, labp, pmask | (1u << pat::pair_index(q, r, nv)));
    return true;
  }
};

// shared-memory map: child quick code -> per-code slot (or kSlotNone)
template <int MODE>
__device__ __forceinline__ u32 smap_get(unsigned long long* mkey, u32* mslot, u32 mcap, u32* used, u32 cslots,
                                        unsigned long long* sinfo, unsigned long long* skey, u32* sid, u64 code,
                                        const FsmArgs& a) {
  u32 h = (u32)hash64(code) & (mcap - 1);
  for (u32 probe = 0; probe < mcap; ++probe) {
    unsigned long long k = mkey[h];
    if (k == 0ull) {
      const unsigned long long prev = atomicCAS(mkey + h, 0ull, (unsigned long long)code);
      if (prev == 0ull) {
        const u32 sl = atomicAdd(used, 1u);
        u32 val = kSlotNone;
        if (sl < cslots) {
          val = sl;
          skey[sl] = code;  // read only after the item's barrier
          // sinfo is shared with the other warps of the item before any
          // barrier: written and read with atomics (published through mslot)
          unsigned long long si = 0ull;
          if (MODE == kDomain) {
            // the code's canonical pattern and PositionMap; a bitmap only if
            // the pattern has one in this round
            const u64 info = hash_info(a.H, hash_find(a.H, code));
            const u32 bs = a.bslot[(u32)(info >> 32)];
            si = (bs >= a.round_lo && bs < a.round_hi) ? (((u64)(bs - a.round_lo) << 32) | (u32)info) : ~0ull;
          }
          atomicExch(sinfo + sl, si);
          if (MODE == kQCD) {
            sid[sl] = hash_add(a.H, code, 0ull);  // dense quick-code id (0: table overflow)
          }
        }
        __threadfence_block();
        atomicExch(mslot + h, val);  // publish (atomics: the flag is not a data race)
        return val;
      }
      k = prev;
    }
    if (k == code) {
      u32 val;
      while ((val = atomicAdd(mslot + h, 0u)) == kSlotPending) {
      }
      __threadfence_block();
      return val;
    }
    h = (h + 1) & (mcap - 1);
  }
  return kSlotNone;
}

// MODE kQC: quick-code counts; kQCD: counts + quick-position domain bitmaps
// per quick-code id (the fused last level); kDomain: canonical-position
// domain bitmaps of the current round (two-pass levels).
template <int LEV, int MODE>
__global__ void __launch_bounds__(kGT, 1) egroup_kernel(FsmArgs a, GroupArgs ga) {
  extern __shared__ __align__(16) unsigned char gsm[];
  unsigned long long* mkey = reinterpret_cast<unsigned long long*>(gsm);
  unsigned long long* sinfo = mkey + ga.mcap;    // kQC/kQCD: count; kDomain: (bitmap slot << 32 | perm) or ~0
  unsigned long long* skey = sinfo + ga.cslots;  // code per slot
  u32* mslot = reinterpret_cast<u32*>(skey + ga.cslots);
  u32* sid = mslot + ga.mcap;                    // kQCD: dense quick-code id per slot
  u32* sbm = sid + ga.cslots;                    // kDomain / kQCD: [cslots][kpos][words]
  constexpr bool kRows = MODE != kQC;
  __shared__ u64 s_item, s_pa, s_pb;
  __shared__ unsigned long long s_next;
  __shared__ u32 s_used;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int NW = kGT / 32;
  constexpr u64 kChunk = 4096;  // candidates per warp grab inside an item
  const u64 rowlen = (u64)a.kpos * a.words;
  unsigned long long acc = 0;
  for (;;) {
    __syncthreads();  // the previous item's flush is done
    if (threadIdx.x == 0) {
      const u64 it = atomicAdd(ga.ctr, 1ull);
      s_item = it;
      s_used = 0;
      if (it < ga.nitems) {
        const u64 j0 = ldg(ga.items + it), j1 = ldg(ga.items + it + 1);
        s_next = j0;
        s_pa = upper_bound_prev(a.Wp, 0, a.np + 1, j0);
        s_pb = upper_bound_prev(a.Wp, s_pa, a.np + 1, j1 - 1);
      }
    }
    for (u32 i = threadIdx.x; i < ga.mcap; i += kGT) {
      mkey[i] = 0ull;
      mslot[i] = kSlotPending;
    }
    if (kRows) {
      const u64 nz = (u64)ga.cslots * rowlen;
      for (u64 i = threadIdx.x; i < nz; i += kGT) sbm[i] = 0u;
    }
    __syncthreads();
    const u64 item = s_item;
    if (item >= ga.nitems) break;
    const u64 j1 = ldg(ga.items + item + 1);
    const u64 ipa = s_pa, ipb = s_pb;
    FCur<LEV> cur;
    for (;;) {  // warps grab kChunk-candidate pieces of the item (balance inside the CTA)
      unsigned long long c0 = 0;
      if (lane == 0) c0 = atomicAdd(&s_next, (unsigned long long)kChunk);
      const u64 wj0 = __shfl_sync(0xffffffffu, c0, 0);
      if (wj0 >= j1) break;
      const u64 wj1 = min(j1, wj0 + kChunk);
      u64 pr = 0;
      if (lane == 0) pr = upper_bound_prev(a.Wp, ipa, ipb + 1, wj0);
      u64 P0 = __shfl_sync(0xffffffffu, pr, 0);
      for (u64 jb = wj0; jb < wj1; jb += 32) {
        const u64 j = jb + lane;
        const u64 x = (P0 + 1 + lane <= a.np) ? ldg(a.Wp + P0 + 1 + lane) : ~0ull;
        const u32 bit = (x - jb < 32) ? (1u << (u32)(x - jb)) : 0u;
        const u32 starts = __reduce_or_sync(0xffffffffu, bit);
        const u64 myp = P0 + __popc(starts & (lanemask_lt() | (1u << lane)));
        P0 += __popc(starts);
        bool ok = false;
        u64 code = 0;
        u32 w = 0;
        int r = 0;
        if (j < wj1) {
          cur.load(a, myp, kRows);
          ok = cur.eval(a, j, code, w, r);
        }
        const u32 mask = __ballot_sync(0xffffffffu, ok);
        if (!mask) continue;
        const u32 peers = __match_any_sync(0xffffffffu, ok ? code : ~0ull);
        const int leader = __ffs(peers) - 1;
        u32 slot = kSlotNone;
        if (ok && lane == leader)
          slot = smap_get<MODE>(mkey, mslot, ga.mcap, &s_used, ga.cslots, sinfo, skey, sid, code, a);
        slot = __shfl_sync(0xffffffffu, slot, leader);
        if (MODE != kDomain) {
          acc += __popc(mask);
          if (ok && lane == leader) {
            if (slot != kSlotNone) atomicAdd(sinfo + slot, (unsigned long long)__popc(peers));
          }
        }
        if (MODE == kQC) {
          if (ok && lane == leader && slot == kSlotNone) hash_add(a.H, code, __popc(peers));
          continue;
        }
        // ---- domains: the child's vertices at its quick positions
        // (lanes with the same code and parent write the parent's positions once)
        const u32 sib = peers & __match_any_sync(0xffffffffu, myp);
        const int first = (lane == __ffs(sib) - 1) ? 0 : cur.nv;
        u32* row = nullptr;
        u32 perm = 0;
        bool permute = false;
        if (MODE == kQCD && ok && slot == kSlotNone) {
          // no shared slot: straight into the code's global rows (old path)
          u32 id = 0;
          if (lane == leader) id = hash_add(a.H, code, __popc(peers));
          id = __shfl_sync(peers, id, leader);
          if (id && id - 1 >= a.qcap) *a.qover = 1;
          else if (id) row = a.qbm + (u64)(id - 1) * rowlen;
        } else if (ok && slot != kSlotNone) {
          if (MODE != kDomain || atomicAdd(sinfo + slot, 0ull) != ~0ull) row = sbm + (u64)slot * rowlen;  // kDomain: bitmap this round?
        } else if (ok) {  // kDomain without a shared slot
          const u64 info = hash_info(a.H, hash_find(a.H, code));
          const u32 bs = a.bslot[(u32)(info >> 32)];
          if (bs >= a.round_lo && bs < a.round_hi) {
            row = a.bitmaps + (u64)(bs - a.round_lo) * rowlen;
            perm = (u32)info;
            permute = true;
          }
        }
        if (row) {
          const int cnv = (r == cur.nv) ? cur.nv + 1 : cur.nv;
          const u32 wl = (r == cur.nv) ? ldg(a.lrank + w) : 0u;
          u32* wp[LEV + 2];
          u32 bm[LEV + 2], old[LEV + 2];
#pragma unroll
          for (int i = 0; i < LEV + 2; ++i) {
            wp[i] = nullptr;
            if (i >= first && i < cnv) {
              const u32 lri = (i < LEV + 1 && i < cur.nv) ? FCur<LEV>::sel(cur.lr, i < LEV + 1 ? i : 0) : wl;
              const u32 cp = permute ? (perm >> (3 * i)) & 7u : (u32)i;
              wp[i] = row + (u64)cp * a.words + (lri >> 5);
              bm[i] = 1u << (lri & 31);
            }
          }
#pragma unroll
          for (int i = 0; i < LEV + 2; ++i) old[i] = wp[i] ? *wp[i] : 0u;
#pragma unroll
          for (int i = 0; i < LEV + 2; ++i)
            if (wp[i] && !(old[i] & bm[i])) atomicOr(wp[i], bm[i]);
        }
      }
    }
    __syncthreads();
    // ---- flush once per code
    const u32 used = min(s_used, ga.cslots);
    if (MODE != kDomain) {
      for (u32 sl = threadIdx.x; sl < used; sl += kGT)
        if (sinfo[sl]) hash_add(a.H, skey[sl], sinfo[sl]);
    }
    if (kRows) {
      for (u64 row = wid; row < (u64)used * a.kpos; row += NW) {
        const u32 sl = (u32)(row / a.kpos);
        const int i = (int)(row % a.kpos);
        if (i >= pat::code_nv(skey[sl])) continue;
        u32* dst;
        if (MODE == kDomain) {
          const u64 info = sinfo[sl];
          if (info == ~0ull) continue;
          const u32 cp = ((u32)info >> (3 * i)) & 7u;
          dst = a.bitmaps + ((info >> 32) * a.kpos + cp) * a.words;
        } else {
          const u32 id = sid[sl];
          if (!id) continue;
          if (id - 1 >= a.qcap) {
            if (lane == 0) *a.qover = 1;
            continue;
          }
          dst = a.qbm + ((u64)(id - 1) * a.kpos + i) * a.words;
        }
        const u32* src = sbm + (u64)sl * rowlen + (u64)i * a.words;
        for (u64 w = lane; w < a.words; w += 32) {
          const u32 val = src[w];
          if (val) atomicOr(dst + w, val);
        }
      }
    }
  }
  if (MODE != kDomain && lane == 0 && acc) atomicAdd(a.accepted, acc);  // acc is warp-uniform
}

// ---------------------------------------------------------------------------
// Fan-out pass of the fused last level.  Parents are sorted
// by their exact quick code; an item is (one parent code P, one extended
// position q, a range of P's parents).  Every child of the item then has the
// quick code
//   new vertex w:   base(P, q) | label(w) << npairs(nv+1)   -> slot label(w)
//   closing w=v_r:  code(P + edge (q, r))                  -> slot NL + r
// so the item's codes are DENSE slots of a per-CTA shared table (counts and
// quick-position domain rows) -- no hashing or code building per child.  A
// child's new vertex sets one bit of its slot's new-vertex row; the parent
// positions' bits are the same for all children of one parent with one slot,
// so each parent ORs its vertices once per slot it produced (a label mask
// reduced over the warp), not once per child.  At the end of the item every
// used slot adds its count to the level's quick-code hash (dense id) and ORs
// its rows into that id's global quick-position bitmaps (qbm) -- the same
// state the rest of the fused path (canonicalise, merge_qbm) consumes.
// Lanes map to the candidates N(v_q) of one parent at a time (coalesced);
// parent descriptors are built 32 at a time, one per lane, into shared memory.
// threads per fan CTA: 14 warps when two such CTAs fit an SM (the fan pass is
// latency-bound at 2 CTAs/SM: FSM17 256 -> 122.4 ms, 320 -> 110.7, 384 ->
// 102.9, 448 -> 97.5; one CTA of 512-704 threads: 123-145 ms), else 8
constexpr int kFT = 256;
constexpr int kFTWide = 448;
constexpr int kRankBits = 27;            // labrank[v] = label << 27 | rank within the label class
constexpr u32 kRankMask = (1u << kRankBits) - 1;
constexpr u32 kFanParents = 4096;        // parents per item (large groups split)

struct FanItem {
  u64 code;    // parent quick code
  u32 pa, pb;  // parents [pa, pb) of the sorted compacted order
  u32 q;       // extended position
  u32 pad;
};

struct FanArgs {
  const FanItem* items;
  u64 nitems;
  unsigned long long* ctr;
  u32 nl;      // new-vertex slots (1 << LB <= 32)
};

template <int LEV>
struct FanDesc {  // per-warp parent descriptors, struct of arrays over 32 lanes
  static constexpr int MV = LEV + 1;
  u64 cb[32];
  u64 thrq[32];
  u64 dupe[LEV][32];
  u64 thr[LEV + 1][32];
  u32 deg[32];
  u32 x[32];
  u32 v[MV][32];
  u32 lr[MV][32];
  u32 stp[32];
};

template <int LEV, int FT>
__global__ void __launch_bounds__(FT, 2) efan_kernel(FsmArgs a, FanArgs fa) {
  constexpr int MV = LEV + 1;
  constexpr int NW = FT / 32;
  extern __shared__ __align__(16) unsigned char fsm_fan_smem[];
  const u32 nslot = fa.nl + MV;
  const u64 rowlen = (u64)a.kpos * a.words;
  u32* rows = reinterpret_cast<u32*>(fsm_fan_smem);          // [nslot][kpos][words]
  u32* cnt = rows + (u64)nslot * rowlen;                      // [nslot]
  u32* sid = cnt + nslot;                                     // [nslot] quick-code id at flush
  const u64 doff = (u64)nslot * rowlen + 2 * nslot;
  FanDesc<LEV>* descs = reinterpret_cast<FanDesc<LEV>*>(rows + doff + (doff & 1));  // 8-byte aligned
  __shared__ u64 s_item;
  __shared__ u32 s_bnext;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  FanDesc<LEV>& D = descs[wid];
  unsigned long long acc = 0;
  for (u64 i = threadIdx.x; i < (u64)nslot * rowlen; i += FT) rows[i] = 0u;
  for (;;) {
    for (u32 i = threadIdx.x; i < nslot; i += FT) cnt[i] = 0u;
    if (threadIdx.x == 0) {
      s_item = atomicAdd(fa.ctr, 1ull);
      if (s_item < fa.nitems) s_bnext = fa.items[s_item].pa;
    }
    __syncthreads();
    const u64 it = s_item;
    if (it >= fa.nitems) break;
    const FanItem item = fa.items[it];
    const int q = (int)item.q;
    int nv;
    u32 plab[8], pmask;
    pat::decode(item.code, a.LB, &nv, plab, &pmask);
    u64 labp = 0;
    for (int i = 0; i < nv; ++i) labp = (labp << a.LB) | plab[i];
    const u32 lshift = (u32)pat::npairs(nv + 1);
    const u64 newbase = pat::make_code_packed(nv + 1, labp << a.LB,
                                              pat::widen_mask(pmask, nv) | (1u << pat::pair_index(q, nv, nv + 1)));
    // ---- warps grab 32-parent batches of the item
    for (;;) {
      u32 b0 = 0;
      if (lane == 0) b0 = atomicAdd(&s_bnext, 32u);
      b0 = __shfl_sync(0xffffffffu, b0, 0);
      if (b0 >= item.pb) break;
      const u32 nb = min(32u, item.pb - b0);
      __syncwarp();
      if ((u32)lane < nb) {
        EEmb<LEV> E;
        reconstruct_e<LEV>(a.L, a.g, ldg(a.pidx + b0 + lane), E);
        u64 dupe[LEV];
#pragma unroll
        for (int j = 0; j < LEV; ++j) dupe[j] = ((u64)E.e0[j] << 32) | E.e1[j];
        u64 thr[LEV + 1];
#pragma unroll
        for (int pp = 1; pp <= LEV; ++pp) {
          u64 t = dupe[0];
#pragma unroll
          for (int s2 = 2; s2 <= LEV; ++s2)
            if (s2 > pp) t = max(t, dupe[s2 - 1]);
          thr[pp] = t;
        }
        thr[0] = thr[1];
        u32 stp = 0, x = 0;
#pragma unroll
        for (int i = 0; i < MV; ++i) {
          const bool in = i < E.nv;
          D.v[i][lane] = in ? E.v[i] : 0xffffffffu;
          D.lr[i][lane] = in ? ldg(a.labrank + E.v[i]) & kRankMask : 0u;
          stp |= (u32)(in ? E.step[i] : 0) << (4 * i);
          if (i == q) x = E.v[i];
        }
#pragma unroll
        for (int j = 0; j < LEV; ++j) D.dupe[j][lane] = dupe[j];
        u64 tq = thr[0];
#pragma unroll
        for (int pp = 0; pp <= LEV; ++pp) {
          D.thr[pp][lane] = thr[pp];
          if (pp == (int)((stp >> (4 * q)) & 15u)) tq = thr[pp];
        }
        const u64 cb = ldg(a.g.off + x);
        D.cb[lane] = cb;
        D.deg[lane] = (u32)(ldg(a.g.off + x + 1) - cb);  // >= 1: x is an endpoint of a parent edge
        D.x[lane] = x;
        D.thrq[lane] = tq;
        D.stp[lane] = stp;
      }
      __syncwarp();
      // flattened (parent, 32-candidate chunk) stream of the batch, the next
      // chunk's candidates in flight while the current one is evaluated
      u32 cj = 0, cjb = 0;
      u32 cw = (u32)lane < D.deg[0] ? ldg(a.g.col + D.cb[0] + lane) : 0u;
      u32 lm = 0, cm = 0;  // labels of new-vertex children / closing positions of parent cj
      while (cj < nb) {
        const u32 cdeg = D.deg[cj];
        u32 nj = cj, njb = cjb + 32;
        if (njb >= cdeg) {
          nj = cj + 1;
          njb = 0;
        }
        u32 nw = 0;
        if (nj < nb && njb + lane < D.deg[nj]) nw = ldg(a.g.col + D.cb[nj] + njb + lane);
        const u32 x = D.x[cj];
        const u64 thrq = D.thrq[cj];
        bool ok = false;
        if (cjb + lane < cdeg) {
          const u32 w = cw;
          const u32 lw = ldg(a.labrank + w);  // issued before the position / threshold tests
          int r = nv;
#pragma unroll
          for (int i = 0; i < MV; ++i)
            if (i < nv && D.v[i][cj] == w) r = i;
          const u64 n = w < x ? (((u64)w << 32) | x) : (((u64)x << 32) | w);
          if (r == nv) {
            ok = n > thrq;
            if (ok) {
              const u32 lab = lw >> kRankBits, lr = lw & kRankMask;
              atomicAdd(cnt + lab, 1u);
              u32* wp = rows + ((u64)lab * a.kpos + nv) * a.words + (lr >> 5);
              const u32 bit = 1u << (lr & 31);
              if (!(*wp & bit)) atomicOr(wp, bit);
              lm |= 1u << lab;
            }
          } else if (r > q) {  // closing edge from its earlier-inserted endpoint
            bool dup = false;
#pragma unroll
            for (int jj = 0; jj < LEV; ++jj) dup |= D.dupe[jj][cj] == n;
            const u32 stp = D.stp[cj];
            const int sq = (int)((stp >> (4 * q)) & 15u), sr = (int)((stp >> (4 * r)) & 15u);
            const int sm = min(sq, sr);
            u64 t = D.thr[0][cj];
#pragma unroll
            for (int pp = 1; pp <= LEV; ++pp)
              if (pp == sm) t = D.thr[pp][cj];
            ok = !dup && n > t;
            if (ok) cm |= 1u << r;
          }
        }
        acc += __popc(__ballot_sync(0xffffffffu, ok));
        if (nj != cj) {
          // end of parent cj: its vertices once per (parent, slot) produced
          lm = __reduce_or_sync(0xffffffffu, lm);
          cm = __reduce_or_sync(0xffffffffu, cm);
          if (lm | cm) {
            u32 plr[MV];
#pragma unroll
            for (int i = 0; i < MV; ++i) plr[i] = D.lr[i][cj];
            if (lm >> lane & 1u) {  // lane = new-vertex label (nl <= 32)
#pragma unroll
              for (int i = 0; i < MV; ++i)
                if (i < nv) {
                  u32* wp = rows + ((u64)lane * a.kpos + i) * a.words + (plr[i] >> 5);
                  const u32 bit = 1u << (plr[i] & 31);
                  if (!(*wp & bit)) atomicOr(wp, bit);
                }
            }
            if (lane < MV && (cm >> lane & 1u)) {
              const u32 sl = fa.nl + lane;
              atomicAdd(cnt + sl, 1u);  // one closing child per (parent, q, r)
#pragma unroll
              for (int i = 0; i < MV; ++i)
                if (i < nv) {
                  u32* wp = rows + ((u64)sl * a.kpos + i) * a.words + (plr[i] >> 5);
                  atomicOr(wp, 1u << (plr[i] & 31));
                }
            }
          }
          lm = 0;
          cm = 0;
        }
        cj = nj;
        cjb = njb;
        cw = nw;
      }
    }
    __syncthreads();
    // ---- flush: count -> quick-code hash (dense id), rows -> the id's qbm rows
    for (u32 sl = threadIdx.x; sl < nslot; sl += FT) {
      u32 id = 0;
      if (cnt[sl]) {
        u64 code;
        if (sl < fa.nl) code = newbase | ((u64)sl << lshift);
        else code = pat::make_code_packed(nv, labp, pmask | (1u << pat::pair_index(q, (int)(sl - fa.nl), nv)));
        id = hash_add(a.H, code, cnt[sl]);
        if (id && id - 1 >= a.qcap) {
          *a.qover = 1;
          id = 0;
        }
      }
      sid[sl] = id;
    }
    __syncthreads();
    for (u64 rr = wid; rr < (u64)nslot * a.kpos; rr += NW) {
      const u32 sl = (u32)(rr / a.kpos);
      const int i = (int)(rr % a.kpos);
      if (!cnt[sl]) continue;
      const int cnv = sl < fa.nl ? nv + 1 : nv;
      if (i >= cnv) continue;
      u32* src = rows + rr * a.words;
      const u32 id = sid[sl];
      u32* dst = id ? a.qbm + ((u64)(id - 1) * a.kpos + i) * a.words : nullptr;
      for (u64 w = lane; w < a.words; w += 32) {
        const u32 val = src[w];
        if (val) {
          if (dst) atomicOr(dst + w, val);
          src[w] = 0u;
        }
      }
    }
    __syncthreads();
  }
  if (lane == 0 && acc) atomicAdd(a.accepted, acc);
}

// exact quick code of every compacted parent (fan grouping key)
template <int LEV>
__global__ void pcode_kernel(DevGraph g, ELevels L, const u32* __restrict__ pidx, u64 nz, int LB,
                             u64* __restrict__ codes) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nz; i += (u64)gridDim.x * blockDim.x) {
    EEmb<LEV> E;
    reconstruct_e<LEV>(L, g, pidx[i], E);
    codes[i] = parent_code<LEV>(E, LB);
  }
}

// codes <-> sort keys: rotate the vertex-count nibble (bits 60-63) to the
// bottom so the occupied bits are contiguous from bit 0 (fewer radix passes)
__global__ void rotl4_kernel(u64* __restrict__ c, u64 n, int left) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u64 x = c[i];
    c[i] = left ? (x << 4) | (x >> 60) : (x >> 4) | (x << 60);
  }
}

__global__ void gstart64_kernel(const u64* __restrict__ keys, u64 n, u8* __restrict__ flag) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void gather_codes_kernel(const u64* __restrict__ codes, const u32* __restrict__ starts, u64 G,
                                    u64* __restrict__ out) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < G; i += (u64)gridDim.x * blockDim.x)
    out[i] = codes[starts[i]];
}

// ---- level 1 (single edges): reduce + filter before the loop
__device__ __forceinline__ u64 l1_code(const DevGraph& g, u32 u, u32 v, int LB) {
  u32 lab[2] = {ldg(g.lab + u), ldg(g.lab + v)};
  return pat::make_code(2, lab, 1u, LB);
}

template <int MODE>
__global__ void l1_kernel(FsmArgs a, const u32* __restrict__ idx, const u32* __restrict__ vid, u64 n,
                          u8* __restrict__ keep) {
  const int lane = threadIdx.x & 31;
  for (u64 i0 = (blockIdx.x * (u64)blockDim.x + threadIdx.x) & ~31ull; i0 < n; i0 += (u64)gridDim.x * blockDim.x) {
    const u64 i = i0 + lane;
    const bool act = i < n;
    u32 u = 0, v = 0;
    u64 code = 0;
    if (act) {
      u = idx[i];
      v = vid[i];
      code = l1_code(a.g, u, v, a.LB);
    }
    if (MODE == kQC) {
      const unsigned long long key = act ? code : ~0ull;
      const u32 peers = __match_any_sync(0xffffffffu, key);
      if (act && lane == __ffs(peers) - 1) hash_add(a.H, code, __popc(peers));
    } else if (MODE == kDomain) {
      if (act) {
        u32 cv[2] = {u, v};
        domain_or<2>(a, hash_info(a.H, hash_find(a.H, code)), cv, 2, 0);
      }
    } else if (MODE == kSparse) {
      u32 cv[2] = {u, v};
      sparse_emit(a, act, act ? hash_info(a.H, hash_find(a.H, code)) : 0ull, cv, 2);
    } else if (act) {
      keep[i] = a.frequent[hash_info(a.H, hash_find(a.H, code)) >> 32];
    }
  }
}

// canonicalize every occupied hash slot once (reduce step 2)
// occupied hash slots -> a dense list (any order; everything after is per
// distinct quick code, so the level's arrays are U-sized instead of cap-sized)
__global__ void occ_kernel(const unsigned long long* __restrict__ ent, u64 cap, unsigned long long* __restrict__ top,
                           u32* __restrict__ occ) {
  for (u64 s = blockIdx.x * (u64)blockDim.x + threadIdx.x; s < cap; s += (u64)gridDim.x * blockDim.x)
    if (ent[2 * s]) occ[atomicAdd(top, 1ull)] = (u32)s;
}

__global__ void canon_slots_kernel(const unsigned long long* __restrict__ ent, const u32* __restrict__ occ, u64 U,
                                   int LB, u64* __restrict__ canon, u32* __restrict__ perm, u64* __restrict__ counts,
                                   u32* __restrict__ ids) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < U; i += (u64)gridDim.x * blockDim.x) {
    const u64 s = occ[i];
    const u64 key = ent[2 * s];
    counts[i] = ent[2 * s + 1] & kCountMask;
    ids[i] = (u32)(ent[2 * s + 1] >> 40);
    int nv;
    u32 lab[8], mask;
    pat::decode(key, LB, &nv, lab, &mask);
    u8 p[8];
    canon[i] = pat::canonicalize(nv, lab, mask, LB, p);
    u32 pk = 0;
    for (int j = 0; j < nv; ++j) pk |= (u32)p[j] << (3 * j);
    perm[i] = pk;
  }
}

// Fused last level: OR each quick code's position bitmaps into its canonical
// pattern's bitmaps through the PositionMap (one warp per quick code).
__global__ void merge_qbm_kernel(const u32* __restrict__ qbm, const u64* __restrict__ canon,
                                 const u32* __restrict__ ids, const u32* __restrict__ perm, u64 cap,
                                 const unsigned long long* __restrict__ ent, const u32* __restrict__ occ,
                                 const u32* __restrict__ bslot, u32 round_lo, u32 round_hi, u32* __restrict__ bitmaps,
                                 u64 words, int kpos) {
  const int lane = threadIdx.x & 31;
  for (u64 sl = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5; sl < cap;
       sl += ((u64)gridDim.x * blockDim.x) >> 5) {
    const u64 c = canon[sl];
    if (c == ~0ull) continue;
    // pattern id of the canonical key: slot_pid_kernel published it in the
    // slot's value (a per-warp binary search over ~10^6 keys was ~20
    // dependent loads per quick code, most of this kernel's time)
    const u32 pid = (u32)(ent[2 * (u64)occ[sl] + 1] >> 32);
    const u32 bs = bslot[pid];
    if (bs < round_lo || bs >= round_hi) continue;
    const int nv = pat::code_nv(c);
    const u32 pm = perm[sl];
    const u32* q = qbm + (u64)(ids[sl] - 1) * kpos * words;
    u32* b = bitmaps + (u64)(bs - round_lo) * kpos * words;
    for (int i = 0; i < nv; ++i) {
      const u32 cp = (pm >> (3 * i)) & 7u;
      for (u64 w = lane; w < words; w += 32) {
        const u32 v = q[(u64)i * words + w];
        if (v) atomicOr(b + (u64)cp * words + w, v);
      }
    }
  }
}

__global__ void slot_pid_kernel(const u64* __restrict__ canon, const u32* __restrict__ occ, u64 U,
                                const u64* __restrict__ gkeys, u64 P, const u32* __restrict__ perm,
                                unsigned long long* __restrict__ ent) {
  for (u64 s = blockIdx.x * (u64)blockDim.x + threadIdx.x; s < U; s += (u64)gridDim.x * blockDim.x) {
    const u64 c = canon[s];
    u64 lo = 0, hi = P;
    while (lo < hi) {
      u64 mid = (lo + hi) >> 1;
      if (gkeys[mid] < c) lo = mid + 1;
      else hi = mid;
    }
    ent[2 * (u64)occ[s] + 1] = ((unsigned long long)lo << 32) | perm[s];
  }
}

// popcount per (pattern, canonical position); MNI = min over positions
// MNI per bitmap pattern: min over positions of the domain size
// (canonical-mapping MNI).  full != 0: full-automorphism
// MNI -- an embedding's mappings include every automorphism
// of the pattern, so a position's domain is the union of the canonical
// domains over its automorphism orbit; min over orbits.
// One warp per bitmap pattern (8 per CTA): ~10^6 patterns of a few KB each
// (a CTA per pattern was ~5 us of scheduling per pattern, 4 ms a level)
__global__ void mni_kernel(const u32* __restrict__ bitmaps, u64 words, int kpos, const u64* __restrict__ gkeys,
                           const u32* __restrict__ bs_to_pid, u32 round_lo, u32 round_n, int LB, int full,
                           unsigned long long* __restrict__ mni) {
  const u32 lane = threadIdx.x & 31;
  const u32 r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);  // bitmap pattern within round
  if (r >= round_n) return;
  const u32 pid = bs_to_pid[round_lo + r];
  const u64 key = gkeys[pid];
  const int nv = pat::code_nv(key);
  // orbit representative of each position, 4 bits each (identity unless full)
  u32 reps = 0x76543210u;
  if (full) {
    if (lane == 0) {
      int n2;
      u32 lab[8], mask;
      u8 rep[8];
      for (int i = 0; i < 8; ++i) rep[i] = (u8)i;
      pat::decode(key, LB, &n2, lab, &mask);
      pat::orbits(nv, lab, mask, rep);
      reps = 0;
      for (int i = 0; i < 8; ++i) reps |= (u32)rep[i] << (4 * i);
    }
    reps = __shfl_sync(0xffffffffu, reps, 0);
  }
  unsigned long long best = ~0ull;
  for (int pos = 0; pos < nv; ++pos) {
    if (((reps >> (4 * pos)) & 15u) != (u32)pos) continue;  // counted with its orbit's representative
    const u32* bm = bitmaps + ((u64)r * kpos + pos) * words;
    u32 c = 0;
    for (u64 w = lane; w < words; w += 32) {
      u32 v = bm[w];
      for (int o = pos + 1; o < nv; ++o)
        if (((reps >> (4 * o)) & 15u) == (u32)pos) v |= bitmaps[((u64)r * kpos + o) * words + w];
      c += __popc(v);
    }
    c = __reduce_add_sync(0xffffffffu, c);  // <= n / labels bits per position
    best = min(best, (unsigned long long)c);
  }
  if (lane == 0) mni[pid] = best;
}

// packed orbit representatives of every sparse slot (identity unless
// full-automorphism MNI)
__global__ void srep_kernel(const u64* __restrict__ gkeys, const u32* __restrict__ sp_to_pid, u64 NS, int LB, int full,
                            u32* __restrict__ srep) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < NS; i += (u64)gridDim.x * blockDim.x) {
    const u64 key = gkeys[sp_to_pid[i]];
    const int nv = pat::code_nv(key);
    u8 rep[8];
    for (int j = 0; j < 8; ++j) rep[j] = (u8)j;
    if (full) {
      int n2;
      u32 lab[8], mask;
      pat::decode(key, LB, &n2, lab, &mask);
      pat::orbits(nv, lab, mask, rep);
    }
    u32 pk = 0;
    for (int j = 0; j < 8; ++j) pk |= (u32)rep[j] << (3 * j);
    srep[i] = pk;
  }
}

// sorted keys -> distinct (slot, position, vertex) per (slot, position)
__global__ void sparse_count_kernel(const unsigned long long* __restrict__ k, u64 n,
                                    unsigned long long* __restrict__ dcnt) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    if (k[i] != ~0ull && (i == 0 || k[i] != k[i - 1])) atomicAdd(dcnt + (k[i] >> 32), 1ull);
}

// MNI of every sparse slot: min over its orbit representatives' domain sizes
__global__ void sparse_mni_kernel(const unsigned long long* __restrict__ dcnt, const u64* __restrict__ gkeys,
                                  const u32* __restrict__ sp_to_pid, const u32* __restrict__ srep, u64 NS,
                                  unsigned long long* __restrict__ mni) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < NS; i += (u64)gridDim.x * blockDim.x) {
    const u32 pid = sp_to_pid[i];
    const int nv = pat::code_nv(gkeys[pid]);
    unsigned long long best = ~0ull;
    for (int j = 0; j < nv; ++j)
      if (((srep[i] >> (3 * j)) & 7u) == (u32)j) best = min(best, dcnt[i * 8 + j]);
    mni[pid] = best;
  }
}

struct NonZeroW {
  const u64* w;
  __device__ __forceinline__ bool operator()(const u32& i) const { return w[i] != 0; }
};

__global__ void egather_kernel(const u64* __restrict__ w, const u32* __restrict__ pidx, u64 nz, u64* __restrict__ Wp) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nz; i += (u64)gridDim.x * blockDim.x)
    Wp[i] = w[pidx[i]];
}

__global__ void iota_kernel(u32* __restrict__ v, u32 n) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) v[i] = (u32)i;
}

// sorted (label, vertex) -> rank of each vertex within its label class; the
// largest class size -> *mx
__global__ void lrank_kernel(const u32* __restrict__ lab, const u32* __restrict__ vid, u32 n, u32* __restrict__ lrank,
                             u32* __restrict__ labrank, unsigned long long* __restrict__ mx) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    // class start: first index with the same label (binary search)
    u64 lo = 0, hi = i;
    const u32 L = lab[i];
    while (lo < hi) {
      const u64 mid = (lo + hi) >> 1;
      if (lab[mid] < L) lo = mid + 1;
      else hi = mid;
    }
    lrank[vid[i]] = (u32)(i - lo);
    if (labrank) labrank[vid[i]] = (L << kRankBits) | ((u32)(i - lo) & kRankMask);
    if (i + 1 == n || lab[i + 1] != L) atomicMax(mx, (unsigned long long)(i - lo + 1));
  }
}

inline unsigned grid1(u64 items) { return (unsigned)std::max<u64>(1, std::min<u64>((items + 255) / 256, 1u << 20)); }

// ------------------------------------------------------------------ host driver
template <class App>
struct Fsm {
  const gpm_graph& G;
  const gpm_config& cfg;
  DevGraph g;
  cudaStream_t s;
  Stats& st;
  Timeline& tl;
  gpm_result& res;
  int k;
  u64 sigma;
  int LB;
  int sms;
  u64 budget;
  u64 prev_unique = 1024;
  DBuf<unsigned long long> d_ctr;
  DBuf<u32> lrank;   // vertex -> rank within its label class
  DBuf<u32> labrank; // vertex -> label << 27 | rank (fan pass; LB <= 5)
  u64 max_class = 1;
  // words of one label-local domain row (padding rows to 16 bytes for
  // vector loads in merge_qbm measured slower: 5.7 -> 11.3 ms, the lanes'
  // ORs no longer coalesce)
  u64 dom_words() const { return (max_class + 31) / 32; }

  // lrank[v] = #{u < v : lab[u] == lab[v]} via a stable sort of (label, v)
  void label_ranks() {
    const u32 n = G.n;
    lrank.alloc(std::max<u32>(1, n), s);
    if (!n) return;
    DBuf<u32> lab2(n, s), vid(n, s), vid2(n, s);
    iota_kernel<<<grid1(n), 256, 0, s>>>(vid.get(), n);
    GPM_CUDA(cudaGetLastError());
    size_t tmp = 0;
    GPM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, G.d_lab, lab2.get(), vid.get(), vid2.get(), (int64_t)n, 0,
                                             std::max(1, LB), s));
    DBuf<u8> t(tmp, s);
    GPM_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, G.d_lab, lab2.get(), vid.get(), vid2.get(), (int64_t)n, 0,
                                             std::max(1, LB), s));
    DBuf<unsigned long long> mx(1, s);
    GPM_CUDA(cudaMemsetAsync(mx.get(), 0, sizeof(unsigned long long), s));
    if (LB <= 5) labrank.alloc(n, s);
    lrank_kernel<<<grid1(n), 256, 0, s>>>(lab2.get(), vid2.get(), n, lrank.get(), LB <= 5 ? labrank.get() : nullptr,
                                          mx.get());
    GPM_CUDA(cudaGetLastError());
    tl.launches += 4;
    max_class = std::max<u64>(1, d2h(mx.get()));
  }

  Fsm(const gpm_graph& G_, const gpm_config& c_, cudaStream_t s_, Stats& st_, Timeline& tl_, gpm_result& r_)
      : G(G_), cfg(c_), g(G_.view()), s(s_), st(st_), tl(tl_), res(r_) {}

  void sync() { GPM_CUDA(cudaStreamSynchronize(s)); }
  // host-side phase trace (GPM_TRACE=1)
  void trace(const char* what, double a = 0, double b = 0) {
    static const bool on = std::getenv("GPM_TRACE") != nullptr;
    if (!on) return;
    sync();
    static auto t0 = std::chrono::steady_clock::now();
    double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[gpm fsm] %10.1f ms  %-24s %.6g %.6g\n", ms, what, a, b);
  }
  template <class T>
  T d2h(const T* p) {
    T v;
    GPM_CUDA(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, s));
    sync();
    return v;
  }

  // Reduce state for one level
  struct Level {
    u64 cap = 0;
    DBuf<unsigned long long> ent, used;
    DBuf<int> overflow;
    DBuf<u64> canon;
    DBuf<u32> perm, bslot, bs_to_pid, ids, occ;  // perm / ids / canon / occ: per occupied slot
    u64 U = 0;
    DBuf<u8> frequent;
    std::vector<u64> gkeys_h, gcount_h, mni_h;  // from / back to the host pool (u64_pool)
    std::vector<u8> freq_h;  // frequent (not pruned) flags, host copy
    Level() = default;
    Level(const Level&) = delete;
    Level& operator=(const Level&) = delete;
    ~Level() {
      give_u64(gkeys_h);
      give_u64(gcount_h);
      give_u64(mni_h);
    }
    DBuf<u64> gkeys;
    u64 P = 0;
    u64 NB = 0;
    // sparse domains: pattern -> sparse slot, slot -> pattern, key capacity
    DBuf<u32> sslot, sp_to_pid;
    u64 NS = 0;
    u64 skeys_total = 0;
  };

  Hash hash_of(Level& R) {
    return Hash{R.ent.get(), R.cap - 1, R.used.get(), R.overflow.get()};
  }

  void alloc_hash(Level& R, u64 cap) {
    R.cap = cap;
    R.ent.alloc(2 * cap, s);
    R.used.alloc(1, s);
    R.overflow.alloc(1, s);
    GPM_CUDA(cudaMemsetAsync(R.ent.get(), 0, sizeof(unsigned long long) * 2 * cap, s));
    GPM_CUDA(cudaMemsetAsync(R.used.get(), 0, sizeof(unsigned long long), s));
    GPM_CUDA(cudaMemsetAsync(R.overflow.get(), 0, sizeof(int), s));
  }

  // After pass A: canonicalize slots, global pattern table (+exchange), pids,
  // count pre-filter, bitmap slots.
  void canon_and_group(Level& R, int kpos, bool allow_sparse) {
    // list the U occupied slots, canonicalize each distinct quick code once,
    // sort by canonical code and reduce by key on the device: only the
    // distinct canonical patterns come back to the host
    const u64 U = d2h(R.used.get());
    R.U = U;
    const u64 U1 = std::max<u64>(1, U);
    R.occ.alloc(U1, s);
    R.canon.alloc(U1, s);
    R.perm.alloc(U1, s);
    R.ids.alloc(U1, s);
    DBuf<u64> ck2(U1, s);
    DBuf<unsigned long long> cc3(U1, s), cc4(U1, s), top(1, s);
    GPM_CUDA(cudaMemsetAsync(top.get(), 0, sizeof(unsigned long long), s));
    occ_kernel<<<grid1(R.cap), 256, 0, s>>>(R.ent.get(), R.cap, top.get(), R.occ.get());
    canon_slots_kernel<<<grid1(U1), 256, 0, s>>>(R.ent.get(), R.occ.get(), U, LB, R.canon.get(), R.perm.get(),
                                                 reinterpret_cast<u64*>(cc3.get()), R.ids.get());
    GPM_CUDA(cudaGetLastError());
    tl.launches += 2;
    DBuf<u64> ck(U1, s);
    if (U) GPM_CUDA(cudaMemcpyAsync(ck.get(), R.canon.get(), sizeof(u64) * U, cudaMemcpyDeviceToDevice, s));
    std::vector<u64> keys = take_u64(), cnts = take_u64();
    if (U) {
      size_t tmp = 0;
      GPM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, ck.get(), ck2.get(), cc3.get(), cc4.get(), (int64_t)U, 0,
                                               64, s));
      DBuf<u8> t(tmp, s);
      GPM_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, ck.get(), ck2.get(), cc3.get(), cc4.get(), (int64_t)U, 0,
                                               64, s));
      DBuf<u64> nuniq(1, s);
      size_t tmp2 = 0;
      GPM_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, tmp2, ck2.get(), ck.get(), cc4.get(), cc3.get(), nuniq.get(),
                                              cuda::std::plus<unsigned long long>{}, (int64_t)U, s));
      DBuf<u8> t2(tmp2, s);
      GPM_CUDA(cub::DeviceReduce::ReduceByKey(t2.get(), tmp2, ck2.get(), ck.get(), cc4.get(), cc3.get(), nuniq.get(),
                                              cuda::std::plus<unsigned long long>{}, (int64_t)U, s));
      const u64 PU = d2h(nuniq.get());
      keys.resize(PU);
      cnts.resize(PU);
      GPM_CUDA(cudaMemcpyAsync(keys.data(), ck.get(), sizeof(u64) * PU, cudaMemcpyDeviceToHost, s));
      GPM_CUDA(cudaMemcpyAsync(cnts.data(), cc3.get(), sizeof(u64) * PU, cudaMemcpyDeviceToHost, s));
      sync();
    }
    trace("canon+sort", (double)U, (double)R.cap);
    // multi-GPU: all-gather every rank's (canonical key, count) list
    if (cfg.world > 1 && cfg.exchange) {
      const int W = cfg.world;
      const u64 nk = keys.size();
      std::vector<u64> lens(W, 0);
      lens[cfg.rank] = nk;
      exchange_sum_host(cfg, lens, s);
      u64 mx = *std::max_element(lens.begin(), lens.end());
      std::vector<u64> buf(2 * mx * W, 0);
      for (u64 i = 0; i < nk; ++i) {
        buf[(u64)cfg.rank * 2 * mx + i] = keys[i];
        buf[(u64)cfg.rank * 2 * mx + mx + i] = cnts[i];
      }
      exchange_sum_host(cfg, buf, s);  // disjoint slots: sum == all-gather
      keys.clear();
      cnts.clear();
      for (int r = 0; r < W; ++r)
        for (u64 i = 0; i < lens[r]; ++i) {
          keys.push_back(buf[(u64)r * 2 * mx + i]);
          cnts.push_back(buf[(u64)r * 2 * mx + mx + i]);
        }
      std::vector<size_t> ord(keys.size());
      for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
      std::sort(ord.begin(), ord.end(), [&](size_t x, size_t y) { return keys[x] < keys[y]; });
      std::vector<u64> k2, c2;
      for (size_t i : ord) {
        k2.push_back(keys[i]);
        c2.push_back(cnts[i]);
      }
      keys.swap(k2);
      cnts.swap(c2);
    }
    // reduce by canonical key (sorted; a single rank's device reduce already
    // made them unique)
    R.gkeys_h.clear();
    R.gcount_h.clear();
    if (!(cfg.world > 1 && cfg.exchange)) {
      R.gkeys_h.swap(keys);
      R.gcount_h.swap(cnts);
    }
    for (size_t i = 0; i < keys.size(); ++i) {
      if (R.gkeys_h.empty() || R.gkeys_h.back() != keys[i]) {
        R.gkeys_h.push_back(keys[i]);
        R.gcount_h.push_back(0);
      }
      R.gcount_h.back() += cnts[i];
    }
    R.P = R.gkeys_h.size();
    give_u64(keys);
    give_u64(cnts);
    trace("host reduce by key", (double)R.P);
    R.gkeys.alloc(std::max<u64>(1, R.P), s);
    if (R.P)
      GPM_CUDA(cudaMemcpyAsync(R.gkeys.get(), R.gkeys_h.data(), sizeof(u64) * R.P, cudaMemcpyHostToDevice, s));
    trace("gkeys h2d", (double)R.P);
    slot_pid_kernel<<<grid1(std::max<u64>(1, R.U)), 256, 0, s>>>(R.canon.get(), R.occ.get(), R.U, R.gkeys.get(), R.P,
                                                                 R.perm.get(), R.ent.get());
    GPM_CUDA(cudaGetLastError());
    ++tl.launches;
    trace("reduce keys + slot pids", (double)R.P, (double)R.U);
    // count pre-filter -> bitmap slots (MNI <= count)
    std::vector<u32>& bslot = host_scratch<u32, 0>();
    std::vector<u32>& bs_to_pid = host_scratch<u32, 1>();
    std::vector<u32>& sslot = host_scratch<u32, 2>();
    std::vector<u32>& sp_to_pid = host_scratch<u32, 3>();
    std::vector<u8>& need = host_scratch<u8, 0>();
    const long long PP = (long long)std::max<u64>(1, R.P);
    bslot.resize(PP);
    sslot.resize(PP);
    need.resize(PP);
    bs_to_pid.clear();
    sp_to_pid.clear();
    // MNI <= count; the full-automorphism MNI unions an orbit's domains: <= nv * count
    // (~10^6 patterns on the last level: the per-pattern host loops run on
    // the host cores, ~9 ms single-threaded on the GPU box)
    const bool full = cfg.mni_mode == GPM_MNI_AUTOMORPHISM;
    const int HT = std::max(1, std::min(host_threads(), (int)(PP >> 14) + 1));
#pragma omp parallel for num_threads(HT) schedule(static)
    for (long long p = 0; p < PP; ++p) {
      need[p] = p < (long long)R.P && App::kDomains &&
                R.gcount_h[p] * (full ? (u64)pat::code_nv(R.gkeys_h[p]) : 1) >= sigma;
      sslot[p] = ~0u;
    }
    // sparse domains: a pattern whose keys (8 B per embedding
    // vertex, x2 for the sort) cost less than its dense label-local bitmap
    // rows -- big label classes, few embeddings -- gets sorted key lists
    // instead, within half the budget (GPM_FSM_SPARSE=1: every pattern).
    // Counts, words and the budget are rank-invariant, so is the choice.
    R.skeys_total = 0;
    if (allow_sparse) {
      const bool force = std::getenv("GPM_FSM_SPARSE") != nullptr;
      const u64 words = dom_words();
      std::vector<std::pair<u64, u32>> cand;
      for (u64 p = 0; p < R.P; ++p) {
        if (!need[p]) continue;
        const u64 keyb = R.gcount_h[p] * (u64)pat::code_nv(R.gkeys_h[p]) * 16;
        if (force || keyb < (u64)kpos * words * 4) cand.emplace_back(keyb, (u32)p);
      }
      std::sort(cand.begin(), cand.end());
      u64 used = 0;
      for (auto [kb, p] : cand) {
        if (used + kb > budget / 2) break;
        used += kb;
        sslot[p] = (u32)sp_to_pid.size();
        sp_to_pid.push_back(p);
        R.skeys_total += kb / 16;
      }
    }
    // dense bitmap slots in pattern order: per-thread counts, prefix, write
    {
      std::vector<u64> part(HT + 1, 0);
#pragma omp parallel num_threads(HT)
      {
        const int t = host_thread();
        const long long b = PP * t / HT, e = PP * (t + 1) / HT;
        u64 c = 0;
        for (long long p = b; p < e; ++p) c += need[p] && sslot[p] == ~0u;
        part[t + 1] = c;
      }
      for (int t = 0; t < HT; ++t) part[t + 1] += part[t];
      bs_to_pid.resize(part[HT]);
#pragma omp parallel num_threads(HT)
      {
        const int t = host_thread();
        const long long b = PP * t / HT, e = PP * (t + 1) / HT;
        u64 o = part[t];
        for (long long p = b; p < e; ++p) {
          if (need[p] && sslot[p] == ~0u) {
            bslot[p] = (u32)o;
            bs_to_pid[o++] = (u32)p;
          } else {
            bslot[p] = ~0u;
          }
        }
      }
    }
    trace("group: host slots", (double)R.P);
    R.NB = bs_to_pid.size();
    R.NS = sp_to_pid.size();
    if (R.NS) st.paths |= GPM_PATH_FSM_SPARSE;
    R.sslot.alloc(sslot.size(), s);
    GPM_CUDA(cudaMemcpyAsync(R.sslot.get(), sslot.data(), sizeof(u32) * sslot.size(), cudaMemcpyHostToDevice, s));
    R.sp_to_pid.alloc(std::max<u64>(1, R.NS), s);
    if (R.NS)
      GPM_CUDA(cudaMemcpyAsync(R.sp_to_pid.get(), sp_to_pid.data(), sizeof(u32) * R.NS, cudaMemcpyHostToDevice, s));
    R.bslot.alloc(bslot.size(), s);
    GPM_CUDA(cudaMemcpyAsync(R.bslot.get(), bslot.data(), sizeof(u32) * bslot.size(), cudaMemcpyHostToDevice, s));
    R.bs_to_pid.alloc(std::max<u64>(1, R.NB), s);
    if (R.NB)
      GPM_CUDA(cudaMemcpyAsync(R.bs_to_pid.get(), bs_to_pid.data(), sizeof(u32) * R.NB, cudaMemcpyHostToDevice, s));
    sync();  // host vectors above are temporaries
    trace("group", (double)R.P, (double)R.NB);
  }

  // Sparse domains: one extend pass emits (slot, position, rank) keys for the
  // children of sparse patterns; sort + unique (+ all-gather across ranks)
  // give every domain exactly; MNI per slot.
  template <class SparseFn>
  void sparse_domains(Level& R, unsigned long long* mni, SparseFn&& run_sparse) {
    DBuf<u32> srep(R.NS, s);
    srep_kernel<<<grid1(R.NS), 256, 0, s>>>(R.gkeys.get(), R.sp_to_pid.get(), R.NS, LB,
                                            cfg.mni_mode == GPM_MNI_AUTOMORPHISM, srep.get());
    GPM_CUDA(cudaGetLastError());
    const u64 cap = std::max<u64>(1, R.skeys_total);
    DBuf<unsigned long long> keys(cap, s), top(1, s);
    GPM_CUDA(cudaMemsetAsync(top.get(), 0, sizeof(unsigned long long), s));
    run_sparse(keys.get(), top.get(), cap, srep.get());
    u64 nk = d2h(top.get());
    if (nk > cap) throw Error(GPM_ENOMEM, "fsm: sparse domain keys exceed the planned capacity");
    DBuf<unsigned long long> sorted(std::max<u64>(1, nk), s);
    auto sort_keys = [&](unsigned long long* in, unsigned long long* out, u64 n) {
      size_t tmp = 0;
      GPM_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, in, out, (int64_t)n, 0, 64, s));
      DBuf<u8> t(tmp, s);
      GPM_CUDA(cub::DeviceRadixSort::SortKeys(t.get(), tmp, in, out, (int64_t)n, 0, 64, s));
      tl.launches += 4;
    };
    if (nk) sort_keys(keys.get(), sorted.get(), nk);
    if (cfg.world > 1 && cfg.exchange) {
      // union over ranks: all-gather every rank's sorted keys (padded with ~0)
      const int W = cfg.world;
      std::vector<u64> lens(W, 0);
      lens[cfg.rank] = nk;
      exchange_sum_host(cfg, lens, s);
      const u64 mx = std::max<u64>(1, *std::max_element(lens.begin(), lens.end()));
      DBuf<unsigned long long> all(mx * W, s), all2(mx * W, s);
      GPM_CUDA(cudaMemsetAsync(all.get(), 0xff, sizeof(unsigned long long) * mx * W, s));
      if (nk)
        GPM_CUDA(cudaMemcpyAsync(all.get() + (u64)cfg.rank * mx, sorted.get(), sizeof(unsigned long long) * nk,
                                 cudaMemcpyDeviceToDevice, s));
      exchange_device(cfg, all.get(), mx, 8, 2, s);
      sort_keys(all.get(), all2.get(), mx * W);
      sorted = std::move(all2);
      nk = 0;
      for (u64 x : lens) nk += x;  // the ~0 padding sorts last
    }
    DBuf<unsigned long long> dcnt(R.NS * 8, s);
    GPM_CUDA(cudaMemsetAsync(dcnt.get(), 0, sizeof(unsigned long long) * R.NS * 8, s));
    if (nk) sparse_count_kernel<<<grid1(nk), 256, 0, s>>>(sorted.get(), nk, dcnt.get());
    sparse_mni_kernel<<<grid1(R.NS), 256, 0, s>>>(dcnt.get(), R.gkeys.get(), R.sp_to_pid.get(), srep.get(), R.NS, mni);
    GPM_CUDA(cudaGetLastError());
    tl.launches += 3;
    trace("sparse domains (slots, keys)", (double)R.NS, (double)nk);
  }

  // Domain pass in rounds that fit the bitmap budget; MNI; frequent flags.
  template <class DomainFn, class SparseFn>
  void domains_and_mni(Level& R, int kpos, DomainFn&& run_domain, SparseFn&& run_sparse) {
    // label-local domain bitmaps: a position's vertices all carry its label,
    // so bits are indexed by the rank within the label class (n/#labels bits
    // per position instead of n)
    const u64 words = dom_words();
    const u64 per_pat = (u64)kpos * words * 4;
    const u64 per_round = std::max<u64>(1, std::min<u64>(R.NB, budget / 2 / std::max<u64>(1, per_pat)));
    DBuf<unsigned long long> mni(std::max<u64>(1, R.P), s);
    GPM_CUDA(cudaMemsetAsync(mni.get(), 0, sizeof(unsigned long long) * std::max<u64>(1, R.P), s));
    if (per_round < R.NB) st.paths |= GPM_PATH_FSM_ROUNDS;
    if (R.NB) {
      DBuf<u32> bm(per_round * kpos * words, s);
      for (u64 lo = 0; lo < R.NB; lo += per_round) {
        const u64 n = std::min(per_round, R.NB - lo);
        GPM_CUDA(cudaMemsetAsync(bm.get(), 0, sizeof(u32) * n * kpos * words, s));
        trace("domain memset", (double)n * kpos * words * 4);
        run_domain(bm.get(), words, kpos, (u32)lo, (u32)(lo + n));
        // multi-GPU: OR the packed domain bitmaps across ranks (SURVEY §5 route ii)
        exchange_device(cfg, bm.get(), n * kpos * words, 4, 1, s);
        trace("domain round", (double)lo, (double)n);
        mni_kernel<<<(unsigned)((n + 7) / 8), 256, 0, s>>>(bm.get(), words, kpos, R.gkeys.get(), R.bs_to_pid.get(), (u32)lo,
                                               (u32)n, LB, cfg.mni_mode == GPM_MNI_AUTOMORPHISM, mni.get());
        GPM_CUDA(cudaGetLastError());
        ++tl.launches;
      }
    }
    if (R.NS) sparse_domains(R, mni.get(), run_sparse);
    give_u64(R.mni_h);
    R.mni_h = take_u64();
    R.mni_h.assign(R.P, 0);
    if (R.P)
      GPM_CUDA(cudaMemcpyAsync(R.mni_h.data(), mni.get(), sizeof(u64) * R.P, cudaMemcpyDeviceToHost, s));
    sync();
    trace("mni kernel + d2h", (double)R.P);
    std::vector<u8>& freq = R.freq_h;
    freq.assign(std::max<u64>(1, R.P), 0);
#pragma omp parallel for schedule(static)
    for (long long p = 0; p < (long long)R.P; ++p) freq[p] = frequent_pat(R, (u64)p) ? 1 : 0;
    R.frequent.alloc(freq.size(), s);
    GPM_CUDA(cudaMemcpyAsync(R.frequent.get(), freq.data(), freq.size(), cudaMemcpyHostToDevice, s));
    sync();
    trace("frequent flags h2d", (double)R.P);
  }

  // filter: keep a pattern iff !App::to_prune (Listing 5: MNI < sigma); mni_h
  // is 0 for patterns without domains (count below the MNI bound)
  bool frequent_pat(const Level& R, u64 p) const {
    PatternInfo pi{R.gkeys_h[p], R.gcount_h[p], R.mni_h[p], sigma, LB, cfg.mni_mode};
    return R.gcount_h[p] > 0 && !App::to_prune(pi);
  }

  // text is formatted on access (gpm_result_pattern): ~10^6 patterns per
  // call, recorded in parallel from the frequent flags (pattern order kept)
  void record(Level& R, int level) {
    const long long P = (long long)R.P;
    const int T = std::max(1, std::min(host_threads(), (int)(P >> 14) + 1));
    std::vector<u64> part(T + 1, 0);
#pragma omp parallel num_threads(T)
    {
      const int t = host_thread();
      const long long b = P * t / T, e = P * (t + 1) / T;
      u64 c = 0;
      for (long long p = b; p < e; ++p) c += R.freq_h[p];
      part[t + 1] = c;
    }
    for (int t = 0; t < T; ++t) part[t + 1] += part[t];
    const size_t base = res.kpatterns.size();
    res.kpatterns.resize(base + part[T]);
#pragma omp parallel num_threads(T)
    {
      const int t = host_thread();
      const long long b = P * t / T, e = P * (t + 1) / T;
      size_t o = base + part[t];
      for (long long p = b; p < e; ++p)
        if (R.freq_h[p]) {
          const PatternInfo pi{R.gkeys_h[p], R.gcount_h[p], R.mni_h[p], sigma, LB, cfg.mni_mode};
          res.kpatterns[o++] = {R.gkeys_h[p], App::support_of(pi), level};
        }
    }
  }

  FsmArgs base_args(Level& R) {
    FsmArgs a{};
    a.g = g;
    a.LB = LB;
    a.H = hash_of(R);
    a.ctr = d_ctr.get();
    return a;
  }

  // ---------------------------------------------------------- level 1
  void level1(DBuf<u32>& idx, DBuf<u32>& vid, u64& n1) {
    Level R;
    u64 cap = 1024;
    while (cap < 4 * std::min<u64>(n1, u64(1) << 22)) cap <<= 1;
    for (;;) {
      alloc_hash(R, cap);
      FsmArgs a = base_args(R);
      if (n1) {
        l1_kernel<kQC><<<grid1(n1), 256, 0, s>>>(a, idx.get(), vid.get(), n1, nullptr);
        GPM_CUDA(cudaGetLastError());
        ++tl.launches;
      }
      if (d2h(R.overflow.get()) == 0) break;
      cap <<= 3;
    }
    prev_unique = d2h(R.used.get());
    canon_and_group(R, 2, true);
    domains_and_mni(
        R, 2,
        [&](u32* bm, u64 words, int kpos, u32 lo, u32 hi) {
          FsmArgs a = base_args(R);
          a.bslot = R.bslot.get();
          a.bitmaps = bm;
          a.words = words;
          a.lrank = lrank.get();
          a.kpos = kpos;
          a.round_lo = lo;
          a.round_hi = hi;
          if (n1) {
            l1_kernel<kDomain><<<grid1(n1), 256, 0, s>>>(a, idx.get(), vid.get(), n1, nullptr);
            GPM_CUDA(cudaGetLastError());
            ++tl.launches;
          }
        },
        [&](unsigned long long* keys, unsigned long long* top, u64 scap, const u32* srep) {
          FsmArgs a = base_args(R);
          a.lrank = lrank.get();
          a.sslot = R.sslot.get();
          a.srep = srep;
          a.skeys = keys;
          a.stop = top;
          a.scap = scap;
          if (n1) {
            l1_kernel<kSparse><<<grid1(n1), 256, 0, s>>>(a, idx.get(), vid.get(), n1, nullptr);
            GPM_CUDA(cudaGetLastError());
            ++tl.launches;
          }
        });
    record(R, 1);
    // filter: keep entries whose pattern is frequent
    if (!n1) return;
    DBuf<u8> keep(n1, s);
    {
      FsmArgs a = base_args(R);
      a.frequent = R.frequent.get();
      l1_kernel<kSCount><<<grid1(n1), 256, 0, s>>>(a, idx.get(), vid.get(), n1, keep.get());
      GPM_CUDA(cudaGetLastError());
      ++tl.launches;
    }
    DBuf<u32> ni(n1, s), nvv(n1, s);
    DBuf<u64> nsel(1, s);
    size_t tmp = 0;
    GPM_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, idx.get(), keep.get(), ni.get(), nsel.get(), (int64_t)n1, s));
    DBuf<u8> t(tmp, s);
    GPM_CUDA(cub::DeviceSelect::Flagged(t.get(), tmp, idx.get(), keep.get(), ni.get(), nsel.get(), (int64_t)n1, s));
    GPM_CUDA(cub::DeviceSelect::Flagged(t.get(), tmp, vid.get(), keep.get(), nvv.get(), nsel.get(), (int64_t)n1, s));
    n1 = d2h(nsel.get());
    idx = std::move(ni);
    vid = std::move(nvv);
    st.survivors[0] = n1;
  }

  // ---------------------------------------------------------- extend levels
  template <int LEV>
  void launch(FsmArgs& a, int mode, const char* name, double bytes) {
    void (*kern)(FsmArgs) = nullptr;
    switch (mode) {
      case kQC: kern = eextend_kernel<App, LEV, kQC>; break;
      case kDomain: kern = eextend_kernel<App, LEV, kDomain>; break;
      case kSCount: kern = eextend_kernel<App, LEV, kSCount>; break;
      case kSparse: kern = eextend_kernel<App, LEV, kSparse>; break;
      default: kern = eextend_kernel<App, LEV, kSWrite>; break;
    }
    int occ = 0;
    GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, 0));
    occ = std::max(1, occ);
    const u64 nb = a.b_end - a.b_begin;
    u64 blocks = std::max<u64>(1, std::min<u64>((u64)sms * occ, (nb * 32 + kThreads - 1) / kThreads));
    a.grab = std::max<u64>(1, std::min<u64>(4, nb / (blocks * (kThreads / 32) * 64)));
    GPM_CUDA(cudaMemsetAsync(d_ctr.get(), 0, sizeof(unsigned long long), s));
    size_t ev = tl.begin(std::string(name) + "_L" + std::to_string(LEV), bytes);
    kern<<<(unsigned)blocks, kThreads, 0, s>>>(a);
    GPM_CUDA(cudaGetLastError());
    tl.end(ev);
    ++tl.launches;
  }

  // ---------------------------------------------------------- grouped passes
  struct Groups {
    DBuf<u64> items;
    u64 nitems = 0;
    bool on = false;
  };

  // Sorts the compacted parents by a hash of their quick code (24-bit radix
  // sort of (key, parent)) so that each item of the candidate space holds the
  // children of a few parent codes.
  template <int LEV>
  void sort_parents(const ELevels& L, DBuf<u32>& pidx, u64 nz, DBuf<u32>& keys) {
    keys.alloc(nz, s);
    pkey_kernel<LEV><<<grid1(nz), 256, 0, s>>>(g, L, pidx.get(), nz, LB, keys.get());
    GPM_CUDA(cudaGetLastError());
    DBuf<u32> k2(nz, s), p2(nz, s);
    size_t tmp = 0;
    GPM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys.get(), k2.get(), pidx.get(), p2.get(), (int64_t)nz, 0,
                                             24, s));
    DBuf<u8> t(tmp, s);
    GPM_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, keys.get(), k2.get(), pidx.get(), p2.get(), (int64_t)nz, 0,
                                             24, s));
    tl.launches += 5;
    keys = std::move(k2);
    pidx = std::move(p2);
  }

  // Items over the sorted candidate space [0, W): each parent group is one
  // item, consecutive small groups are merged up to kMinItem candidates and
  // large groups split into kMaxItem pieces.
  void build_items(const DBuf<u32>& keys, u64 nz, const DBuf<u64>& Wp, u64 W, Groups& gr) {
    constexpr u64 kMinItem = u64(1) << 16, kMaxItem = u64(1) << 21;
    DBuf<u8> flag(nz, s);
    gstart_kernel<<<grid1(nz), 256, 0, s>>>(keys.get(), nz, flag.get());
    DBuf<u32> starts(nz, s);
    DBuf<u64> ng(1, s);
    size_t tmp = 0;
    thrust::counting_iterator<u32> it(0);
    GPM_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, flag.get(), starts.get(), ng.get(), (int64_t)nz, s));
    DBuf<u8> t(tmp, s);
    GPM_CUDA(cub::DeviceSelect::Flagged(t.get(), tmp, it, flag.get(), starts.get(), ng.get(), (int64_t)nz, s));
    const u64 G = d2h(ng.get());
    DBuf<u64> gw(G, s);
    gather_starts_kernel<<<grid1(G), 256, 0, s>>>(Wp.get(), starts.get(), G, gw.get());
    GPM_CUDA(cudaGetLastError());
    tl.launches += 4;
    std::vector<u64> gs(G);
    GPM_CUDA(cudaMemcpyAsync(gs.data(), gw.get(), sizeof(u64) * G, cudaMemcpyDeviceToHost, s));
    sync();
    std::vector<u64> b{0};
    for (u64 i = 0; i < G; ++i) {
      const u64 a0 = gs[i], a1 = i + 1 < G ? gs[i + 1] : W;
      if (a1 - a0 > kMaxItem) {
        if (b.back() < a0) b.push_back(a0);
        const u64 np_ = (a1 - a0 + kMaxItem - 1) / kMaxItem;
        for (u64 q = 1; q < np_; ++q) b.push_back(a0 + (a1 - a0) * q / np_);
        b.push_back(a1);
      } else if (a1 - b.back() >= kMinItem) {
        b.push_back(a1);
      }
    }
    if (b.back() < W) b.push_back(W);
    gr.nitems = b.size() - 1;
    gr.items.alloc(b.size(), s);
    GPM_CUDA(cudaMemcpyAsync(gr.items.get(), b.data(), sizeof(u64) * b.size(), cudaMemcpyHostToDevice, s));
    sync();
    trace("groups -> items", (double)G, (double)gr.nitems);
  }

  // shared-memory geometry of a grouped pass; false = does not fit (the
  // ungrouped kernels run instead)
  bool group_geometry(int mode, int kpos, u64 words, GroupArgs& ga, size_t& smem) {
    int maxs = 0;
    GPM_CUDA(cudaDeviceGetAttribute(&maxs, cudaDevAttrMaxSharedMemoryPerBlockOptin, G.device));
    const size_t avail = (size_t)maxs - 1024;  // static shared + slack
    u32 cs = 1024;
    if (mode != kQC) {
      const size_t per = (size_t)kpos * words * 4 + 20 + 24;  // rows + sinfo/skey/sid + 2 map entries
      cs = (u32)std::min<size_t>(256, avail / per) & ~7u;
      if (cs < 16) return false;
    }
    u32 mc = 64;
    while (mc < 2 * cs) mc <<= 1;
    ga.mcap = mc;
    ga.cslots = cs;
    auto bytes = [&](u32 c, u32 m) {
      return (size_t)m * 12 + (size_t)c * 20 + (mode != kQC ? (size_t)c * kpos * words * 4 : 0);
    };
    while (bytes(cs, mc) > avail && cs > 16) {
      cs -= 8;
      mc = 64;
      while (mc < 2 * cs) mc <<= 1;
    }
    ga.mcap = mc;
    ga.cslots = cs;
    smem = bytes(cs, mc);
    return smem <= avail;
  }

  template <int LEV>
  void launch_group(FsmArgs& a, const Groups& gr, int mode, const char* name, double bytes) {
    if constexpr (!App::kBuiltin) {
      throw Error(GPM_EINVAL, "fsm: grouped passes are builtin-only");
    } else {
    GroupArgs ga{};
    size_t smem = 0;
    if (!group_geometry(mode, a.kpos, a.words, ga, smem)) throw Error(GPM_EINVAL, "fsm: grouped pass does not fit");
    ga.items = gr.items.get();
    ga.nitems = gr.nitems;
    ga.ctr = d_ctr.get();
    auto kern = mode == kQC ? egroup_kernel<LEV, kQC> : mode == kQCD ? egroup_kernel<LEV, kQCD> : egroup_kernel<LEV, kDomain>;
    GPM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int occ = 0;
    GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kGT, smem));
    occ = std::max(1, occ);
    const u64 blocks = std::max<u64>(1, std::min<u64>((u64)sms * occ, gr.nitems));
    GPM_CUDA(cudaMemsetAsync(d_ctr.get(), 0, sizeof(unsigned long long), s));
    st.paths |= GPM_PATH_FSM_GROUPED;
    size_t ev = tl.begin(std::string(name) + "_L" + std::to_string(LEV), bytes);
    kern<<<(unsigned)blocks, kGT, smem, s>>>(a, ga);
    GPM_CUDA(cudaGetLastError());
    tl.end(ev);
    ++tl.launches;
    }
  }

  // ---------------------------------------------------------- fan-out pass (last level)
  size_t fan_smem(int LEVv, int kpos, u64 words, int ft = kFT) const {
    const u64 nslot = (u64(1) << LB) + LEVv + 1;
    const u64 desc = (u64)(ft / 32) * (8 * 32 * (2 + 2 * LEVv + 1) + 4 * 32 * (3 + 2 * (LEVv + 1))) + 64;
    return (size_t)(4 * (nslot * kpos * words + 2 * nslot + 2) + desc);
  }
  bool fan_fits(int LEVv, int kpos, u64 words) const {
    if (LB > 5 || !labrank.get() || max_class >= (u64(1) << kRankBits)) return false;  // label slots = lanes
    int maxs = 0;
    GPM_CUDA(cudaDeviceGetAttribute(&maxs, cudaDevAttrMaxSharedMemoryPerBlockOptin, G.device));
    return fan_smem(LEVv, kpos, words) + 1024 <= (size_t)maxs;
  }

  // compacted parents sorted by their exact quick code; codes sorted alongside
  template <int LEV>
  void sort_parents_exact(const ELevels& L, DBuf<u32>& pidx, u64 nz, DBuf<u64>& codes) {
    codes.alloc(nz, s);
    pcode_kernel<LEV><<<grid1(nz), 256, 0, s>>>(g, L, pidx.get(), nz, LB, codes.get());
    GPM_CUDA(cudaGetLastError());
    // a parent has LEV edges, so <= LEV + 1 vertices: its code below bit 60
    // fits npairs + nv x LB bits; with the nv nibble rotated to the bottom the
    // sort needs 4 + that many bits (FSM17 level 2: 22 instead of 64)
    const int nvmax = LEV + 1;
    const int bits = std::min(64, 4 + pat::npairs(nvmax) + nvmax * LB);
    rotl4_kernel<<<grid1(nz), 256, 0, s>>>(codes.get(), nz, 1);
    DBuf<u64> k2(nz, s);
    DBuf<u32> p2(nz, s);
    size_t tmp = 0;
    GPM_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, codes.get(), k2.get(), pidx.get(), p2.get(), (int64_t)nz, 0,
                                             bits, s));
    DBuf<u8> t(tmp, s);
    GPM_CUDA(cub::DeviceRadixSort::SortPairs(t.get(), tmp, codes.get(), k2.get(), pidx.get(), p2.get(), (int64_t)nz, 0,
                                             bits, s));
    rotl4_kernel<<<grid1(nz), 256, 0, s>>>(k2.get(), nz, 0);
    GPM_CUDA(cudaGetLastError());
    tl.launches += 11;
    codes = std::move(k2);
    pidx = std::move(p2);
  }

  // items: (parent code group, extended position q, <= kFanParents parents)
  void build_fan_items(const DBuf<u64>& codes, u64 nz, DBuf<FanItem>& items, u64& nitems) {
    DBuf<u8> flag(nz, s);
    gstart64_kernel<<<grid1(nz), 256, 0, s>>>(codes.get(), nz, flag.get());
    DBuf<u32> starts(nz, s);
    DBuf<u64> ng(1, s);
    size_t tmp = 0;
    thrust::counting_iterator<u32> it(0);
    GPM_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, flag.get(), starts.get(), ng.get(), (int64_t)nz, s));
    DBuf<u8> t(tmp, s);
    GPM_CUDA(cub::DeviceSelect::Flagged(t.get(), tmp, it, flag.get(), starts.get(), ng.get(), (int64_t)nz, s));
    const u64 G_ = d2h(ng.get());
    DBuf<u64> gc(std::max<u64>(1, G_), s);
    gather_codes_kernel<<<grid1(std::max<u64>(1, G_)), 256, 0, s>>>(codes.get(), starts.get(), G_, gc.get());
    GPM_CUDA(cudaGetLastError());
    tl.launches += 4;
    std::vector<u32> hs(G_);
    std::vector<u64> hc(G_);
    GPM_CUDA(cudaMemcpyAsync(hs.data(), starts.get(), sizeof(u32) * G_, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaMemcpyAsync(hc.data(), gc.get(), sizeof(u64) * G_, cudaMemcpyDeviceToHost, s));
    sync();
    trace("fan group starts d2h", (double)G_);
    // items, large first (tail balance): a stable counting sort by size
    // (sizes are 1..kFanParents), O(items) instead of a comparison sort
    std::vector<u64> bucket(kFanParents + 2, 0);
    u64 ntot = 0;
    for (u64 i = 0; i < G_; ++i) {
      const u32 a0 = hs[i], a1 = i + 1 < G_ ? hs[i + 1] : (u32)nz;
      const int nvv = pat::code_nv(hc[i]);
      for (u32 b = a0; b < a1; b += kFanParents) {
        bucket[kFanParents - std::min<u32>(a1 - b, kFanParents)] += (u64)nvv;
        ntot += (u64)nvv;
      }
    }
    u64 acc = 0;
    for (auto& x : bucket) {
      const u64 c = x;
      x = acc;
      acc += c;
    }
    std::vector<FanItem>& v = host_scratch<FanItem, 0>();
    v.resize(ntot);  // every element is written below
    for (u64 i = 0; i < G_; ++i) {
      const u32 a0 = hs[i], a1 = i + 1 < G_ ? hs[i + 1] : (u32)nz;
      const int nvv = pat::code_nv(hc[i]);
      for (int q = 0; q < nvv; ++q)
        for (u32 b = a0; b < a1; b += kFanParents) {
          const u32 e = std::min<u32>(a1, b + kFanParents);
          v[bucket[kFanParents - (e - b)]++] = FanItem{hc[i], b, e, (u32)q, 0};
        }
    }
    trace("fan items host sort", (double)v.size());
    nitems = v.size();
    items.alloc(std::max<u64>(1, nitems), s);
    if (nitems) GPM_CUDA(cudaMemcpyAsync(items.get(), v.data(), sizeof(FanItem) * nitems, cudaMemcpyHostToDevice, s));
    sync();
    trace("fan groups -> items", (double)G_, (double)nitems);
  }

  template <int LEV>
  void launch_fan(FsmArgs& a, const DBuf<FanItem>& items, u64 nitems, const char* name, double bytes) {
    if constexpr (!App::kBuiltin) {
      throw Error(GPM_EINVAL, "fsm: the fan pass is builtin-only");
    } else {
    FanArgs fa{};
    fa.items = items.get();
    fa.nitems = nitems;
    fa.ctr = d_ctr.get();
    fa.nl = 1u << LB;
    // wide CTAs when two of them fit an SM, else the 8-warp CTA
    size_t smem = fan_smem(LEV, a.kpos, a.words, kFTWide);
    auto kern = efan_kernel<LEV, kFTWide>;
    int ft = kFTWide, occ = 0, maxs = 0;
    GPM_CUDA(cudaDeviceGetAttribute(&maxs, cudaDevAttrMaxSharedMemoryPerBlockOptin, G.device));
    if (smem + 1024 <= (size_t)maxs && !std::getenv("GPM_FSM_FAN_NARROW")) {
      GPM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFTWide, smem));
    }
    if (occ < 2) {
      smem = fan_smem(LEV, a.kpos, a.words, kFT);
      kern = efan_kernel<LEV, kFT>;
      ft = kFT;
      GPM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFT, smem));
    }
    occ = std::max(1, occ);
    const u64 blocks = std::max<u64>(1, std::min<u64>((u64)sms * occ, nitems));
    GPM_CUDA(cudaMemsetAsync(d_ctr.get(), 0, sizeof(unsigned long long), s));
    st.paths |= GPM_PATH_FSM_FAN;
    size_t ev = tl.begin(std::string(name) + "_L" + std::to_string(LEV), bytes);
    kern<<<(unsigned)blocks, ft, smem, s>>>(a, fa);
    GPM_CUDA(cudaGetLastError());
    tl.end(ev);
    ++tl.launches;
    }
  }

  // Extends level LEV (np parents) -> reduce (+ filter into out arrays unless last)
  template <int LEV>
  void extend_level(const ELevels& L, u64 np, bool last, DBuf<u32>& oi, DBuf<u32>& ov, DBuf<u8>& oh, u64& nout) {
    nout = 0;
    // work + compaction + scan
    DBuf<u64> w(std::max<u64>(1, np), s);
    DBuf<unsigned long long> nvsum(1, s);
    GPM_CUDA(cudaMemsetAsync(nvsum.get(), 0, sizeof(unsigned long long), s));
    if (np) {
      ework_kernel<App, LEV><<<grid1(np), kThreads, 0, s>>>(g, L, np, w.get(), nvsum.get());
      GPM_CUDA(cudaGetLastError());
      ++tl.launches;
    }
    DBuf<u32> pidx(std::max<u64>(1, np), s);
    DBuf<u64> nsel(1, s);
    u64 nz = 0;
    if (np) {
      size_t tmp = 0;
      thrust::counting_iterator<u32> it(0);
      GPM_CUDA(cub::DeviceSelect::If(nullptr, tmp, it, pidx.get(), nsel.get(), (int64_t)np, NonZeroW{w.get()}, s));
      DBuf<u8> t(tmp, s);
      GPM_CUDA(cub::DeviceSelect::If(t.get(), tmp, it, pidx.get(), nsel.get(), (int64_t)np, NonZeroW{w.get()}, s));
      nz = d2h(nsel.get());
    }
    // grouped passes: parents sorted by quick code
    Groups gr;
    DBuf<u32> gkeys_sorted;
    // fused last level: the fan-out pass over parents grouped by exact code
    // (the grouped and fan passes inline the builtin to_add_edge: builtin FSM only)
    const bool fan_ok = App::kBuiltin && last && nz && !std::getenv("GPM_FSM_NOFAN") &&
                        !std::getenv("GPM_FSM_TWO_PASS") && fan_fits(LEV, LEV + 2, dom_words());
    {
      GroupArgs probe{};
      size_t sm = 0;
      gr.on = App::kBuiltin && nz && !fan_ok && !std::getenv("GPM_FSM_UNGROUPED") &&
              group_geometry(kDomain, LEV + 2, dom_words(), probe, sm);
    }
    if (gr.on) sort_parents<LEV>(L, pidx, nz, gkeys_sorted);
    DBuf<u64> Wp(nz + 1, s);
    GPM_CUDA(cudaMemsetAsync(Wp.get() + nz, 0, sizeof(u64), s));
    if (nz) {
      egather_kernel<<<grid1(nz), 256, 0, s>>>(w.get(), pidx.get(), nz, Wp.get());
      GPM_CUDA(cudaGetLastError());
      ++tl.launches;
    }
    scan_inplace(Wp.get(), nz + 1, s);
    const u64 W = d2h(Wp.get() + nz);
    const u64 nvs = d2h(nvsum.get());
    if (gr.on && W) build_items(gkeys_sorted, nz, Wp, W, gr);
    gkeys_sorted.release();
    st.candidates[LEV] += W;
    const double bytes_in = 8.0 * LEV * np + 16.0 * nvs + 4.0 * W;
    st.balg += bytes_in;
    const u64 nb = (W + kBatch - 1) / kBatch;

    Level R;
    DBuf<unsigned long long> accepted(1, s);
    auto args = [&](Level& RR) {
      FsmArgs a = base_args(RR);
      a.L = L;
      a.Wp = Wp.get();
      a.pidx = pidx.get();
      a.np = nz;
      a.W = W;
      a.B = kBatch;
      a.b_begin = 0;
      a.b_end = nb;
      a.accepted = accepted.get();
      return a;
    };
    // first guess: previous level's distinct quick codes x fan-out, grown x8 on overflow
    // distinct quick codes <= accepted <= candidates W: size for 2 W (capped at
    // 2^26 entries = 1 GB) so the pass rarely has to regrow and re-run
    // A child's quick code is a function of (parent quick code, extended
    // position, new vertex label | closing position), so the level has at most
    // prev_unique x (LEV + 1) x (2^LB + LEV + 1) distinct codes: a table of
    // twice that never overflows (load <= 1/2) and is 4-250x smaller than the
    // 2 W guess, i.e. mostly L2-resident probes instead of DRAM ones.
    const u64 fan = (u64)(LEV + 1) * ((u64(1) << LB) + LEV + 1);
    const u64 bound = prev_unique > (u64(1) << 40) / fan ? (u64(1) << 40) : prev_unique * fan;
    u64 want = std::min<u64>(u64(1) << 26, std::max<u64>(2 * W, 64 * prev_unique));
    want = std::min<u64>(want, 2 * bound + 2);
    u64 cap = 1u << 16;
    while (cap < want) cap <<= 1;
    // Last level: fuse the domain pass into pass A.  Children OR their vertices
    // into per-quick-code bitmaps (label-local, quick positions); after
    // canonicalisation these are merged into the canonical patterns' bitmaps
    // through the PositionMaps, so the level is extended once, not twice.
    const int kposL = LEV + 2;
    const u64 wordsL = dom_words();
    const u64 per_id = (u64)kposL * wordsL * 4;
    DBuf<u32> qbm;
    DBuf<int> qover(1, s);
    u64 qcap = 0;
    if (App::kDomains && last && nb && !std::getenv("GPM_FSM_TWO_PASS")) {
      qcap = std::min<u64>(cap / 2, budget / 2 / std::max<u64>(1, per_id));
      if (qcap >= 1024) qbm.alloc(qcap * kposL * wordsL, s);
      else qcap = 0;
    }
    DBuf<FanItem> fitems;
    u64 nfan = 0;
    const bool use_fan = fan_ok && qcap && nb;
    trace("qbm alloc", (double)qcap);
    if (use_fan) {
      DBuf<u64> pcodes;
      sort_parents_exact<LEV>(L, pidx, nz, pcodes);
      trace("sort parents", (double)nz);
      // Wp in the new parent order (the unfused fallback passes read it)
      egather_kernel<<<grid1(nz), 256, 0, s>>>(w.get(), pidx.get(), nz, Wp.get());
      GPM_CUDA(cudaGetLastError());
      ++tl.launches;
      GPM_CUDA(cudaMemsetAsync(Wp.get() + nz, 0, sizeof(u64), s));
      scan_inplace(Wp.get(), nz + 1, s);
      trace("egather + scan", (double)nz);
      build_fan_items(pcodes, nz, fitems, nfan);
    }
    for (;;) {
      alloc_hash(R, cap);
      GPM_CUDA(cudaMemsetAsync(accepted.get(), 0, sizeof(unsigned long long), s));
      GPM_CUDA(cudaMemsetAsync(qover.get(), 0, sizeof(int), s));
      if (qcap) GPM_CUDA(cudaMemsetAsync(qbm.get(), 0, sizeof(u32) * qcap * kposL * wordsL, s));
      if (nb) {
        FsmArgs a = args(R);
        if (qcap) {
          a.qbm = qbm.get();
          a.qcap = qcap;
          a.qover = qover.get();
          a.kpos = kposL;
          a.words = wordsL;
          a.lrank = lrank.get();
        }
        a.labrank = labrank.get();
        if (use_fan) launch_fan<LEV>(a, fitems, nfan, "fsm_fan_qc_domain", bytes_in);
        else if (gr.on) launch_group<LEV>(a, gr, qcap ? kQCD : kQC, qcap ? "fsm_group_qc_domain" : "fsm_group_qc", bytes_in);
        else launch<LEV>(a, kQC, qcap ? "fsm_extend_qc_domain" : "fsm_extend_qc", bytes_in);
      }
      if (d2h(R.overflow.get()) == 0) break;
      cap <<= 3;
    }
    const bool fused = qcap && d2h(qover.get()) == 0;
    if (fused) st.paths |= GPM_PATH_FSM_FUSED_LAST;
    if (!fused) qbm.release();  // more quick codes than bitmaps: separate domain pass
    trace(fused ? "pass A fused (qcap, ids)" : "pass A unfused (qcap, ids)", (double)qcap, (double)d2h(R.used.get()));
    u64 acc = d2h(accepted.get());
    prev_unique = d2h(R.used.get());
    trace("pass A (qc)", (double)acc, (double)R.cap);
    if (cfg.world > 1 && cfg.exchange) {
      std::vector<u64> v{acc};
      exchange_sum_host(cfg, v, s);
      acc = v[0];
    }
    st.level_sizes[LEV] += acc;
    canon_and_group(R, LEV + 2, !fused);
    domains_and_mni(R, LEV + 2, [&](u32* bm, u64 words, int kpos, u32 lo, u32 hi) {
      if (!nb) return;
      if (fused) {
        merge_qbm_kernel<<<grid1(std::max<u64>(1, R.U) * 32), 256, 0, s>>>(qbm.get(), R.canon.get(), R.ids.get(), R.perm.get(), R.U,
                                                           R.ent.get(), R.occ.get(), R.bslot.get(), lo, hi, bm, words, kpos);
        GPM_CUDA(cudaGetLastError());
        ++tl.launches;
        return;
      }
      FsmArgs a = args(R);
      a.bslot = R.bslot.get();
      a.bitmaps = bm;
      a.words = words;
      a.lrank = lrank.get();
      a.kpos = kpos;
      a.round_lo = lo;
      a.round_hi = hi;
      if (gr.on) launch_group<LEV>(a, gr, kDomain, "fsm_group_domain", bytes_in);
      else launch<LEV>(a, kDomain, "fsm_extend_domain", bytes_in);
    }, [&](unsigned long long* keys, unsigned long long* top, u64 scap, const u32* srep) {
      if (!nb) return;
      FsmArgs a = args(R);
      a.lrank = lrank.get();
      a.sslot = R.sslot.get();
      a.srep = srep;
      a.skeys = keys;
      a.stop = top;
      a.scap = scap;
      launch<LEV>(a, kSparse, "fsm_extend_sparse", bytes_in);
    });
    trace("mni done", (double)R.P);
    record(R, LEV + 1);
    trace("mni+record", (double)R.P);
    if (last || !nb) return;
    // filter + write survivors (inspection-execution)
    DBuf<u64> cnt(nb + 1, s);
    GPM_CUDA(cudaMemsetAsync(cnt.get() + nb, 0, sizeof(u64), s));
    {
      FsmArgs a = args(R);
      a.frequent = R.frequent.get();
      a.cnt = cnt.get();
      launch<LEV>(a, kSCount, "fsm_extend_filter_count", bytes_in);
    }
    scan_inplace(cnt.get(), nb + 1, s);
    const u64 T = d2h(cnt.get() + nb);
    if (T >= (u64(1) << 32)) throw Error(GPM_ENOMEM, "fsm level exceeds 2^32 embeddings");
    nout = T;
    oi.alloc(std::max<u64>(1, T), s);
    ov.alloc(std::max<u64>(1, T), s);
    oh.alloc(std::max<u64>(1, T), s);
    if (T) {
      FsmArgs a = args(R);
      a.frequent = R.frequent.get();
      a.boffs = cnt.get();
      a.out_base = 0;
      a.out_idx = oi.get();
      a.out_vid = ov.get();
      a.out_his = oh.get();
      launch<LEV>(a, kSWrite, "fsm_extend_filter_write", bytes_in + 9.0 * T);
    }
    st.survivors[LEV] = T;
    st.balg += 9.0 * T;
  }

  void run() {
    k = cfg.k;
    sigma = cfg.min_support;
    if (!G.labeled) throw Error(GPM_EINVAL, "fsm: graph is unlabeled");
    if (G.oriented) throw Error(GPM_EINVAL, "fsm: graph must be undirected");
    if (k < 2 || k > kMaxEdges + 1) throw Error(GPM_EINVAL, "fsm: k must be in [2,6]");
    LB = std::max(1, G.label_bits);
    if (pat::code_bits(k, LB) > pat::kCodeBits)
      throw Error(GPM_EINVAL, "fsm: too many distinct labels for a packed pattern code at this k");
    sms = sm_count();
    const size_t freeb = device_free_bytes();
    budget = cfg.mem_budget ? cfg.mem_budget : (u64)(0.5 * (double)freeb);
    // the bitmap rounds (one OR collective each) and the fused/two-pass
    // choice follow from the budget: every rank must plan with the same one
    budget = exchange_min_host(cfg, budget, s);
    d_ctr.alloc(1, s);
    label_ranks();
    const int levels = k - 1;
    st.ensure(levels);
    DBuf<u32> l1i, l1v;
    u64 n1 = 0;
    build_level1(G, l1i, l1v, n1, s, tl);
    u64 lo = 0, hi = n1;
    if (cfg.root_hi > 0) {
      lo = std::min(cfg.root_lo, n1);
      hi = std::max(lo, std::min(cfg.root_hi, n1));
    } else {
      root_split(G, l1i.get(), l1v.get(), n1, GPM_APP_MC, cfg.rank, std::max(1, cfg.world), lo, hi, s, tl);
    }
    // slice level 1 into owned arrays
    u64 nr = hi - lo;
    {
      DBuf<u32> a(std::max<u64>(1, nr), s), b(std::max<u64>(1, nr), s);
      if (nr) {
        GPM_CUDA(cudaMemcpyAsync(a.get(), l1i.get() + lo, sizeof(u32) * nr, cudaMemcpyDeviceToDevice, s));
        GPM_CUDA(cudaMemcpyAsync(b.get(), l1v.get() + lo, sizeof(u32) * nr, cudaMemcpyDeviceToDevice, s));
      }
      l1i = std::move(a);
      l1v = std::move(b);
    }
    u64 nl1 = nr;
    if (cfg.world > 1 && cfg.exchange) {
      std::vector<u64> v{nr};
      exchange_sum_host(cfg, v, s);
      nl1 = v[0];
    }
    st.level_sizes[0] = nl1;
    level1(l1i, l1v, nr);
    DBuf<u8> l1h(std::max<u64>(1, nr), s);
    GPM_CUDA(cudaMemsetAsync(l1h.get(), 0, std::max<u64>(1, nr), s));
    std::vector<DBuf<u32>> li(levels), lv(levels);
    std::vector<DBuf<u8>> lh(levels);
    li[0] = std::move(l1i);
    lv[0] = std::move(l1v);
    lh[0] = std::move(l1h);
    u64 np = nr;
    ELevels L{};
    for (int lev = 1; lev <= levels - 1; ++lev) {
      L.idx[lev - 1] = li[lev - 1].get();
      L.vid[lev - 1] = lv[lev - 1].get();
      L.his[lev - 1] = lh[lev - 1].get();
      const bool last = (lev == levels - 1);
      u64 nout = 0;
      switch (lev) {
        case 1: extend_level<1>(L, np, last, li[lev], lv[lev], lh[lev], nout); break;
        case 2: extend_level<2>(L, np, last, li[lev], lv[lev], lh[lev], nout); break;
        case 3: extend_level<3>(L, np, last, li[lev], lv[lev], lh[lev], nout); break;
        case 4: extend_level<4>(L, np, last, li[lev], lv[lev], lh[lev], nout); break;
        default: throw Error(GPM_EINVAL, "fsm: level out of range");
      }
      np = nout;
    }
    if (cfg.world > 1 && cfg.exchange) {
      // level sizes except the already-reduced accepted counts: survivors per rank
      std::vector<u64> v(st.survivors.begin(), st.survivors.end());
      std::vector<u64> c(st.candidates.begin(), st.candidates.end());
      v.insert(v.end(), c.begin(), c.end());
      v.push_back((u64)st.balg);
      exchange_sum_host(cfg, v, s);
      const size_t L2 = st.survivors.size();
      for (size_t i = 0; i < L2; ++i) st.survivors[i] = v[i];
      for (size_t i = 0; i < st.candidates.size(); ++i) st.candidates[i] = v[L2 + i];
      st.balg = (double)v.back();
    }
    // (level, support desc, canonical key): integer compares only
    // ~10^6 records: libstdc++'s OpenMP parallel sort on the host cores
    __gnu_parallel::sort(res.kpatterns.begin(), res.kpatterns.end(),
                         [](const gpm_result::KeyPattern& x, const gpm_result::KeyPattern& y) {
      if (x.level != y.level) return x.level < y.level;
      if (x.support != y.support) return x.support > y.support;
      return x.key < y.key;
    });
    res.label_bits = LB;
    res.label_values = G.label_values;
  }
};

}  // namespace

// mine() for an edge-mode App (FSM and user apps on the same engine).
template <class App>
void mine_edges(const gpm_graph& g, const gpm_config& cfg, cudaStream_t s, gpm_result& res, Stats& st, Timeline& tl) {
  Fsm<App> f(g, cfg, s, st, tl, res);
  f.run();
}

}  // namespace fsm_engine
}  // namespace gpm
