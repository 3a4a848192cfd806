// vertex.cu — vertex-induced extend-reduce engine for TC, CF (k-clique) and
// MC (k-motif) on sm_100a.
//
// Reference: Alg. 1 / Alg. 2, engine module SPEC.md:344-379,
// apps, Listings 3/4/6.
//
// Design (B200-first):
//  * Levels are SoA (idx u32, vid u32) in HBM (Fig. 7, embedding_list.hpp:19-40);
//    level 1 is the CSR edge range (DAG edges or u<v pairs).
//  * Work is balanced over CANDIDATES, not parents: a work pass computes, per
//    parent, w = sum of deg over positions passing to_extend; an exclusive scan
//    gives the candidate space [0, W).  The space is cut into fixed batches of
//    B candidates; a persistent grid of warps pulls batches from an atomic
//    counter.  Each lane owns one candidate per step (coalesced neighbour-list
//    reads), locates its parent by binary search over the work prefix, and
//    evaluates to_add with binary-search probes (§5.4).  Power-law hubs
//    are split across many warps; tiny parents pack 32 candidates per step.
//  * Inspection-execution: COUNT writes accepted children
//    per batch, a device scan gives batch offsets, WRITE re-walks the batch and
//    writes idx/vid at offset + warp-ballot rank: no atomics on the store, and
//    the output order is exactly the sequential (parent, pos, neighbour) order.
//  * The last level is never materialised ("reduce only on the
//    last iteration" + loop fusion §5.2): FUSED counts (TC/CF) or classifies by
//    connectivity code with warp-aggregated (__match_any_sync) shared-memory
//    atomics (MC, Listing 6 / Fig. 6).
//  * A planner splits a level whose children exceed the memory budget (or
//    2^32-1 entries, the u32 idx limit of embedding_list.hpp:20) into batch
//    ranges processed depth-first: generalised edge blocking.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>

#include "engine.hpp"
#include "pattern.cuh"

namespace gpm {

void scan_inplace(u64* data, u64 n, cudaStream_t s);

namespace {

enum { kAppTC = 0, kAppCF = 1, kAppMC = 2 };
enum { kCount = 1, kWrite = 2, kFused = 3 };

constexpr int kThreads = 256;
constexpr u64 kBatch = 2048;  // candidates per warp batch

constexpr u64 kItemGrab = 8;        // root-kernel work items per atomic grab
constexpr u64 kBatchGrab = 4;       // generic-engine batches per atomic grab
constexpr u32 kHashSlots = 1024;    // per-warp exact hash set of the root's out-list (4 KB)
constexpr u32 kFilterMax = 512;     // out-lists longer than this are probed by binary search
constexpr u64 kMaskChunk = 4096;    // ballot-mask words a warp reserves at a time
constexpr u32 kSparseWords = 64;    // accepted (parent, u) children recorded per CF item

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

struct ExtendArgs {
  DevGraph g;
  VLevels L;
  const u64* Wp;   // exclusive work prefix over compacted parents, np+1 entries
  const u32* pidx; // compacted parent -> level index
  // CF/TC on a DAG: per compacted parent, candidate-list begin and packed probe
  // lists (begin | deg << 40) of emb[0..S-2]; replaces the reconstruct chain
  const u64* dcbeg;
  const u64* dq[kMaxLevels];
  u64 np, W, B;    // np = number of parents with non-zero work
  u64 b_begin, b_end;
  u64 grab;          // batches per atomic grab
  unsigned long long* ctr;
  u64* cnt;          // COUNT: accepted per batch (index b - b_begin)
  const u64* boffs;  // WRITE: exclusive offsets per batch (absolute b)
  u64 out_base;
  u32* out_idx;
  u32* out_vid;
  u32* masks;        // COUNT writes / WRITE reads one ballot word per 32 candidates
  u64 mask_base;     // batch index of masks[0]
  unsigned long long* hist;   // FUSED MC: per connectivity code
  unsigned long long* total;  // FUSED TC/CF
  int k;
};

// Per-parent work: sum of deg(emb[pos]) over positions passing to_extend.
template <int APP, int LEV>
__global__ void __launch_bounds__(kThreads) work_kernel(DevGraph g, VLevels L, u64 np, u64* __restrict__ W) {
  constexpr int S = LEV + 1;
  for (u64 p = blockIdx.x * (u64)blockDim.x + threadIdx.x; p < np; p += (u64)gridDim.x * blockDim.x) {
    u32 emb[S];
    reconstruct<LEV>(L, p, emb);
    u64 w = 0;
    if (APP == kAppMC) {
#pragma unroll
      for (int t = 0; t < S; ++t) w += ldg(g.off + emb[t] + 1) - ldg(g.off + emb[t]);
    } else {
      w = ldg(g.off + emb[S - 1] + 1) - ldg(g.off + emb[S - 1]);  // Listing 3: last vertex only
    }
    W[p] = w;
  }
}

// Per-lane cursor over the candidate space: caches the parent embedding that
// owns candidate j.  Parents are addressed in the COMPACTED index space of
// parents with non-zero work (a.pidx maps back to level indices).
template <int APP, int LEV, bool PMASK>
struct Cursor {
  static constexpr int S = LEV + 1;
  static constexpr int NPOS = (APP == kAppMC) ? S : 1;
  static constexpr int NPROBE = (APP == kAppMC) ? 1 : S - 1;
  u64 cp = ~0ull, cWb = 0, cWe = 0;
  u32 parent = 0;  // level index of the parent
  u32 emb[S];
  u64 pbeg[NPOS];
  u32 pdeg[NPOS];
  u64 qbeg[NPROBE];  // CF/TC: probe lists N+(emb[t]), t < S-1
  u32 qdeg[NPROBE];
  u32 pmask = 0;

  __device__ __forceinline__ void load(const ExtendArgs& a, u64 p) {
    if (p == cp) return;
    cp = p;
    cWb = ldg(a.Wp + p);
    cWe = ldg(a.Wp + p + 1);
    parent = ldg(a.pidx + p);
    if (APP != kAppMC && a.dcbeg) {  // descriptor path: independent loads, no chain
      pbeg[0] = ldg(a.dcbeg + p);
#pragma unroll
      for (int t = 0; t < S - 1; ++t) {
        const u64 q = ldg(a.dq[t] + p);
        qbeg[t] = q & ((u64(1) << 40) - 1);
        qdeg[t] = (u32)(q >> 40);
      }
      return;
    }
    reconstruct<LEV>(a.L, parent, emb);
    const DevGraph& g = a.g;
    if (APP == kAppMC) {
#pragma unroll
      for (int t = 0; t < S; ++t) {
        pbeg[t] = ldg(g.off + emb[t]);
        pdeg[t] = (u32)(ldg(g.off + emb[t] + 1) - pbeg[t]);
      }
      if (PMASK) {
        pmask = 1u << pat::pair_index(0, 1, S + 1);
#pragma unroll
        for (int bb = 2; bb < S; ++bb)
#pragma unroll
          for (int aa = 0; aa < bb; ++aa)
            if (has_edge_sym(g, emb[aa], emb[bb])) pmask |= 1u << pat::pair_index(aa, bb, S + 1);
      }
    } else {
      pbeg[0] = ldg(g.off + emb[S - 1]);
      pdeg[0] = (u32)(ldg(g.off + emb[S - 1] + 1) - pbeg[0]);
#pragma unroll
      for (int t = 0; t < S - 1; ++t) {
        qbeg[t] = ldg(g.off + emb[t]);
        qdeg[t] = (u32)(ldg(g.off + emb[t] + 1) - qbeg[t]);
      }
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
    if (APP == kAppMC) {
      pos = 0;
#pragma unroll
      for (int t = 0; t < S - 1; ++t)
        if (pos == t && local >= pdeg[t]) {
          local -= pdeg[t];
          pos = t + 1;
        }
      return ldg(g.col + pbeg[pos] + local);
    }
    pos = S - 1;
    return ldg(g.col + pbeg[0] + local);
  }
};

template <int APP, int LEV, int MODE>
__global__ void __launch_bounds__(kThreads, 2) extend_kernel(ExtendArgs a) {
  constexpr int S = LEV + 1;  // parent embedding size
  constexpr int kWords = (int)(kBatch / 32);
  extern __shared__ unsigned long long shist[];
  __shared__ __align__(16) u32 s_hash[(APP != kAppMC) ? kThreads / 32 : 1][(APP != kAppMC) ? kHashSlots : 4];
  const int lane = threadIdx.x & 31;
  u32* filt = s_hash[(APP != kAppMC) ? (threadIdx.x >> 5) : 0];
  u32 fsh = 0, fmask = 0;
  const DevGraph& g = a.g;
  int nbins = 0;
  if (MODE == kFused && APP == kAppMC) {
    nbins = 1 << pat::npairs(a.k);
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) shist[i] = 0;
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
    Cursor<APP, LEV, MODE == kFused> cur;

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
    u64 fkey = ~0ull;  // begin of the root out-list held in the hash set
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
      if (APP != kAppMC) {
        // warp-shared exact hash set of N+(emb[0]) (the root's out-list,
        // shared by all parents of one root): the emb[0] probe costs one or
        // two shared-memory loads instead of a global binary search
        const u32 act = __ballot_sync(0xffffffffu, j < j1);
        const int leader = __ffs(act) - 1;
        const u64 key = __shfl_sync(0xffffffffu, cur.qbeg[0] | ((u64)cur.qdeg[0] << 40), leader);
        if (key != fkey) {
          fkey = key;
          const u32 d = (u32)(key >> 40);
          const u64 qb = key & ((u64(1) << 40) - 1);
          fok = d <= kFilterMax;
          if (fok) hs_stage_warp(filt, g.col, qb, d, kHashSlots, fsh, fmask);
        }
      }
      if (j < j1) {
        int pos;
        u = cur.candidate(g, j, pos);
        const u32* emb = cur.emb;
        bool inemb = false;
        // SPEC.md:392.  On the DAG descriptor path every emb[t] precedes u in
        // the orientation order (u in N+(emb[S-1])), so u cannot be in emb.
        if (APP == kAppMC || !a.dcbeg) {
#pragma unroll
          for (int t = 0; t < S; ++t) inemb |= (emb[t] == u);
        }
        if (!inemb) {
          if (APP == kAppMC) {
            // is_auto_canonical_vertex + source position
            ok = u > emb[0];
#pragma unroll
            for (int t = 1; t < S; ++t)
              if (t > pos && u <= emb[t]) ok = false;
#pragma unroll
            for (int t = 0; t < S - 1; ++t)
              if (ok && t < pos && has_edge_sym(g, emb[t], u)) ok = false;
            if (ok && MODE == kFused) {
              code = cur.pmask | (1u << pat::pair_index(pos, S, S + 1));
#pragma unroll
              for (int t = 1; t < S; ++t)
                if (t > pos && has_edge_sym(g, emb[t], u)) code |= 1u << pat::pair_index(t, S, S + 1);
            }
          } else {
            // Listing 3 / TC: connected (directed) to every earlier vertex
            ok = true;
            int t0 = 0;
            if (fok && (cur.qbeg[0] | ((u64)cur.qdeg[0] << 40)) == fkey) {
              ok = hs_has(filt, fsh, fmask, u);  // exact: emb[0] needs no further probe
              t0 = 1;
            }
#pragma unroll
            for (int t = 0; t < S - 1; ++t)
              if (t >= t0 && ok && !contains_sorted(g.col + cur.qbeg[t], cur.qdeg[t], u)) ok = false;
          }
        }
      }
      const u32 mask = __ballot_sync(0xffffffffu, ok);
      if (MODE == kCount) {
        c += __popc(mask);
        if (a.masks) {
          if ((it & 31) == lane) myword = mask;
          if ((it & 31) == 31) {
            a.masks[(b - a.mask_base) * kWords + (it - 31) + lane] = myword;
          }
        }
      } else if (MODE == kWrite) {
        if (ok) {
          const u64 o = wpos + __popc(mask & lanemask_lt());
          a.out_idx[o] = cur.parent;
          a.out_vid[o] = u;
        }
        wpos += __popc(mask);
      } else {  // FUSED
        if (APP == kAppMC) {
          if (mask) {
            const u32 key = ok ? code : 0xffffffffu;
            const u32 peers = __match_any_sync(0xffffffffu, key);
            if (ok && lane == __ffs(peers) - 1) atomicAdd(&shist[code], (unsigned long long)__popc(peers));
          }
        } else {
          wtotal += __popc(mask);
        }
      }
    }
    if (MODE == kCount) {
      if (a.masks && (it & 31) != 0 && lane < (it & 31)) a.masks[(b - a.mask_base) * kWords + (it & ~31) + lane] = myword;
      if (lane == 0) a.cnt[b - a.b_begin] = c;
    }
  }
  if (MODE == kFused) {
    if (APP == kAppMC) {
      __syncthreads();
      for (int i = threadIdx.x; i < nbins; i += blockDim.x)
        if (shist[i]) atomicAdd(a.hist + i, shist[i]);
    } else if (lane == 0 && wtotal) {
      atomicAdd(a.total, wtotal);
    }
  }
}

struct NonZeroW {
  const u64* w;
  __device__ __forceinline__ bool operator()(const u32& i) const { return w[i] != 0; }
};

__global__ void gather_kernel(const u64* __restrict__ w, const u32* __restrict__ pidx, u64 nz, u64* __restrict__ Wp) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nz; i += (u64)gridDim.x * blockDim.x)
    Wp[i] = w[pidx[i]];
}

template <int LEV>
__global__ void desc_kernel(DevGraph g, VLevels L, const u32* __restrict__ pidx, u64 nz, u64* __restrict__ cbeg,
                            ExtendArgs a) {
  constexpr int S = LEV + 1;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nz; i += (u64)gridDim.x * blockDim.x) {
    u32 emb[S];
    reconstruct<LEV>(L, pidx[i], emb);
    cbeg[i] = ldg(g.off + emb[S - 1]);
#pragma unroll
    for (int t = 0; t < S - 1; ++t) {
      const u64 b = ldg(g.off + emb[t]), e = ldg(g.off + emb[t] + 1);
      const_cast<u64*>(a.dq[t])[i] = b | ((e - b) << 40);
    }
  }
}

// ---------------------------------------------------------------------------
// First extension of TC / CF on the DAG (Listing 3: parents are level-1 edges
// (v0, v1); candidates u in N+(v1); to_add = u in N+(v0)).  Work item = 32
// consecutive level-1 edges (one per lane), which may span several roots v0.
// The warp stages the out-lists of the item's distinct roots in ONE exact
// shared-memory hash set keyed (u << 5 | root slot), streams the concatenated
// candidate lists N+(v1) 32 at a time (lanes -> parents by one OR-reduction
// over start offsets) and probes each candidate with its parent's root slot.
// Fixed-size edge items keep the per-item cost amortised over ~all 32 lanes
// even when most roots own only a handful of out-edges (power-law DAGs).
// Output order = sequential (parent, candidate) order, as the generic engine.
struct EdgeArgs {
  DevGraph g;
  const u32* src;      // level-1 v0 per DAG edge (absolute edge index)
  u64 lo, hi;          // level-1 slice (edge indices of the DAG CSR)
  u64 ibeg, iend;      // items processed by this launch: [ibeg, iend), item = 32 edges
  u64 grab;            // items per atomic grab
  unsigned long long* ctr;
  u64* cnt;            // COUNT: accepted per item
  const u64* offs;     // WRITE: exclusive offsets per item (absolute index)
  u64 out_base;
  u32* out_idx;
  u32* out_vid;
  u32* masks;          // COUNT writes / WRITE reads ballot words (per-warp chunks)
  u64* moff;           // per item: word offset into masks, or ~0 (no masks)
  unsigned long long* mtop;
  u64 mcap;
  unsigned long long* total;  // FUSED
  unsigned long long* cand;   // candidates streamed (stats)
  u32 hstride;                // per-warp hash slots (power of two)
  const u32* wv;              // SIB: new vertex per entry (level vid array)
};

// SIB = false: level-1 edges (src = v0, new vertex col[e], root list N+(v0)).
// SIB = true: last CF level (k >= 4): entries of a materialised level, src =
// parent index (sorted), new vertex w = wv[e], "root list" = the parent's
// children wv[group] (= the common out-neighbours of the parent embedding, so
// u ~ every earlier vertex <=> u in the group; Listing 3), FUSED only.
template <int MODE, bool SIB>
__global__ void __launch_bounds__(kThreads, 5) edge_chunk_kernel(EdgeArgs a) {
  extern __shared__ __align__(16) u32 s_rhash[];  // [kThreads/32][hstride]
  __shared__ u64 s_cp[kThreads / 32][64];   // per parent rank: &col[cb] - 4 * exclusive start (byte address)
  __shared__ u32 s_ex[kThreads / 32][64];   // per parent rank: exclusive candidate start; ~0 past nnz
  __shared__ u32 s_ei[kThreads / 32][64];   // per parent rank: parent index (slice-relative)
  __shared__ u32 s_sl[kThreads / 32][64];   // per parent rank: root slot
  __shared__ u64 s_rb[kThreads / 32][32];   // per root slot: out-list begin
  __shared__ u32 s_rk[kThreads / 32][64];   // per root slot: exclusive key start; ~0 past the roots
  __shared__ u32 s_rd[kThreads / 32][32];   // per root slot: out-degree
  __shared__ __align__(8) u32 s_mw[kThreads / 32][2 * kSparseWords];  // COUNT: accepted (parent, u) pairs
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const u32 lemask = lanemask_lt() | (1u << lane);
  u32* T = s_rhash + wid * a.hstride;
  u64* const scp = s_cp[wid];
  u32* const sex = s_ex[wid];
  u32* const sei = s_ei[wid];
  u32* const ssl = s_sl[wid];
  u64* const srb = s_rb[wid];
  u32* const srk = s_rk[wid];
  u32* const srd = s_rd[wid];
  u32* const smw = s_mw[wid];
  sex[32 + lane] = 0xffffffffu;
  srk[32 + lane] = 0xffffffffu;
  const DevGraph& g = a.g;
  unsigned long long acc_total = 0, acc_cand = 0;
  u32 mbase = 0, mend = 0;  // this warp's chunk of ballot-mask words (mcap <= 2^28)
  u64 grab = 0, grab_left = 0;
  // WRITE items are (mostly) a copy of recorded children: uniform cost, so
  // warps take them in a static stride instead of contending on the counter
  const u64 gwarp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
  const u64 nwarps = ((u64)gridDim.x * blockDim.x) >> 5;
  u64 sitem = a.ibeg + gwarp;
  for (;;) {
    u64 item;
    if (MODE == kWrite) {
      item = sitem;
      sitem += nwarps;
    } else {
      if (grab_left == 0) {
        u64 it_ = 0;
        if (lane == 0) it_ = atomicAdd(a.ctr, (unsigned long long)a.grab) + a.ibeg;
        grab = __shfl_sync(0xffffffffu, it_, 0);
        grab_left = a.grab;
      }
      item = grab++;
      --grab_left;
    }
    if (item >= a.iend) break;
    u64 wpos = 0, mo = ~0ull;
    if (MODE == kWrite) {
      wpos = ldg(a.offs + item);
      const u64 wend = ldg(a.offs + item + 1);
      if (wend == wpos) continue;
      mo = ldg(a.moff + item);
      wpos -= a.out_base;
      if (mo != ~0ull) {
        // execution from the inspection's recorded children: a coalesced copy
        const u32 nc = (u32)(wend - (wpos + a.out_base));
        for (u32 i = lane; i < nc; i += 32) {
          const uint2 pr = reinterpret_cast<const uint2*>(a.masks + mo)[i];
          a.out_idx[wpos + i] = pr.x;
          a.out_vid[wpos + i] = pr.y;
        }
        continue;
      }
    }
    constexpr bool from_masks = false;
    const u64 e = a.lo + item * 32 + lane;
    const bool valid = e < a.hi;
    const u32 v0 = valid ? ldg(a.src + e) : 0xffffffffu;
    const u32* const keysrc = SIB ? a.wv : g.col;
    const u32 v1 = valid ? ldg(keysrc + e) : 0u;
    // distinct roots of the item (edges are sorted by v0): slot = root rank
    const u32 vprev = __shfl_up_sync(0xffffffffu, v0, 1);
    const bool lead = valid && (lane == 0 || v0 != vprev);
    const u32 lmask = __ballot_sync(0xffffffffu, lead);
    const u32 slot = __popc(lmask & lemask) - 1;
    bool use_hash = false;
    u32 sh = 0, hmask = 0;
    if (!from_masks) {
      // ---- stage the roots' out-lists, key = u << 5 | slot
      u64 rb = 0;
      u32 rd = 0;
      if (lead) {
        if (SIB) {  // the parent's whole child group [gb, ge) (may extend past the item)
          u64 lo_ = 0, hi_ = e;
          while (lo_ < hi_) {
            const u64 mid = (lo_ + hi_) >> 1;
            if (ldg(a.src + mid) < v0) lo_ = mid + 1;
            else hi_ = mid;
          }
          rb = lo_;
          lo_ = e + 1;
          hi_ = a.hi;
          while (lo_ < hi_) {
            const u64 mid = (lo_ + hi_) >> 1;
            if (ldg(a.src + mid) <= v0) lo_ = mid + 1;
            else hi_ = mid;
          }
          rd = (u32)(lo_ - rb);
        } else {
          rb = ldg(g.off + v0);
          rd = (u32)(ldg(g.off + v0 + 1) - rb);
        }
      }
      u32 kin = rd;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, kin, o);
        if (lane >= o) kin += t;
      }
      const u32 K = __shfl_sync(0xffffffffu, kin, 31);
      const u32 nr = __popc(lmask);
      __syncwarp();
      srk[lane] = 0xffffffffu;
      __syncwarp();
      if (lead) {
        srb[slot] = rb;
        srk[slot] = kin - rd;
        srd[slot] = rd;
      }
      __syncwarp();
      use_hash = 2 * K <= a.hstride;
      if (use_hash) {
        u32 cap = 64;
        while (cap < 8 * K && cap < a.hstride) cap <<= 1;
        hb_geom(cap, sh, hmask);  // bucketised: one LDS.128 per probe
        for (u32 i = lane * 4; i < cap; i += 128)
          *reinterpret_cast<uint4*>(T + i) = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
        __syncwarp();
        u32 R = 0;  // root owning key kb
        for (u32 kb = 0; kb < K; kb += 32) {
          const u32 d = srk[R + 1 + lane] - kb;
          const u32 starts = __reduce_or_sync(0xffffffffu, d < 32u ? (1u << d) : 0u);
          const u32 r = min(R + __popc(starts & lemask), nr - 1);
          R += __popc(starts);
          const u32 k = kb + lane;
          if (k < K) hb_insert(T, sh, hmask, (ldg(keysrc + srb[r] + (k - srk[r])) << 5) | r);
        }
        __syncwarp();
      }
    }
    // ---- parents' candidate lists N+(v1), concatenated
    u64 cb = 0;
    u32 w = 0;
    if (valid) {
      cb = ldg(g.off + v1);
      w = (u32)(ldg(g.off + v1 + 1) - cb);
    }
    u32 incl = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const u32 total = __shfl_sync(0xffffffffu, incl, 31);
    if (MODE != kWrite) acc_cand += total;
    if (total == 0) {
      if (MODE == kCount && lane == 0) {
        a.cnt[item] = 0;
        a.moff[item] = ~0ull;
      }
      continue;
    }
    const u32 nzmask = __ballot_sync(0xffffffffu, w > 0);
    const u32 rank = __popc(nzmask & lanemask_lt());
    const u32 nnz = __popc(nzmask);
    __syncwarp();
    sex[lane] = 0xffffffffu;
    __syncwarp();
    if (w > 0) {
      scp[rank] = reinterpret_cast<u64>(g.col) + 4 * (cb - (u64)(incl - w));
      sex[rank] = incl - w;
      sei[rank] = (u32)(e - a.lo);
      ssl[rank] = slot;
    }
    __syncwarp();
    u32 P = 0, c = 0, wi = 0;
    // lane -> parent for the step at jb: one OR-reduction over the next
    // parents' start offsets (sex is padded with ~0 past the last parent)
    auto map_step = [&](u32 jb) -> u32 {
      const u32 d = sex[P + 1 + lane] - jb;
      const u32 starts = __reduce_or_sync(0xffffffffu, d < 32u ? (1u << d) : 0u);
      const u32 myp = P + __popc(starts & lemask);
      P += __popc(starts);
      return myp;
    };
    {
      // software pipeline: the next step's candidate load is in flight while
      // the current one is probed
      u32 myp = map_step(0);
      u32 u = lane < total ? ldg(reinterpret_cast<const u32*>(scp[myp]) + lane) : 0u;
      for (u32 jb = 0; jb < total; jb += 32, ++wi) {
        const u32 j = jb + lane;
        u32 nmyp = 0, nu = 0;
        if (jb + 32 < total) {
          nmyp = map_step(jb + 32);
          if (j + 32 < total) nu = ldg(reinterpret_cast<const u32*>(scp[nmyp]) + j + 32);
        }
        bool ok = false;
        if (j < total) {
          if (use_hash) {
            ok = hb_has(T, sh, hmask, (u << 5) | ssl[myp]);
          } else {
            const u32 r = ssl[myp];
            ok = contains_sorted(keysrc + srb[r], srd[r], u);
          }
        }
        const u32 mask = __ballot_sync(0xffffffffu, ok);
        if (MODE == kWrite) {
          if (ok) {
            const u64 o = wpos + __popc(mask & lanemask_lt());
            a.out_idx[o] = sei[myp];
            a.out_vid[o] = u;
          }
          wpos += __popc(mask);
        } else {
          if (MODE == kCount && mask) {
            // record the accepted children (sequential order) for execution
            const u32 slot = c + __popc(mask & lanemask_lt());
            if (ok && slot < kSparseWords) {
              smw[2 * slot] = sei[myp];
              smw[2 * slot + 1] = u;
            }
          }
          c += __popc(mask);
        }
        myp = nmyp;
        u = nu;
      }
    }
    if (MODE == kCount) {
      // keep the non-zero ballots (step, mask) when they fit; the execution
      // pass then touches accepted candidates only (else it recomputes)
      mo = ~0ull;
      const u32 nzw = c;
      if (nzw && nzw <= kSparseWords && a.masks) {
        if (mbase + 2 * nzw > mend) {  // per-warp chunk: one global atomic per chunk
          unsigned long long t = 0;
          if (lane == 0) t = atomicAdd(a.mtop, (unsigned long long)kMaskChunk);
          t = __shfl_sync(0xffffffffu, t, 0);
          if (t + kMaskChunk <= a.mcap) {
            mbase = (u32)t;
            mend = (u32)(t + kMaskChunk);
          } else {
            mbase = mend = 0;
          }
        }
        if (mbase + 2 * nzw <= mend) {
          __syncwarp();
          for (u32 i = lane; i < 2 * nzw; i += 32) a.masks[mbase + i] = smw[i];
          mo = mbase;
          mbase += 2 * nzw;
        }
      }
      if (lane == 0) {
        a.cnt[item] = c;
        a.moff[item] = mo;
      }
    }
    if (MODE == kFused) acc_total += c;
    __syncwarp();
  }
  if (lane == 0) {
    if (MODE == kFused && acc_total) atomicAdd(a.total, acc_total);
    if (MODE != kWrite && acc_cand) atomicAdd(a.cand, acc_cand);
  }
}

// Canonical code of every connectivity mask over k positions (reduce step 2:
// canonicalize once per quick pattern).
__global__ void canon_masks_kernel(int k, u64* __restrict__ keys) {
  const int nm = 1 << pat::npairs(k);
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < nm; m += gridDim.x * blockDim.x) {
    u32 lab[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    keys[m] = pat::canonicalize(k, lab, (u32)m, 0, nullptr);
  }
}

struct Ctx {
  const gpm_graph* G;
  DevGraph g;
  int app, k;
  cudaStream_t s;
  Timeline* tl;
  Stats* st;
  int sms;
  u64 cap_entries;
  u64 mask_budget;
  unsigned long long* d_total;
  unsigned long long* d_hist;
  unsigned long long* d_ctr;
  bool siblings_complete;   // every child of each level parent is in this chunk
  bool generic_mc;   // GPM_GENERIC_MC: per-candidate binary-search path for MC
  // listing mode (gpm_config.list_fn): the last level is materialised and
  // streamed to the host instead of being counted in the fused kernel
  gpm_list_fn list_fn;
  void* list_ctx;
  u64 listed;
};

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

template <int LEV>
void emit_dispatch(Ctx& c, const VLevels& L, u64 n) {
  if constexpr (LEV + 1 < kMaxLevels) emit_rows<LEV>(c, L, n);
  else throw Error(GPM_EINVAL, "listing: level out of range");
}

template <int APP, int LEV, int MODE>
void launch_extend(Ctx& c, ExtendArgs& a, const char* what, double bytes) {
  auto kern = extend_kernel<APP, LEV, MODE>;
  size_t smem = (MODE == kFused && APP == kAppMC) ? sizeof(unsigned long long) * (size_t(1) << pat::npairs(c.k)) : 0;
  static std::atomic<int> occ_slot{0};  // per template instantiation
  const int occ = cached_occupancy(occ_slot, [&] {
    int o = 0;
    GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kThreads, smem));
    return o;
  });
  const u64 nb = a.b_end - a.b_begin;
  const u64 warps_needed = nb;
  u64 blocks = std::min<u64>((u64)c.sms * occ, (warps_needed * 32 + kThreads - 1) / kThreads);
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

template <int APP, int LEV>
void run_work(Ctx& c, const VLevels& L, u64 np, u64* W) {
  unsigned blocks = (unsigned)std::min<u64>((np + kThreads - 1) / kThreads, (u64)c.sms * 16);
  work_kernel<APP, LEV><<<std::max(1u, blocks), kThreads, 0, c.s>>>(c.g, L, np, W);
  GPM_CUDA(cudaGetLastError());
  ++c.tl->launches;
}

void cf_last_siblings(Ctx& c, const u32* idx, const u32* vid, u64 np, int lev);

template <int APP, int LEV>
void process(Ctx& c, VLevels L, u64 np);

template <int APP>
void process_dispatch(Ctx& c, int lev, const VLevels& L, u64 np) {
  switch (lev) {
#define GPM_LEV(X) \
  case X:          \
    if constexpr (APP != kAppMC || X <= 3) { process<APP, X>(c, L, np); return; } break;
    GPM_LEV(1) GPM_LEV(2) GPM_LEV(3) GPM_LEV(4) GPM_LEV(5) GPM_LEV(6) GPM_LEV(7)
#undef GPM_LEV
    default:
      break;
  }
  throw Error(GPM_EINVAL, "unsupported level " + std::to_string(lev));
}

template <int APP, int LEV>
void process(Ctx& c, VLevels L, u64 np) {
  constexpr int S = LEV + 1;
  constexpr int NPOS = (APP == kAppMC) ? S : 1;
  const bool last = (LEV == c.k - 2);
  Stats& st = *c.st;
  if (np == 0) return;
  if constexpr (APP == kAppMC && LEV == 2) {
    if (last && c.k == 4 && !c.generic_mc && c.G->n < (1u << 30)) {  // union-set tags need ids < 2^30
      mc4_last_staged(*c.G, L.idx[0], L.vid[0], L.idx[1], L.vid[1], np, c.d_hist, c.s, *c.tl, st);
      return;
    }
  }
  if constexpr (APP == kAppCF && LEV >= 2) {
    if (last && !c.list_fn && c.g.oriented && c.siblings_complete && c.G->n < (1u << 27) &&
        !std::getenv("GPM_GENERIC_CF")) {
      cf_last_siblings(c, L.idx[LEV - 1], L.vid[LEV - 1], np, LEV);
      return;
    }
  }
  // ---- work pass, compaction of parents with work, scan: candidate space
  u64 nz = 0;
  DBuf<u32> pidx;
  DBuf<u64> Wp;
  {
    DBuf<u64> w(np, c.s);
    htrace(c.s, "generic: alloc w");
    run_work<APP, LEV>(c, L, np, w.get());
    htrace(c.s, "generic: work kernel");
    pidx.alloc(np, c.s);
    htrace(c.s, "generic: alloc pidx");
    DBuf<u64> nsel(1, c.s);
    size_t tmp = 0;
    thrust::counting_iterator<u32> it(0);
    GPM_CUDA(cub::DeviceSelect::If(nullptr, tmp, it, pidx.get(), nsel.get(), (int64_t)np, NonZeroW{w.get()}, c.s));
    DBuf<u8> t(tmp, c.s);
    GPM_CUDA(cub::DeviceSelect::If(t.get(), tmp, it, pidx.get(), nsel.get(), (int64_t)np, NonZeroW{w.get()}, c.s));
    GPM_CUDA(cudaMemcpyAsync(&nz, nsel.get(), sizeof(u64), cudaMemcpyDeviceToHost, c.s));
    GPM_CUDA(cudaStreamSynchronize(c.s));
    htrace(c.s, "generic: select");
    Wp.alloc(nz + 1, c.s);
    htrace(c.s, "generic: alloc Wp");
    GPM_CUDA(cudaMemsetAsync(Wp.get() + nz, 0, sizeof(u64), c.s));
    if (nz) {
      gather_kernel<<<(unsigned)std::min<u64>((nz + 255) / 256, 1u << 20), 256, 0, c.s>>>(w.get(), pidx.get(), nz,
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
  const double bytes_in = 8.0 * LEV * np + 16.0 * NPOS * np + 4.0 * W;
  st.balg += bytes_in;
  htrace(c.s, "generic: work+select+scan");
  if (W == 0) return;
  const u64 nb = (W + kBatch - 1) / kBatch;
  ExtendArgs a{};
  a.g = c.g;
  a.L = L;
  a.Wp = Wp.get();
  a.pidx = pidx.get();
  a.np = nz;
  a.W = W;
  DBuf<u64> dcbeg, dq;
  if (APP != kAppMC && c.g.oriented && c.G->m < (u64(1) << 40)) {
    dcbeg.alloc(nz, c.s);
    dq.alloc(nz * (S - 1), c.s);
    for (int t = 0; t < S - 1; ++t) a.dq[t] = dq.get() + (u64)t * nz;
    a.dcbeg = dcbeg.get();
    desc_kernel<LEV><<<(unsigned)std::min<u64>((nz + 255) / 256, 1u << 20), 256, 0, c.s>>>(c.g, L, pidx.get(), nz,
                                                                                       dcbeg.get(), a);
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
    launch_extend<APP, LEV, kFused>(c, a, "extend_fused", bytes_in);
    htrace(c.s, "generic: fused");
    return;
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
  launch_extend<APP, LEV, kCount>(c, a, "extend_count", bytes_in);
  htrace(c.s, "generic: count");
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
    htrace(c.s, "generic: alloc level");
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
    launch_extend<APP, LEV, kWrite>(c, w, "extend_write", wbytes + 8.0 * Tc);
    htrace(c.s, "generic: write");
    VLevels nl = L;
    nl.idx[LEV] = oi.get();
    nl.vid[LEV] = ov.get();
    c.siblings_complete = chunks.size() == 1;  // planner chunks may split a parent's children
    if (last) emit_dispatch<LEV + 1>(c, nl, Tc);
    else process_dispatch<APP>(c, LEV + 1, nl, Tc);
  }
}

template <int MODE, bool SIB = false>
void launch_edge(Ctx& c, EdgeArgs& a, const std::string& what, double bytes) {
  auto kern = edge_chunk_kernel<MODE, SIB>;
  // hash capacity: keys of one item <= 32 + 2 x max out-degree in practice
  const u32 md = c.G->max_deg ? c.G->max_deg : kFilterMax;
  u32 hs = 256;
  while (hs < 2 * (32 + 2 * std::min<u32>(md, kFilterMax)) && hs < kHashSlots) hs <<= 1;
  a.hstride = hs;
  const size_t smem = (size_t)(kThreads / 32) * hs * sizeof(u32);
  static std::atomic<int> occ_by_hs[16];  // zero-initialised (static storage)
  const int occ = cached_occupancy(occ_by_hs[31 - __builtin_clz(hs)], [&] {
    GPM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kThreads / 32 * kHashSlots * 4)));
    int o = 0;
    GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kThreads, smem));
    return o;
  });
  const u64 ni = a.iend - a.ibeg;
  u64 blocks = std::max<u64>(1, std::min<u64>((u64)c.sms * occ, (ni * 32 + kThreads - 1) / kThreads));
  // coarse grabs only when every warp gets many items (tail balance first)
  a.grab = std::max<u64>(1, std::min<u64>(kItemGrab, ni / (blocks * (kThreads / 32) * 64)));
  GPM_CUDA(cudaMemsetAsync(c.d_ctr, 0, sizeof(unsigned long long), c.s));
  a.ctr = c.d_ctr;
  size_t ev = c.tl->begin(what, bytes);
  kern<<<(unsigned)blocks, kThreads, smem, c.s>>>(a);
  GPM_CUDA(cudaGetLastError());
  c.tl->end(ev);
  ++c.tl->launches;
}

// Last extension of CF (k >= 4) over a complete materialised level: the
// edge-chunk kernel in sibling mode (one probe into the parent's child group
// replaces the LEV binary searches of the generic to_add).
void cf_last_siblings(Ctx& c, const u32* idx, const u32* vid, u64 np, int lev) {
  DBuf<unsigned long long> cand(1, c.s);
  GPM_CUDA(cudaMemsetAsync(cand.get(), 0, sizeof(unsigned long long), c.s));
  EdgeArgs a{};
  a.g = c.g;
  a.src = idx;
  a.wv = vid;
  a.lo = 0;
  a.hi = np;
  a.ibeg = 0;
  a.iend = (np + 31) / 32;
  a.total = c.d_total;
  a.cand = cand.get();
  size_t rec = c.tl->recs.size();
  c.st->paths |= GPM_PATH_CF_SIBLINGS;
  launch_edge<kFused, true>(c, a, "extend_fused_L" + std::to_string(lev), 0.0);
  unsigned long long W = 0;
  GPM_CUDA(cudaMemcpyAsync(&W, cand.get(), sizeof W, cudaMemcpyDeviceToHost, c.s));
  GPM_CUDA(cudaStreamSynchronize(c.s));
  const double bytes = 8.0 * lev * np + 16.0 * np + 4.0 * (double)W;  // SURVEY §8d (one extended position)
  c.tl->recs[rec].bytes = bytes;
  c.st->candidates[lev] += W;
  c.st->balg += bytes;
}

// First extension of TC/CF on a DAG through the edge-chunk kernel; deeper
// levels continue in the generic engine.  src = level-1 v0 (absolute index).
void process_l1_cf(Ctx& c, const VLevels& L, const u32* src, u64 lo, u64 hi) {
  Stats& st = *c.st;
  const u64 np = hi - lo;
  if (np == 0) return;
  const bool last = (c.k == 3);
  const u64 NI = (np + 31) / 32;
  st.paths |= GPM_PATH_CF_EDGE_CHUNK;
  DBuf<unsigned long long> cand(1, c.s);
  GPM_CUDA(cudaMemsetAsync(cand.get(), 0, sizeof(unsigned long long), c.s));
  EdgeArgs a{};
  a.g = c.g;
  a.src = src;
  a.lo = lo;
  a.hi = hi;
  a.ibeg = 0;
  a.iend = NI;
  a.cand = cand.get();
  if (last) {
    a.total = c.d_total;
    size_t rec = c.tl->recs.size();
    launch_edge<kFused>(c, a, "extend_fused_L1", 0.0);
    unsigned long long W = 0;
    GPM_CUDA(cudaMemcpyAsync(&W, cand.get(), sizeof W, cudaMemcpyDeviceToHost, c.s));
    GPM_CUDA(cudaStreamSynchronize(c.s));
    const double bytes = 8.0 * np + 16.0 * np + 4.0 * W;
    c.tl->recs[rec].bytes = bytes;
    st.candidates[1] += W;
    st.balg += bytes;
    return;
  }
  DBuf<u64> cnt(NI + 1, c.s), moff(NI + 1, c.s);
  GPM_CUDA(cudaMemsetAsync(cnt.get() + NI, 0, sizeof(u64), c.s));
  // ballot masks: 1 bit per candidate, per-warp chunks
  // recorded children: <= kSparseWords pairs per item + one chunk of slack per warp
  const u64 mwant = 2 * kSparseWords * NI + (u64)c.sms * 64 * kMaskChunk;
  const u64 mcap = std::max<u64>(1, std::min<u64>({c.mask_budget / 4, u64(1) << 28, mwant}));
  DBuf<u32> masks(mcap, c.s);
  DBuf<unsigned long long> mtop(1, c.s);
  GPM_CUDA(cudaMemsetAsync(mtop.get(), 0, sizeof(unsigned long long), c.s));
  a.cnt = cnt.get();
  a.moff = moff.get();
  a.masks = masks.get();
  a.mtop = mtop.get();
  a.mcap = mcap;
  size_t rec = c.tl->recs.size();
  launch_edge<kCount>(c, a, "extend_count_L1", 0.0);
  scan_inplace(cnt.get(), NI + 1, c.s);
  unsigned long long W = 0;
  u64 T = 0;
  GPM_CUDA(cudaMemcpyAsync(&W, cand.get(), sizeof W, cudaMemcpyDeviceToHost, c.s));
  GPM_CUDA(cudaMemcpyAsync(&T, cnt.get() + NI, sizeof(u64), cudaMemcpyDeviceToHost, c.s));
  GPM_CUDA(cudaStreamSynchronize(c.s));
  const double bytes_in = 8.0 * np + 16.0 * np + 4.0 * W;
  c.tl->recs[rec].bytes = bytes_in;
  st.candidates[1] += W;
  st.balg += bytes_in + 8.0 * T;
  st.level_sizes[1] += T;
  if (T == 0) return;
  std::vector<std::pair<u64, u64>> chunks;  // item ranges
  if (T <= c.cap_entries) {
    chunks.emplace_back(0, NI);
  } else {
    std::vector<u64> h(NI + 1);
    GPM_CUDA(cudaMemcpyAsync(h.data(), cnt.get(), sizeof(u64) * (NI + 1), cudaMemcpyDeviceToHost, c.s));
    GPM_CUDA(cudaStreamSynchronize(c.s));
    u64 r0 = 0;
    while (r0 < NI) {
      u64 key = h[r0] + c.cap_entries;
      u64 r1 = (u64)(std::upper_bound(h.begin() + r0 + 1, h.end(), key) - h.begin()) - 1;
      if (r1 <= r0) r1 = r0 + 1;
      chunks.emplace_back(r0, r1);
      r0 = r1;
    }
  }
  st.chunks += chunks.size() - 1;
  for (auto [r0, r1] : chunks) {
    u64 base = 0, end = 0;
    GPM_CUDA(cudaMemcpyAsync(&base, cnt.get() + r0, sizeof(u64), cudaMemcpyDeviceToHost, c.s));
    GPM_CUDA(cudaMemcpyAsync(&end, cnt.get() + r1, sizeof(u64), cudaMemcpyDeviceToHost, c.s));
    GPM_CUDA(cudaStreamSynchronize(c.s));
    const u64 Tc = end - base;
    if (Tc == 0) continue;
    DBuf<u32> oi(Tc, c.s), ov(Tc, c.s);
    EdgeArgs w = a;
    w.ibeg = r0;
    w.iend = r1;
    w.offs = cnt.get();
    w.out_base = base;
    w.out_idx = oi.get();
    w.out_vid = ov.get();
    const double frac = (double)(r1 - r0) / (double)NI;
    launch_edge<kWrite>(c, w, "extend_write_L1", frac * (double)W / 8.0 + 24.0 * Tc);
    htrace(c.s, "l1: write");
    VLevels nl = L;
    nl.idx[1] = oi.get();
    nl.vid[1] = ov.get();
    c.siblings_complete = true;  // item-aligned chunks never split an edge's children
    process_dispatch<kAppCF>(c, 2, nl, Tc);
  }
}

}  // namespace


void mine_vertex(const gpm_graph& G0, const gpm_config& cfg, cudaStream_t s, gpm_result& res, Stats& st,
                 Timeline& tl) {
  int app = cfg.app;
  int k = cfg.k;
  if (app == GPM_APP_TC) k = 3;
  if (app == GPM_APP_CF && (k < 3 || k > 9)) throw Error(GPM_EINVAL, "clique_find: k must be in [3,9]");
  if (app == GPM_APP_MC && (k < 3 || k > 5)) throw Error(GPM_EINVAL, "motif_count: k must be in {3,4,5}");
  res.k = k;
  // TC/CF run on the degree-ordered DAG; MC unoriented (:457)
  std::unique_ptr<gpm_graph> dag;
  const gpm_graph* G = &G0;
  if (app != GPM_APP_MC && !G0.oriented && !cfg.no_orient) {
    dag = std::make_unique<gpm_graph>();
    dag->device = G0.device;
    dag->stream = s;            // orient on the engine stream; freed on it too
    dag->owns_stream = false;
    orient_on_device(G0, *dag);
    tl.launches += 4;
    G = dag.get();
  }
  if (app == GPM_APP_MC && G0.oriented) throw Error(GPM_EINVAL, "motif_count needs an undirected graph");

  const int levels = k - 1;
  st.ensure(levels);
  htrace(s, "mine_vertex: start (orient done)");
  DBuf<u32> l1i, l1v;
  DBuf<u64> l1s;
  u64 n1 = 0;
  const u32* l1vid = nullptr;
  build_level1(*G, l1i, l1v, n1, s, tl, &l1vid, &l1s);
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
    root_split_bounds(*G, l1i.get(), l1vid, n1, app, world, bounds, s, tl);
    lo = bounds[cfg.rank];
    hi = bounds[cfg.rank + 1];
  }
  htrace(s, "level1 built");

  Ctx c{};
  c.G = G;
  c.g = G->view();
  c.app = app;
  c.k = k;
  c.s = s;
  c.tl = &tl;
  c.st = &st;
  c.sms = sm_count();
  c.generic_mc = std::getenv("GPM_GENERIC_MC") != nullptr;
  c.list_fn = cfg.list_fn;
  c.list_ctx = cfg.list_ctx;
  c.listed = 0;
  if (c.list_fn && app == GPM_APP_MC) throw Error(GPM_EINVAL, "listing mode: TC/CF only (SPEC.md:458)");
  const size_t freeb = device_free_bytes();
  u64 budget = cfg.mem_budget ? cfg.mem_budget : (u64)(0.6 * (double)freeb);
  const int mat_levels = std::max(1, k - 3);
  c.cap_entries = std::max<u64>(kBatch, std::min<u64>((u64(1) << 32) - 1, budget / 16 / mat_levels));
  c.mask_budget = budget / 4;
  const int nbins = (app == GPM_APP_MC) ? (1 << pat::npairs(k)) : 1;
  DBuf<unsigned long long> d_total(1, s), d_hist(nbins, s), d_ctr(1, s);
  GPM_CUDA(cudaMemsetAsync(d_total.get(), 0, sizeof(unsigned long long), s));
  GPM_CUDA(cudaMemsetAsync(d_hist.get(), 0, sizeof(unsigned long long) * nbins, s));
  c.d_total = d_total.get();
  c.d_hist = d_hist.get();
  c.d_ctr = d_ctr.get();

  htrace(s, "setup (meminfo, counters)");
  const int appk = (app == GPM_APP_MC) ? kAppMC : kAppCF;  // TC == CF with k=3 (Listing 3)
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
    if (appk == kAppMC && k == 3 && l1s.get() && !c.generic_mc) {
      mc3_staged(*G, l1s.get(), slo, shi, c.d_hist, s, tl, st);
    } else if (appk == kAppMC) {
      process_dispatch<kAppMC>(c, 1, L, np);
    } else if (G->oriented && G->n < (1u << 27) && !c.list_fn && !std::getenv("GPM_GENERIC_L1")) {  // key = u << 5 | slot
      process_l1_cf(c, L, l1i.get(), slo, shi);
    } else {
      process_dispatch<kAppCF>(c, 1, L, np);
    }
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
    const u64 chunk = cfg.steal_chunk ? cfg.steal_chunk : std::max<u64>(1024, tsum / ((u64)world * 32));
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

  htrace(s, "levels processed");
  if (c.list_fn && k > 2) {  // listed rows play the fused kernel's count (exchanged below)
    const unsigned long long v = c.listed;
    GPM_CUDA(cudaMemcpyAsync(d_total.get(), &v, sizeof v, cudaMemcpyHostToDevice, s));
    GPM_CUDA(cudaStreamSynchronize(s));
  }
  // multi-GPU: the only collectives are the per-pattern counts and the
  // per-level size vectors
  if (cfg.world > 1 && cfg.exchange) {
    if (app == GPM_APP_MC) exchange_device(cfg, d_hist.get(), nbins, 8, 0, s);
    else exchange_device(cfg, d_total.get(), 1, 8, 0, s);
    std::vector<u64> v;
    for (auto x : st.level_sizes) v.push_back(x);
    for (auto x : st.candidates) v.push_back(x);
    v.push_back((u64)st.balg);
    exchange_sum_host(cfg, v, s);
    const size_t L = st.level_sizes.size();
    for (size_t i = 0; i < L; ++i) st.level_sizes[i] = v[i];
    for (size_t i = 0; i < st.candidates.size(); ++i) st.candidates[i] = v[L + i];
    st.balg = (double)v.back();
    // the fused last level is re-derived from the reduced counters below
    st.level_sizes[levels - 1] = 0;
  }

  if (app == GPM_APP_MC) {
    std::vector<unsigned long long> h(nbins);
    std::vector<u64> keys(nbins);
    DBuf<u64> dk(nbins, s);
    canon_masks_kernel<<<(nbins + 127) / 128, 128, 0, s>>>(k, dk.get());
    GPM_CUDA(cudaGetLastError());
    ++tl.launches;
    GPM_CUDA(cudaMemcpyAsync(h.data(), d_hist.get(), sizeof(unsigned long long) * nbins, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaMemcpyAsync(keys.data(), dk.get(), sizeof(u64) * nbins, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaStreamSynchronize(s));
    std::map<u64, u64> agg;
    u64 acc = 0;
    for (int m = 0; m < nbins; ++m)
      if (h[m]) {
        agg[keys[m]] += h[m];
        acc += h[m];
      }
    for (auto& [key, cnt] : agg) res.patterns.push_back({canon_text(key, k, 0, nullptr), cnt, k});
    std::sort(res.patterns.begin(), res.patterns.end(),
              [](const gpm_result::Pattern& x, const gpm_result::Pattern& y) { return x.text < y.text; });
    st.level_sizes[levels - 1] += acc;
    res.total = acc;
  } else if (k > 2) {
    unsigned long long t = 0;
    GPM_CUDA(cudaMemcpyAsync(&t, d_total.get(), sizeof t, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaStreamSynchronize(s));
    res.total = t;
    st.level_sizes[levels - 1] += t;
  }
}

}  // namespace gpm
