// vertex.cu — the builtin vertex-mode apps (TC, k-CL, k-MC) on the
// header-only hook engine (include/gpm_engine.cuh) plus their specialised
// sm_100a kernels, selected under the same App contract.
//
// Reference: Alg. 1 / Alg. 2, engine module SPEC.md:344-379,
// apps, Listings 3/4/6.  The App structs are in
// include/gpm_apps.cuh; the generic inspection-execution extend, the memory
// planner, listing, root split / stealing and the count exchange are the
// engine's.  This file holds the specialisations:
//  * CF/TC first extension on the DAG: edge-chunk kernel;
//  * CF last extension over complete sibling groups;
//  * MC staged last levels (mc_staged.cu).
#include <cstdlib>
#include <cstring>

#include "gpm_apps.cuh"

namespace gpm {

using engine::Ctx;
using engine::VLevels;
using engine::kCount;
using engine::kWrite;
using engine::kFused;
using engine::kThreads;

namespace {

constexpr u64 kItemGrab = 8;        // root-kernel work items per atomic grab
constexpr u32 kHashSlots = 1024;    // per-warp hash slots of the edge-chunk kernel
constexpr u32 kFilterMax = 512;     // out-lists longer than this are probed by binary search
constexpr u64 kMaskChunk = 4096;    // record words a warp reserves at a time
constexpr u32 kSparseWords = 64;    // accepted (parent, u) children recorded per CF item

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


// Hybrid variant of edge_chunk_kernel for the inspection (COUNT) and fused
// (FUSED) passes: same items, staging and results.  The whole 32-candidate
// chunks of a candidate list N+(v1) are streamed by the whole warp, one parent
// at a time (no lane -> parent mapping, the probe's root slot is
// warp-uniform); the remaining w mod 32 candidates of every list are packed
// 32 per step with the OR-reduction mapping of edge_chunk_kernel, so no step
// is wasted on a partial chunk.  Accepted
// children are rare (PAT: 1 in 400): COUNT records them as (parent lane,
// index within the parent) -- the index from a per-parent shared counter
// plus the rank among same-parent lanes of the step, so it follows u order
// -- and places them at prefix(parent) + index, i.e. in the sequential
// (parent, u) order the execution pass copies.  The execution pass (WRITE)
// stays on edge_chunk_kernel.

template <int MODE, bool SIB>
__global__ void __launch_bounds__(kThreads, 5) edge_lane_kernel(EdgeArgs a) {
  static_assert(MODE != kWrite, "execution runs on edge_chunk_kernel");
  extern __shared__ __align__(16) u32 s_rhash[];  // [kThreads/32][hstride]
  __shared__ u64 s_cp[kThreads / 32][32];   // short parent rank: &col[cb] - 4 * exclusive start
  __shared__ u32 s_ex[kThreads / 32][64];   // short parent rank: exclusive start; ~0 past the last
  __shared__ u32 s_sl[kThreads / 32][32];   // short parent rank: (lane << 8) | root slot
  __shared__ u64 s_rb[kThreads / 32][32];   // per root slot: out-list begin
  __shared__ u32 s_rk[kThreads / 32][64];   // per root slot: exclusive key start; ~0 past the roots
  __shared__ u32 s_rd[kThreads / 32][32];   // per root slot: out-degree
  __shared__ u32 s_pc[kThreads / 32][32];   // COUNT: accepted children per parent lane
  __shared__ __align__(8) u32 s_ac[kThreads / 32][2 * kSparseWords];  // COUNT: (lane << 16 | idx, u)
  __shared__ __align__(8) u32 s_mw[kThreads / 32][2 * kSparseWords];  // COUNT: ordered (parent, u) pairs
  __shared__ u32 s_na[kThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const u32 lemask = lanemask_lt() | (1u << lane);
  u32* T = s_rhash + wid * a.hstride;
  u64* const scp = s_cp[wid];
  u32* const sex = s_ex[wid];
  u32* const ssl = s_sl[wid];
  u64* const srb = s_rb[wid];
  u32* const srk = s_rk[wid];
  u32* const srd = s_rd[wid];
  u32* const spc = s_pc[wid];
  u32* const sac = s_ac[wid];
  u32* const smw = s_mw[wid];
  srk[32 + lane] = 0xffffffffu;
  sex[32 + lane] = 0xffffffffu;
  const DevGraph& g = a.g;
  unsigned long long acc_total = 0, acc_cand = 0;
  u32 mbase = 0, mend = 0;
  u64 grab = 0, grab_left = 0;
  const u32* const keysrc = SIB ? a.wv : g.col;
  for (;;) {
    if (grab_left == 0) {
      u64 it_ = 0;
      if (lane == 0) it_ = atomicAdd(a.ctr, (unsigned long long)a.grab) + a.ibeg;
      grab = __shfl_sync(0xffffffffu, it_, 0);
      grab_left = a.grab;
    }
    const u64 item = grab++;
    --grab_left;
    if (item >= a.iend) break;
    const u64 e = a.lo + item * 32 + lane;
    const bool valid = e < a.hi;
    const u32 v0 = valid ? ldg(a.src + e) : 0xffffffffu;
    const u32 v1 = valid ? ldg(keysrc + e) : 0u;
    // ---- roots of the item and their staged out-lists (as edge_chunk_kernel)
    const u32 vprev = __shfl_up_sync(0xffffffffu, v0, 1);
    const bool lead = valid && (lane == 0 || v0 != vprev);
    const u32 lmask = __ballot_sync(0xffffffffu, lead);
    const u32 slot = __popc(lmask & lemask) - 1;
    u64 rb = 0;
    u32 rd = 0;
    if (lead) {
      if (SIB) {
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
    sex[lane] = 0xffffffffu;
    if (MODE == kCount) {
      spc[lane] = 0;
      if (lane == 0) s_na[wid] = 0;
    }
    __syncwarp();
    if (lead) {
      srb[slot] = rb;
      srk[slot] = kin - rd;
      srd[slot] = rd;
    }
    __syncwarp();
    const bool use_hash = 2 * K <= a.hstride;
    u32 sh = 0, hmask = 0;
    if (use_hash) {
      u32 cap = 64;
      while (cap < 8 * K && cap < a.hstride) cap <<= 1;
      hb_geom(cap, sh, hmask);
      for (u32 i = lane * 4; i < cap; i += 128)
        *reinterpret_cast<uint4*>(T + i) = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
      __syncwarp();
      u32 R = 0;
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
    auto probe = [&](u32 u, u32 sl) -> bool {
      if (use_hash) return hb_has(T, sh, hmask, (u << 5) | sl);
      return contains_sorted(keysrc + srb[sl], srd[sl], u);
    };
    // record an accepted child of parent lane pl at index idx (COUNT)
    auto record = [&](u32 pl, u32 idx, u32 u) {
      const u32 qd = atomicAdd(&s_na[wid], 1u);
      if (qd < kSparseWords) {
        sac[2 * qd] = (pl << 16) | idx;
        sac[2 * qd + 1] = u;
      }
    };
    // ---- this lane's parent: candidates N+(v1)
    u64 cb = 0;
    u32 w = 0;
    if (valid) {
      cb = ldg(g.off + v1);
      w = (u32)(ldg(g.off + v1 + 1) - cb);
    }
    const u32 total = __reduce_add_sync(0xffffffffu, w);
    acc_cand += total;
    if (total == 0) {
      if (MODE == kCount && lane == 0) {
        a.cnt[item] = 0;
        a.moff[item] = ~0ull;
      }
      continue;
    }
    u32 c = 0;  // accepted children of the item (warp-uniform)
    // ---- heads of the long lists (whole 32-candidate chunks), warp-cooperative
    for (u32 lm = __ballot_sync(0xffffffffu, w >= 32); lm; lm &= lm - 1) {
      const int p = __ffs(lm) - 1;
      const u64 pcb = __shfl_sync(0xffffffffu, cb, p);
      const u32 pw = __shfl_sync(0xffffffffu, w, p) & ~31u;
      const u32 psl = __shfl_sync(0xffffffffu, slot, p);
      const u32* const pl = g.col + pcb;
      u32 pc = 0;
      u32 u = lane < pw ? ldg(pl + lane) : 0u;
      for (u32 jb = 0; jb < pw; jb += 32) {
        const u32 nu = jb + 32 + lane < pw ? ldg(pl + jb + 32 + lane) : 0u;
        const bool ok = jb + lane < pw && probe(u, psl);
        const u32 m = __ballot_sync(0xffffffffu, ok);
        if (MODE == kCount && ok) record((u32)p, pc + __popc(m & lanemask_lt()), u);
        pc += __popc(m);
        u = nu;
      }
      if (MODE == kCount && lane == 0) spc[p] = pc;
      c += pc;
    }
    // ---- the tails (w mod 32 candidates of every list), packed 32 per step
    const u32 tw = w & 31u, head = w & ~31u;
    const bool sp = tw > 0;
    const u32 smask = __ballot_sync(0xffffffffu, sp);
    if (smask) {
      u32 incl = tw;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const u32 stot = __shfl_sync(0xffffffffu, incl, 31);
      const u32 rank = __popc(smask & lanemask_lt());
      if (sp) {
        scp[rank] = reinterpret_cast<u64>(g.col) + 4 * (cb + head - (u64)(incl - tw));
        sex[rank] = incl - tw;
        ssl[rank] = ((u32)lane << 8) | slot;
      }
      __syncwarp();
      u32 P = 0;
      auto map_step = [&](u32 jb) -> u32 {
        const u32 d = sex[P + 1 + lane] - jb;
        const u32 starts = __reduce_or_sync(0xffffffffu, d < 32u ? (1u << d) : 0u);
        const u32 myp = P + __popc(starts & lemask);
        P += __popc(starts);
        return myp;
      };
      u32 myp = map_step(0);
      u32 u = lane < stot ? ldg(reinterpret_cast<const u32*>(scp[myp]) + lane) : 0u;
      for (u32 jb = 0; jb < stot; jb += 32) {
        const u32 j = jb + lane;
        u32 nmyp = 0, nu = 0;
        if (jb + 32 < stot) {
          nmyp = map_step(jb + 32);
          if (j + 32 < stot) nu = ldg(reinterpret_cast<const u32*>(scp[nmyp]) + j + 32);
        }
        const u32 sl = j < stot ? ssl[myp] : 0u;
        const bool ok = j < stot && probe(u, sl & 0xffu);
        const u32 m = __ballot_sync(0xffffffffu, ok);
        if (MODE == kCount && m) {
          // index within the parent: its count so far + rank among same-parent lanes
          const u32 peers = __match_any_sync(0xffffffffu, ok ? myp : 0xffffffffu);
          if (ok) {
            const int leader = __ffs(peers) - 1;
            const u32 pl = sl >> 8;
            u32 base = 0;
            if (lane == leader) base = atomicAdd(&spc[pl], (u32)__popc(peers));
            base = __shfl_sync(peers, base, leader);
            record(pl, base + __popc(peers & lanemask_lt()), u);
          }
        }
        c += __popc(m);
        myp = nmyp;
        u = nu;
      }
    }
    if (MODE == kFused) acc_total += c;
    if (MODE == kCount) {
      __syncwarp();
      u64 mo = ~0ull;
      if (c && c <= kSparseWords && a.masks) {
        // order the records: (parent lane, index) -> prefix(parent lane) + index
        u32 pcnt = spc[lane], pincl = pcnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const u32 t = __shfl_up_sync(0xffffffffu, pincl, o);
          if (lane >= o) pincl += t;
        }
        const u32 pre = pincl - pcnt;
        for (u32 ib = 0; ib < c; ib += 32) {
          const u32 i = ib + lane;
          const u32 key = i < c ? sac[2 * i] : 0u;
          const u32 pos = __shfl_sync(0xffffffffu, pre, key >> 16) + (key & 0xffffu);
          if (i < c) {
            smw[2 * pos] = (u32)(item * 32 + (key >> 16));
            smw[2 * pos + 1] = sac[2 * i + 1];
          }
        }
        __syncwarp();
        if (mbase + 2 * c > mend) {
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
        if (mbase + 2 * c <= mend) {
          for (u32 i = lane; i < 2 * c; i += 32) a.masks[mbase + i] = smw[i];
          mo = mbase;
          mbase += 2 * c;
        }
      }
      if (lane == 0) {
        a.cnt[item] = c;
        a.moff[item] = mo;
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    if (MODE == kFused && acc_total) atomicAdd(a.total, acc_total);
    if (acc_cand) atomicAdd(a.cand, acc_cand);
  }
}

template <int MODE, bool SIB = false>
void launch_edge(Ctx& c, EdgeArgs& a, const std::string& what, double bytes) {
  // GPM_CF_STREAM=1: the packed-stream kernel (all lanes on the concatenated
  // candidate lists) instead of the lane-per-parent one
  // FUSED counts run on the hybrid kernel (whole 32-candidate chunks without
  // the lane -> parent mapping: TC16 0.264 -> 0.215 ms); the inspection pass
  // stays on the packed stream, which measured faster on short-list DAGs
  // (PAT 4-CL: 1.20 vs 1.45 ms; profiles/r02).  GPM_CF_STREAM=1 / GPM_CF_HYBRID=1
  // force one or the other.
  static const bool stream_env = std::getenv("GPM_CF_STREAM") != nullptr;
  static const bool hybrid_env = std::getenv("GPM_CF_HYBRID") != nullptr;
  const bool stream = stream_env || MODE == kWrite || (MODE == kCount && !hybrid_env);
  void (*kern)(EdgeArgs) = edge_chunk_kernel<MODE, SIB>;
  if constexpr (MODE != kWrite) {
    if (!stream) kern = edge_lane_kernel<MODE, SIB>;
  }
  // hash capacity: keys of one item <= 32 + 2 x max out-degree in practice
  const u32 md = c.G->max_deg ? c.G->max_deg : kFilterMax;
  u32 hs = 256;
  while (hs < 2 * (32 + 2 * std::min<u32>(md, kFilterMax)) && hs < kHashSlots) hs <<= 1;
  a.hstride = hs;
  const size_t smem = (size_t)(kThreads / 32) * hs * sizeof(u32);
  static std::atomic<int> occ_by_hs[2][16];  // zero-initialised (static storage)
  const int occ = cached_occupancy(occ_by_hs[stream][31 - __builtin_clz(hs)], [&] {
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
    engine::process_dispatch<CliqueApp>(c, 2, nl, Tc);
  }
}


}  // namespace

namespace engine {

bool cf_local_roots(Ctx& c, const u32* l1_src, u64 slo, u64 shi);  // clique_local.cu

// Builtin specialisations of a level (gpm_engine.cuh process()).
bool builtin_level(Ctx& c, int kind, int lev, const VLevels& L, u64 np) {
  const bool last = (lev == c.k - 2);
  if (kind == kBuiltinClique && lev >= 2 && last && !c.list_fn && c.g.oriented && c.siblings_complete &&
      c.G->n < (1u << 27) && !std::getenv("GPM_GENERIC_CF")) {
    cf_last_siblings(c, L.idx[lev - 1], L.vid[lev - 1], np, lev);
    return true;
  }
  return false;
}

// Builtin specialisations of a root slice (level-1 entries [slo, shi)).
bool builtin_roots(Ctx& c, int kind, const VLevels& L, const u32* l1_src, const u64* l1_start, u64 slo, u64 shi) {
  if (kind == kBuiltinMotif && c.k == 3 && l1_start && !std::getenv("GPM_GENERIC_MC")) {
    mc3_staged(*c.G, l1_start, slo, shi, c.d_hist, c.s, *c.tl, *c.st);
    return true;
  }
  if (kind == kBuiltinMotif && c.k == 4 && c.G->n < (1u << 30) &&  // union-set tags need ids < 2^30
      !std::getenv("GPM_GENERIC_MC")) {
    mc4_roots_staged(*c.G, L.idx[0], L.vid[0], shi - slo, c.d_hist, c.s, *c.tl, *c.st);
    return true;
  }
  if (kind == kBuiltinClique && c.G->oriented && c.G->n < (1u << 27) && !c.list_fn &&
      !std::getenv("GPM_GENERIC_L1")) {  // key = u << 5 | slot
    if (cf_local_roots(c, l1_src, slo, shi)) return true;  // k >= 4 counts on local rows
    process_l1_cf(c, L, l1_src, slo, shi);
    return true;
  }
  return false;
}

}  // namespace engine

void mine_vertex(const gpm_graph& G0, const gpm_config& cfg, cudaStream_t s, gpm_result& res, Stats& st,
                 Timeline& tl) {
  if (cfg.list_fn && cfg.app == GPM_APP_MC) throw Error(GPM_ECONFIG, "listing mode: TC/CF only (SPEC.md:458)");
  if (cfg.app == GPM_APP_MC) engine::mine<MotifApp>(G0, cfg, s, res, st, tl);
  else engine::mine<CliqueApp>(G0, cfg, s, res, st, tl);  // TC == CF with k = 3 (Listing 3)
}

}  // namespace gpm
