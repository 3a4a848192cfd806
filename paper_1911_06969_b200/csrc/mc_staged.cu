// mc_staged.cu — the last extension of 3-motif counting with the root's
// adjacency staged on chip (sm_100a).
//
// Reference: extend (Alg. 2) with MC's
// to_add = is_auto_canonical_vertex (Listing 4) and reduce by
// connectivity code (Listing 6), fused on the last level
// (PAPER.md:742-744).  DESIGN.md §3b.
//
// Level 1 of MC is every edge (v0, v1) with v0 < v1 (embedding_list.hpp:
// 178-192); the parents of one root v0 are S0 = {v in N(v0) : v > v0}, the
// upper suffix of v0's sorted CSR list.  Every 3-vertex candidate u satisfies
// u > v0, so only S0 matters for the membership tests.  Per parent (v0, v1):
//   pos 0: u in N(v0), u > v1          -> always accepted;
//          triangle iff u in N(v1), else wedge centred at v0
//   pos 1: u in N(v1), u > v0          -> accepted iff u not in N(v0);
//          wedge centred at v1
// The pos-1 candidates are streamed from HBM (coalesced, one lane per
// candidate) and tested against S0 held in a shared-memory hash set; a hit is
// the pair predicate adj(v0,u) = adj(v1,u) for the same u, which also decides
// the class of the pos-0 candidate u (u > v1).  So one streamed pass over the
// pos-1 candidates evaluates every candidate's to_add and pattern predicate:
//   tri(v0,v1)   = #{u in N(v1) ∩ S0 : u > v1}
//   X(v0,v1)     = #{u in N(v1) ∩ S0}
//   wedge@v0     = #{u in S0 : u > v1} - tri
//   wedge@v1     = #{u in N(v1) : u > v0} - X
// Roots with |S0| <= kWKeys stage S0 per warp (warp kernel); larger roots
// stage S0 per CTA in tiles of kBKeys (block kernel), each tile owning an id
// range so that every pos-1 candidate is streamed exactly once.
#include <cub/cub.cuh>

#include <algorithm>

#include "engine.hpp"
#include "pattern.cuh"

namespace gpm {

void scan_inplace(u64* data, u64 n, cudaStream_t s);

namespace {

constexpr int kT = 256;
constexpr int kWarps = kT / 32;
constexpr u32 kWSlots = 1024;   // per-warp hash slots (4 KB): load <= 1/8 up to kWKeys
constexpr u32 kWKeys = 256;     // roots with |S0| <= this use the warp kernel (load <= 1/4)
constexpr u32 kBSlots = 8192;   // default per-CTA hash slots (32 KB)
constexpr u32 kBKeys = 2048;    // default S0 tile of the block kernel (load 1/4; 1024: 130.8 ms, 2048: 127.5 ms on LJ22)
constexpr u32 kPB = 4096;       // parents per block item (warps grab 32 at a time)

// first index i in [b, e) with col[i] >= key
__device__ __forceinline__ u64 lower_bound_col(const u32* __restrict__ col, u64 b, u64 e, u32 key) {
  while (b < e) {
    const u64 mid = (b + e) >> 1;
    if (ldg(col + mid) < key) b = mid + 1;
    else e = mid;
  }
  return b;
}

struct Mc3Args {
  DevGraph g;
  const u64* l1s;        // first level-1 index per vertex (n+1 entries)
  u64 lo, hi;            // level-1 slice
  u32 vlo;               // root of level-1 index lo
  const u64* istart;     // per root (r - vlo): first item; nr+1 entries
  const u32* iroot;      // per item: r - vlo
  u64 nitems;
  u64 grab;
  unsigned long long* ctr;
  unsigned long long* hist;
  unsigned long long* cand;
  unsigned long long* moved;  // [0] streamed candidates, [1] staged keys, [2] parent visits, [3] pos-0 counted
  u32 codeT, codeW0, codeW1;
  u32 bkeys, bslots;          // block kernel: S0 tile keys, hash slots (shared memory)
};

// Per-root item counts.  small: |S0| <= kWKeys -> ceil(npar/32) warp items;
// big: ntiles * ceil(npar/kPB) block items.
__global__ void mc3_items_kernel(const u64* __restrict__ l1s, u64 lo, u64 hi, u32 vlo, u32 nr, u32 bkeys,
                                 u64* __restrict__ small, u64* __restrict__ big) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nr; i += (u64)gridDim.x * blockDim.x) {
    const u32 r = vlo + (u32)i;
    const u64 s = l1s[r], e = l1s[r + 1];
    const u64 ns = e - s;
    const u64 pa = max(s, lo), pb = min(e, hi);
    const u64 np = pb > pa ? pb - pa : 0;
    u64 cs = 0, cb = 0;
    if (np) {
      if (ns <= kWKeys) cs = (np + 31) / 32;
      else cb = ((ns + bkeys - 1) / bkeys) * ((np + kPB - 1) / kPB);
    }
    small[i] = cs;
    big[i] = cb;
  }
}

__global__ void mc3_iroot_kernel(const u64* __restrict__ istart, u32 nr, u32* __restrict__ iroot) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < nr; i += (u64)gridDim.x * blockDim.x)
    for (u64 t = istart[i], te = istart[i + 1]; t < te; ++t) iroot[t] = (u32)i;
}

// root owning level-1 index e: last r with l1s[r] <= e
__global__ void mc3_root_of_kernel(const u64* __restrict__ l1s, u32 n, u64 e0, u64 e1, u32* __restrict__ out) {
  const int t = threadIdx.x;
  if (t > 1) return;
  const u64 e = t == 0 ? e0 : e1;
  u64 lo = 0, hi = n;
  while (lo < hi) {
    const u64 mid = (lo + hi + 1) >> 1;
    if (l1s[mid] <= e) lo = mid;
    else hi = mid - 1;
  }
  out[t] = (u32)lo;
}

// Streams the pos-1 candidate ranges of <= 32 parents (lane i: col[st, st+len),
// parent vertex v1) against the staged set; adds the warp's hits (X) and hits
// above v1 (tri).  Segments of >= 32 candidates are streamed one at a time
// (warp-uniform parent, coalesced, two loads in flight); shorter ones are
// packed 32 candidates per step with the OR-reduction lane -> parent map.
__device__ __forceinline__ void stream_parents(const u32* __restrict__ col, const u32* T, u32 sh, u32 mask, u64 st,
                                               u32 len, u32 v1, u64* scb, u32* sex, u32* sv1, unsigned long long& X,
                                               unsigned long long& tri) {
  const int lane = threadIdx.x & 31;
  u32 cx = 0, ct = 0;
  // ---- long segments, one after the other
  u32 todo = __ballot_sync(0xffffffffu, len >= 32);
  while (todo) {
    const int i = __ffs(todo) - 1;
    todo &= todo - 1;
    const u64 b = __shfl_sync(0xffffffffu, st, i);
    const u32 L = __shfl_sync(0xffffffffu, len, i);
    const u32 w = __shfl_sync(0xffffffffu, v1, i);
    u32 j = 0;
    for (; j + 256 <= L; j += 256) {  // eight loads in flight per lane
      u32 u[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) u[q] = ldg(col + b + j + 32 * q + lane);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const bool h = hb_has(T, sh, mask, u[q]);
        cx += __popc(__ballot_sync(0xffffffffu, h));
        ct += __popc(__ballot_sync(0xffffffffu, h && u[q] > w));
      }
    }
    for (; j + 128 <= L; j += 128) {  // four loads in flight per lane
      u32 u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) u[q] = ldg(col + b + j + 32 * q + lane);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool h = hb_has(T, sh, mask, u[q]);
        cx += __popc(__ballot_sync(0xffffffffu, h));
        ct += __popc(__ballot_sync(0xffffffffu, h && u[q] > w));
      }
    }
    for (; j + 64 <= L; j += 64) {
      const u32 u0 = ldg(col + b + j + lane);
      const u32 u1 = ldg(col + b + j + 32 + lane);
      const bool h0 = hb_has(T, sh, mask, u0);
      const bool h1 = hb_has(T, sh, mask, u1);
      cx += __popc(__ballot_sync(0xffffffffu, h0)) + __popc(__ballot_sync(0xffffffffu, h1));
      ct += __popc(__ballot_sync(0xffffffffu, h0 && u0 > w)) + __popc(__ballot_sync(0xffffffffu, h1 && u1 > w));
    }
    for (; j < L; j += 32) {
      const bool v = j + lane < L;
      const u32 u0 = v ? ldg(col + b + j + lane) : 0u;
      const bool h0 = v && hb_has(T, sh, mask, u0);
      cx += __popc(__ballot_sync(0xffffffffu, h0));
      ct += __popc(__ballot_sync(0xffffffffu, h0 && u0 > w));
    }
  }
  // ---- short segments, packed
  const u32 sl = len < 32 ? len : 0u;
  u32 incl = sl;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  const u32 total = __shfl_sync(0xffffffffu, incl, 31);
  if (total) {
    const u32 nz = __ballot_sync(0xffffffffu, sl > 0);
    const u32 rank = __popc(nz & lanemask_lt());
    __syncwarp();
    if (sl > 0) {
      scb[rank] = st;
      sex[rank] = incl - sl;
      sv1[rank] = v1;
    }
    const u32 nnz = __popc(nz);
    __syncwarp();
    u32 P = 0;
    for (u32 jb = 0; jb < total; jb += 32) {
      const u32 jj = jb + lane;
      const u32 x = (P + 1 + lane < nnz) ? sex[P + 1 + lane] : 0xffffffffu;
      const u32 bit = (x - jb < 32u) ? (1u << (x - jb)) : 0u;
      const u32 starts = __reduce_or_sync(0xffffffffu, bit);
      const u32 myp = min(P + __popc(starts & (lanemask_lt() | (1u << lane))), nnz - 1);
      P += __popc(starts);
      bool hit = false, t = false;
      if (jj < total) {
        const u32 u = ldg(col + scb[myp] + (jj - sex[myp]));
        hit = hb_has(T, sh, mask, u);
        t = hit && u > sv1[myp];
      }
      cx += __popc(__ballot_sync(0xffffffffu, hit));
      ct += __popc(__ballot_sync(0xffffffffu, t));
    }
    __syncwarp();
  }
  X += cx;
  tri += ct;
}

// 5 CTAs / SM for both 3-MC kernels (LJ22: 218.6 -> 216.2 ms; 6: 218.3 ms)
__global__ void __launch_bounds__(kT, 5) mc3_warp_kernel(Mc3Args a) {
  extern __shared__ __align__(16) u32 s_wtab[];  // [kWarps][kWSlots]
  __shared__ u64 s_cb[kWarps][32];
  __shared__ u32 s_ex[kWarps][32];
  __shared__ u32 s_v1[kWarps][32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  u32* T = s_wtab + wid * kWSlots;
  const DevGraph& g = a.g;
  unsigned long long aX = 0, aTri = 0, aC0 = 0, aLen = 0, aCand = 0, aStg = 0, aVis = 0;
  u32 troot = 0xffffffffu, sh = 0, mask = 0;
  u64 grab = 0, left = 0;
  for (;;) {
    if (left == 0) {
      u64 g_ = 0;
      if (lane == 0) g_ = atomicAdd(a.ctr, (unsigned long long)a.grab);
      grab = __shfl_sync(0xffffffffu, g_, 0);
      left = a.grab;
    }
    const u64 item = grab++;
    --left;
    if (item >= a.nitems) break;
    const u32 rr = ldg(a.iroot + item);
    const u32 r = a.vlo + rr;
    const u64 s = ldg(a.l1s + r), e = ldg(a.l1s + r + 1);
    const u32 ns = (u32)(e - s);
    const u64 ob = ldg(g.off + r), oe = ldg(g.off + r + 1);
    const u64 sb = oe - ns;  // S0 = col[sb, oe)
    if (r != troot) {
      troot = r;
      u32 cap = 64;
      while (cap < 8 * ns && cap < kWSlots) cap <<= 1;
      hb_geom(cap, sh, mask);  // bucketised table: mask = bucket mask
      for (u32 i = lane * 4; i < cap; i += 128) *reinterpret_cast<uint4*>(T + i) = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
      __syncwarp();
      for (u32 i = lane; i < ns; i += 32) hb_insert(T, sh, mask, ldg(g.col + sb + i));
      if (lane == 0) aStg += ns;
      __syncwarp();
    }
    const u64 pa0 = max(s, a.lo);
    const u64 pa = pa0 + 32 * (item - ldg(a.istart + rr));
    const u64 pb = min(min(e, a.hi), pa + 32);
    const u64 p = pa + lane;
    u64 st = 0;
    u32 len = 0, v1 = 0;
    if (p < pb) {
      const u32 ip = (u32)(p - s);
      v1 = ldg(g.col + sb + ip);
      const u64 b1 = ldg(g.off + v1), e1 = ldg(g.off + v1 + 1);
      st = lower_bound_col(g.col, b1, e1, r + 1);
      len = (u32)(e1 - st);
      aC0 += ns - ip - 1;
      aLen += len;
      aCand += (oe - ob) + (e1 - b1);
      ++aVis;
    }
    stream_parents(g.col, T, sh, mask, st, len, v1, s_cb[wid], s_ex[wid], s_v1[wid], aX, aTri);
  }
  // per-lane partials (aC0, aLen, aCand, aVis) + warp-uniform (aX, aTri)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    aC0 += __shfl_xor_sync(0xffffffffu, aC0, o);
    aLen += __shfl_xor_sync(0xffffffffu, aLen, o);
    aCand += __shfl_xor_sync(0xffffffffu, aCand, o);
    aVis += __shfl_xor_sync(0xffffffffu, aVis, o);
  }
  if (lane == 0) {
    if (aTri) atomicAdd(a.hist + a.codeT, aTri);
    if (aC0 - aTri) atomicAdd(a.hist + a.codeW0, aC0 - aTri);
    if (aLen - aX) atomicAdd(a.hist + a.codeW1, aLen - aX);
    if (aCand) atomicAdd(a.cand, aCand);
    atomicAdd(a.moved + 0, aLen);
    atomicAdd(a.moved + 1, aStg);
    atomicAdd(a.moved + 2, aVis);
    atomicAdd(a.moved + 3, aC0);
  }
}

// Roots with |S0| > kWKeys: item = (root, S0 tile, chunk of <= kPB parents).
// The CTA stages the tile; warps grab 32 parents at a time from the chunk and
// stream their candidates inside the tile's id range [idlo, idhi).
__global__ void __launch_bounds__(kT, 5) mc3_block_kernel(Mc3Args a) {
  extern __shared__ __align__(16) u32 s_btab[];
  __shared__ u64 s_cb[kWarps][32];
  __shared__ u32 s_ex[kWarps][32];
  __shared__ u32 s_v1[kWarps][32];
  __shared__ u64 s_item;
  __shared__ u32 s_next;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const DevGraph& g = a.g;
  unsigned long long aX = 0, aTri = 0, aC0 = 0, aLen = 0, aCand = 0, aStg = 0, aVis = 0;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) {
      s_item = atomicAdd(a.ctr, 1ull);
      s_next = 0;
    }
    __syncthreads();
    const u64 item = s_item;
    if (item >= a.nitems) break;
    const u32 rr = ldg(a.iroot + item);
    const u32 r = a.vlo + rr;
    const u64 s = ldg(a.l1s + r), e = ldg(a.l1s + r + 1);
    const u32 ns = (u32)(e - s);
    const u64 ob = ldg(g.off + r), oe = ldg(g.off + r + 1);
    const u64 sb = oe - ns;
    const u64 pa0 = max(s, a.lo), pe = min(e, a.hi);
    const u64 nch = (pe - pa0 + kPB - 1) / kPB;
    const u32 ntiles = (ns + a.bkeys - 1) / a.bkeys;
    const u64 q = item - ldg(a.istart + rr);
    const u32 t = (u32)(q / nch);
    const u64 c = q % nch;
    const u32 k0 = t * a.bkeys, k1 = min(ns, k0 + a.bkeys);
    u32 cap = 1024;  // table sized to the tile: load <= 1/8, cleared in O(cap)
    while (cap < 8 * (k1 - k0) && cap < a.bslots) cap <<= 1;
    u32 sh, mask;
    hb_geom(cap, sh, mask);
    for (u32 i = threadIdx.x * 4; i < cap; i += kT * 4)
      *reinterpret_cast<uint4*>(s_btab + i) = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    __syncthreads();
    for (u32 i = k0 + threadIdx.x; i < k1; i += kT) hb_insert(s_btab, sh, mask, ldg(g.col + sb + i));
    if (threadIdx.x == 0) aStg += k1 - k0;
    __syncthreads();
    if (threadIdx.x == 0 && ntiles > 1) a.moved[4] = 1;  // path flag (tests)
    const u32 idlo = (t == 0) ? r + 1 : ldg(g.col + sb + k0);
    const bool last_tile = (t + 1 == ntiles);
    const u32 idhi = last_tile ? 0xffffffffu : ldg(g.col + sb + k1);
    const u64 cb = pa0 + c * kPB;
    const u32 cn = (u32)(min(pe, cb + kPB) - cb);
    for (;;) {
      u32 sub = 0;
      if (lane == 0) sub = atomicAdd(&s_next, 32u);
      sub = __shfl_sync(0xffffffffu, sub, 0);
      if (sub >= cn) break;
      const u64 p = cb + sub + lane;
      u64 st = 0;
      u32 len = 0, v1 = 0;
      if (sub + lane < cn) {
        const u32 ip = (u32)(p - s);
        v1 = ldg(g.col + sb + ip);
        const u64 b1 = ldg(g.off + v1), e1 = ldg(g.off + v1 + 1);
        st = lower_bound_col(g.col, b1, e1, idlo);
        const u64 en = last_tile ? e1 : lower_bound_col(g.col, st, e1, idhi);
        len = (u32)(en - st);
        aLen += len;
        ++aVis;
        if (t == 0) {
          aC0 += ns - ip - 1;
          aCand += (oe - ob) + (e1 - b1);
        }
      }
      stream_parents(g.col, s_btab, sh, mask, st, len, v1, s_cb[wid], s_ex[wid], s_v1[wid], aX, aTri);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    aC0 += __shfl_xor_sync(0xffffffffu, aC0, o);
    aLen += __shfl_xor_sync(0xffffffffu, aLen, o);
    aCand += __shfl_xor_sync(0xffffffffu, aCand, o);
    aVis += __shfl_xor_sync(0xffffffffu, aVis, o);
  }
  if (lane == 0) {
    if (aTri) atomicAdd(a.hist + a.codeT, aTri);
    if (aC0 - aTri) atomicAdd(a.hist + a.codeW0, aC0 - aTri);  // mod 2^64: partial sums may be negative
    if (aLen - aX) atomicAdd(a.hist + a.codeW1, aLen - aX);
    if (aCand) atomicAdd(a.cand, aCand);
    atomicAdd(a.moved + 0, aLen);
    if (aStg) atomicAdd(a.moved + 1, aStg);
    atomicAdd(a.moved + 2, aVis);
    atomicAdd(a.moved + 3, aC0);
  }
}

// ---------------------------------------------------------------------------
// 4-MC last extension.  Parents are level-2 embeddings (v0, v1, v2) whose
// level-1 parent q = (v0, v1) groups them (the level is written in parent
// order).  With S_i = N(v_i) ∩ (>v0), m = max(v1, v2), the candidates are
//   pos 0: u in S0, u > m                 -> accepted; class by (u~v1, u~v2)
//   pos 1: u in S1, u > v2, u not in S0   -> accepted; class by u~v2
//   pos 2: u in S2, u not in S0 ∪ S1      -> accepted
// (SPEC.md:214 + "emit u only from its first adjacent position").  The warp
// stages S0 (per root) and S1 (per group) as shared-memory hash sets and
// I01 = S0 ∩ S1 (sorted, per-warp scratch); each child streams S2 from HBM,
// one lane per candidate, probing both sets:
//   e2  = #{u in S2 : u !in S0, u !in S1}
//   e11 = #{u in S2 : u in S0, u in S1, u > m}
//   e01 = #{u in S2 : u in S0, u !in S1, u > m}
//   e12 = #{u in S2 : u in S1, u !in S0, u > v2}
// and the classes follow from the same predicates:
//   pos0 (v1,v2 adj) e11 | (v1) #I01>m - e11 | (v2) e01 | () #S0>m - #I01>m - e01
//   pos1 (v2 adj) e12    | () #S1>v2 - #I01>v2 - e12          pos2: e2
// Sets larger than the hash capacity are probed by binary search in HBM.
constexpr int kT4 = 256;
constexpr int kW4 = kT4 / 32;
constexpr u32 k4Slots = 1024;  // per-warp union table S0 ∪ S1 (4 KB)
constexpr u32 k4Keys = 512;    // |S0| + |S1| above this -> binary search in HBM
constexpr u64 k4Q = 8;         // level-1 parents per warp work item

struct Mc4Args {
  DevGraph g;
  const u32* l1i;   // level-1 v0 (slice-relative)
  const u32* l1v;   // level-1 v1
  u64 nq;           // level-1 parents in the slice
  u64 nitems;
  unsigned long long* ctr;
  unsigned long long* hist;   // 64 bins
  unsigned long long* cand;   // [0] level-2 candidates, [1] level-3 candidates
  unsigned long long* moved;  // [0] streamed S2 candidates, [1] staged keys, [2] level-2 children, [3] rank-counted, [4] path flag
  u32* scratch;               // per warp: max_deg entries for I01
  u64 scratch_stride;
  u32 pm_bits[4];             // pmask value for (v0~v2, v1~v2)
  u32 cl_bits[7];
};

// Union hash set of S0 and S1: slot = (id << 2) | (in S0) | (in S1) << 1
// (ids < 2^30).  One probe answers both memberships.
__device__ __forceinline__ u32 us_flags(const u32* T, u32 sh, u32 bmask, u32 v) {
  // slot = id << 2 | flags: (slot ^ v << 2) < 4 <=> same id; the empty slot
  // ~0u never matches (ids < 2^30 - 1)
  const u32 vk = v << 2;
  u32 b = (v * kHashMul) >> sh;  // bucketised (4 slots, one LDS.128), see hb_has
  for (;;) {
    const uint4 x = *reinterpret_cast<const uint4*>(T + 4 * b);
    if ((x.x ^ vk) < 4u) return x.x & 3u;
    if ((x.y ^ vk) < 4u) return x.y & 3u;
    if ((x.z ^ vk) < 4u) return x.z & 3u;
    if ((x.w ^ vk) < 4u) return x.w & 3u;
    if (x.w == kEmpty) return 0;
    b = (b + 1) & bmask;
  }
}
// insert v with flag f; if v is present OR the flag in; returns true if present
// (keys inserted concurrently are distinct, so a lost CAS just moves on)
__device__ __forceinline__ bool us_add(u32* T, u32 sh, u32 bmask, u32 v, u32 f) {
  u32 b = (v * kHashMul) >> sh;
  for (;;) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      u32 x = T[4 * b + k];
      if (x == kEmpty) {
        x = atomicCAS(T + 4 * b + k, kEmpty, (v << 2) | f);
        if (x == kEmpty) return false;
      }
      if ((x >> 2) == v) {
        atomicOr(T + 4 * b + k, f);
        return true;
      }
    }
    b = (b + 1) & bmask;
  }
}

// #{x in sorted a[0, n) : x > key}
__device__ __forceinline__ u32 count_gt_global(const u32* __restrict__ a, u32 n, u32 key) {
  u32 lo = 0, hi = n;
  while (lo < hi) {
    const u32 mid = (lo + hi) >> 1;
    if (ldg(a + mid) <= key) lo = mid + 1;
    else hi = mid;
  }
  return n - lo;
}
__device__ __forceinline__ u32 count_gt_plain(const u32* a, u32 n, u32 key) {
  u32 lo = 0, hi = n;
  while (lo < hi) {
    const u32 mid = (lo + hi) >> 1;
    if (a[mid] <= key) lo = mid + 1;
    else hi = mid;
  }
  return n - lo;
}

// The HBM fallback is out of line: the kernels inline flags() at ~10 sites
// and their loop bodies are instruction-cache sensitive (a second inlined
// copy of the 4-MC step body measured 2x slower).
__device__ __forceinline__ u32 us_flags_sorted(const u32* s0, u32 n0, const u32* s1, u32 n1, u32 v) {
  return (contains_sorted(s0, n0, v) ? 1u : 0u) | (contains_sorted(s1, n1, v) ? 2u : 0u);
}
struct UnionSet {
  const u32* T;      // nullptr -> probe the sorted lists in HBM
  const u32* s0;
  const u32* s1;
  u32 n0, n1, sh, mask;
  __device__ __forceinline__ u32 flags(u32 v) const {
    if (T) return us_flags(T, sh, mask, v);
    return us_flags_sorted(s0, n0, s1, n1, v);
  }
};

// Fused level 2 + last level of 4-MC: items are ranges of level-1 parents
// q = (v0, v1); per q the warp stages S0 ∪ S1 once and walks q's level-2
// children in place -- {u in S0 : u > v1} (pos 0, the contiguous suffix of
// the sorted S0 above v1) then {u in S1 : u !in S0} (pos 1, first-adjacent
// rule) -- so level 2 is never materialised (no inspection / execution
// passes, no idx2 / vid2 round trip through HBM).  The children are exactly
// is_auto_canonical_vertex's accepted candidates of (v0, v1)
// (gpm_engine.cuh).
// 5 CTAs / SM (48 registers, ~90 B of spills): latency-bound probes and
// searches want warps more than registers (4 CTAs: 386 ms, 5: 366 ms on MC4)
__global__ void __launch_bounds__(kT4, 5) mc4_roots_kernel(Mc4Args a) {
  __shared__ __align__(16) u32 s_tab[kW4][k4Slots];
  __shared__ u64 s_cb[kW4][32];
  __shared__ u32 s_ex[kW4][32];
  __shared__ u32 s_v2[kW4][32];
  __shared__ unsigned long long s_h[kW4][32];
  __shared__ unsigned long long s_kids[kW4], s_cand[kW4];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const DevGraph& g = a.g;
  u32* T = s_tab[wid];
  u32* I01 = a.scratch + (blockIdx.x * (u64)kW4 + wid) * a.scratch_stride;
  s_h[wid][lane] = 0;
  if (lane == 0) s_kids[wid] = s_cand[wid] = 0;
  // per-item counters (streamed, staged, rank-counted), folded into the
  // unused class slot 7 of each parent-mask row of s_h per item
  u32 aLen = 0, aStg = 0, aRank = 0;
  UnionSet U{};
  u32 v0 = 0, v1 = 0, n01 = 0;
  u32 deg01 = 0, deg0 = 0;  // degrees < 2^32
  u32 cur_v0 = 0xffffffffu;

  // one warp step over up to 32 children (lane-owned v2 where valid).  The
  // classes only matter summed per parent-mask value pv, so event counts go
  // straight into s_h (val[1] = Im - e11 etc.: +e into one class, -e into
  // its rank partner; the u64 sums wrap back to the exact totals).
  // a0 / b1: #S0 > max(v1, v2) / #S1 > v2 when known from the child's index
  // in the staged list (~0u: binary search).
  auto step = [&](bool valid, u32 v2, u32 a0, u32 b1) {
    u32 len = 0, pmv = 0;
    u64 st = 0;
    if (valid) {
      const u64 b2 = ldg(g.off + v2), e2 = ldg(g.off + v2 + 1);
      st = lower_bound_col(g.col, b2, e2, v0 + 1);
      len = (u32)(e2 - st);
      pmv = U.flags(v2);  // bit 0: v2 ~ v0, bit 1: v2 ~ v1
      aLen += len;
    }
    {  // level-3 candidates of the step's children (deg v0 + deg v1 + deg v2),
       // summed in 16-bit halves so the warp sums fit 32 bits
      const u32 cc = valid ? deg01 + (u32)(ldg(g.off + v2 + 1) - ldg(g.off + v2)) : 0u;
      const u32 lo = __reduce_add_sync(0xffffffffu, cc & 0xffffu), hi = __reduce_add_sync(0xffffffffu, cc >> 16);
      if (lane == 0) s_cand[wid] += (unsigned long long)lo + ((unsigned long long)hi << 16);
    }
    // long S2 ranges (>= 32 candidates): one child at a time, warp-uniform
    // thresholds, coalesced loads, two in flight (4: 366 ms, 2: 361, 1: 365),
    // per-lane event counters
    u32 todo = __ballot_sync(0xffffffffu, len >= 32);
    while (todo) {
      const int i = __ffs(todo) - 1;
      todo &= todo - 1;
      const u64 b = __shfl_sync(0xffffffffu, st, i);
      const u32 L = __shfl_sync(0xffffffffu, len, i);
      const u32 cv2 = __shfl_sync(0xffffffffu, v2, i);
      const u32 cpv = __shfl_sync(0xffffffffu, pmv, i);
      const u32 cm = max(v1, cv2);
      u32 c2 = 0, c11 = 0, c01 = 0, c12 = 0;
      u32 j = 0;
      for (; j + 64 <= L; j += 64) {
        u32 u[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) u[q] = ldg(g.col + b + j + 32 * q + lane);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const u32 f = U.flags(u[q]);
          c2 += (f == 0 && u[q] > v0);
          c11 += (f == 3 && u[q] > cm);
          c01 += (f == 1 && u[q] > cm);
          c12 += (f == 2 && u[q] > cv2);
        }
      }
      for (; j < L; j += 32) {
        const bool ok = j + lane < L;
        const u32 u0 = ok ? ldg(g.col + b + j + lane) : 0u;
        const u32 f0 = ok ? U.flags(u0) : 4u;
        c2 += (f0 == 0 && u0 > v0);
        c11 += (f0 == 3 && u0 > cm);
        c01 += (f0 == 1 && u0 > cm);
        c12 += (f0 == 2 && u0 > cv2);
      }
      c2 = __reduce_add_sync(0xffffffffu, c2);
      c11 = __reduce_add_sync(0xffffffffu, c11);
      c01 = __reduce_add_sync(0xffffffffu, c01);
      c12 = __reduce_add_sync(0xffffffffu, c12);
      if (lane == 0) {
        unsigned long long* h = s_h[wid] + cpv * 8;
        h[0] += c11;
        h[1] -= c11;
        h[2] += c01;
        h[3] -= c01;
        h[4] += c12;
        h[5] -= c12;
        h[6] += c2;
        aRank -= c11 + c01 + c12;
      }
    }
    // short S2 ranges: packed 32 candidates per step (OR-reduction lane ->
    // child map); each candidate adds one to a packed per-lane counter of its
    // (child pv, event) bin -- 8-bit fields, a lane sees < 32 candidates here
    const u32 sl = len < 32 ? len : 0u;
    u32 incl = sl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const u32 total = __shfl_sync(0xffffffffu, incl, 31);
    if (total) {
      const u32 nz = __ballot_sync(0xffffffffu, sl > 0);
      const u32 rank = __popc(nz & lanemask_lt());
      const u32 nnz = __popc(nz);
      if (sl > 0) {
        s_cb[wid][rank] = st;
        s_ex[wid][rank] = incl - sl;
        s_v2[wid][rank] = v2 | (pmv << 30);  // ids < 2^30
      }
      __syncwarp();
      u32 acc0 = 0, acc1 = 0, acc2 = 0;  // pv 1, 2, 3 (pv 0 never occurs); 8-bit field per event
      u32 P = 0;
      for (u32 jb = 0; jb < total; jb += 32) {
        const u32 j = jb + lane;
        const u32 x = (P + 1 + lane < nnz) ? s_ex[wid][P + 1 + lane] : 0xffffffffu;
        const u32 bit = (x - jb < 32u) ? (1u << (x - jb)) : 0u;
        const u32 starts = __reduce_or_sync(0xffffffffu, bit);
        const u32 c = P + __popc(starts & (lanemask_lt() | (1u << lane)));
        P += __popc(starts);
        if (j < total) {
          const u32 u = ldg(g.col + s_cb[wid][c] + (j - s_ex[wid][c]));
          const u32 w = s_v2[wid][c];
          const u32 cv2 = w & 0x3fffffffu;
          const u32 f = U.flags(u);
          // event field: 0 e11, 1 e01, 2 e12, 3 e2
          const bool hit = f == 0 ? u > v0 : (f == 2 ? u > cv2 : u > max(v1, cv2));
          const u32 ev = f == 0 ? 3u : (f == 3 ? 0u : f);
          const u32 inc = hit ? 1u << (8 * ev) : 0u;
          const u32 k = w >> 30;
          acc0 += k == 1 ? inc : 0u;
          acc1 += k == 2 ? inc : 0u;
          acc2 += k == 3 ? inc : 0u;
        }
      }
      // fields summed over the warp as 16-bit lanes (< 32 x 32 per field)
#pragma unroll
      for (int pv = 1; pv <= 3; ++pv) {
        const u32 A = pv == 1 ? acc0 : (pv == 2 ? acc1 : acc2);
        const u32 lo = __reduce_add_sync(0xffffffffu, A & 0x00ff00ffu);         // events 0, 2
        const u32 hi = __reduce_add_sync(0xffffffffu, (A >> 8) & 0x00ff00ffu);  // events 1, 3
        if (lane == 0 && (lo | hi)) {
          const u32 e11 = lo & 0xffffu, e12 = lo >> 16, e01 = hi & 0xffffu, e2 = hi >> 16;
          unsigned long long* h = s_h[wid] + pv * 8;
          h[0] += e11;
          h[1] -= e11;
          h[2] += e01;
          h[3] -= e01;
          h[4] += e12;
          h[5] -= e12;
          h[6] += e2;
          aRank -= e11 + e01 + e12;
        }
      }
      __syncwarp();
    }
    // ---- per-child rank terms, reduced per parent-mask value
    u32 r1 = 0, r3 = 0, r5 = 0;
    if (valid) {
      const u32 m = max(v1, v2);
      const u32 A0 = a0 != ~0u ? a0 : count_gt_global(U.s0, U.n0, m);
      const u32 B1 = b1 != ~0u ? b1 : count_gt_global(U.s1, U.n1, v2);
      const u32 Im = count_gt_plain(I01, n01, m);
      const u32 I2 = count_gt_plain(I01, n01, v2);
      r1 = Im;
      r3 = A0 - Im;
      r5 = B1 - I2;
      aRank += r1 + r3 + r5;
    }
#pragma unroll
    for (u32 pv = 1; pv < 4; ++pv) {
      const bool mine = valid && pmv == pv;
      if (__ballot_sync(0xffffffffu, mine) == 0) continue;
      const u32 s1_ = __reduce_add_sync(0xffffffffu, mine ? r1 : 0u);
      const u32 s3_ = __reduce_add_sync(0xffffffffu, mine ? r3 : 0u);
      const u32 s5_ = __reduce_add_sync(0xffffffffu, mine ? r5 : 0u);
      if (lane == 0) {
        s_h[wid][pv * 8 + 1] += s1_;
        s_h[wid][pv * 8 + 3] += s3_;
        s_h[wid][pv * 8 + 5] += s5_;
      }
    }
    __syncwarp();
  };

  for (;;) {
    u64 it_ = 0;
    if (lane == 0) it_ = atomicAdd(a.ctr, 1ull);
    const u64 item = __shfl_sync(0xffffffffu, it_, 0);
    if (item >= a.nitems) break;
    const u64 qend = min(a.nq, (item + 1) * k4Q);
    for (u64 q = item * k4Q; q < qend; ++q) {
      // ---- stage S0 ∪ S1 (flags) and I01 = S0 ∩ S1 in ascending order
      const u32 nv0 = ldg(a.l1i + q);
      v1 = ldg(a.l1v + q);
      if (nv0 != cur_v0) {  // level 1 is in v0 order: S0 is found once per root
        cur_v0 = v0 = nv0;
        const u64 b0 = ldg(g.off + v0), e0 = ldg(g.off + v0 + 1);
        const u64 s0b = lower_bound_col(g.col, b0, e0, v0 + 1);
        U.s0 = g.col + s0b;
        U.n0 = (u32)(e0 - s0b);
        deg0 = (u32)(e0 - b0);
      }
      const u64 b1 = ldg(g.off + v1), e1 = ldg(g.off + v1 + 1);
      const u64 s1b = lower_bound_col(g.col, b1, e1, v0 + 1);
      U.s1 = g.col + s1b;
      U.n1 = (u32)(e1 - s1b);
      deg01 = deg0 + (u32)(e1 - b1);
      const bool fits = U.n0 + U.n1 <= k4Keys;
      if (fits) {
        u32 cap = 64;
        while (cap < 8 * (U.n0 + U.n1) && cap < k4Slots) cap <<= 1;  // load <= 1/8 while it fits
        hb_geom(cap, U.sh, U.mask);
        __syncwarp();
        for (u32 i = lane * 4; i < cap; i += 128)
          *reinterpret_cast<uint4*>(T + i) = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
        __syncwarp();
        for (u32 i = lane; i < U.n0; i += 32) us_add(T, U.sh, U.mask, ldg(U.s0 + i), 1u);
        __syncwarp();
      }
      n01 = 0;
      for (u32 jb = 0; jb < U.n1; jb += 32) {
        const u32 j = jb + lane;
        u32 u = 0;
        bool hit = false;
        if (j < U.n1) {
          u = ldg(U.s1 + j);
          hit = fits ? us_add(T, U.sh, U.mask, u, 2u) : contains_sorted(U.s0, U.n0, u);
        }
        const u32 bm = __ballot_sync(0xffffffffu, hit);
        if (hit) I01[n01 + __popc(bm & lanemask_lt())] = u;
        n01 += __popc(bm);
      }
      U.T = fits ? T : nullptr;
      if (!fits && lane == 0) a.moved[4] = 1;  // path flag (tests)
      if (lane == 0) {
        aStg += (fits ? U.n0 : 0u) + U.n1;
        s_h[wid][23] += deg01;      // slot 23 (pv 2, class 7): level-2 candidates
      }
      __syncwarp();
      // ---- level-2 children: pos 0 = the suffix of S0 above v1, then pos 1 =
      // the S1 members not adjacent to v0; one step loop over the
      // concatenation (one inlined copy of the step body)
      const u32 p1 = U.n0 - count_gt_global(U.s0, U.n0, v1);
      const u32 nA = U.n0 - p1, nAll = nA + U.n1;
      for (u32 jb = 0; jb < nAll; jb += 32) {
        const u32 j = jb + lane;
        bool valid = j < nAll;
        u32 v2 = 0, a0 = ~0u, b1 = ~0u;
        if (valid) {
          if (j < nA) {  // v2 = S0[p1 + j] > v1: #S0 > v2 from its index
            v2 = ldg(U.s0 + p1 + j);
            a0 = nA - j - 1;
          } else {  // v2 = S1[t]: #S1 > v2 from its index
            v2 = ldg(U.s1 + (j - nA));
            b1 = nAll - j - 1;
            valid = !(U.flags(v2) & 1u);
          }
        }
        const u32 nk = __popc(__ballot_sync(0xffffffffu, valid));
        if (lane == 0) s_kids[wid] += nk;
        step(valid, v2, a0, b1);
      }
    }
    {
      const u32 l = __reduce_add_sync(0xffffffffu, aLen), rk = __reduce_add_sync(0xffffffffu, aRank);
      if (lane == 0) {
        s_h[wid][7] += l;
        s_h[wid][15] += aStg;
        s_h[wid][31] += rk;
      }
      aLen = aStg = aRank = 0;
    }
  }
  __syncwarp();
  {  // slots 7 / 15 / 31: streamed, staged, rank-counted; 23: level-2 candidates
    const unsigned long long v = lane < 4 ? s_h[wid][8 * lane + 7] : 0ull;
    if (v) atomicAdd(lane == 2 ? a.cand : a.moved + lane, v);
  }
  {
    const u32 pv = lane >> 3, cl = lane & 7;
    const unsigned long long v = s_h[wid][lane];
    if (cl < 7 && v) atomicAdd(a.hist + (a.pm_bits[pv] | a.cl_bits[cl]), v);
  }
  if (lane == 0) {
    if (s_cand[wid]) atomicAdd(a.cand + 1, s_cand[wid]);
    if (s_kids[wid]) atomicAdd(a.moved + 2, s_kids[wid]);
  }
}

inline unsigned grid1(u64 items) { return (unsigned)std::max<u64>(1, std::min<u64>((items + 255) / 256, 1u << 20)); }

}  // namespace

void mc3_staged(const gpm_graph& G, const u64* l1s, u64 lo, u64 hi, unsigned long long* d_hist, cudaStream_t s,
                Timeline& tl, Stats& st) {
  if (hi <= lo) return;
  const u64 np = hi - lo;
  DBuf<u32> vv(2, s);
  mc3_root_of_kernel<<<1, 32, 0, s>>>(l1s, G.n, lo, hi - 1, vv.get());
  GPM_CUDA(cudaGetLastError());
  u32 vr[2];
  GPM_CUDA(cudaMemcpyAsync(vr, vv.get(), sizeof vr, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  const u32 nr = vr[1] - vr[0] + 1;
  DBuf<u64> ismall(nr + 1, s), ibig(nr + 1, s);
  GPM_CUDA(cudaMemsetAsync(ismall.get() + nr, 0, sizeof(u64), s));
  GPM_CUDA(cudaMemsetAsync(ibig.get() + nr, 0, sizeof(u64), s));
  // block-kernel tile: GPM_MC3_TILE keys (default kBKeys) at load <= 1/4..1/8
  // (the tile's hash has a power-of-two capacity: the knob is rounded up to
  // a power of two in [256, 8192]; 3072 used to overrun the table)
  static const u32 tile_env = [] {
    const char* e = std::getenv("GPM_MC3_TILE");
    const long t = e ? std::atol(e) : 0;
    if (t <= 0) return 0u;
    u32 p = 256;
    while (p < (u32)std::min<long>(t, 8192)) p <<= 1;
    return p;
  }();
  const u32 bkeys = tile_env ? tile_env : kBKeys;
  const u32 bslots = std::max<u32>(kBSlots, bkeys * 4 > kBSlots ? (bkeys * 4 + 1023) & ~1023u : kBSlots);
  mc3_items_kernel<<<grid1(nr), 256, 0, s>>>(l1s, lo, hi, vr[0], nr, bkeys, ismall.get(), ibig.get());
  GPM_CUDA(cudaGetLastError());
  scan_inplace(ismall.get(), nr + 1, s);
  scan_inplace(ibig.get(), nr + 1, s);
  u64 NS = 0, NB = 0;
  GPM_CUDA(cudaMemcpyAsync(&NS, ismall.get() + nr, sizeof(u64), cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaMemcpyAsync(&NB, ibig.get() + nr, sizeof(u64), cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  tl.launches += 6;
  DBuf<u32> rs(std::max<u64>(1, NS), s), rb(std::max<u64>(1, NB), s);
  if (NS) mc3_iroot_kernel<<<grid1(nr), 256, 0, s>>>(ismall.get(), nr, rs.get());
  if (NB) mc3_iroot_kernel<<<grid1(nr), 256, 0, s>>>(ibig.get(), nr, rb.get());
  GPM_CUDA(cudaGetLastError());
  DBuf<unsigned long long> ctr(2, s), cand(6, s);
  GPM_CUDA(cudaMemsetAsync(ctr.get(), 0, 2 * sizeof(unsigned long long), s));
  GPM_CUDA(cudaMemsetAsync(cand.get(), 0, 6 * sizeof(unsigned long long), s));

  Mc3Args a{};
  a.g = G.view();
  a.l1s = l1s;
  a.lo = lo;
  a.hi = hi;
  a.vlo = vr[0];
  a.hist = d_hist;
  a.cand = cand.get();
  a.moved = cand.get() + 1;
  a.codeT = (1u << pat::pair_index(0, 1, 3)) | (1u << pat::pair_index(0, 2, 3)) | (1u << pat::pair_index(1, 2, 3));
  a.codeW0 = (1u << pat::pair_index(0, 1, 3)) | (1u << pat::pair_index(0, 2, 3));
  a.codeW1 = (1u << pat::pair_index(0, 1, 3)) | (1u << pat::pair_index(1, 2, 3));
  a.bkeys = bkeys;
  a.bslots = bslots;
  const int sms = sm_count();
  size_t rec = tl.recs.size();
  if (NS) {
    const size_t wsmem = (size_t)kWarps * kWSlots * sizeof(u32);
    static std::atomic<int> occ_slot{0};
    const int occ = cached_occupancy(occ_slot, [&] {
      GPM_CUDA(cudaFuncSetAttribute(mc3_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsmem));
      int o = 0;
      GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, mc3_warp_kernel, kT, wsmem));
      return o;
    });
    const u64 blocks = std::max<u64>(1, std::min<u64>((u64)sms * occ, (NS + kWarps - 1) / kWarps));
    Mc3Args w = a;
    w.istart = ismall.get();
    w.iroot = rs.get();
    w.nitems = NS;
    w.ctr = ctr.get();
    w.grab = std::max<u64>(1, std::min<u64>(4, NS / (blocks * kWarps * 64)));
    size_t ev = tl.begin("extend_fused_L1", 0.0);
    mc3_warp_kernel<<<(unsigned)blocks, kT, wsmem, s>>>(w);
    GPM_CUDA(cudaGetLastError());
    tl.end(ev);
    ++tl.launches;
  }
  if (NB) {
    const size_t smem = (size_t)bslots * sizeof(u32);
    static thread_local std::pair<size_t, int> occb_c{0, 0};
    if (occb_c.first != smem) {
      GPM_CUDA(cudaFuncSetAttribute(mc3_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int o = 0;
      GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, mc3_block_kernel, kT, smem));
      occb_c = {smem, std::max(1, o)};
    }
    const int occb = occb_c.second;
    const u64 blocks = std::max<u64>(1, std::min<u64>((u64)sms * occb, NB));
    Mc3Args b = a;
    b.istart = ibig.get();
    b.iroot = rb.get();
    b.nitems = NB;
    b.ctr = ctr.get() + 1;
    size_t ev = tl.begin("extend_fused_L1", 0.0);
    mc3_block_kernel<<<(unsigned)blocks, kT, smem, s>>>(b);
    GPM_CUDA(cudaGetLastError());
    tl.end(ev);
    ++tl.launches;
  }
  unsigned long long W[6] = {0, 0, 0, 0, 0, 0};
  GPM_CUDA(cudaMemcpyAsync(W, cand.get(), sizeof W, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  // SURVEY §8d B_alg of the level: 8*l per parent + (16 + 4 deg) per position
  const double bytes = 8.0 * np + 16.0 * 2 * np + 4.0 * (double)W[0];
  // what the kernels actually read: the streamed pos-1 suffixes and staged S0
  // keys (4 B each) + per parent visit its v1 and offsets pair (20 B);
  // binary-search probes excluded as in B_alg.  The pos-0 candidates u > v1
  // are never streamed: their class is the pair predicate decided by the
  // stream from the other side, so they are counted, not read.
  const double moved = 4.0 * (double)(W[1] + W[2]) + 20.0 * (double)W[3];
  if (rec < tl.recs.size()) {  // both launches are named extend_fused_L1: totals on the first
    tl.recs[rec].bytes = bytes;
    tl.recs[rec].moved = moved;
  }
  st.candidates[1] += W[0];
  st.streamed += W[1] + W[2];
  st.counted += W[4];
  st.balg += bytes;
  st.bmoved += moved;
  st.paths |= (NS ? (u32)GPM_PATH_MC3_WARP : 0u) | (NB ? (u32)GPM_PATH_MC3_BLOCK : 0u) |
              (W[5] ? (u32)GPM_PATH_MC3_MULTITILE : 0u);
}

void mc4_roots_staged(const gpm_graph& G, const u32* l1i, const u32* l1v, u64 nq, unsigned long long* d_hist,
                      cudaStream_t s, Timeline& tl, Stats& st) {
  if (nq == 0) return;
  static std::atomic<int> occ_slot{0};
  const int occ = cached_occupancy(occ_slot, [] {
    int o = 0;
    GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, mc4_roots_kernel, kT4, 0));
    return o;
  });
  const u64 nitems = (nq + k4Q - 1) / k4Q;
  const u64 blocks = std::max<u64>(1, std::min<u64>((u64)sm_count() * occ, (nitems + kW4 - 1) / kW4));
  const u64 stride = std::max<u64>(32, ((u64)G.max_deg + 31) / 32 * 32);
  DBuf<u32> scratch(blocks * kW4 * stride, s);
  DBuf<unsigned long long> ctr(1, s), cand(7, s);
  GPM_CUDA(cudaMemsetAsync(ctr.get(), 0, sizeof(unsigned long long), s));
  GPM_CUDA(cudaMemsetAsync(cand.get(), 0, 7 * sizeof(unsigned long long), s));
  htrace(s, "mc4: scratch");
  Mc4Args a{};
  a.g = G.view();
  a.l1i = l1i;
  a.l1v = l1v;
  a.nq = nq;
  a.nitems = nitems;
  a.ctr = ctr.get();
  a.hist = d_hist;
  a.cand = cand.get();
  a.moved = cand.get() + 2;
  a.scratch = scratch.get();
  a.scratch_stride = stride;
  auto P = [](int i, int j) { return 1u << pat::pair_index(i, j, 4); };
  for (u32 pv = 0; pv < 4; ++pv) a.pm_bits[pv] = P(0, 1) | ((pv & 1) ? P(0, 2) : 0u) | ((pv & 2) ? P(1, 2) : 0u);
  a.cl_bits[0] = P(0, 3) | P(1, 3) | P(2, 3);
  a.cl_bits[1] = P(0, 3) | P(1, 3);
  a.cl_bits[2] = P(0, 3) | P(2, 3);
  a.cl_bits[3] = P(0, 3);
  a.cl_bits[4] = P(1, 3) | P(2, 3);
  a.cl_bits[5] = P(1, 3);
  a.cl_bits[6] = P(2, 3);
  size_t ev = tl.begin("extend_fused_L1L2", 0.0);
  mc4_roots_kernel<<<(unsigned)blocks, kT4, 0, s>>>(a);
  GPM_CUDA(cudaGetLastError());
  tl.end(ev);
  tl.launches += 1;
  // W: level-2 candidates, level-3 candidates, streamed S2, staged keys,
  // level-2 children, rank-counted, path flag
  unsigned long long W[7] = {0, 0, 0, 0, 0, 0, 0};
  GPM_CUDA(cudaMemcpyAsync(W, cand.get(), sizeof W, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  const double T = (double)W[4];
  // SURVEY §8d B_alg of both levels, as the level-by-level engine counts
  // them (level 1: 8 B + two 16 B offset pairs per parent + 4 B per
  // candidate + 8 B per child; level 2: 16 B + three offset pairs per parent
  // + 4 B per candidate)
  const double bytes = (8.0 + 32.0) * (double)nq + 4.0 * (double)W[0] + 8.0 * T + (16.0 + 48.0) * T +
                       4.0 * (double)W[1];
  // read by the kernel: streamed S2 suffixes + staged S0/S1 keys (4 B each),
  // 24 B per level-1 parent (v0, v1, offsets) and 20 B per child (its id,
  // re-read from the staged list, and its offsets pair)
  const double moved = 4.0 * (double)(W[2] + W[3]) + 24.0 * (double)nq + 20.0 * T;
  tl.recs[ev].bytes = bytes;
  tl.recs[ev].moved = moved;
  st.candidates[1] += W[0];
  st.candidates[2] += W[1];
  st.level_sizes[1] += W[4];
  st.streamed += W[2];
  st.counted += W[5];
  st.balg += bytes;
  st.bmoved += moved;
  st.paths |= GPM_PATH_MC4_STAGED | (W[6] ? (u32)GPM_PATH_MC4_HBM_SETS : 0u);
}

}  // namespace gpm
