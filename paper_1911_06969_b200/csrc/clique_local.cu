// clique_local.cu — k-CL (k >= 4) counting on the degree-ordered DAG with the
// levels >= 2 evaluated on per-root local adjacency rows.
//
// Reference semantics: Listing 3 under Alg. 1 / Alg. 2
// (PAPER.md:688-772): parents at level 1 are the DAG edges (v0, v1),
// candidates at every level are the out-list of the last vertex, and to_add
// accepts u iff u is an out-neighbour of every earlier vertex.  For a root v0
// every accepted vertex lies in N+(v0), so the whole subtree of embeddings
// rooted at v0 lives in the local graph induced on N+(v0):
//
//   level 1 (edges -> triangles): every candidate u in N+(v1) is probed
//     against an on-chip hash of N+(v0) (the same per-candidate probe as the
//     edge-chunk kernel); an accepted u sets bit j(u) of row[v1], where j is
//     u's position in N+(v0).  row[v1] is therefore exactly the set of
//     children of the parent (v0, v1), i.e. {u in N+(v1) : u in N+(v0)}.
//   level l >= 2: the candidates of a parent (v0, v1, .., x) are N+(x); those
//     outside N+(v0) were already rejected by the level-1 probe of the edge
//     (v0, x) (row[x] holds exactly the ones inside), so the children are
//     S(parent) & row[x], evaluated 32 candidates per AND, where S(parent)
//     is the parent's own child set (= the common out-neighbours of its
//     vertices inside N+(v0)).
//
// Every level's size, candidate count (sum of out-degrees of the parents'
// last vertices) and SURVEY §8d algorithmic bytes are the engine's exactly;
// no level is materialised in HBM, so the inspection / execution passes,
// the sibling-group last level and their host round trips disappear.
//
// Work split: roots with out-degree <= 32 are packed into warp items (the
// roots whose first out-edge lies in one 32-edge block of the DAG CSR: <= 32
// roots, <= 63 edges, one 32-bit row per edge); a root with out-degree in
// (32, 64] is one warp item (2-word rows); roots with out-degree in
// (64, kBigMax] and the (at most two) roots cut by the slice bounds go to a
// CTA-per-root kernel (run first) with rows of ceil(d/32) words in shared
// memory.
#include <cstdlib>

#include "gpm_apps.cuh"

namespace gpm {
namespace engine {

namespace {

constexpr u32 kBigMax = 1024;     // largest out-degree handled on chip
constexpr u32 kMidMax = 64;       // largest out-degree of a warp item
constexpr int kSmallThreads = 256;
constexpr int kBigThreads = 128;
constexpr int kAcc = 2 * kMaxLevels;  // [0, kMaxLevels): children per level; [kMaxLevels, ..): candidates per level

struct LocalArgs {
  DevGraph g;
  u64 lo, hi;           // level-1 slice = DAG edge range
  u64 blo, nblk;        // 32-edge blocks [blo, blo + nblk)
  u32* item_root;       // per block: smallest small root whose first edge lies in the block, or ~0
  u32* big;             // roots for the CTA kernel
  unsigned long long* nbig;
  u32* mid;             // roots of out-degree (32, 64] (one warp item each, after the blocks)
  unsigned long long* nmid;
  unsigned long long* ctr;   // [0] warp-item grabs, [1] big-root grabs
  unsigned long long* acc;   // [3][kAcc]: small, medium, big
  unsigned long long* total; // last-level count (engine d_total)
  u32* vr;                   // vertex range of the slice (device)
  int k;
};

__device__ __forceinline__ u32 hb_insert_at(u32* T, u32 sh, u32 bmask, u32 v) {
  u32 b = (v * kHashMul) >> sh;
  for (;;) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const u32 old = atomicCAS(T + 4 * b + q, kEmpty, v);
      if (old == kEmpty || old == v) return 4 * b + q;
    }
    b = (b + 1) & bmask;
  }
}

// slot of v in the bucketised table, or ~0
__device__ __forceinline__ u32 hb_find(const u32* T, u32 sh, u32 bmask, u32 v) {
  u32 b = (v * kHashMul) >> sh;
  for (;;) {
    const uint4 x = *reinterpret_cast<const uint4*>(T + 4 * b);
    if (x.x == v || x.y == v || x.z == v || x.w == v)
      return 4 * b + (x.x == v ? 0u : x.y == v ? 1u : x.z == v ? 2u : 3u);
    if (x.w == kEmpty) return ~0u;
    b = (b + 1) & bmask;
  }
}

// warp-aggregated append of v to list (one atomic per warp and list)
__device__ __forceinline__ void warp_append(bool take, u32 v, u32* list, unsigned long long* n) {
  const u32 m = __ballot_sync(__activemask(), take);
  if (!m) return;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(n, (unsigned long long)__popc(m));
  base = __shfl_sync(__activemask(), base, leader);
  if (take) list[base + __popc(m & lanemask_lt())] = v;
}

// Classifies the roots of the slice (thread per vertex whose out-edge range
// meets [lo, hi)): medium / big roots are appended to their lists; every
// 32-edge block b gets item_root[b] = the first vertex whose list starts at
// or after 32 b (written by exactly that vertex: no atomics), from which the
// warp item scans the small roots that start inside the block.
// <<<2, kVrThreads>>>: block 0 -> vr[0] = root of edge lo (last v in [0, n)
// with off[v] <= lo); block 1 -> vr[1] = first v in [0, n] with off[v] >= hi.
// A kVrThreads-ary search: ~3 rounds of one load per thread instead of ~22
// dependent loads of one thread (~17 us on PAT after the L2 flush, in front
// of every k-CL step).
constexpr int kVrThreads = 1024;
__global__ void __launch_bounds__(kVrThreads) local_vrange_kernel(LocalArgs a) {
  // P(v): off[v] <= lo (block 0) / off[v] < hi (block 1): true at v = 0,
  // monotone; find the last v in [0, n) with P(v)
  const bool first = blockIdx.x == 0;
  const u64 key = first ? a.lo : a.hi;
  u64 l = 0, h = a.g.n;  // P(l) holds (off[0] = 0; hi > lo >= 0), answer < h
  while (h - l > 1) {
    const u64 span = h - l;
    const u64 sp = l + span * threadIdx.x / kVrThreads;
    const u64 o = ldg(a.g.off + sp);
    const int cnt = __syncthreads_count(first ? o <= key : o < key);  // samples monotone in threadIdx
    const u64 nl = l + span * (u64)(cnt - 1) / kVrThreads;
    const u64 nh = cnt < kVrThreads ? l + span * (u64)cnt / kVrThreads : h;
    l = nl;
    h = nh;
  }
  if (threadIdx.x == 0) {
    const u32 r = first ? (u32)l : (u32)(l + 1);
    a.vr[blockIdx.x] = r;
    // block blo's lower-bound vertex may precede the slice (its list starts
    // before lo): scanning block blo from the root of edge lo finds every
    // small root that starts inside the slice (the prep may lower it no further)
    if (first && a.nblk) a.item_root[0] = r;
  }
}

__global__ void local_prep_kernel(LocalArgs a) {
  // the slice's vertex range [vr[0], vr[1]] (grid-stride: any grid covers it)
  const u64 vend = ((u64)a.vr[1] + 1 < (u64)a.g.n) ? (u64)a.vr[1] + 1 : (u64)a.g.n;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 vb = a.vr[0] + blockIdx.x * (u64)blockDim.x; vb < vend; vb += stride) {
    const u64 v = vb + threadIdx.x;
    const bool valid = v < vend;
    // one offset load per lane; the neighbours' from the adjacent lanes
    const int lane = threadIdx.x & 31;
    const u64 ob = v <= a.g.n ? ldg(a.g.off + v) : 0;
    u64 oe = __shfl_down_sync(0xffffffffu, ob, 1), prev = __shfl_up_sync(0xffffffffu, ob, 1);
    if (lane == 31 && valid) oe = ldg(a.g.off + v + 1);
    if (lane == 0 && v) prev = ldg(a.g.off + v - 1);
    if (valid) {
      const u64 b0 = max(v ? prev / 32 + 1 : 0, a.blo), b1 = ob / 32 + 1;  // b in [b0, b1)
      for (u64 b = b0; b < b1 && b < a.blo + a.nblk; ++b) a.item_root[b - a.blo] = (u32)v;
    }
    const bool in = valid && !(oe <= a.lo || ob >= a.hi || ob == oe);
    const u64 d = valid ? oe - ob : 0;
    const bool big = in && (ob < a.lo || oe > a.hi || d > kMidMax);
    warp_append(big, (u32)v, a.big, a.nbig);
    warp_append(in && !big && d > 32, (u32)v, a.mid, a.nmid);
  }
}

// ---------------------------------------------------------------------------
// Warp items.  An item is either the small roots (out-degree <= 32) whose
// first out-edge lies in one 32-edge block of the DAG CSR (<= 32 roots,
// <= 63 edges, 1-word rows), or one medium root (out-degree in (32, 64],
// rows of 2 words).  Per warp in shared memory: a bucketised hash of the
// item's keys (u << 5 | root slot) -> local position, the rows, and the
// candidate stream's descriptors.  The stream (the concatenated out-lists of
// the item's edges) is walked 32 positions per window; a per-window bitmap of
// entry starts (built once per item) maps lanes to entries with two POPCs,
// and keys that all sit in their primary bucket are probed with ONE LDS.128
// (items whose insert overflowed a bucket, or whose stream exceeds the window
// bitmap, take the general loop: OR-reduction mapping + chained probe).
constexpr u32 ilog2(u32 x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

template <int KMAX, int NB, int WMAX, int WIN = 256, int UNROLL = 4, int MINB = 4>
struct WarpCfg {
  static constexpr int kKeys = KMAX;     // edges (keys) per item
  static constexpr int kBuckets = NB;    // 4 slots each
  static constexpr int kWords = WMAX;    // row words per edge
  static constexpr int kWin = WIN;       // stream windows with a start bitmap (32 positions each)
  static constexpr int kUnroll = UNROLL; // windows per loop step (loads in flight per warp)
  static constexpr int kMinBlocks = MINB;  // (software-pipelining the next step's loads needed 78
                                          // registers -> 3 CTAs/SM and measured slower: 1.00 vs 0.89 ms)
};
using SmallCfg = WarpCfg<64, 128, 2, 128>;   // small-root blocks (1-word rows) and roots of out-degree <= 64

template <class C>
struct WarpSmem {
  uint4 T[C::kBuckets];           // keys (kEmpty = free)
  u32 F[256];                     // 8192-bit blocked Bloom filter of the keys (2 bits per key)
  u8 V[C::kBuckets * 4];          // local position of the key in its root's list
  u32 rows[C::kKeys * C::kWords];
  __align__(16) u32 wm[C::kWin + C::kUnroll];  // per window: bit p = an entry starts at window position p
  uint2 ent[C::kKeys];            // per entry: (cb - exclusive start) mod 2^32, root slot
  u8 ekk[C::kKeys];               // per entry: its edge kk
  u32 ex[C::kKeys + 32];          // per entry: exclusive start, ~0 past the entries
  u32 dp[C::kKeys];               // per edge: out-degree of its v1
  u8 base[C::kKeys];              // per edge: first edge index of its root
  u64 rb[32];                     // per root slot: first out-edge
  u32 rk[64];                     // per root slot: first edge index; ~0 past the roots
  unsigned long long acc[kAcc];   // levels >= 2 (generic DFS)
};

// children of the level-1 parent kk: row words R[0..W); levels >= 2 below it
template <int WMAX>
__device__ __forceinline__ void count_subtree(const u32* rows, const u32* dp, u32 kbase, u32 kk, u32 W, int last,
                                              unsigned long long& l2, unsigned long long& c2,
                                              unsigned long long* sacc) {
  u32 S[WMAX];
#pragma unroll
  for (int w = 0; w < WMAX; ++w) S[w] = w < (int)W ? rows[kk * W + w] : 0u;
  if (last == 2) {
    // 4-CL: the children's children are counted, not visited
#pragma unroll
    for (int w = 0; w < WMAX; ++w) {
      u32 m = S[w];
      while (m) {
        const u32 j = kbase + w * 32 + __ffs(m) - 1;
        m &= m - 1;
        c2 += dp[j];
        u32 cnt = 0;
#pragma unroll
        for (int x = 0; x < WMAX; ++x)
          if (x < (int)W) cnt += __popc(S[x] & rows[j * W + x]);
        l2 += cnt;
      }
    }
    return;
  }
  // k >= 5: DFS over the child sets (per level W words, local memory)
  u32 set[kMaxLevels][WMAX], cw[kMaxLevels], cb[kMaxLevels];
#pragma unroll
  for (int w = 0; w < WMAX; ++w) set[1][w] = S[w];
  int lev = 1;
  cw[1] = 0;
  cb[1] = S[0];
  while (lev >= 1) {
    while (cb[lev] == 0 && cw[lev] + 1 < W) cb[lev] = set[lev][++cw[lev]];
    if (cb[lev] == 0) {
      --lev;
      continue;
    }
    const u32 j = kbase + cw[lev] * 32 + __ffs(cb[lev]) - 1;
    cb[lev] &= cb[lev] - 1;
    atomicAdd(sacc + kMaxLevels + lev + 1, (unsigned long long)dp[j]);
    const bool deeper = lev + 1 < last;
    u32 cnt = 0;
    for (u32 w = 0; w < W; ++w) {
      const u32 x = set[lev][w] & rows[j * W + w];
      cnt += __popc(x);
      if (deeper) set[lev + 1][w] = x;
    }
    if (cnt) atomicAdd(sacc + lev + 1, (unsigned long long)cnt);
    if (deeper && cnt) {
      ++lev;
      cw[lev] = 0;
      cb[lev] = set[lev][0];
    }
  }
}

// Items [0, nblk) are small-root blocks, then one item per root of out-degree
// in (32, 64] (a.mid).
template <class C>
__global__ void __launch_bounds__(kSmallThreads, C::kMinBlocks) local_warp_kernel(LocalArgs a) {
  extern __shared__ __align__(16) unsigned char wsm[];
  WarpSmem<C>* const s_w = reinterpret_cast<WarpSmem<C>*>(wsm);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const u32 lt = lanemask_lt(), lemask = lt | (1u << lane);
  WarpSmem<C>& S = s_w[wid];
  u32* const Tw = reinterpret_cast<u32*>(S.T);
  constexpr u32 sh = 32 - ilog2(C::kBuckets);
  constexpr u32 bmask = C::kBuckets - 1;
  for (int i = lane; i < kAcc; i += 32) S.acc[i] = 0;
  for (int i = lane; i < C::kBuckets; i += 32) S.T[i] = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
  for (int i = lane; i < 256; i += 32) S.F[i] = 0;
  S.rk[32 + lane] = 0xffffffffu;
  __syncwarp();
  const DevGraph& g = a.g;
  const int last = a.k - 2;
  unsigned long long l1 = 0, c1 = 0, l2 = 0, c2 = 0;
  const u64 nblk = a.nblk;
  const u64 nitems = nblk + *reinterpret_cast<volatile unsigned long long*>(a.nmid);
  const u32* const rootlist = a.mid;
  constexpr u64 kGrab = 4;
  u64 grab = 0, grab_left = 0;
  for (;;) {
    if (grab_left == 0) {
      u64 it_ = 0;
      if (lane == 0) it_ = atomicAdd(a.ctr, kGrab);
      grab = __shfl_sync(0xffffffffu, it_, 0);
      grab_left = kGrab;
    }
    const u64 item = grab++;
    --grab_left;
    if (item >= nitems) break;
    // ---- the item's roots -> slots (rb, rk = degree then exclusive start)
    u32 nr = 0;
    if (item >= nblk) {
      if (lane == 0) {
        const u32 v = rootlist[item - nblk];
        S.rb[0] = ldg(g.off + v);
        S.rk[0] = (u32)(ldg(g.off + v + 1) - S.rb[0]);
      }
      nr = 1;
    } else {
      const u32 ra = a.item_root[item];
      if (ra == 0xffffffffu) continue;
      const u64 bend = (a.blo + item + 1) * 32;
      for (u32 vb = ra;; vb += 32) {
        const u32 v = vb + lane;
        u64 ob = ~0ull, oe = 0;
        if (v < g.n) {
          ob = ldg(g.off + v);
          oe = ldg(g.off + v + 1);
        }
        const bool q = ob < bend && oe > ob && oe - ob <= 32 && ob >= a.lo && oe <= a.hi;
        const u32 qm = __ballot_sync(0xffffffffu, q);
        if (q) {
          const u32 s = nr + __popc(qm & lt);
          S.rb[s] = ob;
          S.rk[s] = (u32)(oe - ob);
        }
        nr += __popc(qm);
        if (__ballot_sync(0xffffffffu, ob >= bend)) break;
      }
    }
    __syncwarp();
    u32 rd = lane < nr ? S.rk[lane] : 0u, kin = rd;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 t = __shfl_up_sync(0xffffffffu, kin, o);
      if (lane >= o) kin += t;
    }
    const u32 K = __shfl_sync(0xffffffffu, kin, 31);
    const u32 W = (K + 31) / 32 > 1 && item >= nblk ? (K + 31) / 32 : 1u;  // blocks: 1-word rows
    __syncwarp();
    S.rk[lane] = lane < nr ? kin - rd : 0xffffffffu;
    __syncwarp();
    // ---- keys (u << 5 | slot) -> local position; per-edge out-lists
    u32 R = 0, nz = 0, run = 0;
    bool ovf = false;
    u32 kpos[C::kKeys / 32], kfw[C::kKeys / 32];
#pragma unroll
    for (int rr = 0; rr < C::kKeys / 32; ++rr) {
      const u32 kb = rr * 32;
      kpos[rr] = ~0u;
      kfw[rr] = 0;
      if (kb >= K) continue;  // warp-uniform
      u32 r = 0;
      if (item < nblk) {
        const u32 dd = S.rk[R + 1 + lane] - kb;
        const u32 starts = __reduce_or_sync(0xffffffffu, dd < 32u ? (1u << dd) : 0u);
        r = min(R + __popc(starts & lemask), nr - 1);
        R += __popc(starts);
      }
      const u32 kk = kb + lane;
      u32 dpv = 0;
      u64 cb = 0;
      if (kk < K) {
        const u32 kbase = S.rk[r], j = kk - kbase;
        const u32 w = ldg(g.col + S.rb[r] + j);
        const u32 key = (w << 5) | r;
        const u32 hv = key * kHashMul;
        // filter: word = hash bits 16..23, two bits = bits 27..31 and 11..15
        // (a blocked Bloom filter: ~0.03 % false positives at 64 keys)
        atomicOr(S.F + ((hv >> 16) & 255u), (1u << (hv >> 27)) | (1u << ((hv >> 11) & 31u)));
        kfw[rr] = (hv >> 16) & 255u;
        u32 b = hv >> sh;
        for (u32 probe = 0;; ++probe) {
          u32 q = 0;
          for (; q < 4; ++q) {
            const u32 old = atomicCAS(Tw + 4 * b + q, kEmpty, key);
            if (old == kEmpty) break;
          }
          if (q < 4) {
            kpos[rr] = 4 * b + q;
            break;
          }
          ovf = true;
          b = (b + 1) & bmask;
        }
        S.V[kpos[rr]] = (u8)j;
        S.base[kk] = (u8)kbase;
        cb = ldg(g.off + w);
        dpv = (u32)(ldg(g.off + w + 1) - cb);
        S.dp[kk] = dpv;
#pragma unroll
        for (int w2 = 0; w2 < C::kWords; ++w2)
          if (w2 < (int)W) S.rows[kk * W + w2] = 0;
      }
      u32 incl = dpv;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const u32 nzm = __ballot_sync(0xffffffffu, dpv > 0);
      if (dpv > 0) {
        const u32 qi = nz + __popc(nzm & lt);
        const u32 ex = run + incl - dpv;
        S.ex[qi] = ex;
        S.ent[qi] = make_uint2((u32)(cb - (u64)ex), r);  // col index = (.x + position) mod 2^32 (m < 2^32)
        S.ekk[qi] = (u8)kk;
      }
      nz += __popc(nzm);
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    const u32 total = run;
    const u32 nwin = (total + 31) >> 5;
    const bool fast = !__any_sync(0xffffffffu, ovf) && nwin <= (u32)C::kWin;
    if (fast) {
      for (u32 i = lane; i < nwin + C::kUnroll; i += 32) S.wm[i] = 0;
    }
    S.ex[nz + lane] = 0xffffffffu;
    __syncwarp();
    if (fast) {
      for (u32 i = lane; i < nz; i += 32) {
        const u32 ex = S.ex[i];
        atomicOr(S.wm + (ex >> 5), 1u << (ex & 31));
      }
    }
    __syncwarp();
    // ---- level 1: every candidate u of the stream probes (u, slot)
    auto hit = [&](u32 key, u32 e) {
      u32 b = (key * kHashMul) >> sh;
      for (;;) {
        const uint4 x = S.T[b];
        if (x.x == key || x.y == key || x.z == key || x.w == key) {
          const u32 j = S.V[4 * b + (x.x == key ? 0u : x.y == key ? 1u : x.z == key ? 2u : 3u)], kk = S.ekk[e];
          atomicOr(S.rows + kk * W + (j >> 5), 1u << (j & 31));
          return;
        }
        if (x.w == kEmpty) return;
        b = (b + 1) & bmask;
      }
    };
    if (fast) {
      // a lane past the stream probes key 0xfffffffe (vertex 2^27 - 1, slot
      // 30): no vertex has that id (n < 2^27) and it is not kEmpty
      static_assert(C::kUnroll == 4, "one LDS.128 of window masks per step");
      u32 P = 0xffffffffu;  // entry holding the position before the window
      const u32* const col = g.col;
      // one step = 4 windows: lane -> entry by the start bitmaps, then the
      // four candidate loads (raw vertex + slot; the key is formed later)
      auto issue = [&](u32 it, u32 (&uq)[4], u32 (&sq)[4], u32 (&eq)[4]) {
        const uint4 w4 = *reinterpret_cast<const uint4*>(S.wm + it);
        const u32 wq[4] = {w4.x, w4.y, w4.z, w4.w};
        const u32 jl = it * 32 + lane;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          eq[q] = P + __popc(wq[q] & lemask);
          P += __popc(wq[q]);
          uq[q] = 0x07ffffffu;
          sq[q] = 30;
          if (jl + 32 * q < total) {
            const uint2 d = S.ent[eq[q]];
            uq[q] = ldg(col + (u32)(d.x + jl + 32 * q));
            sq[q] = d.y;
          }
        }
      };
      // filter bit first (one LDS.32 per window); the bucket (LDS.128, ~4x
      // the shared-memory wavefronts) only for filter-positive lanes, which
      // are rare: any positive lane re-probes its 4 keys exactly
      auto probe = [&](const u32 (&uq)[4], const u32 (&sq)[4], const u32 (&eq)[4]) {
        u32 key[4], pm = 0;  // pm: windows whose key passed the filter
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          key[q] = (uq[q] << 5) | sq[q];
          const u32 hv = key[q] * kHashMul;
          const u32 f = S.F[__byte_perm(hv, 0, 0x4442)];
          const u32 m2 = (1u << (hv >> 27)) | (1u << ((hv >> 11) & 31u));
          pm |= (u32)((f & m2) == m2) << q;
        }
        if (pm) {  // rare: true hits (~0.3 % of candidates) and filter false positives
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (pm & (1u << q)) hit(key[q], eq[q]);  // static indices: key / eq stay in registers
        }
      };
      {
        for (u32 it = 0; it < nwin; it += 4) {
          u32 uq[4], sq[4], eq[4];
          issue(it, uq, sq, eq);
          probe(uq, sq, eq);
        }
      }
    } else {
      u32 P = 0;
      for (u32 jb = 0; jb < total; jb += 32) {
        const u32 d = S.ex[P + 1 + lane] - jb;
        const u32 st = __reduce_or_sync(0xffffffffu, d < 32u ? (1u << d) : 0u);
        const u32 myp = P + __popc(st & lemask);
        P += __popc(st);
        const u32 jj = jb + lane;
        if (jj < total) {
          const uint2 dd = S.ent[myp];
          const u32 u = ldg(g.col + (u32)(dd.x + jj));
          hit((u << 5) | dd.y, myp);
        }
      }
    }
    __syncwarp();
    // ---- levels >= 2 on the rows
    for (u32 kk = lane; kk < K; kk += 32) {
      const u32 kbase = S.base[kk];
      u32 n1 = 0;
#pragma unroll
      for (int w = 0; w < C::kWords; ++w)
        if (w < (int)W) n1 += __popc(S.rows[kk * W + w]);
      l1 += n1;
      c1 += S.dp[kk];
      if (n1) count_subtree<C::kWords>(S.rows, S.dp, kbase, kk, W, last, l2, c2, S.acc);
    }
    __syncwarp();
    // ---- free the item's keys and filter words
#pragma unroll
    for (int rr = 0; rr < C::kKeys / 32; ++rr)
      if (kpos[rr] != ~0u) {
        Tw[kpos[rr]] = kEmpty;
        S.F[kfw[rr]] = 0;
      }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l1 += __shfl_xor_sync(0xffffffffu, l1, o);
    c1 += __shfl_xor_sync(0xffffffffu, c1, o);
    l2 += __shfl_xor_sync(0xffffffffu, l2, o);
    c2 += __shfl_xor_sync(0xffffffffu, c2, o);
  }
  __syncwarp();
  if (lane == 0) {
    S.acc[1] += l1;
    S.acc[kMaxLevels + 1] += c1;
    S.acc[2] += l2;
    S.acc[kMaxLevels + 2] += c2;
  }
  __syncwarp();
  unsigned long long* const gacc = a.acc;
  for (int i = lane; i < kAcc; i += 32) {
    const unsigned long long x = S.acc[i];
    if (!x) continue;
    if (i == last) atomicAdd(a.total, x);
    else atomicAdd(gacc + i, x);
  }
}

// Dynamic shared-memory layout of local_big_kernel (32-bit word offsets):
// hash keys (cap), u16 local positions (cap), rows (dmax x ceil(dmax/32)),
// per-edge out-degrees, stream starts (+33 sentinels), list addresses (u64),
// stream entry -> edge.
struct BigLayout {
  u32 cap, T, V, rows, dp, ex, cp, inf, words;
  __host__ __device__ explicit BigLayout(u32 dmax) {
    cap = 128;
    while (cap < 4 * dmax) cap <<= 1;
    T = 0;
    V = cap;
    rows = V + cap / 2;
    dp = rows + dmax * ((dmax + 31) / 32);
    ex = dp + dmax;
    cp = (ex + dmax + 33 + 1) & ~1u;
    inf = cp + 2 * dmax;
    words = inf + dmax;
  }
};

// One root per CTA (out-degree in (32, kBigMax], or cut by the slice bounds):
// hash of N+(v0) (key u -> local position), ceil(d/32)-word rows, the
// root's candidate stream split evenly over the warps.
__global__ void __launch_bounds__(kBigThreads) local_big_kernel(LocalArgs a, u32 dmax) {
  extern __shared__ __align__(16) u32 sm[];
  constexpr int NW = kBigThreads / 32;
  const BigLayout L(dmax);
  u32* const T = sm + L.T;
  uint16_t* const V = reinterpret_cast<uint16_t*>(sm + L.V);
  u32* const rows = sm + L.rows;
  u32* const sdp = sm + L.dp;
  u32* const sex = sm + L.ex;
  u64* const scp = reinterpret_cast<u64*>(sm + L.cp);
  u32* const sinf = sm + L.inf;
  __shared__ u32 s_wsum[NW + 1];
  __shared__ u64 s_item;
  __shared__ unsigned long long s_acc[kAcc];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const u32 lt = lanemask_lt(), lemask = lt | (1u << lane);
  const DevGraph& g = a.g;
  const int last = a.k - 2;
  for (int i = tid; i < kAcc; i += kBigThreads) s_acc[i] = 0;
  for (;;) {
    __syncthreads();
    if (tid == 0) s_item = atomicAdd(a.ctr + 1, 1ull);
    __syncthreads();
    const u64 item = s_item;
    if (item >= *reinterpret_cast<volatile unsigned long long*>(a.nbig)) break;
    const u32 v0 = a.big[item];
    const u64 ob = ldg(g.off + v0), oe = ldg(g.off + v0 + 1);
    const u32 d = (u32)(oe - ob);
    const u32 W = (d + 31) / 32;
    // counted edges [k0, k1) (a root cut by the slice bounds); every edge's
    // row is built, since a child's position in N+(v0) (id order) may lie
    // before or after its parent's
    const u32 k0 = (u32)(max(ob, a.lo) - ob), k1 = (u32)(min(oe, a.hi) - ob);
    u32 c = 128;
    while (c < 4 * d) c <<= 1;
    const u32 sh = 32 - (31 - __clz(c / 4)), bmask = c / 4 - 1;
    for (u32 i = tid * 4; i < c; i += 4 * kBigThreads) *reinterpret_cast<uint4*>(T + i) = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
    for (u32 i = tid; i < d * W; i += kBigThreads) rows[i] = 0;
    __syncthreads();
    // stage keys, per-edge out-degrees and list starts
    for (u32 kk = tid; kk < d; kk += kBigThreads) {
      const u32 w = ldg(g.col + ob + kk);
      V[hb_insert_at(T, sh, bmask, w)] = (uint16_t)kk;
      const u64 cb = ldg(g.off + w);
      sdp[kk] = (u32)(ldg(g.off + w + 1) - cb);
      scp[kk] = cb;
    }
    __syncthreads();
    // stream entries: edges kk in [0, d) with non-empty lists, in order
    // (one warp compacts; d <= kBigMax)
    if (wid == 0) {
      u32 nz = 0, run = 0;
      for (u32 kb = 0; kb < d; kb += 32) {
        const u32 kk = kb + lane;
        const u32 dp = kk < d ? sdp[kk] : 0u;
        u32 incl = dp;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const u32 nzm = __ballot_sync(0xffffffffu, dp > 0);
        // scp is rewritten in place for entries <= kk (nz <= kk)
        u64 cb = kk < d ? scp[kk] : 0;
        __syncwarp();
        if (dp > 0) {
          const u32 qi = nz + __popc(nzm & lt);
          const u32 ex = run + incl - dp;
          sex[qi] = ex;
          scp[qi] = reinterpret_cast<u64>(g.col) + 4 * (cb - (u64)ex);
          sinf[qi] = kk;
        }
        __syncwarp();
        nz += __popc(nzm);
        run += __shfl_sync(0xffffffffu, incl, 31);
      }
      for (u32 i = nz + lane; i < nz + 33; i += 32) sex[i] = 0xffffffffu;
      if (lane == 0) {
        s_wsum[0] = run;
        s_wsum[1] = nz;
      }
    }
    __syncthreads();
    const u32 total = s_wsum[0], nzt = s_wsum[1];
    // ---- level 1: warp w streams candidates [t0, t1)
    {
      const u32 t0 = (u32)((u64)total * wid / NW), t1 = (u32)((u64)total * (wid + 1) / NW);
      if (t0 < t1) {
        // P = the entry holding t0: last entry with sex <= t0
        u32 l_ = 0, h_ = nzt;
        while (h_ - l_ > 1) {
          const u32 mid = (l_ + h_) >> 1;
          if (sex[mid] <= t0) l_ = mid;
          else h_ = mid;
        }
        u32 P = l_;
        // first map_step may see starts at P (already counted) only via d < 32
        auto map_step = [&](u32 jb) -> u32 {
          const u32 dd = sex[P + 1 + lane] - jb;
          const u32 st = __reduce_or_sync(0xffffffffu, dd < 32u ? (1u << dd) : 0u);
          const u32 myp = P + __popc(st & lemask);
          P += __popc(st);
          return myp;
        };
        for (u32 jb = t0; jb < t1; jb += 32) {
          const u32 myp = map_step(jb);
          const u32 jj = jb + lane;
          if (jj < t1) {
            const u32 u = ldg(reinterpret_cast<const u32*>(scp[myp]) + jj);
            const u32 pos = hb_find(T, sh, bmask, u);
            if (pos != ~0u) {
              const u32 j = V[pos], kk = sinf[myp];
              atomicOr(rows + (size_t)kk * W + (j >> 5), 1u << (j & 31));
            }
          }
        }
      }
    }
    __syncthreads();
    // ---- levels: counted edges [k0, k1)
    for (u32 kk = k0 + tid; kk < k1; kk += kBigThreads) {
      const u32* R0 = rows + (size_t)kk * W;
      u32 S1 = 0;
      for (u32 w = 0; w < W; ++w) S1 += __popc(R0[w]);
      atomicAdd(s_acc + kMaxLevels + 1, (unsigned long long)sdp[kk]);
      if (S1) atomicAdd(s_acc + 1, (unsigned long long)S1);
      if (last < 2 || !S1) continue;
      // DFS over the local rows (sets of W words, in local memory)
      u32 set[kMaxLevels][kBigMax / 32];
      u32 cw[kMaxLevels], cb_[kMaxLevels];
      int lev = 1;
      for (u32 w = 0; w < W; ++w) set[1][w] = R0[w];
      cw[1] = 0;
      cb_[1] = set[1][0];
      while (lev >= 1) {
        while (cb_[lev] == 0 && cw[lev] + 1 < W) cb_[lev] = set[lev][++cw[lev]];
        if (cb_[lev] == 0) {
          --lev;
          continue;
        }
        const u32 j = cw[lev] * 32 + __ffs(cb_[lev]) - 1;
        cb_[lev] &= cb_[lev] - 1;
        atomicAdd(s_acc + kMaxLevels + lev + 1, (unsigned long long)sdp[j]);
        const u32* Rj = rows + (size_t)j * W;
        const bool deeper = lev + 1 < last;
        u32 cnt = 0;
        for (u32 w = 0; w < W; ++w) {
          const u32 x = set[lev][w] & Rj[w];
          cnt += __popc(x);
          if (deeper) set[lev + 1][w] = x;
        }
        if (cnt) atomicAdd(s_acc + lev + 1, (unsigned long long)cnt);
        if (deeper && cnt) {
          ++lev;
          cw[lev] = 0;
          cb_[lev] = set[lev][0];
        }
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < kAcc; i += kBigThreads) {
    const unsigned long long x = s_acc[i];
    if (!x) continue;
    if (i == last) atomicAdd(a.total, x);
    else atomicAdd(a.acc + 2 * kAcc + i, x);
  }
}


}  // namespace

// Timeline record on a stream other than the timeline's own (marked side:
// overlapped, not a phase of the step)
size_t tl_begin_on(Timeline& tl, const char* name, cudaStream_t st) {
  Timeline::Rec r{name, nullptr, nullptr, 0.0, -1, st != tl.s};
  GPM_CUDA(cudaEventCreate(&r.a));
  GPM_CUDA(cudaEventCreate(&r.b));
  GPM_CUDA(cudaEventRecord(r.a, st));
  tl.recs.push_back(r);
  return tl.recs.size() - 1;
}

// Side stream of the calling thread on the current device
cudaStream_t side_stream() {
  int dev = 0;
  GPM_CUDA(cudaGetDevice(&dev));
  static thread_local std::vector<cudaStream_t> ss;
  if ((int)ss.size() <= dev) ss.resize(dev + 1, nullptr);
  if (!ss[dev]) {
    // highest priority: its CTAs are dispatched before the small-item grid's
    int lo = 0, hi = 0;
    GPM_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    GPM_CUDA(cudaStreamCreateWithPriority(&ss[dev], cudaStreamNonBlocking, hi));
  }
  return ss[dev];
}

template <class C>
size_t launch_warp(Ctx& c, LocalArgs& a, u64 max_blocks, const char* name, cudaStream_t st) {
  auto kern = local_warp_kernel<C>;
  const size_t smem = sizeof(WarpSmem<C>) * (kSmallThreads / 32);
  static std::atomic<int> occ{0};
  const int o = cached_occupancy(occ, [&] {
    GPM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int r = 0;
    GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, kern, kSmallThreads, smem));
    return r;
  });
  const u64 blocks = std::max<u64>(1, std::min<u64>((u64)c.sms * o, max_blocks));
  size_t rec = c.tl->begin(name, 0.0);
  kern<<<(unsigned)blocks, kSmallThreads, smem, st>>>(a);
  GPM_CUDA(cudaGetLastError());
  c.tl->end(rec);
  return rec;
}

// k-CL (k >= 4) count of the level-1 slice [slo, shi) on local rows; false
// when the preconditions do not hold (the caller runs the edge-chunk path).
bool cf_local_applicable(const gpm_graph& G, int k, bool listing) {
  return k >= 4 && !listing && G.oriented && G.max_deg <= kBigMax && G.n < (1u << 27) && G.m < (u64(1) << 32) &&
         !std::getenv("GPM_CF_NOLOCAL");
}

bool cf_local_roots(Ctx& c, const u32*, u64 slo, u64 shi) {
  if (!cf_local_applicable(*c.G, c.k, c.list_fn != nullptr)) return false;
  const u64 np = shi - slo;
  Stats& st = *c.st;
  st.paths |= GPM_PATH_CF_LOCAL;
  const u64 blo = slo / 32, nblk = (shi - 1) / 32 - blo + 1;
  const u64 bigcap = np / 33 + 3;
  DBuf<u32> item(nblk, c.s), big(bigcap, c.s), mid(bigcap, c.s);
  constexpr int kCtl = 8;
  DBuf<unsigned long long> ctl(kCtl + 3 * kAcc, c.s);
  GPM_CUDA(cudaMemsetAsync(item.get(), 0xff, sizeof(u32) * nblk, c.s));
  GPM_CUDA(cudaMemsetAsync(ctl.get(), 0, sizeof(unsigned long long) * (kCtl + 3 * kAcc), c.s));
  LocalArgs a{};
  a.g = c.g;
  a.lo = slo;
  a.hi = shi;
  a.blo = blo;
  a.nblk = nblk;
  a.item_root = item.get();
  a.big = big.get();
  a.nbig = ctl.get();
  a.ctr = ctl.get() + 1;
  a.mid = mid.get();
  a.nmid = ctl.get() + 4;
  a.acc = ctl.get() + kCtl;
  a.total = c.d_total;
  a.k = c.k;
  // the slice's vertices: at most (hi - lo) non-empty ones plus the empty
  // vertices between them; whole-graph bound when that is smaller
  DBuf<u32> vr(2, c.s);
  a.vr = vr.get();
  local_vrange_kernel<<<2, kVrThreads, 0, c.s>>>(a);
  const u64 vcap = std::min<u64>(c.G->n, np + (u64(1) << 20));  // grid size only: the kernel strides
  const unsigned pg = (unsigned)std::max<u64>(1, (vcap + 255) / 256);
  local_prep_kernel<<<pg, 256, 0, c.s>>>(a);
  GPM_CUDA(cudaGetLastError());
  // roots of out-degree > 64 (and slice-cut roots): one CTA each, ~50 us on
  // PAT.  (Heavy medium-root warp CTAs -- 94 KB of shared memory -- launched
  // beside the persistent small-item grid only got SMs once it drained, i.e.
  // ran as a tail; light CTAs dispatched first co-reside with it.)
  size_t rec[3] = {0, 0, 0};
  const u32 dmax = std::max<u32>(kMidMax + 1, c.G->max_deg);
  const size_t smem = 4 * (size_t)BigLayout(dmax).words;
  // attribute + occupancy once per shared-memory size (per thread: the
  // attribute is per device and threads may run on different devices)
  static thread_local std::pair<size_t, int> big_occ{0, 0};
  if (big_occ.first != smem) {
    GPM_CUDA(cudaFuncSetAttribute(local_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int o = 0;
    GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, local_big_kernel, kBigThreads, smem));
    big_occ = {smem, o};
  }
  const int ob = big_occ.second;
  const u64 bb = std::max<u64>(1, std::min<u64>((u64)c.sms * std::max(1, ob), bigcap));
  // the CTA kernel (few, light CTAs: 128 threads, ~12 KB) is dispatched
  // first on a side stream, the small-item grid right after on the main one:
  // they share the SMs while the big roots run instead of serialising
  cudaStream_t ss = side_stream();
  cudaEvent_t fork = nullptr, join = nullptr;
  GPM_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  GPM_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
  struct EvGuard {
    cudaEvent_t* e[2];
    ~EvGuard() {
      for (auto* x : e)
        if (*x) cudaEventDestroy(*x);
    }
  } evg{{&fork, &join}};
  GPM_CUDA(cudaEventRecord(fork, c.s));
  GPM_CUDA(cudaStreamWaitEvent(ss, fork, 0));
  rec[2] = tl_begin_on(*c.tl, "extend_local_big", ss);
  local_big_kernel<<<(unsigned)bb, kBigThreads, smem, ss>>>(a, dmax);
  GPM_CUDA(cudaGetLastError());
  GPM_CUDA(cudaEventRecord(c.tl->recs[rec[2]].b, ss));
  GPM_CUDA(cudaEventRecord(join, ss));
  rec[0] = launch_warp<SmallCfg>(c, a, (nblk + bigcap + 7) / 8, "extend_local_small", c.s);
  GPM_CUDA(cudaStreamWaitEvent(c.s, join, 0));
  c.tl->launches += 4;
  std::vector<unsigned long long> h(kCtl + 3 * kAcc);
  GPM_CUDA(cudaMemcpyAsync(h.data(), ctl.get(), sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost, c.s));
  GPM_CUDA(cudaStreamSynchronize(c.s));
  if (h[0] > 0) st.paths |= GPM_PATH_CF_LOCAL_BIG;
  // stats and SURVEY §8d bytes per kernel: level lev parents P_lev (P_1 = the
  // slice's edges), candidates C_lev, children L_lev (the last level's
  // children are the engine's total, added from d_total by the caller)
  const int last = c.k - 2;
  double bytes[3] = {0, 0, 0};
  for (int kind = 0; kind < 3; ++kind) {
    const unsigned long long* A = h.data() + kCtl + kind * kAcc;
    for (int lev = 1; lev <= last; ++lev) {
      const u64 C = A[kMaxLevels + lev];
      st.candidates[lev] += C;
      bytes[kind] += 4.0 * (double)C;
      if (lev < last) {
        st.level_sizes[lev] += A[lev];
        bytes[kind] += 8.0 * (double)A[lev];  // stored children (engine model)
      }
    }
    // parents per level: P_1 from the level-1 candidates' owners is np in
    // total; deeper levels' parents are the previous level's children
    for (int lev = 2; lev <= last; ++lev) bytes[kind] += (8.0 * lev + 16.0) * (double)A[lev - 1];
  }
  // level-1 parents: every edge of the slice, (8 + 16) B each; attributed to
  // the kernels in proportion to their level-1 candidates
  double c1[3], c1t = 0;
  for (int kind = 0; kind < 3; ++kind) c1t += (c1[kind] = (double)h[kCtl + kind * kAcc + kMaxLevels + 1]);
  for (int kind = 0; kind < 3; kind += 2) {  // kind 1 (the old medium-root kernel) is unused
    bytes[kind] += 24.0 * (double)np * (c1t > 0 ? c1[kind] / c1t : (kind == 0 ? 1.0 : 0.0));
    c.tl->recs[rec[kind]].bytes = bytes[kind];
    st.balg += bytes[kind];
  }
  return true;
}

}  // namespace engine
}  // namespace gpm
