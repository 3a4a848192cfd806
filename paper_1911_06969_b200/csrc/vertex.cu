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
  u64 np, W, B;    // np = number of parents with non-zero work
  u64 b_begin, b_end;
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
__global__ void __launch_bounds__(kThreads) extend_kernel(ExtendArgs a) {
  constexpr int S = LEV + 1;  // parent embedding size
  constexpr int kWords = (int)(kBatch / 32);
  extern __shared__ unsigned long long shist[];
  const int lane = threadIdx.x & 31;
  const DevGraph& g = a.g;
  int nbins = 0;
  if (MODE == kFused && APP == kAppMC) {
    nbins = 1 << pat::npairs(a.k);
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) shist[i] = 0;
    __syncthreads();
  }
  unsigned long long wtotal = 0;

  for (;;) {
    u64 b = 0;
    if (lane == 0) b = atomicAdd(a.ctr, 1ull) + a.b_begin;
    b = __shfl_sync(0xffffffffu, b, 0);
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
      if (j < j1) {
        cur.load(a, myp);
        int pos;
        u = cur.candidate(g, j, pos);
        const u32* emb = cur.emb;
        bool inemb = false;
#pragma unroll
        for (int t = 0; t < S; ++t) inemb |= (emb[t] == u);
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
#pragma unroll
            for (int t = 0; t < S - 1; ++t)
              if (ok && !contains_sorted(g.col + cur.qbeg[t], cur.qdeg[t], u)) ok = false;
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
};

template <int APP, int LEV, int MODE>
void launch_extend(Ctx& c, ExtendArgs& a, const char* what, double bytes) {
  auto kern = extend_kernel<APP, LEV, MODE>;
  size_t smem = (MODE == kFused && APP == kAppMC) ? sizeof(unsigned long long) * (size_t(1) << pat::npairs(c.k)) : 0;
  static int occ = 0;  // per template instantiation
  if (occ == 0) {
    GPM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem));
    occ = std::max(1, occ);
  }
  const u64 nb = a.b_end - a.b_begin;
  const u64 warps_needed = nb;
  u64 blocks = std::min<u64>((u64)c.sms * occ, (warps_needed * 32 + kThreads - 1) / kThreads);
  blocks = std::max<u64>(1, blocks);
  GPM_CUDA(cudaMemsetAsync(c.d_ctr, 0, sizeof(unsigned long long), c.s));
  a.ctr = c.d_ctr;
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
  // ---- work pass, compaction of parents with work, scan: candidate space
  u64 nz = 0;
  DBuf<u32> pidx;
  DBuf<u64> Wp;
  {
    DBuf<u64> w(np, c.s);
    run_work<APP, LEV>(c, L, np, w.get());
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
  if (W == 0) return;
  const u64 nb = (W + kBatch - 1) / kBatch;
  ExtendArgs a{};
  a.g = c.g;
  a.L = L;
  a.Wp = Wp.get();
  a.pidx = pidx.get();
  a.np = nz;
  a.W = W;
  a.B = kBatch;
  a.b_begin = 0;
  a.b_end = nb;
  a.k = c.k;
  if (last) {
    a.hist = c.d_hist;
    a.total = c.d_total;
    launch_extend<APP, LEV, kFused>(c, a, "extend_fused", bytes_in);
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
  scan_inplace(cnt.get(), nb + 1, c.s);
  u64 T = 0;
  GPM_CUDA(cudaMemcpyAsync(&T, cnt.get() + nb, sizeof(u64), cudaMemcpyDeviceToHost, c.s));
  GPM_CUDA(cudaStreamSynchronize(c.s));
  st.level_sizes[LEV] += T;
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
    launch_extend<APP, LEV, kWrite>(c, w, "extend_write", wbytes + 8.0 * Tc);
    VLevels nl = L;
    nl.idx[LEV] = oi.get();
    nl.vid[LEV] = ov.get();
    process_dispatch<APP>(c, LEV + 1, nl, Tc);
  }
}

}  // namespace

void build_level1(const gpm_graph& g, DBuf<u32>& idx, DBuf<u32>& vid, u64& count, cudaStream_t s, Timeline& tl);

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
  DBuf<u32> l1i, l1v;
  u64 n1 = 0;
  build_level1(*G, l1i, l1v, n1, s, tl);
  u64 lo = 0, hi = n1;
  if (cfg.root_hi > 0) {
    lo = std::min(cfg.root_lo, n1);
    hi = std::min(cfg.root_hi, n1);
    if (hi < lo) hi = lo;
  } else {
    root_split(*G, l1i.get(), l1v.get(), n1, app, cfg.rank, std::max(1, cfg.world), lo, hi, s, tl);
  }
  const u64 nroot = hi - lo;
  if (nroot >= (u64(1) << 32)) throw Error(GPM_EINVAL, "level 1 exceeds 2^32 entries");
  st.level_sizes[0] = nroot;

  Ctx c{};
  c.G = G;
  c.g = G->view();
  c.app = app;
  c.k = k;
  c.s = s;
  c.tl = &tl;
  c.st = &st;
  c.sms = sm_count();
  size_t freeb = 0, totalb = 0;
  GPM_CUDA(cudaMemGetInfo(&freeb, &totalb));
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

  VLevels L{};
  L.idx[0] = l1i.get() + lo;
  L.vid[0] = l1v.get() + lo;
  const int appk = (app == GPM_APP_MC) ? kAppMC : kAppCF;  // TC == CF with k=3 (Listing 3)
  if (k == 2 || nroot == 0) {
    res.total = (k == 2) ? nroot : 0;
  } else if (appk == kAppMC) {
    process_dispatch<kAppMC>(c, 1, L, nroot);
  } else {
    process_dispatch<kAppCF>(c, 1, L, nroot);
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
  } else if (k > 2 && nroot > 0) {
    unsigned long long t = 0;
    GPM_CUDA(cudaMemcpyAsync(&t, d_total.get(), sizeof t, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaStreamSynchronize(s));
    res.total = t;
    st.level_sizes[levels - 1] += t;
  }
}

}  // namespace gpm
