// graph.cu — device CSR lifecycle: upload + validation (graph.hpp:29-55),
// degree-ordered orientation (graph.hpp:121-132), level-1 init
// (embedding_list.hpp:178-192), batched is_connected (graph.hpp:93-104) and
// the degree-weighted root split.
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>

#include "engine.hpp"

namespace gpm {
namespace {

// Warp per vertex: validates strictly ascending lists, ids < n, no loops.
__global__ void validate_kernel(const u64* __restrict__ off, const u32* __restrict__ col, u32 n, u64 m,
                                int* __restrict__ bad, u32* __restrict__ maxdeg) {
  const int lane = threadIdx.x & 31;
  const u64 warp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
  const u64 nwarps = (gridDim.x * (u64)blockDim.x) >> 5;
  __shared__ u32 smax;
  __shared__ int sbad;
  if (threadIdx.x == 0) {
    smax = 0;
    sbad = 0;
  }
  __syncthreads();
  u32 mymax = 0;
  int mybad = 0;
  for (u64 v = warp; v < n; v += nwarps) {
    u64 b = off[v], e = off[v + 1];
    if (e < b || e > m) {
      mybad |= 1;
      continue;
    }
    mymax = max(mymax, (u32)(e - b));
    for (u64 i = b + lane; i < e; i += 32) {
      u32 x = col[i];
      bool ok = x < n && x != v && (i == b || col[i - 1] < x);
      if (!ok) mybad |= 2;
    }
  }
  mymax = __reduce_max_sync(0xffffffffu, mymax);
  mybad = (int)__reduce_or_sync(0xffffffffu, (unsigned)mybad);
  if (lane == 0) {
    atomicMax(&smax, mymax);
    atomicOr(&sbad, mybad);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (smax) atomicMax(maxdeg, smax);
    if (sbad) atomicOr(bad, sbad);
  }
}

// u32 degrees (and the offsets' validity, graph.hpp:29-55) for the
// orientation's (deg, id) order: one 4-byte random read per edge.
__global__ void deg32_kernel(const u64* __restrict__ off, u32 vb, u32 ve, u64 m, u32* __restrict__ deg,
                             int* __restrict__ bad) {
  int mybad = 0;
  for (u64 v = vb + blockIdx.x * (u64)blockDim.x + threadIdx.x; v < ve; v += (u64)gridDim.x * blockDim.x) {
    const u64 b = off[v], e = off[v + 1];
    const bool ok = e >= b && e <= m;
    if (!ok) mybad = 1;
    deg[v] = ok ? (u32)(e - b) : 0u;
  }
  if (mybad) atomicOr(bad, 1);
}

// Edge-balanced orientation of a vertex range [vb, ve) whose out-lists are
// the edge range [eb, ee) (graph.hpp:121-132): the DAG's column array is the
// kept half-edges in their original order, so every pass is one thread per
// edge or per vertex -- no warp walks a hub's list alone:
//   src[i]  = source vertex of edge i (scatter at list starts + max-scan)
//   keep[i] = (deg u, u) < (deg v, v), plus the graph.hpp:29-55 validation
//   kpos    = exclusive scan of keep;  dcol[base + kpos[i]] = col[i]
//   doff[u] = base + kpos[off[u] - eb]; base[k+1] = base[k] + kept in chunk k
__global__ void src_mark_kernel(const u64* __restrict__ off, u32 vb, u32 ve, u64 eb, u32* __restrict__ src) {
  for (u64 u = vb + blockIdx.x * (u64)blockDim.x + threadIdx.x; u < ve; u += (u64)gridDim.x * blockDim.x) {
    const u64 b = off[u], e = off[u + 1];
    if (e > b && b >= eb) src[b - eb] = (u32)u;
  }
}
__global__ void keep_kernel(const u64* __restrict__ off, const u32* __restrict__ col, const u32* __restrict__ deg,
                            u32 n, u64 eb, u64 ee, const u32* __restrict__ src, int validate, u32* __restrict__ keep,
                            int* __restrict__ bad) {
  int mybad = 0;
  for (u64 i = eb + blockIdx.x * (u64)blockDim.x + threadIdx.x; i < ee; i += (u64)gridDim.x * blockDim.x) {
    const u32 u = src[i - eb], v = col[i];
    if (validate && !(v < n && v != u && (i == off[u] || col[i - 1] < v))) mybad = 2;
    bool k = false;
    if (v < n) {
      const u32 du = deg[u], dv = deg[v];
      k = du != dv ? du < dv : u < v;
    }
    keep[i - eb] = k ? 1u : 0u;
  }
  mybad = (int)__reduce_or_sync(__activemask(), (unsigned)mybad);
  if (mybad && (threadIdx.x & 31) == __ffs(__activemask()) - 1) atomicOr(bad, mybad);
}
__global__ void chunk_base_kernel(const u32* __restrict__ keep, const u32* __restrict__ kpos, u64 ne, u64* __restrict__ base,
                                  int k) {
  base[k + 1] = base[k] + (ne ? (u64)kpos[ne - 1] + keep[ne - 1] : 0);
}
__global__ void dag_write_kernel(const u32* __restrict__ col, const u32* __restrict__ keep, const u32* __restrict__ kpos,
                                 u64 eb, u64 ee, const u64* __restrict__ base, int k, u32* __restrict__ dcol) {
  const u64 b0 = base[k];
  for (u64 i = eb + blockIdx.x * (u64)blockDim.x + threadIdx.x; i < ee; i += (u64)gridDim.x * blockDim.x)
    if (keep[i - eb]) dcol[b0 + kpos[i - eb]] = col[i];
}
__global__ void dag_off_kernel(const u64* __restrict__ off, u32 vb, u32 ve, u64 eb, u64 ee, const u32* __restrict__ kpos,
                               const u64* __restrict__ base, int k, u64* __restrict__ doff, u32* __restrict__ md) {
  const u64 b0 = base[k], tot = base[k + 1] - b0;
  u32 best = 0;
  for (u64 u = vb + blockIdx.x * (u64)blockDim.x + threadIdx.x; u < ve; u += (u64)gridDim.x * blockDim.x) {
    const u64 b = off[u], e = off[u + 1];
    const u64 ks = b < ee ? kpos[b - eb] : tot, ke = e < ee ? kpos[e - eb] : tot;
    doff[u] = b0 + ks;
    best = max(best, (u32)(ke - ks));
  }
  best = __reduce_max_sync(__activemask(), best);
  if ((threadIdx.x & 31) == __ffs(__activemask()) - 1 && best) atomicMax(md, best);
}

// doff[n] = total; md = max out-degree

// level 1 of an undirected graph: per vertex, entries v > u (u<v rule).
// max_v (off[v+1] - off[v]) -> *md (atomicMax per warp)
__global__ void max_degree_kernel(const u64* __restrict__ off, u32 n, u32* __restrict__ md) {
  u32 best = 0;
  for (u64 v = blockIdx.x * (u64)blockDim.x + threadIdx.x; v < n; v += (u64)gridDim.x * blockDim.x)
    best = max(best, (u32)(off[v + 1] - off[v]));
  best = __reduce_max_sync(0xffffffffu, best);
  if ((threadIdx.x & 31) == 0 && best) atomicMax(md, best);
}

__global__ void l1_count_kernel(const u64* __restrict__ off, const u32* __restrict__ col, u32 n,
                                u64* __restrict__ cnt) {
  u64 u = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  if (u >= n) return;
  u64 b = off[u], e = off[u + 1];
  // first position with col > u
  u64 lo = b, hi = e;
  while (lo < hi) {
    u64 mid = (lo + hi) >> 1;
    if (col[mid] <= u) lo = mid + 1;
    else hi = mid;
  }
  cnt[u] = e - lo;
}

__global__ void l1_fill_kernel(const u64* __restrict__ off, const u32* __restrict__ col, u32 n, int oriented,
                               const u64* __restrict__ pos, u32* __restrict__ idx, u32* __restrict__ vid) {
  const int lane = threadIdx.x & 31;
  const u64 warp = (blockIdx.x * (u64)blockDim.x + threadIdx.x) >> 5;
  const u64 nwarps = (gridDim.x * (u64)blockDim.x) >> 5;
  for (u64 u = warp; u < n; u += nwarps) {
    u64 b = off[u], e = off[u + 1];
    u64 w = oriented ? b : pos[u];
    u64 start = oriented ? b : e - (pos[u + 1] - pos[u]);
    for (u64 i = start + lane; i < e; i += 32) {
      idx[w + (i - start)] = (u32)u;
      vid[w + (i - start)] = col[i];
    }
  }
}

__global__ void l1_idx_kernel(const u64* __restrict__ off, u32 n, u32* __restrict__ idx) {
  for (u64 v = blockIdx.x * (u64)blockDim.x + threadIdx.x; v < n; v += (u64)gridDim.x * blockDim.x)
    for (u64 e = off[v], ee = off[v + 1]; e < ee; ++e) idx[e] = (u32)v;
}

__global__ void is_connected_kernel(DevGraph g, const u32* __restrict__ us, const u32* __restrict__ vs, u64 q,
                                    u8* __restrict__ out) {
  u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  if (i >= q) return;
  out[i] = has_edge(g, us[i], vs[i]) ? 1 : 0;
}

__global__ void root_weight_kernel(const u64* __restrict__ off, const u32* __restrict__ idx,
                                   const u32* __restrict__ vid, u64 n1, int both, u64* __restrict__ w) {
  u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  if (i >= n1) return;
  u32 a = idx[i], b = vid[i];
  u64 x = off[b + 1] - off[b];
  if (both) x += off[a + 1] - off[a];
  w[i] = x + 1;  // +1: every root unit costs at least its own visit
}

__global__ void lower_bound_kernel(const u64* __restrict__ pre, u64 n, const u64* __restrict__ keys, int nk,
                                   u64* __restrict__ out) {
  int t = threadIdx.x;
  if (t >= nk) return;
  u64 key = keys[t], lo = 0, hi = n;
  while (lo < hi) {
    u64 mid = (lo + hi) >> 1;
    if (pre[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  out[t] = lo;
}

void exclusive_scan_u64(u64* data, u64 n, cudaStream_t s) {
  size_t tmp = 0;
  GPM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, data, data, n, s));
  DBuf<u8> t(tmp, s);
  GPM_CUDA(cub::DeviceScan::ExclusiveSum(t.get(), tmp, data, data, n, s));
}

inline unsigned grid_for(u64 items, int per_block) {
  u64 g = (items + per_block - 1) / per_block;
  return (unsigned)std::max<u64>(1, std::min<u64>(g, 1u << 20));
}

}  // namespace

void scan_inplace(u64* data, u64 n, cudaStream_t s) { exclusive_scan_u64(data, n, s); }

// Keep freed stream-ordered allocations cached in the device pool instead of
// returning them to the driver at every synchronisation: level buffers are
// re-allocated every gpm_mine call and every level.
void keep_pool_warm(int device) {
  static bool done[64] = {false};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    u64 thr = ~u64(0);
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done[device] = true;
}

void build_level1(const gpm_graph& g, DBuf<u32>& idx, DBuf<u32>& vid, u64& count, cudaStream_t s, Timeline& tl,
                  const u32** vid_view, DBuf<u64>* l1_start, bool need_idx) {
  if (g.oriented) {
    // level 1 of a DAG is the CSR edge range itself: vid aliases col (no copy)
    count = g.m;
    if (!need_idx && vid_view) {
      *vid_view = g.d_col;
      return;
    }
    idx.alloc(std::max<u64>(1, g.m), s);
    if (vid_view) {
      *vid_view = g.d_col;
    } else {
      vid.alloc(std::max<u64>(1, g.m), s);
      if (g.m) GPM_CUDA(cudaMemcpyAsync(vid.get(), g.d_col, sizeof(u32) * g.m, cudaMemcpyDeviceToDevice, s));
    }
    if (g.m && g.n) {
      ++tl.launches;
      l1_idx_kernel<<<grid_for(g.n, 256), 256, 0, s>>>(g.d_off, g.n, idx.get());
      GPM_CUDA(cudaGetLastError());
    }
    return;
  }
  if (vid_view) *vid_view = nullptr;
  DBuf<u64> pos(g.n + 1, s);
  GPM_CUDA(cudaMemsetAsync(pos.get(), 0, sizeof(u64) * (g.n + 1), s));
  if (g.n) {
    ++tl.launches;
    l1_count_kernel<<<grid_for(g.n, 256), 256, 0, s>>>(g.d_off, g.d_col, g.n, pos.get());
    GPM_CUDA(cudaGetLastError());
  }
  exclusive_scan_u64(pos.get(), g.n + 1, s);
  GPM_CUDA(cudaMemcpyAsync(&count, pos.get() + g.n, sizeof(u64), cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  idx.alloc(std::max<u64>(1, count), s);
  vid.alloc(std::max<u64>(1, count), s);
  if (count) {
    ++tl.launches;
    l1_fill_kernel<<<grid_for((u64)g.n * 32, 256), 256, 0, s>>>(g.d_off, g.d_col, g.n, 0, pos.get(), idx.get(),
                                                                 vid.get());
    GPM_CUDA(cudaGetLastError());
  }
  if (l1_start) *l1_start = std::move(pos);
}

void root_split_bounds(const gpm_graph& g, const u32* idx, const u32* vid, u64 n1, int app, int world,
                       std::vector<u64>& bounds, cudaStream_t s, Timeline& tl) {
  bounds.assign(world + 1, n1);
  bounds[0] = 0;
  if (world <= 1 || n1 == 0) return;
  DBuf<u64> w(n1 + 1, s);
  GPM_CUDA(cudaMemsetAsync(w.get() + n1, 0, sizeof(u64), s));
  ++tl.launches;
  root_weight_kernel<<<grid_for(n1, 256), 256, 0, s>>>(g.d_off, idx, vid, n1, app == GPM_APP_MC ? 1 : 0, w.get());
  GPM_CUDA(cudaGetLastError());
  exclusive_scan_u64(w.get(), n1 + 1, s);
  u64 total = 0;
  GPM_CUDA(cudaMemcpyAsync(&total, w.get() + n1, sizeof(u64), cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  std::vector<u64> keys(world - 1);
  for (int r = 1; r < world; ++r) keys[r - 1] = (u64)((unsigned __int128)total * (u64)r / (u64)world);
  DBuf<u64> dk(world - 1, s), dout(world - 1, s);
  GPM_CUDA(cudaMemcpyAsync(dk.get(), keys.data(), sizeof(u64) * (world - 1), cudaMemcpyHostToDevice, s));
  ++tl.launches;
  lower_bound_kernel<<<(world + 31) / 32, 32, 0, s>>>(w.get(), n1 + 1, dk.get(), world - 1, dout.get());
  GPM_CUDA(cudaGetLastError());
  std::vector<u64> res(world - 1);
  GPM_CUDA(cudaMemcpyAsync(res.data(), dout.get(), sizeof(u64) * (world - 1), cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  for (int r = 1; r < world; ++r) bounds[r] = std::min(std::max(res[r - 1], bounds[r - 1]), n1);
}

void root_split(const gpm_graph& g, const u32* idx, const u32* vid, u64 n1, int app, int rank, int world, u64& lo,
                u64& hi, cudaStream_t s, Timeline& tl) {
  std::vector<u64> b;
  root_split_bounds(g, idx, vid, n1, app, world, b, s, tl);
  lo = b[rank];
  hi = b[rank + 1];
}

// Work-stealing grab (device side): one thread walks the ranks' tail counters
// from its own rank on and claims the next chunk with a system-scope atomic on
// the (possibly NVLink-peer-mapped) counter.  out = [lo, hi) or [0, 0).
__global__ void steal_grab_kernel(unsigned long long* ctrs, const u64* __restrict__ tlo, const u64* __restrict__ thi,
                                  int world, int rank, u64 chunk, u64* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int k = 0; k < world; ++k) {
    const int v = (rank + k) % world;
    const u64 len = thi[v] - tlo[v];
    if (*(volatile unsigned long long*)(ctrs + v) >= len) continue;
    const u64 t = atomicAdd_system(ctrs + v, (unsigned long long)chunk);
    if (t < len) {
      out[0] = tlo[v] + t;
      out[1] = tlo[v] + min(t + chunk, len);
      return;
    }
  }
  out[0] = out[1] = 0;
}

void steal_grab(unsigned long long* ctrs, const u64* d_tlo, const u64* d_thi, int world, int rank, u64 chunk,
                u64* d_out, u64& lo, u64& hi, cudaStream_t s) {
  steal_grab_kernel<<<1, 32, 0, s>>>(ctrs, d_tlo, d_thi, world, rank, chunk, d_out);
  GPM_CUDA(cudaGetLastError());
  u64 r[2];
  GPM_CUDA(cudaMemcpyAsync(r, d_out, sizeof r, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  lo = r[0];
  hi = r[1];
}

// out-degree maximum of a freshly built device CSR (sets gpm_graph::max_deg)
void set_max_degree(gpm_graph& out, cudaStream_t s) {
  DBuf<u32> md(1, s);
  GPM_CUDA(cudaMemsetAsync(md.get(), 0, sizeof(u32), s));
  if (out.n) {
    max_degree_kernel<<<std::min<unsigned>(grid_for(out.n, 256), 1184u), 256, 0, s>>>(out.d_off, out.n, md.get());
    GPM_CUDA(cudaGetLastError());
  }
  GPM_CUDA(cudaMemcpyAsync(&out.max_deg, md.get(), sizeof(u32), cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
}

// Orientation of chunk k = vertices [vb, ve), edges [eb, ee) of (off, col)
// into (doff, dcol) with the edge-balanced passes above; base[k] must hold
// the kept half-edges of the earlier chunks (base[0] = 0).
struct OrientScratch {
  DBuf<u32> src, keep, kpos;
  DBuf<u8> tmax, tsum;
  size_t nmax = 0, nsum = 0;
  OrientScratch(u64 cap, cudaStream_t s) : src(std::max<u64>(1, cap), s), keep(std::max<u64>(1, cap), s),
                                           kpos(std::max<u64>(1, cap), s) {
    GPM_CUDA(cub::DeviceScan::InclusiveScan(nullptr, nmax, src.get(), src.get(), cuda::maximum<u32>{}, (int64_t)std::max<u64>(1, cap), s));
    GPM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, nsum, keep.get(), kpos.get(), (int64_t)std::max<u64>(1, cap), s));
    tmax.alloc(std::max<size_t>(1, nmax), s);
    tsum.alloc(std::max<size_t>(1, nsum), s);
  }
};
void orient_chunk(const u64* off, const u32* col, const u32* deg, u32 n, u32 vb, u32 ve, u64 eb, u64 ee, int validate,
                  OrientScratch& X, u64* base, int k, u64* doff, u32* dcol, u32* md, int* bad, cudaStream_t s) {
  const u64 ne = ee - eb;
  const unsigned gv = std::min<unsigned>(grid_for(std::max<u32>(1, ve - vb), 256), 2368u);
  const unsigned ge = std::min<unsigned>(grid_for(std::max<u64>(1, ne), 256), 4736u);
  if (ne) {
    GPM_CUDA(cudaMemsetAsync(X.src.get(), 0, sizeof(u32) * ne, s));
    src_mark_kernel<<<gv, 256, 0, s>>>(off, vb, ve, eb, X.src.get());
    GPM_CUDA(cub::DeviceScan::InclusiveScan(X.tmax.get(), X.nmax, X.src.get(), X.src.get(), cuda::maximum<u32>{},
                                            (int64_t)ne, s));
    keep_kernel<<<ge, 256, 0, s>>>(off, col, deg, n, eb, ee, X.src.get(), validate, X.keep.get(), bad);
    GPM_CUDA(cub::DeviceScan::ExclusiveSum(X.tsum.get(), X.nsum, X.keep.get(), X.kpos.get(), (int64_t)ne, s));
  }
  chunk_base_kernel<<<1, 1, 0, s>>>(X.keep.get(), X.kpos.get(), ne, base, k);
  if (ne) dag_write_kernel<<<ge, 256, 0, s>>>(col, X.keep.get(), X.kpos.get(), eb, ee, base, k, dcol);
  if (ve > vb) dag_off_kernel<<<gv, 256, 0, s>>>(off, vb, ve, eb, ee, X.kpos.get(), base, k, doff, md);
  GPM_CUDA(cudaGetLastError());
}
__global__ void dag_end_kernel(const u64* __restrict__ base, int k, u64* __restrict__ doff, u32 n) { doff[n] = base[k]; }

void orient_on_device(const gpm_graph& g, gpm_graph& out) {
  cudaStream_t s = out.stream;
  out.n = g.n;
  out.oriented = true;
  out.labeled = g.labeled;
  out.label_values = g.label_values;
  out.label_bits = g.label_bits;
  GPM_CUDA(cudaStreamSynchronize(g.stream));  // source graph ordered before our stream
  out.sz_off = sizeof(u64) * (g.n + 1);
  GPM_CUDA(dev_malloc((void**)&out.d_off, out.sz_off, s));
  // the DAG keeps m/2 half-edges of a symmetric CSR; m bounds any input
  out.sz_col = sizeof(u32) * std::max<u64>(1, g.m);
  GPM_CUDA(dev_malloc((void**)&out.d_col, out.sz_col, s));
  DBuf<int> bad(1, s);
  DBuf<u32> md(1, s), deg(std::max<u32>(1, g.n), s);
  DBuf<u64> base(2, s);
  GPM_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
  GPM_CUDA(cudaMemsetAsync(md.get(), 0, sizeof(u32), s));
  GPM_CUDA(cudaMemsetAsync(base.get(), 0, sizeof(u64), s));
  if (g.n) {
    deg32_kernel<<<std::min<unsigned>(grid_for(g.n, 256), 2368u), 256, 0, s>>>(g.d_off, 0, g.n, g.m, deg.get(), bad.get());
    GPM_CUDA(cudaGetLastError());
  }
  OrientScratch X(g.m, s);
  orient_chunk(g.d_off, g.d_col, deg.get(), g.n, 0, g.n, 0, g.m, 0, X, base.get(), 0, out.d_off, out.d_col, md.get(),
               bad.get(), s);
  dag_end_kernel<<<1, 1, 0, s>>>(base.get(), 1, out.d_off, g.n);
  GPM_CUDA(cudaGetLastError());
  u64 m = 0;
  GPM_CUDA(cudaMemcpyAsync(&m, out.d_off + g.n, sizeof(u64), cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaMemcpyAsync(&out.max_deg, md.get(), sizeof(u32), cudaMemcpyDeviceToHost, s));
  if (g.labeled) {
    out.sz_lab = sizeof(u32) * std::max<u32>(1, g.n);
    GPM_CUDA(dev_malloc((void**)&out.d_lab, out.sz_lab, s));
    GPM_CUDA(cudaMemcpyAsync(out.d_lab, g.d_lab, sizeof(u32) * g.n, cudaMemcpyDeviceToDevice, s));
  }
  GPM_CUDA(cudaStreamSynchronize(s));
  out.m = m;
}

// Host CSR -> device DAG in one pipelined call: the column array is copied in
// vertex-range chunks on a copy stream while a compute stream validates and
// counts the orientation of every chunk that has landed (graph.hpp:29-55 +
// :121-132).  The undirected copy is dropped afterwards.
void create_dag_pipelined(const u64* h_off, const u32* h_col, const u32* labels, u32 n, u64 m, gpm_graph& out) {
  // Per column chunk (vertex range) as soon as it lands: validate + count the
  // kept out-edges, scan the chunk onto the running offsets (no host round
  // trip: the base is read on the device) and write its DAG lists, so the
  // whole orientation overlaps the host->device copy of the later chunks.
  cudaStream_t s = out.stream;
  cudaStream_t cs;
  GPM_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t x;
    ~StreamGuard() {
      if (!x) return;
      cudaStreamSynchronize(x);
      cudaStreamDestroy(x);
    }
  };
  StreamGuard early{cs};  // owns cs until the buffers below exist
  DBuf<u64> uoff(n + 1, s);
  DBuf<u32> ucol(std::max<u64>(1, m), s);
  DBuf<int> bad(1, s);
  DBuf<u32> md(1, s);
  // declared after the buffers, so it is destroyed first: on an exception the
  // copies still in flight on cs finish before the buffers go back to s
  early.x = nullptr;
  StreamGuard guard{cs};
  GPM_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
  GPM_CUDA(cudaMemsetAsync(md.get(), 0, sizeof(u32), s));
  out.sz_off = sizeof(u64) * (n + 1);
  GPM_CUDA(dev_malloc((void**)&out.d_off, out.sz_off, s));
  // a valid undirected CSR keeps exactly m/2 entries; m bounds any input
  out.sz_col = sizeof(u32) * std::max<u64>(1, m);
  GPM_CUDA(dev_malloc((void**)&out.d_col, out.sz_col, s));
  cudaEvent_t ready;
  GPM_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  GPM_CUDA(cudaEventRecord(ready, s));  // allocations visible to the copy stream
  GPM_CUDA(cudaStreamWaitEvent(cs, ready, 0));
  // GPM_TRACE: device timeline of the copies and the per-chunk orientation
  static const bool tr = std::getenv("GPM_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto tmark = [&](cudaStream_t st) {
    if (!tr) return;
    cudaEvent_t e;
    GPM_CUDA(cudaEventCreate(&e));
    GPM_CUDA(cudaEventRecord(e, st));
    tev.push_back(e);
  };
  const auto th0 = std::chrono::steady_clock::now();
  tmark(cs);
  GPM_CUDA(cudaMemcpyAsync(uoff.get(), h_off, sizeof(u64) * (n + 1), cudaMemcpyHostToDevice, cs));
  tmark(cs);
  // degrees (u32) as soon as the offsets have landed
  DBuf<u32> deg(std::max<u32>(1, n), s);
  cudaEvent_t offev;
  GPM_CUDA(cudaEventCreateWithFlags(&offev, cudaEventDisableTiming));
  GPM_CUDA(cudaEventRecord(offev, cs));
  GPM_CUDA(cudaStreamWaitEvent(s, offev, 0));
  if (n) deg32_kernel<<<std::min<unsigned>(grid_for(n, 256), 2368u), 256, 0, s>>>(uoff.get(), 0, n, m, deg.get(), bad.get());
  GPM_CUDA(cudaGetLastError());
  const int K = m > (u64(1) << 22) ? 8 : 1;
  std::vector<cudaEvent_t> evs;
  std::vector<std::pair<u32, u32>> ranges;
  u32 vb = 0;
  for (int k = 0; k < K && vb < n; ++k) {
    // vertex range whose edges end near (k+1)/K of m
    const u64 target = (k == K - 1) ? m : m / K * (k + 1);
    const u32 ve = (k == K - 1) ? n : (u32)(std::upper_bound(h_off, h_off + n + 1, target) - h_off - 1);
    const u32 vend = std::max(ve, vb + 1 <= n ? vb + 1 : n);
    const u64 eb = h_off[vb], ee = h_off[vend];
    if (ee > eb)
      GPM_CUDA(cudaMemcpyAsync(ucol.get() + eb, h_col + eb, sizeof(u32) * (ee - eb), cudaMemcpyHostToDevice, cs));
    cudaEvent_t ev;
    GPM_CUDA(cudaEventCreateWithFlags(&ev, tr ? 0 : cudaEventDisableTiming));
    GPM_CUDA(cudaEventRecord(ev, cs));
    evs.push_back(ev);
    ranges.emplace_back(vb, vend);
    vb = vend;
  }
  u64 maxe = 1;
  for (auto [a, b] : ranges) maxe = std::max<u64>(maxe, h_off[b] - h_off[a]);
  OrientScratch X(maxe, s);
  DBuf<u64> base(ranges.size() + 1, s);
  GPM_CUDA(cudaMemsetAsync(base.get(), 0, sizeof(u64), s));
  for (size_t k = 0; k < ranges.size(); ++k) {
    const auto [rb, re] = ranges[k];
    GPM_CUDA(cudaStreamWaitEvent(s, evs[k], 0));
    orient_chunk(uoff.get(), ucol.get(), deg.get(), n, rb, re, h_off[rb], h_off[re], 1, X, base.get(), (int)k, out.d_off,
                 out.d_col, md.get(), bad.get(), s);
    tmark(s);
  }
  dag_end_kernel<<<1, 1, 0, s>>>(base.get(), (int)ranges.size(), out.d_off, n);
  GPM_CUDA(cudaGetLastError());
  if (labels) {
    out.sz_lab = sizeof(u32) * std::max<u32>(1, n);
    GPM_CUDA(dev_malloc((void**)&out.d_lab, out.sz_lab, s));
  }
  u64 dm = 0;
  int hb = 0;
  GPM_CUDA(cudaMemcpyAsync(&dm, out.d_off + n, sizeof(u64), cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaMemcpyAsync(&out.max_deg, md.get(), sizeof(u32), cudaMemcpyDeviceToHost, s));
  tmark(s);
  GPM_CUDA(cudaStreamSynchronize(s));
  if (tr) {
    const double host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count();
    std::fprintf(stderr, "[gpm dag] host %.3f ms; device marks (ms from the first copy):", host_ms);
    for (size_t i = 1; i < tev.size(); ++i) {
      float t = 0;
      cudaEventElapsedTime(&t, tev[0], tev[i]);
      std::fprintf(stderr, " %.3f", t);
    }
    std::fprintf(stderr, "  (off copied, orient chunk 1..K, end); copies done:");
    for (auto e : evs) {
      float t = 0;
      cudaEventElapsedTime(&t, tev[0], e);
      std::fprintf(stderr, " %.3f", t);
    }
    std::fprintf(stderr, "\n");
    for (auto e : tev) cudaEventDestroy(e);
  }
  for (auto e : evs) cudaEventDestroy(e);
  cudaEventDestroy(ready);
  cudaEventDestroy(offev);
  if (hb & 1) throw Error(GPM_EINVAL, "row_offsets not non-decreasing / out of range");
  if (hb & 2) throw Error(GPM_EINVAL, "neighbor list not strictly ascending, self-loop, or id out of range");
  out.n = n;
  out.m = dm;
  out.oriented = true;
}

}  // namespace gpm

// ---------------------------------------------------------------- C ABI: graph
using namespace gpm;

gpm_graph::~gpm_graph() {
  cudaSetDevice(device);
  cudaStream_t s = stream ? stream : 0;
  dev_free(d_off, sz_off, device, s);
  dev_free(d_col, sz_col, device, s);
  dev_free(d_lab, sz_lab, device, s);
  if (stream) {
    cudaStreamSynchronize(stream);
    if (owns_stream) cudaStreamDestroy(stream);
  }
}

extern "C" int gpm_graph_create_csr(const uint64_t* row_offsets, const uint32_t* col, const uint32_t* labels,
                                    uint32_t n, uint64_t m, int oriented, int device, gpm_graph** out) {
  if (!out || !row_offsets || (m && !col)) {
    set_last_error("gpm_graph_create_csr: null argument");
    return GPM_EINVAL;
  }
  *out = nullptr;
  return guarded([&] {
    if (row_offsets[0] != 0 || row_offsets[n] != m) throw Error(GPM_EINVAL, "row_offsets must start at 0 and end at m");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw Error(GPM_ECUDA, "no CUDA device visible");
    }
    if (device < 0 || device >= ndev) throw Error(GPM_EINVAL, "device index out of range");
    GPM_CUDA(cudaSetDevice(device));
    keep_pool_warm(device);
    auto g = std::make_unique<gpm_graph>();
    g->device = device;
    g->n = n;
    g->m = m;
    g->oriented = oriented != 0;
    GPM_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    cudaStream_t s = g->stream;
    g->sz_off = sizeof(u64) * (n + 1);
    GPM_CUDA(dev_malloc((void**)&g->d_off, g->sz_off, s));
    g->sz_col = sizeof(u32) * std::max<u64>(1, m);
    GPM_CUDA(dev_malloc((void**)&g->d_col, g->sz_col, s));
    GPM_CUDA(cudaMemcpyAsync(g->d_off, row_offsets, sizeof(u64) * (n + 1), cudaMemcpyHostToDevice, s));
    if (m) GPM_CUDA(cudaMemcpyAsync(g->d_col, col, sizeof(u32) * m, cudaMemcpyHostToDevice, s));
    if (labels) {
      // order-preserving dense label ranks (canonical order is unchanged)
      std::vector<u32> vals(labels, labels + n);
      std::sort(vals.begin(), vals.end());
      vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
      g->label_values = vals;
      int lb = 0;
      while ((u64(1) << lb) < std::max<size_t>(1, vals.size())) ++lb;
      g->label_bits = lb;
      std::vector<u32> ranks(n);
      for (u32 v = 0; v < n; ++v)
        ranks[v] = (u32)(std::lower_bound(vals.begin(), vals.end(), labels[v]) - vals.begin());
      g->labeled = true;
      g->sz_lab = sizeof(u32) * std::max<u32>(1, n);
      GPM_CUDA(dev_malloc((void**)&g->d_lab, g->sz_lab, s));
      GPM_CUDA(cudaMemcpyAsync(g->d_lab, ranks.data(), sizeof(u32) * n, cudaMemcpyHostToDevice, s));
      GPM_CUDA(cudaStreamSynchronize(s));  // ranks is a host temporary
    }
    DBuf<int> bad(1, s);
    DBuf<u32> md(1, s);
    GPM_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
    GPM_CUDA(cudaMemsetAsync(md.get(), 0, sizeof(u32), s));
    if (n) {
      validate_kernel<<<grid_for((u64)n * 32, 256), 256, 0, s>>>(g->d_off, g->d_col, n, m, bad.get(), md.get());
      GPM_CUDA(cudaGetLastError());
    }
    int hb = 0;
    GPM_CUDA(cudaMemcpyAsync(&hb, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaMemcpyAsync(&g->max_deg, md.get(), sizeof(u32), cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaStreamSynchronize(s));
    if (hb & 1) throw Error(GPM_EINVAL, "row_offsets not non-decreasing / out of range");
    if (hb & 2) throw Error(GPM_EINVAL, "neighbor list not strictly ascending, self-loop, or id out of range");
    *out = g.release();
  });
}

extern "C" int gpm_graph_create_dag_csr(const uint64_t* row_offsets, const uint32_t* col, const uint32_t* labels,
                                        uint32_t n, uint64_t m, int device, gpm_graph** out) {
  if (!out || !row_offsets || (m && !col)) {
    set_last_error("gpm_graph_create_dag_csr: null argument");
    return GPM_EINVAL;
  }
  *out = nullptr;
  return guarded([&] {
    if (row_offsets[0] != 0 || row_offsets[n] != m) throw Error(GPM_EINVAL, "row_offsets must start at 0 and end at m");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw Error(GPM_ECUDA, "no CUDA device visible");
    }
    if (device < 0 || device >= ndev) throw Error(GPM_EINVAL, "device index out of range");
    GPM_CUDA(cudaSetDevice(device));
    keep_pool_warm(device);
    auto g = std::make_unique<gpm_graph>();
    g->device = device;
    GPM_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    if (labels) {
      std::vector<u32> vals(labels, labels + n);
      std::sort(vals.begin(), vals.end());
      vals.erase(std::unique(vals.begin(), vals.end()), vals.end());
      g->label_values = vals;
      int lb = 0;
      while ((u64(1) << lb) < std::max<size_t>(1, vals.size())) ++lb;
      g->label_bits = lb;
      g->labeled = true;
    }
    create_dag_pipelined(row_offsets, col, labels, n, m, *g);
    if (labels) {
      std::vector<u32> ranks(n);
      for (u32 v = 0; v < n; ++v)
        ranks[v] = (u32)(std::lower_bound(g->label_values.begin(), g->label_values.end(), labels[v]) -
                         g->label_values.begin());
      GPM_CUDA(cudaMemcpyAsync(g->d_lab, ranks.data(), sizeof(u32) * n, cudaMemcpyHostToDevice, g->stream));
      GPM_CUDA(cudaStreamSynchronize(g->stream));
    }
    *out = g.release();
  });
}

extern "C" int gpm_graph_orient_dag(const gpm_graph* g, gpm_graph** out) {
  if (!g || !out) {
    set_last_error("gpm_graph_orient_dag: null argument");
    return GPM_EINVAL;
  }
  *out = nullptr;
  return guarded([&] {
    if (g->oriented) throw Error(GPM_EINVAL, "orient_dag: graph is already oriented");
    GPM_CUDA(cudaSetDevice(g->device));
    auto o = std::make_unique<gpm_graph>();
    o->device = g->device;
    GPM_CUDA(cudaStreamCreateWithFlags(&o->stream, cudaStreamNonBlocking));
    orient_on_device(*g, *o);
    *out = o.release();
  });
}

extern "C" int gpm_graph_info(const gpm_graph* g, uint32_t* n, uint64_t* m, int* oriented, int* labeled) {
  if (!g) {
    set_last_error("null graph");
    return GPM_EINVAL;
  }
  if (n) *n = g->n;
  if (m) *m = g->m;
  if (oriented) *oriented = g->oriented;
  if (labeled) *labeled = g->labeled;
  return GPM_OK;
}

extern "C" int gpm_graph_download(const gpm_graph* g, uint64_t* row_offsets, uint32_t* col) {
  if (!g || !row_offsets || (g->m && !col)) {
    set_last_error("null argument");
    return GPM_EINVAL;
  }
  return guarded([&] {
    GPM_CUDA(cudaSetDevice(g->device));
    GPM_CUDA(cudaMemcpyAsync(row_offsets, g->d_off, sizeof(u64) * (g->n + 1), cudaMemcpyDeviceToHost, g->stream));
    if (g->m) GPM_CUDA(cudaMemcpyAsync(col, g->d_col, sizeof(u32) * g->m, cudaMemcpyDeviceToHost, g->stream));
    GPM_CUDA(cudaStreamSynchronize(g->stream));
  });
}

extern "C" int gpm_graph_is_connected(const gpm_graph* g, const uint32_t* us, const uint32_t* vs, uint64_t q,
                                      uint8_t* out) {
  if (!g || (q && (!us || !vs || !out))) {
    set_last_error("null argument");
    return GPM_EINVAL;
  }
  return guarded([&] {
    for (u64 i = 0; i < q; ++i)
      if (us[i] >= g->n || vs[i] >= g->n) throw Error(GPM_EINVAL, "is_connected: vertex id out of range");
    if (!q) return;
    GPM_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = g->stream;
    DBuf<u32> du(q, s), dv(q, s);
    DBuf<u8> dr(q, s);
    GPM_CUDA(cudaMemcpyAsync(du.get(), us, sizeof(u32) * q, cudaMemcpyHostToDevice, s));
    GPM_CUDA(cudaMemcpyAsync(dv.get(), vs, sizeof(u32) * q, cudaMemcpyHostToDevice, s));
    is_connected_kernel<<<grid_for(q, 256), 256, 0, s>>>(g->view(), du.get(), dv.get(), q, dr.get());
    GPM_CUDA(cudaGetLastError());
    GPM_CUDA(cudaMemcpyAsync(out, dr.get(), q, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" int gpm_level1(const gpm_graph* g, uint32_t* idx, uint32_t* vid, uint64_t cap, uint64_t* n_out) {
  if (!g || !n_out) {
    set_last_error("null argument");
    return GPM_EINVAL;
  }
  return guarded([&] {
    GPM_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = g->stream;
    Timeline tl(s);
    DBuf<u32> di, dv;
    u64 cnt = 0;
    build_level1(*g, di, dv, cnt, s, tl);
    *n_out = cnt;
    u64 c = std::min<u64>(cap, cnt);
    if (c && idx) GPM_CUDA(cudaMemcpyAsync(idx, di.get(), sizeof(u32) * c, cudaMemcpyDeviceToHost, s));
    if (c && vid) GPM_CUDA(cudaMemcpyAsync(vid, dv.get(), sizeof(u32) * c, cudaMemcpyDeviceToHost, s));
    GPM_CUDA(cudaStreamSynchronize(s));
  });
}

extern "C" void gpm_graph_free(gpm_graph* g) { delete g; }
