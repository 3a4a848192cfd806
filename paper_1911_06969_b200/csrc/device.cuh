// device.cuh — device-side graph view, connectivity probes, memory + launch
// helpers shared by the engine translation units.
#pragma once
#include <atomic>
#include <mutex>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "common.hpp"

namespace gpm {

#define GPM_CUDA(x)                                                                                   \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess) {                                                                          \
      if (e_ == cudaErrorMemoryAllocation) throw ::gpm::Error(GPM_ENOMEM, std::string(#x) + ": out of device memory"); \
      throw ::gpm::Error(GPM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));                 \
    }                                                                                                 \
  } while (0)

constexpr int kMaxLevels = 10;   // k <= 9 vertices (CF) -> 8 stored levels
constexpr int kWarp = 32;

// Immutable CSR in HBM (graph.hpp:22-115): u64 offsets, u32 ascending lists,
// optional u32 dense label ranks.
struct DevGraph {
  const u64* __restrict__ off;
  const u32* __restrict__ col;
  const u32* __restrict__ lab;
  u32 n;
  u64 m;
  int oriented;
};

__device__ __forceinline__ u32 ldg(const u32* p) { return __ldg(p); }
__device__ __forceinline__ u64 ldg(const u64* p) { return __ldg(reinterpret_cast<const unsigned long long*>(p)); }

// Binary-search membership over a sorted list (graph.hpp:101-104, PAPER.md
// §5.4 "binary search for the connectivity check").
__device__ __forceinline__ bool contains_sorted(const u32* __restrict__ a, u32 len, u32 key) {
  const u32* base = a;
  u32 n = len;
  while (n > 1) {
    u32 half = n >> 1;
    base = (ldg(base + half - 1) < key) ? base + half : base;
    n -= half;
  }
  return n == 1 && ldg(base) == key;
}

// Directed probe x -> u (on a DAG tests the oriented edge).
__device__ __forceinline__ bool has_edge(const DevGraph& g, u32 x, u32 u) {
  u64 b = ldg(g.off + x), e = ldg(g.off + x + 1);
  return contains_sorted(g.col + b, (u32)(e - b), u);
}

// Undirected probe: search the shorter of the two lists (same answer by
// symmetry), bounding the hub cost of power-law graphs.
__device__ __forceinline__ bool has_edge_sym(const DevGraph& g, u32 x, u32 u) {
  u64 bx = ldg(g.off + x), ex = ldg(g.off + x + 1);
  u64 bu = ldg(g.off + u), eu = ldg(g.off + u + 1);
  if (ex - bx <= eu - bu) return contains_sorted(g.col + bx, (u32)(ex - bx), u);
  return contains_sorted(g.col + bu, (u32)(eu - bu), x);
}

// Open-addressing set of distinct u32 vertex ids in shared memory (linear
// probing, multiplicative hash, capacity a power of two >= 2 x keys): the
// on-chip staging of a source adjacency list.  sh = 32 -
// log2(capacity).
constexpr u32 kEmpty = 0xffffffffu;
constexpr u32 kHashMul = 0x9E3779B1u;
__device__ __forceinline__ void hs_insert(u32* T, u32 sh, u32 mask, u32 v) {
  u32 h = (v * kHashMul) >> sh;
  for (;;) {
    const u32 old = atomicCAS(T + h, kEmpty, v);
    if (old == kEmpty || old == v) return;
    h = (h + 1) & mask;
  }
}
__device__ __forceinline__ bool hs_has(const u32* T, u32 sh, u32 mask, u32 v) {
  u32 h = (v * kHashMul) >> sh;
  for (;;) {
    const u32 x = T[h];
    if (x == v) return true;
    if (x == kEmpty) return false;
    h = (h + 1) & mask;
  }
}
// Bucketised variant (4 slots = 16 B per bucket): a lookup is one LDS.128 and
// four compares; the next bucket is visited only when a bucket is full, which
// at load <= 1/4 almost never happens for any lane of a warp (linear probing
// sends most warps round a second probe).  Buckets fill left to right, so an
// empty last slot ends the search.  sh = 32 - log2(capacity / 4).
__device__ __forceinline__ void hb_insert(u32* T, u32 sh, u32 bmask, u32 v) {
  u32 b = (v * kHashMul) >> sh;
  for (;;) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const u32 old = atomicCAS(T + 4 * b + k, kEmpty, v);
      if (old == kEmpty || old == v) return;
    }
    b = (b + 1) & bmask;
  }
}
__device__ __forceinline__ bool hb_has(const u32* T, u32 sh, u32 bmask, u32 v) {
  u32 b = (v * kHashMul) >> sh;
  for (;;) {
    const uint4 x = *reinterpret_cast<const uint4*>(T + 4 * b);
    if (x.x == v || x.y == v || x.z == v || x.w == v) return true;
    if (x.w == kEmpty) return false;
    b = (b + 1) & bmask;
  }
}
// (sh, bmask) of a bucketised table of cap slots (cap a power of two >= 64)
__device__ __forceinline__ void hb_geom(u32 cap, u32& sh, u32& bmask) {
  const u32 nb = cap >> 2;
  bmask = nb - 1;
  sh = 32 - (31 - __clz(nb));
}

// Warp-collective: stages col[b, b+len) into T (maxcap >= 2 len slots) with
// the smallest power-of-two capacity >= 8 len (load <= 1/8, short probe runs)
// that fits maxcap; returns (sh, mask).
__device__ __forceinline__ void hs_stage_warp(u32* T, const u32* __restrict__ col, u64 b, u32 len, u32 maxcap,
                                              u32& sh, u32& mask) {
  const int lane = threadIdx.x & 31;
  u32 cap = 64;
  while (cap < 8 * len && cap < maxcap) cap <<= 1;
  mask = cap - 1;
  sh = 32 - (31 - __clz(cap));
  __syncwarp();
  for (u32 i = lane * 4; i < cap; i += 128)
    *reinterpret_cast<uint4*>(T + i) = make_uint4(kEmpty, kEmpty, kEmpty, kEmpty);
  __syncwarp();
  for (u32 i = lane; i < len; i += 32) hs_insert(T, sh, mask, __ldg(col + b + i));
  __syncwarp();
}

// Last index i in [lo, hi) with W[i] <= key (W non-decreasing).
__device__ __forceinline__ u64 upper_bound_prev(const u64* __restrict__ W, u64 lo, u64 hi, u64 key) {
  // find first i in [lo,hi) with W[i] > key, return i-1
  u64 l = lo, h = hi;
  while (l < h) {
    u64 mid = (l + h) >> 1;
    if (ldg(W + mid) <= key) l = mid + 1;
    else h = mid;
  }
  return l - 1;
}

__device__ __forceinline__ u32 lanemask_lt() {
  u32 r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// Large buffers (level columns, hash tables, bitmaps: 64 MiB .. tens of GB)
// come from an explicit per-process cache of cudaMalloc blocks in size
// classes of 1/8 of a power of two; small temporaries use the default
// stream-ordered pool.  With stream-ordered pools the driver kept re-mapping
// multi-GB blocks between calls (0.1-1.4 s stalls inside cudaMallocAsync on a
// 0.44 s 4-MC step, GPM_TRACE); cached blocks never go back to the driver
// unless an allocation fails.  A released block carries an event recorded on
// the releasing stream; the next owner's stream waits on it.
// Bumped when the library hands memory back to the driver outside a mine
// call (gpm_release_cached) or after an allocation failure: invalidates the
// cached free-memory readings of device_free_bytes().
inline std::atomic<unsigned>& mem_generation() {
  static std::atomic<unsigned> g{0};
  return g;
}
// Running balance of the library's own >= 64 MiB allocations per device
// (BigCache blocks handed out: -bytes, handed back: +bytes).  A cached
// free-memory reading is corrected by the change of this balance since it
// was taken, so graphs created or freed between two calls are accounted
// without another cudaMemGetInfo.
inline std::atomic<long long>& lib_delta(int dev) {
  static std::atomic<long long> d[64];
  return d[dev & 63];
}

constexpr size_t kBigAlloc = size_t(64) << 20;
inline size_t big_size_class(size_t bytes) {
  size_t p = size_t(1) << (63 - __builtin_clzll((unsigned long long)bytes));
  const size_t step = p / 8;
  return (bytes + step - 1) / step * step;
}
struct BigCache {
  struct Blk {
    void* p;
    size_t bytes;
    int dev;
    cudaEvent_t ev;
  };
  std::mutex mu;
  std::vector<Blk> free_;
  // returns every cached block of `dev` to the driver
  void trim(int dev) {
    std::vector<Blk> keep, drop;
    {
      std::lock_guard<std::mutex> lk(mu);
      for (auto& b : free_) (b.dev == dev ? drop : keep).push_back(b);
      free_.swap(keep);
    }
    for (auto& b : drop) {
      cudaEventSynchronize(b.ev);
      cudaEventDestroy(b.ev);
      cudaFree(b.p);
    }
  }
  size_t cached(int dev) {
    std::lock_guard<std::mutex> lk(mu);
    size_t t = 0;
    for (auto& b : free_)
      if (b.dev == dev) t += b.bytes;
    return t;
  }
};
inline BigCache& big_cache() {
  static BigCache* c = new BigCache;  // never destroyed: blocks may outlive static destructors
  return *c;
}
inline void* big_alloc(size_t bytes, int dev, cudaStream_t st) {
  const size_t cls = big_size_class(bytes);
  BigCache& C = big_cache();
  {
    std::lock_guard<std::mutex> lk(C.mu);
    for (size_t i = 0; i < C.free_.size(); ++i) {
      if (C.free_[i].dev == dev && C.free_[i].bytes == cls) {
        BigCache::Blk b = C.free_[i];
        C.free_[i] = C.free_.back();
        C.free_.pop_back();
        cudaStreamWaitEvent(st, b.ev, 0);
        cudaEventDestroy(b.ev);
        lib_delta(dev).fetch_sub((long long)cls, std::memory_order_relaxed);
        return b.p;
      }
    }
  }
  void* p = nullptr;
  if (cudaMalloc(&p, cls) != cudaSuccess) {
    cudaGetLastError();
    C.trim(dev);  // other size classes (and the default pool's cache): hand them back, retry once
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      cudaDeviceSynchronize();
      cudaMemPoolTrimTo(pool, 0);
    }
    cudaGetLastError();
    if (cudaMalloc(&p, cls) != cudaSuccess) {
      cudaGetLastError();
      mem_generation().fetch_add(1, std::memory_order_relaxed);
      return nullptr;
    }
  }
  lib_delta(dev).fetch_sub((long long)cls, std::memory_order_relaxed);
  return p;
}
inline void big_release(void* p, size_t bytes, int dev, cudaStream_t st) {
  cudaEvent_t ev = nullptr;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess || cudaEventRecord(ev, st) != cudaSuccess) {
    cudaGetLastError();
    cudaStreamSynchronize(st);
    if (ev) cudaEventDestroy(ev);
    cudaFree(p);
    lib_delta(dev).fetch_add((long long)big_size_class(bytes), std::memory_order_relaxed);
    return;
  }
  BigCache& C = big_cache();
  std::lock_guard<std::mutex> lk(C.mu);
  C.free_.push_back({p, big_size_class(bytes), dev, ev});
  lib_delta(dev).fetch_add((long long)big_size_class(bytes), std::memory_order_relaxed);
}

// Raw allocations outside DBuf (graph CSR arrays): same policy as DBuf.
inline cudaError_t dev_malloc(void** p, size_t bytes, cudaStream_t s) {
  if (bytes >= kBigAlloc) {
    int dev = 0;
    cudaGetDevice(&dev);
    *p = big_alloc(bytes, dev, s);
    return *p ? cudaSuccess : cudaErrorMemoryAllocation;
  }
  return cudaMallocAsync(p, bytes, s);
}
inline void dev_free(void* p, size_t bytes, int dev, cudaStream_t s) {
  if (!p) return;
  if (bytes >= kBigAlloc) big_release(p, bytes, dev, s);
  else cudaFreeAsync(p, s);
}

// Device buffer: >= 64 MiB from BigCache, else the stream-ordered default pool.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = 0;
  int dev = -1;  // >= 0: a BigCache block of that device
  DBuf() = default;
  DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) {
      const size_t bytes = count * sizeof(T);
      cudaError_t e = cudaSuccess;
      if (bytes >= kBigAlloc) {
        cudaGetDevice(&dev);
        p = static_cast<T*>(big_alloc(bytes, dev, st));
        if (!p) {
          e = cudaErrorMemoryAllocation;
          dev = -1;
        }
      } else {
        dev = -1;
        e = cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, st);
        if (e != cudaSuccess) {  // the big-buffer cache may hold the memory: hand it back, retry
          cudaGetLastError();
          int d = 0;
          cudaGetDevice(&d);
          big_cache().trim(d);
          e = cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, st);
        }
      }
      if (e != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        n = 0;
        throw Error(GPM_ENOMEM, "device allocation of " + std::to_string(count * sizeof(T)) + " bytes failed");
      }
    }
  }
  void release() {
    if (p) {
      if (dev >= 0) big_release(p, n * sizeof(T), dev, s);
      else cudaFreeAsync(p, s);
    }
    p = nullptr;
    n = 0;
    dev = -1;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s), dev(o.dev) { o.p = nullptr; o.n = 0; o.dev = -1; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s; dev = o.dev;
      o.p = nullptr; o.n = 0; o.dev = -1;
    }
    return *this;
  }
  T* get() const { return p; }
};

// Kernel timing + launch accounting for gpm_stats (CUDA events on the
// engine's stream, resolved once at the end of gpm_mine).
struct Timeline {
  struct Rec {
    std::string name;
    cudaEvent_t a, b;
    double bytes;
    double moved = -1;  // bytes the kernel actually reads when they differ from B_alg (< 0: = bytes)
    bool side = false;  // ran on a side stream beside the main stream's kernels (not a step phase)
  };
  cudaStream_t s;
  std::vector<Rec> recs;
  u64 launches = 0;
  explicit Timeline(cudaStream_t st) : s(st) {}
  ~Timeline() {
    for (auto& r : recs) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
  }
  size_t begin(const std::string& name, double bytes) {
    Rec r{name, nullptr, nullptr, bytes, -1};
    GPM_CUDA(cudaEventCreate(&r.a));
    GPM_CUDA(cudaEventCreate(&r.b));
    GPM_CUDA(cudaEventRecord(r.a, s));
    recs.push_back(r);
    return recs.size() - 1;
  }
  void end(size_t i) { GPM_CUDA(cudaEventRecord(recs[i].b, s)); }
};

// Host-side phase trace (GPM_TRACE=1): synchronises the stream and prints the
// wall time since the previous trace point.
inline void htrace(cudaStream_t s, const char* what) {
  static const bool on = std::getenv("GPM_TRACE") != nullptr;
  if (!on) return;
  cudaStreamSynchronize(s);
  static auto t0 = std::chrono::steady_clock::now();
  auto t1 = std::chrono::steady_clock::now();
  std::fprintf(stderr, "[gpm host] %8.3f ms  %s\n", std::chrono::duration<double, std::milli>(t1 - t0).count(), what);
  t0 = t1;
}

// Occupancy (blocks per SM) of a kernel, computed once per cache slot; the
// slots are shared by every thread that runs the engine.
template <class F>
inline int cached_occupancy(std::atomic<int>& slot, F&& compute) {
  int v = slot.load(std::memory_order_acquire);
  if (v == 0) {
    v = std::max(1, compute());
    slot.store(v, std::memory_order_release);
  }
  return v;
}

// Device bytes available to the engine: free memory plus what the stream-
// ordered pool holds reserved but unused (the pool keeps released blocks,
// keep_pool_warm), so the planner's budget does not shrink from call to call.
inline size_t device_free_bytes() {
  // cudaMemGetInfo costs ~1 ms of host time, and tens of ms when an NVML
  // client (nvidia-smi) is polling the device: reuse a reading taken in the
  // last 2 s on this device (the planner budgets a fraction of it, and an
  // allocation that still fails raises GPM_ENOMEM)
  int dev = 0;
  cudaGetDevice(&dev);
  struct Cached {
    int dev = -1;
    unsigned gen = 0;
    long long delta = 0;
    size_t bytes = 0;
    std::chrono::steady_clock::time_point at;
  };
  static thread_local Cached cache;
  const auto now = std::chrono::steady_clock::now();
  const unsigned gen = mem_generation().load(std::memory_order_relaxed);
  const long long delta = lib_delta(dev).load(std::memory_order_relaxed);
  if (cache.dev == dev && cache.gen == gen && now - cache.at < std::chrono::milliseconds(2000)) {
    const long long v = (long long)cache.bytes + (delta - cache.delta);
    return v > 0 ? (size_t)v : 0;
  }
  size_t freeb = 0, totalb = 0;
  GPM_CUDA(cudaMemGetInfo(&freeb, &totalb));
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long reserved = 0, used = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) == cudaSuccess &&
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess && reserved > used)
      freeb += (size_t)(reserved - used);
  }
  freeb += big_cache().cached(dev);
  cudaGetLastError();
  cache.dev = dev;
  cache.gen = gen;
  cache.delta = delta;
  cache.bytes = freeb;
  cache.at = now;
  return freeb;
}

inline int sm_count() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

}  // namespace gpm
