// api.cu — C ABI: mine(), results, stats, errors (include/gpm.h).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <array>
#include <map>
#include <memory>

#include "engine.hpp"
#include "pattern.cuh"

namespace gpm {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

// SPEC.md:252 stable text "k=<n>;L=<l0,...>;E=(i,j)(i,j)..."
std::string canon_text(u64 key, int nv_hint, int label_bits, const std::vector<u32>* label_values) {
  int nv = 0;
  u32 lab[8] = {0};
  u32 mask = 0;
  pat::decode(key, label_bits, &nv, lab, &mask);
  (void)nv_hint;
  // "k=<n>;L=l0,l1,..;E=(i,j)..", formatted without iostreams:
  // FSM can emit ~10^6 patterns per call
  char buf[512];
  char* o = buf;
  auto put_u = [&](u32 v) {
    char t[12];
    int n = 0;
    do {
      t[n++] = (char)('0' + v % 10);
      v /= 10;
    } while (v);
    while (n) *o++ = t[--n];
  };
  *o++ = 'k';
  *o++ = '=';
  put_u((u32)nv);
  *o++ = ';';
  *o++ = 'L';
  *o++ = '=';
  for (int i = 0; i < nv; ++i) {
    if (i) *o++ = ',';
    u32 v = lab[i];
    if (label_values && !label_values->empty()) v = (*label_values)[lab[i]];
    put_u(v);
  }
  *o++ = ';';
  *o++ = 'E';
  *o++ = '=';
  for (int a = 0; a < nv; ++a)
    for (int b = a + 1; b < nv; ++b)
      if (mask >> pat::pair_index(a, b, nv) & 1u) {
        *o++ = '(';
        put_u((u32)a);
        *o++ = ',';
        put_u((u32)b);
        *o++ = ')';
      }
  return std::string(buf, o);
}

// Sum a host u64 vector across ranks through the exchange hook.
void exchange_sum_host(const gpm_config& cfg, std::vector<u64>& v, cudaStream_t s) {
  if (cfg.world <= 1 || !cfg.exchange || v.empty()) return;
  DBuf<u64> d(v.size(), s);
  GPM_CUDA(cudaMemcpyAsync(d.get(), v.data(), sizeof(u64) * v.size(), cudaMemcpyHostToDevice, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  if (cfg.exchange(cfg.exchange_ctx, d.get(), v.size(), 8, 0, s) != 0) throw Error(GPM_ENCCL, "exchange(sum) failed");
  GPM_CUDA(cudaMemcpyAsync(v.data(), d.get(), sizeof(u64) * v.size(), cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
}

// Minimum of a host u64 across ranks (all-gather, op 2): planner sizes that
// decide how many collectives a level issues must agree on every rank.
u64 exchange_min_host(const gpm_config& cfg, u64 v, cudaStream_t s) {
  if (cfg.world <= 1 || !cfg.exchange) return v;
  const int W = cfg.world;
  std::vector<u64> h(W, ~0ull);
  h[cfg.rank] = v;
  DBuf<u64> d(W, s);
  GPM_CUDA(cudaMemcpyAsync(d.get(), h.data(), sizeof(u64) * W, cudaMemcpyHostToDevice, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  if (cfg.exchange(cfg.exchange_ctx, d.get(), 1, 8, 2, s) != 0) throw Error(GPM_ENCCL, "exchange(all-gather) failed");
  GPM_CUDA(cudaMemcpyAsync(h.data(), d.get(), sizeof(u64) * W, cudaMemcpyDeviceToHost, s));
  GPM_CUDA(cudaStreamSynchronize(s));
  return *std::min_element(h.begin(), h.end());
}

void exchange_device(const gpm_config& cfg, void* dev, u64 count, int elem_bytes, int op, cudaStream_t s) {
  if (cfg.world <= 1 || !cfg.exchange || count == 0) return;
  GPM_CUDA(cudaStreamSynchronize(s));
  if (cfg.exchange(cfg.exchange_ctx, dev, count, elem_bytes, op, s) != 0) throw Error(GPM_ENCCL, "exchange failed");
}

// One thread per pattern: the device canonicaliser the FSM / MC reduce steps
// use (pattern.cuh), exposed for batches of arbitrary patterns (tests, tools).
__global__ void canon_batch_kernel(int nv, u64 count, const u32* __restrict__ lab, const u32* __restrict__ masks,
                                   int LB, u64* __restrict__ codes, u32* __restrict__ perms) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < count; i += (u64)gridDim.x * blockDim.x) {
    u32 l[8];
    for (int j = 0; j < nv; ++j) l[j] = lab[i * nv + j];
    u8 p[8];
    codes[i] = pat::canonicalize(nv, l, masks[i], LB, p);
    u32 pk = 0;
    for (int j = 0; j < nv; ++j) pk |= (u32)p[j] << (3 * j);
    perms[i] = pk;
  }
}

}  // namespace gpm

using namespace gpm;

extern "C" {

const char* gpm_last_error(void) { return g_last_error.c_str(); }

int gpm_canonicalize_batch(int device, int nv, uint64_t count, const uint32_t* labels, const uint32_t* masks,
                           uint32_t* canon_labels, uint32_t* canon_masks, uint8_t* perms) {
  return guarded([&] {
    if (nv < 1 || nv > 8) throw Error(GPM_EINVAL, "canonicalize: 1 <= nv <= 8 (SPEC.md:204)");
    if (count && (!masks || !canon_masks)) throw Error(GPM_EINVAL, "null argument");
    const int np = pat::npairs(nv);
    for (u64 i = 0; i < count; ++i)
      if (np < 32 && (masks[i] >> np)) throw Error(GPM_EINVAL, "mask has bits beyond the nv*(nv-1)/2 pairs");
    // dense, order-preserving label ranks PER PATTERN (the canonical form only
    // depends on the order of a pattern's own labels): <= nv distinct values,
    // so 3 label bits always fit the packed code (8 * 3 + 28 <= 60)
    const int LB = 3;
    std::vector<u32> rk(count * nv, 0);
    std::vector<u32> vals(count * nv, 0);  // per pattern: rank -> value
    if (labels)
      for (u64 i = 0; i < count; ++i) {
        u32* v = vals.data() + i * nv;
        std::copy(labels + i * nv, labels + (i + 1) * nv, v);
        std::sort(v, v + nv);
        const int nu = (int)(std::unique(v, v + nv) - v);
        for (int j = 0; j < nv; ++j) rk[i * nv + j] = (u32)(std::lower_bound(v, v + nu, labels[i * nv + j]) - v);
      }
    if (count == 0) return;
    GPM_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    GPM_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct SG { cudaStream_t s; ~SG() { cudaStreamSynchronize(s); cudaStreamDestroy(s); } } sg{st};
    DBuf<u32> dl(count * nv, st), dm(count, st), dp(count, st);
    DBuf<u64> dc(count, st);
    GPM_CUDA(cudaMemcpyAsync(dl.get(), rk.data(), sizeof(u32) * count * nv, cudaMemcpyHostToDevice, st));
    GPM_CUDA(cudaMemcpyAsync(dm.get(), masks, sizeof(u32) * count, cudaMemcpyHostToDevice, st));
    canon_batch_kernel<<<(unsigned)std::min<u64>(4096, (count + 127) / 128), 128, 0, st>>>(nv, count, dl.get(), dm.get(),
                                                                                           LB, dc.get(), dp.get());
    GPM_CUDA(cudaGetLastError());
    std::vector<u64> codes(count);
    std::vector<u32> pk(count);
    GPM_CUDA(cudaMemcpyAsync(codes.data(), dc.get(), sizeof(u64) * count, cudaMemcpyDeviceToHost, st));
    GPM_CUDA(cudaMemcpyAsync(pk.data(), dp.get(), sizeof(u32) * count, cudaMemcpyDeviceToHost, st));
    GPM_CUDA(cudaStreamSynchronize(st));
    for (u64 i = 0; i < count; ++i) {
      int cn = 0;
      u32 cl[8], cm = 0;
      pat::decode(codes[i], LB, &cn, cl, &cm);
      canon_masks[i] = cm;
      for (int j = 0; j < nv; ++j) {
        if (canon_labels) canon_labels[i * nv + j] = labels ? vals[i * nv + cl[j]] : 0u;
        if (perms) perms[i * nv + j] = (u8)((pk[i] >> (3 * j)) & 7u);
      }
    }
  });
}

const char* gpm_version(void) { return "gpm-b200 0.1 (sm_100a)"; }

int gpm_release_cached(int device) {
  return guarded([&] {
    int nd = 0;
    GPM_CUDA(cudaGetDeviceCount(&nd));
    int cur = 0;
    GPM_CUDA(cudaGetDevice(&cur));
    for (int d = 0; d < nd; ++d) {
      if (device >= 0 && d != device) continue;
      GPM_CUDA(cudaSetDevice(d));
      big_cache().trim(d);
    }
    mem_generation().fetch_add(1, std::memory_order_relaxed);
    GPM_CUDA(cudaSetDevice(cur));
  });
}

void gpm_config_default(gpm_config* cfg) {
  if (!cfg) return;
  std::memset(cfg, 0, sizeof(*cfg));
  cfg->app = GPM_APP_TC;
  cfg->k = 3;
  cfg->world = 1;
}

int gpm_steal_create(int device, int world, void** dev_ptr, void* ipc_handle_out) {
  if (!dev_ptr || world < 1) {
    set_last_error("gpm_steal_create: bad argument");
    return GPM_EINVAL;
  }
  return guarded([&] {
    GPM_CUDA(cudaSetDevice(device));
    void* p = nullptr;
    GPM_CUDA(cudaMalloc(&p, sizeof(unsigned long long) * world));  // not pooled: IPC-exportable
    GPM_CUDA(cudaMemset(p, 0, sizeof(unsigned long long) * world));
    if (ipc_handle_out) {
      cudaIpcMemHandle_t h;
      GPM_CUDA(cudaIpcGetMemHandle(&h, p));
      std::memcpy(ipc_handle_out, &h, sizeof h);
    }
    *dev_ptr = p;
  });
}

int gpm_steal_open(int device, const void* ipc_handle, void** dev_ptr) {
  if (!ipc_handle || !dev_ptr) {
    set_last_error("gpm_steal_open: null argument");
    return GPM_EINVAL;
  }
  return guarded([&] {
    GPM_CUDA(cudaSetDevice(device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, ipc_handle, sizeof h);
    GPM_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  });
}

int gpm_steal_reset(void* dev_ptr, int world, void* stream) {
  if (!dev_ptr || world < 1) {
    set_last_error("gpm_steal_reset: bad argument");
    return GPM_EINVAL;
  }
  return guarded([&] {
    cudaStream_t s = (cudaStream_t)stream;
    GPM_CUDA(cudaMemsetAsync(dev_ptr, 0, sizeof(unsigned long long) * world, s));
    GPM_CUDA(cudaStreamSynchronize(s));
  });
}

int gpm_steal_release(void* dev_ptr, int opened) {
  if (!dev_ptr) return GPM_OK;
  return guarded([&] {
    if (opened) GPM_CUDA(cudaIpcCloseMemHandle(dev_ptr));
    else GPM_CUDA(cudaFree(dev_ptr));
  });
}

}  // extern "C"

namespace gpm {

// gpm_mine's validation of the builtin apps' config (SPEC.md:375 conflicts).
static void check_builtin_config(const gpm_config* cfg) {
  if (cfg->app < GPM_APP_TC || cfg->app > GPM_APP_FSM) throw Error(GPM_EINVAL, "unknown app");
  if (cfg->mni_mode != GPM_MNI_CANONICAL && cfg->mni_mode != GPM_MNI_AUTOMORPHISM)
    throw Error(GPM_EINVAL, "unknown mni_mode");
  // config conflicts ("chunking + filter -> error"): the FSM
  // filter needs every root's embeddings before the next extend, so a
  // root slice is only legal as one rank's share of an exchanged job;
  // listing is a TC/CF mode; stealing only applies to the count apps
  if (cfg->list_fn && cfg->app != GPM_APP_TC && cfg->app != GPM_APP_CF)
    throw Error(GPM_ECONFIG, "listing mode: TC/CF only (SPEC.md:458)");
  if (cfg->app == GPM_APP_FSM && cfg->root_hi > 0 && !(cfg->world > 1 && cfg->exchange))
    throw Error(GPM_ECONFIG, "fsm: a root slice without a cross-rank exchange would filter on partial supports "
                             "(SPEC.md:160, :375)");
  if (cfg->app == GPM_APP_FSM && cfg->steal_ctrs)
    throw Error(GPM_ECONFIG, "fsm: work stealing conflicts with the per-level exchange (static split only)");
  if (cfg->steal_ctrs && cfg->root_hi > 0)
    throw Error(GPM_ECONFIG, "steal_ctrs and an explicit root slice are mutually exclusive");
}

// Stream, timing events and the stats record around one mine body (a builtin
// app or a user App instantiated from include/gpm_engine.cuh).
static int mine_once(const gpm_graph* g, const gpm_config* cfg, gpm_result** out, MineBody body, bool builtin) {
  *out = nullptr;
  return guarded([&] {
    if (builtin) check_builtin_config(cfg);
    if (cfg->world < 0 || (cfg->world > 1 && (cfg->rank < 0 || cfg->rank >= cfg->world)))
      throw Error(GPM_EINVAL, "bad rank/world");
    GPM_CUDA(cudaSetDevice(g->device));
    cudaStream_t s = cfg->stream ? (cudaStream_t)cfg->stream : g->stream;
    if (cfg->stream) GPM_CUDA(cudaStreamSynchronize(g->stream));  // graph upload ordered before the caller's stream
    auto res = std::make_unique<gpm_result>();
    res->app = cfg->app;
    res->k = cfg->k;
    Stats st;
    Timeline tl(s);
    cudaEvent_t e0, e1;
    GPM_CUDA(cudaEventCreate(&e0));
    GPM_CUDA(cudaEventCreate(&e1));
    GPM_CUDA(cudaEventRecord(e0, s));
    try {
      body(*g, *cfg, s, *res, st, tl);
    } catch (...) {
      cudaStreamSynchronize(s);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      throw;
    }
    GPM_CUDA(cudaEventRecord(e1, s));
    GPM_CUDA(cudaStreamSynchronize(s));
    float ms = 0;
    GPM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    struct EvDrop {
      cudaEvent_t a, b;
      ~EvDrop() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
      }
    } ev_drop{e0, e1};  // kept for the trace's per-kernel start offsets

    gpm_stats& S = res->stats;
    std::memset(&S, 0, sizeof S);
    S.n_levels = (int)std::min<size_t>(16, st.level_sizes.size());
    for (int i = 0; i < S.n_levels; ++i) {
      S.level_sizes[i] = st.level_sizes[i];
      S.candidates[i] = i < (int)st.candidates.size() ? st.candidates[i] : 0;
      S.survivors[i] = i < (int)st.survivors.size() ? st.survivors[i] : 0;
    }
    for (auto x : st.level_sizes) S.n_explored += x;
    S.b_alg = st.balg;
    S.ms_total = ms;
    S.launches = tl.launches;
    S.chunks = st.chunks;
    S.n_counted = st.counted;
    S.paths = st.paths | (st.chunks ? (u32)GPM_PATH_PLANNER_CHUNKS : 0u);
    std::map<std::string, std::array<double, 3>> per;  // name -> (ms, bytes, moved)
    static const bool trace = std::getenv("GPM_TRACE") != nullptr;
    if (trace) std::fprintf(stderr, "[gpm] mine app=%d k=%d total %.3f ms, %zu timed launches\n", cfg->app, cfg->k, ms, tl.recs.size());
    for (auto& r : tl.recs) {
      float t = 0;
      GPM_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
      if (trace) {
        float t0 = 0;
        GPM_CUDA(cudaEventElapsedTime(&t0, e0, r.a));
        std::fprintf(stderr, "[gpm]   %-28s %10.3f ms  %12.4g B_alg  (starts at %.3f ms%s)\n", r.name.c_str(), t, r.bytes,
                     t0, r.side ? ", side stream" : "");
      }
      if (r.side) continue;  // overlapped with the main stream: neither a phase nor the dominant kernel
      per[r.name][0] += t;
      per[r.name][1] += r.bytes;
      per[r.name][2] += r.moved >= 0 ? r.moved : r.bytes;
      S.ms_extend += t;
    }
    double best = -1;
    for (auto& [name, v] : per)
      if (v[0] > best) {
        best = v[0];
        S.ms_dominant = v[0];
        S.b_dominant = v[1];
        S.b_moved_dominant = v[2];
        std::snprintf(S.dominant, sizeof S.dominant, "%s", name.c_str());
      }
    *out = res.release();
  });
}

static int mine_with(const gpm_graph* g, const gpm_config* cfg, gpm_result** out, MineBody body, bool builtin) {
  if (!g || !cfg || !out) {
    set_last_error("gpm_mine: null argument");
    return GPM_EINVAL;
  }
  int rc = mine_once(g, cfg, out, body, builtin);
  // The planner sizes levels from a cached free-memory reading; memory the
  // caller allocated since (e.g. torch tensors) can make a level allocation
  // fail.  Re-plan once from a fresh reading with the library's cached
  // blocks handed back -- unless other ranks already entered collectives
  // (FSM exchanges per level) or stolen chunks would be lost.
  const bool solo = cfg->world <= 1 || !cfg->exchange;
  if (rc == GPM_ENOMEM && !cfg->steal_ctrs && (solo || cfg->app != GPM_APP_FSM)) {
    int dev = 0;
    cudaGetDevice(&dev);
    big_cache().trim(dev);
    mem_generation().fetch_add(1, std::memory_order_relaxed);
    rc = mine_once(g, cfg, out, body, builtin);
  }
  return rc;
}

static void builtin_body(const gpm_graph& g, const gpm_config& cfg, cudaStream_t s, gpm_result& res, Stats& st,
                         Timeline& tl) {
  if (cfg.app == GPM_APP_FSM) mine_fsm(g, cfg, s, res, st, tl);
  else mine_vertex(g, cfg, s, res, st, tl);
}

int run_custom(const gpm_graph* g, const gpm_config* cfg, gpm_result** out, MineBody body) {
  return mine_with(g, cfg, out, body, false);
}

}  // namespace gpm

extern "C" {

int gpm_mine(const gpm_graph* g, const gpm_config* cfg, gpm_result** out) {
  return mine_with(g, cfg, out, builtin_body, true);
}

int gpm_result_total(const gpm_result* r, uint64_t* total) {
  if (!r || !total) {
    set_last_error("null argument");
    return GPM_EINVAL;
  }
  *total = r->total;
  return GPM_OK;
}

int gpm_result_num_patterns(const gpm_result* r, uint64_t* n) {
  if (!r || !n) {
    set_last_error("null argument");
    return GPM_EINVAL;
  }
  *n = r->patterns.size() + r->kpatterns.size();
  return GPM_OK;
}

int gpm_result_pattern(const gpm_result* r, uint64_t i, char* text, size_t cap, uint64_t* support, int* level) {
  if (!r || i >= r->patterns.size() + r->kpatterns.size()) {
    set_last_error("pattern index out of range");
    return GPM_EINVAL;
  }
  if (i >= r->patterns.size()) {  // FSM record: format the canonical key now
    const auto& q = r->kpatterns[i - r->patterns.size()];
    if (text && cap) {
      const std::string t = canon_text(q.key, 0, r->label_bits, &r->label_values);
      size_t c = std::min(cap - 1, t.size());
      std::memcpy(text, t.data(), c);
      text[c] = 0;
    }
    if (support) *support = q.support;
    if (level) *level = q.level;
    return GPM_OK;
  }
  auto& p = const_cast<gpm_result*>(r)->patterns[i];
  if (p.text.empty() && p.key) p.text = canon_text(p.key, 0, r->label_bits, &r->label_values);
  if (text && cap) {
    size_t c = std::min(cap - 1, p.text.size());
    std::memcpy(text, p.text.data(), c);
    text[c] = 0;
  }
  if (support) *support = p.support;
  if (level) *level = p.level;
  return GPM_OK;
}

int gpm_result_stats(const gpm_result* r, gpm_stats* out) {
  if (!r || !out) {
    set_last_error("null argument");
    return GPM_EINVAL;
  }
  *out = r->stats;
  return GPM_OK;
}

void gpm_result_free(gpm_result* r) { delete r; }

}  // extern "C"
