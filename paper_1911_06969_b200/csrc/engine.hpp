// engine.hpp — internal (C++) engine interfaces behind the C ABI.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "common.hpp"
#include "device.cuh"

struct gpm_graph {
  int device = 0;
  gpm::u32 n = 0;
  gpm::u64 m = 0;
  bool oriented = false;
  bool labeled = false;
  gpm::u64* d_off = nullptr;
  gpm::u32* d_col = nullptr;
  gpm::u32* d_lab = nullptr;            // dense label ranks (order-preserving)
  size_t sz_off = 0, sz_col = 0, sz_lab = 0;  // allocation bytes (>= 64 MiB: BigCache blocks)
  std::vector<gpm::u32> label_values;   // rank -> original label value
  int label_bits = 0;
  gpm::u32 max_deg = 0;
  cudaStream_t stream = nullptr;        // stream the arrays were allocated on
  bool owns_stream = true;              // destroy `stream` with the graph
  ~gpm_graph();
  gpm::DevGraph view() const { return gpm::DevGraph{d_off, d_col, d_lab, n, m, oriented ? 1 : 0}; }
};

struct gpm_result {
  int app = 0;
  int k = 0;
  gpm::u64 total = 0;
  struct Pattern {
    std::string text;   // empty while only the canonical key is known (FSM: formatted on access)
    gpm::u64 support;
    int level;
    gpm::u64 key = 0;   // packed canonical code (pattern.cuh)
  };
  std::vector<Pattern> patterns;
  // FSM: ~10^6 patterns per call kept as 24-byte (key, support, level)
  // records; the canonical text is formatted by gpm_result_pattern on access
  struct KeyPattern {
    gpm::u64 key;
    gpm::u64 support;
    int level;
    // no zero-fill on resize(): the ~17 MB of records are first touched by
    // the parallel writers in record() (host page faults cost ~1 ms per MB)
    KeyPattern() {}
    KeyPattern(gpm::u64 k, gpm::u64 s, int l) : key(k), support(s), level(l) {}
  };
  std::vector<KeyPattern> kpatterns;
  int label_bits = 0;                      // for formatting FSM keys lazily
  std::vector<gpm::u32> label_values;      // dense label rank -> original label
  gpm_stats stats{};
};

namespace gpm {

struct Stats {
  std::vector<u64> level_sizes, candidates, survivors;
  double balg = 0;
  double bmoved = 0;   // bytes read by kernels whose reads differ from B_alg (staged MC)
  u64 streamed = 0;    // of which: neighbour-list entries read one by one
  u64 counted = 0;     // accepted embeddings whose class came from a rank/count, not a per-candidate read
  u64 chunks = 0;
  u32 paths = 0;       // GPM_PATH_* bits
  void ensure(size_t L) {
    if (level_sizes.size() < L) level_sizes.resize(L, 0);
    if (candidates.size() < L) candidates.resize(L, 0);
    if (survivors.size() < L) survivors.resize(L, 0);
  }
};

// Level-1 build on the device (embedding_list.hpp:178-192): DAG -> every
// edge; undirected -> (u,v) with u<v.  idx[i] = first endpoint, vid[i] = second.
// Undirected graphs: *l1_start (optional) receives the exclusive prefix over
// vertices of |{v in N(u) : v > u}|, i.e. the first level-1 index of root u.
// need_idx = false (DAG only): the per-edge v0 array is not built (the k-CL
// local-row path reads the CSR offsets instead).
void build_level1(const gpm_graph& g, DBuf<u32>& idx, DBuf<u32>& vid, u64& count, cudaStream_t s, Timeline& tl,
                  const u32** vid_view = nullptr, DBuf<u64>* l1_start = nullptr, bool need_idx = true);

// Last extension of 3-MC with the root's upper adjacency staged on chip
// (mc_staged.cu): adds the 3-vertex connectivity-code counts of the level-1
// slice [lo, hi) into d_hist (8 bins) and the candidates / B_alg to st.
void mc3_staged(const gpm_graph& g, const u64* l1_start, u64 lo, u64 hi, unsigned long long* d_hist, cudaStream_t s,
                Timeline& tl, Stats& st);
// Levels 2 and 3 of 4-MC fused over the level-1 slice (l1i = v0, l1v = v1,
// nq parents): S0 / S1 staged on chip per parent, the parent's level-2
// children walked in place (never materialised); adds 6-pair code counts to
// d_hist and both levels' candidates / level size / B_alg to st.
void mc4_roots_staged(const gpm_graph& G, const u32* l1i, const u32* l1v, u64 nq, unsigned long long* d_hist,
                      cudaStream_t s, Timeline& tl, Stats& st);

// Degree-weighted static split of [0, n1) root units into `world` parts
// (SURVEY §8e); weight = candidate count of each level-1 entry.
void root_split(const gpm_graph& g, const u32* idx, const u32* vid, u64 n1, int app, int rank, int world, u64& lo,
                u64& hi, cudaStream_t s, Timeline& tl);
// The same split for every rank: bounds[r]..bounds[r+1] (world+1 entries).
void root_split_bounds(const gpm_graph& g, const u32* idx, const u32* vid, u64 n1, int app, int world,
                       std::vector<u64>& bounds, cudaStream_t s, Timeline& tl);
// Device-side work-stealing grab over the ranks' tail ranges [tlo, thi)
// (gpm_config.steal_ctrs); [lo, hi) = claimed chunk, lo == hi when all done.
void steal_grab(unsigned long long* ctrs, const u64* d_tlo, const u64* d_thi, int world, int rank, u64 chunk,
                u64* d_out, u64& lo, u64& hi, cudaStream_t s);

void keep_pool_warm(int device);

// Device orientation (graph.hpp:121-132).
void orient_on_device(const gpm_graph& g, gpm_graph& out);
void create_dag_pipelined(const u64* h_off, const u32* h_col, const u32* labels, u32 n, u64 m, gpm_graph& out);

void mine_vertex(const gpm_graph& g, const gpm_config& cfg, cudaStream_t s, gpm_result& res, Stats& st, Timeline& tl);

// One mine body run inside gpm_mine's bookkeeping (stream, events, stats).
using MineBody = void (*)(const gpm_graph&, const gpm_config&, cudaStream_t, gpm_result&, Stats&, Timeline&);
// gpm_mine for a user App instantiated from include/gpm_engine.cuh
// (gpm::mine_app<App>): same bookkeeping, no builtin-app config checks.
int run_custom(const gpm_graph* g, const gpm_config* cfg, gpm_result** out, MineBody body);
void mine_fsm(const gpm_graph& g, const gpm_config& cfg, cudaStream_t s, gpm_result& res, Stats& st, Timeline& tl);

// Collective hooks (multi-GPU, one process per GPU): sum a host vector or
// exchange a device buffer in place through gpm_config.exchange.
void exchange_sum_host(const gpm_config& cfg, std::vector<u64>& v, cudaStream_t s);
void exchange_device(const gpm_config& cfg, void* dev, u64 count, int elem_bytes, int op, cudaStream_t s);
u64 exchange_min_host(const gpm_config& cfg, u64 v, cudaStream_t s);

// Canonical pattern text from a packed canonical key (pattern.cuh).
std::string canon_text(u64 key, int nv, int label_bits, const std::vector<u32>* label_values);

}  // namespace gpm
