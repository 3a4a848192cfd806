// oracle/oracle.cpp — TEST INFRASTRUCTURE ONLY (the CPU checker, never the product).
//
// A plain C++20 + OpenMP restatement of the Pangolin extend-reduce-filter engine
// as specified in /root/reference/SPEC.md (modules pattern, support, engine,
// apps) and /root/reference/PAPER.md (Alg. 1 / Alg. 2, Listings 3-6), on top of
// a restatement of the CSR primitives of /root/reference/proj/include/gpmine.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library.  The product (libgpm.so) never
// links or calls it.
//
// Parity pinning: the graph primitives are checked against the reference
// headers compiled into oracle/_ref (see oracle/ref_shim.cpp); the engine is
// checked against every SPEC.md known answer and against independent
// brute-force Python oracles (tests/test_oracle_*.py).  The hot path itself
// (engine/pattern/support/apps) exists only as SPEC text in the reference, so
// these known answers + brute force are the pin.
//
// Conventions pinned here (and restated independently by the CUDA path):
//  * orientation: keep u->v iff (deg u, u) < (deg v, v)          graph.hpp:121-132
//  * level 1: all DAG edges, or undirected (u,v) with u<v, CSR order
//                                                        embedding_list.hpp:178-192
//  * vertex-mode extend: for pos with to_extend, for u in N(emb[pos]) ascending,
//    reject u in emb, then to_add
//  * MC to_add = is_auto_canonical_vertex + "emit only from p"
//  * FSM to_add = is_auto_canonical_edge + closing edge only from its
//    earlier-inserted endpoint
//  * canonicalize: lexicographic minimum of (labels, sorted edge list) over
//    all permutations in std::next_permutation order; first minimiser wins
//                                                        SPEC.md:202-210, :245-247
//  * MNI: canonical-mapping domains
//  * reduce only on the last level unless filter is on
//  * FSM: level-1 reduce+filter before the loop
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include <omp.h>

namespace orc {

using u8 = std::uint8_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;

enum App { TC = 0, CF = 1, MC = 2, FSM = 3 };

// ---------------------------------------------------------------- graph core
// Restates gpmine::Graph (graph.hpp:22-115): CSR, ascending neighbour lists,
// binary-search connectivity (graph.hpp:93-104).
struct Graph {
  u32 n = 0;
  std::vector<u64> off;
  std::vector<u32> col;
  std::vector<u32> lab;
  bool oriented = false;

  u32 deg(u32 v) const { return static_cast<u32>(off[v + 1] - off[v]); }
  const u32* nb(u32 v) const { return col.data() + off[v]; }
  bool has_edge(u32 u, u32 v) const {
    const u32* b = nb(u);
    return std::binary_search(b, b + deg(u), v);
  }
  u32 label(u32 v) const { return lab.empty() ? 0u : lab[v]; }
};

// graph.hpp:121-132: keep each undirected edge once, towards the endpoint with
// higher (degree, id).
Graph orient_dag(const Graph& g) {
  if (g.oriented) throw std::runtime_error("orient_dag: graph is already oriented");
  Graph r;
  r.n = g.n;
  r.lab = g.lab;
  r.oriented = true;
  r.off.assign(g.n + 1, 0);
  auto precedes = [&](u32 a, u32 b) {
    return g.deg(a) != g.deg(b) ? g.deg(a) < g.deg(b) : a < b;
  };
  for (u32 u = 0; u < g.n; ++u) {
    u64 c = 0;
    for (u64 e = g.off[u]; e < g.off[u + 1]; ++e) c += precedes(u, g.col[e]);
    r.off[u + 1] = r.off[u] + c;
  }
  r.col.resize(r.off[g.n]);
#pragma omp parallel for schedule(dynamic, 4096)
  for (long long uu = 0; uu < (long long)g.n; ++uu) {
    u32 u = (u32)uu;
    u64 w = r.off[u];
    for (u64 e = g.off[u]; e < g.off[u + 1]; ++e)
      if (precedes(u, g.col[e])) r.col[w++] = g.col[e];
  }
  return r;
}

// ---------------------------------------------------------------- pattern
// SPEC.md:176-190 QuickPattern / CanonicalPattern, literal form.
struct Pat {
  int nv = 0;
  std::vector<u32> lab;                      // per position
  std::vector<std::pair<int, int>> e;        // sorted, i<j
  bool operator<(const Pat& o) const {
    if (lab != o.lab) return lab < o.lab;    // labels before edges
    return e < o.e;
  }
  bool operator==(const Pat& o) const { return nv == o.nv && lab == o.lab && e == o.e; }
};

static Pat permute(const Pat& q, const std::vector<int>& perm) {
  Pat r;
  r.nv = q.nv;
  r.lab.assign(q.nv, 0);
  for (int i = 0; i < q.nv; ++i) r.lab[perm[i]] = q.lab[i];
  r.e.reserve(q.e.size());
  for (auto [a, b] : q.e) {
    int x = perm[a], y = perm[b];
    r.e.emplace_back(std::min(x, y), std::max(x, y));
  }
  std::sort(r.e.begin(), r.e.end());
  return r;
}

struct Canon {
  Pat pat;
  std::vector<int> perm;  // quick position -> canonical position
};

// brute-force lexicographic minimisation; first minimiser in
// std::next_permutation order is kept (tie-break pinned, SURVEY §7 hard part 2).
Canon canonicalize(const Pat& q) {
  if (q.nv > 8) throw std::runtime_error("canonicalize: more than 8 vertices");
  std::vector<int> p(q.nv);
  std::iota(p.begin(), p.end(), 0);
  Canon best;
  bool have = false;
  do {
    Pat c = permute(q, p);
    if (!have || c < best.pat) {
      best.pat = std::move(c);
      best.perm = p;
      have = true;
    }
  } while (std::next_permutation(p.begin(), p.end()));
  return best;
}

// SPEC.md:252 textual form "k=<n>;L=<l0,...>;E=(i,j)(i,j)..."
std::string pattern_text(const Pat& p) {
  std::string s = "k=" + std::to_string(p.nv) + ";L=";
  for (int i = 0; i < p.nv; ++i) {
    if (i) s += ",";
    s += std::to_string(p.lab[i]);
  }
  s += ";E=";
  for (auto [a, b] : p.e) s += "(" + std::to_string(a) + "," + std::to_string(b) + ")";
  return s;
}

// pair index in lexicographic order (0,1),(0,2),..,(0,k-1),(1,2),...
static inline int pair_index(int i, int j, int k) {
  // i<j
  return i * k - i * (i + 1) / 2 + (j - i - 1);
}

static Pat pat_from_mask(int k, u64 mask, const u32* labels) {
  Pat p;
  p.nv = k;
  p.lab.assign(k, 0);
  if (labels)
    for (int i = 0; i < k; ++i) p.lab[i] = labels[i];
  for (int i = 0; i < k; ++i)
    for (int j = i + 1; j < k; ++j)
      if (mask >> pair_index(i, j, k) & 1) p.e.emplace_back(i, j);
  return p;
}

// Listing 6 / SPEC.md:229-237
static bool classify_3_vertex_is_triangle(int n_edges) { return n_edges == 3; }

// ---------------------------------------------------------------- stats
struct Stats {
  std::vector<u64> level_sizes;   // |L1|, accepted per extend level
  std::vector<u64> candidates;    // per extend level: sum of deg over extended positions
  std::vector<u64> survivors;     // FSM: per level after filter
  double balg = 0;                // SURVEY §8d algorithmic bytes
  void ensure(size_t L) {
    if (level_sizes.size() < L) level_sizes.resize(L, 0);
    if (candidates.size() < L) candidates.resize(L, 0);
    if (survivors.size() < L) survivors.resize(L, 0);
  }
};

// ---------------------------------------------------------------- vertex mode
struct VLevel {
  std::vector<u32> idx, vid;
  size_t size() const { return vid.size(); }
};

// embedding_list.hpp:73-115 (vertex branch): walk idx links to level 1.
static inline void reconstruct_v(const std::vector<VLevel>& L, int lev, u64 i, u32* emb) {
  u64 p = i;
  for (int k = lev; k >= 2; --k) {
    emb[k] = L[k - 1].vid[p];
    p = L[k - 1].idx[p];
  }
  emb[0] = L[0].idx[p];
  emb[1] = L[0].vid[p];
}

static inline bool to_extend_v(int app, int s, int pos) {
  // CF/TC: Listing 3 "emb.getLastVertex() == v"; MC default true
  return app == MC ? true : pos == s - 1;
}

static inline bool to_add_v(const Graph& g, int app, const u32* emb, int s, int pos, u32 u) {
  switch (app) {
    case TC:  // PAPER.md:982-984 "check whether v2 is connected to v0"
      return g.has_edge(emb[0], u);
    case CF:  // Listing 3: connected to every earlier vertex
      for (int t = 0; t < s - 1; ++t)
        if (!g.has_edge(emb[t], u)) return false;
      return true;
    case MC: {  // SPEC.md:214 + source-position rule
      if (u <= emb[0]) return false;
      int p = -1;
      for (int t = 0; t < s; ++t)
        if (g.has_edge(emb[t], u)) { p = t; break; }
      if (p != pos) return false;
      for (int t = p + 1; t < s; ++t)
        if (u <= emb[t]) return false;
      return true;
    }
  }
  return false;
}

struct VResult {
  Stats st;
  u64 total = 0;                           // TC / CF
  std::map<std::string, u64> patterns;     // MC
};

// Alg. 1 in the edge-blocked schedule (PAPER.md:1296-1331,
// SPEC.md:142-160): level-1 chunks run through all levels; the last level is
// reduced as it is generated (reduce only on the last iteration).
VResult mine_vertex(const Graph& g, int app, int k, u64 chunk, u64 root_lo, u64 root_hi) {
  VResult R;
  const int levels = k - 1;  // L1..L_{k-1}
  R.st.ensure(levels);
  // init_single_edges (embedding_list.hpp:178-192)
  VLevel L1;
  for (u32 u = 0; u < g.n; ++u)
    for (u64 e = g.off[u]; e < g.off[u + 1]; ++e) {
      u32 v = g.col[e];
      if (!g.oriented && u >= v) continue;
      L1.idx.push_back(u);
      L1.vid.push_back(v);
    }
  root_hi = std::min<u64>(root_hi, L1.size());
  root_lo = std::min(root_lo, root_hi);
  const u64 nroot = root_hi - root_lo;
  R.st.level_sizes[0] = nroot;
  if (k <= 2 || nroot == 0) {
    R.total = (k <= 2) ? nroot : 0;
    return R;
  }
  if (chunk == 0) chunk = nroot;
  const u64 nchunks = (nroot + chunk - 1) / chunk;
  const int npairs = k * (k - 1) / 2;
  const size_t nmask = (app == MC) ? (size_t(1) << npairs) : 1;

  int nthr = omp_get_max_threads();
  std::vector<Stats> tst(nthr);
  std::vector<std::vector<u64>> tmask(nthr, std::vector<u64>(nmask, 0));
  std::vector<u64> ttotal(nthr, 0);

#pragma omp parallel
  {
    int tid = omp_get_thread_num();
    Stats& st = tst[tid];
    st.ensure(levels);
    std::vector<u64>& mcount = tmask[tid];
    u64& total = ttotal[tid];
    std::vector<VLevel> L(levels);
    std::vector<u32> cnt;
    std::vector<u64> offs;
    u32 emb[16];
#pragma omp for schedule(dynamic, 1)
    for (long long c = 0; c < (long long)nchunks; ++c) {
      u64 b = root_lo + (u64)c * chunk, e = std::min(root_hi, b + chunk);
      L[0].idx.assign(L1.idx.begin() + b, L1.idx.begin() + e);
      L[0].vid.assign(L1.vid.begin() + b, L1.vid.begin() + e);
      for (int lev = 1; lev <= levels - 1; ++lev) {
        const bool last = (lev == levels - 1);
        const int s = lev + 1;  // parent embedding size
        const VLevel& P = L[lev - 1];
        const u64 np = P.size();
        if (!last) {
          // inspection
          cnt.assign(np, 0);
          for (u64 i = 0; i < np; ++i) {
            reconstruct_v(L, lev, i, emb);
            u32 c2 = 0;
            for (int pos = 0; pos < s; ++pos) {
              if (!to_extend_v(app, s, pos)) continue;
              u32 v = emb[pos];
              st.candidates[lev] += g.deg(v);
              st.balg += 16.0 + 4.0 * g.deg(v);
              for (const u32* q = g.nb(v); q != g.nb(v) + g.deg(v); ++q) {
                u32 u = *q;
                bool inemb = false;
                for (int t = 0; t < s; ++t) inemb |= (emb[t] == u);
                if (inemb) continue;
                c2 += to_add_v(g, app, emb, s, pos, u);
              }
            }
            st.balg += 8.0 * lev;
            cnt[i] = c2;
          }
          // exclusive scan -> start indices
          offs.assign(np + 1, 0);
          for (u64 i = 0; i < np; ++i) offs[i + 1] = offs[i] + cnt[i];
          const u64 tot = offs[np];
          if (tot >= (u64(1) << 32)) throw std::runtime_error("level exceeds 2^32 entries; lower chunk size");
          VLevel& O = L[lev];
          O.idx.assign(tot, 0);
          O.vid.assign(tot, 0);
          // execution: write at reserved offsets
          for (u64 i = 0; i < np; ++i) {
            if (!cnt[i]) continue;
            reconstruct_v(L, lev, i, emb);
            u64 w = offs[i];
            for (int pos = 0; pos < s; ++pos) {
              if (!to_extend_v(app, s, pos)) continue;
              u32 v = emb[pos];
              for (const u32* q = g.nb(v); q != g.nb(v) + g.deg(v); ++q) {
                u32 u = *q;
                bool inemb = false;
                for (int t = 0; t < s; ++t) inemb |= (emb[t] == u);
                if (inemb) continue;
                if (to_add_v(g, app, emb, s, pos, u)) {
                  O.idx[w] = (u32)i;
                  O.vid[w] = u;
                  ++w;
                }
              }
            }
          }
          st.level_sizes[lev] += tot;
          st.balg += 8.0 * tot;
        } else {
          // last level: extend fused with reduce (never materialised)
          u64 acc = 0;
          for (u64 i = 0; i < np; ++i) {
            reconstruct_v(L, lev, i, emb);
            u64 pmask = 0;
            if (app == MC) {
              for (int a = 0; a < s; ++a)
                for (int bb = a + 1; bb < s; ++bb)
                  if (g.has_edge(emb[a], emb[bb])) pmask |= u64(1) << pair_index(a, bb, k);
            }
            for (int pos = 0; pos < s; ++pos) {
              if (!to_extend_v(app, s, pos)) continue;
              u32 v = emb[pos];
              st.candidates[lev] += g.deg(v);
              st.balg += 16.0 + 4.0 * g.deg(v);
              for (const u32* q = g.nb(v); q != g.nb(v) + g.deg(v); ++q) {
                u32 u = *q;
                bool inemb = false;
                for (int t = 0; t < s; ++t) inemb |= (emb[t] == u);
                if (inemb) continue;
                if (!to_add_v(g, app, emb, s, pos, u)) continue;
                ++acc;
                if (app == MC) {
                  // quick pattern = induced edges among positions
                  u64 m = pmask;
                  for (int t = 0; t < s; ++t)
                    if (t == pos || g.has_edge(emb[t], u)) m |= u64(1) << pair_index(t, s, k);
                  ++mcount[m];
                }
              }
            }
            st.balg += 8.0 * lev;
          }
          st.level_sizes[lev] += acc;
          total += acc;
        }
      }
    }
  }
  for (int t = 0; t < nthr; ++t) {
    for (int l = 1; l < levels; ++l) {
      R.st.level_sizes[l] += tst[t].level_sizes[l];
      R.st.candidates[l] += tst[t].candidates[l];
    }
    R.st.balg += tst[t].balg;
    R.total += ttotal[t];
  }
  if (app == MC) {
    // two-level reduce: quick pattern (mask) -> canonical pattern
    std::vector<u64> merged(nmask, 0);
    for (int t = 0; t < nthr; ++t)
      for (size_t m = 0; m < nmask; ++m) merged[m] += tmask[t][m];
    std::string tri, wedge;
    if (k == 3) {
      tri = pattern_text(canonicalize(pat_from_mask(3, 7, nullptr)).pat);
      wedge = pattern_text(canonicalize(pat_from_mask(3, 3, nullptr)).pat);
    }
    for (size_t m = 0; m < nmask; ++m) {
      if (!merged[m]) continue;
      std::string key;
      if (k == 3)  // customised classifier, Listing 6
        key = classify_3_vertex_is_triangle(__builtin_popcountll(m)) ? tri : wedge;
      else
        key = pattern_text(canonicalize(pat_from_mask(k, m, nullptr)).pat);
      R.patterns[key] += merged[m];
    }
  }
  return R;
}

// ---------------------------------------------------------------- edge mode (FSM)
struct ELevel {
  std::vector<u32> idx, vid;
  std::vector<u8> his;
  size_t size() const { return vid.size(); }
};

struct EEmb {
  int nv = 0, ne = 0;
  u32 v[10];
  int slot[10];   // chain slot where the position's vertex was introduced
  int step[10];   // edge step after which the vertex belongs to V_t
  std::pair<u32, u32> e[10];   // normalised edges e_1..e_ne (vertex ids)
  int ea[10], eb[10];          // position pairs
  int pos_of(u32 w) const {
    for (int i = 0; i < nv; ++i)
      if (v[i] == w) return i;
    return nv;
  }
};

static inline std::pair<u32, u32> norm(u32 a, u32 b) { return a < b ? std::make_pair(a, b) : std::make_pair(b, a); }

// embedding_list.hpp:73-115 (edge branch): dedup the chain into vertices,
// translate (his, slot) pairs into position pairs.
static void reconstruct_e(const std::vector<ELevel>& L, int lev, u64 i, EEmb& E) {
  u32 chain[12];
  int his[12];
  u64 p = i;
  for (int k = lev; k >= 2; --k) {
    chain[k] = L[k - 1].vid[p];
    his[k] = L[k - 1].his[p];
    p = L[k - 1].idx[p];
  }
  chain[0] = L[0].idx[p];
  chain[1] = L[0].vid[p];
  his[1] = 0;
  int slotpos[12];
  E.nv = 0;
  for (int j = 0; j <= lev; ++j) {
    int at = E.pos_of(chain[j]);
    if (at == E.nv) {
      E.v[E.nv] = chain[j];
      E.slot[E.nv] = j;
      E.step[E.nv] = std::max(1, j);
      ++E.nv;
    }
    slotpos[j] = at;
  }
  E.ne = lev;
  for (int j = 1; j <= lev; ++j) {
    E.e[j - 1] = norm(chain[his[j]], chain[j]);
    E.ea[j - 1] = slotpos[his[j]];
    E.eb[j - 1] = slotpos[j];
  }
}

// quick pattern key: nv, edge mask over position pairs, labels
using QKey = std::array<u32, 8>;  // [nv, mask, l0..l5]
struct QKeyHash {
  size_t operator()(const QKey& k) const {
    u64 h = 1469598103934665603ull;
    for (u32 x : k) { h ^= x; h *= 1099511628211ull; }
    return (size_t)h;
  }
};

static QKey quick_key(const Graph& g, const EEmb& E) {
  QKey k{};
  k[0] = (u32)E.nv;
  u32 m = 0;
  for (int j = 0; j < E.ne; ++j) {
    int a = std::min(E.ea[j], E.eb[j]), b = std::max(E.ea[j], E.eb[j]);
    m |= 1u << pair_index(a, b, E.nv);
  }
  k[1] = m;
  for (int i = 0; i < E.nv; ++i) k[2 + i] = g.label(E.v[i]);
  return k;
}

static Pat pat_from_qkey(const QKey& k) {
  Pat p;
  p.nv = (int)k[0];
  p.lab.assign(p.nv, 0);
  for (int i = 0; i < p.nv; ++i) p.lab[i] = k[2 + i];
  for (int i = 0; i < p.nv; ++i)
    for (int j = i + 1; j < p.nv; ++j)
      if (k[1] >> pair_index(i, j, p.nv) & 1) p.e.emplace_back(i, j);
  return p;
}

// Enumerate accepted children of parent i at level lev.
template <class F>
static void extend_edge_parent(const Graph& g, const EEmb& E, u64 i, Stats* st, int lev, F&& emit) {
  for (int q = 0; q < E.nv; ++q) {
    const u32 x = E.v[q];
    if (st) {
      st->candidates[lev] += g.deg(x);
      st->balg += 16.0 + 4.0 * g.deg(x);
    }
    for (const u32* it = g.nb(x); it != g.nb(x) + g.deg(x); ++it) {
      const u32 w = *it;
      auto ne = norm(x, w);
      bool dup = false;
      for (int j = 0; j < E.ne; ++j) dup |= (E.e[j] == ne);
      if (dup) continue;                    // e not in emb
      const int r = E.pos_of(w);
      if (r < E.nv && r < q) continue;      // closing edge: earlier-inserted endpoint only
      if (!(ne > E.e[0])) continue;         // e > e_1
      int p = E.step[q];
      if (r < E.nv) p = std::min(p, E.step[r]);
      bool ok = true;
      for (int s = p + 1; s <= E.ne; ++s)
        if (!(ne > E.e[s - 1])) { ok = false; break; }
      if (!ok) continue;
      emit(q, w, r);
    }
  }
  if (st) st->balg += 8.0 * lev;
}

static void child_emb(const EEmb& P, int q, u32 w, int r, EEmb& C) {
  C = P;
  int wpos = r;
  if (r == P.nv) {
    C.v[C.nv] = w;
    C.slot[C.nv] = P.ne + 1;
    C.step[C.nv] = P.ne + 1;
    wpos = C.nv;
    ++C.nv;
  }
  C.e[C.ne] = norm(P.v[q], w);
  C.ea[C.ne] = q;
  C.eb[C.ne] = wpos;
  ++C.ne;
}

struct FSMPattern {
  int level;
  std::string text;
  u64 support;
};

struct FResult {
  Stats st;
  std::vector<FSMPattern> patterns;
};

// Per-level reduce: quick pattern -> canonical pattern, counts, MNI domains.
struct ReduceState {
  std::unordered_map<QKey, u64, QKeyHash> qcount;
  std::unordered_map<QKey, std::pair<int, std::vector<int>>, QKeyHash> qinfo;  // pid, perm
  std::vector<Pat> pats;
  std::vector<u64> pcount;
  std::vector<int> slot;                      // pid -> bitmap slot or -1
  std::vector<std::vector<std::atomic<u64>>*> bits;  // slot -> nv*words
  std::vector<u64> mni;
  size_t words = 0;
  ~ReduceState() {
    for (auto* b : bits) delete b;
  }
};

static bool g_mni_full = false;  // full-automorphism MNI (oracle_mine_json mni_mode)

// Builds pids from merged quick counts; allocates domain bitsets for
// count-frequent patterns (count >= sigma is necessary for MNI >= sigma).
static void reduce_canon(ReduceState& RS, u32 n, u64 sigma) {
  std::map<std::string, int> by_text;
  for (auto& [qk, c] : RS.qcount) {
    Canon cn = canonicalize(pat_from_qkey(qk));
    std::string t = pattern_text(cn.pat);
    auto it = by_text.find(t);
    int pid;
    if (it == by_text.end()) {
      pid = (int)RS.pats.size();
      by_text.emplace(t, pid);
      RS.pats.push_back(cn.pat);
      RS.pcount.push_back(0);
    } else {
      pid = it->second;
    }
    RS.pcount[pid] += c;
    RS.qinfo.emplace(qk, std::make_pair(pid, cn.perm));
  }
  RS.words = (n + 63) / 64;
  RS.slot.assign(RS.pats.size(), -1);
  for (size_t p = 0; p < RS.pats.size(); ++p) {
    // MNI <= count (one vertex per domain per embedding); the full-automorphism
    // MNI unions an orbit's domains, so only MNI <= nv * count holds there
    if (RS.pcount[p] * (g_mni_full ? (u64)RS.pats[p].nv : 1) >= sigma) {
      RS.slot[p] = (int)RS.bits.size();
      auto* b = new std::vector<std::atomic<u64>>(RS.words * RS.pats[p].nv);
      for (auto& x : *b) x.store(0, std::memory_order_relaxed);
      RS.bits.push_back(b);
    }
  }
}

// domain_support + merge_domain: domains[perm[i]] |= {v_i}
static void reduce_domain(ReduceState& RS, const Graph& g, const EEmb& E) {
  QKey qk = quick_key(g, E);
  auto it = RS.qinfo.find(qk);
  if (it == RS.qinfo.end()) return;
  int pid = it->second.first;
  int sl = RS.slot[pid];
  if (sl < 0) return;
  auto& b = *RS.bits[sl];
  const auto& perm = it->second.second;
  for (int i = 0; i < E.nv; ++i) {
    u32 v = E.v[i];
    b[(size_t)perm[i] * RS.words + (v >> 6)].fetch_or(u64(1) << (v & 63), std::memory_order_relaxed);
  }
}

// Automorphism orbits of a canonical pattern ("true MNI would
// union over all isomorphic mappings including pattern automorphisms"):
// brute force over every permutation; orbit id = smallest member.
static std::vector<int> automorphism_orbits(const Pat& P) {
  std::vector<int> rep(P.nv), p(P.nv);
  std::iota(rep.begin(), rep.end(), 0);
  std::iota(p.begin(), p.end(), 0);
  do {
    if (permute(P, p) == P)
      for (int j = 0; j < P.nv; ++j) {
        int a = rep[j], b = rep[p[j]];
        if (a == b) continue;
        int lo = std::min(a, b), hi = std::max(a, b);
        for (int& x : rep)
          if (x == hi) x = lo;
      }
  } while (std::next_permutation(p.begin(), p.end()));
  return rep;
}

// mni; full-automorphism variant: min over automorphism
// orbits of the union of the orbit's canonical domains
static void reduce_mni(ReduceState& RS) {
  RS.mni.assign(RS.pats.size(), 0);
  for (size_t p = 0; p < RS.pats.size(); ++p) {
    int sl = RS.slot[p];
    if (sl < 0) continue;
    auto& b = *RS.bits[sl];
    const int nv = RS.pats[p].nv;
    std::vector<int> rep(nv);
    if (g_mni_full) rep = automorphism_orbits(RS.pats[p]);
    else std::iota(rep.begin(), rep.end(), 0);
    u64 mn = ~u64(0);
    for (int pos = 0; pos < nv; ++pos) {
      if (rep[pos] != pos) continue;
      u64 c = 0;
      for (size_t w = 0; w < RS.words; ++w) {
        u64 x = 0;
        for (int o = 0; o < nv; ++o)
          if (rep[o] == pos) x |= b[o * RS.words + w].load(std::memory_order_relaxed);
        c += __builtin_popcountll(x);
      }
      mn = std::min(mn, c);
    }
    RS.mni[p] = mn;
  }
}

static int pid_of(const ReduceState& RS, const Graph& g, const EEmb& E) {
  return RS.qinfo.at(quick_key(g, E)).first;
}

FResult mine_fsm(const Graph& g, int k, u64 sigma, u64 root_lo = 0, u64 root_hi = ~u64(0)) {
  if (g.lab.empty()) throw std::runtime_error("fsm: graph is unlabeled");
  if (g.oriented) throw std::runtime_error("fsm: graph must be undirected");
  if (k < 2 || k > 6) throw std::runtime_error("fsm: k must be in [2,6]");
  FResult R;
  const int levels = k - 1;  // number of edges of the largest pattern
  R.st.ensure(levels);
  std::vector<ELevel> L(levels);
  for (u32 u = 0; u < g.n; ++u)
    for (u64 e = g.off[u]; e < g.off[u + 1]; ++e) {
      u32 v = g.col[e];
      if (u >= v) continue;
      L[0].idx.push_back(u);
      L[0].vid.push_back(v);
      L[0].his.push_back(0);
    }
  // optional level-1 slice (bounded CPU samples / partition tests)
  root_hi = std::min<u64>(root_hi, L[0].size());
  root_lo = std::min(root_lo, root_hi);
  if (root_lo > 0 || root_hi < L[0].size()) {
    ELevel S;
    S.idx.assign(L[0].idx.begin() + root_lo, L[0].idx.begin() + root_hi);
    S.vid.assign(L[0].vid.begin() + root_lo, L[0].vid.begin() + root_hi);
    S.his.assign(root_hi - root_lo, 0);
    L[0] = std::move(S);
  }
  R.st.level_sizes[0] = L[0].size();
  const int nthr = omp_get_max_threads();

  auto record = [&](ReduceState& RS, int lev) {
    for (size_t p = 0; p < RS.pats.size(); ++p)
      if (RS.slot[p] >= 0 && RS.mni[p] >= sigma)
        R.patterns.push_back({lev, pattern_text(RS.pats[p]), RS.mni[p]});
  };

  // merge per-thread quick counts
  auto merge_counts = [&](std::vector<std::unordered_map<QKey, u64, QKeyHash>>& tq, ReduceState& RS) {
    for (auto& m : tq)
      for (auto& [kk, c] : m) RS.qcount[kk] += c;
  };

  // ---- level 1: reduce + filter before the main loop
  {
    ReduceState RS;
    const u64 np = L[0].size();
    std::vector<std::unordered_map<QKey, u64, QKeyHash>> tq(nthr);
#pragma omp parallel
    {
      auto& m = tq[omp_get_thread_num()];
      EEmb E;
#pragma omp for schedule(static)
      for (long long i = 0; i < (long long)np; ++i) {
        reconstruct_e(L, 1, (u64)i, E);
        ++m[quick_key(g, E)];
      }
    }
    merge_counts(tq, RS);
    reduce_canon(RS, g.n, sigma);
#pragma omp parallel
    {
      EEmb E;
#pragma omp for schedule(static)
      for (long long i = 0; i < (long long)np; ++i) {
        reconstruct_e(L, 1, (u64)i, E);
        reduce_domain(RS, g, E);
      }
    }
    reduce_mni(RS);
    record(RS, 1);
    // filter: keep iff !(MNI < sigma)
    ELevel F;
    for (u64 i = 0; i < np; ++i) {
      EEmb E;
      reconstruct_e(L, 1, i, E);
      int pid = pid_of(RS, g, E);
      if (RS.slot[pid] >= 0 && RS.mni[pid] >= sigma) {
        F.idx.push_back(L[0].idx[i]);
        F.vid.push_back(L[0].vid[i]);
        F.his.push_back(0);
      }
    }
    L[0] = std::move(F);
    R.st.survivors[0] = L[0].size();
  }

  for (int lev = 1; lev <= levels - 1; ++lev) {
    const bool last = (lev == levels - 1);
    const u64 np = L[lev - 1].size();
    ReduceState RS;
    std::vector<Stats> tst(nthr);
    for (auto& s : tst) s.ensure(levels);
    // pass 1: per-parent accepted counts + quick-pattern counts
    std::vector<u32> cnt(np, 0);
    std::vector<std::unordered_map<QKey, u64, QKeyHash>> tq(nthr);
#pragma omp parallel
    {
      int tid = omp_get_thread_num();
      auto& m = tq[tid];
      EEmb P, C;
#pragma omp for schedule(dynamic, 256)
      for (long long ii = 0; ii < (long long)np; ++ii) {
        u64 i = (u64)ii;
        reconstruct_e(L, lev, i, P);
        u32 c = 0;
        extend_edge_parent(g, P, i, &tst[tid], lev, [&](int q, u32 w, int r) {
          child_emb(P, q, w, r, C);
          ++m[quick_key(g, C)];
          ++c;
        });
        cnt[i] = c;
      }
    }
    u64 acc = 0;
    for (u64 i = 0; i < np; ++i) acc += cnt[i];
    for (auto& s : tst) {
      R.st.candidates[lev] += s.candidates[lev];
      R.st.balg += s.balg;
    }
    R.st.level_sizes[lev] = acc;
    merge_counts(tq, RS);
    reduce_canon(RS, g.n, sigma);
    // pass 2: domains
#pragma omp parallel
    {
      EEmb P, C;
#pragma omp for schedule(dynamic, 256)
      for (long long ii = 0; ii < (long long)np; ++ii) {
        u64 i = (u64)ii;
        if (!cnt[i]) continue;
        reconstruct_e(L, lev, i, P);
        extend_edge_parent(g, P, i, nullptr, lev, [&](int q, u32 w, int r) {
          child_emb(P, q, w, r, C);
          reduce_domain(RS, g, C);
        });
      }
    }
    reduce_mni(RS);
    record(RS, lev + 1);
    if (last) break;
    // filter fused with the write pass (inspection-execution of survivors)
    std::vector<u32> scnt(np, 0);
#pragma omp parallel
    {
      EEmb P, C;
#pragma omp for schedule(dynamic, 256)
      for (long long ii = 0; ii < (long long)np; ++ii) {
        u64 i = (u64)ii;
        if (!cnt[i]) continue;
        reconstruct_e(L, lev, i, P);
        u32 c = 0;
        extend_edge_parent(g, P, i, nullptr, lev, [&](int q, u32 w, int r) {
          child_emb(P, q, w, r, C);
          int pid = pid_of(RS, g, C);
          c += (RS.slot[pid] >= 0 && RS.mni[pid] >= sigma);
        });
        scnt[i] = c;
      }
    }
    std::vector<u64> offs(np + 1, 0);
    for (u64 i = 0; i < np; ++i) offs[i + 1] = offs[i] + scnt[i];
    const u64 tot = offs[np];
    ELevel& O = L[lev];
    O.idx.assign(tot, 0);
    O.vid.assign(tot, 0);
    O.his.assign(tot, 0);
#pragma omp parallel
    {
      EEmb P, C;
#pragma omp for schedule(dynamic, 256)
      for (long long ii = 0; ii < (long long)np; ++ii) {
        u64 i = (u64)ii;
        if (!scnt[i]) continue;
        reconstruct_e(L, lev, i, P);
        u64 w = offs[i];
        extend_edge_parent(g, P, i, nullptr, lev, [&](int q, u32 wv, int r) {
          child_emb(P, q, wv, r, C);
          int pid = pid_of(RS, g, C);
          if (RS.slot[pid] >= 0 && RS.mni[pid] >= sigma) {
            O.idx[w] = (u32)i;
            O.vid[w] = wv;
            O.his[w] = (u8)P.slot[q];
            ++w;
          }
        });
      }
    }
    R.st.survivors[lev] = tot;
    R.st.balg += 9.0 * tot;
  }
  return R;
}

}  // namespace orc

// ---------------------------------------------------------------- C ABI (tests only)
namespace {
char* dup_string(const std::string& s) {
  char* p = (char*)std::malloc(s.size() + 1);
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}
std::string json_u64_list(const std::vector<orc::u64>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) s += ",";
    s += std::to_string(v[i]);
  }
  return s + "]";
}
orc::Graph make_graph(const orc::u64* off, const orc::u32* col, const orc::u32* lab, orc::u32 n, orc::u64 m, int oriented) {
  orc::Graph g;
  g.n = n;
  g.off.assign(off, off + n + 1);
  g.col.assign(col, col + m);
  if (lab) g.lab.assign(lab, lab + n);
  g.oriented = oriented != 0;
  return g;
}
}  // namespace

extern "C" {

void oracle_free(char* p) { std::free(p); }

// Returns a malloc'd JSON record; {"error": "..."} on failure.
char* oracle_mine_json(const std::uint64_t* off, const std::uint32_t* col, const std::uint32_t* labels,
                       std::uint32_t n, std::uint64_t m, int oriented, int app, int k,
                       std::uint64_t min_support, int threads, std::uint64_t chunk_size,
                       std::uint64_t root_lo, std::uint64_t root_hi, int no_orient, int mni_mode) {
  try {
    orc::g_mni_full = mni_mode == 1;
    if (threads > 0) omp_set_num_threads(threads);
    orc::Graph g = make_graph(off, col, labels, n, m, oriented);
    std::string out = "{";
    auto t0 = std::chrono::steady_clock::now();
    double ms = 0;
    if (app == orc::FSM) {
      auto R = orc::mine_fsm(g, k, min_support, root_lo, root_hi);
      ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      std::sort(R.patterns.begin(), R.patterns.end(), [](const orc::FSMPattern& a, const orc::FSMPattern& b) {
        if (a.level != b.level) return a.level < b.level;
        if (a.support != b.support) return a.support > b.support;
        return a.text < b.text;
      });
      out += "\"app\":\"fsm\",\"patterns\":[";
      for (size_t i = 0; i < R.patterns.size(); ++i) {
        if (i) out += ",";
        out += "[" + std::to_string(R.patterns[i].level) + ",\"" + R.patterns[i].text + "\"," +
               std::to_string(R.patterns[i].support) + "]";
      }
      out += "],\"level_sizes\":" + json_u64_list(R.st.level_sizes) +
             ",\"candidates\":" + json_u64_list(R.st.candidates) +
             ",\"survivors\":" + json_u64_list(R.st.survivors);
      orc::u64 nexp = 0;
      for (auto x : R.st.level_sizes) nexp += x;
      out += ",\"n_explored\":" + std::to_string(nexp);
      char buf[64];
      std::snprintf(buf, sizeof buf, "%.0f", R.st.balg);
      out += ",\"b_alg\":" + std::string(buf);
    } else {
      if (app != orc::TC && app != orc::CF && app != orc::MC) throw std::runtime_error("unknown app");
      if (app == orc::TC) k = 3;
      if (app == orc::MC && (k < 3 || k > 5)) throw std::runtime_error("motif_count: k must be in {3,4,5}");
      if (app == orc::CF && (k < 3 || k > 9)) throw std::runtime_error("clique_find: k must be in [3,9]");
      orc::Graph h;
      const orc::Graph* gp = &g;
      if ((app == orc::TC || app == orc::CF) && !g.oriented && !no_orient) {
        h = orc::orient_dag(g);
        gp = &h;
      }
      t0 = std::chrono::steady_clock::now();
      auto R = orc::mine_vertex(*gp, app, k, chunk_size, root_lo, root_hi);
      ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      static const char* names[] = {"tc", "cf", "mc"};
      out += "\"app\":\"" + std::string(names[app]) + "\",\"total\":" + std::to_string(R.total);
      out += ",\"patterns\":[";
      bool first = true;
      for (auto& [t, c] : R.patterns) {
        if (!first) out += ",";
        first = false;
        out += "[" + std::to_string(k) + ",\"" + t + "\"," + std::to_string(c) + "]";
      }
      out += "],\"level_sizes\":" + json_u64_list(R.st.level_sizes) +
             ",\"candidates\":" + json_u64_list(R.st.candidates);
      orc::u64 nexp = 0;
      for (auto x : R.st.level_sizes) nexp += x;
      out += ",\"n_explored\":" + std::to_string(nexp);
      char buf[64];
      std::snprintf(buf, sizeof buf, "%.0f", R.st.balg);
      out += ",\"b_alg\":" + std::string(buf);
    }
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.3f", ms);
    out += ",\"ms\":" + std::string(buf) + ",\"threads\":" + std::to_string(omp_get_max_threads()) + "}";
    return dup_string(out);
  } catch (const std::exception& e) {
    return dup_string(std::string("{\"error\":\"") + e.what() + "\"}");
  }
}

// orient_dag restatement, for checking against oracle/_ref. Caller frees with oracle_free_buf.
int oracle_orient_dag(const std::uint64_t* off, const std::uint32_t* col, std::uint32_t n, std::uint64_t m,
                      std::uint64_t** out_off, std::uint32_t** out_col, std::uint64_t* out_m) {
  try {
    orc::Graph g = make_graph(off, col, nullptr, n, m, 0);
    orc::Graph h = orc::orient_dag(g);
    *out_off = (std::uint64_t*)std::malloc(sizeof(std::uint64_t) * (n + 1));
    *out_col = (std::uint32_t*)std::malloc(sizeof(std::uint32_t) * std::max<size_t>(1, h.col.size()));
    std::memcpy(*out_off, h.off.data(), sizeof(std::uint64_t) * (n + 1));
    if (!h.col.empty()) std::memcpy(*out_col, h.col.data(), sizeof(std::uint32_t) * h.col.size());
    *out_m = h.col.size();
    return 0;
  } catch (...) {
    return 1;
  }
}

void oracle_free_buf(void* p) { std::free(p); }

// SURVEY.md §8d synthetic input, restated independently of the product's
// generator so the reference arm of bench.py and the golden scripts never
// load libgpm.so: splitmix64 quadrant draws per (edge, bit), a seeded
// Fisher-Yates permutation of [0, 2^scale), self-loops dropped, then
// graph_io.hpp:83-116 cleaning (ids compacted ascending, symmetrised,
// deduplicated, ascending lists) done here by sorting packed (u, v) keys.
// Labels: uniform in [0, n_labels) per dense vertex.  Caller frees the
// three buffers with oracle_free_buf.
int oracle_generate_rmat(int scale, double ef, double a, double b, double c, std::uint64_t seed,
                         std::uint32_t n_labels, std::uint64_t label_seed, std::uint64_t** out_off,
                         std::uint32_t** out_col, std::uint32_t** out_lab, std::uint32_t* out_n,
                         std::uint64_t* out_m) {
  using orc::u32;
  using orc::u64;
  try {
    auto sm = [](u64 x) {
      x += 0x9E3779B97F4A7C15ull;
      x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
      x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
      return x ^ (x >> 31);
    };
    if (scale < 1 || scale > 31) return 1;
    const u64 N = u64(1) << scale;
    const u64 m0 = (u64)std::llround(ef * (double)N);
    std::vector<u64> perm(N);
    std::iota(perm.begin(), perm.end(), u64(0));
    u64 st = sm(seed ^ 0x5EEDC0FFEEull);
    for (u64 i = N - 1; i > 0; --i) {
      st = sm(st);
      std::swap(perm[i], perm[st % (i + 1)]);
    }
    // packed undirected pairs (both directions), self-loops dropped
    std::vector<u64> keys(2 * m0);
    std::vector<unsigned char> keep(m0);
#pragma omp parallel for schedule(static)
    for (long long ii = 0; ii < (long long)m0; ++ii) {
      u64 x = sm(seed ^ sm((u64)ii + 1)), u = 0, v = 0;
      for (int bit = 0; bit < scale; ++bit) {
        x = sm(x);
        const double r = (double)(x >> 11) * (1.0 / 9007199254740992.0);
        const int q = r < a ? 0 : r < a + b ? 1 : r < a + b + c ? 2 : 3;
        u = (u << 1) | (u64)(q >> 1);
        v = (v << 1) | (u64)(q & 1);
      }
      u = perm[u];
      v = perm[v];
      keep[ii] = u != v;
      keys[2 * ii] = (u << 32) | v;
      keys[2 * ii + 1] = (v << 32) | u;
    }
    u64 w = 0;
    for (u64 i = 0; i < m0; ++i)
      if (keep[i]) {
        keys[w++] = keys[2 * i];
        keys[w++] = keys[2 * i + 1];
      }
    keys.resize(w);
    if (keys.empty()) return 1;
    // dense ids = rank among the ids that occur (ascending)
    std::vector<unsigned char> seen(N, 0);
    for (u64 k : keys) seen[k >> 32] = 1;
    std::vector<u32> dense(N, 0);
    u32 n = 0;
    for (u64 x = 0; x < N; ++x)
      if (seen[x]) dense[x] = n++;
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < (long long)keys.size(); ++i)
      keys[i] = ((u64)dense[keys[i] >> 32] << 32) | dense[keys[i] & 0xffffffffull];
    // sort: per-thread std::sort of contiguous blocks, then pairwise merges
    {
      const int T = std::max(1, omp_get_max_threads());
      std::vector<size_t> cut(T + 1);
      for (int t = 0; t <= T; ++t) cut[t] = keys.size() * (size_t)t / (size_t)T;
#pragma omp parallel for schedule(static, 1)
      for (int t = 0; t < T; ++t) std::sort(keys.begin() + cut[t], keys.begin() + cut[t + 1]);
      for (int width = 1; width < T; width *= 2) {
#pragma omp parallel for schedule(dynamic, 1)
        for (int t = 0; t < T; t += 2 * width) {
          if (t + width >= T) continue;
          std::inplace_merge(keys.begin() + cut[t], keys.begin() + cut[t + width],
                             keys.begin() + cut[std::min(T, t + 2 * width)]);
        }
      }
    }
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    u64* off = (u64*)std::calloc(n + 1, sizeof(u64));
    u32* col = (u32*)std::malloc(sizeof(u32) * keys.size());
    u32* lab = n_labels ? (u32*)std::malloc(sizeof(u32) * std::max<u32>(1, n)) : nullptr;
    if (!off || !col || (n_labels && !lab)) return 1;
    for (size_t i = 0; i < keys.size(); ++i) {
      ++off[(keys[i] >> 32) + 1];
      col[i] = (u32)(keys[i] & 0xffffffffull);
    }
    for (u32 v = 0; v < n; ++v) off[v + 1] += off[v];
    for (u32 v = 0; n_labels && v < n; ++v) lab[v] = (u32)(sm(label_seed ^ sm((u64)v + 0x1234567ull)) % n_labels);
    *out_off = off;
    *out_col = col;
    *out_lab = lab;
    *out_n = n;
    *out_m = keys.size();
    return 0;
  } catch (...) {
    return 1;
  }
}

// canonicalize restatement exposed for tests: returns "text|p0,p1,..."
char* oracle_canonicalize(int nv, const std::uint32_t* labels, int ne, const int* edges) {
  try {
    orc::Pat q;
    q.nv = nv;
    q.lab.assign(labels, labels + nv);
    for (int i = 0; i < ne; ++i) {
      int a = edges[2 * i], b = edges[2 * i + 1];
      q.e.emplace_back(std::min(a, b), std::max(a, b));
    }
    std::sort(q.e.begin(), q.e.end());
    auto c = orc::canonicalize(q);
    std::string s = orc::pattern_text(c.pat) + "|";
    for (int i = 0; i < nv; ++i) {
      if (i) s += ",";
      s += std::to_string(c.perm[i]);
    }
    return dup_string(s);
  } catch (const std::exception& e) {
    return dup_string(std::string("error:") + e.what());
  }
}

}  // extern "C"
