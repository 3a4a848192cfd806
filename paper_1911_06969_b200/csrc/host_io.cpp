// host_io.cpp — host input pipeline: text loaders with the exact semantics of
// the reference loaders (graph_io.hpp:83-116 load_edge_list, :126-211
// load_labeled_graph), a cleaned-CSR builder, and the seeded RMAT generator of
// SURVEY.md §8d.  Parsing is a single pass over the file image with manual
// digit scanning (no per-line istringstream, the reference's cost centre,
// SURVEY §3 stack 1); CSR construction is counting-based and OpenMP-parallel.
#include <omp.h>
#include <parallel/algorithm>
#include <sys/stat.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.hpp"

namespace gpm {
namespace {

inline bool is_space(unsigned char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

// graph_io.hpp:48-57 parse_u64: digits only, overflow rejected.
inline bool parse_u64(const char* b, const char* e, u64& out) {
  if (b == e) return false;
  u64 v = 0;
  for (const char* p = b; p != e; ++p) {
    unsigned c = (unsigned char)*p - '0';
    if (c > 9) return false;
    if (v > (UINT64_MAX - c) / 10) return false;
    v = v * 10 + c;
  }
  out = v;
  return true;
}

std::string read_file(const char* path) {
  FILE* f = std::fopen(path, "rb");
  if (!f) throw Error(GPM_EINVAL, std::string("cannot open ") + path);
  std::fseek(f, 0, SEEK_END);
  long sz = std::ftell(f);
  std::fseek(f, 0, SEEK_SET);
  std::string buf;
  // resize_and_overwrite-style: grow without the zero fill of std::string(n, '\0')
  buf.reserve(sz > 0 ? (size_t)sz : 0);
  buf.resize(sz > 0 ? (size_t)sz : 0);
  if (sz > 0 && std::fread(buf.data(), 1, (size_t)sz, f) != (size_t)sz) {
    std::fclose(f);
    throw Error(GPM_EINVAL, std::string("short read on ") + path);
  }
  std::fclose(f);
  return buf;
}

struct Tok {
  const char* b;
  const char* e;
};

// Splits one line (without '\n') into whitespace tokens (istringstream >>
// semantics); returns the number of tokens, storing up to `cap`.
inline int tokenize(const char* b, const char* e, Tok* t, int cap) {
  int n = 0;
  const char* p = b;
  while (p < e) {
    while (p < e && is_space((unsigned char)*p)) ++p;
    if (p >= e) break;
    const char* s = p;
    while (p < e && !is_space((unsigned char)*p)) ++p;
    if (n < cap) t[n] = {s, p};
    ++n;
  }
  return n;
}

// graph_io.hpp:32-41 blank / comment.
inline bool blank_line(const char* b, const char* e) {
  for (const char* p = b; p < e; ++p)
    if (!is_space((unsigned char)*p)) return false;
  return true;
}
inline bool comment_line(const char* b, const char* e) {
  const char* p = b;
  while (p < e && (*p == ' ' || *p == '\t')) ++p;
  return p < e && (*p == '#' || *p == '%');
}

template <class F>
void for_each_line(const std::string& buf, F&& f) {
  const char* p = buf.data();
  const char* end = p + buf.size();
  u64 lineno = 0;
  while (p < end) {
    const char* nl = (const char*)std::memchr(p, '\n', end - p);
    const char* le = nl ? nl : end;
    ++lineno;
    const char* ce = le;
    if (ce > p && ce[-1] == '\r') --ce;  // chomp (graph_io.hpp:27-29)
    f(p, ce, lineno);
    p = nl ? nl + 1 : end;
  }
}

// Dense ids ascending over `ids` (graph_io.hpp:57-66 compact_ids).  Returns the
// sorted unique id list; `lookup` maps id -> dense index.
struct Compactor {
  std::vector<u64> uniq;
  bool dense_range = false;
  std::vector<u32> table;  // when ids are small: id -> dense
  std::unordered_map<u64, u32> map;

  // ids = a ++ b (two halves, no concatenated copy on the dense path)
  void build2(const std::vector<u64>& a, const std::vector<u64>& b) {
    u64 mx = 0;
    const long long na = (long long)a.size(), nt = na + (long long)b.size();
#pragma omp parallel for reduction(max : mx) schedule(static)
    for (long long i = 0; i < nt; ++i) mx = std::max(mx, i < na ? a[i] : b[i - na]);
    if (nt > 0 && mx < (u64(1) << 32) && mx <= 4 * (u64)nt + 1024) {
      dense_range = true;
      std::vector<u8> seen(mx + 1, 0);
      u8* sp = seen.data();
#pragma omp parallel for schedule(static)
      for (long long i = 0; i < nt; ++i) sp[i < na ? a[i] : b[i - na]] = 1;  // benign same-value writes
      table.assign(mx + 1, UINT32_MAX);
      u32 d = 0;
      for (u64 x = 0; x <= mx; ++x)
        if (seen[x]) {
          table[x] = d++;
          uniq.push_back(x);
        }
      if (uniq.size() >= (u64(1) << 32)) throw Error(GPM_EINVAL, "too many vertices for 32-bit ids");
      return;
    }
    std::vector<u64> ids;
    ids.reserve(nt);
    ids.insert(ids.end(), a.begin(), a.end());
    ids.insert(ids.end(), b.begin(), b.end());
    build(std::move(ids));
  }
  void build(std::vector<u64> ids) {
    u64 mx = 0;
#pragma omp parallel for reduction(max : mx) schedule(static)
    for (long long i = 0; i < (long long)ids.size(); ++i) mx = std::max(mx, ids[i]);
    if (!ids.empty() && mx < (u64(1) << 32) && mx <= 4 * ids.size() + 1024) {
      dense_range = true;
      std::vector<u8> seen(mx + 1, 0);
      u8* sp = seen.data();
#pragma omp parallel for schedule(static)
      for (long long i = 0; i < (long long)ids.size(); ++i) sp[ids[i]] = 1;  // benign same-value writes
      table.assign(mx + 1, UINT32_MAX);
      u32 d = 0;
      for (u64 x = 0; x <= mx; ++x)
        if (seen[x]) {
          table[x] = d++;
          uniq.push_back(x);
        }
    } else {
      __gnu_parallel::sort(ids.begin(), ids.end());
      ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
      uniq = std::move(ids);
      map.reserve(uniq.size() * 2);
      for (size_t i = 0; i < uniq.size(); ++i) map.emplace(uniq[i], (u32)i);
    }
    if (uniq.size() >= (u64(1) << 32)) throw Error(GPM_EINVAL, "too many vertices for 32-bit ids");
  }
  u32 operator()(u64 id) const { return dense_range ? table[id] : map.at(id); }
};

// Symmetrise, sort, dedup (graph_io.hpp:68-73, :119-126).  Degrees and the
// scatter use relaxed atomics across threads; every list is sorted afterwards,
// so the result does not depend on the scatter order.
void build_csr(u32 n, const std::vector<u32>& su, const std::vector<u32>& sv, gpm_csr* out) {
  const long long ne = (long long)su.size();
  std::vector<u64> deg(n + 1, 0);
  u64* dp = deg.data();
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < ne; ++i) {
    __atomic_fetch_add(dp + su[i] + 1, 1, __ATOMIC_RELAXED);
    __atomic_fetch_add(dp + sv[i] + 1, 1, __ATOMIC_RELAXED);
  }
  for (u32 v = 0; v < n; ++v) deg[v + 1] += deg[v];
  std::vector<u32> adj(deg[n]);
  {
    std::vector<u64> pos(deg.begin(), deg.end() - 1);
    u64* pp = pos.data();
    u32* ap = adj.data();
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < ne; ++i) {
      ap[__atomic_fetch_add(pp + su[i], 1, __ATOMIC_RELAXED)] = sv[i];
      ap[__atomic_fetch_add(pp + sv[i], 1, __ATOMIC_RELAXED)] = su[i];
    }
  }
  std::vector<u64> cnt(n + 1, 0);
#pragma omp parallel for schedule(dynamic, 1024)
  for (long long vv = 0; vv < (long long)n; ++vv) {
    u32 v = (u32)vv;
    auto b = adj.begin() + deg[v], e = adj.begin() + deg[v + 1];
    std::sort(b, e);
    cnt[v + 1] = (u64)(std::unique(b, e) - b);
  }
  for (u32 v = 0; v < n; ++v) cnt[v + 1] += cnt[v];
  out->n = n;
  out->m = cnt[n];
  out->row_offsets = (u64*)std::malloc(sizeof(u64) * (n + 1));
  out->col = (u32*)std::malloc(sizeof(u32) * std::max<u64>(1, cnt[n]));
  if (!out->row_offsets || !out->col) throw Error(GPM_ENOMEM, "csr allocation failed");
  std::memcpy(out->row_offsets, cnt.data(), sizeof(u64) * (n + 1));
#pragma omp parallel for schedule(dynamic, 1024)
  for (long long vv = 0; vv < (long long)n; ++vv) {
    u32 v = (u32)vv;
    std::memcpy(out->col + cnt[v], adj.data() + deg[v], sizeof(u32) * (cnt[v + 1] - cnt[v]));
  }
}

void finish_ids(const Compactor& C, gpm_csr* out) {
  out->original_ids = (u64*)std::malloc(sizeof(u64) * std::max<size_t>(1, C.uniq.size()));
  if (!out->original_ids) throw Error(GPM_ENOMEM, "id allocation failed");
  std::memcpy(out->original_ids, C.uniq.data(), sizeof(u64) * C.uniq.size());
}

void csr_from_pairs(const std::vector<u64>& a, const std::vector<u64>& b, gpm_csr* out) {
  static const bool tr = std::getenv("GPM_IO_TRACE") != nullptr;
  double t0 = omp_get_wtime();
  auto mark = [&](const char* w) {
    if (tr) std::fprintf(stderr, "[gpm io] %-12s %.3f s\n", w, omp_get_wtime() - t0);
  };
  Compactor C;
  C.build2(a, b);
  mark("compact");
  std::vector<u32> su(a.size()), sv(a.size());
#pragma omp parallel for schedule(static)
  for (long long i = 0; i < (long long)a.size(); ++i) {
    su[i] = C(a[i]);
    sv[i] = C(b[i]);
  }
  mark("map");
  build_csr((u32)C.uniq.size(), su, sv, out);
  mark("build_csr");
  out->labels = nullptr;
  finish_ids(C, out);
}

// splitmix64 (counter-based, reproducible across thread counts)
inline u64 mix64(u64 x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

}  // namespace

// Parallel single pass over the file image: the buffer is cut into one
// range per thread at line starts, each thread parses its lines into local
// (u, v) vectors, and a parse error reports the globally FIRST bad line (its
// number = lines of the earlier ranges + its rank inside its own range), as
// the reference's sequential loop would (graph_io.hpp:88-98).
void load_edge_list(const char* path, gpm_csr* out) {
  static const bool tr = std::getenv("GPM_IO_TRACE") != nullptr;
  const double t0 = omp_get_wtime();
  auto mark = [&](const char* w) {
    if (tr) std::fprintf(stderr, "[gpm io] %-12s %.3f s\n", w, omp_get_wtime() - t0);
  };
  std::string buf = read_file(path);
  mark("read");
  const char* base = buf.data();
  const char* end = base + buf.size();
  const int T = std::max(1, std::min(omp_get_max_threads(), (int)(buf.size() >> 20) + 1));
  std::vector<const char*> cut(T + 1, end);
  cut[0] = base;
  for (int t = 1; t < T; ++t) {
    const char* p = std::max(base + buf.size() * t / T, cut[t - 1]);
    const char* nl = p < end ? (const char*)std::memchr(p, '\n', end - p) : nullptr;
    cut[t] = nl ? nl + 1 : end;
  }
  std::vector<std::vector<u64>> A(T), B(T);
  std::vector<u64> nlines(T, 0), bad(T, 0);  // bad: 1-based line inside the range (0 = none)
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int t = 0; t < T; ++t) {
    auto& a = A[t];
    auto& b = B[t];
    a.reserve((cut[t + 1] - cut[t]) / 12 + 16);
    b.reserve((cut[t + 1] - cut[t]) / 12 + 16);
    const char* p = cut[t];
    const char* e = cut[t + 1];
    u64 ln = 0;
    while (p < e) {
      const char* nl = (const char*)std::memchr(p, '\n', e - p);
      const char* le = nl ? nl : e;
      ++ln;
      const char* lb = p;
      const char* ce = le;
      if (ce > lb && ce[-1] == '\r') --ce;  // chomp (graph_io.hpp:27-29)
      p = nl ? nl + 1 : e;
      if (bad[t]) continue;  // keep counting lines only
      if (blank_line(lb, ce) || comment_line(lb, ce)) continue;
      Tok tk[3];
      const int nt = tokenize(lb, ce, tk, 3);
      u64 u, v;
      if (nt != 2 || !parse_u64(tk[0].b, tk[0].e, u) || !parse_u64(tk[1].b, tk[1].e, v)) {
        bad[t] = ln;
        continue;
      }
      if (u == v) continue;  // self-loop
      a.push_back(u);
      b.push_back(v);
    }
    nlines[t] = ln;
  }
  mark("parse");
  u64 before = 0;
  for (int t = 0; t < T; ++t) {
    if (bad[t]) {
      const u64 lineno = before + bad[t];
      throw Error(GPM_EPARSE, "line " + std::to_string(lineno) + ": expected two non-negative integers", lineno);
    }
    before += nlines[t];
  }
  std::string().swap(buf);
  u64 tot = 0;
  for (int t = 0; t < T; ++t) tot += A[t].size();
  if (tot == 0) throw Error(GPM_EINVAL, "edge list is empty after cleaning");
  std::vector<u64> a(tot), b(tot);
  std::vector<u64> at(T + 1, 0);
  for (int t = 0; t < T; ++t) at[t + 1] = at[t] + A[t].size();
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int t = 0; t < T; ++t) {
    std::memcpy(a.data() + at[t], A[t].data(), sizeof(u64) * A[t].size());
    std::memcpy(b.data() + at[t], B[t].data(), sizeof(u64) * B[t].size());
    std::vector<u64>().swap(A[t]);
    std::vector<u64>().swap(B[t]);
  }
  mark("concat");
  csr_from_pairs(a, b, out);
}

void load_labeled_graph(const char* path, gpm_csr* out) {
  std::string buf = read_file(path);
  std::vector<std::pair<u64, std::string>> decls;
  std::vector<u64> ea, eb, eline;
  std::unordered_map<u64, size_t> declared;
  for_each_line(buf, [&](const char* lb, const char* le, u64 lineno) {
    if (blank_line(lb, le) || comment_line(lb, le)) return;
    Tok t[5];
    int nt = tokenize(lb, le, t, 5);
    std::string tag(t[0].b, t[0].e);
    if (tag == "t") return;  // gSpan transaction header
    if (tag == "v") {
      u64 id;
      if (nt != 3 || !parse_u64(t[1].b, t[1].e, id))
        throw Error(GPM_EPARSE, "line " + std::to_string(lineno) + ": expected 'v <id> <label>'", lineno);
      if (!declared.emplace(id, decls.size()).second)
        throw Error(GPM_EPARSE,
                    "line " + std::to_string(lineno) + ": vertex " + std::string(t[1].b, t[1].e) + " declared twice",
                    lineno);
      decls.emplace_back(id, std::string(t[2].b, t[2].e));
    } else if (tag == "e") {
      u64 u, v;
      if ((nt != 3 && nt != 4) || !parse_u64(t[1].b, t[1].e, u) || !parse_u64(t[2].b, t[2].e, v))
        throw Error(GPM_EPARSE, "line " + std::to_string(lineno) + ": expected 'e <u> <v> [label]'", lineno);
      if (u == v) return;
      ea.push_back(u);
      eb.push_back(v);
      eline.push_back(lineno);
    } else {
      throw Error(GPM_EPARSE, "line " + std::to_string(lineno) + ": unknown line tag '" + tag + "'", lineno);
    }
  });
  for (size_t i = 0; i < ea.size(); ++i)
    for (u64 id : {ea[i], eb[i]})
      if (!declared.count(id))
        throw Error(GPM_EPARSE,
                    "line " + std::to_string(eline[i]) + ": edge references undeclared vertex " + std::to_string(id),
                    eline[i]);
  if (ea.empty()) throw Error(GPM_EINVAL, "labeled graph has no edges after cleaning");

  std::vector<u64> ids;
  ids.reserve(decls.size());
  for (auto& d : decls) ids.push_back(d.first);
  Compactor C;
  C.build(std::move(ids));
  // numeric labels keep their value; other tokens interned above them,
  // first-appearance order (graph_io.hpp:168-190)
  u64 max_numeric = 0;
  bool any_numeric = false;
  for (auto& d : decls) {
    u64 val;
    if (parse_u64(d.second.data(), d.second.data() + d.second.size(), val)) {
      if (val > 0xFFFFFFFFull) throw Error(GPM_EINVAL, "vertex label too large: " + d.second);
      max_numeric = std::max(max_numeric, val);
      any_numeric = true;
    }
  }
  std::unordered_map<std::string, u32> interned;
  u64 next_id = any_numeric ? max_numeric + 1 : 0;
  const u32 n = (u32)C.uniq.size();
  std::vector<u32> labels(n, 0);
  for (auto& d : decls) {
    u64 val;
    u32 lab;
    if (parse_u64(d.second.data(), d.second.data() + d.second.size(), val)) {
      lab = (u32)val;
    } else {
      auto it = interned.find(d.second);
      if (it == interned.end()) {
        if (next_id > 0xFFFFFFFFull) throw Error(GPM_EINVAL, "too many distinct labels");
        it = interned.emplace(d.second, (u32)next_id++).first;
      }
      lab = it->second;
    }
    labels[C(d.first)] = lab;
  }
  std::vector<u32> su(ea.size()), sv(ea.size());
  for (size_t i = 0; i < ea.size(); ++i) {
    su[i] = C(ea[i]);
    sv[i] = C(eb[i]);
  }
  build_csr(n, su, sv, out);
  out->labels = (u32*)std::malloc(sizeof(u32) * std::max<u32>(1, n));
  if (!out->labels) throw Error(GPM_ENOMEM, "label allocation failed");
  std::memcpy(out->labels, labels.data(), sizeof(u32) * n);
  finish_ids(C, out);
}

void csr_from_edges(const u64* src, const u64* dst, u64 ne, gpm_csr* out) {
  std::vector<u64> a, b;
  a.reserve(ne);
  b.reserve(ne);
  for (u64 i = 0; i < ne; ++i) {
    if (src[i] == dst[i]) continue;
    a.push_back(src[i]);
    b.push_back(dst[i]);
  }
  if (a.empty()) throw Error(GPM_EINVAL, "edge list is empty after cleaning");
  csr_from_pairs(a, b, out);
}

// SURVEY.md §8d RMAT: for each edge and each bit, pick a quadrant with
// probabilities (a, b, c, 1-a-b-c); then a seeded permutation of [0, 2^scale)
// on both endpoints; then load_edge_list cleaning (ids compacted).
void generate_rmat(int scale, double ef, double a, double b, double c, u64 seed, u32 n_labels, u64 label_seed,
                   gpm_csr* out) {
  if (scale < 1 || scale > 31) throw Error(GPM_EINVAL, "rmat scale must be in [1,31]");
  if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0)) throw Error(GPM_EINVAL, "bad rmat probabilities");
  const u64 N = u64(1) << scale;
  const u64 m0 = (u64)std::llround(ef * (double)N);
  std::vector<u64> perm(N);
  std::iota(perm.begin(), perm.end(), 0);
  u64 st = mix64(seed ^ 0x5EEDC0FFEEull);
  for (u64 i = N - 1; i > 0; --i) {
    st = mix64(st);
    u64 j = st % (i + 1);
    std::swap(perm[i], perm[j]);
  }
  const double ab = a + b, abc = a + b + c;
  std::vector<u64> su(m0), sv(m0);
#pragma omp parallel for schedule(static)
  for (long long ii = 0; ii < (long long)m0; ++ii) {
    u64 x = mix64(seed ^ mix64((u64)ii + 1));
    u64 u = 0, v = 0;
    for (int bit = 0; bit < scale; ++bit) {
      x = mix64(x);
      double r = (double)(x >> 11) * (1.0 / 9007199254740992.0);
      u64 bu, bv;
      if (r < a) { bu = 0; bv = 0; }
      else if (r < ab) { bu = 0; bv = 1; }
      else if (r < abc) { bu = 1; bv = 0; }
      else { bu = 1; bv = 1; }
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    su[ii] = perm[u];
    sv[ii] = perm[v];
  }
  // drop self-loops (load_edge_list semantics) then compact + clean
  std::vector<u64> fa, fb;
  fa.reserve(m0);
  fb.reserve(m0);
  for (u64 i = 0; i < m0; ++i)
    if (su[i] != sv[i]) {
      fa.push_back(su[i]);
      fb.push_back(sv[i]);
    }
  su.clear();
  su.shrink_to_fit();
  sv.clear();
  sv.shrink_to_fit();
  if (fa.empty()) throw Error(GPM_EINVAL, "rmat produced no edges");
  csr_from_pairs(fa, fb, out);
  if (n_labels > 0) {
    out->labels = (u32*)std::malloc(sizeof(u32) * std::max<u32>(1, out->n));
    if (!out->labels) throw Error(GPM_ENOMEM, "label allocation failed");
    for (u32 v = 0; v < out->n; ++v) out->labels[v] = (u32)(mix64(label_seed ^ mix64((u64)v + 0x1234567ull)) % n_labels);
  }
}

// ---------------------------------------------------------------------------
// Binary CSR cache: the cleaned CSR of a text input,
// written once and mapped back with a few large reads instead of re-parsing
// (the reference re-parses every run, graph_io.hpp:83-116).  Layout, little
// endian: CacheHeader, row_offsets u64[n+1], col u32[m], labels u32[n] (flag
// 1), original_ids u64[n] (flag 2).  The header records the source file's
// size and mtime so a stale cache is detected, and a checksum over the arrays.
namespace {
constexpr char kCacheMagic[8] = {'G', 'P', 'M', 'C', 'S', 'R', '0', '1'};
struct CacheHeader {
  char magic[8];
  u32 version;
  u32 flags;
  u32 n;
  u32 pad;
  u64 m;
  u64 src_size;
  u64 src_mtime_ns;
  u64 checksum;
};
static_assert(sizeof(CacheHeader) == 56, "cache header layout");

// word-parallel checksum: mix64 of each 8-byte word (position-salted), summed
u64 checksum_bytes(const void* p, size_t nbytes, u64 salt) {
  const unsigned char* b = static_cast<const unsigned char*>(p);
  const size_t nw = nbytes / 8;
  u64 s = 0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (long long i = 0; i < (long long)nw; ++i) {
    u64 w;
    std::memcpy(&w, b + 8 * i, 8);
    s += mix64(w ^ mix64(salt + (u64)i));
  }
  u64 tail = 0;
  std::memcpy(&tail, b + 8 * nw, nbytes - 8 * nw);
  return s + mix64(tail ^ salt ^ (u64)nbytes);
}

u64 csr_checksum(const gpm_csr* c) {
  u64 s = checksum_bytes(c->row_offsets, sizeof(u64) * ((u64)c->n + 1), 1);
  s += checksum_bytes(c->col, sizeof(u32) * c->m, 2);
  if (c->labels) s += checksum_bytes(c->labels, sizeof(u32) * (u64)c->n, 3);
  if (c->original_ids) s += checksum_bytes(c->original_ids, sizeof(u64) * (u64)c->n, 4);
  return s;
}

bool file_stamp(const char* path, u64& size, u64& mtime_ns) {
  struct stat st;
  if (!path || ::stat(path, &st) != 0) return false;
  size = (u64)st.st_size;
  mtime_ns = (u64)st.st_mtim.tv_sec * 1000000000ull + (u64)st.st_mtim.tv_nsec;
  return true;
}

void write_all(FILE* f, const void* p, size_t n, const char* path) {
  if (n && std::fwrite(p, 1, n, f) != n) {
    std::fclose(f);
    throw Error(GPM_EINVAL, std::string("short write on ") + path);
  }
}

template <class T>
T* read_array(FILE* f, u64 count, const char* path) {
  T* p = (T*)std::malloc(sizeof(T) * std::max<u64>(1, count));
  if (!p) throw Error(GPM_ENOMEM, "cache allocation failed");
  if (count && std::fread(p, sizeof(T), count, f) != count) {
    std::free(p);
    throw Error(GPM_EINVAL, std::string("truncated cache file ") + path);
  }
  return p;
}
}  // namespace

void csr_save(const char* path, const gpm_csr* c, const char* src_path) {
  if (!c->row_offsets || (c->m && !c->col)) throw Error(GPM_EINVAL, "csr_save: empty csr");
  CacheHeader h{};
  std::memcpy(h.magic, kCacheMagic, 8);
  h.version = 1;
  h.flags = (c->labels ? 1u : 0u) | (c->original_ids ? 2u : 0u);
  h.n = c->n;
  h.m = c->m;
  if (src_path && !file_stamp(src_path, h.src_size, h.src_mtime_ns))
    throw Error(GPM_EINVAL, std::string("cannot stat ") + src_path);
  h.checksum = csr_checksum(c);
  const std::string tmp = std::string(path) + ".tmp";
  FILE* f = std::fopen(tmp.c_str(), "wb");
  if (!f) throw Error(GPM_EINVAL, std::string("cannot create ") + tmp);
  write_all(f, &h, sizeof h, path);
  write_all(f, c->row_offsets, sizeof(u64) * ((u64)c->n + 1), path);
  write_all(f, c->col, sizeof(u32) * c->m, path);
  if (c->labels) write_all(f, c->labels, sizeof(u32) * (u64)c->n, path);
  if (c->original_ids) write_all(f, c->original_ids, sizeof(u64) * (u64)c->n, path);
  if (std::fclose(f) != 0) throw Error(GPM_EINVAL, std::string("close failed on ") + tmp);
  if (std::rename(tmp.c_str(), path) != 0) throw Error(GPM_EINVAL, std::string("cannot rename to ") + path);
}

// Returns false (and leaves `out` empty) when the cache is absent or was
// written for another version of src_path; a corrupt cache is an error.
bool csr_load(const char* path, const char* src_path, gpm_csr* out) {
  FILE* f = std::fopen(path, "rb");
  if (!f) return false;
  CacheHeader h{};
  if (std::fread(&h, sizeof h, 1, f) != 1 || std::memcmp(h.magic, kCacheMagic, 8) != 0 || h.version != 1) {
    std::fclose(f);
    throw Error(GPM_EINVAL, std::string("not a gpm CSR cache: ") + path);
  }
  if (src_path) {
    u64 sz = 0, mt = 0;
    if (!file_stamp(src_path, sz, mt) || sz != h.src_size || mt != h.src_mtime_ns) {
      std::fclose(f);
      return false;  // stale
    }
  }
  try {
    out->n = h.n;
    out->m = h.m;
    out->row_offsets = read_array<u64>(f, (u64)h.n + 1, path);
    out->col = read_array<u32>(f, h.m, path);
    if (h.flags & 1u) out->labels = read_array<u32>(f, h.n, path);
    if (h.flags & 2u) out->original_ids = read_array<u64>(f, h.n, path);
  } catch (...) {
    std::fclose(f);
    throw;
  }
  std::fclose(f);
  if (csr_checksum(out) != h.checksum) throw Error(GPM_EINVAL, std::string("cache checksum mismatch: ") + path);
  if (out->row_offsets[0] != 0 || out->row_offsets[h.n] != h.m) throw Error(GPM_EINVAL, "cache offsets inconsistent");
  return true;
}

}  // namespace gpm

extern "C" {

static void zero_csr(gpm_csr* out) { std::memset(out, 0, sizeof(*out)); }

int gpm_load_edge_list(const char* path, gpm_csr* out, uint64_t* err_line) {
  if (!path || !out) {
    gpm::set_last_error("null argument");
    return GPM_EINVAL;
  }
  zero_csr(out);
  int rc = gpm::guarded([&] { gpm::load_edge_list(path, out); }, err_line);
  if (rc != GPM_OK) gpm_csr_free(out);
  return rc;
}

int gpm_load_labeled_graph(const char* path, gpm_csr* out, uint64_t* err_line) {
  if (!path || !out) {
    gpm::set_last_error("null argument");
    return GPM_EINVAL;
  }
  zero_csr(out);
  int rc = gpm::guarded([&] { gpm::load_labeled_graph(path, out); }, err_line);
  if (rc != GPM_OK) gpm_csr_free(out);
  return rc;
}

int gpm_csr_from_edges(const uint64_t* src, const uint64_t* dst, uint64_t n_edges, gpm_csr* out) {
  if (!out || (n_edges && (!src || !dst))) {
    gpm::set_last_error("null argument");
    return GPM_EINVAL;
  }
  zero_csr(out);
  int rc = gpm::guarded([&] { gpm::csr_from_edges(src, dst, n_edges, out); });
  if (rc != GPM_OK) gpm_csr_free(out);
  return rc;
}

int gpm_generate_rmat(int scale, double edge_factor, double a, double b, double c, uint64_t seed,
                      uint32_t n_labels, uint64_t label_seed, gpm_csr* out) {
  if (!out) {
    gpm::set_last_error("null argument");
    return GPM_EINVAL;
  }
  zero_csr(out);
  int rc = gpm::guarded([&] { gpm::generate_rmat(scale, edge_factor, a, b, c, seed, n_labels, label_seed, out); });
  if (rc != GPM_OK) gpm_csr_free(out);
  return rc;
}

int gpm_csr_save(const char* path, const gpm_csr* csr, const char* src_path) {
  if (!path || !csr) {
    gpm::set_last_error("null argument");
    return GPM_EINVAL;
  }
  return gpm::guarded([&] { gpm::csr_save(path, csr, src_path); });
}

int gpm_csr_load(const char* path, gpm_csr* out) {
  if (!path || !out) {
    gpm::set_last_error("null argument");
    return GPM_EINVAL;
  }
  zero_csr(out);
  int rc = gpm::guarded([&] {
    if (!gpm::csr_load(path, nullptr, out)) throw gpm::Error(GPM_EINVAL, std::string("cannot open ") + path);
  });
  if (rc != GPM_OK) gpm_csr_free(out);
  return rc;
}

int gpm_load_cached(const char* path, int labeled, const char* cache_path, gpm_csr* out, uint64_t* err_line,
                    int* cache_hit) {
  if (!path || !out) {
    gpm::set_last_error("null argument");
    return GPM_EINVAL;
  }
  zero_csr(out);
  if (cache_hit) *cache_hit = 0;
  const std::string cp = cache_path ? std::string(cache_path) : std::string(path) + ".gpmcsr";
  int rc = gpm::guarded(
      [&] {
        bool hit = false;
        try {
          hit = gpm::csr_load(cp.c_str(), path, out);
        } catch (const gpm::Error&) {
          gpm_csr_free(out);  // unreadable cache: rebuild it from the text
          hit = false;
        }
        if (hit) {
          if (cache_hit) *cache_hit = 1;
          if (labeled && !out->labels) throw gpm::Error(GPM_EINVAL, "cache holds an unlabeled graph");
          return;
        }
        gpm_csr_free(out);
        if (labeled) gpm::load_labeled_graph(path, out);
        else gpm::load_edge_list(path, out);
        gpm::csr_save(cp.c_str(), out, path);
      },
      err_line);
  if (rc != GPM_OK) gpm_csr_free(out);
  return rc;
}

void gpm_csr_free(gpm_csr* csr) {
  if (!csr) return;
  std::free(csr->row_offsets);
  std::free(csr->col);
  std::free(csr->labels);
  std::free(csr->original_ids);
  std::memset(csr, 0, sizeof(*csr));
}

}  // extern "C"
