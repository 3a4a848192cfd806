// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A C shim over the UNMODIFIED reference headers in
// /root/reference/proj/include/gpmine (included by path, never copied), built
// by oracle/Makefile into oracle/_ref/libref.so.  It exposes the reference's
// own loaders, CSR, orientation, level-1 init and reconstruction so tests can
// pin the oracle and the product's host code against the reference itself:
//   load_edge_list        graph_io.hpp:83-116
//   load_labeled_graph    graph_io.hpp:126-211
//   orient_dag            graph.hpp:121-132
//   init_single_edges     embedding_list.hpp:178-192
//   has_edge              graph.hpp:101-104
// plus a triangle count composed only of reference primitives (the survey's
// "reference-primitive TC") used as an extra CPU baseline.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>

#include "gpmine/embedding_list.hpp"
#include "gpmine/graph.hpp"
#include "gpmine/graph_io.hpp"

namespace {
thread_local std::string g_err;

struct RefCsr {
  std::uint32_t n;
  std::uint64_t m;
  std::uint64_t* off;
  std::uint32_t* col;
  std::uint32_t* lab;  // may be null
  std::uint64_t* orig;
};

void export_graph(const gpmine::Graph& g, RefCsr* out) {
  out->n = g.num_vertices();
  out->m = g.num_edges();
  out->off = (std::uint64_t*)std::malloc(sizeof(std::uint64_t) * (out->n + 1));
  out->col = (std::uint32_t*)std::malloc(sizeof(std::uint32_t) * (out->m ? out->m : 1));
  std::memcpy(out->off, g.row_offsets().data(), sizeof(std::uint64_t) * (out->n + 1));
  if (out->m) std::memcpy(out->col, g.column_indices().data(), sizeof(std::uint32_t) * out->m);
  out->lab = nullptr;
  if (g.labeled()) {
    out->lab = (std::uint32_t*)std::malloc(sizeof(std::uint32_t) * (out->n ? out->n : 1));
    if (out->n) std::memcpy(out->lab, g.labels().data(), sizeof(std::uint32_t) * out->n);
  }
  out->orig = (std::uint64_t*)std::malloc(sizeof(std::uint64_t) * (out->n ? out->n : 1));
  for (std::uint32_t v = 0; v < out->n; ++v) out->orig[v] = g.original_id(v);
}

gpmine::Graph import_graph(const std::uint64_t* off, const std::uint32_t* col, const std::uint32_t* lab,
                           std::uint32_t n, int oriented) {
  std::vector<std::vector<gpmine::VertexId>> adj(n);
  for (std::uint32_t v = 0; v < n; ++v) adj[v].assign(col + off[v], col + off[v + 1]);
  std::vector<std::uint32_t> labels;
  if (lab) labels.assign(lab, lab + n);
  return gpmine::Graph(std::move(adj), std::move(labels), {}, oriented != 0);
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_free(void* p) { std::free(p); }

// 0 ok, 1 error, 2 parse error (line in *err_line)
int ref_load(const char* path, int labeled, RefCsr* out, std::uint64_t* err_line) {
  try {
    std::ifstream in(path, std::ios::binary);
    if (!in) {
      g_err = "cannot open file";
      return 1;
    }
    gpmine::Graph g = labeled ? gpmine::load_labeled_graph(in) : gpmine::load_edge_list(in);
    export_graph(g, out);
    return 0;
  } catch (const gpmine::parse_error& e) {
    g_err = e.what();
    if (err_line) *err_line = e.line();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_orient_dag(const std::uint64_t* off, const std::uint32_t* col, std::uint32_t n, RefCsr* out) {
  try {
    gpmine::Graph g = import_graph(off, col, nullptr, n, 0);
    export_graph(gpmine::orient_dag(g), out);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Level-1 entries (idx = first endpoint, vid = second).  Caller frees.
int ref_init_single_edges(const std::uint64_t* off, const std::uint32_t* col, std::uint32_t n, int oriented,
                          std::uint32_t** idx, std::uint32_t** vid, std::uint64_t* count) {
  try {
    gpmine::Graph g = import_graph(off, col, nullptr, n, oriented);
    auto list = gpmine::init_single_edges(g, gpmine::Mode::vertex_induced);
    const auto& l1 = list.level(1);
    *count = l1.size();
    *idx = (std::uint32_t*)std::malloc(sizeof(std::uint32_t) * (l1.size() ? l1.size() : 1));
    *vid = (std::uint32_t*)std::malloc(sizeof(std::uint32_t) * (l1.size() ? l1.size() : 1));
    if (l1.size()) {
      std::memcpy(*idx, l1.idx.data(), sizeof(std::uint32_t) * l1.size());
      std::memcpy(*vid, l1.vid.data(), sizeof(std::uint32_t) * l1.size());
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int ref_has_edge(const std::uint64_t* off, const std::uint32_t* col, std::uint32_t n, int oriented,
                 const std::uint32_t* us, const std::uint32_t* vs, std::uint64_t q, std::uint8_t* out) {
  try {
    gpmine::Graph g = import_graph(off, col, nullptr, n, oriented);
    for (std::uint64_t i = 0; i < q; ++i) out[i] = g.is_connected(us[i], vs[i]) ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Triangle count composed of reference primitives only: orient_dag,
// init_single_edges and has_edge (SURVEY.md §6 "reference-primitive TC").
int ref_triangle_count(const std::uint64_t* off, const std::uint32_t* col, std::uint32_t n,
                       std::uint64_t* triangles, std::uint64_t* candidates) {
  try {
    gpmine::Graph g = import_graph(off, col, nullptr, n, 0);
    gpmine::Graph d = gpmine::orient_dag(g);
    auto list = gpmine::init_single_edges(d, gpmine::Mode::vertex_induced);
    const auto& l1 = list.level(1);
    std::uint64_t t = 0, c = 0;
    const long long ne = (long long)l1.size();
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : t, c)
    for (long long i = 0; i < ne; ++i) {
      auto v0 = l1.idx[i], v1 = l1.vid[i];
      for (auto u : d.neighbors(v1)) {
        ++c;
        t += d.has_edge(v0, u);
      }
    }
    *triangles = t;
    *candidates = c;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Reconstruct an edge-mode embedding through the reference's own
// EmbeddingList::reconstruct (embedding_list.hpp:73-115): levels given as
// flat arrays; returns vertices and (src_pos,dst_pos) edges.
int ref_reconstruct_edge(int nlev, const std::uint64_t* sizes, const std::uint32_t* const* idx,
                         const std::uint32_t* const* vid, const std::uint8_t* const* his, int lev,
                         std::uint64_t pos, std::uint32_t* verts, int* nverts, std::uint32_t* edges, int* nedges) {
  try {
    gpmine::EmbeddingList list(gpmine::Mode::edge_induced);
    for (int l = 0; l < nlev; ++l) {
      gpmine::Level L;
      L.idx.assign(idx[l], idx[l] + sizes[l]);
      L.vid.assign(vid[l], vid[l] + sizes[l]);
      L.his.assign(his[l], his[l] + sizes[l]);
      list.push_level(std::move(L));
    }
    list.validate();
    auto e = list.reconstruct(lev, pos);
    *nverts = (int)e.vertices.size();
    for (size_t i = 0; i < e.vertices.size(); ++i) verts[i] = e.vertices[i];
    *nedges = (int)e.edges.size();
    for (size_t i = 0; i < e.edges.size(); ++i) {
      edges[2 * i] = e.edges[i].src_pos;
      edges[2 * i + 1] = e.edges[i].dst_pos;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // extern "C"
