/* gpm.h — C ABI of the B200-native extend-reduce-filter engine (libgpm.so).
 *
 * Drop-in boundary for the Pangolin hot path (arXiv 1911.06969).  Every entry
 * point names the reference interface it replaces.  Reference paths are
 * relative to /root/reference:
 *   proj/include/gpmine/graph.hpp, graph_io.hpp, embedding_list.hpp, error.hpp
 *   SPEC.md (engine / apps / cli modules; the hot path exists only as spec)
 *   PAPER.md (Alg. 1, Alg. 2, Listings 1-6)
 *
 * Conventions: plain pointers and sizes only; the caller owns input arrays
 * (copied at create time); the library owns graphs/results until *_free.
 * Exceptions never cross the ABI: every function returns a gpm_status and a
 * thread-local message is available from gpm_last_error()
 * (replaces gpmine::error / parse_error, error.hpp:10-25).
 */
#ifndef GPM_H_
#define GPM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum gpm_status {
  GPM_OK = 0,
  GPM_EINVAL = 1,   /* bad argument / out-of-range id                 */
  GPM_EPARSE = 2,   /* input text malformed (parse_error, error.hpp:16) */
  GPM_ENOMEM = 3,   /* host or device allocation failed               */
  GPM_ECUDA = 4,    /* CUDA runtime error / no device                 */
  GPM_ENCCL = 5,    /* collective exchange callback failed            */
  GPM_ECONFIG = 6   /* config conflict, e.g. chunking + filter */
} gpm_status;

typedef enum gpm_app {
  GPM_APP_TC = 0,   /* triangle_count       */
  GPM_APP_CF = 1,   /* clique_find(k)  SPEC.md:423-431, Listing 3 */
  GPM_APP_MC = 2,   /* motif_count(k)  SPEC.md:432-440, Listing 4 */
  GPM_APP_FSM = 3   /* fsm(k, sigma)   SPEC.md:441-449, Listing 5 */
} gpm_app;

typedef struct gpm_graph gpm_graph;
typedef struct gpm_result gpm_result;

/* Collective hook for multi-GPU runs (one process per GPU).  The library calls
 * it with a DEVICE buffer on `stream`; the host side performs the exchange
 * (torch.distributed / NCCL over NVLink) in place and returns 0 on success.
 *   op 0 = sum over ranks (uint64 elements)
 *   op 1 = bitwise OR over ranks (uint32 words; FSM domain bitmaps)
 *   op 2 = all-gather: buf holds world*count elements, slot `rank` filled  */
typedef int (*gpm_exchange_fn)(void* ctx, void* dev_buf, uint64_t count, int elem_bytes, int op, void* stream);

/* EngineConfig + CliConfig knobs. */
/* Listing sink ("an optional listing mode dumps final-level
 * embeddings"; PAPER.md:907-910 clique-listing).  Called on the host, in
 * order, with batches of final-level embeddings: `verts` holds n rows of k
 * vertex ids (insertion order, i.e. DAG order v0 -> v1 -> ... for TC/CF) in a
 * pinned staging buffer that is reused once the call returns.  A non-zero
 * return aborts the job with GPM_EINVAL. */
typedef int (*gpm_list_fn)(void* ctx, const uint32_t* verts, uint64_t n, int k);

typedef struct gpm_config {
  int app;                  /* gpm_app                                            */
  int k;                    /* MAX_SIZE: vertices (TC/CF/MC); edges+1 (FSM)       */
  uint64_t min_support;     /* sigma for FSM (to_prune = MNI < sigma)              */
  uint64_t mem_budget;      /* device bytes for materialised levels; 0 = auto     */
  int no_orient;            /* TC/CF: skip degree-ordered DAG orientation         */
  int rank, world;          /* root-unit partition (degree-weighted static split) */
  uint64_t root_lo, root_hi;/* explicit level-1 slice; root_hi=0 -> whole/split   */
  void* stream;             /* cudaStream_t to launch on; NULL = library stream   */
  gpm_exchange_fn exchange; /* optional collective hook (world > 1)               */
  void* exchange_ctx;
  /* Device-side work-stealing tail (world > 1, TC/CF/MC): device
   * pointer, valid on this rank's GPU, to `world` uint64 counters shared by all
   * ranks (gpm_steal_create / gpm_steal_open) and zeroed before the call
   * (gpm_steal_reset + a barrier).  Each rank mines the head of its static
   * range, then claims chunks of every rank's tail with system-scope atomics
   * on the counters (own tail first).  NULL = static split only. */
  void* steal_ctrs;
  uint64_t steal_chunk;     /* level-1 entries per stolen chunk; 0 = auto          */
  /* Listing mode (TC/CF): the final level is materialised chunk by chunk
   * (inspection-execution under the memory planner), reconstructed on the
   * device into k-vertex rows and streamed device -> pinned host through a
   * double buffer into `list_fn`.  result total = rows listed (summed over
   * ranks by the exchange when world > 1; each rank lists its own roots). */
  gpm_list_fn list_fn;      /* NULL = count only                                  */
  void* list_ctx;
  /* FSM support measure: GPM_MNI_CANONICAL (default) maps an
   * embedding's vertex i to domain perm[i] of the canonical pattern only;
   * GPM_MNI_AUTOMORPHISM also applies every automorphism of the pattern
   * ("true MNI", open question :318), i.e. each position's domain
   * is the union over its automorphism orbit. */
  int mni_mode;
} gpm_config;

enum { GPM_MNI_CANONICAL = 0, GPM_MNI_AUTOMORPHISM = 1 };

void gpm_config_default(gpm_config* cfg);

/* In-library NCCL implementation of gpm_exchange_fn (one process per GPU; no
 * Python on the exchange path).  Rank 0 calls gpm_nccl_unique_id and ships
 * the GPM_NCCL_ID_BYTES bytes to every rank by any means (MPI, file, socket,
 * torch.distributed); each rank then calls gpm_exchange_nccl_create, or
 * wraps a communicator it already owns (ncclComm_t) with
 * gpm_exchange_nccl_wrap.  Set gpm_config.exchange = gpm_exchange_nccl_fn()
 * and exchange_ctx = ctx.  Ops: 0 = ncclAllReduce(sum, u64); 1 = bitwise OR
 * of u32 words, owner-based (grouped ncclSend/ncclRecv all-to-all of 1/N
 * slices, device OR, ncclAllGather): 2(N-1)/N of the bytes per GPU;
 * 2 = in-place ncclAllGather. */
#define GPM_NCCL_ID_BYTES 128
int gpm_nccl_unique_id(void* id_out);
int gpm_exchange_nccl_create(const void* unique_id, int rank, int world, int device, void** ctx);
int gpm_exchange_nccl_wrap(void* nccl_comm, void** ctx);
gpm_exchange_fn gpm_exchange_nccl_fn(void);
int gpm_exchange_nccl_destroy(void* ctx);

/* Shared steal counters for gpm_config.steal_ctrs.  One rank creates them on
 * its device and exports a CUDA IPC handle (64 bytes) that the other ranks open
 * (peer mapping over NVLink); ranks in one process may share the pointer.
 * reset zeroes the `world` counters on `stream` (NULL = legacy stream). */
int gpm_steal_create(int device, int world, void** dev_ptr, void* ipc_handle_out);
int gpm_steal_open(int device, const void* ipc_handle, void** dev_ptr);
int gpm_steal_reset(void* dev_ptr, int world, void* stream);
int gpm_steal_release(void* dev_ptr, int opened);

/* ---------------------------------------------------------------- graph core */

/* Graph ctor (graph.hpp:29-55): validates strictly ascending lists, no
 * self-loops, ids < n; uploads CSR (u64 offsets, u32 col, optional u32 labels)
 * to `device`.  oriented != 0 marks a DAG input. */
int gpm_graph_create_csr(const uint64_t* row_offsets, const uint32_t* col, const uint32_t* labels, uint32_t n,
                         uint64_t m, int oriented, int device, gpm_graph** out);

/* Graph ctor + orient_dag fused (graph.hpp:29-55, :121-132): uploads an
 * UNDIRECTED host CSR and returns the degree-ordered DAG, overlapping the
 * chunked host->device copy with validation and orientation on the device.
 * Same result as gpm_graph_create_csr followed by gpm_graph_orient_dag. */
int gpm_graph_create_dag_csr(const uint64_t* row_offsets, const uint32_t* col, const uint32_t* labels, uint32_t n,
                             uint64_t m, int device, gpm_graph** out);

/* orient_dag (graph.hpp:121-132): keep u->v iff (deg u, u) < (deg v, v); runs
 * on the device.  Errors if already oriented. */
int gpm_graph_orient_dag(const gpm_graph* g, gpm_graph** out);

/* num_vertices / num_edges / oriented (graph.hpp:60-72). */
int gpm_graph_info(const gpm_graph* g, uint32_t* n, uint64_t* m, int* oriented, int* labeled);

/* Copy the device CSR back (for tests of orient_dag). */
int gpm_graph_download(const gpm_graph* g, uint64_t* row_offsets, uint32_t* col);

/* is_connected (graph.hpp:93-97) batched on the device: out[i] = v_i in N(u_i). */
int gpm_graph_is_connected(const gpm_graph* g, const uint32_t* us, const uint32_t* vs, uint64_t q, uint8_t* out);

/* init_single_edges (embedding_list.hpp:178-192), vertex mode: level-1 idx/vid
 * as built on the device (tests / listing). cap in entries. */
int gpm_level1(const gpm_graph* g, uint32_t* idx, uint32_t* vid, uint64_t cap, uint64_t* n_out);

void gpm_graph_free(gpm_graph* g);

/* ---------------------------------------------------------------- engine */

/* mine (Alg. 1) with the app's hooks
 * (to_extend / to_add / get_pattern / to_prune) compiled into the kernels.
 * TC/CF orient internally unless no_orient or the graph is already a DAG
 * (apps).  Blocking; one in-flight job per graph. */
int gpm_mine(const gpm_graph* g, const gpm_config* cfg, gpm_result** out);

/* TC/CF total count (AppResult.total_count). */
int gpm_result_total(const gpm_result* r, uint64_t* total);

/* PatternMap: n patterns; text in the stable form
 * "k=<n>;L=..;E=(i,j)..".  FSM patterns carry their level
 * (edges) and MNI support, ordered by (level, support desc, canonical code),
 * and their text is formatted on first access (do not read one result from
 * several threads at once); MC patterns carry counts (level = k). */
int gpm_result_num_patterns(const gpm_result* r, uint64_t* n);
int gpm_result_pattern(const gpm_result* r, uint64_t i, char* text, size_t cap, uint64_t* support, int* level);

/* Stats record: per-level sizes (|L1|, accepted per extend level),
 * candidates per extend level, FSM survivors per level, N_explored, B_alg
 * and device ms per phase. Arrays are copied up to cap. */
typedef struct gpm_stats {
  int n_levels;
  uint64_t level_sizes[16];
  uint64_t candidates[16];
  uint64_t survivors[16];
  uint64_t n_explored;
  double b_alg;
  double ms_total;          /* device time of gpm_mine (events on its stream)    */
  double ms_extend;         /* extend kernels (count/write/fused)                */
  double ms_dominant;       /* the dominant extend kernel's total time           */
  double b_dominant;        /* algorithmic bytes of the dominant kernel          */
  uint64_t launches;        /* kernels launched by this gpm_mine call            */
  uint64_t chunks;          /* planner chunks used                               */
  char dominant[64];        /* name of the dominant kernel                       */
  double b_moved_dominant;  /* bytes the dominant kernel actually reads (staged MC
                               kernels read staged sets once per root/group and
                               never stream pos-0 candidates; = b_dominant else) */
  uint64_t n_counted;       /* accepted embeddings whose class was derived from a
                               count/rank (staged MC pos-0), not a per-candidate
                               read; included in n_explored                        */
  uint32_t paths;           /* GPM_PATH_* bits: which kernel paths ran (tests)     */
} gpm_stats;

/* gpm_stats.paths bits */
enum {
  GPM_PATH_GENERIC = 1u << 0,          /* generic inspection-execution extend     */
  GPM_PATH_CF_EDGE_CHUNK = 1u << 1,    /* TC/CF first extension, edge-chunk kernel */
  GPM_PATH_CF_SIBLINGS = 1u << 2,      /* CF last level over sibling groups        */
  GPM_PATH_MC3_WARP = 1u << 3,         /* 3-MC staged, per-warp root sets          */
  GPM_PATH_MC3_BLOCK = 1u << 4,        /* 3-MC staged, per-CTA root tiles          */
  GPM_PATH_MC3_MULTITILE = 1u << 5,    /* ... a root needed more than one tile     */
  GPM_PATH_MC4_STAGED = 1u << 6,       /* 4-MC staged last level                   */
  GPM_PATH_MC4_HBM_SETS = 1u << 7,     /* ... |S0|+|S1| beyond the on-chip set     */
  GPM_PATH_PLANNER_CHUNKS = 1u << 8,   /* a level was split by the memory planner  */
  GPM_PATH_FSM_ROUNDS = 1u << 9,       /* FSM domain bitmaps in several rounds     */
  GPM_PATH_FSM_FUSED_LAST = 1u << 10,  /* FSM last level: domain pass fused        */
  GPM_PATH_FSM_GROUPED = 1u << 11,     /* FSM passes over parents grouped by code  */
  GPM_PATH_FSM_FAN = 1u << 12,         /* FSM last level: fan-out pass (dense slots) */
  GPM_PATH_FSM_SPARSE = 1u << 13,     /* FSM sparse (sorted-key) domains            */
  GPM_PATH_CF_LOCAL = 1u << 14,       /* k-CL (k >= 4) counts on per-root local rows */
  GPM_PATH_CF_LOCAL_BIG = 1u << 15    /* ... CTA-per-root kernel (out-degree > 32)   */
};
int gpm_result_stats(const gpm_result* r, gpm_stats* out);

void gpm_result_free(gpm_result* r);

/* ---------------------------------------------------------------- host input
 * Host-side loaders with the exact graph_io.hpp semantics (symmetrise, drop
 * self-loops, dedup, ids compacted ascending; gSpan labels interned).  The
 * returned arrays are malloc'd; release with gpm_csr_free. */
typedef struct gpm_csr {
  uint32_t n;
  uint64_t m;
  uint64_t* row_offsets;
  uint32_t* col;
  uint32_t* labels;        /* NULL for edge lists */
  uint64_t* original_ids;  /* dense -> input id   */
} gpm_csr;

/* load_edge_list (graph_io.hpp:83-116); *err_line set on GPM_EPARSE. */
int gpm_load_edge_list(const char* path, gpm_csr* out, uint64_t* err_line);
/* load_labeled_graph (graph_io.hpp:126-211). */
int gpm_load_labeled_graph(const char* path, gpm_csr* out, uint64_t* err_line);
/* Build a cleaned CSR from an in-memory edge list (same cleaning rules). */
int gpm_csr_from_edges(const uint64_t* src, const uint64_t* dst, uint64_t n_edges, gpm_csr* out);
/* Seeded RMAT generator: m0 = round(ef * 2^scale) edges,
 * quadrant probabilities (a,b,c,1-a-b-c), seeded vertex permutation, then
 * load_edge_list cleaning; labels uniform in [0,n_labels) when n_labels > 0. */
int gpm_generate_rmat(int scale, double edge_factor, double a, double b, double c, uint64_t seed,
                      uint32_t n_labels, uint64_t label_seed, gpm_csr* out);
void gpm_csr_free(gpm_csr* csr);

/* Binary CSR cache (replaces re-running
 * load_edge_list / load_labeled_graph, graph_io.hpp:83-211, on every run).
 * gpm_csr_save writes the cleaned CSR (+ labels, original ids) with a
 * checksum; src_path (nullable) stamps the source file's size and mtime.
 * gpm_csr_load reads it back (checksum verified).  gpm_load_cached loads
 * `path` (labeled != 0: gSpan, else edge list) through the cache at
 * cache_path (NULL: path + ".gpmcsr"): a cache whose stamp matches the source
 * is read, otherwise the text is parsed and the cache (re)written;
 * *cache_hit reports which. */
int gpm_csr_save(const char* path, const gpm_csr* csr, const char* src_path);
int gpm_csr_load(const char* path, gpm_csr* out);
int gpm_load_cached(const char* path, int labeled, const char* cache_path, gpm_csr* out, uint64_t* err_line,
                    int* cache_hit);

/* canonicalize (the paper's getIsoCanonicalBliss,
 * PAPER.md:939-954) of `count` patterns of nv <= 8 vertices on `device`, with
 * the same device canonicaliser the reduce steps use.  labels: count*nv
 * position labels (NULL = unlabeled); masks: natural pair masks, bit
 * p(i,j) = i*nv - i*(i+1)/2 + (j-i-1) set iff positions i<j are adjacent.
 * Outputs: canonical labels (nullable), canonical masks, and the
 * PositionMap perms[i*nv + q] = canonical position of quick position q
 * (nullable; first minimiser in next_permutation order). */
int gpm_canonicalize_batch(int device, int nv, uint64_t count, const uint32_t* labels, const uint32_t* masks,
                           uint32_t* canon_labels, uint32_t* canon_masks, uint8_t* perms);

/* Returns the device buffers the library keeps cached between gpm_mine calls
 * (level columns, hash tables, bitmaps >= 64 MiB) to the driver; the next
 * call re-allocates them.  For callers that share the GPU with other
 * allocators.  device < 0: every device. */
int gpm_release_cached(int device);

/* Diagnostic: best-of-`reps` read bandwidth (GB/s) of one persistent grid of
 * 16-byte loads over a `bytes` device buffer -- 64 MiB measures the L2 read
 * rate the L2-resident workloads' roofline uses (bench.py roofline.l2), a few
 * GiB the HBM read rate.  Not on the mining path. */
int gpm_probe_read_bandwidth(int device, uint64_t bytes, int reps, double* gbs);

const char* gpm_last_error(void);
const char* gpm_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GPM_H_ */
