"""paper_1911_06969_b200 — B200-native extend-reduce-filter graph pattern
mining (Pangolin, arXiv 1911.06969): TC, k-clique, k-motif and FSM through
hand-written sm_100a kernels behind the C ABI in include/gpm.h."""
from ._lib import GpmError, ParseError, lib  # noqa: F401  (raises ImportError if libgpm.so is missing)
from .api import (Graph, HostGraph, MineResult, canonicalize, clique_find, csr_from_edges, fsm,  # noqa: F401
                  generate_rmat, list_embeddings, load_cached, load_csr, load_edge_list, load_labeled_graph, save_csr, mine, mine_custom, motif_count,
                  pattern_tsv, probe_read_bandwidth, release_cached, triangle_count)

lib()  # fail loudly at import if the CUDA library is absent
