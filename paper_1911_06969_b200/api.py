"""Host-side mirror of the reference interface, over the C ABI (libgpm.so).

Reference surface mirrored here (paths relative to /root/reference):

=====================================  ==========================================
reference                              here
=====================================  ==========================================
``load_edge_list`` graph_io.hpp:83      :func:`load_edge_list`
``load_labeled_graph`` graph_io.hpp:126 :func:`load_labeled_graph`
``Graph`` graph.hpp:22                  :class:`HostGraph` (host CSR), :class:`Graph` (device)
``orient_dag`` graph.hpp:121            :meth:`Graph.orient_dag`
``is_connected`` graph.hpp:93           :meth:`Graph.is_connected`
``init_single_edges`` emb_list.hpp:178  :meth:`Graph.level1`
``mine`` SPEC.md:371                    :func:`mine` (EngineConfig SPEC.md:337)
``triangle_count`` SPEC.md:414          :func:`triangle_count`
``clique_find`` SPEC.md:423             :func:`clique_find`
``motif_count`` SPEC.md:432             :func:`motif_count`
``fsm`` SPEC.md:441                     :func:`fsm`
``error`` / ``parse_error`` error.hpp   :class:`GpmError` / :class:`ParseError`
=====================================  ==========================================

All mining runs in the sm_100a kernels of libgpm.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np

from . import _lib as _L
from ._lib import GpmError, ParseError, check, lib

APP_IDS = {"tc": _L.APP_TC, "cf": _L.APP_CF, "mc": _L.APP_MC, "fsm": _L.APP_FSM}


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


@dataclass
class HostGraph:
    """Host CSR (graph.hpp:22-115): u64 row offsets, u32 ascending neighbour
    lists, optional u32 labels, dense -> input id map."""
    off: np.ndarray
    col: np.ndarray
    labels: Optional[np.ndarray] = None
    original_ids: Optional[np.ndarray] = None
    oriented: bool = False

    @property
    def n(self) -> int:
        return len(self.off) - 1

    @property
    def m(self) -> int:
        return len(self.col)

    def degree(self) -> np.ndarray:
        return np.diff(self.off.astype(np.int64))


def _take_csr(cs: _L.CsrStruct) -> HostGraph:
    n, m = cs.n, cs.m
    off = np.ctypeslib.as_array(C.cast(cs.row_offsets, C.POINTER(C.c_uint64)), shape=(n + 1,)).copy()
    col = (np.ctypeslib.as_array(C.cast(cs.col, C.POINTER(C.c_uint32)), shape=(m,)).copy()
           if m else np.zeros(0, np.uint32))
    lab = (np.ctypeslib.as_array(C.cast(cs.labels, C.POINTER(C.c_uint32)), shape=(n,)).copy()
           if cs.labels and n else None)
    ids = (np.ctypeslib.as_array(C.cast(cs.original_ids, C.POINTER(C.c_uint64)), shape=(n,)).copy()
           if cs.original_ids and n else None)
    lib().gpm_csr_free(C.byref(cs))
    return HostGraph(off, col, lab, ids)


def load_edge_list(path: str) -> HostGraph:
    cs, line = _L.CsrStruct(), C.c_uint64(0)
    rc = lib().gpm_load_edge_list(str(path).encode(), C.byref(cs), C.byref(line))
    check(rc, line.value)
    return _take_csr(cs)


def load_labeled_graph(path: str) -> HostGraph:
    cs, line = _L.CsrStruct(), C.c_uint64(0)
    rc = lib().gpm_load_labeled_graph(str(path).encode(), C.byref(cs), C.byref(line))
    check(rc, line.value)
    return _take_csr(cs)


def _as_csr(g: HostGraph) -> Tuple[_L.CsrStruct, list]:
    keep = [np.ascontiguousarray(g.off, dtype=np.uint64), np.ascontiguousarray(g.col, dtype=np.uint32)]
    cs = _L.CsrStruct(g.n, g.m, keep[0].ctypes.data, keep[1].ctypes.data if g.m else None, None, None)
    if g.labels is not None:
        keep.append(np.ascontiguousarray(g.labels, dtype=np.uint32))
        cs.labels = keep[-1].ctypes.data
    if g.original_ids is not None:
        keep.append(np.ascontiguousarray(g.original_ids, dtype=np.uint64))
        cs.original_ids = keep[-1].ctypes.data
    return cs, keep


def save_csr(path: str, g: HostGraph, src_path: Optional[str] = None) -> None:
    """Binary CSR cache writer (gpm_csr_save)."""
    cs, _keep = _as_csr(g)
    check(lib().gpm_csr_save(str(path).encode(), C.byref(cs), None if src_path is None else str(src_path).encode()))


def load_csr(path: str) -> HostGraph:
    """Binary CSR cache reader (gpm_csr_load; checksum verified)."""
    cs = _L.CsrStruct()
    check(lib().gpm_csr_load(str(path).encode(), C.byref(cs)))
    return _take_csr(cs)


def load_cached(path: str, labeled: bool = False, cache_path: Optional[str] = None) -> Tuple[HostGraph, bool]:
    """load_edge_list / load_labeled_graph through the binary cache
    (gpm_load_cached): returns (graph, cache_hit)."""
    cs, line, hit = _L.CsrStruct(), C.c_uint64(0), C.c_int(0)
    rc = lib().gpm_load_cached(str(path).encode(), int(labeled),
                               None if cache_path is None else str(cache_path).encode(), C.byref(cs),
                               C.byref(line), C.byref(hit))
    check(rc, line.value)
    return _take_csr(cs), bool(hit.value)


def csr_from_edges(src, dst) -> HostGraph:
    s = np.ascontiguousarray(src, dtype=np.uint64)
    d = np.ascontiguousarray(dst, dtype=np.uint64)
    cs = _L.CsrStruct()
    check(lib().gpm_csr_from_edges(_p(s), _p(d), len(s), C.byref(cs)))
    return _take_csr(cs)


def generate_rmat(scale: int, edge_factor: float, a: float, b: float, c: float, seed: int = 1,
                  n_labels: int = 0, label_seed: int = 101) -> HostGraph:
    cs = _L.CsrStruct()
    check(lib().gpm_generate_rmat(scale, edge_factor, a, b, c, seed, n_labels, label_seed, C.byref(cs)))
    return _take_csr(cs)


class Graph:
    """Immutable device CSR (one per GPU; "safe for unrestricted
    concurrent reads")."""

    def __init__(self, host: HostGraph = None, device: int = 0, *, orient: bool = False, _handle=None):
        """Uploads `host`.  orient=True returns the degree-ordered DAG directly
        (pipelined upload + orientation, == Graph(host).orient_dag())."""
        L = lib()
        if _handle is not None:
            self._h = _handle
        elif orient:
            off = np.ascontiguousarray(host.off, dtype=np.uint64)
            col = np.ascontiguousarray(host.col, dtype=np.uint32)
            lab = None if host.labels is None else np.ascontiguousarray(host.labels, dtype=np.uint32)
            h = C.c_void_p()
            check(L.gpm_graph_create_dag_csr(_p(off), _p(col), _p(lab), host.n, host.m, device, C.byref(h)))
            self._h = h
        else:
            off = np.ascontiguousarray(host.off, dtype=np.uint64)
            col = np.ascontiguousarray(host.col, dtype=np.uint32)
            lab = None if host.labels is None else np.ascontiguousarray(host.labels, dtype=np.uint32)
            h = C.c_void_p()
            check(L.gpm_graph_create_csr(_p(off), _p(col), _p(lab), host.n, host.m, int(host.oriented), device,
                                         C.byref(h)))
            self._h = h
        n, m, o, lb = C.c_uint32(), C.c_uint64(), C.c_int(), C.c_int()
        check(L.gpm_graph_info(self._h, C.byref(n), C.byref(m), C.byref(o), C.byref(lb)))
        self.n, self.m, self.oriented, self.labeled = n.value, m.value, bool(o.value), bool(lb.value)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _L._lib is not None:
            _L._lib.gpm_graph_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def orient_dag(self) -> "Graph":
        h = C.c_void_p()
        check(lib().gpm_graph_orient_dag(self._h, C.byref(h)))
        return Graph(_handle=h)

    def download(self) -> HostGraph:
        off = np.zeros(self.n + 1, np.uint64)
        col = np.zeros(max(self.m, 1), np.uint32)
        check(lib().gpm_graph_download(self._h, _p(off), _p(col)))
        return HostGraph(off, col[:self.m], oriented=self.oriented)

    def is_connected(self, us, vs) -> np.ndarray:
        u = np.ascontiguousarray(us, dtype=np.uint32).reshape(-1)
        v = np.ascontiguousarray(vs, dtype=np.uint32).reshape(-1)
        out = np.zeros(len(u), np.uint8)
        check(lib().gpm_graph_is_connected(self._h, _p(u), _p(v), len(u), _p(out)))
        return out.astype(bool)

    def level1(self) -> Tuple[np.ndarray, np.ndarray]:
        n = C.c_uint64()
        check(lib().gpm_level1(self._h, None, None, 0, C.byref(n)))
        idx = np.zeros(max(n.value, 1), np.uint32)
        vid = np.zeros(max(n.value, 1), np.uint32)
        check(lib().gpm_level1(self._h, _p(idx), _p(vid), n.value, C.byref(n)))
        return idx[:n.value], vid[:n.value]


class MineResult:
    """AppResult + engine stats.  The PatternMap is copied
    out of the library result lazily, on first access of ``patterns`` (FSM can
    return ~10^6 patterns; callers timing gpm_mine do not pay for it)."""

    def __init__(self, app: str, k: int, total: int, stats: Dict, handle, npat: int):
        self.app, self.k, self.total, self.stats = app, k, total, stats
        self._handle, self._npat, self._patterns = handle, npat, None

    @property
    def patterns(self) -> List[Tuple[int, str, int]]:  # (level, canonical text, support)
        if self._patterns is None:
            L = lib()
            pats = []
            buf = C.create_string_buffer(512)
            for i in range(self._npat):
                sup, lev = C.c_uint64(), C.c_int()
                check(L.gpm_result_pattern(self._handle, i, buf, 512, C.byref(sup), C.byref(lev)))
                pats.append((lev.value, buf.value.decode(), sup.value))
            if self.app == "fsm":
                pats.sort(key=lambda x: (x[0], -x[2], x[1]))
            self._patterns = pats
            self._release()
        return self._patterns

    def _release(self):
        if self._handle is not None:
            lib().gpm_result_free(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self._release()
        except Exception:
            pass

    def pattern_map(self) -> Dict[str, int]:
        return {t: s for _, t, s in self.patterns}

    def to_tsv(self) -> str:
        """PatternMap serialisation: `pattern<TAB>support` rows."""
        return pattern_tsv(self.patterns)

    def to_record(self) -> str:
        """AppResult as a single-line JSON record."""
        import json
        rec = {"app": self.app, "k": self.k, "total_count": self.total,
               "elapsed_s": self.stats.get("ms_total", 0.0) / 1e3,
               "n_explored": self.stats.get("n_explored", 0),
               "patterns": [[t, s] for t, s in _tsv_order(self.patterns)]}
        return json.dumps(rec, separators=(",", ":"))


def _tsv_order(patterns) -> List[Tuple[str, int]]:
    """Descending support, then pattern text.  Patterns of
    several levels (FSM) share one table; a canonical text names one level."""
    return sorted(((t, int(s)) for _, t, s in patterns), key=lambda x: (-x[1], x[0]))


def pattern_tsv(patterns) -> str:
    """`pattern<TAB>support` lines for (level, text, support) tuples, sorted by
    descending support then pattern text."""
    return "".join(f"{t}\t{s}\n" for t, s in _tsv_order(patterns))


def make_config(app: str, k: int = 3, min_support: int = 0, *, mem_budget: int = 0, no_orient: bool = False,
                rank: int = 0, world: int = 1, root_lo: int = 0, root_hi: int = 0, stream: int = 0,
                exchange=None, exchange_ctx: int = 0, steal_ctrs: int = 0, steal_chunk: int = 0,
                list_fn=None, mni: str = "canonical") -> _L.Config:
    cfg = _L.Config()
    lib().gpm_config_default(C.byref(cfg))
    cfg.app = APP_IDS[app]
    cfg.k = k
    cfg.min_support = min_support
    cfg.mem_budget = mem_budget
    cfg.no_orient = int(no_orient)
    cfg.rank, cfg.world = rank, world
    cfg.root_lo, cfg.root_hi = root_lo, root_hi
    cfg.stream = stream or None
    if exchange is not None:
        cfg.exchange = exchange
        cfg.exchange_ctx = exchange_ctx or None
    cfg.steal_ctrs = steal_ctrs or None
    cfg.steal_chunk = steal_chunk
    if list_fn is not None:
        cfg.list_fn = list_fn
    cfg.mni_mode = {"canonical": 0, "automorphism": 1}[mni]
    return cfg


def mine(g: Graph, app: str, k: int = 3, min_support: int = 0, **kw) -> MineResult:
    """mine(g, cfg): extend/reduce/filter level loop."""
    cfg = make_config(app, k, min_support, **kw)
    r = C.c_void_p()
    check(lib().gpm_mine(g.handle, C.byref(cfg), C.byref(r)))
    return _collect(r, app, k)


def mine_custom(entry, g: Graph, k: int, *, name: str = "custom", min_support: int = 0, **kw) -> MineResult:
    """Runs a user App compiled against include/gpm_engine.cuh (vertex mode,
    gpm::mine_app<App>) or include/gpm_fsm_engine.cuh (edge mode,
    gpm::mine_edge_app<App>; k = edges + 1, min_support = sigma): `entry` is
    a ctypes function with gpm_mine's signature (graph, config, result**)
    (tests/apps/test_apps.cu)."""
    cfg = make_config("tc", k, min_support, **kw)
    cfg.app = -1  # not a builtin app
    r = C.c_void_p()
    check(entry(g.handle, C.byref(cfg), C.byref(r)))
    return _collect(r, name, k)


def _collect(r, app: str, k: int) -> MineResult:
    L = lib()
    try:
        total = C.c_uint64()
        check(L.gpm_result_total(r, C.byref(total)))
        npat = C.c_uint64()
        check(L.gpm_result_num_patterns(r, C.byref(npat)))
        st = _L.Stats()
        check(L.gpm_result_stats(r, C.byref(st)))
        nl = st.n_levels
        stats = dict(level_sizes=list(st.level_sizes[:nl]), candidates=list(st.candidates[:nl]),
                     survivors=list(st.survivors[:nl]), n_explored=st.n_explored, b_alg=st.b_alg,
                     ms_total=st.ms_total, ms_extend=st.ms_extend, ms_dominant=st.ms_dominant,
                     b_dominant=st.b_dominant, launches=st.launches, chunks=st.chunks,
                     dominant=st.dominant.decode(), b_moved_dominant=st.b_moved_dominant,
                     n_counted=st.n_counted, paths=st.paths)
    except Exception:
        L.gpm_result_free(r)
        raise
    return MineResult(app, k, total.value, stats, r, npat.value)


def list_embeddings(g: Graph, app: str, k: int, **kw):
    """Listing mode (SPEC.md:458, PAPER.md:907-910 clique-listing): returns
    (rows, result) where rows is a uint32 array of shape (count, k) holding
    every final-level embedding in insertion order (DAG order for TC/CF),
    streamed from the device through gpm_config.list_fn."""
    chunks = []

    def sink(_ctx, verts, n, kk):
        try:
            if n:
                a = np.ctypeslib.as_array(verts, shape=(n * kk,))
                chunks.append(a.reshape(n, kk).copy())
            return 0
        except Exception:  # never let an exception unwind through C
            return 1

    cb = _L.LIST_FN(sink)
    res = mine(g, app, k, list_fn=cb, **kw)
    kk = res.k
    rows = np.concatenate(chunks) if chunks else np.zeros((0, kk), dtype=np.uint32)
    return rows, res


def canonicalize(patterns, nv: int, device: int = 0) -> List[Tuple[str, List[int]]]:
    """Device canonicalize of patterns given as
    (labels or None, [(i, j), ...]) over nv positions; returns the SPEC.md:252
    text and the PositionMap (quick -> canonical position) of each."""
    cnt = len(patterns)
    labeled = any(l is not None for l, _ in patterns)
    lab = np.zeros((cnt, nv), np.uint32)
    masks = np.zeros(cnt, np.uint32)
    for i, (l, edges) in enumerate(patterns):
        if l is not None:
            lab[i] = l
        for a, b in edges:
            a, b = min(a, b), max(a, b)
            masks[i] |= np.uint32(1 << (a * nv - a * (a + 1) // 2 + (b - a - 1)))
    cl = np.zeros((cnt, nv), np.uint32)
    cm = np.zeros(cnt, np.uint32)
    pm = np.zeros((cnt, nv), np.uint8)
    check(lib().gpm_canonicalize_batch(device, nv, cnt, _p(lab) if labeled else None, _p(masks), _p(cl), _p(cm),
                                       _p(pm)))
    out = []
    pairs = [(a, b) for a in range(nv) for b in range(a + 1, nv)]
    for i in range(cnt):
        e = "".join(f"({a},{b})" for p_, (a, b) in enumerate(pairs) if int(cm[i]) >> p_ & 1)
        out.append((f"k={nv};L=" + ",".join(str(int(x)) for x in cl[i]) + ";E=" + e, [int(x) for x in pm[i]]))
    return out


def probe_read_bandwidth(nbytes: int, device: int = 0, reps: int = 10) -> float:
    """Best-of-reps read GB/s over an nbytes device buffer (64 MiB: the L2
    read rate; GiBs: HBM) -- the L2 roofline denominator of bench.py."""
    v = C.c_double()
    check(lib().gpm_probe_read_bandwidth(device, nbytes, reps, C.byref(v)))
    return v.value


def release_cached(device: int = -1) -> None:
    """Hands the library's cached >= 64 MiB device buffers back to the driver
    (gpm_release_cached); device < 0: every device."""
    check(lib().gpm_release_cached(device))


def triangle_count(g: Graph, **kw) -> int:
    """SPEC.md:414-422 / PAPER.md:982-984."""
    return mine(g, "tc", 3, **kw).total


def clique_find(g: Graph, k: int, **kw) -> int:
    """SPEC.md:423-431 / Listing 3."""
    return mine(g, "cf", k, **kw).total


def motif_count(g: Graph, k: int, **kw) -> Dict[str, int]:
    """SPEC.md:432-440 / Listings 4, 6."""
    return mine(g, "mc", k, **kw).pattern_map()


def fsm(g: Graph, k: int, sigma: int, **kw) -> List[Tuple[int, str, int]]:
    """SPEC.md:441-449 / Listing 5: frequent patterns with up to k-1 edges."""
    return mine(g, "fsm", k, sigma, **kw).patterns
