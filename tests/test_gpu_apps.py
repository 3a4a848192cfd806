"""GPU: user-defined apps through the header-only hook engine
(include/gpm_engine.cuh).  tests/apps/test_apps.cu defines
four apps the way a reference user writes them with Pangolin's API
(toExtend / toAdd / getPattern / toPrune), compiled against
the engine header and linked to libgpm.so; each is checked against a brute
force restated from vertex SETS (tests/bruteforce.py)."""
import ctypes as C
import itertools
import os
from collections import defaultdict

import numpy as np
import pytest

import bruteforce as BF

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
APPS = {"label_clique": 0, "star": 1, "cycle": 2, "wedge_grown_motif": 3}


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1911_06969_b200 as P
    return P


@pytest.fixture(scope="module")
def testapps(P):
    path = os.path.join(HERE, "apps", "libgpm_testapps.so")
    assert os.path.exists(path), "tests/apps/libgpm_testapps.so not built (__graft_entry__.build())"
    from paper_1911_06969_b200 import _lib
    L = C.CDLL(path)
    L.testapp_mine.restype = C.c_int
    L.testapp_mine.argtypes = [C.c_int, C.c_void_p, C.POINTER(_lib.Config), C.POINTER(C.c_void_p)]

    def entry(which):
        def fn(g, cfg, out):
            return L.testapp_mine(which, g, cfg, out)
        return fn
    return {name: entry(i) for name, i in APPS.items()}


def graph(P, oracle, E, n, labels=None):
    c = oracle.csr_from_edges(E, n, labels)
    hg = P.HostGraph(c.off, c.col, None if labels is None else np.asarray(labels, np.uint32))
    return P.Graph(hg), BF.adjacency(c.off, c.col)


CASES = [(40, 0.25, 1), (60, 0.15, 2), (90, 0.08, 3)]


@pytest.mark.parametrize("n,p,seed", CASES)
@pytest.mark.parametrize("k", [3, 4, 5])
def test_label_clique_app(P, oracle, testapps, n, p, seed, k):
    rng = np.random.default_rng(seed)
    labels = rng.integers(0, 2, n).tolist()
    g, adj = graph(P, oracle, BF.gnp(n, p, seed), n, labels)
    want = 0
    for S in itertools.combinations(range(n), k):
        if len({labels[v] for v in S}) == 1 and all(b in adj[a] for a, b in itertools.combinations(S, 2)):
            want += 1
    r = P.api.mine_custom(testapps["label_clique"], g, k)
    assert r.total == want


@pytest.mark.parametrize("n,p,seed", CASES)
@pytest.mark.parametrize("k", [3, 4, 5])
def test_star_app(P, oracle, testapps, n, p, seed, k):
    g, adj = graph(P, oracle, BF.gnp(n, p, seed), n)
    want = 0
    for c in range(n):
        up = sorted(v for v in adj[c] if v > c)
        for L in itertools.combinations(up, k - 1):
            if all(b not in adj[a] for a, b in itertools.combinations(L, 2)):
                want += 1
    r = P.api.mine_custom(testapps["star"], g, k)
    assert r.total == want
    assert r.stats["level_sizes"][0] == sum(len(a) for a in adj) // 2


def _connected_sets(adj, k):
    n = len(adj)
    for S in itertools.combinations(range(n), k):
        order = BF.canonical_vertex_order(adj, S)
        if order is not None:
            yield order


@pytest.mark.parametrize("n,p,seed", CASES)
def test_cycle_app(P, oracle, testapps, n, p, seed):
    g, adj = graph(P, oracle, BF.gnp(n, p, seed), n)
    cyc = other = 0
    for order in _connected_sets(adj, 4):
        deg = [sum(1 for w in order if w != v and w in adj[v]) for v in order]
        if deg == [2, 2, 2, 2]:
            cyc += 1
        else:
            other += 1
    r = P.api.mine_custom(testapps["cycle"], g, 4)
    assert dict((t, s) for _, t, s in r.patterns) == {k_: v for k_, v in (("cycle4", cyc), ("other4", other)) if v}
    assert r.total == cyc + other


@pytest.mark.parametrize("n,p,seed", CASES)
def test_filter_app_prunes_triangle_prefixes(P, oracle, testapps, n, p, seed):
    """toPrune on an intermediate level: 4-vertex motifs whose canonical
    3-vertex prefix (SPEC.md:214 generation order) is a triangle are dropped."""
    g, adj = graph(P, oracle, BF.gnp(n, p, seed), n)
    want = defaultdict(int)
    for order in _connected_sets(adj, 4):
        a, b, c = order[:3]
        if b in adj[a] and c in adj[a] and c in adj[b]:
            continue
        edges = [(i, j) for i in range(4) for j in range(i + 1, 4) if order[j] in adj[order[i]]]
        (lab, es), _ = BF.canon(4, [0] * 4, edges)
        want[BF.text(4, lab, es)] += 1
    r = P.api.mine_custom(testapps["wedge_grown_motif"], g, 4)
    assert dict((t, s) for _, t, s in r.patterns) == dict(want)
    # the same hooks without the filter = motif counting (the builtin app)
    full = P.motif_count(g, 4)
    assert sum(full.values()) >= sum(want.values())


# ---------------------------------------------------------------- edge mode
@pytest.fixture(scope="module")
def edgeapps(P):
    path = os.path.join(HERE, "apps", "libgpm_testapps.so")
    from paper_1911_06969_b200 import _lib
    L = C.CDLL(path)
    L.testapp_mine_edges.restype = C.c_int
    L.testapp_mine_edges.argtypes = [C.c_int, C.c_void_p, C.POINTER(_lib.Config), C.POINTER(C.c_void_p)]
    return {name: (lambda i: (lambda g, cfg, out: L.testapp_mine_edges(i, g, cfg, out)))(i)
            for name, i in {"label_subset": 0, "count_support": 1}.items()}


@pytest.mark.parametrize("seed", range(3))
def test_edge_app_label_subset_equals_induced_fsm(P, oracle, edgeapps, seed):
    """toAdd(edge) + toPrune restricted to labels {0, 1} == the builtin FSM
    (the oracle) on the subgraph induced by those vertices."""
    rng = np.random.default_rng(60 + seed)
    n = 90
    lab = rng.integers(0, 4, n)
    lab[:4] = [0, 1, 2, 3]  # every label present: dense ranks == values
    E = BF.gnp(n, 0.09, 60 + seed)
    g, _ = graph(P, oracle, E, n, lab)
    keep = lab < 2
    Es = [(a, b) for a, b in E if keep[a] and keep[b]]
    sub = oracle.csr_from_edges(Es, n, lab)
    for k, sigma in ((2, 2), (3, 3), (4, 3)):
        r = P.api.mine_custom(edgeapps["label_subset"], g, k, name="fsm", min_support=sigma)
        o = oracle.mine(sub, "fsm", k, sigma)
        assert [tuple(p) for p in r.patterns] == [tuple(p) for p in o["patterns"]], (k, sigma)


@pytest.mark.parametrize("seed", range(3))
def test_edge_app_count_support_vs_bruteforce(P, oracle, edgeapps, seed):
    """toPrune on the embedding count (no domains) vs brute force over
    connected edge subsets with the same filter semantics."""
    rng = np.random.default_rng(70 + seed)
    n = int(rng.integers(14, 24))
    lab = rng.integers(0, 2, n)
    E = BF.gnp(n, 0.2, 70 + seed)
    g, adj = graph(P, oracle, E, n, lab)
    for k, sigma in ((2, 2), (3, 4), (4, 6)):
        r = P.api.mine_custom(edgeapps["count_support"], g, k, name="fsm", min_support=sigma)
        want, sizes = BF.fsm(adj, lab, k, sigma, support="count")
        assert [tuple(p) for p in r.patterns] == want, (k, sigma)
        assert r.stats["level_sizes"][:len(sizes)] == sizes
