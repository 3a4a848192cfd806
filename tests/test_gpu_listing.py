"""Listing mode ("an optional listing mode dumps final-level
embeddings"; PAPER.md:907-910 clique-listing) through gpm_config.list_fn:
the listed rows are exactly the brute-force clique set, each row in DAG
insertion order, and the count equals the oracle's / the count-only path."""
import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1911_06969_b200 as P
    return P


def gnp(n, p, seed):
    rng = np.random.default_rng(seed)
    return [(u, v) for u in range(n) for v in range(u + 1, n) if rng.random() < p]


def brute_cliques(n, E, k):
    adj = [set() for _ in range(n)]
    for u, v in E:
        adj[u].add(v)
        adj[v].add(u)
    out = set()

    def rec(cl, cands):
        if len(cl) == k:
            out.add(tuple(cl))
            return
        for v in sorted(cands):
            if not cl or v > cl[-1]:
                rec(cl + [v], cands & adj[v])

    rec([], set(range(n)))
    return out


def dag_rank(hg):
    deg = np.diff(hg.off.astype(np.int64))
    return {v: (int(deg[v]), v) for v in range(hg.n)}


def check_rows(rows, k, expect, hg):
    assert rows.shape == (len(expect), k)
    srt = {tuple(sorted(int(x) for x in r)) for r in rows}
    assert len(srt) == len(rows), "a clique was listed twice"
    assert srt == expect
    rank = dag_rank(hg)
    for r in rows[:2000]:  # insertion order follows the degree-ordered DAG
        for i, j in itertools.combinations(range(k), 2):
            assert rank[int(r[i])] < rank[int(r[j])]


@pytest.mark.parametrize("seed", range(4))
def test_list_cliques_gnp(P, oracle, seed):
    n = 60
    E = gnp(n, 0.25, seed)
    c = oracle.csr_from_edges(E, n)
    hg = P.HostGraph(c.off, c.col)
    g = P.Graph(hg)
    for app, k in (("tc", 3), ("cf", 3), ("cf", 4), ("cf", 5)):
        rows, res = P.list_embeddings(g, app, k)
        expect = brute_cliques(n, E, k)
        check_rows(rows, k, expect, hg)
        o = oracle.mine(c, app, k)
        assert res.total == o["total"] == len(expect)
        assert res.stats["n_explored"] == o["n_explored"]
        assert res.stats["level_sizes"][:len(o["level_sizes"])] == o["level_sizes"]


def test_list_matches_count_rmat_multi_piece(P):
    # > 2^20 rows: several staging pieces through the double buffer
    hg = P.generate_rmat(15, 16, 0.57, 0.19, 0.19, seed=1)
    g = P.Graph(hg).orient_dag()
    base = P.mine(g, "tc", 3)
    assert base.total > (1 << 21)
    rows, res = P.list_embeddings(g, "tc", 3)
    assert res.total == base.total == len(rows)
    assert res.stats["n_explored"] == base.stats["n_explored"]
    key = np.sort(rows, axis=1).astype(np.uint64)
    packed = (key[:, 0] << np.uint64(42)) | (key[:, 1] << np.uint64(21)) | key[:, 2]
    assert len(np.unique(packed)) == len(rows)
    off, col = hg.off, hg.col
    # every listed triple is a triangle of the undirected graph
    sample = rows[:: max(1, len(rows) // 5000)]
    for a, b, cc in sample:
        for u, v in ((a, b), (b, cc), (a, cc)):
            nb = col[off[u]:off[u + 1]]
            i = np.searchsorted(nb, v)
            assert i < len(nb) and nb[i] == v


def test_list_chunked_and_sliced(P):
    hg = P.generate_rmat(12, 8, 0.57, 0.19, 0.19, seed=5)
    g = P.Graph(hg)
    full, res = P.list_embeddings(g, "cf", 4)
    assert res.total == P.mine(g, "cf", 4).total == len(full)
    # planner chunks (tiny budget) list the same set, possibly in another order
    tiny, rt = P.list_embeddings(g, "cf", 4, mem_budget=1 << 16)
    assert rt.stats["chunks"] > 0
    assert sorted(map(tuple, tiny)) == sorted(map(tuple, full))
    # two root slices (rank / world without exchange) partition the listing
    parts = [P.list_embeddings(g, "cf", 4, rank=r, world=2)[0] for r in range(2)]
    assert sorted(map(tuple, np.concatenate(parts))) == sorted(map(tuple, full))


def test_list_errors(P):
    hg = P.generate_rmat(9, 8, 0.57, 0.19, 0.19, seed=2)
    g = P.Graph(hg)
    with pytest.raises(P.GpmError):
        P.list_embeddings(g, "mc", 3)

    import ctypes as C
    from paper_1911_06969_b200 import _lib as L

    calls = []

    def stop(_ctx, _v, n, _k):
        calls.append(n)
        return 1

    with pytest.raises(P.GpmError):
        P.mine(g, "tc", 3, list_fn=L.LIST_FN(stop))
    assert len(calls) == 1
    # the library stays usable after an aborted listing
    assert P.mine(g, "tc", 3).total == len(P.list_embeddings(g, "tc", 3)[0])
    del C


def test_release_cached_between_calls(P):
    # the big-buffer cache is handed back to the driver and rebuilt transparently
    hg = P.generate_rmat(14, 16, 0.57, 0.19, 0.19, seed=7)
    g = P.Graph(hg)
    a = P.mine(g, "mc", 3)
    P.release_cached()
    P.release_cached(0)
    b = P.mine(g, "mc", 3)
    assert a.total == b.total and a.patterns == b.patterns
    assert a.stats["n_explored"] == b.stats["n_explored"]


def test_pattern_tsv_and_record(P, oracle):
    # PatternMap TSV and the single-line AppResult record (:463)
    import json
    hg = P.generate_rmat(11, 8, 0.45, 0.15, 0.15, seed=3, n_labels=4, label_seed=101)
    g = P.Graph(hg)
    oc = oracle.Csr(hg.off, hg.col, hg.labels)
    for app, k, sigma in (("mc", 4, 0), ("fsm", 3, 40)):
        r = P.mine(g, app, k, sigma)
        o = oracle.mine(oc, app, k, sigma)
        assert r.to_tsv() == P.pattern_tsv([tuple(x) for x in o["patterns"]])
        rec = json.loads(r.to_record())
        assert rec["app"] == app and rec["total_count"] == r.total
        assert [tuple(x) for x in rec["patterns"]] == [tuple(ln.split("\t")[:1]) + (int(ln.split("\t")[1]),)
                                                      for ln in r.to_tsv().splitlines()]
