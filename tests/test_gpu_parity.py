"""GPU parity: the sm_100a path through the C ABI vs the CPU oracle and the
committed golden vectors.  Bit-exact for every count, pattern, per-level size,
candidate count and B_alg."""
import json
import math
import os

import numpy as np
import pytest

import bruteforce as BF

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1911_06969_b200 as P
    return P


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(HERE, "golden", "golden.json")) as f:
        return json.load(f)["graphs"]


def host(P, oracle, E, n, labels=None):
    c = oracle.csr_from_edges(E, n, labels)
    return P.HostGraph(c.off, c.col, None if labels is None else np.asarray(labels, np.uint32))


def same(r, o, keys=("level_sizes", "candidates", "n_explored", "b_alg")):
    for k in keys:
        a, b = r.stats[k], o[k]
        if isinstance(b, list):
            a = a[:len(b)]
        assert a == b, (k, a, b)


# ----------------------------------------------------------------- golden
def test_golden_vectors(P, oracle, golden):
    for rec in golden:
        hg = host(P, oracle, [tuple(e) for e in rec["edges"]], rec["n"], rec["labels"])
        g = P.Graph(hg)
        d = g.orient_dag().download()
        assert list(d.off) == rec["ref_dag_off"] and list(d.col) == rec["ref_dag_col"], rec["name"]
        gu = P.Graph(P.HostGraph(hg.off, hg.col))
        idx, vid = gu.level1()
        assert [[int(a), int(b)] for a, b in zip(idx, vid)] == rec["ref_l1_undirected"]
        r = P.mine(g, "tc")
        assert r.total == rec["ref_tc"] and r.stats["candidates"][1] == rec["ref_tc_candidates"], rec["name"]
        for k in (3, 4, 5):
            assert P.clique_find(g, k) == rec["bf_cliques"][str(k)], (rec["name"], k)
        for k in (3, 4):
            assert P.motif_count(gu, k) == rec["bf_motifs"][str(k)], (rec["name"], k)


def test_spec_known_answers(P, oracle):
    K = lambda n: [(i, j) for i in range(n) for j in range(i + 1, n)]
    g = P.Graph(host(P, oracle, K(8), 8))
    assert [P.clique_find(g, k) for k in (3, 4, 5)] == [56, 70, 56]
    assert P.motif_count(P.Graph(host(P, oracle, K(4), 4)), 4) == {
        "k=4;L=0,0,0,0;E=(0,1)(0,2)(0,3)(1,2)(1,3)(2,3)": 1}
    for n in range(3, 11):
        gk = P.Graph(host(P, oracle, K(n), n))
        for k in (3, 4, 5):
            if k <= n:
                assert P.clique_find(gk, k) == math.comb(n, k)
    assert P.triangle_count(P.Graph(host(P, oracle, [(i, i + 1) for i in range(10)], 11))) == 0


# ----------------------------------------------------------------- random graphs vs oracle
@pytest.mark.parametrize("seed", range(8))
def test_gnp_parity(P, oracle, seed):
    n = [40, 80, 120, 200][seed % 4]
    p = [0.3, 0.12, 0.08, 0.05][seed % 4]
    hg = host(P, oracle, BF.gnp(n, p, 300 + seed), n)
    g = P.Graph(hg)
    oc = oracle.Csr(hg.off, hg.col)
    for app, k in (("tc", 3), ("cf", 3), ("cf", 4), ("cf", 5), ("mc", 3), ("mc", 4), ("mc", 5)):
        r = P.mine(g, app, k)
        o = oracle.mine(oc, app, k)
        assert r.total == o["total"], (app, k)
        if app == "mc":
            assert r.pattern_map() == {t: c for _, t, c in o["patterns"]}, (app, k)
        same(r, o)


@pytest.mark.parametrize("scale,ef", [(10, 8), (12, 8), (13, 6)])
def test_rmat_parity(P, oracle, scale, ef):
    hg = P.generate_rmat(scale, ef, 0.57, 0.19, 0.19, seed=scale)
    g = P.Graph(hg)
    oc = oracle.Csr(hg.off, hg.col)
    cases = [("tc", 3), ("cf", 4), ("cf", 5), ("mc", 3)] + ([("mc", 4)] if scale <= 12 else [])
    for app, k in cases:
        r = P.mine(g, app, k)
        o = oracle.mine(oc, app, k)
        assert r.total == o["total"], (app, k)
        if app == "mc":
            assert r.pattern_map() == {t: c for _, t, c in o["patterns"]}
        same(r, o)


def test_wedge_formula_and_tc_consistency(P):
    # SPEC.md:439 and :452-454 at a size the oracle is not needed for
    hg = P.generate_rmat(15, 16, 0.57, 0.19, 0.19, seed=7)
    g = P.Graph(hg)
    T = P.triangle_count(g)
    mc = P.motif_count(g, 3)
    deg = hg.degree()
    assert mc["k=3;L=0,0,0;E=(0,1)(0,2)(1,2)"] == T
    assert mc["k=3;L=0,0,0;E=(0,1)(0,2)"] == int((deg * (deg - 1) // 2).sum()) - 3 * T
    assert P.clique_find(g, 3) == T
    assert P.clique_find(g, 4) == P.motif_count(g, 4)["k=4;L=0,0,0,0;E=(0,1)(0,2)(0,3)(1,2)(1,3)(2,3)"]


def test_planner_chunking_invariance(P, oracle, monkeypatch):
    hg = P.generate_rmat(12, 8, 0.57, 0.19, 0.19, seed=3)
    g = P.Graph(hg)
    for app, k in (("cf", 4), ("cf", 5), ("mc", 4)):
        base = P.mine(g, app, k)
        if app == "cf":  # k-CL counts run on local rows: force the level engine to chunk
            monkeypatch.setenv("GPM_CF_NOLOCAL", "1")
        else:  # 4-MC's fused roots kernel has no materialised level to chunk
            monkeypatch.setenv("GPM_GENERIC_MC", "1")
        tiny = P.mine(g, app, k, mem_budget=1 << 16)   # forces many planner chunks
        monkeypatch.delenv("GPM_CF_NOLOCAL", raising=False)
        monkeypatch.delenv("GPM_GENERIC_MC", raising=False)
        assert tiny.stats["chunks"] > 0
        assert tiny.total == base.total and tiny.patterns == base.patterns
        same(tiny, base.stats)


def test_root_partition_sums(P):
    hg = P.generate_rmat(12, 8, 0.57, 0.19, 0.19, seed=4)
    g = P.Graph(hg)
    for app, k in (("tc", 3), ("cf", 4), ("mc", 3), ("mc", 4)):
        full = P.mine(g, app, k)
        parts = [P.mine(g, app, k, rank=r, world=3) for r in range(3)]
        assert sum(p.total for p in parts) == full.total
        assert sum(p.stats["n_explored"] for p in parts) == full.stats["n_explored"]
        if app == "mc":
            agg = {}
            for p in parts:
                for t, c in p.pattern_map().items():
                    agg[t] = agg.get(t, 0) + c
            assert agg == full.pattern_map()


def test_is_connected_and_orient(P, oracle):
    hg = host(P, oracle, BF.gnp(300, 0.05, 1), 300)
    g = P.Graph(hg)
    rng = np.random.default_rng(0)
    us = rng.integers(0, 300, 20000)
    vs = rng.integers(0, 300, 20000)
    adj = BF.adjacency(hg.off, hg.col)
    want = np.array([int(v) in adj[int(u)] for u, v in zip(us, vs)])
    assert (g.is_connected(us, vs) == want).all()
    d = g.orient_dag().download()
    o = oracle.orient_dag(oracle.Csr(hg.off, hg.col))
    assert np.array_equal(d.off, o.off) and np.array_equal(d.col, o.col)
    with pytest.raises(P.GpmError):
        P.Graph(hg).orient_dag().orient_dag()


def test_create_dag_matches_orient(P, oracle):
    for hg in (P.generate_rmat(14, 8, 0.57, 0.19, 0.19, seed=2), host(P, oracle, BF.gnp(90, 0.1, 3), 90),
               P.generate_rmat(12, 4, 0.45, 0.15, 0.15, seed=3, n_labels=5)):
        a = P.Graph(hg).orient_dag().download()
        gd = P.Graph(hg, orient=True)
        b = gd.download()
        assert gd.oriented and np.array_equal(a.off, b.off) and np.array_equal(a.col, b.col)
        assert P.triangle_count(gd) == P.triangle_count(P.Graph(hg))
    with pytest.raises(P.GpmError):
        P.Graph(P.HostGraph(np.array([0, 2, 2], np.uint64), np.array([1, 1], np.uint32)), orient=True)


def test_edge_cases(P, oracle):
    # no edges / isolated vertices / single edge
    empty = P.HostGraph(np.zeros(4, np.uint64), np.zeros(0, np.uint32))
    g = P.Graph(empty)
    assert P.triangle_count(g) == 0 and P.motif_count(g, 3) == {} and P.clique_find(g, 4) == 0
    one = P.Graph(host(P, oracle, [(0, 1)], 5))
    assert P.triangle_count(one) == 0
    assert P.mine(one, "mc", 3).stats["level_sizes"][:2] == [1, 0]
    with pytest.raises(P.GpmError):
        P.Graph(P.HostGraph(np.array([0, 2, 2], np.uint64), np.array([1, 1], np.uint32)))  # duplicate
    with pytest.raises(P.GpmError):
        P.Graph(P.HostGraph(np.array([0, 1], np.uint64), np.array([0], np.uint32)))        # self-loop
    with pytest.raises(P.GpmError):
        P.mine(P.Graph(host(P, oracle, [(0, 1)], 2)), "mc", 7)


# ----------------------------------------------------------------- FSM (edge-induced)
def test_fsm_golden(P, oracle, golden):
    for rec in golden:
        if rec["labels"] is None:
            continue
        g = P.Graph(host(P, oracle, [tuple(e) for e in rec["edges"]], rec["n"], rec["labels"]))
        for key, want in rec["bf_fsm"].items():
            k, sigma = map(int, key.split(","))
            r = P.mine(g, "fsm", k, sigma)
            assert [list(p) for p in r.patterns] == want["patterns"], (rec["name"], key)
            assert r.stats["level_sizes"][:len(want["level_sizes"])] == want["level_sizes"], (rec["name"], key)


@pytest.mark.parametrize("seed", range(6))
def test_fsm_gnp_parity(P, oracle, seed):
    rng = np.random.default_rng(700 + seed)
    n = int(rng.integers(30, 120))
    lab = rng.integers(0, [2, 3, 5][seed % 3], n)
    hg = host(P, oracle, BF.gnp(n, 0.08, 700 + seed), n, lab)
    g = P.Graph(hg)
    oc = oracle.Csr(hg.off, hg.col, hg.labels)
    for k in (2, 3, 4, 5):
        for sigma in (0, 2, 5):
            r = P.mine(g, "fsm", k, sigma)
            o = oracle.mine(oc, "fsm", k, sigma)
            assert [tuple(p) for p in r.patterns] == [tuple(p) for p in o["patterns"]], (k, sigma)
            same(r, o, ("level_sizes", "candidates", "survivors", "n_explored", "b_alg"))


@pytest.mark.parametrize("labels,sigma", [(4, 20), (8, 40), (32, 5)])
def test_fsm_rmat_parity(P, oracle, labels, sigma):
    hg = P.generate_rmat(12, 6, 0.45, 0.15, 0.15, seed=labels, n_labels=labels, label_seed=101)
    g = P.Graph(hg)
    oc = oracle.Csr(hg.off, hg.col, hg.labels)
    r = P.mine(g, "fsm", 4, sigma)
    o = oracle.mine(oc, "fsm", 4, sigma)
    assert [tuple(p) for p in r.patterns] == [tuple(p) for p in o["patterns"]]
    same(r, o, ("level_sizes", "candidates", "survivors", "n_explored", "b_alg"))


def test_fsm_errors_and_sparse_labels(P, oracle):
    g = P.Graph(host(P, oracle, [(0, 1), (1, 2)], 3))
    with pytest.raises(P.GpmError):
        P.mine(g, "fsm", 3, 1)                                   # unlabeled
    # large, sparse label values keep their identity in the pattern text
    hg = host(P, oracle, [(0, 1), (1, 2), (2, 3), (3, 0)], 4, [7, 1000000, 7, 1000000])
    r = P.mine(P.Graph(hg), "fsm", 3, 1)
    o = oracle.mine(oracle.Csr(hg.off, hg.col, hg.labels), "fsm", 3, 1)
    assert [tuple(p) for p in r.patterns] == [tuple(p) for p in o["patterns"]]


@pytest.mark.parametrize("seed", range(4))
def test_fsm_full_automorphism_mni_vs_oracle(P, oracle, seed):
    # full-automorphism MNI: GPU orbit-union domains vs the oracle
    rng = np.random.default_rng(40 + seed)
    n = int(rng.integers(40, 120))
    lab = rng.integers(0, [1, 2, 3, 2][seed], n)
    hg = host(P, oracle, BF.gnp(n, 0.08, 40 + seed), n, lab)
    g = P.Graph(hg)
    oc = oracle.Csr(hg.off, hg.col, hg.labels)
    for k in (2, 3, 4):
        for sigma in (2, 5, 9):
            r = P.mine(g, "fsm", k, sigma, mni="automorphism")
            o = oracle.mine(oc, "fsm", k, sigma, mni="automorphism")
            assert [tuple(p) for p in r.patterns] == [tuple(p) for p in o["patterns"]], (k, sigma)
            same(r, o, ("level_sizes", "candidates", "survivors", "n_explored"))


def test_fsm_full_automorphism_rmat(P, oracle):
    hg = P.generate_rmat(11, 6, 0.45, 0.15, 0.15, seed=2, n_labels=3, label_seed=5)
    g = P.Graph(hg)
    oc = oracle.Csr(hg.off, hg.col, hg.labels)
    for k, sigma in ((3, 40), (4, 80)):
        r = P.mine(g, "fsm", k, sigma, mni="automorphism")
        o = oracle.mine(oc, "fsm", k, sigma, mni="automorphism")
        assert [tuple(p) for p in r.patterns] == [tuple(p) for p in o["patterns"]]
        same(r, o, ("level_sizes", "candidates", "survivors", "n_explored"))
        # automorphisms only add mappings: every canonical-MNI frequent pattern stays frequent
        canon = {t for _, t, _ in P.mine(g, "fsm", k, sigma).patterns}
        assert canon <= {t for _, t, _ in r.patterns}
