"""Pins the CPU oracle (oracle/oracle.cpp) before it is trusted as the parity
checker: every SPEC.md known answer, brute-force oracles on random graphs, and
exactly-once enumeration.  CPU only."""
import itertools
import math

import numpy as np
import pytest

import bruteforce as BF


def K(n):
    return [(i, j) for i in range(n) for j in range(i + 1, n)]


def csr(oracle, edges, n=None, labels=None):
    return oracle.csr_from_edges(edges, n, labels)


# ----------------------------------------------------------------- known answers
def test_tc_known(oracle):
    assert oracle.mine(csr(oracle, [(0, 1), (1, 2), (2, 0)]), "tc")["total"] == 1
    assert oracle.mine(csr(oracle, K(4)), "tc")["total"] == 4
    path = [(i, i + 1) for i in range(10)]
    assert oracle.mine(csr(oracle, path), "tc")["total"] == 0


def test_cf_known(oracle):
    g = csr(oracle, K(8))
    assert [oracle.mine(g, "cf", k)["total"] for k in (3, 4, 5)] == [56, 70, 56]
    bip = [(i, 5 + j) for i in range(5) for j in range(5)]
    assert oracle.mine(csr(oracle, bip), "cf", 3)["total"] == 0
    for n in range(3, 11):
        for k in (3, 4, 5):
            if k <= n:
                assert oracle.mine(csr(oracle, K(n)), "cf", k)["total"] == math.comb(n, k)


def test_mc_known(oracle):
    r = oracle.mine(csr(oracle, K(4)), "mc", 3)
    assert dict((t, c) for _, t, c in r["patterns"]) == {"k=3;L=0,0,0;E=(0,1)(0,2)(1,2)": 4}
    r = oracle.mine(csr(oracle, K(4)), "mc", 4)
    assert [c for _, _, c in r["patterns"]] == [1]


def test_fsm_known(oracle):
    E = [(2 * i, 2 * i + 1) for i in range(5)]
    g = csr(oracle, E, labels=np.zeros(10))
    assert oracle.mine(g, "fsm", 2, 5)["patterns"] == [[1, "k=2;L=0,0;E=(0,1)", 5]]
    assert oracle.mine(g, "fsm", 2, 6)["patterns"] == []


def test_fsm_star_canonical_mapping(oracle):
    # K_{1,4}, same labels, single-edge pattern: canonical-mapping MNI = 1
    # (SURVEY §7 hard part 2 resolves SPEC.md:302; full-automorphism MNI would be 5)
    g = csr(oracle, [(0, i) for i in range(1, 5)], labels=np.zeros(5))
    assert oracle.mine(g, "fsm", 2, 1)["patterns"] == [[1, "k=2;L=0,0;E=(0,1)", 1]]


def test_fsm_star_full_automorphism(oracle):
    # the same star under full-automorphism MNI: both
    # positions of the edge pattern are one orbit -> domain = all 5 vertices
    g = csr(oracle, [(0, i) for i in range(1, 5)], labels=np.zeros(5))
    assert oracle.mine(g, "fsm", 2, 1, mni="automorphism")["patterns"] == [[1, "k=2;L=0,0;E=(0,1)", 5]]
    # Fig. 2-style chain with distinct end labels: no non-trivial automorphism, both measures agree
    g = csr(oracle, [(0, 1), (1, 2)], labels=np.array([1, 0, 2]))
    assert oracle.mine(g, "fsm", 3, 1)["patterns"] == oracle.mine(g, "fsm", 3, 1, mni="automorphism")["patterns"]


@pytest.mark.parametrize("seed", range(6))
def test_fsm_full_automorphism_bruteforce(oracle, seed):
    # the oracle's orbit-union MNI == brute force over ALL isomorphic mappings
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(10, 24))
    E = BF.gnp(n, 0.18, 900 + seed)
    lab = rng.integers(0, 2, n)
    g = csr(oracle, E, n, lab)
    adj = BF.adjacency(g.off, g.col)
    for k in (2, 3, 4):
        for sigma in (1, 3, 5):
            r = oracle.mine(g, "fsm", k, sigma, mni="automorphism")
            want, sizes = BF.fsm(adj, lab, k, sigma, full=True)
            assert [tuple(x) for x in r["patterns"]] == want, (k, sigma)
            assert r["level_sizes"] == sizes


def test_canonicalize_known(oracle):
    # wedge with centre at position 0 and at position 1 -> identical form
    t0, _ = oracle.canonicalize(3, [0, 0, 0], [(0, 1), (0, 2)])
    t1, _ = oracle.canonicalize(3, [0, 0, 0], [(0, 1), (1, 2)])
    assert t0 == t1
    # 2 connected 3-vertex and 6 connected 4-vertex unlabeled classes
    for k, expect in ((3, 2), (4, 6)):
        pairs = [(i, j) for i in range(k) for j in range(i + 1, k)]
        forms = set()
        for mask in range(1 << len(pairs)):
            es = [pairs[i] for i in range(len(pairs)) if mask >> i & 1]
            adj = [set() for _ in range(k)]
            for a, b in es:
                adj[a].add(b)
                adj[b].add(a)
            if BF.canonical_vertex_order(adj, range(k)) is None:
                continue
            forms.add(oracle.canonicalize(k, [0] * k, es)[0])
        assert len(forms) == expect


def test_canonicalize_relabel_invariance(oracle):
    # SPEC.md:510 (acceptance 6), scaled: random patterns, random relabelings
    rng = np.random.default_rng(7)
    for trial in range(150):
        nv = int(rng.integers(2, 7))
        pairs = [(i, j) for i in range(nv) for j in range(i + 1, nv)]
        es = [p for p in pairs if rng.random() < 0.5]
        lab = [int(x) for x in rng.integers(0, 3, nv)] if trial % 2 else [0] * nv
        t, perm = oracle.canonicalize(nv, lab, es)
        (bl, be), bperm = BF.canon(nv, lab, es)
        assert t == BF.text(nv, bl, be) and perm == bperm
        for _ in range(5):
            pi = rng.permutation(nv)
            lab2 = [0] * nv
            for i in range(nv):
                lab2[pi[i]] = lab[i]
            es2 = [(int(pi[a]), int(pi[b])) for a, b in es]
            assert oracle.canonicalize(nv, lab2, es2)[0] == t


# ----------------------------------------------------------------- brute force
@pytest.mark.parametrize("seed", range(12))
def test_tc_cf_bruteforce(oracle, seed):
    n = [30, 60, 100][seed % 3]
    p = [0.05, 0.1, 0.3][seed % 3]
    E = BF.gnp(n, p, seed)
    g = csr(oracle, E, n)
    adj = BF.adjacency(g.off, g.col)
    t = BF.triangles(adj)
    assert oracle.mine(g, "tc")["total"] == t
    assert oracle.mine(g, "cf", 3)["total"] == t
    if n <= 60:
        for k in (4, 5):
            assert oracle.mine(g, "cf", k)["total"] == BF.cliques(adj, k)


@pytest.mark.parametrize("seed", range(6))
def test_mc_bruteforce(oracle, seed):
    n = 24 if seed % 2 else 16
    E = BF.gnp(n, 0.2, 100 + seed)
    g = csr(oracle, E, n)
    adj = BF.adjacency(g.off, g.col)
    for k in (3, 4):
        r = oracle.mine(g, "mc", k)
        got = {t: c for _, t, c in r["patterns"]}
        assert got == BF.motifs(adj, k)
        # mass conservation
        assert sum(got.values()) == r["level_sizes"][-1]
    # wedge = sum C(d,2) - 3T
    r = {t: c for _, t, c in oracle.mine(g, "mc", 3)["patterns"]}
    deg = np.diff(g.off.astype(np.int64))
    T = BF.triangles(adj)
    assert r.get("k=3;L=0,0,0;E=(0,1)(0,2)", 0) == int((deg * (deg - 1) // 2).sum()) - 3 * T
    assert r.get("k=3;L=0,0,0;E=(0,1)(0,2)(1,2)", 0) == T


def test_mc_exactly_once_small_graphs(oracle):
    # every connected graph |V|<=8 -> each connected induced k-subgraph once
    rng = np.random.default_rng(3)
    for trial in range(40):
        n = int(rng.integers(4, 9))
        E = BF.gnp(n, 0.45, 1000 + trial)
        g = csr(oracle, E, n)
        adj = BF.adjacency(g.off, g.col)
        for k in (3, 4):
            if k > n:
                continue
            got = {t: c for _, t, c in oracle.mine(g, "mc", k)["patterns"]}
            assert got == BF.motifs(adj, k)


@pytest.mark.parametrize("seed", range(10))
def test_fsm_bruteforce(oracle, seed):
    # SPEC.md:508 (acceptance 4): n<=40, 3 labels, sigma in {2,3,5}, k in {3,4}
    rng = np.random.default_rng(500 + seed)
    n = int(rng.integers(10, 26))
    E = BF.gnp(n, 0.15, 500 + seed)
    lab = rng.integers(0, 3, n)
    g = csr(oracle, E, n, lab)
    adj = BF.adjacency(g.off, g.col)
    for k in (3, 4):
        for sigma in (2, 3, 5):
            r = oracle.mine(g, "fsm", k, sigma)
            want, sizes = BF.fsm(adj, lab, k, sigma)
            assert [tuple(x) for x in r["patterns"]] == want
            assert r["level_sizes"] == sizes


def test_fsm_exactly_once_edges(oracle):
    # sigma=0 disables pruning: level sizes = number of connected edge subsets
    rng = np.random.default_rng(11)
    for trial in range(25):
        n = int(rng.integers(3, 8))
        E = BF.gnp(n, 0.5, 2000 + trial)
        if not E:
            continue
        g = csr(oracle, E, n, np.zeros(n))
        adj = BF.adjacency(g.off, g.col)
        r = oracle.mine(g, "fsm", 4, 0)
        sizes = [sum(1 for _ in BF.connected_edge_subsets(adj, s)) for s in (1, 2, 3)]
        assert r["level_sizes"] == sizes


def test_chunk_and_thread_invariance(oracle):
    # SPEC.md:511 (acceptance 7): identical across threads and chunk sizes
    E = BF.gnp(120, 0.12, 42)
    g = csr(oracle, E, 120)
    for app, k in (("tc", 3), ("cf", 4), ("mc", 3), ("mc", 4)):
        base = oracle.mine(g, app, k, threads=1, chunk_size=0)
        for th, ch in ((2, 16), (8, 1024), (8, 1)):
            r = oracle.mine(g, app, k, threads=th, chunk_size=ch)
            for key in ("total", "patterns", "level_sizes", "candidates", "n_explored", "b_alg"):
                assert r[key] == base[key], (app, k, th, ch, key)


def test_root_partition_sums(oracle):
    # partition invariance: disjoint level-1 slices sum to the whole
    E = BF.gnp(150, 0.1, 77)
    g = csr(oracle, E, 150)
    for app, k in (("tc", 3), ("cf", 4), ("mc", 4)):
        full = oracle.mine(g, app, k)
        n1 = full["level_sizes"][0]
        cuts = [0, n1 // 3, n1 // 2, n1]
        parts = [oracle.mine(g, app, k, root_lo=a, root_hi=b) for a, b in zip(cuts, cuts[1:])]
        assert sum(p["total"] for p in parts) == full["total"]
        assert sum(p["n_explored"] for p in parts) == full["n_explored"]
        if app == "mc":
            agg = {}
            for p in parts:
                for _, t, c in p["patterns"]:
                    agg[t] = agg.get(t, 0) + c
            assert agg == {t: c for _, t, c in full["patterns"]}


def test_errors(oracle):
    g = csr(oracle, K(4))
    with pytest.raises(RuntimeError):
        oracle.mine(g, "fsm", 3, 1)          # unlabeled graph
    with pytest.raises(RuntimeError):
        oracle.mine(g, "mc", 7)              # unsupported k
    with pytest.raises(ValueError):
        oracle.canonicalize(9, [0] * 9, [])  # cap 8 vertices
