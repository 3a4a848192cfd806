"""Pins the oracle's graph primitives against the reference's OWN code
(/root/reference/proj/include/gpmine compiled into oracle/_ref/libref.so by
oracle/Makefile).  Skipped where the reference build is absent."""
import numpy as np
import pytest

import bruteforce as BF

pytestmark = pytest.mark.skipif(
    not __import__("pyoracle").ref_available(), reason="oracle/_ref not built (no /root/reference)")


def test_orient_spec_examples(oracle):
    # SPEC.md:61 path 0-1-2 -> 0->1, 2->1 ; SPEC.md:62 triangle -> 0->1,0->2,1->2
    for edges, want in (([(0, 1), (1, 2)], {(0, 1), (2, 1)}), ([(0, 1), (1, 2), (2, 0)], {(0, 1), (0, 2), (1, 2)})):
        g = oracle.csr_from_edges(edges)
        for d in (oracle.orient_dag(g), oracle.ref_orient_dag(g)):
            got = {(u, int(v)) for u in range(d.n) for v in d.col[d.off[u]:d.off[u + 1]]}
            assert got == want


@pytest.mark.parametrize("seed", range(8))
def test_orient_matches_reference(oracle, seed):
    n = 200
    g = oracle.csr_from_edges(BF.gnp(n, 0.05 + 0.02 * seed, seed), n)
    a, b = oracle.orient_dag(g), oracle.ref_orient_dag(g)
    assert np.array_equal(a.off, b.off) and np.array_equal(a.col, b.col)
    assert a.m * 2 == g.m  # SPEC.md:76 orientation preserves |E|


@pytest.mark.parametrize("seed", range(6))
def test_level1_and_tc_match_reference(oracle, seed):
    n = 300
    g = oracle.csr_from_edges(BF.gnp(n, 0.06, 10 + seed), n)
    d = oracle.ref_orient_dag(g)
    idx, vid = oracle.ref_init_single_edges(d)
    r = oracle.mine(g, "tc")
    assert r["level_sizes"][0] == len(idx)
    t, c = oracle.ref_triangle_count(g)
    assert r["total"] == t and r["candidates"][1] == c
    # undirected level 1: u < v pairs
    idx2, vid2 = oracle.ref_init_single_edges(g)
    assert (idx2 < vid2).all() and len(idx2) * 2 == g.m
    assert oracle.mine(g, "mc", 3)["level_sizes"][0] == len(idx2)


def test_ref_loader_cleaning(oracle, tmp_path):
    p = tmp_path / "a.el"
    p.write_text("# c\n0 0\n0 1\r\n1 0\n\n% x\n")
    g = oracle.ref_load(str(p))
    assert g.n == 2 and g.m == 2
    p.write_text("0 1\n1 x\n")
    with pytest.raises(oracle.RefParseError) as e:
        oracle.ref_load(str(p))
    assert e.value.line == 2
