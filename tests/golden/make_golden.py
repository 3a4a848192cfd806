"""Generates tests/golden/golden.json — committed golden vectors.

Run in the build container (needs /root/reference for oracle/_ref):
    python tests/golden/make_golden.py

For each small graph it records
  * the reference's OWN outputs (oracle/_ref = reference headers):
    oriented CSR, level-1 entries, triangle count and candidate count
    composed of reference primitives (orient_dag/init_single_edges/has_edge),
  * brute-force pattern answers (tests/bruteforce.py: triangles, cliques,
    connected induced motifs, FSM with canonical-mapping MNI),
  * SPEC.md known answers.
The GPU parity tests read this file on the GPU box (where /root/reference
does not exist) and compare the CUDA path with it.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
sys.path.insert(0, os.path.join(HERE, ".."))
import bruteforce as BF  # noqa: E402
import pyoracle as P  # noqa: E402


def K(n):
    return [(i, j) for i in range(n) for j in range(i + 1, n)]


def graphs():
    yield "triangle", [(0, 1), (1, 2), (2, 0)], 3, None
    yield "path3", [(0, 1), (1, 2)], 3, None
    yield "K4", K(4), 4, None
    yield "K8", K(8), 8, None
    yield "K55", [(i, 5 + j) for i in range(5) for j in range(5)], 10, None
    yield "path11", [(i, i + 1) for i in range(10)], 11, None
    yield "disjoint5", [(2 * i, 2 * i + 1) for i in range(5)], 10, [0] * 10
    yield "star14", [(0, i) for i in range(1, 5)], 5, [0] * 5
    for s in range(4):
        n = 18 + 4 * s
        yield f"gnp{s}", BF.gnp(n, 0.25, 900 + s), n, [int(x) for x in np.random.default_rng(s).integers(0, 3, n)]


def main():
    out = []
    for name, E, n, lab in graphs():
        g = P.csr_from_edges(E, n, lab)
        adj = BF.adjacency(g.off, g.col)
        rec = {"name": name, "n": n, "edges": [list(map(int, e)) for e in E], "labels": lab}
        d = P.ref_orient_dag(g)
        rec["ref_dag_off"] = [int(x) for x in d.off]
        rec["ref_dag_col"] = [int(x) for x in d.col]
        idx, vid = P.ref_init_single_edges(g)
        rec["ref_l1_undirected"] = [[int(a), int(b)] for a, b in zip(idx, vid)]
        t, c = P.ref_triangle_count(g)
        rec["ref_tc"] = int(t)
        rec["ref_tc_candidates"] = int(c)
        rec["bf_triangles"] = BF.triangles(adj)
        rec["bf_cliques"] = {str(k): BF.cliques(adj, k) for k in (3, 4, 5)}
        rec["bf_motifs"] = {str(k): BF.motifs(adj, k) for k in (3, 4)}
        if lab is not None:
            rec["bf_fsm"] = {}
            for k in (2, 3, 4):
                for sigma in (1, 2, 3):
                    pats, sizes = BF.fsm(adj, lab, k, sigma)
                    rec["bf_fsm"][f"{k},{sigma}"] = {"patterns": [list(p) for p in pats], "level_sizes": sizes}
        assert rec["ref_tc"] == rec["bf_triangles"]
        out.append(rec)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "graphs": out}, f, indent=0, sort_keys=True)
    print("wrote", len(out), "graphs")


if __name__ == "__main__":
    main()
