"""Small mines over every kernel path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):
    compute-sanitizer --tool racecheck python tools/sanitize_target.py
Paths: CF edge-chunk + siblings, generic CF/MC (planner chunks), 3-MC warp +
block (multi-tile) kernels, 4-MC staged + HBM union sets, FSM grouped /
ungrouped / two-pass / fused, listing, canonicaliser, is_connected, orient."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_06969_b200 as P  # noqa: E402


def hub_graph(n, p, hubs, seed):
    rng = np.random.default_rng(seed)
    m = int(p * n * (n - 1) / 2)
    e = rng.integers(0, n, size=(m, 2))
    parts = [e]
    for v, d in hubs:
        nb = rng.choice(np.arange(v + 1, n), size=d, replace=False)
        parts.append(np.stack([np.full(d, v), nb], 1))
    e = np.concatenate(parts).astype(np.uint64)
    return P.csr_from_edges(e[:, 0], e[:, 1])


def main():
    out = []
    hg = P.generate_rmat(9, 8, 0.57, 0.19, 0.19, seed=3)
    g = P.Graph(hg)
    d = g.orient_dag()
    out.append(("tc", P.mine(d, "tc").total))
    out.append(("cf4", P.mine(d, "cf", 4).total))
    out.append(("cf5", P.mine(d, "cf", 5).total))
    out.append(("cf4_chunks", P.mine(d, "cf", 4, mem_budget=1 << 14).total))
    out.append(("mc3", len(P.mine(g, "mc", 3).patterns)))
    out.append(("mc4", len(P.mine(g, "mc", 4).patterns)))
    out.append(("mc4_chunks", len(P.mine(g, "mc", 4, mem_budget=1 << 14).patterns)))
    hb = P.Graph(hub_graph(2600, 0.002, [(0, 1500), (2, 450), (3, 300)], seed=2))
    out.append(("mc3_block", len(P.mine(hb, "mc", 3).patterns)))
    out.append(("mc4_hbm", len(P.mine(hb, "mc", 4).patterns)))
    lg = P.Graph(P.generate_rmat(9, 6, 0.45, 0.15, 0.15, seed=3, n_labels=4, label_seed=7))
    out.append(("fsm3", len(P.mine(lg, "fsm", 3, 10).patterns)))
    out.append(("fsm4", len(P.mine(lg, "fsm", 4, 20).patterns)))
    out.append(("fsm4_rounds", len(P.mine(lg, "fsm", 4, 20, mem_budget=1 << 12).patterns)))
    out.append(("list_cf4", len(P.list_embeddings(d, "cf", 4)[0])))
    out.append(("canon8", P.canonicalize([(None, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7)])], 8)[0][0]))
    out.append(("is_connected", int(g.is_connected(np.arange(50), np.arange(1, 51)).sum())))
    print(out)


if __name__ == "__main__":
    main()
