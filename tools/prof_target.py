"""Runs one workload once (after one warm-up) for ncu captures:
   python tools/prof_target.py cf4|tc|mc3s|mc4s|fsms"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_06969_b200 as P
W = {
    "cf4": ("cf", 4, 0, (22, 3.35, .50, .20, .20, 1, 0)),
    "tc": ("tc", 3, 0, (16, 16, .57, .19, .19, 1, 0)),
    "mc3s": ("mc", 3, 0, (19, 16, .57, .19, .19, 1, 0)),
    "mc4s": ("mc", 4, 0, (19, 8.6, .45, .15, .15, 1, 0)),
    "fsms": ("fsm", 4, 100, (15, 11, .45, .15, .15, 1, 32)),
    "mc3": ("mc", 3, 0, (22, 16, .57, .19, .19, 1, 0)),
    "mc4": ("mc", 4, 0, (22, 8.6, .45, .15, .15, 1, 0)),
    "fsm": ("fsm", 4, 300, (17, 11, .45, .15, .15, 1, 32)),
}
app, k, sigma, (sc, ef, a, b, c, seed, nl) = W[sys.argv[1]]
hg = P.generate_rmat(sc, ef, a, b, c, seed, nl, 101)
g = P.Graph(hg)
if app in ("tc", "cf"):
    g = g.orient_dag()
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    r = P.mine(g, app, k, sigma)
print(sys.argv[1], r.total, r.stats["n_explored"], r.stats["dominant"], r.stats["ms_dominant"], r.stats["ms_total"])
