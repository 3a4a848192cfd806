"""tests/golden/make_config_goldens.py — full-size parity vectors for the five
BASELINE.json configs (TEST INFRASTRUCTURE; run in the CPU container).

    python tests/golden/make_config_goldens.py [name ...]   # default: all

Every graph comes from the oracle's own restatement of SURVEY §8d's generator
(oracle.cpp `oracle_generate_rmat`, no libgpm.so); every number comes from the
CPU oracle (oracle/liboracle.so), except the 3-MC split on the LiveJournal-sized
graph, which uses SPEC.md:439's closed form wedge = sum C(d,2) - 3T with the
oracle's triangle count T (the per-candidate oracle would take ~40 min on the
8 cores here; the identity is exact and is itself oracle-checked on smaller
graphs by tests/test_oracle.py).  FSM pattern sets are stored as a count per
level, the support sum and a sha256 over the sorted (level, text, support)
lines (~7e5 patterns at sigma 100/300 would not make a small fixture).

Writes tests/golden/configs.json incrementally (one key per config), keyed by
generator version + parameters so a generator change invalidates them.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import pyoracle as O  # noqa: E402

GEN_VERSION = "splitmix64-v1"
OUT = os.path.join(HERE, "configs.json")

# name: (app, k, sigma, rmat (scale, ef, a, b, c, seed, n_labels, label_seed))
CONFIGS = {
    "tc16": ("tc", 3, 0, (16, 16.0, 0.57, 0.19, 0.19, 1, 0, 101)),
    "pat_cf4": ("cf", 4, 0, (22, 3.35, 0.50, 0.20, 0.20, 1, 0, 101)),
    "lj22_mc3": ("mc", 3, 0, (22, 16.0, 0.57, 0.19, 0.19, 1, 0, 101)),
    "fsm17_s3000": ("fsm", 4, 3000, (17, 11.0, 0.45, 0.15, 0.15, 1, 32, 101)),
    "fsm17_s1000": ("fsm", 4, 1000, (17, 11.0, 0.45, 0.15, 0.15, 1, 32, 101)),
    "fsm17_s300": ("fsm", 4, 300, (17, 11.0, 0.45, 0.15, 0.15, 1, 32, 101)),
    "fsm17_s100": ("fsm", 4, 100, (17, 11.0, 0.45, 0.15, 0.15, 1, 32, 101)),
    "mc4_mc4": ("mc", 4, 0, (22, 8.6, 0.45, 0.15, 0.15, 1, 0, 101)),
}


def pattern_digest(patterns) -> dict:
    rows = sorted((int(l), str(t), int(s)) for l, t, s in patterns)
    h = hashlib.sha256("".join(f"{l}\t{t}\t{s}\n" for l, t, s in rows).encode()).hexdigest()
    per_level = {}
    for l, _, _ in rows:
        per_level[str(l)] = per_level.get(str(l), 0) + 1
    return {"count": len(rows), "per_level": per_level, "support_sum": sum(s for _, _, s in rows), "sha256": h}


def graph_digest(g) -> dict:
    return {"n": g.n, "m": g.m, "off_sha256": hashlib.sha256(np.ascontiguousarray(g.off).tobytes()).hexdigest(),
            "col_sha256": hashlib.sha256(np.ascontiguousarray(g.col).tobytes()).hexdigest()}


def mc3_closed_form(g, threads):
    """wedges = sum_v C(d_v, 2) - 3T; triangles T from the oracle's TC."""
    t0 = time.time()
    tc = O.mine(g, "tc", 3, 0, threads=threads)
    d = np.diff(g.off.astype(np.int64))
    T = int(tc["total"])
    wedges = int((d * (d - 1) // 2).sum()) - 3 * T
    nl1 = g.m // 2
    cand = int((d * d).sum())  # sum over u<v edges of deg(u) + deg(v)
    return {"total": T + wedges,
            "patterns": [[3, "k=3;L=0,0,0;E=(0,1)(0,2)", wedges], [3, "k=3;L=0,0,0;E=(0,1)(0,2)(1,2)", T]],
            "level_sizes": [nl1, T + wedges], "candidates": [0, cand], "n_explored": nl1 + T + wedges,
            "source": "closed form SPEC.md:439 with oracle TC (T=%d), %.1f s" % (T, time.time() - t0)}


def run(name, threads):
    app, k, sigma, rm = CONFIGS[name]
    g = O.generate_rmat(*rm)
    t0 = time.time()
    if name == "lj22_mc3":
        rec = mc3_closed_form(g, threads)
    else:
        r = O.mine(g, app, k, sigma, threads=threads)
        rec = {key: r[key] for key in ("level_sizes", "candidates", "n_explored", "b_alg") if key in r}
        if app == "fsm":
            rec["survivors"] = r["survivors"]
            rec["patterns_digest"] = pattern_digest(r["patterns"])
        else:
            rec["total"] = r["total"]
            rec["patterns"] = r["patterns"]
        rec["source"] = "oracle/liboracle.so, %d threads, %.1f s" % (threads, time.time() - t0)
    rec.update({"app": app, "k": k, "min_support": sigma, "generator": GEN_VERSION,
                "rmat": dict(zip(("scale", "edge_factor", "a", "b", "c", "seed", "n_labels", "label_seed"), rm)),
                "graph": graph_digest(g)})
    return rec


def main():
    names = sys.argv[1:] or list(CONFIGS)
    threads = int(os.environ.get("GOLDEN_THREADS", os.cpu_count() or 1))
    for name in names:
        t = time.time()
        rec = run(name, threads)
        data = {}
        if os.path.exists(OUT):
            with open(OUT) as f:
                data = json.load(f)
        data[name] = rec
        with open(OUT + ".tmp", "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
        os.replace(OUT + ".tmp", OUT)
        print(f"{name}: {time.time() - t:.1f} s", flush=True)


if __name__ == "__main__":
    main()
