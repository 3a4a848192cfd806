"""Input-pipeline throughput: the reference's own
load_edge_list (graph_io.hpp:83-116, compiled from /root/reference into
oracle/_ref/libref.so) vs this repo's parallel loader (gpm_load_edge_list) and
its binary CSR cache (gpm_load_cached hit), on text edge lists of the
Patent-like (PAT) and LiveJournal-sized (LJ22) configs.

    python tools/loader_bench.py [pat|lj22 ...] [--out profiles/r02/loader.json] [--skip-ref]

The text file holds every undirected edge once (u < v, original ids, fields
right-aligned in fixed-width columns), i.e. the cleaned RMAT edge set of the
config; all three loaders must return the identical CSR (checked)."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

CONFIGS = {"pat": (22, 3.35, 0.50, 0.20, 0.20), "lj22": (22, 16.0, 0.57, 0.19, 0.19)}


def write_edge_list(path, hg):
    ids = hg.original_ids.astype(np.uint64)
    deg = np.diff(hg.off.astype(np.int64))
    src = np.repeat(np.arange(hg.n, dtype=np.int64), deg)
    keep = hg.col.astype(np.int64) > src
    u, v = ids[src[keep]], ids[hg.col[keep].astype(np.int64)]
    width = max(1, len(str(int(ids.max()))))
    pw = (10 ** np.arange(width - 1, -1, -1, dtype=np.uint64))
    with open(path, "wb") as f:
        for s in range(0, len(u), 1 << 22):
            a, b = u[s:s + (1 << 22)], v[s:s + (1 << 22)]
            n = len(a)
            buf = np.full((n, 2 * width + 2), ord(" "), dtype=np.uint8)
            for j, x in enumerate((a, b)):
                d = (x[:, None] // pw) % 10
                ch = (d + ord("0")).astype(np.uint8)
                lead = np.cumsum(d != 0, axis=1) == 0
                lead[:, -1] = False
                ch[lead] = ord(" ")
                buf[:, j * (width + 1):j * (width + 1) + width] = ch
            buf[:, -1] = ord("\n")
            f.write(buf.tobytes())
    return len(u)


def timed(f, reps=1):
    best, out = None, None
    for _ in range(reps):
        t = time.perf_counter()
        out = f()
        dt = time.perf_counter() - t
        best = dt if best is None else min(best, dt)
    return best, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="*", default=["pat", "lj22"])
    ap.add_argument("--out", default=None)
    ap.add_argument("--skip-ref", action="store_true")
    ap.add_argument("--dir", default="/tmp/gpm_loader")
    args = ap.parse_args()
    import paper_1911_06969_b200 as P
    import pyoracle as O
    os.makedirs(args.dir, exist_ok=True)
    recs = {}
    for name in args.names:
        hg = P.generate_rmat(*CONFIGS[name], seed=1)
        path = os.path.join(args.dir, f"{name}.el")
        lines = write_edge_list(path, hg)
        size = os.path.getsize(path)
        cache = path + ".gpmcsr"
        if os.path.exists(cache):
            os.remove(cache)
        t_ours, g = timed(lambda: P.load_edge_list(path), 2)
        assert np.array_equal(g.off, hg.off) and np.array_equal(g.col, hg.col)
        t_miss, (gm, hit) = timed(lambda: P.load_cached(path))
        assert not hit
        t_hit, (gh, hit) = timed(lambda: P.load_cached(path), 3)
        assert hit and np.array_equal(gh.col, hg.col) and np.array_equal(gh.off, hg.off)
        rec = {"lines": lines, "text_bytes": size, "n": hg.n, "m_half_edges": hg.m,
               "threads": os.cpu_count(), "ours_text_s": round(t_ours, 3),
               "ours_text_mb_s": round(size / t_ours / 1e6, 1),
               "ours_cache_write_s": round(t_miss - t_ours, 3) if t_miss > t_ours else None,
               "ours_cache_hit_s": round(t_hit, 3), "cache_bytes": os.path.getsize(cache)}
        if not args.skip_ref and O.ref_available():
            t_ref, r = timed(lambda: O.ref_load(path))
            assert np.array_equal(r.off, hg.off) and np.array_equal(r.col, hg.col)
            rec["reference_s"] = round(t_ref, 3)
            rec["speedup_text"] = round(t_ref / t_ours, 1)
            rec["speedup_cache"] = round(t_ref / t_hit, 1)
        recs[name] = rec
        print(name, json.dumps(rec), flush=True)
        os.remove(path)
        os.remove(cache)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"what": __doc__.split("\n\n")[0], "cpu": open("/proc/cpuinfo").read().split("model name")[1]
                       .split("\n")[0].strip(" :\t"), "results": recs}, f, indent=1)


if __name__ == "__main__":
    main()
