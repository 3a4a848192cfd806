"""CPU tests of the product's host side: the C ABI library loads and exports
every symbol in include/gpm.h, the loaders match the reference's own loaders
(oracle/_ref), the RMAT generator is deterministic, and device calls fail
loudly (no CPU fallback) where no GPU exists."""
import os
import re

import numpy as np
import pytest

import bruteforce as BF

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_header_symbols():
    import ctypes
    from paper_1911_06969_b200 import _lib
    hdr = open(os.path.join(ROOT, "include", "gpm.h")).read()
    declared = set(re.findall(r"\b(gpm_[a-z0-9_]+)\s*\(", hdr)) - {"gpm_exchange_fn"}
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(L, name), f"libgpm.so does not export {name}"
    assert declared <= set(_lib.EXPORTS) | {"gpm_exchange_fn"}


def test_version_and_error_model():
    import paper_1911_06969_b200 as P
    assert b"sm_100a" in P.lib().gpm_version()


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


ref_only = pytest.mark.skipif(not __import__("pyoracle").ref_available(), reason="oracle/_ref not built")


@ref_only
@pytest.mark.parametrize("seed", range(5))
def test_edge_list_loader_matches_reference(oracle, tmp_path, seed):
    import paper_1911_06969_b200 as P
    rng = np.random.default_rng(seed)
    m = 400
    ids = rng.choice(10**12, 120, replace=False) if seed % 2 else rng.integers(0, 150, 120)
    u = ids[rng.integers(0, len(ids), m)]
    v = ids[rng.integers(0, len(ids), m)]
    lines = ["# header", "% other comment", ""]
    for a, b in zip(u, v):
        lines.append(f"{a}\t{b}" if rng.random() < 0.3 else f"  {a} {b} ")
    text = "\r\n".join(lines) + "\n" if seed == 3 else "\n".join(lines)
    path = _write(tmp_path, "g.el", text)
    mine = P.load_edge_list(path)
    ref = oracle.ref_load(path)
    assert np.array_equal(mine.off, ref.off)
    assert np.array_equal(mine.col, ref.col)
    assert np.array_equal(mine.original_ids, ref.orig)


@ref_only
def test_labeled_loader_matches_reference(oracle, tmp_path):
    import paper_1911_06969_b200 as P
    text = "t # 0\nv 5 alpha\nv 1 7\nv 9 beta\nv 3 alpha\ne 5 1\ne 1 9 2\ne 9 9\ne 3 5\n"
    path = _write(tmp_path, "g.lg", text)
    mine = P.load_labeled_graph(path)
    ref = oracle.ref_load(path, labeled=True)
    assert np.array_equal(mine.off, ref.off) and np.array_equal(mine.col, ref.col)
    assert np.array_equal(mine.labels, ref.labels)
    assert np.array_equal(mine.original_ids, ref.orig)


@ref_only
@pytest.mark.parametrize("text,line", [("0 1\n1 x\n", 2), ("0 1\n\n1 2 3\n", 3), ("5\n", 1), ("0 -1\n", 1)])
def test_parse_errors_match_reference(oracle, tmp_path, text, line):
    import paper_1911_06969_b200 as P
    path = _write(tmp_path, "bad.el", text)
    with pytest.raises(P.ParseError) as e:
        P.load_edge_list(path)
    assert e.value.line == line
    with pytest.raises(oracle.RefParseError) as r:
        oracle.ref_load(path)
    assert r.value.line == line


@ref_only
def test_parallel_parse_matches_reference_and_first_error(oracle, tmp_path):
    """Files of several MiB are parsed in one range per thread: same CSR as the
    reference loader, and the FIRST bad line is reported even when a later
    range holds another one."""
    import paper_1911_06969_b200 as P
    rng = np.random.default_rng(11)
    m = 700_000
    u = rng.integers(0, 50_000, m)
    v = rng.integers(0, 50_000, m)
    lines = [f"{a} {b}" if i % 97 else f"# c {i}" for i, (a, b) in enumerate(zip(u, v))]
    lines[1234] = "  "
    text = "\n".join(lines) + "\n"
    path = _write(tmp_path, "big.el", text)
    mine = P.load_edge_list(path)
    ref = oracle.ref_load(path)
    assert np.array_equal(mine.off, ref.off) and np.array_equal(mine.col, ref.col)
    assert np.array_equal(mine.original_ids, ref.orig)
    bad = list(lines)
    bad[450_000] = "1 2 3"
    bad[650_000] = "x"
    path = _write(tmp_path, "bad.el", "\n".join(bad) + "\n")
    with pytest.raises(P.ParseError) as e:
        P.load_edge_list(path)
    assert e.value.line == 450_001
    with pytest.raises(oracle.RefParseError) as r:
        oracle.ref_load(path)
    assert r.value.line == 450_001


def test_binary_csr_cache(tmp_path):
    import paper_1911_06969_b200 as P
    src = _write(tmp_path, "g.el", "".join(f"{a} {b}\n" for a, b in BF.gnp(300, 0.05, 2)))
    cache = str(tmp_path / "g.el.gpmcsr")
    g0 = P.load_edge_list(src)
    g1, hit = P.load_cached(src)
    assert not hit and os.path.exists(cache)
    g2, hit = P.load_cached(src)
    assert hit
    for g in (g1, g2, P.load_csr(cache)):
        assert np.array_equal(g.off, g0.off) and np.array_equal(g.col, g0.col)
        assert np.array_equal(g.original_ids, g0.original_ids)
    # a changed source invalidates the cache
    with open(src, "a") as f:
        f.write("1000 1001\n")
    g3, hit = P.load_cached(src)
    assert not hit and g3.n == g0.n + 2
    assert P.load_cached(src)[1]
    # a corrupt cache is detected (direct load) and rebuilt (cached load)
    raw = bytearray(open(cache, "rb").read())
    raw[-3] ^= 0xFF
    open(cache, "wb").write(bytes(raw))
    with pytest.raises(P.GpmError):
        P.load_csr(cache)
    g4, hit = P.load_cached(src)
    assert not hit and np.array_equal(g4.col, g3.col)
    # labeled graphs keep their labels; save/load of any host graph
    lg = _write(tmp_path, "l.lg", "v 0 1\nv 1 2\nv 2 1\ne 0 1\ne 1 2\n")
    a, _ = P.load_cached(lg, labeled=True)
    b, hit = P.load_cached(lg, labeled=True)
    assert hit and list(b.labels) == [1, 2, 1] and np.array_equal(a.col, b.col)
    hg = P.generate_rmat(10, 4, 0.57, 0.19, 0.19, seed=3, n_labels=5)
    P.save_csr(str(tmp_path / "r.bin"), hg)
    r = P.load_csr(str(tmp_path / "r.bin"))
    assert np.array_equal(r.off, hg.off) and np.array_equal(r.col, hg.col) and np.array_equal(r.labels, hg.labels)
    with pytest.raises(P.GpmError):
        P.load_csr(str(tmp_path / "missing.bin"))


def test_loader_spec_examples(tmp_path):
    import paper_1911_06969_b200 as P
    g = P.load_edge_list(_write(tmp_path, "t.el", "0 1\n1 2\n2 0\n"))
    assert g.n == 3 and g.m == 6
    g = P.load_edge_list(_write(tmp_path, "c.el", "0 0\n0 1\n1 0\n"))
    assert g.n == 2 and g.m == 2
    g = P.load_labeled_graph(_write(tmp_path, "l.lg", "v 0 1\nv 1 2\ne 0 1\n"))
    assert list(g.labels) == [1, 2] and g.m == 2
    with pytest.raises(P.ParseError):
        P.load_labeled_graph(_write(tmp_path, "u.lg", "v 0 5\ne 0 1\n"))
    with pytest.raises(P.ParseError):                                  # SPEC.md:50 declared twice
        P.load_labeled_graph(_write(tmp_path, "d.lg", "v 0 5\nv 0 6\ne 0 0\n"))
    with pytest.raises(P.GpmError):                                    # empty edge set
        P.load_edge_list(_write(tmp_path, "e.el", "# nothing\n3 3\n"))


def test_csr_from_edges_matches_python_cleaning(oracle):
    import paper_1911_06969_b200 as P
    E = BF.gnp(80, 0.1, 5)
    src = np.array([a for a, b in E] + [3, 7], dtype=np.uint64)
    dst = np.array([b for a, b in E] + [3, 2], dtype=np.uint64)
    g = P.csr_from_edges(src, dst)
    # compacted ids ascending; compare on the compacted id space
    ids = np.unique(np.concatenate([src[src != dst], dst[src != dst]]))
    remap = {int(x): i for i, x in enumerate(ids)}
    e2 = [(remap[int(a)], remap[int(b)]) for a, b in zip(src, dst) if a != b]
    ref = oracle.csr_from_edges(e2, len(ids))
    assert np.array_equal(g.off, ref.off) and np.array_equal(g.col, ref.col)


def test_rmat_deterministic_and_clean():
    import paper_1911_06969_b200 as P
    a = P.generate_rmat(10, 8, 0.57, 0.19, 0.19, seed=1, n_labels=32, label_seed=101)
    b = P.generate_rmat(10, 8, 0.57, 0.19, 0.19, seed=1, n_labels=32, label_seed=101)
    c = P.generate_rmat(10, 8, 0.57, 0.19, 0.19, seed=2)
    assert np.array_equal(a.off, b.off) and np.array_equal(a.col, b.col) and np.array_equal(a.labels, b.labels)
    assert not (a.m == c.m and np.array_equal(a.col, c.col))
    assert a.labels.max() < 32
    for v in range(a.n):
        nb = a.col[a.off[v]:a.off[v + 1]]
        assert (np.diff(nb.astype(np.int64)) > 0).all() and v not in nb


def test_device_calls_fail_loudly_without_gpu():
    import torch
    import paper_1911_06969_b200 as P
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = P.generate_rmat(6, 4, 0.57, 0.19, 0.19)
    with pytest.raises(P.GpmError) as e:
        P.Graph(g)
    assert e.value.code == 4  # GPM_ECUDA: no silent CPU fallback
    with pytest.raises(P.GpmError):
        P.release_cached()


def test_ctypes_structs_match_header(tmp_path):
    """The ctypes mirror of gpm_config / gpm_stats has the C layout of
    include/gpm.h (sizes and the offsets of the trailing fields)."""
    import shutil
    import subprocess
    import ctypes as C
    from paper_1911_06969_b200 import _lib as L
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    src = tmp_path / "layout.c"
    src.write_text('#include <stddef.h>\n#include <stdio.h>\n#include "gpm.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu\\n", sizeof(gpm_config),'
                   ' offsetof(gpm_config, steal_chunk), offsetof(gpm_config, list_fn),'
                   ' offsetof(gpm_config, list_ctx), sizeof(gpm_stats));return 0;}\n')
    exe = tmp_path / "layout"
    subprocess.run([cc, "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()]
    want = [C.sizeof(L.Config), L.Config.steal_chunk.offset, L.Config.list_fn.offset, L.Config.list_ctx.offset,
            C.sizeof(L.Stats)]
    assert got == want


def test_pattern_tsv_order(oracle):
    """descending support, then pattern text; one row per pattern."""
    import paper_1911_06969_b200 as P
    g = oracle.csr_from_edges([(0, 1), (1, 2), (2, 0), (2, 3), (3, 4)], 5)
    o = oracle.mine(g, "mc", 3)
    tsv = P.pattern_tsv([tuple(x) for x in o["patterns"]])
    rows = [ln.split("\t") for ln in tsv.splitlines()]
    assert len(rows) == len(o["patterns"])
    keys = [(-int(s), t) for t, s in rows]
    assert keys == sorted(keys)
    assert sum(int(s) for _, s in rows) == o["total"]


@pytest.mark.parametrize("args", [(11, 8.0, 0.57, 0.19, 0.19, 1, 0, 101), (13, 11.0, 0.45, 0.15, 0.15, 1, 32, 101),
                                  (12, 3.35, 0.50, 0.20, 0.20, 7, 4, 5)])
def test_oracle_generator_restatement_matches_product(oracle, args):
    """The oracle's own SURVEY §8d generator (used by the reference arm, the
    CPU baseline and the golden scripts, never libgpm.so) produces the same
    cleaned CSR and labels as gpm_generate_rmat."""
    import paper_1911_06969_b200 as P
    a = oracle.generate_rmat(*args)
    b = P.generate_rmat(*args)
    assert np.array_equal(a.off, b.off) and np.array_equal(a.col, b.col)
    if args[6]:
        assert np.array_equal(a.labels, b.labels)
    else:
        assert a.labels is None and b.labels is None


def test_reference_arm_never_loads_the_product(tmp_path):
    """bench.py --impl reference runs the CPU port only: the product package
    (and libgpm.so) is never imported, and its config equals the GPU arm's."""
    import json
    import subprocess
    import sys
    code = ("import runpy, sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--app', 'tc', '--steps', '1',"
            " '--warmup', '0', '--cpu-budget', '0.2']; runpy.run_path('bench.py', run_name='__main__');"
            " assert 'paper_1911_06969_b200' not in sys.modules, 'product imported';"
            " import os; maps = open('/proc/self/maps').read(); assert 'libgpm.so' not in maps, 'libgpm.so mapped'")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["config"]["app"] == "tc"
    sys.path.insert(0, ROOT)
    import bench
    import pyoracle
    g = pyoracle.generate_rmat(16, 16, 0.57, 0.19, 0.19, 1)
    assert line["config"] == bench.workload_config("tc", g.n, g.m, 0)


def test_engine_header_test_apps_built_and_linked():
    """tests/apps/libgpm_testapps.so (user apps on include/gpm_engine.cuh)
    loads against libgpm.so and exports its entry point (no GPU call)."""
    import ctypes
    import paper_1911_06969_b200  # noqa: F401  (loads libgpm.so)
    path = os.path.join(ROOT, "tests", "apps", "libgpm_testapps.so")
    assert os.path.exists(path), "run __graft_entry__.build()"
    L = ctypes.CDLL(path)
    assert hasattr(L, "testapp_mine")
