"""oracle/pyoracle.py — TEST INFRASTRUCTURE ONLY.

ctypes front-end for the CPU checkers built by oracle/Makefile:

* ``liboracle.so``  — C++20/OpenMP restatement of the SPEC.md engine
  (oracle/oracle.cpp), the parity oracle for every GPU result.
* ``_ref/libref.so`` — the reference's own headers
  (/root/reference/proj/include/gpmine) behind a C shim (oracle/ref_shim.cpp).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
APPS = {"tc": 0, "cf": 1, "mc": 2, "fsm": 3}

_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError("oracle/liboracle.so missing: run `make -C oracle`")
        L = C.CDLL(path)
        L.oracle_mine_json.restype = C.c_void_p
        L.oracle_mine_json.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64, C.c_int,
                                       C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64,
                                       C.c_uint64, C.c_int, C.c_int]
        L.oracle_free.argtypes = [C.c_void_p]
        L.oracle_canonicalize.restype = C.c_void_p
        L.oracle_canonicalize.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p]
        L.oracle_orient_dag.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64,
                                        C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]
        L.oracle_free_buf.argtypes = [C.c_void_p]
        L.oracle_generate_rmat.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                           C.c_uint32, C.c_uint64, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                           C.POINTER(C.c_void_p), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64)]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(os.path.join(HERE, "_ref", "libref.so"))


class _RefCsr(C.Structure):
    _fields_ = [("n", C.c_uint32), ("m", C.c_uint64), ("off", C.c_void_p), ("col", C.c_void_p),
                ("lab", C.c_void_p), ("orig", C.c_void_p)]


def ref():
    global _ref
    if _ref is None:
        path = os.path.join(HERE, "_ref", "libref.so")
        if not os.path.exists(path):
            raise RuntimeError("oracle/_ref/libref.so missing (needs /root/reference at build time)")
        L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(_RefCsr), C.POINTER(C.c_uint64)]
        L.ref_orient_dag.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(_RefCsr)]
        L.ref_init_single_edges.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_int,
                                            C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_uint64)]
        L.ref_has_edge.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_int, C.c_void_p, C.c_void_p,
                                   C.c_uint64, C.c_void_p]
        L.ref_triangle_count.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_uint64)]
        L.ref_reconstruct_edge.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                           C.c_uint64, C.c_void_p, C.POINTER(C.c_int), C.c_void_p,
                                           C.POINTER(C.c_int)]
        L.ref_free.argtypes = [C.c_void_p]
        _ref = L
    return _ref


@dataclass
class Csr:
    """Host CSR: offsets u64[n+1], col u32[m], optional labels u32[n]."""
    off: np.ndarray
    col: np.ndarray
    labels: Optional[np.ndarray] = None
    oriented: bool = False
    orig: Optional[np.ndarray] = None

    @property
    def n(self) -> int:
        return len(self.off) - 1

    @property
    def m(self) -> int:
        return len(self.col)


def _p(a):
    return None if a is None else a.ctypes.data


def csr_from_edges(edges, n: Optional[int] = None, labels=None) -> Csr:
    """Clean like graph_io.hpp:83-116 but WITHOUT id compaction when n is given:
    symmetrise, drop self-loops, dedup, ascending lists."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if n is None:
        n = int(e.max()) + 1 if len(e) else 0
    e = e[e[:, 0] != e[:, 1]]
    both = np.concatenate([e, e[:, ::-1]]) if len(e) else e
    if len(both):
        key = np.unique(both[:, 0] * (n + 1) + both[:, 1])
        src, dst = key // (n + 1), key % (n + 1)
    else:
        src = dst = np.zeros(0, dtype=np.int64)
    off = np.zeros(n + 1, dtype=np.uint64)
    np.add.at(off, src + 1, 1)
    off = np.cumsum(off).astype(np.uint64)
    lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.uint32)
    return Csr(off, dst.astype(np.uint32), lab)


def mine(g: Csr, app: str, k: int = 3, min_support: int = 0, threads: int = 0, chunk_size: int = 1024,
         root_lo: int = 0, root_hi: int = 2**64 - 1, no_orient: bool = False, mni: str = "canonical") -> dict:
    L = lib()
    off = np.ascontiguousarray(g.off, dtype=np.uint64)
    col = np.ascontiguousarray(g.col, dtype=np.uint32)
    lab = None if g.labels is None else np.ascontiguousarray(g.labels, dtype=np.uint32)
    p = L.oracle_mine_json(_p(off), _p(col), _p(lab), g.n, g.m, int(g.oriented), APPS[app], k, min_support,
                           threads, chunk_size, root_lo, root_hi, int(no_orient),
                           {"canonical": 0, "automorphism": 1}[mni])
    s = C.string_at(p).decode()
    L.oracle_free(p)
    d = json.loads(s)
    if "error" in d:
        raise RuntimeError(d["error"])
    return d


def canonicalize(nv: int, labels, edges):
    L = lib()
    lab = np.ascontiguousarray(labels, dtype=np.uint32)
    ed = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1))
    p = L.oracle_canonicalize(nv, _p(lab), len(ed) // 2, _p(ed) if len(ed) else None)
    s = C.string_at(p).decode()
    L.oracle_free(p)
    if s.startswith("error:"):
        raise ValueError(s)
    text, perm = s.split("|")
    return text, [int(x) for x in perm.split(",")]


def orient_dag(g: Csr) -> Csr:
    L = lib()
    oo, oc, om = C.c_void_p(), C.c_void_p(), C.c_uint64()
    off = np.ascontiguousarray(g.off, dtype=np.uint64)
    col = np.ascontiguousarray(g.col, dtype=np.uint32)
    if L.oracle_orient_dag(_p(off), _p(col), g.n, g.m, C.byref(oo), C.byref(oc), C.byref(om)) != 0:
        raise RuntimeError("oracle orient failed")
    o = np.ctypeslib.as_array(C.cast(oo, C.POINTER(C.c_uint64)), shape=(g.n + 1,)).copy()
    c = (np.ctypeslib.as_array(C.cast(oc, C.POINTER(C.c_uint32)), shape=(om.value,)).copy()
         if om.value else np.zeros(0, np.uint32))
    L.oracle_free_buf(oo)
    L.oracle_free_buf(oc)
    return Csr(o, c, g.labels, True)


def generate_rmat(scale: int, edge_factor: float, a: float, b: float, c: float, seed: int = 1,
                  n_labels: int = 0, label_seed: int = 101) -> Csr:
    """SURVEY §8d synthetic graph, restated in oracle.cpp (no libgpm.so)."""
    L = lib()
    po, pc, pl = C.c_void_p(), C.c_void_p(), C.c_void_p()
    n, m = C.c_uint32(), C.c_uint64()
    if L.oracle_generate_rmat(scale, edge_factor, a, b, c, seed, n_labels, label_seed, C.byref(po), C.byref(pc),
                              C.byref(pl), C.byref(n), C.byref(m)) != 0:
        raise RuntimeError("oracle_generate_rmat failed")
    off = np.ctypeslib.as_array(C.cast(po, C.POINTER(C.c_uint64)), shape=(n.value + 1,)).copy()
    col = np.ctypeslib.as_array(C.cast(pc, C.POINTER(C.c_uint32)), shape=(m.value,)).copy()
    lab = (np.ctypeslib.as_array(C.cast(pl, C.POINTER(C.c_uint32)), shape=(n.value,)).copy()
           if pl.value else None)
    for p_ in (po, pc, pl):
        if p_.value:
            L.oracle_free_buf(p_)
    return Csr(off, col, lab)


def _take_ref_csr(r: _RefCsr, oriented=False) -> Csr:
    R = ref()
    off = np.ctypeslib.as_array(C.cast(r.off, C.POINTER(C.c_uint64)), shape=(r.n + 1,)).copy()
    col = (np.ctypeslib.as_array(C.cast(r.col, C.POINTER(C.c_uint32)), shape=(r.m,)).copy()
           if r.m else np.zeros(0, np.uint32))
    lab = (np.ctypeslib.as_array(C.cast(r.lab, C.POINTER(C.c_uint32)), shape=(r.n,)).copy()
           if r.lab and r.n else None)
    orig = (np.ctypeslib.as_array(C.cast(r.orig, C.POINTER(C.c_uint64)), shape=(r.n,)).copy()
            if r.n else np.zeros(0, np.uint64))
    for ptr in (r.off, r.col, r.lab, r.orig):
        if ptr:
            R.ref_free(ptr)
    return Csr(off, col, lab, oriented, orig)


class RefParseError(RuntimeError):
    def __init__(self, msg, line):
        super().__init__(msg)
        self.line = line


def ref_load(path: str, labeled: bool = False) -> Csr:
    R = ref()
    r = _RefCsr()
    line = C.c_uint64(0)
    rc = R.ref_load(path.encode(), int(labeled), C.byref(r), C.byref(line))
    if rc == 2:
        raise RefParseError(R.ref_last_error().decode(), line.value)
    if rc != 0:
        raise RuntimeError(R.ref_last_error().decode())
    return _take_ref_csr(r)


def ref_orient_dag(g: Csr) -> Csr:
    R = ref()
    r = _RefCsr()
    off = np.ascontiguousarray(g.off, dtype=np.uint64)
    col = np.ascontiguousarray(g.col, dtype=np.uint32)
    if R.ref_orient_dag(_p(off), _p(col), g.n, C.byref(r)) != 0:
        raise RuntimeError(R.ref_last_error().decode())
    out = _take_ref_csr(r, True)
    out.orig = None
    return out


def ref_init_single_edges(g: Csr):
    R = ref()
    pi, pv, cnt = C.c_void_p(), C.c_void_p(), C.c_uint64()
    off = np.ascontiguousarray(g.off, dtype=np.uint64)
    col = np.ascontiguousarray(g.col, dtype=np.uint32)
    if R.ref_init_single_edges(_p(off), _p(col), g.n, int(g.oriented), C.byref(pi), C.byref(pv), C.byref(cnt)):
        raise RuntimeError(R.ref_last_error().decode())
    n = cnt.value
    idx = np.ctypeslib.as_array(C.cast(pi, C.POINTER(C.c_uint32)), shape=(max(n, 1),))[:n].copy()
    vid = np.ctypeslib.as_array(C.cast(pv, C.POINTER(C.c_uint32)), shape=(max(n, 1),))[:n].copy()
    R.ref_free(pi)
    R.ref_free(pv)
    return idx, vid


def ref_triangle_count(g: Csr):
    R = ref()
    t, c = C.c_uint64(), C.c_uint64()
    off = np.ascontiguousarray(g.off, dtype=np.uint64)
    col = np.ascontiguousarray(g.col, dtype=np.uint32)
    if R.ref_triangle_count(_p(off), _p(col), g.n, C.byref(t), C.byref(c)):
        raise RuntimeError(R.ref_last_error().decode())
    return t.value, c.value
