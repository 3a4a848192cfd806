"""Independent brute-force oracles (pure Python, small graphs only).

These restate the SPEC.md definitions directly from edge/vertex SETS, not by
incremental extension, so they check both the C++ oracle and the CUDA path:

* triangles by O(n^3) triple loop
* k-cliques by subset check
* connected induced k-subgraphs, classified by a permutation canonicaliser
                                                        SPEC.md:440, :507, :509
* connected edge subsets with their canonical generation order, canonical-
  mapping MNI with the level-wise filter semantics of Alg. 1
                                                        SPEC.md:449, :508, :509
"""
from __future__ import annotations

import itertools
from collections import defaultdict

import numpy as np


def adjacency(off, col):
    n = len(off) - 1
    return [set(int(x) for x in col[off[v]:off[v + 1]]) for v in range(n)]


def canon(nv, labels, edges):
    """Lexicographic minimum of (labels, sorted edge list) over permutations in
    lexicographic permutation order; the first minimiser wins."""
    best = None
    bperm = None
    for perm in itertools.permutations(range(nv)):
        lab = [0] * nv
        for i in range(nv):
            lab[perm[i]] = labels[i]
        es = sorted((min(perm[a], perm[b]), max(perm[a], perm[b])) for a, b in edges)
        key = (lab, es)
        if best is None or key < best:
            best, bperm = key, perm
    return best, list(bperm)


def canon_all(nv, labels, edges):
    """Every permutation achieving the canonical form (all isomorphic mappings
    of the embedding onto the canonical pattern, automorphisms included)."""
    best, _ = canon(nv, labels, edges)
    out = []
    for perm in itertools.permutations(range(nv)):
        lab = [0] * nv
        for i in range(nv):
            lab[perm[i]] = labels[i]
        es = sorted((min(perm[a], perm[b]), max(perm[a], perm[b])) for a, b in edges)
        if (lab, es) == best:
            out.append(list(perm))
    return best, out


def text(nv, labels, edges):
    return "k=%d;L=%s;E=%s" % (nv, ",".join(str(x) for x in labels), "".join("(%d,%d)" % e for e in edges))


def triangles(adj):
    n = len(adj)
    t = 0
    for a in range(n):
        for b in adj[a]:
            if b <= a:
                continue
            for c in adj[b]:
                if c > b and c in adj[a]:
                    t += 1
    return t


def cliques(adj, k):
    n = len(adj)
    cnt = 0

    def rec(cands, size):
        nonlocal cnt
        if size == k:
            cnt += 1
            return
        for v in sorted(cands):
            rec({u for u in cands if u > v and u in adj[v]}, size + 1)

    rec(set(range(n)), 0)
    return cnt


def canonical_vertex_order(adj, S):
    """Canonical generation order of a connected vertex set."""
    S = set(S)
    order = [min(S)]
    chosen = {order[0]}
    while len(order) < len(S):
        cand = [u for u in S - chosen if any(u in adj[v] for v in chosen)]
        if not cand:
            return None  # disconnected
        u = min(cand)
        order.append(u)
        chosen.add(u)
    return order


def motifs(adj, k):
    """Connected induced k-subgraphs -> canonical pattern text -> count."""
    n = len(adj)
    out = defaultdict(int)
    for S in itertools.combinations(range(n), k):
        order = canonical_vertex_order(adj, S)
        if order is None:
            continue
        edges = [(i, j) for i in range(k) for j in range(i + 1, k) if order[j] in adj[order[i]]]
        (lab, es), _ = canon(k, [0] * k, edges)
        out[text(k, lab, es)] += 1
    return dict(out)


def _norm(a, b):
    return (a, b) if a < b else (b, a)


def canonical_edge_order(S):
    """Canonical generation order of a connected edge set."""
    S = set(S)
    seq = [min(S)]
    verts = set(seq[0])
    while len(seq) < len(S):
        cand = [e for e in S - set(seq) if e[0] in verts or e[1] in verts]
        if not cand:
            return None
        e = min(cand)
        seq.append(e)
        verts |= set(e)
    return seq


def edge_emb_quick(seq, labels):
    """Vertex insertion order, position labels and position edges of an
    edge-mode embedding given its edge sequence."""
    verts = [seq[0][0], seq[0][1]]
    for a, b in seq[1:]:
        for x in (a, b):
            if x not in verts:
                verts.append(x)
    pos = {v: i for i, v in enumerate(verts)}
    edges = sorted(_norm(pos[a], pos[b]) for a, b in seq)
    lab = [int(labels[v]) for v in verts]
    return verts, lab, edges


def connected_edge_subsets(adj, size):
    """All connected edge subsets with `size` edges (as canonical sequences)."""
    n = len(adj)
    E = sorted({_norm(a, b) for a in range(n) for b in adj[a] if a != b})
    seen = set()
    frontier = {frozenset([e]) for e in E}
    for _ in range(size - 1):
        nxt = set()
        for S in frontier:
            vs = set()
            for a, b in S:
                vs |= {a, b}
            for v in vs:
                for w in adj[v]:
                    e = _norm(v, w)
                    if e not in S:
                        nxt.add(S | {e})
        frontier = nxt
    for S in frontier:
        if S in seen:
            continue
        seen.add(S)
        yield canonical_edge_order(S)


def fsm(adj, labels, k, sigma, full=False, support="mni"):
    """Level-wise FSM with canonical-mapping MNI (full=True: true MNI over all
    isomorphic mappings) and Alg. 1 filter semantics.
    Returns ([(level, text, mni)...], level_sizes)."""
    result = []
    level_sizes = []
    survivors = None  # set of frozenset edge sets surviving the previous level
    for lev in range(1, k):
        embs = []
        for seq in connected_edge_subsets(adj, lev):
            if lev > 1 and frozenset(seq[:-1]) not in survivors:
                continue
            embs.append(seq)
        level_sizes.append(len(embs))
        dom = {}
        pat_of = {}
        for seq in embs:
            verts, lab, edges = edge_emb_quick(seq, labels)
            if full:
                (cl, ce), perms = canon_all(len(verts), lab, edges)
            else:
                (cl, ce), perm = canon(len(verts), lab, edges)
                perms = [perm]
            t = text(len(verts), cl, ce)
            d = dom.setdefault(t, [set() for _ in range(len(verts))])
            for perm in perms:
                for i, v in enumerate(verts):
                    d[perm[i]].add(v)
            pat_of[frozenset(seq)] = t
        if support == "count":  # embedding-count support (SPEC.md CountSupport)
            cnt = defaultdict(int)
            for S, t in pat_of.items():
                cnt[t] += 1
            mni = dict(cnt)
        else:
            mni = {t: min(len(s) for s in d) for t, d in dom.items()}
        for t, m in mni.items():
            if m >= sigma:
                result.append((lev, t, m))
        survivors = {S for S, t in pat_of.items() if mni[t] >= sigma}
    result.sort(key=lambda r: (r[0], -r[2], r[1]))
    return result, level_sizes


def gnp(n, p, seed):
    rng = np.random.default_rng(seed)
    iu = np.triu_indices(n, 1)
    mask = rng.random(len(iu[0])) < p
    return list(zip(iu[0][mask].tolist(), iu[1][mask].tolist()))
