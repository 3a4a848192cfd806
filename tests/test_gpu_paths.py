"""GPU: every specialised kernel path equals the generic engine bit for bit.

The engine picks on-chip staged kernels where their preconditions hold
(DESIGN.md §3a/§3b/§4) and keeps the generic per-candidate extend as the
fallback; environment switches force the fallback so both can be compared on
the same inputs (totals, pattern maps, per-level sizes, candidates, B_alg):
  GPM_GENERIC_L1   CF/TC first level: generic batches instead of edge chunks
  GPM_GENERIC_CF   CF last level: generic to_add instead of the sibling probe
  GPM_CF_NOLOCAL   k-CL (k >= 4): level-by-level instead of per-root local rows
  GPM_GENERIC_MC   MC: per-candidate binary search instead of staged sets
  GPM_FSM_TWO_PASS FSM last level: separate domain pass instead of the fused one
  GPM_FSM_FAN_NARROW FSM fan pass: 8-warp CTAs instead of 14-warp ones
"""
import os

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1911_06969_b200 as P
    return P


def _run(P, g, app, k, sigma=0, env=None, **kw):
    old = {}
    for name in (env or []):
        old[name] = os.environ.get(name)
        os.environ[name] = "1"
    try:
        return P.mine(g, app, k, sigma, **kw)
    finally:
        for name, v in old.items():
            if v is None:
                del os.environ[name]
            else:
                os.environ[name] = v


def _same(a, b):
    assert a.total == b.total
    assert a.patterns == b.patterns
    for key in ("level_sizes", "candidates", "n_explored", "b_alg"):
        assert a.stats[key] == b.stats[key], key


@pytest.mark.parametrize("scale,ef,abc", [(11, 16, (0.57, 0.19, 0.19)), (13, 8, (0.45, 0.15, 0.15)),
                                          (12, 24, (0.6, 0.15, 0.15))])
def test_cf_paths(P, scale, ef, abc):
    g = P.Graph(P.generate_rmat(scale, ef, *abc, seed=scale)).orient_dag()
    for k in (3, 4, 5, 6):
        base = _run(P, g, "cf", k)
        _same(base, _run(P, g, "cf", k, env=["GPM_GENERIC_L1"]))
        _same(base, _run(P, g, "cf", k, env=["GPM_GENERIC_CF"]))
        _same(base, _run(P, g, "cf", k, env=["GPM_GENERIC_L1", "GPM_GENERIC_CF"]))
        _same(base, _run(P, g, "cf", k, env=["GPM_CF_NOLOCAL"]))  # local rows vs level by level


@pytest.mark.parametrize("scale,ef,abc", [(11, 16, (0.57, 0.19, 0.19)), (13, 8, (0.45, 0.15, 0.15)),
                                          (14, 16, (0.57, 0.19, 0.19))])
def test_mc_paths(P, scale, ef, abc):
    # staged vs generic MC (GPU vs GPU); RMAT-14 ef16 has roots with |S0| above
    # the warp-kernel limit (3-MC block kernel).  The oracle-checked big-root
    # paths (multi-tile 3-MC, 4-MC HBM union sets) are tests/test_gpu_bigpaths.py
    g = P.Graph(P.generate_rmat(scale, ef, *abc, seed=scale + 1))
    for k in ((3, 4) if scale < 14 else (3,)):
        _same(_run(P, g, "mc", k), _run(P, g, "mc", k, env=["GPM_GENERIC_MC"]))


def test_mc_paths_under_planner_chunks(P):
    g = P.Graph(P.generate_rmat(12, 8, 0.57, 0.19, 0.19, seed=9))
    # the fused 4-MC roots kernel materialises nothing (no chunks, any
    # budget); the level engine under a tiny budget chunks level 2
    base = _run(P, g, "mc", 4, mem_budget=1 << 16)
    tiny = _run(P, g, "mc", 4, env=["GPM_GENERIC_MC"], mem_budget=1 << 16)
    assert base.stats["chunks"] == 0 and tiny.stats["chunks"] > 0
    _same(base, tiny)


@pytest.mark.parametrize("labels,sigma,k", [(4, 30, 4), (16, 10, 4), (8, 20, 3), (6, 40, 5)])
def test_fsm_paths(P, labels, sigma, k):
    g = P.Graph(P.generate_rmat(12, 8, 0.45, 0.15, 0.15, seed=3, n_labels=labels, label_seed=7))
    _same(_run(P, g, "fsm", k, sigma), _run(P, g, "fsm", k, sigma, env=["GPM_FSM_TWO_PASS"]))


@pytest.mark.parametrize("labels,sigma,k", [(4, 30, 4), (8, 20, 3), (6, 40, 5), (1, 50, 3)])
def test_fsm_sparse_domains_equal_bitmaps(P, labels, sigma, k):
    # GPM_FSM_SPARSE: every pattern's domains as sorted (slot, position, vertex)
    # keys instead of bitmaps, with the separate domain pass
    from paper_1911_06969_b200 import _lib
    g = P.Graph(P.generate_rmat(12, 8, 0.45, 0.15, 0.15, seed=3, n_labels=labels, label_seed=7))
    for mni in ("canonical", "automorphism"):
        sp = _run(P, g, "fsm", k, sigma, env=["GPM_FSM_SPARSE", "GPM_FSM_TWO_PASS"], mni=mni)
        assert sp.stats["paths"] & _lib.PATH_FSM_SPARSE
        _same(sp, _run(P, g, "fsm", k, sigma, env=["GPM_FSM_TWO_PASS"], mni=mni))


@pytest.mark.parametrize("labels,sigma,k", [(8, 20, 3), (16, 10, 4)])
def test_fsm_fan_narrow_ctas(P, labels, sigma, k):
    # the fan pass runs 14-warp CTAs when two fit an SM, else 8-warp CTAs
    # (GPM_FSM_FAN_NARROW forces the latter): same patterns and supports
    g = P.Graph(P.generate_rmat(12, 8, 0.45, 0.15, 0.15, seed=5, n_labels=labels, label_seed=9))
    _same(_run(P, g, "fsm", k, sigma), _run(P, g, "fsm", k, sigma, env=["GPM_FSM_FAN_NARROW"]))

