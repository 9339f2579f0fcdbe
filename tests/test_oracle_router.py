"""Pins for oracle O2 (router/gating) and O3 (D_e permutation, histogram) — CPU only.

P:217-220: "tokens ... first pass through a gating network, which determines
their assignment to different experts"; activation frequency =
activated tokens / total tokens; D_e = tokens passing through e.
Softmax/top-k and the tie-break are reading R2; the stable order is R3.
"""
import itertools
import json
import os

import numpy as np
import pytest
from scipy.special import softmax as scipy_softmax

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _router_from_z(z, k, norm):
    # H = 1, x = [1]: z_e = W_r[e][0]
    z = np.asarray(z, np.float64)
    return oracle.router(np.ones((1, 1)), z[:, None], k, norm)


def test_worked_example():
    g = json.load(open(os.path.join(GOLD, "router_example.json")))
    z = g["z"]
    for kk, want in g["topk_sets"].items():
        k = int(kk)
        _, ids, w, m = _router_from_z(z, k, 0)
        assert list(ids[0]) == want
        if kk in g["margins"]:
            assert m[0] == g["margins"][kk]
    p = np.exp(z) / np.exp(z).sum()
    _, ids, w, _ = _router_from_z(z, 2, 0)
    assert np.allclose(w[0], p[[1, 2]], rtol=0, atol=1e-15)
    assert np.allclose(np.round(p, 6), g["softmax_6dp"])
    _, ids, w, _ = _router_from_z(z, 2, 1)
    assert np.allclose(w[0], g["weights_norm1_k2"], atol=1e-15)


def _brute_topk(z, k):
    """Max-sum k-subset; ties -> lexicographically smallest sorted index tuple."""
    best, best_s = None, -np.inf
    for S in itertools.combinations(range(len(z)), k):
        s = sum(z[i] for i in S)
        if s > best_s:
            best, best_s = S, s
    return set(best)


@pytest.mark.parametrize("E,k", [(4, 1), (5, 2), (8, 2), (8, 3), (6, 6)])
def test_brute_force_subsets(E, k):
    rng = np.random.default_rng(E * 10 + k)
    for trial in range(60):
        if trial % 3 == 0:  # integer logits: many exact ties
            z = rng.integers(-2, 3, size=E).astype(np.float64)
        else:
            z = rng.standard_normal(E)
        _, ids, w, m = _router_from_z(z, k, trial % 2)
        assert set(ids[0]) == _brute_topk(list(z), k)
        # listed in descending z
        assert all(z[ids[0][j]] >= z[ids[0][j + 1]] for j in range(k - 1))
        if k < E:
            rest = [e for e in range(E) if e not in set(ids[0])]
            assert m[0] == z[ids[0][-1]] - max(z[rest])


def test_softmax_against_scipy():
    rng = np.random.default_rng(1)
    H, E, T = 16, 12, 40
    x = rng.standard_normal((T, H))
    wr = rng.standard_normal((E, H))
    z, ids, w, _ = oracle.router(x, wr, 3, 0)
    assert np.allclose(z, x @ wr.T, rtol=1e-13, atol=1e-13)
    p = scipy_softmax(x @ wr.T, axis=1)
    assert np.allclose(w, np.take_along_axis(p, ids, 1), rtol=1e-12)
    _, _, w1, _ = oracle.router(x, wr, 3, 1)
    ps = np.take_along_axis(p, ids, 1)
    assert np.allclose(w1, ps / ps.sum(1, keepdims=True), rtol=1e-12)
    assert np.allclose(w1.sum(1), 1.0)


def test_degenerate_cases():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((10, 8))
    # k == E: every expert chosen, margin = inf
    _, ids, _, m = oracle.router(x, rng.standard_normal((5, 8)), 5, 0)
    assert all(sorted(r) == list(range(5)) for r in ids) and np.all(np.isinf(m))
    # E == 1: weight 1
    _, ids, w, _ = oracle.router(x, rng.standard_normal((1, 8)), 1, 0)
    assert np.all(ids == 0) and np.allclose(w, 1.0)
    # all-zero router: all logits tie -> experts 0..k-1
    _, ids, _, m = oracle.router(x, np.zeros((6, 8)), 3, 1)
    assert np.all(ids == np.arange(3)) and np.all(m == 0)


def test_permute_against_sorted_and_invariants():
    rng = np.random.default_rng(3)
    T, E, k = 57, 7, 3
    ids = np.stack([rng.permutation(E)[:k] for _ in range(T)]).astype(np.int32)
    hist, off, ti, inv = oracle.permute(ids, E)
    assert hist.sum() == T * k and off[-1] == T * k
    assert np.array_equal(hist, np.bincount(ids.ravel(), minlength=E))
    assert np.array_equal(np.diff(off), hist)
    for e in range(E):
        want = sorted(t for t in range(T) if e in ids[t])
        assert list(ti[off[e]:off[e + 1]]) == want
    # every (t, j) appears exactly once and inv_pos points back at it
    assert sorted(inv.ravel()) == list(range(T * k))
    for t in range(T):
        for j in range(k):
            p = inv[t, j]
            assert ti[p] == t and off[ids[t, j]] <= p < off[ids[t, j] + 1]


def test_hist_k_equals_E():
    ids = np.tile(np.arange(4, dtype=np.int32), (9, 1))
    hist, *_ = oracle.permute(ids, 4)
    assert np.all(hist == 9)
