"""Pins for oracle O9 (eq.(1) layer budget) and O10 (eq.(2) merge) — CPU only."""
import json
import os

import numpy as np

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- eq.(1)
def _hist_with_variance(v, E=2, T=10**9):
    """Counts whose frequencies f = hist/T have population variance ~v (two experts: mean ± sqrt(v))."""
    d = np.sqrt(v)
    f = np.array([0.5 + d, 0.5 - d])
    return np.round(f * T).astype(np.int64)


def test_budget_worked_example():
    g = json.load(open(os.path.join(GOLD, "budget_example.json")))
    T = 10 ** 9
    hist = np.stack([_hist_with_variance(v, T=T) for v in g["v"]])
    C, b, v, over = oracle.layer_budget(hist, T, g["B_non"], n_non=np.full(g["L"], 64))
    assert np.allclose(v, g["v"], rtol=1e-6)
    assert np.allclose(b, g["b"], rtol=1e-5)
    assert list(C) == g["B"]
    assert over == sum(g["B"]) - g["B_non"]


def test_budget_equal_variance_is_linear_in_depth():
    L, T = 6, 10 ** 6
    hist = np.stack([_hist_with_variance(0.01, T=T)] * L)
    C, b, _, _ = oracle.layer_budget(hist, T, 210, n_non=np.full(L, 1000))
    # b_l ∝ L-l+1 = 6..1, sum 21 -> B = 210*b/21 = 60,50,...,10 exactly (up to the floor)
    assert np.allclose(b / b[-1], np.arange(L, 0, -1))
    assert list(C) == [60, 50, 40, 30, 20, 10] or list(C) == [59, 49, 39, 29, 19, 9] or \
        all(abs(c - w) <= 1 for c, w in zip(C, [60, 50, 40, 30, 20, 10]))


def test_budget_skewed_layer_gets_smaller_budget():
    # highly skewed layers need a smaller merging budget (divide by v)
    T = 10 ** 6
    hist = np.stack([_hist_with_variance(0.04, T=T), _hist_with_variance(0.01, T=T)])
    C, *_ = oracle.layer_budget(hist, T, 40, n_non=np.array([64, 64]))
    # b = [2/0.04, 1/0.01] = [50, 100]
    assert C[0] < C[1]


def test_budget_clamps():
    T = 10 ** 6
    hist = np.stack([_hist_with_variance(0.01, T=T)] * 3)
    C, *_ = oracle.layer_budget(hist, T, 1, n_non=np.array([5, 5, 5]))
    assert list(C) == [1, 1, 1]  # never zero experts in a layer
    C, *_ = oracle.layer_budget(hist, T, 3000, n_non=np.array([5, 5, 5]))
    assert list(C) == [5, 5, 5]  # never more than the layer's non-tuning experts
    E = hist.shape[1]
    C, *_ = oracle.layer_budget(hist, T, 10 * E)
    assert list(C) == [E, E, E]  # no n_non: every expert is non-tuning, so at most E (R9)


# ---------------------------------------------------------------- eq.(2)
def test_merge_worked_examples():
    g = json.load(open(os.path.join(GOLD, "merge_example.json")))
    fo = g["freq_only"]
    out, remap = oracle.merge(np.array(fo["W"])[:, None], [0, 0], fo["f"], 1)
    assert out[0, 0] == fo["W_c"] and list(remap) == [0, 0]
    af = g["att_freq"]
    alpha = np.array(af["f"]) * np.array(af["abar"])
    out, _ = oracle.merge(np.array(fo["W"])[:, None], [0, 0], alpha, 1)
    assert abs(out[0, 0] - af["W_c"]) < 1e-15


def test_merge_singleton_identity_and_mean():
    rng = np.random.default_rng(0)
    E, n = 6, 1000
    W = oracle.bf16_round(rng.standard_normal((E, n)))
    cl = np.arange(E)  # every expert its own cluster
    out, remap = oracle.merge(W, cl, rng.uniform(0, 1, E), E)
    assert np.array_equal(out, W)  # |E_c| = 1 -> bit-exact identity
    out, _ = oracle.merge(W, np.zeros(E, np.int32), np.full(E, 0.3), 1)
    assert np.allclose(out[0], W.mean(0), rtol=0, atol=1e-14)  # equal alpha -> mean


def test_merge_invariances_and_zero_alpha():
    rng = np.random.default_rng(1)
    E, n, C = 8, 300, 3
    W = rng.standard_normal((E, n))
    cl = np.array([0, 1, 2, 0, 1, 2, 0, 1], np.int32)
    a = rng.uniform(0.01, 1, E)
    o1, _ = oracle.merge(W, cl, a, C)
    o2, _ = oracle.merge(W, cl, a * 7.5, C)  # scale invariance
    assert np.allclose(o1, o2, atol=1e-13)
    perm = rng.permutation(E)  # member order invariance
    o3, _ = oracle.merge(W[perm], cl[perm], a[perm], C)
    assert np.allclose(o1, o3, atol=1e-13)
    # convex combination: weights sum to one -> merging a constant gives the constant
    o4, _ = oracle.merge(np.full((E, 4), 2.5), cl, a, C)
    assert np.allclose(o4, 2.5, atol=1e-14)
    # all-zero alpha cluster -> plain mean (R10)
    a0 = a.copy()
    a0[cl == 2] = 0
    o5, _ = oracle.merge(W, cl, a0, C)
    assert np.allclose(o5[2], W[cl == 2].mean(0), atol=1e-14)


def test_merge_remap_tuning_first():
    cl = np.array([-1, 0, 1, -1, 0, 1, 1], np.int32)
    _, remap = oracle.merge(np.zeros((7, 2)), cl, np.ones(7), 2)
    # tuning experts 0, 3 -> slots 0, 1; cluster 0 -> 2, cluster 1 -> 3
    assert list(remap) == [0, 2, 3, 1, 2, 3, 3]
