"""Shared helpers for the GPU-vs-oracle parity tests.

The parity contract (from BASELINE.json's north_star):
  * quantized weights: bit-exact
  * router logits: per token ||z_gpu - z_ref||_inf <= 1e-3 * ||z_ref||_inf
  * routing: margin m_t = z_(k) - z_(k+1) (oracle fp64 logits).  m_t > 1e-3: the
    GPU's set equals the oracle's; otherwise the GPU set must be valid:
    min chosen z_ref >= max unchosen z_ref - 1e-3
  * gate weights: relative 1e-3 on margin-clear tokens
  * layer outputs (bf16): per token ||y_gpu - y_ref||_2 <= 2e-2 ||y_ref||_2 on
    margin-clear tokens
  * histograms: hist == bincount(GPU ids) exactly; equal to the oracle's on
    margin-clear tokens
Tokens are followed free-running through the layers: the oracle sees only x_0
and the weights.  A token whose (valid, near-tie) routing differs from the
oracle's stops being compared at the following layers.
"""
from __future__ import annotations

import numpy as np

MARGIN = 1e-3
LOGIT_TOL = 1e-3
W_TOL = 1e-3
Y_TOL = 2e-2


class LayerReport:
    def __init__(self):
        self.n_cmp = 0
        self.n_tie = 0
        self.n_div = 0


def input_bound(x_gpu, x_ref, wr):
    """Free-running layers: the router is linear, so a difference in its input (the previous
    layer's bf16 output, within the 2e-2 output tolerance) moves logit e by at most
    Σ_d |W_r[e][d]|·|x_gpu[d] - x_ref[d]|.  Zero at layer 0 (identical generated inputs)."""
    if x_gpu is None:
        return np.zeros((x_ref.shape[0], wr.shape[0]))
    return np.abs(x_gpu.astype(np.float64) - x_ref) @ np.abs(wr.astype(np.float64)).T


def compare_layer(l, ref, gpu, alive, dz=None):
    """ref: oracle dict (x, z, ids, w, y, margin); gpu: dict of numpy arrays (logits, ids, w, y) for the
    same tokens; dz: input_bound() [T][E] or None.  alive: bool mask, updated in place."""
    rep = LayerReport()
    z_ref, z_gpu = ref["z"], gpu["logits"]
    k = ref["ids"].shape[1]
    if dz is None:
        dz = np.zeros_like(z_ref)
    idx = np.nonzero(alive)[0]
    rep.n_cmp = len(idx)
    for t in idx:
        zr = z_ref[t]
        err = np.abs(z_gpu[t] - zr)
        assert np.all(err <= LOGIT_TOL * max(np.max(np.abs(zr)), 1e-30) + dz[t]), (l, t, err.max(), dz[t].max())
        s_ref, s_gpu = set(ref["ids"][t]), set(gpu["ids"][t].tolist())
        assert len(s_gpu) == k, (l, t, gpu["ids"][t])
        eff = MARGIN + 2 * dz[t].max()
        clear = ref["margin"][t] > eff
        if clear:
            assert s_gpu == s_ref, (l, t, s_gpu, s_ref, ref["margin"][t])
            order = np.argsort(ref["ids"][t])
            order_g = np.argsort(gpu["ids"][t])
            wr = ref["w"][t][order]
            wg = gpu["w"][t][order_g]
            assert np.all(np.abs(wg - wr) <= (W_TOL + 2 * dz[t].max()) * np.abs(wr) + 1e-9), (l, t, wg, wr)
            yr, yg = ref["y"][t], gpu["y"][t]
            assert np.linalg.norm(yg - yr) <= Y_TOL * np.linalg.norm(yr), (l, t, np.linalg.norm(yg - yr) /
                                                                          np.linalg.norm(yr))
        else:
            rep.n_tie += 1
            chosen = [zr[e] for e in s_gpu]
            unchosen = [zr[e] for e in range(len(zr)) if e not in s_gpu]
            if unchosen:
                assert min(chosen) >= max(unchosen) - eff, (l, t)
            if s_gpu != s_ref:
                rep.n_div += 1
                alive[t] = False
            else:
                yr, yg = ref["y"][t], gpu["y"][t]
                assert np.linalg.norm(yg - yr) <= Y_TOL * np.linalg.norm(yr)
    return rep


def check_hist_and_de(ids_gpu, hist_gpu, offsets_gpu, token_index_gpu, E):
    """Properties that hold at any size: hist == bincount(ids), D_e CSR is the stable grouping.
    ids -1 (a pick folded by gate re-routing, NEXT-2) own no row and are not counted."""
    T, k = ids_gpu.shape
    flat = ids_gpu.ravel()
    live = flat >= 0
    cnt = np.bincount(flat[live], minlength=E)
    assert np.array_equal(hist_gpu, cnt)
    assert hist_gpu.sum() == live.sum()
    # every token's live experts are distinct
    for t in range(T) if k > 1 and not live.all() else []:
        row = ids_gpu[t][ids_gpu[t] >= 0]
        assert len(set(row.tolist())) == len(row)
    if live.all() and k > 1:
        s = np.sort(ids_gpu, axis=1)
        assert np.all(s[:, 1:] != s[:, :-1])
    if offsets_gpu is None:
        return
    assert offsets_gpu[0] == 0 and np.array_equal(np.diff(offsets_gpu), cnt)
    # stable grouping: for each expert, the ascending token ids that chose it
    order = np.argsort(flat, kind="stable")
    order = order[flat[order] >= 0]
    want = (order // k).astype(np.int32)
    assert np.array_equal(token_index_gpu[:len(want)], want)


# ---------------------------------------------------------------------------------------------
# MoE-branch parity (residual r = 0, so y = bf16(sh + Σ_j w_j o_j) is the expert branch alone)
# ---------------------------------------------------------------------------------------------
# Element-wise, condition-aware bounds.  From the oracle, per output element:
#   cond = |sh| + Σ_j w_j|o_j|                 magnitude of the terms of the O6 sum
#   dmax = max_f|a_sh,f ŵ_hf| + Σ_j w_j max_f|a_jf ŵ_hf|   largest down-projection term behind it
# Two correct implementations of R4/R6 differ only where a bf16 storage point rounds to the other
# neighbour: an o_j or sh (<= one bf16 ulp <= 2^-7 of it), an act value a_f (moves its down term by
# <= 2^-7 of it; a few per expert row at most), and y itself (one ulp).  So
#   arithmetic bound:   |Δy| <= ulp(y) + 2^-7·(cond + 2·dmax)      (allows two act flips per element)
#   north star (2e-2):  |Δy| <= ulp(y) + 2e-2·(cond + dmax)
# Where the terms do not cancel and no single down term dominates, cond + dmax ≈ |y| and the north
# star's bound reads |Δy| <= 2e-2·|y| + 1 ulp.
BRANCH_TOL = 2e-2
BRANCH_TIGHT = 2.0 ** -7


def bf16_ulp(v):
    """ulp of the bf16 format (8 significant bits) at |v|; the smallest subnormal at 0."""
    m = np.abs(np.asarray(v, np.float64))
    e = np.floor(np.log2(np.where(m > 0, m, 1.0)))
    return np.where(m > 0, 2.0 ** (e - 7), 2.0 ** -133)


def branch_bound(y_gpu, y_ref, cond, dmax, tight):
    u = bf16_ulp(np.maximum(np.abs(y_gpu), np.abs(y_ref)))
    return u + (BRANCH_TIGHT * (cond + 2 * dmax) if tight else BRANCH_TOL * (cond + dmax))


def branch_violations(y_gpu, y_ref, cond, dmax, tight):
    """Boolean mask of elements outside the bound (tight = the arithmetic bound, else the north star's)."""
    d = np.abs(np.asarray(y_gpu, np.float64) - y_ref)
    return d > branch_bound(y_gpu, y_ref, cond, dmax, tight)


def compare_branch(ref, gpu, tight=True, stats=None):
    """ref: oracle.model.branch_tokens() dict; gpu: logits, ids, w, y for the same tokens (layer input =
    the generated x_0, identical on both sides, so no input term).  Asserts the router contract and the
    element-wise bounds on every token with the oracle's routing; returns (n_compared, n_near_tie, worst
    ratio |Δ| / north-star bound).  stats (dict, optional) collects ratio arrays for reports."""
    z_ref, k = ref["z"], ref["ids"].shape[1]
    n_cmp = n_tie = 0
    worst = 0.0
    for t in range(z_ref.shape[0]):
        zr = z_ref[t]
        assert np.all(np.abs(gpu["logits"][t] - zr) <= LOGIT_TOL * max(np.max(np.abs(zr)), 1e-30)), t
        s_ref, s_gpu = set(ref["ids"][t].tolist()), set(gpu["ids"][t].tolist())
        if ref["margin"][t] <= MARGIN:
            n_tie += 1
            chosen = [zr[e] for e in s_gpu]
            unchosen = [zr[e] for e in range(len(zr)) if e not in s_gpu]
            if unchosen:
                assert min(chosen) >= max(unchosen) - MARGIN, t
            if s_gpu != s_ref:
                continue  # a valid near-tie routing: a different (correct) output
        else:
            assert s_gpu == s_ref, (t, s_gpu, s_ref)
        assert len(s_gpu) == k
        yg, yr, c, dm = gpu["y"][t], ref["y"][t], ref["cond"][t], ref["dmag"][t]
        d = np.abs(yg - yr)
        r_ns = d / branch_bound(yg, yr, c, dm, False)
        r_t = d / branch_bound(yg, yr, c, dm, True)
        if stats is not None:
            stats.setdefault("ns", []).append(r_ns)
            stats.setdefault("tight", []).append(r_t)
            stats.setdefault("literal", []).append(d / (BRANCH_TOL * np.abs(yr) + bf16_ulp(yr)))
            stats.setdefault("exact", []).append(d == 0)
        else:
            bad = r_ns > 1
            assert not bad.any(), ("2e-2", t, np.nonzero(bad)[0][:8], yg[bad][:8], yr[bad][:8])
            bad = r_t > 1
            if tight:
                assert not bad.any(), ("tight", t, np.nonzero(bad)[0][:8], yg[bad][:8], yr[bad][:8], c[bad][:8],
                                       dm[bad][:8])
        worst = max(worst, float(r_ns.max()))
        n_cmp += 1
    return n_cmp, n_tie, worst
