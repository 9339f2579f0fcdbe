"""Pins for oracle O4-O6 (quantized MoE layer forward) — CPU only.

P:196-220: an MoE layer routes each token through the experts its gating
network selects.  Expert form (SwiGLU), bf16 storage points and the residual
are readings R4-R6.  Pins use independent formulations:
  * E = 1, k = 1 reduces to a dense SwiGLU MLP -> torch fp64 matmuls;
  * a dense-equivalent layer (every expert on every token, then masked by the
    selected set, with the INT8 scale applied as s ⊙ (x·qᵀ)) -> numpy;
  * shared experts add the same dense MLP to every token.
"""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")


def _bf16_torch(t):
    # fp64 -> bf16 via torch (fp64 -> fp32 -> bf16); identical to direct RNE except at
    # double-rounding ties, which these random inputs do not hit (checked by ulps below)
    return t.to(torch.float32).to(torch.bfloat16).to(torch.float64)


def _rand_expert(rng, H, F, wbits, g, scale=1.0):
    mats = []
    for rows, K in ((F, H), (F, H), (H, F)):
        w = (rng.standard_normal((rows, K)) * scale / np.sqrt(K)).astype(np.float32)
        w = oracle.bf16_round(w).astype(np.float32)
        q, s = oracle.quantize(w, wbits, g)
        mats += [q, s]
    return oracle.QExpert(*mats)


def _deq(q, s, grouped):
    """Reading R1b, restated with torch's own bf16 conversions: grouped -> bf16(q * bf16(s)); per channel -> q*s."""
    g = q.shape[1] // s.shape[1]
    srep = np.repeat(s, g, axis=1)
    if not grouped:
        return q.astype(np.float64) * srep.astype(np.float64)
    sb = torch.from_numpy(srep).to(torch.bfloat16).to(torch.float32)
    return (torch.from_numpy(q.astype(np.float32)) * sb).to(torch.bfloat16).to(torch.float64).numpy()


def _bf16_x(rng, n, H):
    return oracle.bf16_round(rng.standard_normal((n, H)))


def _ulps_close(a, b, max_ulps=1):
    # a, b bf16-valued: compare in units of the bf16 ulp of max(|a|,|b|)
    m = np.maximum(np.abs(a), np.abs(b))
    ulp = 2.0 ** (np.floor(np.log2(np.where(m > 0, m, 1.0))) - 7)
    return np.abs(a - b) <= max_ulps * ulp + 1e-300


@pytest.mark.parametrize("wbits,g", [(8, 0), (4, 32)])
def test_single_expert_is_dense_swiglu(wbits, g):
    rng = np.random.default_rng(7)
    H, F, n = 64, 96, 20
    ex = _rand_expert(rng, H, F, wbits, g)
    x = _bf16_x(rng, n, H)
    wr = rng.standard_normal((1, H))
    y, ids, w, _, _ = oracle.moe_tokens(x, wr, [ex], None, k=1, group_size=g, norm=0)
    assert np.all(ids == 0) and np.allclose(w, 1.0)
    qg, sg, qu, su, qd, sd = [ex.arrs[i] for i in (0, 3, 1, 4, 2, 5)]
    X = torch.from_numpy(x)
    Wg, Wu, Wd = (torch.from_numpy(_deq(a, b, g != 0)) for a, b in ((qg, sg), (qu, su), (qd, sd)))
    a = _bf16_torch(torch.nn.functional.silu(X @ Wg.T) * (X @ Wu.T))
    o = _bf16_torch(a @ Wd.T)
    ref = _bf16_torch(X + o).numpy()
    assert np.mean(y == ref) > 0.99 and np.all(_ulps_close(y, ref))


@pytest.mark.parametrize("norm", [0, 1])
def test_sparse_equals_dense_equivalent(norm):
    rng = np.random.default_rng(11 + norm)
    H, F, E, k, n = 32, 48, 6, 2, 30
    experts = [_rand_expert(rng, H, F, 8, 0) for _ in range(E)]
    x = _bf16_x(rng, n, H)
    wr = rng.standard_normal((E, H))
    y, ids, w, z, _ = oracle.moe_tokens(x, wr, experts, None, k=k, group_size=0, norm=norm)
    # dense-equivalent: all experts on all tokens, INT8 per-channel scale applied after the dot product
    outs = []
    for ex in experts:
        qg, qu, qd, sg, su, sd = ex.arrs
        g_ = (x @ qg.T.astype(np.float64)) * sg[:, 0].astype(np.float64)
        u_ = (x @ qu.T.astype(np.float64)) * su[:, 0].astype(np.float64)
        a = oracle.bf16_round(g_ / (1 + np.exp(-g_)) * u_)
        outs.append(oracle.bf16_round((a @ qd.T.astype(np.float64)) * sd[:, 0].astype(np.float64)))
    outs = np.stack(outs, 1)  # [n][E][H]
    p = np.exp(z - z.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    mask = np.zeros((n, E))
    for t in range(n):
        sel = np.argsort(-z[t], kind="stable")[:k]
        mask[t, sel] = p[t, sel] / (p[t, sel].sum() if norm else 1.0)
    ref = oracle.bf16_round(x + np.einsum("te,teh->th", mask, outs))
    assert np.all(_ulps_close(y, ref)) and np.mean(y == ref) > 0.98


def test_shared_expert_adds_dense_mlp():
    rng = np.random.default_rng(13)
    H, F, Fs, E, k, n = 32, 32, 64, 4, 2, 16
    experts = [_rand_expert(rng, H, F, 4, 16) for _ in range(E)]
    sh = _rand_expert(rng, H, Fs, 4, 16)
    x = _bf16_x(rng, n, H)
    wr = np.zeros((E, H))  # routing fixed to experts {0,1}
    y_sh, *_ = oracle.moe_tokens(x, wr, experts, sh, k=k, group_size=16, norm=0)
    y_no, *_ = oracle.moe_tokens(x, wr, experts, None, k=k, group_size=16, norm=0)
    # shared output computed independently (single dense expert with weight 1)
    o_sh, *_ = oracle.moe_tokens(x, np.zeros((1, H)), [sh], None, k=1, group_size=16, norm=0)
    sh_only = o_sh - x  # = bf16(x + o) - x; compare loosely (two roundings)
    diff = y_sh - y_no
    assert np.allclose(diff, sh_only, atol=0.05 * np.abs(sh_only).max())


def test_zero_down_row_keeps_bias_feature():
    # the synthetic recipe's bias feature: W_down row 0 == 0 keeps y[:,0] == x[:,0]
    rng = np.random.default_rng(17)
    H, F, E = 16, 16, 3
    experts = []
    for _ in range(E):
        ex = _rand_expert(rng, H, F, 8, 0)
        ex.arrs[2][0, :] = 0  # q_down row 0
        experts.append(ex)
    x = _bf16_x(rng, 8, H)
    x[:, 0] = 1.0
    y, *_ = oracle.moe_tokens(x, rng.standard_normal((E, H)), experts, None, k=2, group_size=0, norm=1)
    assert np.all(y[:, 0] == 1.0)


def _dense_equivalent(x, z, experts, k, norm, grouped, shared=None):
    """Independent numpy/torch formulation of O4-O6 without the residual: every expert on every token
    (weights dequantized per R1b with torch's bf16 conversions), masked by the top-k set; returns
    (branch sum Σ_j w_j o_j + sh [n][H] unrounded, magnitude Σ_j w_j|o_j| + |sh| [n][H])."""
    n = x.shape[0]
    E = len(experts)
    X = torch.from_numpy(x)

    def run(ex, want_mag=False):
        qg, qu, qd, sg, su, sd = ex.arrs
        Wg, Wu, Wd = (torch.from_numpy(_deq(a, b, grouped)) for a, b in ((qg, sg), (qu, su), (qd, sd)))
        a = _bf16_torch(torch.nn.functional.silu(X @ Wg.T) * (X @ Wu.T))
        if want_mag:  # max_f |a_f·ŵd_hf|
            return (a.abs()[:, None, :] * Wd.abs()[None, :, :]).amax(-1).numpy()
        return _bf16_torch(a @ Wd.T).numpy()

    outs = np.stack([run(ex) for ex in experts], 1)  # [n][E][H]
    dots = np.stack([run(ex, True) for ex in experts], 1)
    p = np.exp(z - z.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    mask = np.zeros((n, E))
    for t in range(n):
        sel = np.argsort(-z[t], kind="stable")[:k]
        mask[t, sel] = p[t, sel] / (p[t, sel].sum() if norm else 1.0)
    branch = np.einsum("te,teh->th", mask, outs)
    mag = np.einsum("te,teh->th", mask, np.abs(outs))
    dmag = np.einsum("te,teh->th", mask, dots)
    if shared is not None:
        o_sh = run(shared)
        branch = branch + o_sh
        mag = mag + np.abs(o_sh)
        dmag = dmag + run(shared, True)
    _dense_equivalent.dmag = dmag
    return branch, mag


@pytest.mark.parametrize("wbits,g,norm,with_shared", [(8, 0, 1, False), (4, 16, 0, True), (4, 32, 1, True)])
def test_zero_residual_is_the_moe_branch(wbits, g, norm, with_shared):
    """R6 with r = 0: y = bf16(sh + Σ_j w_j o_j) — the MoE branch alone, checked against the
    dense-equivalent formulation; cond = |sh| + Σ_j w_j|o_j| exactly (up to summation order)."""
    rng = np.random.default_rng(31 + wbits + g)
    H, F, Fs, E, k, n = 64, 64, 96, 6, 2, 40
    experts = [_rand_expert(rng, H, F, wbits, g) for _ in range(E)]
    sh = _rand_expert(rng, H, Fs, wbits, g) if with_shared else None
    x = _bf16_x(rng, n, H)
    wr = rng.standard_normal((E, H))
    y, ids, w, z, _, cond, dmag = oracle.moe_tokens(x, wr, experts, sh, k=k, group_size=g, norm=norm,
                                                    residual=np.zeros_like(x), with_cond=True)
    branch, mag = _dense_equivalent(x, z, experts, k, norm, g != 0, sh)
    ref = oracle.bf16_round(branch)
    assert np.all(_ulps_close(y, ref)) and np.mean(y == ref) > 0.98
    assert np.allclose(cond, mag, rtol=1e-12, atol=1e-300)
    assert np.allclose(dmag, _dense_equivalent.dmag, rtol=1e-12, atol=1e-300)
    assert np.all(cond <= dmag * 64 * (1 + 2.0 ** -8) + 1e-300)  # |o_h| <= F·max_f |a_f w_hf| (F = 64)
    # the zero-residual output is NOT the residual output minus x: the residual changes the rounding
    y_r, *_ = oracle.moe_tokens(x, wr, experts, sh, k=k, group_size=g, norm=norm)
    assert np.all(_ulps_close(y_r, oracle.bf16_round(x + branch)))
    assert np.abs(y).max() < np.abs(y_r).max()  # the branch alone is small next to the residual stream


def test_residual_array_and_cond_bound():
    """An explicit residual r replaces x in O6 (R6); cond = |r| + |sh| + Σ w|o| bounds |y| (up to the
    final rounding) and equals |y| exactly when every term of the sum is non-negative."""
    rng = np.random.default_rng(41)
    H, F, E, k, n = 32, 48, 5, 3, 25
    experts = [_rand_expert(rng, H, F, 8, 0) for _ in range(E)]
    x = _bf16_x(rng, n, H)
    r = _bf16_x(rng, n, H)
    wr = rng.standard_normal((E, H))
    y, ids, w, z, _, cond, dmag = oracle.moe_tokens(x, wr, experts, None, k=k, group_size=0, norm=0, residual=r,
                                                    with_cond=True)
    branch, mag = _dense_equivalent(x, z, experts, k, 0, False)
    assert np.all(_ulps_close(y, oracle.bf16_round(r + branch)))
    assert np.allclose(cond, np.abs(r) + mag, rtol=1e-12)
    assert np.all(np.abs(y) <= cond * (1 + 2.0 ** -8) + 1e-300)
    # all terms non-negative: zero routed weights (E experts, q_down = 0) and r >= 0 -> cond == |r| == |y|
    for ex in experts:
        ex.arrs[2][:] = 0
    y0, *_, cond0, _ = oracle.moe_tokens(x, wr, experts, None, k=k, group_size=0, norm=0, residual=np.abs(r),
                                      with_cond=True)
    assert np.array_equal(cond0, np.abs(r)) and np.array_equal(y0, np.abs(r))


def test_exact_dequant_variant():
    """SURVEY O4's literal reading ŵ = q·s (kept only to show that R1b is not load-bearing): identical to
    R1b for per-channel codes; for grouped codes it equals a dense layer with the exact q·s weights."""
    rng = np.random.default_rng(43)
    H, F, E, k, n = 64, 64, 4, 2, 20
    x = _bf16_x(rng, n, H)
    wr = rng.standard_normal((E, H))
    pc = [_rand_expert(rng, H, F, 8, 0) for _ in range(E)]
    a = oracle.moe_tokens(x, wr, pc, None, k=k, group_size=0, norm=1)[0]
    b = oracle.moe_tokens(x, wr, pc, None, k=k, group_size=0, norm=1, exact_dequant=True)[0]
    assert np.array_equal(a, b)
    gr = [_rand_expert(rng, H, F, 4, 16) for _ in range(E)]
    y, ids, w, z, _ = oracle.moe_tokens(x, wr, gr, None, k=k, group_size=16, norm=1, exact_dequant=True,
                                        residual=np.zeros_like(x))
    X = torch.from_numpy(x)
    outs = []
    for ex in gr:
        qg, qu, qd, sg, su, sd = ex.arrs
        Wg, Wu, Wd = (torch.from_numpy(q.astype(np.float64) * np.repeat(s, 16, axis=1).astype(np.float64))
                      for q, s in ((qg, sg), (qu, su), (qd, sd)))
        act = _bf16_torch(torch.nn.functional.silu(X @ Wg.T) * (X @ Wu.T))
        outs.append(_bf16_torch(act @ Wd.T).numpy())
    outs = np.stack(outs, 1)
    ref = oracle.bf16_round(np.stack([sum(w[t, j] * outs[t, ids[t, j]] for j in range(k)) for t in range(n)]))
    assert np.all(_ulps_close(y, ref))
    y_r1b = oracle.moe_tokens(x, wr, gr, None, k=k, group_size=16, norm=1, residual=np.zeros_like(x))[0]
    assert not np.array_equal(y, y_r1b)  # the two readings differ (by bf16 rounding of the weights)
