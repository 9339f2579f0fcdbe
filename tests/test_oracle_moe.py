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
