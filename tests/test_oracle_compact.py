"""Pins for O11 (NEXT-2): gate re-routing after merging (§7) and the compact-model
forward (reading R14) — CPU only.

* identity remap over weights that are exactly q·s  ==  the quantized-model forward O4-O6 (pinned
  separately), bit for bit;
* experts with identical weights merged into one slot: the folded pick computes the same expert
  output, so the compact forward equals the original forward up to one rounding;
* one cluster of identical experts with renormalised gates: y = bf16(x + o(x)) with o from an
  independent numpy SwiGLU;
* re-routing invariants (distinct non-empty slots, slot weights = sums of the original picks'
  weights), singleton clusters = the original model (output error 0), empty picks in O3.
"""
import numpy as np

import oracle
import oracle.model as om
import synth


def _bf16(a):
    return oracle.bf16_round(np.asarray(a, np.float64))


def _rand_layer(rng, E, H, F, scale=0.3):
    mk = lambda *s: _bf16(scale * rng.standard_normal(s))  # noqa: E731
    return mk(E, H), mk(E, F, H), mk(E, F, H), mk(E, H, F)


def test_identity_remap_equals_quantized_forward():
    rng = np.random.default_rng(0)
    E, H, F, k, n = 6, 32, 48, 2, 40
    # per-channel quantized weights whose ŵ = q·s is exact: s = powers of two
    qs = []
    dense = []
    for rows, K in ((F, H), (F, H), (H, F)):
        q = rng.integers(-127, 128, size=(E, rows, K)).astype(np.int8)
        s = (2.0 ** rng.integers(-12, -6, size=(E, rows, 1))).astype(np.float32)
        qs.append((q, s))
        dense.append(q.astype(np.float64) * s.astype(np.float64))
    experts = [oracle.QExpert(qs[0][0][e], qs[0][1][e], qs[1][0][e], qs[1][1][e], qs[2][0][e], qs[2][1][e])
               for e in range(E)]
    wr = _bf16(0.2 * rng.standard_normal((E, H)))
    x = _bf16(rng.standard_normal((n, H)))
    for norm in (0, 1):
        y_q, ids_q, w_q, _, _ = oracle.moe_tokens(x, wr, experts, None, k=k, group_size=0, norm=norm)
        y_c, ids_c, w_c, _, _ = oracle.compact_tokens(x, wr, np.arange(E), *dense, k=k, norm=norm)
        assert np.array_equal(ids_q, ids_c) and np.array_equal(w_q, w_c)
        assert np.array_equal(y_q, y_c)
        # the MoE branch alone (r = 0, R6) and its condition terms agree between the two formulations too
        z0 = np.zeros_like(x)
        bq = oracle.moe_tokens(x, wr, experts, None, k=k, group_size=0, norm=norm, residual=z0, with_cond=True)
        bc = oracle.compact_tokens(x, wr, np.arange(E), *dense, k=k, norm=norm, residual=z0, with_cond=True)
        assert np.array_equal(bq[0], bc[0]) and np.array_equal(bq[5], bc[5]) and np.array_equal(bq[6], bc[6])
        assert not np.array_equal(bc[0], y_c)  # the residual is really gone


def test_identical_experts_fold_to_original():
    rng = np.random.default_rng(1)
    E, H, F, k, n = 6, 32, 40, 3, 60
    wr, g, u, d = _rand_layer(rng, E, H, F)
    for a, b in ((1, 4), (2, 5)):  # make pairs identical
        g[b], u[b], d[b] = g[a], u[a], d[a]
    cluster_of = np.array([-1, 0, 1, -1, 0, 1])
    alpha = rng.random(E)
    x = _bf16(rng.standard_normal((n, H)))
    wr_c, gc, uc, dc, _, remap = om.compact_layer((wr, g, u, d, None), cluster_of, alpha)
    assert list(remap) == [0, 2, 3, 1, 2, 3]
    for norm in (0, 1):
        y0, ids0, w0, _, _ = oracle.compact_tokens(x, wr, np.arange(E), g, u, d, k=k, norm=norm)
        y1, ids1, w1, _, _ = oracle.compact_tokens(x, wr_c, remap, gc, uc, dc, k=k, norm=norm)
        # the same outputs up to the rounding of (w_i + w_j)·o vs w_i·o + w_j·o: at most one bf16 step
        diff = np.abs(y1 - y0)
        assert np.all(diff <= 2.0 ** -7 * np.abs(y0) + 1e-30)
        assert np.mean(diff == 0) > 0.95
        folded = (ids1 < 0).any(1)
        assert folded.any()  # the case is exercised


def test_one_cluster_closed_form():
    rng = np.random.default_rng(2)
    E, H, F, k, n = 5, 32, 64, 3, 25
    wr, g, u, d = _rand_layer(rng, E, H, F)
    g[:], u[:], d[:] = g[0], u[0], d[0]
    x = _bf16(rng.standard_normal((n, H)))
    _, gc, uc, dc, _, remap = om.compact_layer((wr, g, u, d, None), np.zeros(E, int), np.ones(E))
    y, ids, w, _, _ = oracle.compact_tokens(x, wr, remap, gc, uc, dc, k=k, norm=1)
    # independent SwiGLU in numpy: a = bf16(SiLU(x·Gᵀ) ⊙ (x·Uᵀ)), o = bf16(a·Dᵀ), y = bf16(x + o)
    gx, ux = x @ g[0].T, x @ u[0].T
    a = _bf16(gx / (1 + np.exp(-gx)) * ux)
    o = _bf16(a @ d[0].T)
    want = _bf16(x + o)
    # Σw = 1 up to one fp64 rounding: exact cancellations x = -o may leave ~1e-16
    assert np.all(np.abs(y - want) <= 2.0 ** -7 * np.abs(want) + 1e-12 * np.abs(o).max())
    assert np.all(ids[:, 0] == 0) and np.all(ids[:, 1:] == -1)
    assert np.allclose(w[:, 0], 1.0, atol=1e-12)


def test_rerouting_invariants_and_singletons():
    cfg = synth.CONFIGS["toy"]
    dense = om.dense_layer(cfg, 0)
    co = synth.cluster_assignment(cfg, 3, n_tuning=2)[0]
    alpha = np.random.default_rng(3).random(cfg.n_experts)
    wr, g, u, d, sh, remap = om.compact_layer(dense, co, alpha)
    x = synth.bf16_bits_to_f32(synth.cpu_rows(synth.spec_x(cfg), np.arange(64))).astype(np.float64)
    _, ids0, w0, _, _ = oracle.router(x, wr, cfg.top_k, cfg.norm_topk)[:3] + (None, None)
    y, ids, w, _, _ = oracle.compact_tokens(x, wr, remap, g, u, d, sh, k=cfg.top_k, norm=cfg.norm_topk)
    for t in range(len(x)):
        slots = ids[t][ids[t] >= 0]
        assert len(set(slots)) == len(slots)
        assert set(slots) == set(remap[ids0[t]])
        for s_ in slots:
            assert np.isclose(w[t][ids[t] == s_].sum(), w0[t][remap[ids0[t]] == s_].sum(), rtol=1e-14)
        assert np.all(w[t][ids[t] < 0] == 0)
    hist, off, ti, inv = oracle.permute(ids, int(remap.max()) + 1)
    assert off[-1] == (ids >= 0).sum() == len(ti) and np.all((inv < 0) == (ids < 0))
    # every expert its own cluster: the compact model is the original model, output error 0
    E = cfg.n_experts
    layers_orig = [om.compact_layer(om.dense_layer(cfg, l), -np.ones(E, int), np.ones(E)) for l in range(2)]
    layers_single = [om.compact_layer(om.dense_layer(cfg, l), np.arange(E), alpha) for l in range(2)]
    a = om.compact_forward(cfg, np.arange(32), layers_orig)[-1]["y"]
    b = om.compact_forward(cfg, np.arange(32), layers_single)[-1]["y"]
    assert np.array_equal(a, b) and abs(om.output_error(b, a)) < 1e-15
