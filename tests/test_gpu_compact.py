"""GPU parity for NEXT-2: gate re-routing + the compact-model forward (§7, reading R14)
and the merge output error, through the C ABI, against oracle O11 on the same seeded
inputs (the oracle's weights come from the CPU generator twin; its cluster assignment and α from
seeded numpy — nothing the CUDA path computes).

Contract: logits as for the quantized path; on margin-clear tokens the set of live
slots and each slot's folded weight equal the oracle's (weights 1e-3 relative) and the empty picks
sit at the same positions; layer outputs 2e-2 relative (bf16); hist == bincount of the live picks,
D_e == their stable grouping; identity merges reproduce the uncompressed model bit for bit."""
import numpy as np
import pytest

import oracle
import oracle.model as om
import synth

from _parity import MARGIN, LOGIT_TOL, W_TOL, Y_TOL, check_hist_and_de, input_bound

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

CASES = {
    # name: (config, clusters, tuning experts per layer, sampled tokens (None = all))
    "toy": (synth.CONFIGS["toy"], 3, 2, None),
    "shared_e16": (synth.MoEConfig("c_e16_shared", 2, 128, 16, 4, 96, 192, 8, 0, 0, 700, synth.BASE_SEED + 21),
                   5, 3, 96),
    "e64_k6": (synth.MoEConfig("c_e64", 2, 128, 64, 6, 128, 256, 4, 128, 0, 520, synth.BASE_SEED + 22), 16, 0, 96),
}


def _alpha(cfg, seed=5):
    return np.random.default_rng(seed).random((cfg.n_layers, cfg.n_experts)).astype(np.float32)


def _gpu_compact(cfg, co, alpha, T, dense=False, with_logits=True):
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import Profiler, compact_model, dense_model
    masters = synthetic.master_weights(cfg)
    if dense:
        model = dense_model(masters)
    else:
        n_tun = int((co[0] < 0).sum())
        C = int(co.max()) + 1
        model = compact_model(masters, torch.from_numpy(alpha).cuda(), torch.from_numpy(co).cuda(), C, n_tun)
    prof = Profiler(model.shape, T, with_logits=with_logits)
    x = synthetic.tokens(cfg, 0, T)
    ys = []
    prof.run(model, x, on_layer=lambda l, y: ys.append(y.float().cpu().numpy()))
    torch.cuda.synchronize()
    return model, prof, ys


def _compare(l, ref, gpu_logits, gpu_ids, gpu_w, gpu_y, alive, dz):
    z_ref = ref["z"]
    for t in np.nonzero(alive)[0]:
        zr = z_ref[t]
        err = np.abs(gpu_logits[t] - zr)
        assert np.all(err <= LOGIT_TOL * np.abs(zr).max() + dz[t]), (l, t)
        eff = MARGIN + 2 * dz[t].max()
        if ref["margin"][t] > eff:
            assert np.array_equal(gpu_ids[t] < 0, ref["ids"][t] < 0), (l, t, gpu_ids[t], ref["ids"][t])
            g = {int(s): float(w) for s, w in zip(gpu_ids[t], gpu_w[t]) if s >= 0}
            r = {int(s): float(w) for s, w in zip(ref["ids"][t], ref["w"][t]) if s >= 0}
            assert g.keys() == r.keys(), (l, t, g, r)
            for s_ in r:
                assert abs(g[s_] - r[s_]) <= (W_TOL + 2 * dz[t].max()) * abs(r[s_]) + 1e-9, (l, t, g, r)
            yr, yg = ref["y"][t], gpu_y[t]
            assert np.linalg.norm(yg - yr) <= Y_TOL * np.linalg.norm(yr), (l, t)
        else:
            alive[t] = False  # a near-tie may legitimately route differently: stop following it


@pytest.mark.parametrize("name", list(CASES))
def test_compact_forward_vs_oracle(name):
    cfg, C, n_tun, n_sample = CASES[name]
    co = synth.cluster_assignment(cfg, C, n_tuning=n_tun)
    alpha = _alpha(cfg)
    T = cfg.tokens
    model, prof, ys = _gpu_compact(cfg, co, alpha, T)
    S = n_tun + C
    toks = np.arange(T) if n_sample is None else np.linspace(0, T - 1, n_sample).astype(np.int64)
    layers = [om.compact_layer(om.dense_layer(cfg, l), co[l], alpha[l].astype(np.float64))
              for l in range(cfg.n_layers)]
    ref = om.compact_forward(cfg, toks, layers)
    alive = np.ones(len(toks), bool)
    x_prev = None
    for l in range(cfg.n_layers):
        assert np.array_equal(model.remap[l].cpu().numpy(), layers[l][5])
        ids = prof.ids[l].cpu().numpy()
        hist = prof.hist[l].cpu().numpy()
        off = prof.offsets[l].cpu().numpy()
        ti = prof.token_index[l].cpu().numpy()
        check_hist_and_de(ids, hist, off, ti, S)
        dz = input_bound(x_prev, ref[l]["x"], layers[l][0])
        _compare(l, ref[l], prof.logits[l].cpu().numpy()[toks], ids[toks], prof.w[l].cpu().numpy()[toks],
                 ys[l][toks], alive, dz)
        x_prev = ys[l][toks]
        if n_sample is None and alive.all():
            h_ref = np.bincount(ref[l]["ids"][ref[l]["ids"] >= 0], minlength=S)
            assert np.array_equal(hist, h_ref)
    assert alive.mean() > 0.8
    folded = (prof.ids.cpu().numpy() < 0).any()
    assert folded or C == cfg.n_experts  # the folding path is exercised


def test_dense_forward_vs_oracle():
    """wbits = 16 without re-routing: the original model in full precision (the error reference)."""
    cfg = synth.CONFIGS["toy"]
    E = cfg.n_experts
    model, prof, ys = _gpu_compact(cfg, None, None, cfg.tokens, dense=True)
    layers = [om.compact_layer(om.dense_layer(cfg, l), -np.ones(E, int), np.ones(E)) for l in range(cfg.n_layers)]
    ref = om.compact_forward(cfg, np.arange(cfg.tokens), layers)
    alive = np.ones(cfg.tokens, bool)
    x_prev = None
    for l in range(cfg.n_layers):
        dz = input_bound(x_prev, ref[l]["x"], layers[l][0])
        _compare(l, ref[l], prof.logits[l].cpu().numpy(), prof.ids[l].cpu().numpy(), prof.w[l].cpu().numpy(), ys[l],
                 alive, dz)
        x_prev = ys[l]
    assert alive.mean() > 0.9


def test_singleton_merge_is_the_original_model_bitwise():
    """Every expert its own cluster: compact slots are bit-exact copies, remap is the identity, so the
    re-routed forward must reproduce the uncompressed forward bit for bit — and the output error is 0."""
    import paper_2508_19078_b200 as F
    cfg = CASES["shared_e16"][0]
    E = cfg.n_experts
    co = np.tile(np.arange(E, dtype=np.int32), (cfg.n_layers, 1))
    alpha = _alpha(cfg)
    _, prof_c, ys_c = _gpu_compact(cfg, co, alpha, cfg.tokens)
    _, prof_d, ys_d = _gpu_compact(cfg, None, None, cfg.tokens, dense=True)
    for l in range(cfg.n_layers):
        assert np.array_equal(ys_c[l], ys_d[l])
        assert np.array_equal(prof_c.ids[l].cpu().numpy(), prof_d.ids[l].cpu().numpy())
    err = F.output_error(prof_c.y[(cfg.n_layers - 1) % 2], prof_d.y[(cfg.n_layers - 1) % 2])
    assert abs(float(err.item())) < 1e-12  # identical outputs: 1 - cos = 0 up to fp64 rounding


def test_output_error_kernel_matches_definition():
    import paper_2508_19078_b200 as F
    rng = np.random.default_rng(9)
    for T, H in ((1, 64), (1000, 128), (20000, 2048)):
        a = torch.from_numpy(rng.standard_normal((T, H)).astype(np.float32)).to(torch.bfloat16)
        b = (a.float() + 0.3 * torch.from_numpy(rng.standard_normal((T, H)).astype(np.float32))).to(torch.bfloat16)
        got = float(F.output_error(a.cuda(), b.cuda()).item())
        A, B = a.double().numpy(), b.double().numpy()
        want = np.mean(1 - (A * B).sum(1) / (np.linalg.norm(A, axis=1) * np.linalg.norm(B, axis=1)))
        assert abs(got - want) <= 1e-12 * max(want, 1e-3), (T, H, got, want)
        again = float(F.output_error(a.cuda(), b.cuda()).item())
        assert got == again  # deterministic


def test_merge_error_falls_with_more_clusters():
    """The paper's merge-quality measure on the synthetic model: merging every expert into one is worse
    than 4 clusters of 4, and singleton clusters (no merging) give 0."""
    import paper_2508_19078_b200 as F
    cfg = CASES["shared_e16"][0]
    _, prof_d, _ = _gpu_compact(cfg, None, None, cfg.tokens, dense=True, with_logits=False)
    last = (cfg.n_layers - 1) % 2
    errs = []
    for C in (1, 4, 16):
        co = synth.cluster_assignment(cfg, C)
        _, prof_c, _ = _gpu_compact(cfg, co, _alpha(cfg), cfg.tokens, with_logits=False)
        errs.append(float(F.output_error(prof_c.y[last], prof_d.y[last]).item()))
    assert abs(errs[2]) < 1e-12 and errs[0] > errs[1] > 1e-6, errs


def test_adaptive_layer_sizes_end_to_end():
    """Per-layer budgets (eq.(1)) through the whole merge path: layer l keeps n_tun[l] tuning
    experts and B(l) merged slots (different per layer), the compact model's forward uses per-layer
    expert counts, and every layer equals the oracle's compact layer (O10/O11).  The budgets come from
    the ORACLE's eq.(1) on the oracle's own routing counts of a token sample."""
    import oracle
    cfg = CASES["shared_e16"][0]
    L, E = cfg.n_layers, cfg.n_experts
    res = om.profile_tokens(cfg, np.arange(256))
    hist = np.stack([np.bincount(r["ids"].ravel(), minlength=E) for r in res]).astype(np.int64)
    n_tun = np.array([2, 0])
    Cl, *_ = oracle.layer_budget(hist, 256, 10, n_non=E - n_tun)
    Cl = np.array([max(2, Cl[0]), min(E - n_tun[1], Cl[1] + 5)])  # make the two layers clearly differ
    co = np.stack([synth.cluster_assignment(cfg, int(Cl[l]), n_tuning=int(n_tun[l]))[l] for l in range(L)])
    alpha = _alpha(cfg, seed=11)
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import Profiler, compact_model, merge_model
    masters = synthetic.master_weights(cfg)
    model = compact_model(masters, torch.from_numpy(alpha).cuda(), torch.from_numpy(co).cuda(), Cl.tolist(),
                          n_tun.tolist())
    S = n_tun + Cl
    assert model.shape.layer_experts == tuple(int(s) for s in S)
    T = cfg.tokens
    prof = Profiler(model.shape, T, with_logits=True)
    ys = []
    prof.run(model, synthetic.tokens(cfg, 0, T), on_layer=lambda l, y: ys.append(y.float().cpu().numpy()))
    torch.cuda.synchronize()
    toks = np.linspace(0, T - 1, 96).astype(np.int64)
    layers = [om.compact_layer(om.dense_layer(cfg, l), co[l], alpha[l].astype(np.float64)) for l in range(L)]
    ref = om.compact_forward(cfg, toks, layers)
    alive = np.ones(len(toks), bool)
    x_prev = None
    for l in range(L):
        assert np.array_equal(model.remap[l].cpu().numpy(), layers[l][5])
        ids = prof.ids[l].cpu().numpy()
        check_hist_and_de(ids, prof.hist[l].cpu().numpy()[:S[l]], prof.offsets[l].cpu().numpy()[:S[l] + 1],
                          prof.token_index[l].cpu().numpy(), int(S[l]))
        assert ids.max() < S[l]
        dz = input_bound(x_prev, ref[l]["x"], layers[l][0])
        _compare(l, ref[l], prof.logits[l].cpu().numpy()[toks], ids[toks], prof.w[l].cpu().numpy()[toks],
                 ys[l][toks], alive, dz)
        x_prev = ys[l][toks]
    assert alive.mean() > 0.8
    # the plain merge with the same per-layer budgets (no tuning experts in layer 1): its slots are the
    # compact model's cluster slots
    merged = merge_model(masters, torch.from_numpy(alpha).cuda(), torch.from_numpy(co).cuda(), Cl.tolist())
    for l in range(L):
        for fam, W in (("gate", model.gate), ("up", model.up), ("down", model.down)):
            got = getattr(merged, fam)[l][:Cl[l]]
            assert torch.equal(got, W[l][n_tun[l]:S[l]]), (l, fam)


@pytest.mark.parametrize("name", list(CASES))
def test_compact_branch_elementwise(name):
    """The compact model's MoE branch alone (all-zero residual, R6), layer by layer on x_0, element by
    element against O11 with r = 0, at the bounds of tests/_parity.py (north star and arithmetic): the
    re-routed picks, the folded weights and the merged bf16 experts are all inside y here."""
    from _parity import BRANCH_TOL, branch_violations
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import Profiler, compact_model
    cfg, C, n_tun, n_sample = CASES[name]
    co = synth.cluster_assignment(cfg, C, n_tuning=n_tun)
    alpha = _alpha(cfg)
    T = cfg.tokens
    masters = synthetic.master_weights(cfg)
    model = compact_model(masters, torch.from_numpy(alpha).cuda(), torch.from_numpy(co).cuda(), C, n_tun)
    prof = Profiler(model.shape, T, with_de=False, with_logits=True)
    x = synthetic.tokens(cfg, 0, T)
    zero = torch.zeros_like(x)
    toks = np.arange(T) if n_sample is None else np.linspace(0, T - 1, n_sample).astype(np.int64)
    x0 = synth.bf16_bits_to_f32(synth.cpu_rows(synth.spec_x(cfg), toks)).astype(np.float64)
    compared = 0
    for l in range(cfg.n_layers):
        y = prof.run_layer(model, l, x, zero).float().cpu().numpy()[toks].astype(np.float64)
        ids = prof.ids[l].cpu().numpy()[toks]
        logits = prof.logits[l].cpu().numpy()[toks]
        wr, g, u, d, sh, remap = om.compact_layer(om.dense_layer(cfg, l), co[l], alpha[l].astype(np.float64))
        yr, idr, wref, zr, mr, cond, dmag = oracle.compact_tokens(x0, wr, remap, g, u, d, sh, k=cfg.top_k,
                                                                   norm=cfg.norm_topk, residual=np.zeros_like(x0),
                                                                   with_cond=True)
        for t in range(len(toks)):
            assert np.all(np.abs(logits[t] - zr[t]) <= LOGIT_TOL * np.abs(zr[t]).max()), (l, t)
            if mr[t] <= MARGIN:
                continue  # a near-tie may route (validly) differently
            assert np.array_equal(ids[t], idr[t]), (l, t, ids[t], idr[t])
            for tight in (False, True):
                bad = branch_violations(y[t], yr[t], cond[t], dmag[t], tight)
                assert not bad.any(), (name, l, t, tight, np.nonzero(bad)[0][:6])
            compared += 1
    assert compared >= 0.8 * cfg.n_layers * len(toks)
    assert BRANCH_TOL == 2e-2
