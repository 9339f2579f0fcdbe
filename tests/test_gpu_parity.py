"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Inputs reach the oracle only through the CPU twin of the
generator; nothing the CUDA path computes is fed to the oracle."""
import numpy as np
import pytest

import oracle
import oracle.model as om
import synth

from _parity import check_hist_and_de, compare_layer, input_bound

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _bits_bf16(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


# small configs the oracle finishes in seconds that still span several tiles + ragged tails
SMALL = {
    "toy": synth.CONFIGS["toy"],
    "int4_shared": synth.MoEConfig("mid_int4_shared", 2, 256, 16, 4, 192, 384, 4, 64, 0, 1000, synth.BASE_SEED + 11),
    "int8_ragged": synth.MoEConfig("mid_int8", 2, 128, 12, 3, 80, 0, 8, 0, 1, 777, synth.BASE_SEED + 12),
    "int4_e64": synth.MoEConfig("e64_int4", 1, 128, 64, 6, 128, 256, 4, 128, 0, 650, synth.BASE_SEED + 13),
    # NEXT-3: the paper's bit-2, grouped and per-channel
    "int2_g64": synth.MoEConfig("int2_g64", 2, 128, 16, 4, 128, 192, 2, 64, 1, 600, synth.BASE_SEED + 14),
    "int2_pc": synth.MoEConfig("int2_pc", 2, 192, 8, 2, 64, 0, 2, 0, 0, 300, synth.BASE_SEED + 15),
    # enough rows per expert for the dequant-pass GEMMs (T·k >= 2048·E): partial last n-tiles
    # (F = 176 -> 128 + 48, F_s = 208 -> 128 + 80, H = 320 -> 256 + 64: trimmed MMAs), full 32-row
    # TMA-store slices and ragged per-thread slices, per-channel scales staged in the epilogue
    "pass_tails": synth.MoEConfig("pass_tails", 1, 320, 4, 2, 176, 208, 8, 0, 1, 4500, synth.BASE_SEED + 16),
    "pass_tails_g64": synth.MoEConfig("pass_tails_g64", 1, 320, 3, 2, 192, 0, 4, 64, 0, 3300, synth.BASE_SEED + 17),
}


def _run_gpu(cfg, T=None):
    import paper_2508_19078_b200 as F  # noqa: F401
    from paper_2508_19078_b200.driver import ModelShape, Profiler, QuantizedModel
    from paper_2508_19078_b200 import synthetic
    T = T or cfg.tokens
    masters = synthetic.master_weights(cfg)
    qm = QuantizedModel(ModelShape.of(cfg))
    qm.quantize_from(masters)
    prof = Profiler(ModelShape.of(cfg), T, with_logits=True)
    x = synthetic.tokens(cfg, 0, T)
    ys = []
    prof.run(qm, x, on_layer=lambda l, y: ys.append(y.float().cpu().numpy()))
    torch.cuda.synchronize()
    return masters, qm, prof, ys


@pytest.mark.parametrize("name", list(SMALL))
def test_quantized_weights_bit_exact(name):
    cfg = SMALL[name]
    masters, qm, prof, ys = _run_gpu(cfg, T=1)
    for l in range(cfg.n_layers):
        for e in [0, cfg.n_experts - 1]:
            for fam, q_t, s_t in (("gate", qm.gate_q, qm.gate_s), ("up", qm.up_q, qm.up_s),
                                  ("down", qm.down_q, qm.down_s)):
                w = om.master_f32(synth.spec_expert(cfg, l, e, fam))
                q, s = oracle.quantize(w, cfg.wbits, cfg.group_size)
                qq = oracle.pack(q, cfg.wbits)
                assert np.array_equal(q_t[l, e].cpu().numpy().view(np.uint8), qq.view(np.uint8)), (l, e, fam)
                assert np.array_equal(s_t[l, e].cpu().numpy(), s), (l, e, fam)


@pytest.mark.parametrize("name", list(SMALL))
def test_profile_pass_parity(name):
    cfg = SMALL[name]
    masters, qm, prof, ys = _run_gpu(cfg)
    ref = om.profile_all(cfg)
    T = cfg.tokens
    alive = np.ones(T, bool)
    for l in range(cfg.n_layers):
        gpu = dict(logits=prof.logits[l].cpu().numpy(), ids=prof.ids[l].cpu().numpy(), w=prof.w[l].cpu().numpy(),
                   y=ys[l])
        wr = om.master_f32(synth.spec_router(cfg, l))
        dz = input_bound(ys[l - 1] if l else None, ref[l]["x"], wr)
        rep = compare_layer(l, ref[l], gpu, alive, dz)
        assert rep.n_cmp > 0.9 * T
        check_hist_and_de(gpu["ids"], prof.hist[l].cpu().numpy(), prof.offsets[l].cpu().numpy(),
                          prof.token_index[l].cpu().numpy(), cfg.n_experts)
        if rep.n_div == 0 and np.all(alive):
            assert np.array_equal(prof.hist[l].cpu().numpy(), ref[l]["hist"])
            assert np.array_equal(prof.token_index[l].cpu().numpy(), ref[l]["token_index"])
            assert np.array_equal(prof.offsets[l].cpu().numpy(), ref[l]["offsets"])


def test_chunk_and_run_invariance():
    """Batch invariance: hist/ids/y do not depend on how the tokens are split; reruns are bitwise equal."""
    cfg = SMALL["int4_shared"]
    from paper_2508_19078_b200.driver import ModelShape, Profiler, QuantizedModel
    from paper_2508_19078_b200 import synthetic
    shape = ModelShape.of(cfg)
    qm = QuantizedModel(shape)
    qm.quantize_from(synthetic.master_weights(cfg))
    T = cfg.tokens
    full = Profiler(shape, T, with_logits=True)
    full.run(qm, synthetic.tokens(cfg, 0, T))
    y_full = full.y[(cfg.n_layers - 1) % 2].clone()
    again = Profiler(shape, T, with_logits=True)
    again.run(qm, synthetic.tokens(cfg, 0, T))
    assert torch.equal(full.ids, again.ids) and torch.equal(full.hist, again.hist)
    assert torch.equal(y_full, again.y[(cfg.n_layers - 1) % 2])
    cut = 389  # ragged split, not a multiple of 128
    a = Profiler(shape, cut)
    b = Profiler(shape, T - cut)
    a.run(qm, synthetic.tokens(cfg, 0, cut))
    b.run(qm, synthetic.tokens(cfg, cut, T - cut))
    assert torch.equal(a.hist + b.hist, full.hist)
    assert torch.equal(torch.cat([a.ids, b.ids], 1), full.ids)
    ya, yb = a.y[(cfg.n_layers - 1) % 2], b.y[(cfg.n_layers - 1) % 2]
    assert torch.equal(torch.cat([ya, yb]), y_full)


# every flux_policy combination the bit-identity test pins (weight path, routed rows, fused combine, static tiles)
POLICIES = [(2, 0, 0, 0), (1, 0, 0, 0), (2, 1, 0, 0), (2, 0, 1, 0), (1, 0, 1, 0), (2, 2, 0, 0), (1, 2, 0, 0),
            (1, 1, 0, 0), (1, 0, 0, 1), (1, 0, 1, 1), (1, 1, 0, 1), (0, 0, 0, 0), (1, 0, 0, 0, 0x100 | 7),
            (1, 0, 0, 0, 0x100 | 0), (1, 0, 0, 0, 0, 2), (1, 0, 0, 0, 0, 1)]


@pytest.mark.parametrize("name", ["int4_shared", "int8_ragged", "int4_e64", "pass_tails", "pass_tails_g64"])
def test_weight_paths_bit_identical(name):
    """Every flux_policy value — in-GEMM dequantization or the separate dequant pass, the routed A rows
    materialised (x_perm), gathered inside the GEMM with cp.async (the pass-path default) or with TMA
    gather4 (test-only), the combine standalone or fused into the shared down GEMM (test-only), claimed or
    static tile order (test-only), every L2-hint combination, gate/up and down as two launches or chained
    in one — produces bit-identical layers: the choice is a pure performance policy."""
    import paper_2508_19078_b200 as F
    from paper_2508_19078_b200.driver import ModelShape, Profiler, QuantizedModel
    from paper_2508_19078_b200 import synthetic
    cfg = SMALL[name]
    shape = ModelShape.of(cfg)
    qm = QuantizedModel(shape)
    qm.quantize_from(synthetic.master_weights(cfg))
    x = synthetic.tokens(cfg, 0, cfg.tokens)
    outs = []
    for pol in POLICIES:
        prof = Profiler(shape, cfg.tokens, policy=F.make_policy(*pol))
        prof.run(qm, x)
        torch.cuda.synchronize()
        outs.append((prof.y[(cfg.n_layers - 1) % 2].clone(), prof.ids.clone(), prof.hist.clone()))
    for y, ids, hist in outs[1:]:
        assert torch.equal(y, outs[0][0]) and torch.equal(ids, outs[0][1]) and torch.equal(hist, outs[0][2])


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("variant", ["balanced", "tuning", "zero_alpha", "singletons"])
def test_merge_parity(dtype, variant):
    import paper_2508_19078_b200 as F
    rng = np.random.default_rng(hash((dtype, variant)) % 2**32)
    cfg = synth.CONFIGS["toy"]
    E, C = 12, 4
    numel = 64 * 96
    W = np.stack([synth.cpu_matrix(synth.Spec(64, 96, cfg.seed, synth.stream_id(synth.KIND_MASTER_F32, 0, e),
                                              synth.scale_c(1.0), 0, 0.0), dtype=dtype) for e in range(E)])
    Wf = W.astype(np.float32) if dtype == "f32" else synth.bf16_bits_to_f32(W)
    cl = (np.arange(E) % C).astype(np.int32)
    alpha = rng.uniform(0.01, 1.0, E).astype(np.float32)
    if variant == "tuning":
        cl[[1, 7]] = -1
    if variant == "zero_alpha":
        alpha[cl == 2] = 0
    if variant == "singletons":
        C = E
        cl = np.arange(E, dtype=np.int32)
    ref, remap_ref = oracle.merge(Wf.reshape(E, numel).astype(np.float64), cl, alpha.astype(np.float64), C)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    dev_W = torch.from_numpy(Wf.reshape(E, numel)).to("cuda", tdt)
    out = torch.empty(C, numel, dtype=tdt, device="cuda")
    remap = torch.empty(E, dtype=torch.int32, device="cuda")
    F.merge_experts(dev_W, torch.from_numpy(cl).cuda(), torch.from_numpy(alpha).cuda(), C, out, remap)
    got = out.float().cpu().numpy().astype(np.float64)
    assert np.array_equal(remap.cpu().numpy(), remap_ref)
    # condition-aware bound: |Δ| <= tol * Σ_e w_e |W_e|
    absw = np.zeros_like(ref)
    for c in range(C):
        mem = np.nonzero(cl == c)[0]
        a = alpha[mem].astype(np.float64)
        wts = a / a.sum() if a.sum() > 0 else np.full(len(mem), 1.0 / len(mem))
        absw[c] = (wts[:, None] * np.abs(Wf.reshape(E, numel)[mem].astype(np.float64))).sum(0)
    tol = 1e-5 if dtype == "f32" else 2e-2
    assert np.all(np.abs(got - ref) <= tol * absw + 1e-30)
    if dtype == "bf16":  # expected within one bf16 rounding of the exact value
        assert np.mean(got == oracle.bf16_round(ref)) > 0.99
    if variant == "singletons":
        assert torch.equal(out, dev_W)  # |E_c| = 1 -> identity, bit for bit


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_merge_packed_stages(dtype):
    """K7's stage packing (merge.cu): slices are packed four per stage ACROSS chunk boundaries, so a
    stage mixes the tail of one chunk with the head of the next.  Cluster sizes 1..9 (K-Means-like),
    an empty cluster (zeros, no error), two tuning experts, and outputs spanning several 16 KB chunks
    with a ragged tail put every slot position, chunk start and chunk end in every combination."""
    import paper_2508_19078_b200 as F
    rng = np.random.default_rng(7 if dtype == "bf16" else 8)
    cfg = synth.CONFIGS["toy"]
    sizes = [1, 9, 0, 2, 5, 3, 1, 4, 7, 6, 2]      # cluster 2 is empty
    E, C = sum(sizes) + 2, len(sizes)
    rows, cols = 41, 488                           # numel 20,008: 2 (bf16) / 4 (fp32) whole chunks + a tail
    numel = rows * cols
    W = np.stack([synth.cpu_matrix(synth.Spec(rows, cols, cfg.seed, synth.stream_id(synth.KIND_MASTER_F32, 1, e),
                                              synth.scale_c(1.0), 0, 0.0), dtype=dtype) for e in range(E)])
    Wf = (W.astype(np.float32) if dtype == "f32" else synth.bf16_bits_to_f32(W)).reshape(E, numel)
    perm = rng.permutation(E)
    cl = np.full(E, -1, np.int32)                  # the last two of perm stay tuning experts
    i = 0
    for c, n in enumerate(sizes):
        cl[perm[i:i + n]] = c
        i += n
    alpha = rng.uniform(0.01, 1.0, E).astype(np.float32)
    tdt = torch.float32 if dtype == "f32" else torch.bfloat16
    dev_W = torch.from_numpy(Wf).to("cuda", tdt)
    out = torch.full((C, numel), 7.0, dtype=tdt, device="cuda")
    remap = torch.empty(E, dtype=torch.int32, device="cuda")
    F.merge_experts(dev_W, torch.from_numpy(cl).cuda(), torch.from_numpy(alpha).cuda(), C, out, remap)
    got = out.float().cpu().numpy().astype(np.float64)
    assert np.all(got[2] == 0.0)                   # the empty cluster: zeros
    live = [c for c in range(C) if sizes[c] > 0]   # the oracle rejects empty clusters: relabel the rest
    relabel = {c: j for j, c in enumerate(live)}
    cl_live = np.array([relabel.get(int(c), -1) if c >= 0 else -1 for c in cl], np.int32)
    ref, _ = oracle.merge(Wf.astype(np.float64), cl_live, alpha.astype(np.float64), len(live))
    tol = 1e-5 if dtype == "f32" else 2e-2
    for j, c in enumerate(live):
        mem = np.nonzero(cl == c)[0]
        wts = alpha[mem].astype(np.float64) / alpha[mem].astype(np.float64).sum()
        absw = (wts[:, None] * np.abs(Wf[mem].astype(np.float64))).sum(0)
        assert np.all(np.abs(got[c] - ref[j]) <= tol * absw + 1e-30), c
        if sizes[c] == 1:
            assert np.array_equal(got[c], Wf[mem[0]].astype(np.float64))  # singleton: bit for bit
        if dtype == "bf16":
            assert np.mean(got[c] == oracle.bf16_round(ref[j])) > 0.99


def test_quantizer_ties_and_extremes_bit_exact():
    """Half-integer quotients (ties to even), saturation, zero and tiny groups: the GPU quantizer's
    reciprocal fast path must fall back to the IEEE division exactly where it matters."""
    import json
    import os
    import paper_2508_19078_b200 as F
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "quantize_examples.json")))
    rng = np.random.default_rng(11)
    for wbits in (2, 4, 8):
        qmax = (1 << (wbits - 1)) - 1
        rows = []
        for c in gold["cases"]:
            rows.append(np.array(c["w"] + [0.0] * 60, np.float32))
        for _ in range(200):  # every element an exact multiple of s/2 -> many exact ties
            s = np.float32(2.0) ** rng.integers(-20, 10)
            k = rng.integers(-2 * qmax - 1, 2 * qmax + 2, size=64).astype(np.float32)
            k[0] = 2 * qmax  # pins max|w| = qmax*s exactly
            rows.append((k * s / 2).astype(np.float32))
        rows.append(np.full(64, 1e-40, np.float32))  # denormal group
        w = np.stack(rows)
        q_ref, s_ref = oracle.quantize(w, wbits, 64)
        tw = torch.from_numpy(w).cuda()
        q = torch.empty(w.shape[0], 64 * wbits // 8, dtype=torch.uint8, device="cuda")
        s = torch.empty(w.shape[0], 1, dtype=torch.float32, device="cuda")
        F.quantize_weights(tw, wbits, 64, q, s)
        qq = oracle.pack(q_ref, wbits).view(np.uint8)
        assert np.array_equal(q.cpu().numpy(), qq), wbits
        assert np.array_equal(s.cpu().numpy(), s_ref), wbits


def test_quantizer_direct_bit_exact():
    import paper_2508_19078_b200 as F
    rng = np.random.default_rng(3)
    for wbits, g, dt in [(8, 0, "bf16"), (4, 128, "bf16"), (4, 64, "f32"), (8, 64, "f32"), (4, 0, "bf16"),
                         (2, 128, "bf16"), (2, 0, "f32"), (2, 64, "bf16")]:
        R, K = 37, 640
        w = (rng.standard_normal((R, K)) * rng.uniform(0.001, 10, (R, 1))).astype(np.float32)
        w[5] = 0
        if dt == "bf16":
            w = oracle.bf16_round(w).astype(np.float32)
        q_ref, s_ref = oracle.quantize(w, wbits, g)
        tw = torch.from_numpy(w).cuda().to(torch.bfloat16 if dt == "bf16" else torch.float32)
        q = torch.empty(R, K * wbits // 8, dtype=torch.uint8, device="cuda")
        s = torch.empty(R, K // (g or K), dtype=torch.float32, device="cuda")
        F.quantize_weights(tw, wbits, g, q, s)
        qq = oracle.pack(q_ref, wbits).view(np.uint8)
        assert np.array_equal(q.cpu().numpy(), qq), (wbits, g, dt)
        assert np.array_equal(s.cpu().numpy(), s_ref), (wbits, g, dt)


def _quantize_both(w, wbits, g, dtype):
    """GPU codes/scales and the oracle's for the same (already representable) values."""
    import paper_2508_19078_b200 as F
    R, K = w.shape
    q_ref, s_ref = oracle.quantize(w, wbits, g)
    tw = torch.from_numpy(w).cuda().to(dtype)
    q = torch.empty(R, K * wbits // 8, dtype=torch.uint8, device="cuda")
    s = torch.empty(R, K // (g or K), dtype=torch.float32, device="cuda")
    F.quantize_weights(tw, wbits, g, q, s)
    return q.cpu().numpy(), s.cpu().numpy(), oracle.pack(q_ref, wbits).view(np.uint8), s_ref


def test_quantizer_exhaustive_bf16():
    """Every (w, s) pair a bf16 group can produce, up to a common power of two: max|w| = a with each
    of the 128 bf16 mantissas, w every bf16 value with |w| <= a over the 10 binades where |w/s| can
    reach 1/2 at qmax = 127 (below them every code is 0), both signs.  The GPU's division-free
    quotient (Markstein correction, quantize.cu) must give the oracle's codes (IEEE division, RNE)
    bit for bit at INT8/INT4/INT2, grouped and per channel."""
    mant = 1.0 + np.arange(128) / 128.0
    cand = np.concatenate([mant * 2.0 ** -e for e in range(10)])
    cand = np.concatenate([cand, -cand, [0.0]]).astype(np.float32)
    rows = []
    for a in mant.astype(np.float32):
        ws = cand[np.abs(cand) <= a]
        for i in range(0, len(ws), 127):
            chunk = ws[i:i + 127]
            rows.append(np.concatenate([[a], chunk, np.zeros(127 - len(chunk), np.float32)]))
    w = np.stack(rows).astype(np.float32)  # every value is exactly representable in bf16
    assert np.array_equal(oracle.bf16_round(w).astype(np.float32), w)
    for wbits in (8, 4, 2):
        for g in (128, 0):
            q, s, q_ref, s_ref = _quantize_both(w, wbits, g, torch.bfloat16)
            assert np.array_equal(s, s_ref), (wbits, g)
            assert np.array_equal(q, q_ref), (wbits, g, int((q != q_ref).sum()))


def test_quantizer_near_ties_f32():
    """fp32 masters: quotients within a few ulps of every half-integer n + 1/2 (the only places where
    a quotient that is not correctly rounded would change a code), for random scales."""
    rng = np.random.default_rng(5)
    for wbits in (8, 4, 2):
        qmax = (1 << (wbits - 1)) - 1
        rows = []
        for _ in range(400):
            a = np.float32(rng.uniform(0.5, 1.0) * 2.0 ** rng.integers(-30, 30))
            s = np.float32(a / np.float32(qmax))
            vals = []
            for n in range(-qmax - 1, qmax):
                h = np.float32((n + 0.5) * np.float64(s))
                v = h
                for _k in range(3):
                    v = np.nextafter(v, np.float32(np.inf))
                    vals.append(v)
                v = h
                for _k in range(3):
                    v = np.nextafter(v, np.float32(-np.inf))
                    vals.append(v)
                vals.append(h)
            vals = np.array([v for v in vals if abs(v) <= a], np.float32)
            for i in range(0, len(vals), 255):  # rows of 256: max|w| = a, then 255 probes
                row = np.zeros(256, np.float32)
                row[0] = a
                row[1:1 + len(vals[i:i + 255])] = vals[i:i + 255]
                rows.append(row)
        w = np.stack(rows)
        q, s, q_ref, s_ref = _quantize_both(w, wbits, 0, torch.float32)
        assert np.array_equal(s, s_ref), wbits
        assert np.array_equal(q, q_ref), (wbits, int((q != q_ref).sum()))


def test_attention_hist_unit_bit_exact():
    """NEXT-3 (α = f·ā, R15): integer fixed-point sums, so the GPU must equal the oracle bit for bit,
    including empty (-1) picks and ties in the 2^-24 rounding."""
    import paper_2508_19078_b200 as F
    rng = np.random.default_rng(21)
    for T, E, k in ((1, 4, 2), (3000, 64, 6), (70001, 128, 8), (5000, 16, 4)):
        ids = np.stack([rng.choice(E, size=k, replace=False) for _ in range(T)]).astype(np.int32)
        ids[rng.random((T, k)) < 0.1] = -1
        a = np.abs(rng.standard_normal(T)).astype(np.float32)
        a[: T // 10] = (rng.integers(0, 64, T // 10) * 2.0 ** -25).astype(np.float32)  # exact ties
        want = oracle.attention_hist(ids, a, E)
        got = torch.zeros(E, dtype=torch.int64, device="cuda")
        F.attention_hist(torch.from_numpy(ids).cuda(), torch.from_numpy(a).cuda(), E, got)
        assert np.array_equal(got.cpu().numpy(), want), (T, E, k)


@pytest.mark.parametrize("name", ["toy", "int4_shared"])
def test_attention_weighted_alpha_through_the_profile(name):
    """Per layer A_e from the profiled routing: equal to the oracle's (its own routing and its own copy
    of the attention values) where every token routes identically, and always consistent with the
    GPU's own picks."""
    import paper_2508_19078_b200 as F  # noqa: F401
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import ModelShape, Profiler, QuantizedModel
    cfg = SMALL[name]
    T = cfg.tokens
    qm = QuantizedModel(ModelShape.of(cfg))
    qm.quantize_from(synthetic.master_weights(cfg))
    prof = Profiler(ModelShape.of(cfg), T)
    attn = synthetic.attention_values(cfg, 0, T)
    prof.run(qm, synthetic.tokens(cfg, 0, T), attn=attn)
    torch.cuda.synchronize()
    ref = om.profile_all(cfg)
    for l in range(cfg.n_layers):
        a_ref = np.abs(synth.cpu_matrix(synth.spec_attn(cfg, l), dtype="f32")[:, 0])
        ids_gpu = prof.ids[l].cpu().numpy()
        A_gpu = prof.ahist[l].cpu().numpy()
        assert np.array_equal(A_gpu, oracle.attention_hist(ids_gpu, a_ref, cfg.n_experts))
        if np.array_equal(np.sort(ids_gpu, 1), np.sort(ref[l]["ids"], 1)):
            assert np.array_equal(A_gpu, oracle.attention_hist(ref[l]["ids"], a_ref, cfg.n_experts))


def test_frequencies_bit_exact():
    """flux_frequencies: α = fl32(count / denom) with the fp64 quotient — exactly numpy's
    (count / denom).astype(float32), for f = hist / T and α = A / (2^24·T) (R15)."""
    import paper_2508_19078_b200 as F
    rng = np.random.default_rng(23)
    for n, hi in ((1, 10), (28 * 64, 262144 * 6), (5000, 2 ** 50)):
        counts = rng.integers(0, hi, n).astype(np.int64)
        for denom in (262144.0, 2097152.0, 16777216.0 * 262144, 3.0):
            a = torch.empty(n, dtype=torch.float32, device="cuda")
            F.frequencies(torch.from_numpy(counts).cuda(), denom, a)
            assert np.array_equal(a.cpu().numpy(), (counts / denom).astype(np.float32)), (n, denom)
