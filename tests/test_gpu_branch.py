"""GPU parity of the MoE branch alone: flux_profile_layer with a ZERO residual buffer, so that
y = bf16(sh + Σ_j w_j o_j) holds only the expert FFNs of the quantized model (the MoE layer
of P:217-220) — compared element by element with the oracle's O4-O6 (oracle.model.branch_tokens,
residual r = 0, reading R6), at the north star's 2e-2 and at the bound the arithmetic allows
(tests/_parity.py: |Δ| <= 2^-7·cond + ulp, cond = |sh| + Σ_j w_j|o_j|).

With the residual in y, the routed experts are only ~1-5% of ||y|| on the synthetic recipe and a
per-token norm check cannot see them; here nothing dilutes them.  Every layer of the small and edge
configs, a DeepSeek-layer-shaped routed-only config through both weight paths (in-GEMM dequant at
1,024 tokens; the dequant pass + in-GEMM cp.async gather at 24,576 tokens), and layer 0 of both
BASELINE shapes at their full token counts (sampled tokens).  A group scale multiplied by 1.1 must
be caught; the check must also hold against the SURVEY's exact ŵ = q·s oracle (R1b not
load-bearing)."""
import numpy as np
import pytest

import oracle.model as om
import synth

from _parity import branch_violations, compare_branch
from test_gpu_edges import EDGE
from test_gpu_parity import SMALL

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

S = synth.BASE_SEED
# DeepSeek-MoE-16B layer shape, routed experts only (no shared MLP), INT4 g128
DS_ROUTED = synth.MoEConfig("ds_routed", 1, 2048, 64, 6, 1408, 0, 4, 128, 0, 1024, S + 31)
WEIGHT_PATH = {"auto": 0, "pass": 1, "fused": 2}  # flux_policy.weight_path


def _gpu_branch(cfg, T, layers, corrupt=None, path="auto"):
    """Quantize on the GPU, then one flux_profile_layer per layer on x_0 with a zero residual.
    Returns (qm, {layer: (logits, ids, w, y)}) as device tensors."""
    import paper_2508_19078_b200 as F
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import ModelShape, Profiler, QuantizedModel
    shape = ModelShape.of(cfg)
    masters = synthetic.master_weights(cfg)
    qm = QuantizedModel(shape)
    qm.quantize_from(masters)
    del masters
    if corrupt is not None:
        corrupt(qm)
    x = synthetic.tokens(cfg, 0, T)
    zero = torch.zeros_like(x)
    prof = Profiler(shape, T, with_de=False, with_logits=True, policy=F.make_policy(WEIGHT_PATH[path]))
    out = {}
    for l in layers:
        y = prof.run_layer(qm, l, x, zero)
        out[l] = (prof.logits[l], prof.ids[l], prof.w[l], y.clone())
    torch.cuda.synchronize()
    return qm, out


def _host(dev, toks):
    t = torch.from_numpy(np.asarray(toks)).cuda()
    logits, ids, w, y = dev
    return dict(logits=logits[t].cpu().numpy(), ids=ids[t].cpu().numpy(), w=w[t].cpu().numpy(),
                y=y[t].float().cpu().numpy().astype(np.float64))


# the largest supported routing: E = 128 experts (router N = 128, all 512 TMEM columns), top-8, INT4 g64
MAXED = {"e128_k8": synth.MoEConfig("e128_k8", 2, 128, 128, 8, 128, 128, 4, 64, 0, 900, S + 33)}
ALL = {**SMALL, **EDGE, **MAXED}


@pytest.mark.parametrize("name", list(ALL))
def test_branch_parity_small(name):
    cfg = ALL[name]
    T = cfg.tokens
    _, dev = _gpu_branch(cfg, T, range(cfg.n_layers))
    toks = np.arange(T)
    for l in range(cfg.n_layers):
        ref = om.branch_tokens(cfg, toks, l)
        n_cmp, n_tie, worst = compare_branch(ref, _host(dev[l], toks))
        assert n_cmp >= 0.9 * T, (l, n_cmp, n_tie)


def _sample(T, n, seed):
    rng = np.random.default_rng(seed)
    fixed = [0, 1, 127, 128, 255, 256, T // 2, T - 2, T - 1]
    return np.unique(np.concatenate([fixed, rng.integers(0, T, n)]))


@pytest.mark.parametrize("path,T,n_sample", [("fused", 1024, None), ("pass", 24576, 160), ("auto", 24576, 96)])
def test_branch_parity_deepseek_layer(path, T, n_sample):
    """H 2048, F 1408, E 64, k 6, INT4 g128, no shared MLP.  'auto' = the library's own policy (the
    dequant pass + cp.async-gathered A rows at this token count, as in the bench)."""
    cfg = DS_ROUTED.with_(tokens=T)
    _, dev = _gpu_branch(cfg, T, [0], path=path)
    toks = np.arange(T) if n_sample is None else _sample(T, n_sample, cfg.seed)
    ref = om.branch_tokens(cfg, toks, 0)
    n_cmp, n_tie, worst = compare_branch(ref, _host(dev[0], toks))
    assert n_cmp >= 0.9 * len(toks)


def test_branch_detects_corrupted_group_scale():
    """One INT4 group scale of one routed expert's down projection multiplied by 1.1 (on the GPU only):
    the element-wise check must fail on the tokens of that expert."""
    cfg = DS_ROUTED
    T = cfg.tokens
    toks = np.arange(T)
    ref = om.branch_tokens(cfg, toks, 0)
    e = int(np.bincount(ref["ids"].ravel(), minlength=cfg.n_experts).argmax())
    h, grp = 5, 2

    def corrupt(qm):
        qm.down_s[0, e, h, grp] *= 1.1

    _, dev = _gpu_branch(cfg, T, [0], corrupt=corrupt)
    gpu = _host(dev[0], toks)
    with pytest.raises(AssertionError):
        compare_branch(ref, gpu)
    # ... at the north star's own tolerance, too, and only in output column h
    bad = branch_violations(gpu["y"], ref["y"], ref["cond"], ref["dmag"], tight=True)
    assert bad.any() and set(np.nonzero(bad)[1].tolist()) == {h}
    # and the uncorrupted run passes
    _, dev = _gpu_branch(cfg, T, [0])
    compare_branch(ref, _host(dev[0], toks))


@pytest.mark.parametrize("name", ["int4_shared", "int4_e64", "pass_tails_g64", "top1_int4", "hot_expert"])
def test_r1b_is_not_load_bearing(name):
    """Against SURVEY O4's literal ŵ = q·s (grouped weights NOT rounded to bf16), the MoE branch still
    meets the north star's 2e-2 per token (||Δy||_2 <= 2e-2·||y||_2 on the branch alone, no residual to
    hide behind): reading R1b does not decide pass/fail at the stated tolerance.  Element-wise, the
    exact-q·s oracle differs from any bf16-weight implementation by the bf16 rounding of every weight
    (2^-9 each, summed over a whole dot product), which exceeds the element-wise condition bound on a few
    cancelling elements: the element-wise contract is stated for R1b (tests above)."""
    cfg = ALL[name]
    assert cfg.group_size > 0
    T = cfg.tokens
    _, dev = _gpu_branch(cfg, T, range(cfg.n_layers))
    toks = np.arange(T)
    for l in range(cfg.n_layers):
        exact = om.branch_tokens(cfg, toks, l, exact_dequant=True)
        r1b = om.branch_tokens(cfg, toks, l)
        gpu = _host(dev[l], toks)
        same = np.array([set(a) == set(b) for a, b in zip(gpu["ids"], exact["ids"])])
        assert same.mean() >= 0.9
        err_exact = np.linalg.norm(gpu["y"] - exact["y"], axis=1) / np.linalg.norm(exact["y"], axis=1)
        err_r1b = np.linalg.norm(gpu["y"] - r1b["y"], axis=1) / np.linalg.norm(r1b["y"], axis=1)
        assert err_exact[same].max() <= 2e-2, (l, err_exact[same].max())
        assert np.median(err_r1b[same]) <= np.median(err_exact[same])  # R1b is the closer reading


@pytest.mark.parametrize("name,n_sample", [("deepseek_moe", 64), ("llama_moe", 64)])
def test_branch_parity_fullsize_layer0(name, n_sample):
    """Layer 0 of the BASELINE shapes at their full token counts (the bench's launch configuration:
    262,144 / 65,536 tokens in one call), zero residual, sampled tokens against the oracle."""
    full = synth.CONFIGS[name]
    cfg = full.with_(n_layers=1)  # layer 0's weights and router skew are those of the full model
    assert synth.router_skew_sigma(cfg, 0) == synth.router_skew_sigma(full, 0)
    T = full.tokens
    _, dev = _gpu_branch(cfg, T, [0])
    toks = _sample(T, n_sample, cfg.seed)
    ref = om.branch_tokens(cfg, toks, 0)
    n_cmp, _, _ = compare_branch(ref, _host(dev[0], toks))
    assert n_cmp >= 0.9 * len(toks)
