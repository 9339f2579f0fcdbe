"""Full-size parity of K7, the eq.(2) merge, in the launch configuration bench.py times:
ONE flux_merge_experts_batch launch over all L x 3 weight families of the DeepSeek-MoE-16B-shaped
model (BASELINE.json configs[3]: 64 -> 16 merged experts per layer, α = activation frequency, bf16).

The oracle (oracle.merge, fp64) is element-wise by definition, so it is evaluated on sampled output
indices only: the members' master values at those indices come from the CPU twin of the generator,
α from the ORACLE's own routing of a token sample (never from the CUDA path).  Samples cover every
output of every job uniformly plus its first / last element and chunk edges (16 KB = 8,192 bf16
elements per chunk); with 148 persistent CTAs each walking ~3,200 chunks, and slices packed four per
stage across chunk boundaries, they hit every part of every CTA's range and every slot position.  Variants: tuning experts
(cluster_of = -1), a cluster whose α are all zero (plain mean, R10), unbalanced clusters including
singletons (bit-exact identity), and per-layer budgets B(l) (eq.(1)).  Bound: |Δ| <= 2e-2·Σ_e w_e|W_e|
(condition-aware, bf16), and >= 99% of outputs equal to the correctly rounded fp64 value."""
import numpy as np
import pytest

import oracle
import oracle.model as om
import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

FAMS = ("gate", "up", "down")


def _alpha_from_oracle_routing(cfg, layer, n_tok=2048):
    """α = f = hist / T of layer `layer`'s router on x_0 of the first n_tok tokens (oracle O2/O3)."""
    x = synth.bf16_bits_to_f32(synth.cpu_rows(synth.spec_x(cfg), np.arange(n_tok))).astype(np.float64)
    wr = om.master_f32(synth.spec_router(cfg, layer)).astype(np.float64)
    _, ids, _, _ = oracle.router(x, wr, cfg.top_k, cfg.norm_topk)
    hist, *_ = oracle.permute(ids, cfg.n_experts)
    return (hist / float(n_tok)).astype(np.float32)


def _variant_clusters(cfg, variant, layer, rng):
    E = cfg.n_experts
    if variant in ("balanced", "zero_alpha"):
        return synth.cluster_assignment(cfg, 16)[layer].copy(), 16
    if variant == "tuning":
        return synth.cluster_assignment(cfg, 16, n_tuning=8)[layer].copy(), 16
    if variant == "unbalanced":  # sizes 1, 1, 2, 3, ... (a random partition with singletons)
        sizes = [1, 1, 2, 3, 5, 8, 13, 31]
        perm = rng.permutation(E)
        co = np.empty(E, np.int32)
        i = 0
        for c, n in enumerate(sizes):
            co[perm[i:i + n]] = c
            i += n
        return co, len(sizes)
    if variant == "budget":  # per-layer C_l from eq.(1) (oracle) on the oracle's own per-layer counts
        return None, None
    raise ValueError(variant)


def _sample_indices(numel, n, rng):
    chunk = 8192  # bf16 elements per 16 KB chunk (merge.cu kSlice)
    edges = [0, 1, 7, 8, chunk - 1, chunk, chunk + 1, 148 * chunk % numel, numel // 2, numel - 8, numel - 1]
    return np.unique(np.concatenate([edges, rng.integers(0, numel, n)]).astype(np.int64))


def _member_values(cfg, layer, fam, experts, idx):
    """master values W_e[idx] (fp32-exact bf16) of the given experts, shape [len(experts)][len(idx)]."""
    spec0 = synth.spec_expert(cfg, layer, 0, fam)
    rows, cols = np.divmod(idx, spec0.cols)
    urows, inv = np.unique(rows, return_inverse=True)
    out = np.empty((len(experts), len(idx)))
    for i, e in enumerate(experts):
        R = synth.bf16_bits_to_f32(synth.cpu_rows(synth.spec_expert(cfg, layer, e, fam), urows))
        out[i] = R[inv, cols]
    return out


@pytest.fixture(scope="module")
def model():
    from paper_2508_19078_b200 import synthetic
    cfg = synth.CONFIGS["deepseek_moe"]
    return cfg, synthetic.master_weights(cfg)


@pytest.mark.parametrize("variant", ["balanced", "tuning", "zero_alpha", "unbalanced", "budget"])
def test_merge_fullsize_batch_parity(model, variant):
    from paper_2508_19078_b200.driver import merge_model
    cfg, masters = model
    L, E = cfg.n_layers, cfg.n_experts
    rng = np.random.default_rng(abs(hash(variant)) % 2**32)
    layers = list(range(L))
    check_layers = [0, 1, L // 2, L - 1]
    alpha = np.zeros((L, E), np.float32)
    for l in check_layers:
        alpha[l] = _alpha_from_oracle_routing(cfg, l)
    for l in layers:
        if l not in check_layers:
            alpha[l] = alpha[check_layers[l % len(check_layers)]]
    cluster_of = np.empty((L, E), np.int32)
    Cl = np.empty(L, np.int32)
    if variant == "budget":
        hist = np.rint(alpha.astype(np.float64) * 2048).astype(np.int64)
        Cl, *_ = oracle.layer_budget(hist, 2048, 16 * L)
        for l in layers:  # a seeded balanced partition into C_l clusters
            perm = np.random.default_rng(cfg.seed + l).permutation(E)
            cluster_of[l, perm] = np.arange(E) % Cl[l]
    else:
        for l in layers:
            cluster_of[l], Cl[l] = _variant_clusters(cfg, variant, l, rng)
    if variant == "zero_alpha":
        for l in layers:
            alpha[l, cluster_of[l] == 3] = 0.0
    n_clusters = Cl.tolist() if variant == "budget" else int(Cl[0])
    merged = merge_model(masters, torch.from_numpy(alpha).cuda(), torch.from_numpy(cluster_of).cuda(), n_clusters)
    torch.cuda.synchronize()

    for l in check_layers:
        C = int(Cl[l])
        remap_ref = None
        for fam in FAMS:
            out = getattr(merged, fam)[l]
            numel = out[0].numel()
            idx = _sample_indices(numel, 384, rng)
            t_idx = torch.from_numpy(idx).cuda()
            got = out.view(out.shape[0], -1)[:C][:, t_idx].float().cpu().numpy().astype(np.float64)
            vals = _member_values(cfg, l, fam, range(E), idx)  # [E][n]
            ref, remap_ref = oracle.merge(vals, cluster_of[l], alpha[l].astype(np.float64), C)
            absw = np.zeros_like(ref)
            for c in range(C):
                mem = np.nonzero(cluster_of[l] == c)[0]
                a = alpha[l, mem].astype(np.float64)
                w = a / a.sum() if a.sum() > 0 else np.full(len(mem), 1.0 / len(mem))
                absw[c] = (w[:, None] * np.abs(vals[mem])).sum(0)
                if len(mem) == 1:  # singleton: the input bit for bit
                    assert np.array_equal(got[c], vals[mem[0]]), (variant, l, fam, c)
            assert np.all(np.abs(got - ref) <= 2e-2 * absw), (variant, l, fam)
            assert np.mean(got == oracle.bf16_round(ref)) > 0.99, (variant, l, fam)
        assert np.array_equal(merged.remap[l].cpu().numpy(), remap_ref), (variant, l)


def test_merge_batch_equals_single_calls(model):
    """The batched launch is bit-identical to one flux_merge_experts call per (layer, family)."""
    import paper_2508_19078_b200 as F
    from paper_2508_19078_b200.driver import merge_model
    cfg, masters = model
    L, E = 3, cfg.n_experts
    co = torch.from_numpy(synth.cluster_assignment(cfg, 16, n_tuning=4)[:L].copy()).cuda()
    alpha = torch.rand(cfg.n_layers, E, device="cuda")
    merged = merge_model(masters, alpha, torch.cat([co, co.new_zeros(cfg.n_layers - L, E)]), 16)
    for l in range(L):
        for fam in FAMS:
            src = getattr(masters, fam)[l].view(E, -1)
            one = torch.empty(16, src.shape[1], dtype=src.dtype, device="cuda")
            rm = torch.empty(E, dtype=torch.int32, device="cuda")
            F.merge_experts(src, co[l], alpha[l], 16, one, rm)
            assert torch.equal(one, getattr(merged, fam)[l].view(16, -1)), (l, fam)
            assert torch.equal(rm, merged.remap[l])
