"""GPU parity for NEXT-1, similarity-based expert clustering (§5.2): the CUDA path
(flux_expert_features, flux_cluster_experts through the C ABI) against oracle/cluster.py on the same
seeded inputs.  Inputs reach the oracle from numpy / the CPU generator twin only.

Tolerances (R12/R13): the Gram matrix accumulates bf16 products in fp32 on the tensor cores
(split-K partials summed in fp64), so |ΔG| <= 1e-4·max diag; eigenvalues and the sign-invariant score
Gram F·Fᵀ then agree to 1e-3 relative where the spectrum is separated.  K-Means runs in fp64 on both
sides from the same fp32 features, so assignments must be identical."""
import numpy as np
import pytest

import oracle.cluster as oc
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _bf16(a):
    """numpy fp32 -> (torch bf16 on cuda, the same values as fp64 numpy)."""
    t = torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16)
    return t.cuda(), t.float().numpy().astype(np.float64)


def _planted_families(rng, E, C, sizes, noise=0.3, spread=None):
    """One layer: E experts drawn around C prototypes; families of the given per-expert sizes."""
    P = sum(sizes)
    scale = np.linspace(2.0, 0.5, C) if spread is None else spread
    protos = rng.standard_normal((C, P)) * scale[:, None]
    labels = rng.permutation(np.arange(E) % C)
    X = protos[labels] + noise * rng.standard_normal((E, P))
    out, o = [], 0
    for n in sizes:
        out.append(X[:, o:o + n])
        o += n
    return out, labels


def _score_gram(F):
    return F @ F.T


@pytest.mark.parametrize("E,sizes,d", [(16, [4096, 1000, 8], 8), (64, [20000, 7704], 16), (7, [640], 6),
                                       (64, [64 * 148 * 3 + 72], 16), (128, [12000, 3000, 800, 64], 24),
                                       (100, [9000], 32), (33, [4096 * 40 + 8], 12),
                                       (32, [64 * 400], 12), (20, [64 * 202 + 8], 8), (24, [64 * 301, 64 * 99], 8),
                                       (16, [64 * 400], 8), (12, [64 * 100, 64 * 100], 6)])
def test_gram_features_vs_oracle(E, sizes, d):
    import paper_2508_19078_b200 as F
    rng = np.random.default_rng(100 + E + len(sizes))
    L = 2
    fams_t, G_ref, feats_ref, lam_ref = [], [], [], []
    for _ in range(L):
        fams, _ = _planted_families(rng, E, max(2, E // 4), sizes)
        pairs = [_bf16(f) for f in fams]
        fams_t.append([p[0] for p in pairs])
        G = oc.gram([p[1] for p in pairs])
        G_ref.append(G)
        f_ref, lam = oc.pca_features(G, d)
        feats_ref.append(f_ref)
        lam_ref.append(lam)
    feats = torch.empty(L, E, d, dtype=torch.float32, device="cuda")
    gram = torch.empty(L, E, E, dtype=torch.float32, device="cuda")
    eig = torch.empty(L, d, dtype=torch.float32, device="cuda")
    F.expert_features(fams_t, d, feats, gram, eig)
    torch.cuda.synchronize()
    for l in range(L):
        g = gram[l].double().cpu().numpy()
        scale = np.abs(np.diag(G_ref[l])).max()
        assert np.abs(g - G_ref[l]).max() <= 1e-4 * scale, l
        lam = eig[l].double().cpu().numpy()
        assert np.allclose(lam, lam_ref[l], rtol=1e-3, atol=1e-5 * lam_ref[l][0]), (lam, lam_ref[l])
        f = feats[l].double().cpu().numpy()
        S, S_ref = _score_gram(f), _score_gram(feats_ref[l])
        assert np.abs(S - S_ref).max() <= 1e-3 * np.abs(S_ref).max(), l
        assert np.allclose(f.sum(0), 0, atol=1e-3 * np.abs(f).max())  # scores of centred data


def test_features_deterministic():
    import paper_2508_19078_b200 as F
    rng = np.random.default_rng(7)
    fams, _ = _planted_families(rng, 64, 8, [30000, 10000])
    t = [[_bf16(f)[0] for f in fams]]
    outs = []
    for _ in range(2):
        feats = torch.empty(1, 64, 16, dtype=torch.float32, device="cuda")
        F.expert_features(t, 16, feats)
        outs.append(feats.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("seed", range(10))
def test_kmeans_vs_oracle(seed):
    import paper_2508_19078_b200 as F
    rng = np.random.default_rng(seed)
    L, E = int(rng.integers(1, 9)), int(rng.choice([5, 16, 37, 64, 100, 128]))
    d = int(rng.integers(1, min(E, 32) + 1))
    feats = rng.standard_normal((L, E, d)).astype(np.float32)
    counts = rng.integers(0, 50, size=(L, E)).astype(np.int64)  # small range: frequency ties occur
    tuning = rng.random((L, E)) < (0.25 if seed % 2 else 0.0)
    n_non = E - tuning.sum(1)
    tuning[n_non == 0, 0] = False
    n_non = E - tuning.sum(1)
    B = np.array([int(rng.integers(1, n + 1)) for n in n_non], np.int32)
    got = F.cluster_experts(torch.from_numpy(feats).cuda(), torch.from_numpy(counts).cuda(), B,
                            tuning if tuning.any() else None, max_iter=40)
    want, _ = oc.fused_kmeans(feats.astype(np.float64), B, tuning, counts.astype(np.float64), max_iter=40)
    assert np.array_equal(got.cpu().numpy(), want)


def test_planted_end_to_end():
    """Weights planted around prototypes: GPU features -> GPU K-Means recovers the planted partition, and
    equals the oracle pipeline on the same bf16 values."""
    import paper_2508_19078_b200 as F
    rng = np.random.default_rng(11)
    L, E, C = 3, 64, 16
    sizes = [2 * 128 * 64, 128 * 64]
    fams_t, labels, feats_ref = [], [], []
    counts = rng.integers(1000, 5000, size=(L, E)).astype(np.int64)
    for l in range(L):
        fams, lab = _planted_families(rng, E, C, sizes, noise=0.05, spread=np.ones(C))
        pairs = [_bf16(f) for f in fams]
        fams_t.append([p[0] for p in pairs])
        labels.append(lab)
        feats_ref.append(oc.pca_features(oc.gram([p[1] for p in pairs]), 15)[0])
        for c in range(C):  # one expert of each planted cluster is the most frequent (R13 init)
            counts[l, np.nonzero(lab == c)[0][0]] += 100000
    feats = torch.empty(L, E, 15, dtype=torch.float32, device="cuda")
    F.expert_features(fams_t, 15, feats)
    got = F.cluster_experts(feats, torch.from_numpy(counts).cuda(), [C] * L).cpu().numpy()
    want, _ = oc.fused_kmeans(np.stack(feats_ref), [C] * L, np.zeros((L, E), bool), counts.astype(np.float64))
    for l in range(L):
        same = got[l][:, None] == got[l][None, :]
        assert np.array_equal(same, labels[l][:, None] == labels[l][None, :]), l
        assert np.array_equal(same, want[l][:, None] == want[l][None, :]), l


def test_fullsize_deepseek_layer_features():
    """DeepSeek-MoE shape (E=64, 3 families of 1408x2048): layer-0 features of the synthetic master weights
    against the oracle Gram built from the CPU generator twin, column chunk by column chunk."""
    import paper_2508_19078_b200 as F
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import expert_features_model
    cfg = synth.CONFIGS["deepseek_moe"].with_(n_layers=1)
    masters = synthetic.master_weights(cfg)
    feats, gram, eig = expert_features_model(masters, 16, with_gram=True)
    torch.cuda.synchronize()
    E = cfg.n_experts
    G = np.zeros((E, E))
    for fam in ("gate", "up", "down"):
        rows = synth.spec_expert(cfg, 0, 0, fam).rows
        for r0 in range(0, rows, 128):
            n = min(128, rows - r0)
            X = np.stack([synth.bf16_bits_to_f32(synth.cpu_matrix(synth.spec_expert(cfg, 0, e, fam), r0, n))
                          .reshape(-1) for e in range(E)]).astype(np.float64)
            G += X @ X.T
    g = gram[0].double().cpu().numpy()
    err = np.abs(g - G)
    i, j = np.unravel_index(np.argmax(err), err.shape)
    assert err.max() <= 1e-4 * np.abs(np.diag(G)).max(), (err.max(), i, j, g[i, j], G[i, j], np.diag(G)[:4])
    f_ref, lam_ref = oc.pca_features(G, 16)
    lam = eig[0].double().cpu().numpy()
    # i.i.d. synthetic experts: a flat spectrum, so compare the subspace-free quantities only
    assert np.allclose(lam, lam_ref, rtol=2e-3)
    f = feats[0].double().cpu().numpy()
    assert np.allclose(np.linalg.norm(f, axis=0), np.sqrt(lam_ref), rtol=2e-3)
    del masters
