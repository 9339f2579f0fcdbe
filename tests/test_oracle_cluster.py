"""Pins for the clustering oracle (§5.2) — CPU only.

* C1 (PCA features through the dual Gram form) against scikit-learn's SVD-based
  PCA on the same vectors (an independent formulation), plus the zero-mean and
  family-concatenation properties;
* C2 (fused, layer-masked K-Means) against an independently written per-layer
  Lloyd iteration (masking cross-layer distances must decouple the layers), a
  planted-cluster recovery case, the Lloyd fixed-point property, tuning-expert
  exclusion and the singleton case.
"""
import numpy as np
import pytest

import oracle.cluster as oc


def _planted(rng, L, E, C, d_raw=200, noise=0.05):
    """L layers of E experts as C well-separated prototypes + small noise; returns (vectors, labels)."""
    X, lab = [], []
    for _ in range(L):
        protos = rng.standard_normal((C, d_raw))
        labels = rng.permutation(np.arange(E) % C)
        X.append(protos[labels] + noise * rng.standard_normal((E, d_raw)))
        lab.append(labels)
    return np.stack(X), np.stack(lab)


def test_pca_features_match_svd_pca():
    sk = pytest.importorskip("sklearn.decomposition")
    rng = np.random.default_rng(0)
    X = rng.standard_normal((24, 300)) @ np.diag(np.linspace(3, 0.1, 300))
    F, lam = oc.pca_features(oc.gram([X]), 6)
    ref = sk.PCA(n_components=6, svd_solver="full").fit_transform(X)
    for j in range(6):  # each component is defined up to sign
        s = np.sign(F[:, j] @ ref[:, j])
        assert np.allclose(F[:, j] * s, ref[:, j], atol=1e-8 * np.abs(ref).max())
    assert np.allclose(F.sum(0), 0, atol=1e-9 * np.abs(F).max())  # scores of centred data
    assert np.all(np.diff(lam) <= 0)


def test_gram_over_families_is_gram_of_concatenation():
    rng = np.random.default_rng(1)
    A, B, C = (rng.standard_normal((10, n)) for n in (7, 13, 5))
    assert np.allclose(oc.gram([A, B, C]), oc.gram([np.concatenate([A, B, C], 1)]))


def _kmeans_layer(F, B, tuning, freq, max_iter):
    """Independent per-layer Lloyd iteration (cosine distance, same init/tie rules as R13)."""
    E = F.shape[0]
    cand = [e for e in sorted(range(E), key=lambda e: (-freq[e], e)) if not tuning[e]]
    mu = F[cand[:B]].copy()
    assign = None

    def cosd(a, b):
        na, nb = np.linalg.norm(a), np.linalg.norm(b)
        return 1.0 if na == 0 or nb == 0 else 1.0 - a @ b / (na * nb)

    for _ in range(max_iter):
        new = np.array([-1 if tuning[e] else int(np.argmin([cosd(F[e], m) for m in mu])) for e in range(E)])
        done = assign is not None and np.array_equal(new, assign)
        assign = new
        for c in range(B):
            if np.any(assign == c):
                mu[c] = F[assign == c].mean(0)
        if done:
            break
    return assign


def test_fused_equals_independent_layers():
    rng = np.random.default_rng(2)
    L, E = 4, 16
    feats = rng.standard_normal((L, E, 5))
    B = [3, 5, 2, 4]
    tuning = rng.random((L, E)) < 0.2
    freq = rng.random((L, E))
    got, _ = oc.fused_kmeans(feats, B, tuning, freq, max_iter=30)
    for l in range(L):
        want = _kmeans_layer(feats[l], B[l], tuning[l], freq[l], 30)
        assert np.array_equal(got[l], want), l


def test_planted_clusters_recovered_through_pca():
    rng = np.random.default_rng(3)
    L, E, C = 3, 24, 4
    X, lab = _planted(rng, L, E, C)
    feats = np.stack([oc.pca_features(oc.gram([X[l]]), 8)[0] for l in range(L)])
    freq = rng.random((L, E))
    for l in range(L):  # the most frequent expert of each planted cluster leads the init (R13)
        for c in range(C):
            freq[l, np.nonzero(lab[l] == c)[0][0]] += 10.0
    got, _ = oc.fused_kmeans(feats, [C] * L, np.zeros((L, E), bool), freq, max_iter=50)
    for l in range(L):
        # same partition up to relabelling: pairs are together iff planted together
        same_got = got[l][:, None] == got[l][None, :]
        same_lab = lab[l][:, None] == lab[l][None, :]
        assert np.array_equal(same_got, same_lab)


def test_fixed_point_tuning_and_singletons():
    rng = np.random.default_rng(4)
    L, E = 2, 12
    feats = rng.standard_normal((L, E, 4))
    tuning = np.zeros((L, E), bool)
    tuning[0, [1, 5]] = True
    freq = rng.random((L, E))
    got, _ = oc.fused_kmeans(feats, [3, 4], tuning, freq, max_iter=100)
    assert np.all(got[0, [1, 5]] == -1) and np.all(got[0, ~tuning[0]] >= 0)
    for l, B in ((0, 3), (1, 4)):
        mask = got[l] >= 0
        mus = np.stack([feats[l][got[l] == c].mean(0) for c in range(B)])
        for e in np.nonzero(mask)[0]:
            d = [1 - feats[l, e] @ m / np.linalg.norm(feats[l, e]) / np.linalg.norm(m) for m in mus]
            assert got[l, e] == int(np.argmin(d))  # Lloyd fixed point: every expert at its nearest centroid
    # B = number of non-tuning experts: every expert its own cluster
    got, _ = oc.fused_kmeans(feats[:1], [E - 2], tuning[:1], freq[:1])
    assert sorted(got[0][got[0] >= 0]) == list(range(E - 2))
