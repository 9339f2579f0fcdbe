"""oracle.cluster — similarity-based expert clustering, §5.2 of the paper.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  numpy fp64; every step is
the paper's, in its order; library primitives: a matmul and a symmetric
eigendecomposition.

C1  features: "reduces the dimensionality of expert parameters
    using ... Principal Component Analysis".  Expert e of a layer is the vector
    of all its parameters (gate | up | down, flattened).  PCA over the E experts
    of the layer: centre the vectors over experts, take the top-d principal
    components; an expert's feature vector is its d PCA scores.  Computed through
    the E x E Gram matrix of the centred vectors, G_c = X_c X_cᵀ = V Λ Vᵀ, whose
    top-d eigenpairs give the scores F = V_d Λ_d^(1/2) (the dual form of PCA;
    pinned against an SVD-based PCA in tests).  d: reading R12.
C2  fused K-Means, reading R13:
    * ΣB(l) centroids, each labelled with its layer;
    * distance(expert of layer l, centroid of layer l') = 1 - cos(f, μ) if l' = l,
      else +inf — the paper's "set to 0" would pull every expert to a
      foreign layer, contradicting "to enforce layer-specific clustering", so it
      is read as the masking value that excludes foreign centroids;
    * init: the B(l) non-tuning experts of layer l with the highest activation
      frequency (ties: lower id), in that order;
    * assignment: argmin distance, ties -> lower centroid index (layer-major order);
    * update: μ = mean of the assigned feature vectors (unchanged if empty);
    * stop: no assignment changed, or max_iter iterations.
    Tuning experts are not clustered (cluster_of = -1).
"""
from __future__ import annotations

import numpy as np


def gram(families) -> np.ndarray:
    """Raw Gram matrix Σ_f X_f X_fᵀ of one layer's experts (families: list of [E][P_f] arrays)."""
    G = None
    for X in families:
        X = np.asarray(X, dtype=np.float64)
        g = X @ X.T
        G = g if G is None else G + g
    return G


def center_gram(G: np.ndarray) -> np.ndarray:
    """Gram matrix of the vectors centred over experts: H G H, H = I - 11ᵀ/E."""
    E = G.shape[0]
    Hm = np.eye(E) - np.full((E, E), 1.0 / E)
    return Hm @ G @ Hm


def pca_features(G_raw: np.ndarray, d: int) -> tuple[np.ndarray, np.ndarray]:
    """C1: top-d PCA scores of the E experts from their raw Gram matrix -> (features [E][d], eigenvalues [d])."""
    w, V = np.linalg.eigh(center_gram(G_raw))
    order = np.argsort(-w, kind="stable")[:d]
    lam = np.maximum(w[order], 0.0)
    return V[:, order] * np.sqrt(lam)[None, :], lam


def _cos_dist(f: np.ndarray, mu: np.ndarray) -> float:
    nf, nm = np.linalg.norm(f), np.linalg.norm(mu)
    if nf == 0.0 or nm == 0.0:
        return 1.0
    return 1.0 - float(f @ mu) / (nf * nm)


def fused_kmeans(features, n_clusters, tuning, freq, max_iter: int = 50):
    """C2 over all layers at once.  features [L][E][d]; n_clusters [L]; tuning [L][E] bool; freq [L][E].
    Returns (cluster_of [L][E] int32 with -1 for tuning experts, iterations run)."""
    F = np.asarray(features, dtype=np.float64)
    L, E, d = F.shape
    tuning = np.asarray(tuning, dtype=bool)
    # centroid table: (layer label, vector), layer-major
    cent_layer, cent = [], []
    for l in range(L):
        cand = [e for e in sorted(range(E), key=lambda e: (-freq[l][e], e)) if not tuning[l][e]]
        for c in range(n_clusters[l]):
            cent_layer.append(l)
            cent.append(F[l, cand[c]].copy())
    cent_layer = np.asarray(cent_layer)
    cent = np.asarray(cent)
    n_cent = len(cent)
    assign = np.full((L, E), -1, dtype=np.int64)  # global centroid index
    it = 0
    for it in range(1, max_iter + 1):
        new = np.full((L, E), -1, dtype=np.int64)
        for l in range(L):
            for e in range(E):
                if tuning[l][e]:
                    continue
                best, best_d = -1, np.inf
                for c in range(n_cent):
                    dist = _cos_dist(F[l, e], cent[c]) if cent_layer[c] == l else np.inf
                    if dist < best_d:
                        best, best_d = c, dist
                new[l, e] = best
        changed = not np.array_equal(new, assign)
        assign = new
        for c in range(n_cent):
            l = cent_layer[c]
            members = [e for e in range(E) if assign[l, e] == c]
            if members:
                cent[c] = F[l, members].mean(axis=0)
        if not changed:
            break
    # global centroid index -> index within its layer
    first = {l: int(np.nonzero(cent_layer == l)[0][0]) for l in range(L) if np.any(cent_layer == l)}
    out = np.full((L, E), -1, dtype=np.int32)
    for l in range(L):
        for e in range(E):
            if assign[l, e] >= 0:
                out[l, e] = assign[l, e] - first[l]
    return out, it
