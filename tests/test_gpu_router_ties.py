"""K1's top-k on exact ties and near-ties (reading R2: the k largest logits in descending order, the
lower expert index first on equal logits), decided in the kernel's own precision: the GPU's fp32
logits (flux_layer_out.router_logits) are re-selected on the host with the definition written out,
and the GPU's ids must equal that selection on EVERY token — including tokens whose top-k
boundary is an exact tie (duplicated router rows give bit-identical logit columns), a near-tie a
few ulps wide (router rows one bf16 ulp apart in one element), logits of ±0 (all-zero router rows)
and expert counts below the kernel's column padding (E = 12, 40).  The weights are checked against the
same definition, w = exp(z_j − max z) / Σ_e exp(z_e − max z) (norm 0) in fp64, at 1e-5 relative
(fp32 evaluation of a 64-term sum).

The kernel selects with truncated integer keys and redoes a row exactly when two of its k+1
largest keys collide (router.cu); these inputs put a large share of the rows on that fallback and
the rest on the fast path, so both are compared."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _topk_r2(z: np.ndarray, k: int) -> np.ndarray:
    """Reading R2 literally: k passes of 'largest remaining, lowest index on ties' over fp32 values."""
    T, E = z.shape
    out = np.empty((T, k), np.int64)
    for t in range(T):
        rem = list(range(E))
        for j in range(k):
            best = rem[0]
            for e in rem[1:]:
                if z[t, e] > z[t, best]:
                    best = e
            out[t, j] = best
            rem.remove(best)
    return out


def _tie_router(wr: torch.Tensor, rng: np.random.Generator) -> torch.Tensor:
    """wr [E][H] bf16 -> rows with exact duplicates, one-ulp near duplicates and zero rows."""
    w = wr.clone()
    E = w.shape[0]
    perm = rng.permutation(E)
    n = max(E // 4, 1)
    for i in range(n):  # exact duplicates: identical logit columns
        w[perm[i]] = w[perm[n + i]]
    for i in range(n):  # near duplicates: one element one bf16 ulp up
        a, b = perm[2 * n + i] if 2 * n + i < E else perm[0], perm[i]
        w[a] = w[b]
        h = int(rng.integers(0, w.shape[1]))
        w[a].view(torch.int16)[h] += 1
    if E >= 8:  # two all-zero rows: logits +0 (or -0)
        w[perm[-1]] = 0
        w[perm[-2]] = 0
    return w


@pytest.mark.parametrize("E,k", [(64, 6), (16, 2), (12, 3), (40, 8), (8, 8)])
def test_router_topk_ties_exact(E, k):
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import ModelShape, Profiler, QuantizedModel
    cfg = synth.MoEConfig(f"ties_E{E}_k{k}", 1, 256, E, k, 128, 0, 8, 0, 0, 1000, synth.BASE_SEED + 60 + E + k)
    shape = ModelShape.of(cfg)
    qm = QuantizedModel(shape)
    qm.quantize_from(synthetic.master_weights(cfg))
    rng = np.random.default_rng(E * 31 + k)
    qm.router[0] = _tie_router(qm.router[0], rng)
    x = synthetic.tokens(cfg, 0, cfg.tokens)
    x[:16] = 0  # all-zero tokens: every logit +0, the selection is experts 0..k-1
    prof = Profiler(shape, cfg.tokens, with_logits=True)
    prof.run(qm, x)
    torch.cuda.synchronize()
    z = prof.logits[0].cpu().numpy()
    ids = prof.ids[0].cpu().numpy()
    w = prof.w[0].cpu().numpy()
    ref = _topk_r2(z, k)
    assert np.array_equal(ids, ref), np.argwhere((ids != ref).any(1))[:10].ravel()
    assert np.array_equal(ids[:16], np.tile(np.arange(k), (16, 1)))
    # the inputs really contain boundary ties: some token's k-th and (k+1)-th logits are equal
    if k < E:
        zs = -np.sort(-z, axis=1)
        assert (zs[16:, k - 1] == zs[16:, k]).sum() >= 1
    zd = z.astype(np.float64)
    p = np.exp(zd - zd.max(1, keepdims=True))
    p /= p.sum(1, keepdims=True)
    wref = np.take_along_axis(p, ref, 1)
    assert np.allclose(w, wref, rtol=1e-5, atol=1e-9), np.abs(w - wref).max()
    hist = prof.hist[0].cpu().numpy()
    assert np.array_equal(hist, np.bincount(ids.ravel(), minlength=E))
