"""Full-size parity at BASELINE.json's sizes, in the launch configuration bench.py
times (one flux_profile_layer call per layer over all tokens of one GPU).

* sampled tokens (tile edges, the ragged end, random ones) are followed by the
  oracle through EVERY layer, free-running from the generated x_0 (the oracle
  never sees a GPU value) and compared per layer with the parity contract;
* properties that hold at any size are checked on every token of every layer:
  hist == bincount(ids), Σ hist = T·k, distinct experts per token, and the
  D_e CSR is exactly the stable grouping of the GPU's own routing;
* the residual stream stays finite and O(1) (the synthetic recipe is sane).
"""
import numpy as np
import pytest

import oracle.model as om
import synth

from _parity import check_hist_and_de, compare_layer, input_bound

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _sample(T, n_rand, seed):
    rng = np.random.default_rng(seed)
    fixed = [0, 1, 127, 128, 129, T // 2, T - 129, T - 2, T - 1]
    return np.unique(np.concatenate([fixed, rng.integers(0, T, n_rand)]))


@pytest.mark.parametrize("name,n_rand", [("deepseek_moe", 23), ("llama_moe", 23)])
def test_fullsize_sampled_parity(name, n_rand):
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import ModelShape, Profiler, QuantizedModel
    cfg = synth.CONFIGS[name]
    T = cfg.tokens
    shape = ModelShape.of(cfg)
    masters = synthetic.master_weights(cfg)
    qm = QuantizedModel(shape)
    qm.quantize_from(masters)
    del masters
    torch.cuda.empty_cache()
    prof = Profiler(shape, T, with_de=True, with_logits=True)
    samp = _sample(T, n_rand, cfg.seed)
    samp_t = torch.from_numpy(samp).cuda()
    ys = []
    rms = []

    def on_layer(l, y):
        ys.append(y[samp_t].float().cpu().numpy())
        rms.append(float(y[:, 1:].float().pow(2).mean().sqrt()))

    prof.run(qm, synthetic.tokens(cfg, 0, T), on_layer=on_layer)
    torch.cuda.synchronize()
    assert all(np.isfinite(rms)) and max(rms) < 4.0, rms

    ref = om.profile_tokens(cfg, samp)
    alive = np.ones(len(samp), bool)
    for l in range(cfg.n_layers):
        ids = prof.ids[l].cpu().numpy()
        check_hist_and_de(ids, prof.hist[l].cpu().numpy(), prof.offsets[l].cpu().numpy(),
                          prof.token_index[l].cpu().numpy(), cfg.n_experts)
        gpu = dict(logits=prof.logits[l][samp_t].cpu().numpy(), ids=ids[samp], w=prof.w[l][samp_t].cpu().numpy(),
                   y=ys[l])
        wr = om.master_f32(synth.spec_router(cfg, l))
        dz = input_bound(ys[l - 1] if l else None, ref[l]["x"], wr)
        compare_layer(l, ref[l], gpu, alive, dz)
    # a token stops being compared after a (validated) near-tie divergence; over 28-32 free-running
    # layers a minority diverge, the rest are still compared at the last layer
    assert alive.mean() >= 0.4, alive
