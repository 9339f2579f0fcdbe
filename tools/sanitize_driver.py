"""Small workload that calls every libflux entry point once (run under compute-sanitizer by
tools/sanitize.sh): quantize (INT8/INT4/INT2), the profile pass on every GEMM path (flux_policy: in-GEMM
dequant, dequant pass with the in-GEMM cp.async gather, materialised x_perm, TMA gather4, fused combine,
static tiles, chained gate/up + down), features + K-Means, merge, compact model forward with gate re-routing, attention histogram,
output error.  Sizes are tiny: the sanitizers replay every memory access."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_19078_b200 as F  # noqa: E402
import synth  # noqa: E402
from paper_2508_19078_b200 import synthetic  # noqa: E402
from paper_2508_19078_b200.driver import (ModelShape, Profiler, QuantizedModel, cluster_model,  # noqa: E402
                                          compact_model, dense_model, expert_features_model, merge_model)

# flux_policy (weight_path, routed_rows, fused_combine, static_tiles)
PATHS = [(2, 0, 0, 0), (1, 0, 0, 0), (1, 1, 0, 0), (1, 2, 0, 0), (1, 0, 1, 0), (1, 0, 0, 1), (1, 0, 0, 0, 0, 2)]


def run(cfg, paths):
    shape = ModelShape.of(cfg)
    masters = synthetic.master_weights(cfg)
    x = synthetic.tokens(cfg, 0, cfg.tokens)
    # plain quantizer + per-call dequantization, then the quantizer that also writes the bf16 operands
    for with_bops in (False, True):
        qm = QuantizedModel(shape, with_bops=with_bops)
        qm.quantize_from(masters)
        for pol in paths:
            prof = Profiler(shape, cfg.tokens, with_de=True, with_logits=True, policy=F.make_policy(*pol))
            prof.run(qm, x)
            torch.cuda.synchronize()
    return masters, prof


def main():
    small = synth.MoEConfig("san_int4_shared", 2, 128, 8, 2, 128, 256, 4, 64, 0, 300, synth.BASE_SEED + 31)
    run(synth.CONFIGS["toy"], PATHS)                                                       # INT8 per channel
    masters, prof = run(small, PATHS)                                                      # INT4 g64 + shared
    run(synth.MoEConfig("san_int2", 1, 128, 8, 2, 64, 0, 2, 64, 1, 200, synth.BASE_SEED + 32), PATHS[-2:])
    cfg = small
    L, E = cfg.n_layers, cfg.n_experts
    feats, _, _ = expert_features_model(masters, 4)                                       # Gram + eig
    cl = cluster_model(feats, prof.hist, 3)                                               # K-Means
    alpha = torch.rand(L, E, device="cuda")
    merge_model(masters, alpha, cl, 3)                                                    # eq.(2)
    co = torch.from_numpy(synth.cluster_assignment(cfg, 3, 2)).cuda()
    cm = compact_model(masters, alpha, co, 3, 2)                                          # compact + re-routing
    p2 = Profiler(cm.shape, cfg.tokens)
    x = synthetic.tokens(cfg, 0, cfg.tokens)
    y_c = p2.run(cm, x)
    dm = dense_model(masters)
    p3 = Profiler(dm.shape, cfg.tokens)
    y_d = p3.run(dm, x)
    if y_c is not None and y_d is not None:
        F.output_error(y_c, y_d)
    ids = prof.ids[0].contiguous()
    attn = torch.rand(cfg.tokens, device="cuda")
    out = torch.zeros(E, dtype=torch.int64, device="cuda")
    F.attention_hist(ids, attn, E, out)
    torch.cuda.synchronize()
    print("sanitize driver: ok")


if __name__ == "__main__":
    main()
