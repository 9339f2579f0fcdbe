"""Per-layer GPU-vs-oracle error report (diagnostic; not a test).

usage: python tools/parity_report.py [config-name ...]
Prints, per layer: tokens compared, near-ties, routing divergences, max/median
relative logit error, max/median relative output error.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import oracle.model as om  # noqa: E402
import synth  # noqa: E402
from paper_2508_19078_b200 import synthetic  # noqa: E402
from paper_2508_19078_b200.driver import ModelShape, Profiler, QuantizedModel  # noqa: E402
from test_gpu_parity import SMALL  # noqa: E402


def report(cfg):
    shape = ModelShape.of(cfg)
    qm = QuantizedModel(shape)
    qm.quantize_from(synthetic.master_weights(cfg))
    prof = Profiler(shape, cfg.tokens, with_logits=True)
    ys = []
    prof.run(qm, synthetic.tokens(cfg, 0, cfg.tokens), on_layer=lambda l, y: ys.append(y.float().cpu().numpy()))
    ref = om.profile_all(cfg)
    alive = np.ones(cfg.tokens, bool)
    print(f"== {cfg.name}: L={cfg.n_layers} H={cfg.hidden} E={cfg.n_experts} k={cfg.top_k} F={cfg.ffn} "
          f"Fs={cfg.shared_ffn} INT{cfg.wbits} g={cfg.group_size} T={cfg.tokens}")
    for l in range(cfg.n_layers):
        z = prof.logits[l].cpu().numpy()
        ids = prof.ids[l].cpu().numpy()
        r = ref[l]
        zr = r["z"]
        lerr = np.abs(z - zr).max(1) / np.abs(zr).max(1)
        yerr = np.linalg.norm(ys[l] - r["y"], axis=1) / np.linalg.norm(r["y"], axis=1)
        same = np.array([set(a) == set(b) for a, b in zip(ids, r["ids"])])
        tie = r["margin"] <= 1e-3
        a = alive.copy()
        print(f" layer {l}: alive {a.sum()} ties {int((tie & a).sum())} div {int((~same & a).sum())} "
              f"(clear-div {int((~same & a & ~tie).sum())}) | logit rel max {lerr[a].max():.2e} med "
              f"{np.median(lerr[a]):.2e} | y rel max {yerr[a & same].max():.2e} med {np.median(yerr[a & same]):.2e}")
        alive &= same


if __name__ == "__main__":
    names = sys.argv[1:] or list(SMALL)
    for n in names:
        report(SMALL[n] if n in SMALL else synth.CONFIGS[n])
