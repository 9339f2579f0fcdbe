"""synthetic — build the seeded synthetic workload of a ``synth.MoEConfig`` on the device.

Uses only the GPU twin of the generator (synth/gen_gpu.cu); holds no
arithmetic of the method.  The recipe (σ per tensor, router skew, bias
feature) lives in ``synth``; DESIGN.md §3 states it.
"""
from __future__ import annotations

import numpy as np
import torch

import synth

from .driver import MasterWeights, ModelShape


def master_weights(cfg, device="cuda", dtype=torch.bfloat16) -> MasterWeights:
    shape = ModelShape.of(cfg)
    m = MasterWeights.empty(shape, device, dtype)
    for l in range(cfg.n_layers):
        synth.gpu_fill(m.router[l], synth.spec_router(cfg, l))
        for e in range(cfg.n_experts):
            synth.gpu_fill(m.gate[l, e], synth.spec_expert(cfg, l, e, "gate"))
            synth.gpu_fill(m.up[l, e], synth.spec_expert(cfg, l, e, "up"))
            synth.gpu_fill(m.down[l, e], synth.spec_expert(cfg, l, e, "down"))
        if cfg.shared_ffn:
            synth.gpu_fill(m.sh_gate[l], synth.spec_expert(cfg, l, synth.SHARED_SLOT, "gate"))
            synth.gpu_fill(m.sh_up[l], synth.spec_expert(cfg, l, synth.SHARED_SLOT, "up"))
            synth.gpu_fill(m.sh_down[l], synth.spec_expert(cfg, l, synth.SHARED_SLOT, "down"))
    return m


def tokens(cfg, t0: int, n: int, device="cuda", out=None) -> torch.Tensor:
    """Rows [t0, t0+n) of x_0 (bf16 [n][H]); a token's values depend only on (seed, t)."""
    x = out if out is not None else torch.empty(n, cfg.hidden, dtype=torch.bfloat16, device=device)
    synth.gpu_fill(x, synth.spec_x(cfg), row0=t0)
    return x


def cluster_assignment(cfg, n_clusters: int, n_tuning: int = 0) -> np.ndarray:
    """cluster_of [L][E] (an input of the merge; see synth.cluster_assignment)."""
    return synth.cluster_assignment(cfg, n_clusters, n_tuning)


def attention_values(cfg, t0: int, n: int, device="cuda") -> torch.Tensor:
    """Per-layer, per-token attention values a_t >= 0 [L][n] fp32 for tokens [t0, t0+n) (synth.spec_attn;
    NEXT-3's α = f·ā needs them from the model's attention layers, which this path does not have)."""
    out = torch.empty(cfg.n_layers, n, 1, dtype=torch.float32, device=device)
    for l in range(cfg.n_layers):
        synth.gpu_fill(out[l], synth.spec_attn(cfg, l), row0=t0)
    return out.abs_().view(cfg.n_layers, n)
