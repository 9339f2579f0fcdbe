"""oracle.model — the oracle run over the synthetic model of ``synth``.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Inputs come from the CPU
twin of the generator (``synth.cpu_*``); nothing here reads anything the CUDA
path produced.

Layer chaining (R7): the hot path has no attention or norm
weights, so layer l+1 consumes y_l directly: x_{l+1} = y_l.  Tokens never
interact, so a SAMPLE of tokens can be followed through all layers exactly
("free-running"): the oracle needs only x_0 of those tokens and the weights.
"""
from __future__ import annotations

import numpy as np

import synth
from . import QExpert, moe_tokens, permute, quantize


def master_f32(spec) -> np.ndarray:
    return synth.bf16_bits_to_f32(synth.cpu_matrix(spec))


def quantized_layer(cfg, layer: int):
    """O1 applied to every expert matrix of one layer (router stays bf16, R1)."""
    g = cfg.group_size
    experts = []
    for e in range(cfg.n_experts):
        mats = []
        for which in ("gate", "up", "down"):
            q, s = quantize(master_f32(synth.spec_expert(cfg, layer, e, which)), cfg.wbits, g)
            mats += [q, s]
        experts.append(QExpert(*mats))
    shared = None
    if cfg.shared_ffn:
        mats = []
        for which in ("gate", "up", "down"):
            q, s = quantize(master_f32(synth.spec_expert(cfg, layer, synth.SHARED_SLOT, which)), cfg.wbits, g)
            mats += [q, s]
        shared = QExpert(*mats)
    wr = master_f32(synth.spec_router(cfg, layer)).astype(np.float64)
    return wr, experts, shared


def profile_tokens(cfg, token_ids, layers=None, quantized=None):
    """Follow the given tokens through layers 0..L-1 of the quantized model.

    Returns a list (one per layer) of dicts: x (input), y, ids, w, z, margin.
    ``quantized`` may pass precomputed quantized_layer() results (index = layer).
    """
    L = cfg.n_layers if layers is None else layers
    x = synth.bf16_bits_to_f32(synth.cpu_rows(synth.spec_x(cfg), token_ids)).astype(np.float64)
    out = []
    for l in range(L):
        wr, experts, shared = quantized[l] if quantized is not None else quantized_layer(cfg, l)
        y, ids, w, z, m = moe_tokens(x, wr, experts, shared, k=cfg.top_k, group_size=cfg.group_size,
                                     norm=cfg.norm_topk)
        out.append(dict(x=x, y=y, ids=ids, w=w, z=z, margin=m))
        x = y
    return out


def profile_all(cfg, quantized=None):
    """Whole-batch oracle for small configs: per layer also the histogram and D_e CSR (O3/O8)."""
    res = profile_tokens(cfg, np.arange(cfg.tokens), quantized=quantized)
    for r in res:
        hist, off, ti, inv = permute(r["ids"], cfg.n_experts)
        r.update(hist=hist, offsets=off, token_index=ti, inv_pos=inv)
    return res
