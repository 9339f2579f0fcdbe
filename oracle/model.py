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
from . import QExpert, bf16_round, compact_tokens, merge, moe_tokens, permute, quantize


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


def branch_tokens(cfg, token_ids, layer: int, quantized=None, exact_dequant=False):
    """The MoE branch of one layer alone (residual r = 0, R6) on the generated x_0 of the given tokens:
    y = bf16(sh + Σ_j w_j o_j).  Returns a dict x, y, ids, w, z, margin, cond (cond = |sh| + Σ_j w_j|o_j|,
    the magnitude of the terms of the O6 sum) and dmag (the largest down-projection term, weighted),
    for condition-aware element-wise bounds."""
    x = synth.bf16_bits_to_f32(synth.cpu_rows(synth.spec_x(cfg), token_ids)).astype(np.float64)
    wr, experts, shared = quantized if quantized is not None else quantized_layer(cfg, layer)
    y, ids, w, z, m, cond, dmag = moe_tokens(x, wr, experts, shared, k=cfg.top_k, group_size=cfg.group_size,
                                             norm=cfg.norm_topk, residual=np.zeros_like(x), with_cond=True,
                                             exact_dequant=exact_dequant)
    return dict(x=x, y=y, ids=ids, w=w, z=z, margin=m, cond=cond, dmag=dmag)


def profile_all(cfg, quantized=None):
    """Whole-batch oracle for small configs: per layer also the histogram and D_e CSR (O3/O8)."""
    res = profile_tokens(cfg, np.arange(cfg.tokens), quantized=quantized)
    for r in res:
        hist, off, ti, inv = permute(r["ids"], cfg.n_experts)
        r.update(hist=hist, offsets=off, token_index=ti, inv_pos=inv)
    return res


# ------------------------------------------------------------------------------------------ NEXT-2
def dense_layer(cfg, layer: int):
    """Full-precision (bf16 master) weights of one layer: (wr, gate [E][F][H], up, down [E][H][F], shared)."""
    E = cfg.n_experts
    fam = {w: np.stack([master_f32(synth.spec_expert(cfg, layer, e, w)) for e in range(E)]).astype(np.float64)
           for w in ("gate", "up", "down")}
    shared = None
    if cfg.shared_ffn:
        shared = tuple(master_f32(synth.spec_expert(cfg, layer, synth.SHARED_SLOT, w)).astype(np.float64)
                       for w in ("gate", "up", "down"))
    wr = master_f32(synth.spec_router(cfg, layer)).astype(np.float64)
    return wr, fam["gate"], fam["up"], fam["down"], shared


def compact_layer(dense, cluster_of, alpha):
    """The compact model of one layer (§5.3 + §7, reading R14): slots = tuning experts (ascending id)
    then the eq.(2) merge of every cluster (O10), stored in bf16 like the GPU's merged weights.
    Returns (wr, gate [S][F][H], up, down, shared, remap [E])."""
    wr, gate, up, down, shared = dense
    E = gate.shape[0]
    cluster_of = np.asarray(cluster_of)
    C = int(cluster_of.max()) + 1 if (cluster_of >= 0).any() else 0
    out = []
    remap = None
    for W in (gate, up, down):
        merged, remap = merge(W.reshape(E, -1), cluster_of, alpha, C) if C else (np.zeros((0, W[0].size)),
                                                                                 np.arange(E, dtype=np.int32))
        S = int(remap.max()) + 1
        slots = np.empty((S,) + W.shape[1:])
        for e in range(E):
            if cluster_of[e] < 0:
                slots[remap[e]] = W[e]
        for c in range(C):
            slots[remap[np.nonzero(cluster_of == c)[0][0]]] = bf16_round(merged[c]).reshape(W.shape[1:])
        out.append(slots)
    return (wr, out[0], out[1], out[2], shared, remap)


def compact_forward(cfg, token_ids, layers_weights):
    """Follow tokens through a stack of (wr, gate, up, down, shared, remap) layers (R7 chaining).
    The original full-precision model is the same call with remap = identity."""
    x = synth.bf16_bits_to_f32(synth.cpu_rows(synth.spec_x(cfg), token_ids)).astype(np.float64)
    out = []
    for wr, gate, up, down, shared, remap in layers_weights:
        y, ids, w, z, m = compact_tokens(x, wr, remap, gate, up, down, shared, k=cfg.top_k, norm=cfg.norm_topk)
        out.append(dict(x=x, y=y, ids=ids, w=w, z=z, margin=m))
        x = y
    return out


def output_error(y_merged, y_orig) -> float:
    """The paper's merge-quality measure: the average cosine distance between
    the final token outputs of the merged model and of the original model."""
    a = np.asarray(y_merged, np.float64)
    b = np.asarray(y_orig, np.float64)
    cos = (a * b).sum(1) / (np.linalg.norm(a, axis=1) * np.linalg.norm(b, axis=1))
    return float(np.mean(1.0 - cos))
