"""driver — the participant-side round of the Flux hot path on one GPU (H2).

One profiling round (paper §4.1-4.2, §5.3; Fig. 7):
  a0  quantize the current model   flux_quantize_weights
  a1-a6  profile local tokens through all layers   flux_profile_layer per layer
  a7  reduce the expert histograms over the box   flux_reduce_stats
  a8-pre per-layer merge budget, eq.(1)   flux_layer_budget (optional)
  NEXT-1 expert clustering, §5.2   flux_expert_features, flux_cluster_experts
  a8  merge the non-tuning experts, eq.(2)   flux_merge_experts
This module owns buffers and sequencing only; all arithmetic is in libflux.
Layer chaining (R7): x_{l+1} = y_l (the path carries no attention/norm weights).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import (FLUX_OK, Comm, LayerOut, QLayer, attention_hist, cluster_experts, expert_features, layer_budget,
               layer_bops_bytes, make_cfg, merge_experts_batch, output_error, profile_layer, profile_layer_bops,
               profile_layer_uses_bops, profile_layer_workspace, quantize_weights, quantize_weights_bops)


@dataclass
class ModelShape:
    n_layers: int
    hidden: int
    n_experts: int
    top_k: int
    ffn: int
    shared_ffn: int
    wbits: int
    group_size: int
    norm_topk: int
    n_router: int = 0  # > 0: gate re-routing (NEXT-2): the router scores n_router original experts
    # per-layer expert (slot) counts of a compact model with adaptive layer sizes (eq.(1)):
    # layer l uses the first layer_experts[l] of the n_experts (= max) slots; None = n_experts everywhere
    layer_experts: tuple | None = None

    @staticmethod
    def of(cfg) -> "ModelShape":
        return ModelShape(cfg.n_layers, cfg.hidden, cfg.n_experts, cfg.top_k, cfg.ffn, cfg.shared_ffn, cfg.wbits,
                          cfg.group_size, cfg.norm_topk)

    def experts_of(self, l: int) -> int:
        return self.n_experts if self.layer_experts is None else int(self.layer_experts[l])

    def ccfg(self, l: int = 0):
        return make_cfg(self.hidden, self.ffn, self.experts_of(l), self.top_k, self.shared_ffn, self.wbits,
                        self.group_size, self.norm_topk, self.n_router)


@dataclass
class MasterWeights:
    """Full-precision (bf16) model on the device, family-major:
    router [L][E][H]; gate/up [L][E][F][H]; down [L][E][H][F]; sh_gate/sh_up [L][Fs][H]; sh_down [L][H][Fs]."""
    shape: ModelShape
    router: torch.Tensor
    gate: torch.Tensor
    up: torch.Tensor
    down: torch.Tensor
    sh_gate: torch.Tensor | None = None
    sh_up: torch.Tensor | None = None
    sh_down: torch.Tensor | None = None

    @staticmethod
    def empty(shape: ModelShape, device="cuda", dtype=torch.bfloat16) -> "MasterWeights":
        L, E, H, F, Fs = shape.n_layers, shape.n_experts, shape.hidden, shape.ffn, shape.shared_ffn
        mk = lambda *s: torch.empty(*s, dtype=dtype, device=device)  # noqa: E731
        return MasterWeights(shape, mk(L, E, H), mk(L, E, F, H), mk(L, E, F, H), mk(L, E, H, F),
                             mk(L, Fs, H) if Fs else None, mk(L, Fs, H) if Fs else None,
                             mk(L, H, Fs) if Fs else None)


class QuantizedModel:
    """Canonical quantized weights (include/flux.h flux_qlayer) for all layers, on the device."""

    def __init__(self, shape: ModelShape, device="cuda", with_bops: bool = False):
        """with_bops: also keep every layer's bf16 B operands (flux_layer_bops_bytes each, ~1.1 GB per
        DeepSeek-shape layer), written by the quantizer in the same pass (flux_quantize_weights_bops), so
        that profiling skips the per-call dequantization pass."""
        self.shape = s = shape
        L, E, H, F, Fs = s.n_layers, s.n_experts, s.hidden, s.ffn, s.shared_ffn
        qdiv = {2: 4, 4: 2}.get(s.wbits, 1)  # codes per byte
        qdt = torch.int8 if s.wbits == 8 else torch.uint8
        gh = s.group_size or H
        gf = s.group_size or F
        gfs = s.group_size or (Fs or 1)
        self.router = torch.empty(L, E, H, dtype=torch.bfloat16, device=device)
        self.gate_q = torch.empty(L, E, F, H // qdiv, dtype=qdt, device=device)
        self.up_q = torch.empty(L, E, F, H // qdiv, dtype=qdt, device=device)
        self.down_q = torch.empty(L, E, H, F // qdiv, dtype=qdt, device=device)
        self.gate_s = torch.empty(L, E, F, H // gh, dtype=torch.float32, device=device)
        self.up_s = torch.empty(L, E, F, H // gh, dtype=torch.float32, device=device)
        self.down_s = torch.empty(L, E, H, F // gf, dtype=torch.float32, device=device)
        if Fs:
            self.sh_gate_q = torch.empty(L, Fs, H // qdiv, dtype=qdt, device=device)
            self.sh_up_q = torch.empty(L, Fs, H // qdiv, dtype=qdt, device=device)
            self.sh_down_q = torch.empty(L, H, Fs // qdiv, dtype=qdt, device=device)
            self.sh_gate_s = torch.empty(L, Fs, H // gh, dtype=torch.float32, device=device)
            self.sh_up_s = torch.empty(L, Fs, H // gh, dtype=torch.float32, device=device)
            self.sh_down_s = torch.empty(L, H, Fs // gfs, dtype=torch.float32, device=device)
        else:
            self.sh_gate_q = self.sh_up_q = self.sh_down_q = None
            self.sh_gate_s = self.sh_up_s = self.sh_down_s = None
        self.bops = None
        if with_bops and s.wbits != 16 and s.layer_experts is None:
            # zeroed once: the rows padding F to a multiple of 128 are never written
            self.bops = torch.zeros(L, layer_bops_bytes(s.ccfg(0)), dtype=torch.uint8, device=device)

    def quantize_from(self, m: MasterWeights, stream=None):
        """a0: quantize every expert matrix of the master model (router copied: not quantized, R1); with
        bops, each family's bf16 B operands are written in the same pass."""
        s = self.shape
        self.router.copy_(m.router)
        pairs = [(m.gate, self.gate_q, self.gate_s), (m.up, self.up_q, self.up_s), (m.down, self.down_q, self.down_s)]
        if s.shared_ffn:
            pairs += [(m.sh_gate, self.sh_gate_q, self.sh_gate_s), (m.sh_up, self.sh_up_q, self.sh_up_s),
                      (m.sh_down, self.sh_down_q, self.sh_down_s)]
        for fam, (w, q, sc) in enumerate(pairs):
            if self.bops is not None:
                quantize_weights_bops(s.ccfg(0), fam, w, s.n_layers, q, sc, self.bops, stream)
            else:
                quantize_weights(w, s.wbits, s.group_size, q, sc, stream)

    def qlayer(self, l: int) -> QLayer:
        p = lambda t: None if t is None else t[l].data_ptr()  # noqa: E731
        return QLayer(p(self.router), p(self.gate_q), p(self.up_q), p(self.down_q), p(self.gate_s), p(self.up_s),
                      p(self.down_s), p(self.sh_gate_q), p(self.sh_up_q), p(self.sh_down_q), p(self.sh_gate_s),
                      p(self.sh_up_s), p(self.sh_down_s))


class DenseWeights:
    """Full-precision (bf16) expert weights run by flux_profile_layer with wbits = 16 (NEXT-2): the original
    model (remap None) or the compact model after merging (slots = tuning experts + clusters; the router keeps
    the E original experts and remap [L][E] re-routes its picks, §7)."""

    def __init__(self, shape: ModelShape, router, gate, up, down, sh_gate=None, sh_up=None, sh_down=None,
                 remap=None):
        self.shape = shape
        self.router, self.gate, self.up, self.down = router, gate, up, down
        self.sh_gate, self.sh_up, self.sh_down = sh_gate, sh_up, sh_down
        self.remap = remap

    def qlayer(self, l: int) -> QLayer:
        p = lambda t: None if t is None else t[l].data_ptr()  # noqa: E731
        q = QLayer(p(self.router), p(self.gate), p(self.up), p(self.down), None, None, None, p(self.sh_gate),
                   p(self.sh_up), p(self.sh_down), None, None, None)
        q.remap = p(self.remap)
        return q


def dense_model(m: MasterWeights) -> DenseWeights:
    """The original model in full precision (the reference for the merge output error)."""
    s = m.shape
    shape = ModelShape(s.n_layers, s.hidden, s.n_experts, s.top_k, s.ffn, s.shared_ffn, 16, 0, s.norm_topk)
    return DenseWeights(shape, m.router, m.gate, m.up, m.down, m.sh_gate, m.sh_up, m.sh_down)


def _per_layer(v, L: int) -> list[int]:
    return [int(v)] * L if np.isscalar(v) else [int(c) for c in v]


def compact_model(m: MasterWeights, alpha: torch.Tensor, cluster_of: torch.Tensor, n_clusters,
                  n_tuning=0, stream=None, out: DenseWeights | None = None) -> DenseWeights:
    """NEXT-2: the compact model (§7 "Customized MoE construction" + "Gate re-routing"): per layer the slots
    [n_tuning[l] tuning experts (ascending id), n_clusters[l] eq.(2) merges] of every weight family and the
    remap of the router's picks — ONE flux_merge_experts_batch launch (compact mode) for all L x 3 families.
    n_clusters / n_tuning: an int (uniform) or per-layer counts (adaptive layer sizes, eq.(1));
    n_tuning[l] must equal the number of -1 entries of cluster_of[l]."""
    s = m.shape
    L, E, F, H = s.n_layers, s.n_experts, s.ffn, s.hidden
    Cl, Tl = _per_layer(n_clusters, L), _per_layer(n_tuning, L)
    Sl = [c + t for c, t in zip(Cl, Tl)]
    S = max(Sl)
    dev = m.gate.device
    if out is not None and out.gate.shape[1] == S:  # reuse the buffers of a previous round
        gate, up, down, remap = out.gate, out.up, out.down, out.remap
    else:
        gate = torch.empty(L, S, F, H, dtype=m.gate.dtype, device=dev)
        up = torch.empty_like(gate)
        down = torch.empty(L, S, H, F, dtype=m.gate.dtype, device=dev)
        remap = torch.empty(L, E, dtype=torch.int32, device=dev)
    jobs = []
    for l in range(L):
        for src, dst, rm in ((m.gate, gate, remap[l]), (m.up, up, None), (m.down, down, None)):
            jobs.append(dict(experts=src[l].view(E, -1), cluster_of=cluster_of[l], alpha=alpha[l], n_clusters=Cl[l],
                             n_tuning=Tl[l], out=dst[l].view(S, -1), remap=rm))
    merge_experts_batch(jobs, compact=True, stream=stream)
    shape = ModelShape(L, H, S, s.top_k, F, s.shared_ffn, 16, 0, s.norm_topk, n_router=E,
                       layer_experts=None if len(set(Sl)) == 1 else tuple(Sl))
    return DenseWeights(shape, m.router, gate, up, down, m.sh_gate, m.sh_up, m.sh_down, remap)


class Profiler:
    """Buffers for profiling T tokens through all layers (a1-a6) on one GPU."""

    def __init__(self, shape: ModelShape, T: int, device="cuda", with_de: bool = True, with_logits: bool = False,
                 policy=None):
        s = self.shape = shape
        self.T = T
        self.policy = policy  # flux_policy (None = the library's measured defaults)
        L, E, H, k = s.n_layers, s.n_experts, s.hidden, s.top_k
        self.cfgs = [s.ccfg(l) for l in range(L)]  # per-layer expert counts (adaptive layer sizes)
        self.cfg = self.cfgs[0]
        ws = max(profile_layer_workspace(c, T, policy) for c in self.cfgs)
        self.ws = torch.empty(max(ws, 1), dtype=torch.uint8, device=device)
        self.y = torch.empty(2, T, H, dtype=torch.bfloat16, device=device)
        self.ids = torch.empty(L, T, k, dtype=torch.int32, device=device)
        self.w = torch.empty(L, T, k, dtype=torch.float32, device=device)
        self.hist = torch.zeros(L, E, dtype=torch.int64, device=device)
        self.offsets = torch.empty(L, E + 1, dtype=torch.int32, device=device) if with_de else None
        self.token_index = torch.empty(L, T * k, dtype=torch.int32, device=device) if with_de else None
        E_r = s.n_router or E  # the router scores the original experts under gate re-routing
        self.logits = torch.empty(L, T, E_r, dtype=torch.float32, device=device) if with_logits else None
        self.ahist = None  # [L][E] int64 attention-weighted counts when run(attn=...) is used (NEXT-3)

    def out(self, l: int) -> LayerOut:
        p = lambda t: None if t is None else t[l].data_ptr()  # noqa: E731
        return LayerOut(self.y[l % 2].data_ptr(), p(self.ids), p(self.w), p(self.hist), p(self.offsets),
                        p(self.token_index), p(self.logits))

    def _layer(self, qm, l: int, x: torch.Tensor, residual, stream):
        bops = getattr(qm, "bops", None)
        if bops is not None and profile_layer_uses_bops(self.cfgs[l], self.T, self.policy):
            # the quantizer already wrote this layer's bf16 B operands: no dequantization pass per call
            profile_layer_bops(self.cfgs[l], qm.qlayer(l), bops[l], x, residual, self.T, self.out(l), self.ws, stream,
                               self.policy)
        else:
            profile_layer(self.cfgs[l], qm.qlayer(l), x, residual, self.T, self.out(l), self.ws, stream, self.policy)

    def run_layer(self, qm, l: int, x: torch.Tensor, residual: torch.Tensor | None = None, stream=None):
        """One flux_profile_layer call with layer l's weights on x (no chaining); residual None = x (R6),
        e.g. a zero buffer so that y is the MoE branch alone.  Accumulates into hist[l]; returns y."""
        self._layer(qm, l, x, residual, stream)
        return self.y[l % 2]

    def run(self, qm: QuantizedModel, x: torch.Tensor, stream=None, on_layer=None, zero_hist: bool = True,
            attn: torch.Tensor | None = None):
        """Profile x [T][H] (bf16, device) through every layer; returns the last layer's y.
        attn [L][T] fp32 (optional, NEXT-3): per-token attention values -> self.ahist, the fixed-point
        attention-weighted counts of eq.(2)'s α = f·ā (flux_attention_hist)."""
        if zero_hist:
            self.hist.zero_()
        if attn is not None:
            if self.ahist is None:
                self.ahist = torch.zeros_like(self.hist)
            elif zero_hist:
                self.ahist.zero_()
        cur = x
        for l in range(self.shape.n_layers):
            torch.cuda.nvtx.range_push(f"layer {l}")  # the chunk x layer timeline under nsys
            self._layer(qm, l, cur, None, stream)
            torch.cuda.nvtx.range_pop()
            if attn is not None:
                attention_hist(self.ids[l], attn[l], self.shape.n_experts, self.ahist[l], stream)
            cur = self.y[l % 2]
            if on_layer is not None:
                on_layer(l, cur)
        return cur


def shard(rank: int, world: int, tokens_per_rank: int) -> tuple[int, int]:
    """Data-parallel split of the global token stream: rank r profiles the contiguous
    tokens [r·T, (r+1)·T); tokens are independent and the statistics additive, so the all-reduced
    histogram equals one GPU profiling the union."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return rank * tokens_per_rank, tokens_per_rank


def frequencies(hist_host: np.ndarray, T_total: int) -> np.ndarray:
    """Activation frequency f = activated tokens / total tokens, fp64 on the host."""
    return hist_host.astype(np.float64) / float(T_total)


@dataclass
class MergedModel:
    gate: torch.Tensor   # [L][C_max][F][H]; layer l uses its first n_clusters[l] rows
    up: torch.Tensor
    down: torch.Tensor   # [L][C_max][H][F]
    remap: torch.Tensor  # [L][E]
    n_clusters: tuple = ()


def merge_model(m: MasterWeights, alpha: torch.Tensor, cluster_of: torch.Tensor, n_clusters,
                out: MergedModel | None = None, stream=None) -> MergedModel:
    """a8: eq.(2) for every layer and weight family in ONE flux_merge_experts_batch launch.
    alpha fp32 [L][E], cluster_of int32 [L][E] (device); n_clusters an int or per-layer budgets B(l)."""
    s = m.shape
    L, E, F, H = s.n_layers, s.n_experts, s.ffn, s.hidden
    Cl = _per_layer(n_clusters, L)
    C = max(Cl)
    if out is None or out.gate.shape[1] != C:
        dev = m.gate.device
        out = MergedModel(torch.empty(L, C, F, H, dtype=m.gate.dtype, device=dev),
                          torch.empty(L, C, F, H, dtype=m.gate.dtype, device=dev),
                          torch.empty(L, C, H, F, dtype=m.gate.dtype, device=dev),
                          torch.empty(L, E, dtype=torch.int32, device=dev))
    out.n_clusters = tuple(Cl)
    jobs = []
    for l in range(L):
        for src, dst, rm in ((m.gate, out.gate, out.remap[l]), (m.up, out.up, None), (m.down, out.down, None)):
            jobs.append(dict(experts=src[l].view(E, -1), cluster_of=cluster_of[l], alpha=alpha[l],
                             n_clusters=Cl[l], out=dst[l].view(C, -1), remap=rm))
    merge_experts_batch(jobs, stream=stream)
    return out


def feature_dim(n_experts: int) -> int:
    """Reading R12: number of PCA components kept per layer, d = min(16, E - 1) (the paper does not fix it;
    E - 1 is the rank of E centred vectors)."""
    return max(1, min(16, n_experts - 1))


def expert_features_model(m: MasterWeights, d: int | None = None, with_gram: bool = False, stream=None):
    """NEXT-1 C1 (§5.2): PCA features [L][E][d] of every layer's experts (gate|up|down)."""
    s = m.shape
    L, E = s.n_layers, s.n_experts
    d = d or feature_dim(E)
    dev = m.gate.device
    feats = torch.empty(L, E, d, dtype=torch.float32, device=dev)
    gram = torch.empty(L, E, E, dtype=torch.float32, device=dev) if with_gram else None
    eig = torch.empty(L, d, dtype=torch.float32, device=dev)
    fams = [[m.gate[l], m.up[l], m.down[l]] for l in range(L)]
    expert_features(fams, d, feats, gram, eig, stream=stream)
    return feats, gram, eig


def cluster_model(features: torch.Tensor, hist_dev: torch.Tensor, n_clusters, tuning=None, max_iter: int = 50,
                  stream=None) -> torch.Tensor:
    """NEXT-1 C2 (§5.2): fused layer-masked K-Means -> cluster_of int32 [L][E] on the device."""
    L = features.shape[0]
    B = np.full(L, n_clusters, np.int32) if np.isscalar(n_clusters) else np.asarray(n_clusters, np.int32)
    return cluster_experts(features, hist_dev, B, tuning, max_iter, stream=stream)


def budgets(hist_host: np.ndarray, T_total: int, B_non: int, n_non=None):
    """a8-pre: eq.(1) layer budgets from the reduced histogram (host, libflux)."""
    return layer_budget(hist_host, T_total, B_non, n_non)


__all__ = ["ModelShape", "MasterWeights", "QuantizedModel", "Profiler", "MergedModel", "merge_model", "frequencies",
           "budgets", "feature_dim", "expert_features_model", "cluster_model", "DenseWeights", "dense_model",
           "compact_model", "output_error", "Comm", "FLUX_OK"]
