"""synth — seeded synthetic workloads shared by the CUDA path and the CPU oracle.

This package holds NO arithmetic of the Flux method (arXiv 2508.19078).  It
defines
  * the workload shapes of BASELINE.json's configs (``CONFIGS``), and
  * the input recipe: which generator stream and which σ each
    tensor uses,
and exposes the counter-based generator G twice: ``*_cpu`` (synth/gen_cpu.c)
and ``*_gpu`` (synth/gen_gpu.cu).  The two are bit-identical
(tests/test_synth.py); the CPU twin feeds the oracle, the GPU twin feeds the
CUDA path, so neither side ever consumes the other's outputs.

Recipe (mirrors Fig. 2 of the paper: layer 1 skewed, later
layers more balanced):
  x_0[t][0] = 1.0 (bias feature), x_0[t][d>0] ~ IH4(σ=1)
  W_r[l][e][0] = β_{l,e} ~ IH4(σ=s_l), s_l linear 0.35 (l=0) → 0.10 (l=L-1)
  W_r[l][e][d>0] ~ IH4(σ=1/√H)
  W_gate, W_up [F][H] ~ IH4(σ=1/√H);  W_down [H][F] ~ IH4(σ=0.1/√F), row 0 = 0
  (0.1 keeps the norm-free residual stream at rms ≈ 1.06 over 28 layers; 0.5 diverges)
  shared experts: one SwiGLU MLP of width F_s (expert slot 1023)
IH4 = Irwin–Hall(4) of 12-bit uniforms, centred and scaled to std σ.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

COL0_ONE = 1
ROW0_ZERO = 2
COL0_C0 = 4

KIND_X, KIND_ROUTER, KIND_GATE, KIND_UP, KIND_DOWN, KIND_MASTER_F32, KIND_ATTN = 1, 2, 3, 4, 5, 6, 7
SHARED_SLOT = 1023
BASE_SEED = 0x250819078


@dataclass(frozen=True)
class MoEConfig:
    """Shape of one synthetic MoE model + profiling batch (BASELINE.json configs)."""
    name: str
    n_layers: int
    hidden: int
    n_experts: int
    top_k: int
    ffn: int
    shared_ffn: int
    wbits: int
    group_size: int  # 0 = per output channel (g = K)
    norm_topk: int   # 0: w = softmax prob (DeepSeek-MoE); 1: renormalised over the top-k
    tokens: int
    seed: int
    skew: str = "fig2"  # "fig2" | "balanced" | "hot" (layer 0: a few experts take most tokens, others none)

    def with_(self, **kw) -> "MoEConfig":
        return replace(self, **kw)


CONFIGS = {
    # BASELINE.json configs[0]
    "toy": MoEConfig("toy", 2, 64, 8, 2, 128, 0, 8, 0, 1, 256, BASE_SEED + 0),
    # configs[1]  (F = 11008/16 = 688 [ext], BJ omits F)
    "llama_moe": MoEConfig("llama_moe_3.5b", 32, 4096, 16, 4, 688, 0, 8, 0, 1, 65536, BASE_SEED + 1),
    # configs[2]  (2 shared experts of width 1408 == one SwiGLU of width 2816)
    "deepseek_moe": MoEConfig("deepseek_moe_16b", 28, 2048, 64, 6, 1408, 2816, 4, 128, 0, 262144, BASE_SEED + 2),
    # configs[4]: the DP workload (2M tokens sharded over ranks)
    "deepseek_moe_dp": MoEConfig("deepseek_moe_16b_dp", 28, 2048, 64, 6, 1408, 2816, 4, 128, 0, 2097152,
                                 BASE_SEED + 2),
}
# configs[3]: layer-aware merge on the DeepSeek shape, 64 -> 16 per layer, bf16
MERGE_CLUSTERS = 16


def stream_id(kind: int, layer: int, expert: int) -> int:
    return (kind << 20) | (layer << 10) | expert


def scale_c(sigma: float) -> float:
    """c = fl32(σ·√3/4096): IH4 of 12-bit uniforms has std 4096/√3."""
    return float(np.float32(sigma * math.sqrt(3.0) / 4096.0))


def router_skew_sigma(cfg: MoEConfig, layer: int) -> float:
    if cfg.skew == "balanced":
        return 0.0
    if cfg.skew == "hot" and layer == 0:  # SURVEY §8d hot-expert variant: σ_β = 2.5 >> the unit logit noise
        return 2.5
    if cfg.n_layers == 1:
        return 0.35
    return 0.35 + (0.10 - 0.35) * layer / (cfg.n_layers - 1)


# --------------------------------------------------------------------------------------
# tensor recipes
# --------------------------------------------------------------------------------------
@dataclass(frozen=True)
class Spec:
    rows: int
    cols: int
    seed: int
    stream: int
    c: float
    flags: int
    c0: float


def spec_x(cfg: MoEConfig):
    return Spec(cfg.tokens, cfg.hidden, cfg.seed, stream_id(KIND_X, 0, 0), scale_c(1.0), COL0_ONE, 0.0)


def spec_attn(cfg: MoEConfig, layer: int):
    """Per-token attention values a_t (NEXT-3, α = f·ā): |N(0, 1)| -> take abs() of the fp32 output.
    The path has no attention layers; these stand in for the values the model's attention supplies."""
    return Spec(cfg.tokens, 1, cfg.seed, stream_id(KIND_ATTN, layer, 0), scale_c(1.0), 0, 0.0)


def spec_router(cfg: MoEConfig, layer: int):
    return Spec(cfg.n_experts, cfg.hidden, cfg.seed, stream_id(KIND_ROUTER, layer, 0),
                scale_c(1.0 / math.sqrt(cfg.hidden)), COL0_C0, scale_c(router_skew_sigma(cfg, layer)))


def spec_expert(cfg: MoEConfig, layer: int, expert: int, which: str):
    """which in {gate, up, down}; expert == SHARED_SLOT selects the shared MLP."""
    F = cfg.shared_ffn if expert == SHARED_SLOT else cfg.ffn
    H = cfg.hidden
    s = cfg.seed
    if which == "gate":
        return Spec(F, H, s, stream_id(KIND_GATE, layer, expert), scale_c(1.0 / math.sqrt(H)), 0, 0.0)
    if which == "up":
        return Spec(F, H, s, stream_id(KIND_UP, layer, expert), scale_c(1.0 / math.sqrt(H)), 0, 0.0)
    if which == "down":
        return Spec(H, F, s, stream_id(KIND_DOWN, layer, expert), scale_c(0.1 / math.sqrt(F)), ROW0_ZERO, 0.0)
    raise ValueError(which)


def cluster_assignment(cfg: MoEConfig, n_clusters: int, n_tuning: int = 0) -> np.ndarray:
    """Seeded balanced partition of every layer's experts into n_clusters (cluster_of [L][E] int32).

    The clustering step itself (§5.2, PCA + K-Means) is not on this path: cluster_of is an
    input of the merge.  The first n_tuning experts of each layer's random order are tuning
    experts (-1), the rest are dealt round-robin to clusters 0..C-1 (M4: 64 -> 16, 4 per cluster).
    """
    rng = np.random.default_rng(cfg.seed ^ 0x5EED)
    out = np.empty((cfg.n_layers, cfg.n_experts), np.int32)
    for l in range(cfg.n_layers):
        order = rng.permutation(cfg.n_experts)
        out[l, order[:n_tuning]] = -1
        rest = order[n_tuning:]
        out[l, rest] = np.arange(len(rest)) % n_clusters
    return out


# --------------------------------------------------------------------------------------
# CPU twin
# --------------------------------------------------------------------------------------
_cpu = None


def _cpu_lib():
    global _cpu
    if _cpu is None:
        path = os.path.join(_HERE, "libsynth_cpu.so")
        if not os.path.exists(path):
            build_cpu()
        lib = ctypes.CDLL(path)
        lib.synth_cpu_matrix.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_float,
                                         ctypes.c_int, ctypes.c_float]
        lib.synth_cpu_rows.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_float,
                                       ctypes.c_int, ctypes.c_float]
        _cpu = lib
    return _cpu


def build_cpu():
    src = os.path.join(_HERE, "gen_cpu.c")
    out = os.path.join(_HERE, "libsynth_cpu.so")
    cmd = f"gcc -O2 -fopenmp -fPIC -shared -ffp-contract=off -o {out} {src}"
    if os.system(cmd) != 0:
        raise RuntimeError("failed: " + cmd)


def build_gpu():
    src = os.path.join(_HERE, "gen_gpu.cu")
    out = os.path.join(_HERE, "libsynth_gpu.so")
    cmd = (f"nvcc -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared "
           f"-fmad=false -o {out} {src}")
    if os.system(cmd) != 0:
        raise RuntimeError("failed: " + cmd)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def cpu_matrix(spec: Spec, row0: int = 0, rows: int | None = None, dtype: str = "bf16") -> np.ndarray:
    """Rows [row0, row0+rows) of a generated matrix. bf16 -> np.uint16 bits; f32 -> np.float32."""
    rows = spec.rows - row0 if rows is None else rows
    out = np.empty((rows, spec.cols), dtype=np.uint16 if dtype == "bf16" else np.float32)
    _cpu_lib().synth_cpu_matrix(out.ctypes.data, 0 if dtype == "bf16" else 1, rows, spec.cols, row0, spec.seed,
                                spec.stream, spec.c, spec.flags, spec.c0)
    return out


def cpu_rows(spec: Spec, row_ids, dtype: str = "bf16") -> np.ndarray:
    ids = np.ascontiguousarray(np.asarray(row_ids, dtype=np.int64))
    out = np.empty((len(ids), spec.cols), dtype=np.uint16 if dtype == "bf16" else np.float32)
    _cpu_lib().synth_cpu_rows(out.ctypes.data, 0 if dtype == "bf16" else 1, ids.ctypes.data, len(ids), spec.cols,
                              spec.seed, spec.stream, spec.c, spec.flags, spec.c0)
    return out


# --------------------------------------------------------------------------------------
# GPU twin (torch tensors on device; torch is plumbing only)
# --------------------------------------------------------------------------------------
_gpu = None


def _gpu_lib():
    global _gpu
    if _gpu is None:
        path = os.path.join(_HERE, "libsynth_gpu.so")
        if not os.path.exists(path):
            raise RuntimeError("synth/libsynth_gpu.so missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        lib.synth_gpu_matrix.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_float,
                                         ctypes.c_int, ctypes.c_float, ctypes.c_void_p]
        lib.synth_gpu_matrix.restype = ctypes.c_int
        _gpu = lib
    return _gpu


def gpu_fill(dst, spec: Spec, row0: int = 0):
    """Fill a contiguous CUDA tensor (bf16 or fp32, last dim = spec.cols) with generated rows row0.."""
    import torch
    C = spec.cols
    assert dst.is_cuda and dst.is_contiguous() and dst.shape[-1] == C
    rows = dst.numel() // C
    dt = 0 if dst.dtype == torch.bfloat16 else 1
    rc = _gpu_lib().synth_gpu_matrix(dst.data_ptr(), dt, rows, C, row0, spec.seed, spec.stream, spec.c, spec.flags,
                                     spec.c0, torch.cuda.current_stream(dst.device).cuda_stream)
    if rc != 0:
        raise RuntimeError(f"synth_gpu_matrix failed: cuda error {rc}")
    return dst
