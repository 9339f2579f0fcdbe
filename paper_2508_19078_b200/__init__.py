"""paper_2508_19078_b200 — B200-native hot path of Flux (arXiv 2508.19078).

Thin ctypes binding over libflux.so (include/flux.h).  This module only
marshals arguments: every step of the computation runs in the library's
sm_100a kernels.  torch supplies device memory, streams and process groups.
There is no CPU fallback: if libflux.so is missing or no sm_100 GPU is
present, calls raise.

Entry points (same names as the C ABI):
  profile_layer_workspace, profile_layer      quantized MoE layer + expert stats (§4.1)
  merge_experts                               eq.(2) merge
  quantize_weights                            INT8/INT4 quantizer
  layer_budget                                eq.(1)
  Comm (comm_unique_id / comm_init / reduce_stats / comm_destroy)   histogram all-reduce
"""
from __future__ import annotations

import ctypes
import os

import torch  # noqa: F401  (load torch's CUDA runtime first: libflux shares it)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libflux.so")

FLUX_OK, FLUX_E_INVALID, FLUX_E_UNSUPPORTED, FLUX_E_WORKSPACE, FLUX_E_CUDA, FLUX_E_NCCL = range(6)
FLUX_BF16, FLUX_FP32 = 0, 1


class FluxError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        detail = _lib().flux_last_error().decode()
        super().__init__(f"{what}: {_lib().flux_status_string(status).decode()} (status {status})"
                         + (f" [{detail}]" if detail else ""))


class MoECfg(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("hidden", "ffn", "n_experts", "top_k", "shared_ffn", "wbits", "group_size", "norm_topk",
                 "n_router")]


class QLayer(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("router_w", "gate_q", "up_q", "down_q", "gate_s", "up_s", "down_s",
                 "sh_gate_q", "sh_up_q", "sh_down_q", "sh_gate_s", "sh_up_s", "sh_down_s", "remap")]


class MergeJob(ctypes.Structure):
    """flux_merge_job (include/flux.h)."""
    _fields_ = [("experts", ctypes.c_void_p), ("cluster_of", ctypes.c_void_p), ("alpha", ctypes.c_void_p),
                ("n_clusters", ctypes.c_int32), ("n_tuning", ctypes.c_int32), ("out", ctypes.c_void_p),
                ("remap", ctypes.c_void_p)]


class Policy(ctypes.Structure):
    """flux_policy (include/flux.h): performance policy of flux_profile_layer_ex; all-zero = defaults.
    Every value gives bit-identical outputs; TEST-ONLY values were measured slower."""
    _fields_ = [("weight_path", ctypes.c_int32), ("routed_rows", ctypes.c_int32), ("fused_combine", ctypes.c_int32),
                ("static_tiles", ctypes.c_int32), ("l2_hints", ctypes.c_int32), ("gemm_chain", ctypes.c_int32)]


WEIGHTS_AUTO, WEIGHTS_DEQUANT_PASS, WEIGHTS_IN_GEMM = 0, 1, 2
ROWS_AUTO, ROWS_MATERIALISED, ROWS_TMA_GATHER4 = 0, 1, 2
L2_SET = 0x100
CHAIN_AUTO, CHAIN_OFF, CHAIN_ON = 0, 1, 2


def make_policy(weight_path=0, routed_rows=0, fused_combine=0, static_tiles=0, l2_hints=0, gemm_chain=0) -> Policy:
    return Policy(weight_path, routed_rows, fused_combine, static_tiles, l2_hints, gemm_chain)


class LayerOut(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("y", "topk_ids", "topk_w", "hist", "expert_offsets", "token_index", "router_logits")]


_L = None


def _lib():
    global _L
    if _L is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
        L.flux_status_string.argtypes = [ctypes.c_int]
        L.flux_status_string.restype = ctypes.c_char_p
        L.flux_profile_layer_workspace.argtypes = [ctypes.POINTER(MoECfg), I64]
        L.flux_profile_layer_workspace.restype = SZ
        L.flux_profile_layer.argtypes = [ctypes.POINTER(MoECfg), ctypes.POINTER(QLayer), P, P, I64,
                                         ctypes.POINTER(LayerOut), P, SZ, P]
        L.flux_profile_layer_workspace_ex.argtypes = [ctypes.POINTER(MoECfg), ctypes.POINTER(Policy), I64]
        L.flux_profile_layer_workspace_ex.restype = SZ
        L.flux_profile_layer_ex.argtypes = [ctypes.POINTER(MoECfg), ctypes.POINTER(Policy), ctypes.POINTER(QLayer),
                                            P, P, I64, ctypes.POINTER(LayerOut), P, SZ, P]
        L.flux_layer_bops_bytes.argtypes = [ctypes.POINTER(MoECfg)]
        L.flux_layer_bops_bytes.restype = SZ
        L.flux_quantize_weights_bops.argtypes = [ctypes.POINTER(MoECfg), I32, ctypes.c_int, P, I32, P, P, P, SZ, P]
        L.flux_dequantize_layer.argtypes = [ctypes.POINTER(MoECfg), ctypes.POINTER(QLayer), P, P]
        L.flux_profile_layer_uses_bops.argtypes = [ctypes.POINTER(MoECfg), ctypes.POINTER(Policy), I64]
        L.flux_profile_layer_uses_bops.restype = I32
        L.flux_profile_layer_workspace_bops.argtypes = [ctypes.POINTER(MoECfg), ctypes.POINTER(Policy), I64]
        L.flux_profile_layer_workspace_bops.restype = SZ
        L.flux_profile_layer_bops.argtypes = [ctypes.POINTER(MoECfg), ctypes.POINTER(Policy), ctypes.POINTER(QLayer),
                                              P, P, P, I64, ctypes.POINTER(LayerOut), P, SZ, P]
        L.flux_merge_experts.argtypes = [ctypes.c_int, I32, I64, P, P, P, I32, P, P, P]
        L.flux_quantize_weights.argtypes = [I32, I32, ctypes.c_int, P, I64, I64, P, P, P]
        L.flux_compact_experts.argtypes = [ctypes.c_int, I32, I64, P, P, P, I32, P, P, P]
        L.flux_merge_experts_batch.argtypes = [ctypes.c_int, I32, I64, I32, P, I32, P]
        L.flux_attention_hist.argtypes = [I64, I32, I32, P, P, P, P]
        L.flux_frequencies.argtypes = [I64, P, ctypes.c_double, P, P]
        L.flux_output_error_workspace.argtypes = []
        L.flux_output_error_workspace.restype = SZ
        L.flux_output_error.argtypes = [I64, I32, P, P, P, P, SZ, P]
        L.flux_layer_budget.argtypes = [I32, I32, P, I64, I64, P, P, P]
        L.flux_expert_features_workspace.argtypes = [I32, I32, I32, P]
        L.flux_expert_features_workspace.restype = SZ
        L.flux_expert_features.argtypes = [I32, I32, I32, P, P, I32, P, P, P, P, SZ, P]
        L.flux_cluster_experts.argtypes = [I32, I32, I32, P, P, P, P, I32, P, P, P]
        L.flux_comm_unique_id.argtypes = [P]
        L.flux_comm_init.argtypes = [ctypes.POINTER(P), P, I32, I32]
        L.flux_reduce_stats.argtypes = [P, P, SZ, P]
        L.flux_comm_destroy.argtypes = [P]
        for f in ("flux_profile_layer", "flux_profile_layer_ex", "flux_profile_layer_bops", "flux_dequantize_layer",
                  "flux_quantize_weights_bops", "flux_merge_experts", "flux_quantize_weights", "flux_layer_budget",
                  "flux_expert_features", "flux_cluster_experts", "flux_compact_experts", "flux_output_error",
                  "flux_merge_experts_batch", "flux_frequencies",
                  "flux_attention_hist",
                  "flux_comm_unique_id", "flux_comm_init", "flux_reduce_stats", "flux_comm_destroy"):
            getattr(L, f).restype = ctypes.c_int
        L.flux_timing_enable.argtypes = [ctypes.c_int]
        L.flux_timing_enable.restype = None
        L.flux_timing_read.argtypes = [P, P, ctypes.c_int, ctypes.c_int]
        L.flux_timing_read.restype = ctypes.c_int
        L.flux_kernel_name.argtypes = [ctypes.c_int]
        L.flux_kernel_name.restype = ctypes.c_char_p
        L.flux_last_error.argtypes = []
        L.flux_last_error.restype = ctypes.c_char_p
        L.flux_timing_clocks.argtypes = [P, ctypes.c_int, ctypes.c_int]
        L.flux_timing_clocks.restype = ctypes.c_int
        L.flux_launch_count.argtypes = []
        L.flux_launch_count.restype = ctypes.c_longlong
        _L = L
    return _L


# ------------------------------------------------------------------------------------------ diagnostics
def timing_enable(on: bool = True):
    _lib().flux_timing_enable(1 if on else 0)


def timing_read(reset: bool = True) -> dict:
    """{kernel name: (total ms, launches)} of the launches recorded while timing was enabled."""
    n = 32
    ms = (ctypes.c_double * n)()
    cnt = (ctypes.c_longlong * n)()
    k = _lib().flux_timing_read(ms, cnt, n, 1 if reset else 0)
    return {_lib().flux_kernel_name(i).decode(): (ms[i], cnt[i]) for i in range(k)}


def timing_clocks(reset: bool = True) -> dict:
    """{kernel name: average SM MHz inside the kernel} for the clock-probed kernels (the expert GEMMs)."""
    n = 32
    mhz = (ctypes.c_double * n)()
    k = _lib().flux_timing_clocks(mhz, n, 1 if reset else 0)
    return {_lib().flux_kernel_name(i).decode(): mhz[i] for i in range(k) if mhz[i] > 0}


def launch_count() -> int:
    return int(_lib().flux_launch_count())


def lib():
    return _lib()


def _check(st: int, what: str):
    if st != FLUX_OK:
        raise FluxError(st, what)


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream(stream=None):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else stream


# ------------------------------------------------------------------------------------------ API
def make_cfg(hidden, ffn, n_experts, top_k, shared_ffn, wbits, group_size, norm_topk, n_router=0) -> MoECfg:
    return MoECfg(hidden, ffn, n_experts, top_k, shared_ffn, wbits, group_size, norm_topk, n_router)


def _pol(policy):
    return ctypes.byref(policy) if policy is not None else None


def profile_layer_workspace(cfg: MoECfg, T: int, policy: Policy | None = None) -> int:
    return int(_lib().flux_profile_layer_workspace_ex(ctypes.byref(cfg), _pol(policy), T))


def profile_layer(cfg: MoECfg, qlayer: QLayer, x, residual, T: int, out: LayerOut, ws, stream=None,
                  policy: Policy | None = None):
    """One quantized MoE layer + statistics (flux_profile_layer_ex). Tensors are CUDA tensors."""
    st = _lib().flux_profile_layer_ex(ctypes.byref(cfg), _pol(policy), ctypes.byref(qlayer), _ptr(x), _ptr(residual),
                                      T, ctypes.byref(out), _ptr(ws),
                                      ws.numel() * ws.element_size() if ws is not None else 0, _stream(stream))
    _check(st, "flux_profile_layer")


def merge_experts(experts, cluster_of, alpha, n_clusters: int, merged, remap=None, stream=None):
    """eq.(2): experts [E][numel] (bf16/fp32 CUDA), cluster_of int32 [E], alpha fp32 [E] -> merged [C][numel]."""
    dt = FLUX_FP32 if experts.dtype == torch.float32 else FLUX_BF16
    E = experts.shape[0]
    numel = experts.numel() // E
    st = _lib().flux_merge_experts(dt, E, numel, _ptr(experts), _ptr(cluster_of), _ptr(alpha), n_clusters,
                                   _ptr(merged), _ptr(remap), _stream(stream))
    _check(st, "flux_merge_experts")


MERGE_MAX_JOBS = 256


def merge_experts_batch(jobs, compact: bool = False, stream=None):
    """eq.(2) for many jobs in ONE launch (flux_merge_experts_batch).  jobs: list of dicts with experts
    [E][numel], cluster_of [E], alpha [E], n_clusters, out, optional remap and (compact) n_tuning; all
    jobs share E, numel and the dtype."""
    if not jobs:
        return
    ex0 = jobs[0]["experts"]
    dt = FLUX_FP32 if ex0.dtype == torch.float32 else FLUX_BF16
    E = ex0.shape[0]
    numel = ex0.numel() // E
    for i in range(0, len(jobs), MERGE_MAX_JOBS):
        part = jobs[i:i + MERGE_MAX_JOBS]
        arr = (MergeJob * len(part))()
        for a, j in zip(arr, part):
            assert j["experts"].dtype == ex0.dtype and j["experts"].numel() == E * numel
            a.experts, a.cluster_of, a.alpha = _ptr(j["experts"]), _ptr(j["cluster_of"]), _ptr(j["alpha"])
            a.n_clusters, a.n_tuning = int(j["n_clusters"]), int(j.get("n_tuning", 0))
            a.out, a.remap = _ptr(j["out"]), _ptr(j.get("remap"))
        st = _lib().flux_merge_experts_batch(dt, E, numel, len(part), ctypes.cast(arr, ctypes.c_void_p),
                                             int(compact), _stream(stream))
        _check(st, "flux_merge_experts_batch")


def compact_experts(experts, cluster_of, alpha, n_clusters: int, compact, remap=None, stream=None):
    """NEXT-2: slots of the compact model (tuning experts, then eq.(2) clusters) -> compact [S][numel]."""
    dt = FLUX_FP32 if experts.dtype == torch.float32 else FLUX_BF16
    E = experts.shape[0]
    numel = experts.numel() // E
    st = _lib().flux_compact_experts(dt, E, numel, _ptr(experts), _ptr(cluster_of), _ptr(alpha), n_clusters,
                                     _ptr(compact), _ptr(remap), _stream(stream))
    _check(st, "flux_compact_experts")


def frequencies(counts, denom: float, alpha, stream=None):
    """alpha = fl32(counts / denom) on the device (flux_frequencies): f = hist / T, or α = A / (2^24·T)."""
    assert counts.dtype == torch.int64 and alpha.dtype == torch.float32 and counts.numel() == alpha.numel()
    st = _lib().flux_frequencies(counts.numel(), _ptr(counts), float(denom), _ptr(alpha), _stream(stream))
    _check(st, "flux_frequencies")


def attention_hist(ids, attn, n_experts: int, out, stream=None):
    """NEXT-3: out int64 [E] += fixed-point attention-weighted counts (α = f·ā = out / (2^24·T))."""
    T, k = ids.shape
    st = _lib().flux_attention_hist(T, k, n_experts, _ptr(ids), _ptr(attn), _ptr(out), _stream(stream))
    _check(st, "flux_attention_hist")


def output_error(a, b, result=None, ws=None, stream=None):
    """Mean cosine distance between two bf16 [T][H] CUDA outputs -> device double [1]."""
    T, H = a.shape
    if result is None:
        result = torch.empty(1, dtype=torch.float64, device=a.device)
    if ws is None:
        ws = torch.empty(int(_lib().flux_output_error_workspace()), dtype=torch.uint8, device=a.device)
    st = _lib().flux_output_error(T, H, _ptr(a), _ptr(b), _ptr(result), _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "flux_output_error")
    return result


def quantize_weights(w, wbits: int, group_size: int, q, s, stream=None):
    """w [R][K] bf16/fp32 CUDA -> q int8 [R][K] or uint8 [R][K/2] (INT4), s fp32 [R][K/g]."""
    dt = FLUX_FP32 if w.dtype == torch.float32 else FLUX_BF16
    K = w.shape[-1]
    R = w.numel() // K
    st = _lib().flux_quantize_weights(wbits, group_size, dt, _ptr(w), R, K, _ptr(q), _ptr(s), _stream(stream))
    _check(st, "flux_quantize_weights")


FAM_GATE, FAM_UP, FAM_DOWN, FAM_SH_GATE, FAM_SH_UP, FAM_SH_DOWN = range(6)


def layer_bops_bytes(cfg: MoECfg) -> int:
    """Bytes of one layer's bf16 B operands (flux_layer_bops_bytes)."""
    return int(_lib().flux_layer_bops_bytes(ctypes.byref(cfg)))


def quantize_weights_bops(cfg: MoECfg, family: int, w, n_layers: int, q, s, bops, stream=None):
    """flux_quantize_weights_bops: quantize one family of n_layers layers (w [n_layers·rows][K]) into q, s and
    write each layer's bf16 B operands of that family into bops [n_layers][layer_bops_bytes] (uint8 CUDA)."""
    dt = FLUX_FP32 if w.dtype == torch.float32 else FLUX_BF16
    st = _lib().flux_quantize_weights_bops(ctypes.byref(cfg), family, dt, _ptr(w), n_layers, _ptr(q), _ptr(s),
                                           _ptr(bops), bops.stride(0) * bops.element_size(), _stream(stream))
    _check(st, "flux_quantize_weights_bops")


def dequantize_layer(cfg: MoECfg, qlayer: QLayer, bops, stream=None):
    """flux_dequantize_layer: the layer's bf16 B operands from its q, s into bops (uint8 CUDA tensor)."""
    _check(_lib().flux_dequantize_layer(ctypes.byref(cfg), ctypes.byref(qlayer), _ptr(bops), _stream(stream)),
           "flux_dequantize_layer")


def profile_layer_uses_bops(cfg: MoECfg, T: int, policy: Policy | None = None) -> bool:
    r = int(_lib().flux_profile_layer_uses_bops(ctypes.byref(cfg), _pol(policy), T))
    if r < 0:
        raise ValueError("flux_profile_layer_uses_bops: invalid arguments")
    return r == 1


def profile_layer_workspace_bops(cfg: MoECfg, T: int, policy: Policy | None = None) -> int:
    return int(_lib().flux_profile_layer_workspace_bops(ctypes.byref(cfg), _pol(policy), T))


def profile_layer_bops(cfg: MoECfg, qlayer: QLayer, bops, x, residual, T: int, out: LayerOut, ws, stream=None,
                       policy: Policy | None = None):
    """flux_profile_layer_bops: profile_layer with this layer's B operands already dequantized."""
    st = _lib().flux_profile_layer_bops(ctypes.byref(cfg), _pol(policy), ctypes.byref(qlayer), _ptr(bops), _ptr(x),
                                        _ptr(residual), T, ctypes.byref(out), _ptr(ws),
                                        ws.numel() * ws.element_size() if ws is not None else 0, _stream(stream))
    _check(st, "flux_profile_layer_bops")


def layer_budget(hist, T: int, B_non: int, n_non=None):
    """eq.(1) on host int64 counts [L][E] -> (C [L] list, overrun)."""
    import numpy as np
    h = np.ascontiguousarray(hist, dtype=np.int64)
    L, E = h.shape
    C = np.empty(L, np.int32)
    nn = None if n_non is None else np.ascontiguousarray(n_non, dtype=np.int32)
    over = ctypes.c_int64(0)
    st = _lib().flux_layer_budget(L, E, h.ctypes.data, T, B_non, None if nn is None else nn.ctypes.data,
                                  C.ctypes.data, ctypes.byref(over))
    _check(st, "flux_layer_budget")
    return C, over.value


def expert_features_workspace(n_layers: int, n_experts: int, fam_numel) -> int:
    import numpy as np
    n = np.ascontiguousarray(fam_numel, dtype=np.int64)
    return int(_lib().flux_expert_features_workspace(n_layers, n_experts, len(n), n.ctypes.data))


def expert_features(families, d: int, features, gram=None, eigvals=None, ws=None, stream=None):
    """§5.2 C1 (flux_expert_features).  families: per layer, a list of bf16 CUDA tensors [E][...]
    (contiguous; same family shapes in every layer) -> features fp32 [L][E][d] (+ raw Gram [L][E][E],
    eigenvalues [L][d])."""
    import numpy as np
    L, nf = len(families), len(families[0])
    E = families[0][0].shape[0]
    numel = np.array([t.numel() // E for t in families[0]], np.int64)
    ptrs = (ctypes.c_void_p * (L * nf))(*[t.data_ptr() for fam in families for t in fam])
    for fam in families:
        for t, n in zip(fam, numel):
            if t.dtype != torch.bfloat16 or not t.is_contiguous() or t.numel() != E * n:
                raise ValueError("expert_features: families must be contiguous bf16 [E][numel] of equal shapes")
    if ws is None:
        ws = torch.empty(expert_features_workspace(L, E, numel), dtype=torch.uint8, device=features.device)
    st = _lib().flux_expert_features(L, E, nf, ptrs, numel.ctypes.data, d, _ptr(features), _ptr(gram),
                                     _ptr(eigvals), _ptr(ws), ws.numel(), _stream(stream))
    _check(st, "flux_expert_features")


def cluster_experts(features, counts, n_clusters, tuning=None, max_iter: int = 50, cluster_of=None,
                    iterations=None, stream=None):
    """§5.2 C2 (flux_cluster_experts).  features fp32 CUDA [L][E][d]; counts int64 CUDA [L][E];
    n_clusters host ints [L]; tuning host bool [L][E] or None -> cluster_of int32 CUDA [L][E]."""
    import numpy as np
    L, E, d = features.shape
    B = np.ascontiguousarray(n_clusters, dtype=np.int32)
    tu = None if tuning is None else np.ascontiguousarray(tuning, dtype=np.uint8)
    if cluster_of is None:
        cluster_of = torch.empty((L, E), dtype=torch.int32, device=features.device)
    st = _lib().flux_cluster_experts(L, E, d, _ptr(features), _ptr(counts), B.ctypes.data,
                                     None if tu is None else tu.ctypes.data, max_iter, _ptr(cluster_of),
                                     _ptr(iterations), _stream(stream))
    _check(st, "flux_cluster_experts")
    return cluster_of


class Comm:
    """NCCL communicator for the histogram all-reduce (flux_comm_*)."""

    def __init__(self, uid: bytes, nranks: int, rank: int):
        self._h = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(uid, 128)
        _check(_lib().flux_comm_init(ctypes.byref(self._h), buf, nranks, rank), "flux_comm_init")

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(_lib().flux_comm_unique_id(buf), "flux_comm_unique_id")
        return buf.raw

    def reduce_stats(self, hist, stream=None):
        _check(_lib().flux_reduce_stats(self._h, _ptr(hist), hist.numel(), _stream(stream)), "flux_reduce_stats")

    def destroy(self):
        if self._h:
            _check(_lib().flux_comm_destroy(self._h), "flux_comm_destroy")
            self._h = ctypes.c_void_p()
