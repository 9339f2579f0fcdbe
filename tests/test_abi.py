"""The C-ABI library: loads, exports every symbol include/flux.h declares, and
validates arguments on the host (no compute calls: these run without a GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def F():
    import paper_2508_19078_b200 as F
    if not os.path.exists(F.LIB_PATH):
        from paper_2508_19078_b200 import build
        build.build()
    F.lib()
    return F


def test_exports_every_declared_symbol(F):
    hdr = open(os.path.join(ROOT, "include", "flux.h")).read()
    names = set(re.findall(r"\b(flux_[a-z_]+)\s*\(", hdr))
    assert {"flux_profile_layer", "flux_merge_experts", "flux_reduce_stats"} <= names
    lib = ctypes.CDLL(F.LIB_PATH)
    for n in sorted(names):
        assert hasattr(lib, n), n


def test_status_strings(F):
    for s in range(6):
        assert F.lib().flux_status_string(s)


def test_host_validation_without_gpu(F):
    L = F.lib()
    bad = F.make_cfg(100, 128, 8, 2, 0, 8, 0, 1)  # hidden % 64 != 0
    assert L.flux_profile_layer_workspace(ctypes.byref(bad), 10) == 0
    out = F.LayerOut()
    ql = F.QLayer()
    assert L.flux_profile_layer(ctypes.byref(bad), ctypes.byref(ql), None, None, 10, ctypes.byref(out), None, 0,
                                None) == F.FLUX_E_UNSUPPORTED
    good = F.make_cfg(64, 128, 8, 2, 0, 8, 0, 1)
    assert L.flux_profile_layer_workspace(ctypes.byref(good), 256) > 0
    # missing required outputs -> invalid, before any device work
    assert L.flux_profile_layer(ctypes.byref(good), ctypes.byref(ql), None, None, 10, ctypes.byref(out), None, 0,
                                None) == F.FLUX_E_INVALID
    # T == 0 is a no-op
    assert L.flux_profile_layer(ctypes.byref(good), ctypes.byref(ql), None, None, 0, ctypes.byref(out), None, 0,
                                None) == F.FLUX_OK
    too_many_k = F.make_cfg(64, 128, 8, 9, 0, 8, 0, 1)
    assert L.flux_profile_layer_workspace(ctypes.byref(too_many_k), 10) == 0
    assert L.flux_quantize_weights(3, 0, 0, None, 4, 64, None, None, None) == F.FLUX_E_UNSUPPORTED
    assert L.flux_quantize_weights(4, 12, 0, None, 4, 96, None, None, None) == F.FLUX_E_UNSUPPORTED
    assert L.flux_quantize_weights(4, 48, 0, None, 4, 96, None, None, None) == F.FLUX_E_INVALID
    assert L.flux_merge_experts(0, 4, 12, None, None, None, 2, None, None, None) == F.FLUX_E_UNSUPPORTED
    assert L.flux_merge_experts(0, 4, 16, None, None, None, 5, None, None, None) == F.FLUX_E_INVALID
    assert L.flux_reduce_stats(None, None, 0, None) == F.FLUX_E_INVALID
    # clustering: E > 64, d > E, odd family size, B(l) above the non-tuning count
    numel = (ctypes.c_int64 * 1)(12)
    assert L.flux_expert_features_workspace(28, 64, 1, numel) > 0
    assert L.flux_expert_features_workspace(0, 64, 1, numel) == 0 and L.flux_expert_features_workspace(1, 129, 1, numel) == 0
    ptr = (ctypes.c_void_p * 1)(None)
    assert L.flux_expert_features(1, 129, 1, ptr, numel, 4, None, None, None, None, 0, None) == F.FLUX_E_INVALID
    assert L.flux_expert_features(1, 8, 1, ptr, numel, 9, None, None, None, None, 0, None) == F.FLUX_E_INVALID
    B = (ctypes.c_int32 * 1)(4)
    tun = (ctypes.c_uint8 * 4)(1, 0, 0, 0)
    assert L.flux_cluster_experts(1, 4, 2, 16, 16, B, tun, 10, 16, None, None) == F.FLUX_E_INVALID
    assert L.flux_cluster_experts(1, 4, 40, 16, 16, B, None, 10, 16, None, None) == F.FLUX_E_INVALID


def test_budget_host_matches_oracle(F):
    import oracle
    rng = np.random.default_rng(9)
    for _ in range(30):
        L, E = int(rng.integers(1, 30)), int(rng.integers(2, 65))
        T = int(rng.integers(100, 10**6))
        hist = rng.integers(0, T, size=(L, E)).astype(np.int64)
        B_non = int(rng.integers(0, 2000))
        n_non = rng.integers(0, E + 1, size=L).astype(np.int32) if rng.random() < 0.5 else None
        C, over = F.layer_budget(hist, T, B_non, n_non)
        Cr, _, _, over_r = oracle.layer_budget(hist, T, B_non, n_non)
        assert np.array_equal(C, Cr) and over == over_r


def test_policy_and_batch_validation_without_gpu(F):
    """flux_policy values are validated on the host (before any launch) and change the workspace only
    through the paths they select; flux_merge_experts_batch validates every job on the host."""
    L = F.lib()
    cfg = F.make_cfg(2048, 1408, 64, 6, 2816, 4, 128, 0)
    T = 262144
    ws_default = L.flux_profile_layer_workspace(ctypes.byref(cfg), T)
    assert ws_default > 0
    assert L.flux_profile_layer_workspace_ex(ctypes.byref(cfg), None, T) == ws_default
    assert L.flux_profile_layer_workspace_ex(ctypes.byref(cfg), ctypes.byref(F.make_policy()), T) == ws_default
    # the materialised routed rows need x_perm (T·k·H·2 bytes more); the in-GEMM dequant materialises the
    # rows too but needs no bf16 B copies (E·3·F·H + 3·F_s·H bf16 weights)
    mat = L.flux_profile_layer_workspace_ex(ctypes.byref(cfg), ctypes.byref(F.make_policy(routed_rows=1)), T)
    assert mat - ws_default >= 2 * T * 6 * 2048
    ing = L.flux_profile_layer_workspace_ex(ctypes.byref(cfg), ctypes.byref(F.make_policy(weight_path=2)), T)
    assert mat - ing >= 2 * (64 * 3 * 1408 + 3 * 2816) * 2048
    chain = L.flux_profile_layer_workspace_ex(ctypes.byref(cfg), ctypes.byref(F.make_policy(gemm_chain=2)), T)
    assert chain > ws_default  # chained GEMMs: m-tile ready flags and prefixes
    for bad in (F.make_policy(weight_path=3), F.make_policy(routed_rows=-1), F.make_policy(fused_combine=2),
                F.make_policy(static_tiles=5), F.make_policy(l2_hints=3), F.make_policy(gemm_chain=7)):
        assert L.flux_profile_layer_workspace_ex(ctypes.byref(cfg), ctypes.byref(bad), T) == 0
        out, ql = F.LayerOut(), F.QLayer()
        assert L.flux_profile_layer_ex(ctypes.byref(cfg), ctypes.byref(bad), ctypes.byref(ql), None, None, 10,
                                       ctypes.byref(out), None, 0, None) == F.FLUX_E_INVALID
    assert L.flux_profile_layer_workspace_ex(ctypes.byref(cfg), ctypes.byref(F.make_policy(l2_hints=F.L2_SET | 5)),
                                             T) == ws_default
    # batch merge: counts, numel % 8, null pointers, C > E, compact slot bounds
    jobs = (F.MergeJob * 2)()
    assert L.flux_merge_experts_batch(0, 4, 16, 0, None, 0, None) == F.FLUX_OK  # nothing to do
    assert L.flux_merge_experts_batch(0, 4, 16, 2, None, 0, None) == F.FLUX_E_INVALID
    assert L.flux_merge_experts_batch(0, 4, 12, 2, ctypes.cast(jobs, ctypes.c_void_p), 0, None) == F.FLUX_E_UNSUPPORTED
    assert L.flux_merge_experts_batch(0, 4, 16, 2, ctypes.cast(jobs, ctypes.c_void_p), 0, None) == F.FLUX_E_INVALID
    assert L.flux_merge_experts_batch(0, 4, 16, 257, ctypes.cast(jobs, ctypes.c_void_p), 0, None) == F.FLUX_E_INVALID
    buf = (ctypes.c_uint8 * 64)()
    p = ctypes.addressof(buf) + (-ctypes.addressof(buf)) % 16  # 16-byte aligned host address (not touched)
    for j in jobs:
        j.experts = j.cluster_of = j.alpha = j.out = p
        j.n_clusters = 5  # > E
    assert L.flux_merge_experts_batch(0, 4, 16, 2, ctypes.cast(jobs, ctypes.c_void_p), 0, None) == F.FLUX_E_INVALID
    for j in jobs:
        j.n_clusters, j.n_tuning = 3, 2  # compact: n_tuning + C > E
    assert L.flux_merge_experts_batch(0, 4, 16, 2, ctypes.cast(jobs, ctypes.c_void_p), 1, None) == F.FLUX_E_INVALID
    assert L.flux_merge_experts_batch(0, 4, 16, 2, ctypes.cast(jobs, ctypes.c_void_p), 2, None) == F.FLUX_E_INVALID


def test_bops_host_functions_without_gpu(F):
    """The quantizer-written B operands (flux_layer_bops_bytes & co.): sizes and path queries are host
    functions; the fused quantizer validates its arguments before touching the device."""
    ds = F.make_cfg(2048, 1408, 64, 6, 2816, 4, 128, 0)
    pad64 = lambda v: (v + 63) // 64 * 64  # noqa: E731
    pad128 = lambda v: (v + 127) // 128 * 128  # noqa: E731
    r256 = lambda b: (b + 255) // 256 * 256  # noqa: E731
    want = (r256(2 * 64 * 2 * pad128(1408) * 2048) + r256(2 * 64 * 2048 * pad64(1408)) +
            r256(2 * 2 * pad128(2816) * 2048) + r256(2 * 2048 * pad64(2816)))
    assert F.layer_bops_bytes(ds) == want
    # the dequant-pass path from T·k >= 2048·E (auto policy), always with the pass policy
    assert F.profile_layer_uses_bops(ds, 262144) and not F.profile_layer_uses_bops(ds, 1024)
    assert F.profile_layer_uses_bops(ds, 1024, F.make_policy(F.WEIGHTS_DEQUANT_PASS))
    with pytest.raises(ValueError):
        F.profile_layer_uses_bops(F.make_cfg(2048, 1408, 64, 6, 2816, 3, 128, 0), 1024)  # wbits 3
    # with caller-supplied operands the workspace holds none of them
    T = 262144
    assert F.profile_layer_workspace(ds, T) - F.profile_layer_workspace_bops(ds, T) == want
    lib = F.lib()
    bad_family = lib.flux_quantize_weights_bops(ctypes.byref(ds), 7, F.FLUX_BF16, None, 1, None, None, None, 0, None)
    assert bad_family == 1  # FLUX_E_INVALID
    small_stride = lib.flux_quantize_weights_bops(ctypes.byref(ds), F.FAM_GATE, F.FLUX_BF16, None, 1, None, None,
                                                  ctypes.c_void_p(256), 64, None)
    assert small_stride == 1
    bf16_model = F.make_cfg(2048, 1408, 64, 6, 2816, 16, 0, 0)
    assert lib.flux_quantize_weights_bops(ctypes.byref(bf16_model), F.FAM_GATE, F.FLUX_BF16, None, 1, None, None,
                                          None, 0, None) == 2  # FLUX_E_UNSUPPORTED
