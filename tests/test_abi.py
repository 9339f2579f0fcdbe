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
