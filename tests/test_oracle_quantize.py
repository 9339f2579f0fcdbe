"""Pins for oracle O1 (quantize) and the bf16 rounding helper — CPU only.

The paper names the bit widths (Fig. 5 legend bit-2/4/8, "e.g.
INT4") but no scheme; R1 fixes it.  Pins: hand-derived worked
examples (tests/golden/quantize_examples.json), the round-trip bound
|w - q·s| <= s/2 that holds for any correct symmetric RNE quantizer, range and
saturation properties, and the canonical INT4 packing.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _s(spec, w):
    if isinstance(spec, (int, float)):
        return np.float32(spec)
    # "fl32(fl32(a)/b)" forms
    if spec == "fl32(fl32(0.9)/127)":
        return np.float32(np.float32(0.9) / np.float32(127))
    if spec == "fl32(fl32(0.9)/7)":
        return np.float32(np.float32(0.9) / np.float32(7))
    if spec == "fl32(8/7)":
        return np.float32(np.float32(8) / np.float32(7))
    raise KeyError(spec)


def test_worked_examples():
    g = json.load(open(os.path.join(GOLD, "quantize_examples.json")))
    for c in g["cases"]:
        w = np.array([c["w"]], np.float32)
        q, s = oracle.quantize(w, c["wbits"], 0)
        assert list(q[0]) == c["q"], c
        assert s[0, 0] == _s(c["s"], w), c


def test_pack_int4_example():
    g = json.load(open(os.path.join(GOLD, "quantize_examples.json")))["pack_int4"]
    out = oracle.pack_int4(np.array([g["q"]], np.int8))
    assert list(out[0]) == g["bytes"]


def test_pack_int2_example():
    g = json.load(open(os.path.join(GOLD, "quantize_examples.json")))["pack_int2"]
    out = oracle.pack_int2(np.array([g["q"]], np.int8))
    assert list(out[0]) == g["bytes"]


@pytest.mark.parametrize("wbits,g", [(8, 0), (4, 128), (4, 32), (8, 64), (2, 128), (2, 0)])
def test_round_trip_bound_and_range(wbits, g):
    rng = np.random.default_rng(wbits * 1000 + g)
    R, K = 37, 256
    w = (rng.standard_normal((R, K)) * rng.uniform(0.01, 3, size=(R, 1))).astype(np.float32)
    w[3, :] = 0.0  # an all-zero row/group
    q, s = oracle.quantize(w, wbits, g)
    gg = g or K
    qmax = (1 << (wbits - 1)) - 1
    srow = np.repeat(s.astype(np.float64), gg, axis=1)
    err = np.abs(w.astype(np.float64) - q.astype(np.float64) * srow)
    assert np.all(err <= srow / 2 + 1e-300)
    assert q.min() >= -qmax and q.max() <= qmax  # symmetric: -qmax-1 never produced
    # the element of largest magnitude of every non-zero group maps to +-qmax exactly
    wg = np.abs(w).reshape(R, K // gg, gg)
    qg = np.abs(q.astype(np.int32)).reshape(R, K // gg, gg)
    nz = wg.max(axis=2) > 0
    assert np.all(qg.max(axis=2)[nz] == qmax)
    assert np.all(q[3] == 0) and np.all(s[3] == 0)


def test_ties_to_even_in_bulk():
    # w = (n + 1/2)·s exactly for s = 1: every value is a tie; RNE picks the even neighbour
    w = np.array([[127.0] + [n + 0.5 for n in range(-10, 10)] + [0.0] * 11], np.float32)
    q, s = oracle.quantize(w, 8, 0)
    assert s[0, 0] == 1.0
    for n, qq in zip(range(-10, 10), q[0, 1:21]):
        lo, hi = n, n + 1
        assert qq == (lo if lo % 2 == 0 else hi)


def test_pack_roundtrip_random():
    rng = np.random.default_rng(5)
    q = rng.integers(-8, 8, size=(9, 64)).astype(np.int8)
    p = oracle.pack_int4(q)
    lo = (p & 0xF).astype(np.int16)
    hi = (p >> 4).astype(np.int16)
    lo[lo > 7] -= 16
    hi[hi > 7] -= 16
    back = np.empty_like(q)
    back[:, 0::2] = lo
    back[:, 1::2] = hi
    assert np.array_equal(back, q)


def test_bf16_round_hand_cases():
    u = 2.0 ** -7  # bf16 ulp at 1.0
    cases = {
        1.0 + u / 2: 1.0,            # tie -> even (1.0)
        1.0 + 3 * u / 2: 1.0 + 2 * u,  # tie between odd 1+u and even 1+2u
        1.0 + u / 2 + 1e-12: 1.0 + u,  # just above the tie
        -(1.0 + u / 2): -1.0,
        3.0: 3.0,
        0.0: 0.0,
    }
    for v, want in cases.items():
        assert oracle.bf16_round([v])[0] == want, v


def test_bf16_round_matches_torch_on_fp32_values():
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(0)
    v = (rng.standard_normal(10000) * 10.0 ** rng.uniform(-6, 6, 10000)).astype(np.float32)
    ref = torch.from_numpy(v).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(oracle.bf16_round(v.astype(np.float64)), ref)


def test_pack_int2_roundtrip_random():
    rng = np.random.default_rng(6)
    q = rng.integers(-2, 2, size=(7, 64)).astype(np.int8)
    p = oracle.pack_int2(q).astype(np.int16)
    back = np.empty_like(q)
    for j in range(4):
        v = (p >> (2 * j)) & 0x3
        v[v > 1] -= 4
        back[:, j::4] = v
    assert np.array_equal(back, q)
