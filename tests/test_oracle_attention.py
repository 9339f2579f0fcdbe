"""Pins for O13 (NEXT-3): the attention-weighted importance α_e = f_e·ā_e of eq.(2),
kept as fixed-point integer sums A_e = Σ_{t∈D_e} RNE(a_t·2^24) (reading R15) — CPU only."""
from fractions import Fraction

import numpy as np

import oracle
import synth


def _ids(rng, T, E, k):
    return np.stack([rng.choice(E, size=k, replace=False) for _ in range(T)]).astype(np.int32)


def test_alpha_is_frequency_times_mean_attention_exactly():
    rng = np.random.default_rng(0)
    T, E, k = 50, 7, 3
    ids = _ids(rng, T, E, k)
    m = rng.integers(0, 1 << 24, size=T)  # a_t = m_t·2^-24: representable, so the fixed point is exact
    a = (m.astype(np.float64) / 2 ** 24).astype(np.float32)
    A = oracle.attention_hist(ids, a, E)
    for e in range(E):
        members = [t for t in range(T) if e in ids[t]]
        f = Fraction(len(members), T)
        abar = sum(Fraction(int(m[t]), 1 << 24) for t in members) / len(members) if members else Fraction(0)
        assert Fraction(int(A[e]), (1 << 24) * T) == f * abar, e


def test_unit_attention_reduces_to_the_histogram():
    rng = np.random.default_rng(1)
    ids = _ids(rng, 80, 9, 4)
    A = oracle.attention_hist(ids, np.ones(80, np.float32), 9)
    hist, _, _, _ = oracle.permute(ids, 9)
    assert np.array_equal(A, hist * (1 << 24))


def test_fixed_point_rounds_half_to_even_and_skips_empty_picks():
    ids = np.array([[0, 1], [1, -1], [2, 0]], np.int32)
    a = np.array([2.0 ** -25, 3 * 2.0 ** -25, 0.75], np.float32)  # 0.5 -> 0, 1.5 -> 2 (ties to even)
    A = oracle.attention_hist(ids, a, 3)
    assert list(A) == [0 + int(0.75 * 2 ** 24), 0 + 2, int(0.75 * 2 ** 24)]


def test_attention_values_generator_is_nonnegative_after_abs():
    cfg = synth.CONFIGS["toy"]
    a = np.abs(synth.cpu_matrix(synth.spec_attn(cfg, 0), dtype="f32")[:, 0])
    assert a.shape == (cfg.tokens,) and np.all(a >= 0) and 0.5 < a.mean() < 1.1  # E|N(0,1)| = 0.80
