"""The seeded generator G: CPU twin pinned against a numpy restatement of the
spec (CPU), and the GPU twin bit-identical to the CPU twin (GPU)."""
import numpy as np
import pytest

import synth

M64 = (1 << 64) - 1


def _splitmix64_np(x):
    x = x.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _spec_numpy(spec, rows, row0=0):
    R = np.arange(row0, row0 + rows, dtype=np.uint64)[:, None]
    Cc = np.arange(spec.cols, dtype=np.uint64)[None, :]
    idx = R * np.uint64(spec.cols) + Cc
    h = _splitmix64_np(np.uint64(spec.seed) ^ (np.uint64(spec.stream) << np.uint64(40)) ^ idx)
    n = sum(((h >> np.uint64(16 * i)) & np.uint64(0xFFF)).astype(np.int64) for i in range(4)) - 8190
    v = n.astype(np.float32) * np.float32(spec.c)
    if spec.flags & synth.COL0_C0:
        hb = _splitmix64_np(np.uint64(spec.seed) ^ (np.uint64(spec.stream | (1 << 19)) << np.uint64(40)) ^ R[:, 0])
        nb = sum(((hb >> np.uint64(16 * i)) & np.uint64(0xFFF)).astype(np.int64) for i in range(4)) - 8190
        v[:, 0] = nb.astype(np.float32) * np.float32(spec.c0)
    if spec.flags & synth.COL0_ONE:
        v[:, 0] = 1.0
    if spec.flags & synth.ROW0_ZERO and row0 == 0:
        v[0, :] = 0.0
    return v


def _to_bf16_bits(v):
    u = v.view(np.uint32).astype(np.uint64)
    u = u + 0x7FFF + ((u >> 16) & 1)
    return (u >> 16).astype(np.uint16)


@pytest.mark.parametrize("which", ["x", "router", "gate", "down"])
def test_cpu_twin_matches_spec(which):
    cfg = synth.CONFIGS["toy"]
    spec = {"x": synth.spec_x(cfg), "router": synth.spec_router(cfg, 1),
            "gate": synth.spec_expert(cfg, 1, 3, "gate"), "down": synth.spec_expert(cfg, 0, 5, "down")}[which]
    rows = min(spec.rows, 64)
    want = _spec_numpy(spec, rows)
    got32 = synth.cpu_matrix(spec, rows=rows, dtype="f32")
    assert np.array_equal(got32, want)
    assert np.array_equal(synth.cpu_matrix(spec, rows=rows), _to_bf16_bits(want))
    # row offsets and row lists address the same global rows
    part = synth.cpu_matrix(spec, row0=3, rows=5)
    assert np.array_equal(part, synth.cpu_matrix(spec, rows=8)[3:])
    assert np.array_equal(synth.cpu_rows(spec, [7, 2, 7]), synth.cpu_matrix(spec, rows=8)[[7, 2, 7]])


def test_distribution_moments():
    cfg = synth.CONFIGS["deepseek_moe"]
    x = synth.bf16_bits_to_f32(synth.cpu_matrix(synth.spec_x(cfg), rows=512))
    assert np.all(x[:, 0] == 1.0)
    assert abs(x[:, 1:].std() - 1.0) < 0.01 and abs(x[:, 1:].mean()) < 0.01
    wd = synth.bf16_bits_to_f32(synth.cpu_matrix(synth.spec_expert(cfg, 0, 0, "down")))
    assert np.all(wd[0] == 0) and abs(wd[1:].std() * np.sqrt(cfg.ffn) - 0.1) < 0.002


@pytest.mark.gpu
def test_gpu_twin_bit_identical():
    import torch
    cfg = synth.CONFIGS["deepseek_moe"]
    for spec, row0, rows in [(synth.spec_x(cfg), 12345, 300), (synth.spec_router(cfg, 3), 0, 64),
                             (synth.spec_expert(cfg, 2, 17, "down"), 0, 2048),
                             (synth.spec_expert(cfg, 1, synth.SHARED_SLOT, "gate"), 0, 2816)]:
        for dt, tdt in (("bf16", torch.bfloat16), ("f32", torch.float32)):
            d = torch.empty(rows, spec.cols, dtype=tdt, device="cuda")
            synth.gpu_fill(d, spec, row0=row0)
            cpu = synth.cpu_matrix(spec, row0=row0, rows=rows, dtype=dt)
            g = d.view(torch.int16).cpu().numpy().view(np.uint16) if dt == "bf16" else d.cpu().numpy()
            assert np.array_equal(g, cpu), (spec, dt)
