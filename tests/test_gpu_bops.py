"""The dequantization pass folded into the quantizer (flux_quantize_weights_bops, include/flux.h): one
pass over the master weights writes the codes and scales AND every layer's bf16 B operands.  Where the
operands come from must not change a byte:
  * q and s equal flux_quantize_weights' (the bit-exact a0 of tests/test_gpu_parity.py);
  * each layer's operands equal flux_dequantize_layer's (the per-call pass) byte for byte — INT4/INT2
    grouped, INT8 per channel, shared experts, F not a multiple of 128 (interleaved pad rows);
  * profiling with them (flux_profile_layer_bops) equals profiling without, bitwise, over several layers."""
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

S = synth.BASE_SEED
CFGS = {
    "int4_g128_shared": synth.MoEConfig("b_int4_sh", 3, 256, 16, 2, 256, 384, 4, 128, 0, 4096, S + 80),
    "int8_channel_pad": synth.MoEConfig("b_int8", 3, 192, 8, 2, 176, 0, 8, 0, 1, 2048, S + 81),
    "int2_g64": synth.MoEConfig("b_int2", 2, 256, 8, 2, 128, 192, 2, 64, 0, 2048, S + 82),
    "int4_channel_pad_shared": synth.MoEConfig("b_int4_pad", 2, 128, 8, 3, 160, 96, 4, 0, 0, 3000, S + 83),
    "deepseek_layers": synth.CONFIGS["deepseek_moe"].with_(n_layers=2, tokens=16384, name="b_ds"),
}


def _pair(cfg):
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import ModelShape, QuantizedModel
    shape = ModelShape.of(cfg)
    m = synthetic.master_weights(cfg)
    qa = QuantizedModel(shape)
    qa.quantize_from(m)
    qb = QuantizedModel(shape, with_bops=True)
    assert qb.bops is not None
    qb.quantize_from(m)
    torch.cuda.synchronize()
    return shape, qa, qb


@pytest.mark.parametrize("name", list(CFGS))
def test_fused_operands_equal_pass(name):
    import paper_2508_19078_b200 as F
    cfg = CFGS[name]
    shape, qa, qb = _pair(cfg)
    for f in ("gate", "up", "down") + (("sh_gate", "sh_up", "sh_down") if cfg.shared_ffn else ()):
        assert torch.equal(getattr(qa, f + "_q"), getattr(qb, f + "_q")), f
        assert torch.equal(getattr(qa, f + "_s"), getattr(qb, f + "_s")), f
    c = shape.ccfg(0)
    for l in range(cfg.n_layers):
        ref = torch.zeros(F.layer_bops_bytes(c), dtype=torch.uint8, device="cuda")
        F.dequantize_layer(c, qa.qlayer(l), ref)
        torch.cuda.synchronize()
        assert torch.equal(qb.bops[l], ref), (l, (qb.bops[l] != ref).nonzero()[:8].ravel().tolist())


@pytest.mark.parametrize("name", ["int4_g128_shared", "int8_channel_pad", "int2_g64", "deepseek_layers"])
def test_profile_with_fused_operands_bitwise(name):
    import paper_2508_19078_b200 as F
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import Profiler
    cfg = CFGS[name]
    shape, qa, qb = _pair(cfg)
    pol = F.make_policy(F.WEIGHTS_DEQUANT_PASS)
    assert F.profile_layer_uses_bops(shape.ccfg(0), cfg.tokens, pol)
    x = synthetic.tokens(cfg, 0, cfg.tokens)
    res = []
    for qm in (qa, qb):
        prof = Profiler(shape, cfg.tokens, with_de=True, policy=pol)
        ys = []
        prof.run(qm, x, on_layer=lambda l, y: ys.append(y.clone()))
        torch.cuda.synchronize()
        res.append((ys, prof.ids.clone(), prof.w.clone(), prof.hist.clone(), prof.offsets.clone(),
                    prof.token_index.clone()))
    (y0, *r0), (y1, *r1) = res
    for a, b in zip(y0, y1):
        assert torch.equal(a, b)
    for a, b in zip(r0, r1):
        assert torch.equal(a, b)


def test_fused_quantizer_argument_errors():
    import paper_2508_19078_b200 as F
    cfg = CFGS["int2_g64"]
    shape, qa, qb = _pair(cfg)
    c = shape.ccfg(0)
    from paper_2508_19078_b200 import synthetic
    m = synthetic.master_weights(cfg)
    with pytest.raises(F.FluxError):  # no such family
        F.quantize_weights_bops(c, 6, m.gate, cfg.n_layers, qa.gate_q, qa.gate_s, qb.bops)
    small = torch.zeros(cfg.n_layers, 64, dtype=torch.uint8, device="cuda")
    with pytest.raises(F.FluxError):  # a layer stride below flux_layer_bops_bytes
        F.quantize_weights_bops(c, F.FAM_GATE, m.gate, cfg.n_layers, qa.gate_q, qa.gate_s, small)
