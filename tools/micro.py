"""Micro-benchmarks of single libflux entry points at BASELINE sizes (diagnostics, not bench lines).

usage: python tools/micro.py [quantize] [merge] [features] [layer]
Each prints achieved algorithmic GB/s (HBM-bound kernels) against MEASURED_PEAKS.json.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2508_19078_b200 as F  # noqa: E402
import synth  # noqa: E402


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p))["hbm_gbs"] if os.path.exists(p) else 6650.0


def quantize():
    cfg = synth.CONFIGS["deepseek_moe"]
    R, K = 4 * cfg.n_experts * cfg.ffn, cfg.hidden  # 4 layers of routed gate weights
    w = torch.randn(R, K, device="cuda").to(torch.bfloat16)
    for wbits, g in ((4, 128), (8, 0)):
        q = torch.empty(R, K // (2 if wbits == 4 else 1), dtype=torch.uint8, device="cuda")
        s = torch.empty(R, K // (g or K), dtype=torch.float32, device="cuda")
        ms = timed(lambda: F.quantize_weights(w, wbits, g, q, s))
        by = w.numel() * 2 + q.numel() + s.numel() * 4
        print(f"quantize INT{wbits} g={g}: {ms:.3f} ms  {by / ms / 1e6:.0f} GB/s  ({by / ms / 1e6 / peak():.2f} of peak)")


def merge():
    cfg = synth.CONFIGS["deepseek_moe"]
    E, C = cfg.n_experts, 16
    numel = cfg.ffn * cfg.hidden
    W = torch.randn(E, numel, device="cuda").to(torch.bfloat16)
    cl = torch.arange(E, dtype=torch.int32, device="cuda") % C
    al = torch.rand(E, device="cuda")
    out = torch.empty(C, numel, dtype=torch.bfloat16, device="cuda")
    ms = timed(lambda: F.merge_experts(W, cl, al, C, out))
    by = W.numel() * 2 + out.numel() * 2
    print(f"merge 64->16 bf16 one family/layer: {ms:.3f} ms  {by / ms / 1e6:.0f} GB/s  ({by / ms / 1e6 / peak():.2f})")


def merge_model():
    """a8 over all 28 DeepSeek layers × 3 families, balanced vs unbalanced clusters, cold vs power-capped."""
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import merge_model as mm
    cfg = synth.CONFIGS["deepseek_moe"]
    m = synthetic.master_weights(cfg)
    L, E, C = cfg.n_layers, cfg.n_experts, 16
    alpha = torch.rand(L, E, device="cuda")
    by = m.gate.numel() * 2 * 3 * (1 + C / E)
    bal = (torch.arange(E, dtype=torch.int32, device="cuda") % C).repeat(L, 1).contiguous()
    g = torch.Generator(device="cuda").manual_seed(1)
    unb = torch.randint(0, C, (L, E), generator=g, device="cuda", dtype=torch.int32)
    unb[:, :C] = torch.arange(C, dtype=torch.int32, device="cuda")
    out = mm(m, alpha, unb if os.environ.get("MICRO_MERGE_FIRST") == "unbalanced" else bal, C)  # first launch (ncu -c 1)
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    for name, cl in (("balanced", bal), ("unbalanced", unb)):
        ms = timed(lambda: mm(m, alpha, cl, C, out), reps=5, warm=2)
        print(f"merge_model {name}: {ms:.2f} ms  {by / ms / 1e6:.0f} GB/s ({by / ms / 1e6 / peak():.2f})")
        for _ in range(300):  # ~1 s of bf16 GEMMs: power-capped clocks, like inside the bench step
            a @ a
        ms = timed(lambda: mm(m, alpha, cl, C, out), reps=1, warm=0)
        print(f"merge_model {name} after GEMM load: {ms:.2f} ms  {by / ms / 1e6:.0f} GB/s ({by / ms / 1e6 / peak():.2f})")


def features():
    """§5.2 C1 over all 28 DeepSeek layers (gate|up|down of 64 experts) + C2 K-Means into 16 clusters."""
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import cluster_model, expert_features_model
    cfg = synth.CONFIGS["deepseek_moe"]
    m = synthetic.master_weights(cfg)
    hist = torch.randint(0, 1000, (cfg.n_layers, cfg.n_experts), dtype=torch.int64, device="cuda")
    F.timing_read(reset=True)
    F.timing_enable(True)
    ms = timed(lambda: expert_features_model(m, 16), reps=5, warm=2)
    feats, _, _ = expert_features_model(m, 16)
    ms_k = timed(lambda: cluster_model(feats, hist, 16), reps=5, warm=2)
    F.timing_enable(False)
    k = F.timing_read(reset=True)
    by = m.gate.numel() * 2 * 3
    print(f"features 28 layers: {ms:.2f} ms  {by / ms / 1e6:.0f} GB/s ({by / ms / 1e6 / peak():.2f} of HBM); "
          f"kmeans {ms_k:.3f} ms;", {n: round(v[0] / max(v[1], 1), 4) for n, v in k.items() if v[1]})
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    for _ in range(300):  # ~1 s of bf16 GEMMs: power-capped clocks, like inside the bench step
        a @ a
    ms = timed(lambda: expert_features_model(m, 16), reps=1, warm=0)
    print(f"features 28 layers after GEMM load: {ms:.2f} ms  {by / ms / 1e6:.0f} GB/s ({by / ms / 1e6 / peak():.2f})")


def layer(name="deepseek_moe"):
    from paper_2508_19078_b200.driver import ModelShape, Profiler, QuantizedModel
    from paper_2508_19078_b200 import synthetic
    cfg = synth.CONFIGS[name].with_(n_layers=1)
    if os.environ.get("MICRO_TOKENS"):  # token-count override for scaling experiments
        cfg = cfg.with_(tokens=int(os.environ["MICRO_TOKENS"]))
    shape = ModelShape.of(cfg)
    qm = QuantizedModel(shape)
    qm.quantize_from(synthetic.master_weights(cfg))
    chain = int(os.environ.get("MICRO_CHAIN", "0"))  # flux_policy.gemm_chain (0 auto, 1 off, 2 on)
    wp = int(os.environ.get("MICRO_WP", "0"))  # flux_policy.weight_path (0 auto, 1 dequant pass, 2 in-GEMM)
    prof = Profiler(shape, cfg.tokens, with_de=True, policy=F.make_policy(weight_path=wp, gemm_chain=chain))
    x = synthetic.tokens(cfg, 0, cfg.tokens)
    F.timing_read(reset=True)
    F.timing_enable(True)
    ms = timed(lambda: prof.run(qm, x), reps=5, warm=2)
    F.timing_enable(False)
    k = F.timing_read(reset=True)
    print(f"one {name} layer, {cfg.tokens} tokens, weight_path={wp} chain={chain}: {ms:.2f} ms;",
          {n: round(v[0] / max(v[1], 1), 3) for n, v in k.items() if v[1]})


def layer_llama():
    layer("llama_moe")


if __name__ == "__main__":
    for what in sys.argv[1:] or ["quantize", "merge", "layer"]:
        globals()[what]()
