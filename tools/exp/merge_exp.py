"""A/B of merge kernel variants, cold and right after ~1 s of bf16 GEMMs (power-capped clocks, as inside
the bench step).  usage (GPU box): python tools/exp/merge_exp.py"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "libmerge_exp.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                       "-o", so, os.path.join(HERE, "merge_exp.cu")])
lib = ctypes.CDLL(so)
P = ctypes.c_void_p

import synth  # noqa: E402
from paper_2508_19078_b200 import synthetic  # noqa: E402
from paper_2508_19078_b200.driver import merge_model  # noqa: E402

try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    clk = lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)  # noqa: E731
except Exception:
    clk = lambda: -1  # noqa: E731

cfg = synth.CONFIGS["deepseek_moe"]
m = synthetic.master_weights(cfg)
L, E, C = cfg.n_layers, cfg.n_experts, 16
alpha = torch.rand(L, E, device="cuda")
co = (torch.arange(E, dtype=torch.int32, device="cuda") % C).repeat(L, 1).contiguous()
ref = merge_model(m, alpha, co, C)
by = m.gate.numel() * 2 * 3 * (1 + C / E)
outs = [torch.empty_like(ref.gate), torch.empty_like(ref.up), torch.empty_like(ref.down)]
jobs = [(getattr(m, f)[l], co[l], alpha[l], outs[i][l]) for l in range(L) for i, f in enumerate(("gate", "up", "down"))]
numel = m.gate[0, 0].numel()
arr = lambda xs: (P * len(xs))(*[x.data_ptr() for x in xs])  # noqa: E731
ex, cl, al, ou = arr([j[0] for j in jobs]), arr([j[1] for j in jobs]), arr([j[2] for j in jobs]), arr([j[3] for j in jobs])
Cs = (ctypes.c_int * len(jobs))(*([C] * len(jobs)))
a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)


def run_variant(v, bps):
    if v == 0:
        merge_model(m, alpha, co, C, ref)
    else:
        rc = lib.merge_exp(v, bps, len(jobs), E, ctypes.c_longlong(numel), ex, cl, al, ou, Cs,
                           P(torch.cuda.current_stream().cuda_stream))
        assert rc == 0


def timed(fn, hot):
    if hot:
        for _ in range(300):
            a @ a
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), clk()


for v, bps in ((0, 1),):
    run_variant(v, bps)
    torch.cuda.synchronize()
    if v:
        assert torch.equal(outs[0], ref.gate) and torch.equal(outs[2], ref.down), v
    res = []
    for hot in (False, True, True):
        ms, c = timed(lambda: run_variant(v, bps), hot)
        res.append(f"{'hot ' if hot else 'cold'} {ms:6.2f} ms {by / ms / 1e6:6.0f} GB/s @{c} MHz")
    print(f"variant {v} blocks/SM {bps}: " + " | ".join(res), flush=True)
