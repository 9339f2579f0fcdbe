"""bench.py — profiled tokens/s/box of the Flux hot path on B200 (BASELINE.json metric).

One step = one participant round of the hot path (all rows):
  a0 quantize the model (INT4 g128 / INT8)   flux_quantize_weights
  a1-a6 profile the rank's tokens through all layers: router+top-k+histogram,
        D_e permutation, grouped SwiGLU expert GEMMs (routed + shared), combine
                                             flux_profile_layer x L
  a7 all-reduce the int64 histograms         flux_reduce_stats (NCCL)
  a8-pre eq.(1) layer budgets (host)         flux_layer_budget
  §5.2 expert clustering (NEXT-1): PCA features of every layer's experts
        + fused K-Means into 16 clusters from the reduced counts
                                             flux_expert_features, flux_cluster_experts
  a8 eq.(2) merge 64 -> 16 experts per layer, α = f (bf16)   flux_merge_experts
Data parallel over tokens, weak scaling: every rank profiles its own shard of
`tokens` tokens (the N=8 run is BASELINE.json's 2M-token DP config).

usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config deepseek_moe|llama_moe]
       python bench.py --impl reference ...   (the CPU oracle, timed on the host cores)
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "profiled tokens/sec/box (quantized MoE fwd + expert stats) at 1/2/4/8 B200; % roofline"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


def workload_config(cfg, tokens_per_gpu, n_gpus):
    return {
        "workload": f"{cfg.name}: INT{cfg.wbits}{'-g' + str(cfg.group_size) if cfg.group_size else ' per-channel'} "
                    f"quantize + profile {cfg.n_layers} layers + NCCL hist all-reduce + PCA/K-Means clustering + eq.(2) merge "
                    f"{cfg.n_experts}->{max(1, cfg.n_experts // 4)} bf16",
        "layers": cfg.n_layers, "hidden": cfg.hidden, "experts": cfg.n_experts, "shared_ffn": cfg.shared_ffn,
        "top_k": cfg.top_k, "ffn": cfg.ffn, "wbits": cfg.wbits, "group_size": cfg.group_size,
        "tokens_per_gpu": tokens_per_gpu, "tokens_total": tokens_per_gpu * n_gpus,
        "parallelism": f"dp{n_gpus}",
        "l2": "inputs larger than L2 (x shard = %.2f GiB, weights %.1f GiB)" % (
            tokens_per_gpu * cfg.hidden * 2 / 2**30,
            cfg.n_layers * (cfg.n_experts * 3 * cfg.ffn + 3 * cfg.shared_ffn) * cfg.hidden * 2 / 2**30),
    }


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, path):
        self.path = path
        self.proc = None

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self, gpus):
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, mx, reasons = [], [], set()
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9 or not p[0].isdigit() or int(p[0]) not in gpus:
                continue
            try:
                sm.append(float(p[1]))
                mx.append(float(p[2]))
            except ValueError:
                continue
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"), p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------------ reference arm
def oracle_rate(cfg, n_tok, n_layers, T_full):
    """Time the oracle (as it stands) on n_tok tokens through n_layers layers; returns (tokens/s scaled to a full
    L-layer pass, threads, sample description, seconds)."""
    import oracle.model as om
    t0 = time.perf_counter()
    q = [om.quantized_layer(cfg, l) for l in range(n_layers)]
    om.profile_tokens(cfg, np.arange(n_tok), layers=n_layers, quantized=q)
    dt = time.perf_counter() - t0
    per_tok = dt / n_tok * (cfg.n_layers / n_layers)
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    sample = (f"{n_tok} tokens x {n_layers} of {cfg.n_layers} layers (oracle quantization of those layers + "
              f"free-running fp64 layer forward), scaled to a {cfg.n_layers}-layer pass; merge not included")
    return 1.0 / per_tok, threads, sample, dt


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    n_tok, n_layers = (args.ref_tokens, args.ref_layers)
    rates = []
    for i in range(args.warmup + args.steps):
        r, threads, sample, dt = oracle_rate(cfg, n_tok, n_layers, cfg.tokens)
        if i >= args.warmup:
            rates.append(r)
    v = statistics.median(rates)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * cfg.tokens / v,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, cfg.tokens, 1),
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": threads, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------ our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="flux", choices=["flux", "reference"])
    ap.add_argument("--config", default="deepseek_moe")
    ap.add_argument("--tokens", type=int, default=0, help="tokens per GPU (default: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-tokens", type=int, default=64)  # oracle sample: ~10 s of host CPU work (16 cores)
    ap.add_argument("--ref-layers", type=int, default=2)
    ap.add_argument("--clusters", type=int, default=0)
    ap.add_argument("--rounds", type=int, default=2,
                    help="NEXT-4: serial vs stale-profiling participant rounds measured after the run (0 = skip)")
    ap.add_argument("--alpha", default="f", choices=["f", "attn"],
                    help="merge importance: activation frequency (BASELINE config) or f·ā with synthetic attention")
    ap.add_argument("--wbits", type=int, default=0, choices=[0, 2, 4, 8],
                    help="override the config's bit level (2 = the paper's bit-2 ablation, NEXT-3)")
    ap.add_argument("--error-tokens", type=int, default=8192,
                    help="tokens for the merged model's output error after the timed run (0 = skip)")
    ap.add_argument("--features-stream", default="main", choices=["main", "side"],
                    help="PCA features in stream order (default) or on a side stream overlapping the profiling")
    ap.add_argument("--clustering", default="pca", choices=["pca", "seeded"],
                    help="pca: §5.2 PCA + K-Means on the GPU inside the step; seeded: a fixed balanced partition")
    args = ap.parse_args()

    import synth
    cfg = synth.CONFIGS[args.config]
    if args.wbits:
        cfg = cfg.with_(wbits=args.wbits, name=f"{cfg.name}_int{args.wbits}")
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2508_19078_b200 as F
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import (ModelShape, Profiler, QuantizedModel, budgets, cluster_model,
                                              expert_features_model, feature_dim, merge_model, shard)

    T = args.tokens or cfg.tokens
    T_total = T * world
    C = args.clusters or max(1, cfg.n_experts // 4)
    shape = ModelShape.of(cfg)
    L, E, H, k = cfg.n_layers, cfg.n_experts, cfg.hidden, cfg.top_k
    stream = torch.cuda.current_stream()

    # ---- setup (not timed): synthetic master weights, this rank's token shard, buffers, NCCL comm
    masters = synthetic.master_weights(cfg)
    qm = QuantizedModel(shape)
    prof = Profiler(shape, T, with_de=True)
    t0, _ = shard(rank, world, T)  # this rank's contiguous slice of the global token stream
    x = synthetic.tokens(cfg, t0, T)
    cluster_of = torch.from_numpy(synth.cluster_assignment(cfg, C)).cuda()
    side = torch.cuda.Stream()
    ev_start, ev_feat = torch.cuda.Event(), torch.cuda.Event()
    d_feat = feature_dim(E)
    alpha = torch.empty(L, E, dtype=torch.float32, device="cuda")
    alpha_host = torch.empty(L, E, dtype=torch.float32).pin_memory()
    hist_host = torch.empty(L, E, dtype=torch.int64).pin_memory()
    ahist_host = torch.empty(L, E, dtype=torch.int64).pin_memory()
    attn = synthetic.attention_values(cfg, t0, T) if args.alpha == "attn" else None
    merged = None
    uid = F.Comm.unique_id() if rank == 0 else None
    if world > 1:
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    comm = F.Comm(uid, world, rank)
    budget_out = {}

    def step(x_in, before_profile=None, after_profile=None):
        nonlocal merged, cluster_of
        if args.clustering == "pca" and args.features_stream == "side":  # §5.2 C1 overlapping a0-a7
            ev_start.record(stream)
            side.wait_event(ev_start)
            with torch.cuda.stream(side):
                feats, _, _ = expert_features_model(masters, d_feat, stream=side)
                ev_feat.record(side)
            feats.record_stream(stream)
        elif args.clustering == "pca":                              # §5.2 C1 in stream order (reads masters only)
            feats, _, _ = expert_features_model(masters, d_feat)
            ev_feat.record(stream)
        qm.quantize_from(masters)                                   # a0
        if before_profile:
            before_profile()
        prof.run(qm, x_in, attn=attn)                               # a1-a6 (hist zeroed first)
        if after_profile:
            after_profile()
        comm.reduce_stats(prof.hist)                                # a7
        if attn is not None:                                        # NEXT-3: Σ_{t∈D_e} a_t, fixed point
            comm.reduce_stats(prof.ahist)
            ahist_host.copy_(prof.ahist, non_blocking=True)
        if args.clustering == "pca":                                # §5.2 C2: K-Means from the reduced counts
            stream.wait_event(ev_feat)
            cluster_of = cluster_model(feats, prof.hist, C)
        hist_host.copy_(prof.hist, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        h = hist_host.numpy()
        if attn is None:
            alpha_host.copy_(torch.from_numpy((h / float(T_total)).astype(np.float32)))  # α = f
        else:  # α = f·ā = Σ_{t∈D_e} a_t / T (eq.(2); R15)
            alpha_host.copy_(torch.from_numpy((ahist_host.numpy() / (16777216.0 * T_total)).astype(np.float32)))
        Cl, over = budgets(h, T_total, C * L)                       # a8-pre, eq.(1)
        budget_out["C"] = Cl
        alpha.copy_(alpha_host, non_blocking=True)
        merged = merge_model(masters, alpha, cluster_of, C, merged)  # a8, eq.(2)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(x)
    barrier()

    clocks = ClockSampler(os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out"))
                                       else "/tmp", f"clocks_rank{rank}.csv"))
    if rank == 0:
        clocks.start()
    F.timing_read(reset=True)
    F.timing_enable(True)
    launches0 = F.launch_count()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step(x)
    ev1.record(stream)
    barrier()
    F.timing_enable(False)
    launches = F.launch_count() - launches0
    kern = F.timing_read(reset=True)
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clk = clocks.stop(gpus=set(range(world))) if rank == 0 else None

    # ---- e2e: the same step through the public API with host buffers: every step copies its tokens
    #      H2D from pinned memory and its profiling result (reduced histogram + D_e CSR of every
    #      layer) D2H.  The copies run on a copy stream, pipelined like a serving loop: step i+1's
    #      tokens go up while step i profiles (double-buffered x), and step i's D_e comes down while
    #      it clusters and merges; step i+1 profiles only after that copy has drained D_e.
    x_host = x.cpu().pin_memory()
    off_host = torch.empty_like(prof.offsets, device="cpu").pin_memory()
    ti_host = torch.empty_like(prof.token_index, device="cpu").pin_memory()
    x_dev = [torch.empty_like(x), torch.empty_like(x)]
    h2d = x_host.numel() * x_host.element_size()
    d2h = hist_host.numel() * 8 + off_host.numel() * 4 + ti_host.numel() * 4
    cstream = torch.cuda.Stream()
    ev_h2d = [torch.cuda.Event(), torch.cuda.Event()]
    ev_prof, ev_d2h = torch.cuda.Event(), torch.cuda.Event()
    state = {"i": 0, "n": 1, "d2h_pending": False}

    def h2d_into(buf):
        with torch.cuda.stream(cstream):
            x_dev[buf].copy_(x_host, non_blocking=True)
            ev_h2d[buf].record(cstream)

    def before_profile():
        stream.wait_event(ev_h2d[state["i"] % 2])  # this step's tokens are on the device
        if state["d2h_pending"]:
            stream.wait_event(ev_d2h)  # the previous step's D_e has left the device

    def after_profile():
        ev_prof.record(stream)
        with torch.cuda.stream(cstream):
            cstream.wait_event(ev_prof)
            off_host.copy_(prof.offsets, non_blocking=True)
            ti_host.copy_(prof.token_index, non_blocking=True)
            ev_d2h.record(cstream)
        state["d2h_pending"] = True
        if state["i"] + 1 < state["n"]:
            h2d_into((state["i"] + 1) % 2)  # the next step's tokens (that buffer's reader is done)

    def e2e_step():
        step(x_dev[state["i"] % 2], before_profile, after_profile)
        state["i"] += 1

    def e2e_drain():
        ev_d2h.synchronize()  # the last step's D_e is on the host
        cstream.synchronize()

    state["n"] = 1
    h2d_into(0)
    e2e_step()
    e2e_drain()
    barrier()
    state.update(i=0, n=args.steps, d2h_pending=False)
    ev0.record(stream)
    cstream.wait_event(ev0)
    h2d_into(0)  # the first timed step's tokens: inside the timed region
    for _ in range(args.steps):
        e2e_step()
    e2e_drain()
    ev1.record(stream)
    barrier()
    ms_e2e = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())

    # ---- merge quality of the round's merged model (not timed): the paper's output error —
    #      mean cosine distance between the final outputs of the compact model (tuning experts + the
    #      eq.(2) merges, gate re-routed, bf16) and of the original bf16 model on the first tokens of x
    merr = None
    if args.error_tokens > 0 and rank == 0:
        from paper_2508_19078_b200.driver import compact_model, dense_model
        n_err = min(args.error_tokens, T)
        dense = dense_model(masters)
        comp = compact_model(masters, alpha, cluster_of, C, 0)
        outs = []
        for mdl in (dense, comp):
            pr = Profiler(mdl.shape, n_err, with_de=False)
            outs.append(pr.run(mdl, x[:n_err]).clone())
            del pr
        merr = {"value": float(F.output_error(outs[1], outs[0]).item()), "tokens": n_err,
                "clusters_per_layer": C, "alpha": args.alpha, "clustering": args.clustering,
                "what": "mean cosine distance of final token outputs, merged vs original bf16 model (P:686-689)"}
        del comp, outs

    # ---- NEXT-4 stale profiling (not part of the timed step): participant rounds, serial (Fig. 7a) vs
    #      stale (Fig. 7b), each round = profile + merge into the compact model + its forward over the
    #      local fine-tuning tokens (the first quarter of x); CUDA events on the round's streams
    stale = None
    if args.rounds > 0 and world == 1:
        from paper_2508_19078_b200.rounds import Participant
        part = Participant(masters, x, x[: max(1, T // 4)], comm, C, T_total, clustering=args.clustering,
                           seeded_cluster_of=cluster_of)
        part.round_serial()  # warm-up; leaves f^r for the first stale round
        ser = [part.round_serial() for _ in range(args.rounds)]
        stl = [part.round_stale() for _ in range(args.rounds)]
        med = lambda rs, k: statistics.median(r[k] for r in rs)  # noqa: E731
        stale = {"serial_round_ms": med(ser, "round_ms"), "serial_ft_start_ms": med(ser, "ft_start_ms"),
                 "stale_round_ms": med(stl, "round_ms"), "stale_ft_start_ms": med(stl, "ft_start_ms"),
                 "stale_profile_done_ms": med(stl, "profile_done_ms"), "rounds": args.rounds,
                 "finetune_tokens": int(max(1, T // 4)),
                 "what": "participant round = profile + merge (compact model) + compact-model forward over the "
                         "fine-tuning tokens; stale = merge with f^(r-1) at once, profile on a low-priority stream"}
        del part

    if rank == 0:
        peaks, peak_src = load_peaks()
        value = T_total * args.steps / (ms / 1000.0)
        # dominant kernel: the gate/up grouped GEMM (routed + shared in one launch, once per layer)
        gu_ms, gu_n = kern.get("gemm_gate_up", (0.0, 0))
        flop_gu = 2.0 * T * (k * H * 2 * cfg.ffn + H * 2 * cfg.shared_ffn)  # per launch (one layer)
        achieved = flop_gu / (gu_ms / gu_n / 1000.0) / 1e12 if gu_n else None
        peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            # dram read+write bytes per launch from the committed `ncu --set full` capture (profiles/)
            traffic = json.load(open(tp)).get(f"{args.config}:{T}:K3/K5 gate/up GEMM (pair)")
        kernels = {n: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps}
                   for n, v in kern.items() if v[1]}
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": workload_config(cfg, T, world),
            "roofline": {"bound": "tensor", "kernel": "gemm_gate_up (K3+K5)", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "peak_source": peak_src + ", bf16 sustained",
                         "flop_per_launch": flop_gu,
                         # context for power-capped runs: the dense bf16 MMA peak at the median SM clock
                         # seen under load (148 SMs x 8192 FLOP/clk/SM = 2.25 PFLOP/s at 1.856 GHz)
                         "peak_at_clock": (148 * 8192 * clk["sm_mhz"] * 1e6 / 1e12) if clk else None,
                         "frac_at_clock": (achieved / (148 * 8192 * clk["sm_mhz"] * 1e6 / 1e12))
                         if (clk and achieved) else None},
            "e2e": {"value": T_total * args.steps / (ms_e2e / 1000.0), "unit": "tokens/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk,
            "kernels": kernels,
            "budget_C": [int(c) for c in budget_out.get("C", [])][:4],
            "merge_output_error": merr,
            "stale_profiling": stale,
        }
        if world == 1 and not args.no_cpu_baseline:
            r, threads, sample, dt = oracle_rate(cfg, args.ref_tokens, args.ref_layers, T)
            line["cpu_baseline"] = {"value": r, "unit": "tokens/s", "cores": threads, "kind": "oracle",
                                    "sample": sample, "seconds": dt}
        print(json.dumps(line), flush=True)
    comm.destroy()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
