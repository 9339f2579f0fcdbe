"""bench.py — profiled tokens/s/box of the Flux hot path on B200 (BASELINE.json metric).

One step = one participant round of the hot path (all rows):
  a0 quantize the model (INT4 g128 / INT8)   flux_quantize_weights
  a1-a6 profile the rank's tokens through all layers: router+top-k+histogram,
        D_e permutation, grouped SwiGLU expert GEMMs (routed + shared), combine
                                             flux_profile_layer x L (x chunks)
  a7 all-reduce the int64 histograms         flux_reduce_stats (NCCL)
  a8-pre eq.(1) layer budgets (host)         flux_layer_budget
  §5.2 expert clustering (NEXT-1): PCA features of every layer's experts
        + fused K-Means into C clusters per layer from the reduced counts
                                             flux_expert_features, flux_cluster_experts
  a8 eq.(2) merge 64 -> 16 experts per layer, α = f (bf16), ONE launch for all
        L x 3 weight families                flux_merge_experts_batch
Data parallel over tokens: one process per GPU; `--gpus N` without torchrun
re-launches itself under torch.distributed.run with N ranks.
  --scaling weak   (default) every rank profiles its own shard of the config's tokens
                   (262,144 per GPU for the DeepSeek shape: N = 8 is BASELINE configs[4]);
  --scaling strong BASELINE configs[4]: 2,097,152 tokens split over the N ranks,
                   profiled in chunks of 262,144 tokens (the library is batch-invariant).

usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config deepseek_moe|llama_moe]
       python bench.py --impl reference ...   (the CPU oracle, timed on the host cores)
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "profiled tokens/sec/box (quantized MoE fwd + expert stats) at 1/2/4/8 B200; % roofline"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
SPEC_HBM_GBS = 8000.0  # the north star's "~8 TB/s" (B200 datasheet), reported beside the measured peak
STRONG_TOKENS = {"deepseek_moe": 2097152, "llama_moe": 524288, "toy": 2048}  # BASELINE configs[4] (M5)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


def workload_config(cfg, tokens_per_gpu, n_gpus, scaling="weak", chunk=None):
    d = {
        "workload": f"{cfg.name}: INT{cfg.wbits}{'-g' + str(cfg.group_size) if cfg.group_size else ' per-channel'} "
                    f"quantize + profile {cfg.n_layers} layers + NCCL hist all-reduce + PCA/K-Means clustering + eq.(2) merge "
                    f"{cfg.n_experts}->{max(1, cfg.n_experts // 4)} bf16",
        "layers": cfg.n_layers, "hidden": cfg.hidden, "experts": cfg.n_experts, "shared_ffn": cfg.shared_ffn,
        "top_k": cfg.top_k, "ffn": cfg.ffn, "wbits": cfg.wbits, "group_size": cfg.group_size,
        "tokens_per_gpu": tokens_per_gpu, "tokens_total": tokens_per_gpu * n_gpus,
        "parallelism": f"dp{n_gpus}", "scaling": scaling,
        "l2": "inputs larger than L2 (x shard = %.2f GiB, weights %.1f GiB)" % (
            tokens_per_gpu * cfg.hidden * 2 / 2**30,
            cfg.n_layers * (cfg.n_experts * 3 * cfg.ffn + 3 * cfg.shared_ffn) * cfg.hidden * 2 / 2**30),
    }
    if chunk and chunk < tokens_per_gpu:
        d["chunk_tokens"] = chunk
    return d


# ------------------------------------------------------------------------------------------ launcher
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_relaunch(args):
    """One process per GPU: `bench.py --gpus N` outside torchrun re-executes itself under
    torch.distributed.run with N ranks (127.0.0.1 rendezvous) and exits with its status; under torchrun
    the world size must equal --gpus."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
            sys.exit(2)
        return
    if args.gpus <= 1:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def launcher_selftest(args):
    """CPU check of the multi-rank plumbing (gloo): every rank contributes 1 to an all-reduce and its
    token shard; rank 0 prints the world it saw."""
    import torch
    import torch.distributed as dist
    from paper_2508_19078_b200.driver import shard
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.tensor([1, shard(rank, world, 1000)[0]], dtype=torch.int64)
    if world > 1:
        dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"n_gpus": world, "ranks_seen": int(t[0]), "shard_starts_sum": int(t[1]),
                          "gpus_arg": args.gpus}), flush=True)
    if world > 1:
        dist.destroy_process_group()


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


# ------------------------------------------------------------------------------------------ oracle timing
def oracle_costs(cfg, n_tok, n_layers, T_full):
    """Time the oracle (as it stands) on a bounded sample and separate its two costs:
      q  = per-layer quantization of the model (O1, once per layer per round),
      c0 = per-layer fixed forward cost (fp64 dequantization of the experts the tokens use),
      c  = per-token, per-layer forward cost (router + expert FFNs + combine, O2-O6),
    from n_tok and n_tok/8 tokens through the first n_layers layers.  Returns (tokens/s of a full
    cfg.n_layers-layer pass over T_full tokens = T_full / (L·(q + c0) + T_full·L·c), details).
    The sampled layers are the LAST ones (the most balanced routing, so both token counts use nearly every
    expert and c0 is the same in both runs); each runs on x_0 (timing only)."""
    import oracle.model as om
    import synth
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    n_small = max(1, n_tok // 2)
    x0 = synth.bf16_bits_to_f32(synth.cpu_rows(synth.spec_x(cfg), np.arange(n_tok))).astype(np.float64)
    tq = tf_small = tf = 0.0
    t_start = time.perf_counter()
    for l in range(cfg.n_layers - n_layers, cfg.n_layers):
        x = x0
        t0 = time.perf_counter()
        wr, experts, shared = om.quantized_layer(cfg, l)
        t1 = time.perf_counter()
        om.moe_tokens(x[:n_small], wr, experts, shared, k=cfg.top_k, group_size=cfg.group_size, norm=cfg.norm_topk)
        t2 = time.perf_counter()
        om.moe_tokens(x, wr, experts, shared, k=cfg.top_k, group_size=cfg.group_size, norm=cfg.norm_topk)
        t3 = time.perf_counter()
        tq += t1 - t0
        tf_small += t2 - t1
        tf += t3 - t2
    seconds = time.perf_counter() - t_start
    q = tq / n_layers
    c = max(tf - tf_small, 0.0) / n_layers / max(n_tok - n_small, 1)
    c0 = max(tf / n_layers - c * n_tok, 0.0)
    L = cfg.n_layers
    full = L * (q + c0) + T_full * L * c
    det = {"cores": threads, "seconds": seconds,
           "quantize_s_per_layer": q, "forward_fixed_s_per_layer": c0, "forward_s_per_token_layer": c,
           "forward_tokens_per_s": 1.0 / (c * L) if c > 0 else None,
           "full_pass_s": full,
           "sample": f"{n_tok} (and {n_small}) tokens through the last {n_layers} of {L} layers: oracle quantization of each "
                     f"layer (q), fp64 layer forward (fixed part c0 + per-token part c, separated by the two token "
                     f"counts); full pass = L·(q + c0) + T·L·c for T = {T_full}; merge not included"}
    return T_full / full, det


def run_reference(args, cfg, rank, world, T_rank):
    if rank != 0:
        return
    rates, secs, det = [], [], None
    for i in range(args.warmup + args.steps):
        r, det = oracle_costs(cfg, args.ref_tokens, args.ref_layers, T_rank * world)
        if i >= args.warmup:
            rates.append(r)
            secs.append(det["seconds"])
    v = statistics.median(rates)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            # the measured wall time of one step = one bounded oracle sample (not the extrapolated pass)
            "ms_per_step": 1000.0 * statistics.median(secs),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(cfg, T_rank, world, args.scaling),
            "cpu_baseline": {"value": v, "unit": "tokens/s", "kind": "oracle", **det},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------ algorithmic bytes
def kernel_bytes(cfg, T, C, n_chunks_T, fused_bops=False):
    """Algorithmic HBM bytes per step of each HBM-bound kernel, for T tokens
    per rank per step in n_chunks_T profiling calls per layer.  fused_bops: the quantizer also writes the
    bf16 B operands (flux_quantize_weights_bops) and no dequantization pass runs.  Keys are
    flux_kernel_name()s."""
    L, E, H, F, Fs, k = cfg.n_layers, cfg.n_experts, cfg.hidden, cfg.ffn, cfg.shared_ffn, cfg.top_k
    n_w = E * 3 * F * H + 3 * Fs * H                           # quantized weights per layer
    per_w_q = {8: 1.0, 4: 0.5, 2: 0.25}[cfg.wbits]             # code bytes per weight
    g = cfg.group_size
    sc = 4.0 / g if g else 0.0                                  # scale bytes per weight (grouped)
    return {
        "router": L * T * (2 * H + 12 * k),                     # read x, write ids / w / rank
        "permute": L * T * 16 * k,                               # K2: read ids + rank, write inv_pos + token_index
        "combine": L * T * (k * H * 2 + 8 * k + H * 2 * (3 if Fs else 2)),
        "dequant": n_chunks_T * L * n_w * (per_w_q + sc + 2.0),  # per profiling call: read codes (+ scales), write bf16
        "quantize": L * n_w * (2.0 + per_w_q + sc + (2.0 if fused_bops else 0.0)),  # read masters, write codes + scales
                                                                                     # (+ the bf16 B operands)
        "merge": L * 3 * F * H * 2 * (E + C),                   # read Σ|W_e|, write Σ|W_c|
        "gram": L * E * 3 * F * H * 2,                          # read every master parameter once
    }


# ------------------------------------------------------------------------------------------ one workload
def measure(args, cfg, T_rank, rank, world, stream_extras=True, steps=None, warmup=None):
    """Run the participant round on this rank's shard: warm-up, K timed steps (device time, max over ranks),
    the e2e variant through host buffers, and (rank 0, main workload) the extras.  Returns a dict."""
    import torch
    import torch.distributed as dist
    import paper_2508_19078_b200 as F
    import synth
    from paper_2508_19078_b200 import synthetic
    from paper_2508_19078_b200.driver import (ModelShape, Profiler, QuantizedModel, budgets, cluster_model,
                                              expert_features_model, feature_dim, merge_model, shard)
    steps = steps or args.steps
    warmup = warmup if warmup is not None else args.warmup
    T_total = T_rank * world
    Tc = min(T_rank, args.chunk or cfg.tokens)                 # tokens per flux_profile_layer call
    n_chunks = (T_rank + Tc - 1) // Tc
    C = args.clusters or max(1, cfg.n_experts // 4)
    shape = ModelShape.of(cfg)
    L, E = cfg.n_layers, cfg.n_experts
    stream = torch.cuda.current_stream()

    # ---- setup (not timed): synthetic master weights, this rank's token shard, buffers, NCCL comm
    masters = synthetic.master_weights(cfg)
    qm = QuantizedModel(shape, with_bops=args.fused_dequant == "on")
    prof = Profiler(shape, Tc, with_de=True, policy=F.make_policy(gemm_chain={"auto": 0, "off": 1, "on": 2}[args.chain]))
    t0, _ = shard(rank, world, T_rank)  # this rank's contiguous slice of the global token stream
    x = synthetic.tokens(cfg, t0, T_rank)
    cluster_of = torch.from_numpy(synth.cluster_assignment(cfg, C)).cuda()
    d_feat = feature_dim(E)
    alpha = torch.empty(L, E, dtype=torch.float32, device="cuda")
    hist_host = torch.empty(L, E, dtype=torch.int64).pin_memory()
    ev_hist = torch.cuda.Event()
    attn = synthetic.attention_values(cfg, t0, T_rank) if args.alpha == "attn" else None
    if attn is not None and n_chunks > 1:
        raise SystemExit("--alpha attn needs one chunk per rank")
    state = {"merged": None, "cluster_of": cluster_of, "C": None}
    uid = F.Comm.unique_id() if rank == 0 else None
    if world > 1:
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    comm = F.Comm(uid, world, rank)

    def step(xs, before_chunk=None, after_chunk=None):
        if args.clustering == "pca":                              # §5.2 C1 (reads the masters only)
            feats, _, _ = expert_features_model(masters, d_feat)
        qm.quantize_from(masters)                                 # a0
        prof.hist.zero_()
        for c in range(n_chunks):                                 # a1-a6 (hist accumulates over chunks)
            if before_chunk:
                before_chunk(c)
            torch.cuda.nvtx.range_push(f"chunk {c}")             # chunk x layer timeline (nsys; no-op otherwise)
            prof.run(qm, xs[c * Tc:(c + 1) * Tc], zero_hist=False, attn=attn)
            torch.cuda.nvtx.range_pop()
            if after_chunk:
                after_chunk(c)
        report_budgets()  # the previous round's eq.(1) on the host, once this round's profiling is enqueued
        comm.reduce_stats(prof.hist)                              # a7
        if attn is None:                                          # α = f = hist / T, on the device
            F.frequencies(prof.hist, float(T_total), alpha)
        else:                                                     # NEXT-3: α = f·ā = Σ_{t∈D_e} a_t / T (R15)
            comm.reduce_stats(prof.ahist)
            F.frequencies(prof.ahist, 16777216.0 * T_total, alpha)
        hist_host.copy_(prof.hist, non_blocking=True)             # the round's statistics leave the device
        ev_hist.record(stream)
        if args.budget == "adaptive":                             # a8-pre, eq.(1) budgets drive this round
            ev_hist.synchronize()
            Cl, _ = budgets(hist_host.numpy(), T_total, C * L)
            state["C"] = Cl
            n_cl = [int(c) for c in Cl]
        else:                                                     # uniform C (BASELINE configs[3]): eq.(1)
            n_cl = C                                              # on the host, off the GPU's critical path
            state["hist_pending"] = True
        if args.clustering == "pca":                              # §5.2 C2: K-Means from the reduced counts
            state["cluster_of"] = cluster_model(feats, prof.hist, n_cl)
        state["merged"] = merge_model(masters, alpha, state["cluster_of"], n_cl, state["merged"])  # a8, eq.(2)

    def report_budgets():
        """a8-pre, eq.(1) on the host from the last round's reduced histogram (uniform mode: the report).
        Called after this round's profiling launches are enqueued: the wait on the last round's histogram
        event then never starves the GPU of queued work (called at the top of the step, it held the host
        until the previous round's profiling had finished, and the launches of the features + quantize
        phase could not stay ahead of the GPU: LLaMA shape 26 ms of idle GPU per step)."""
        if state.get("hist_pending"):
            ev_hist.synchronize()
            state["C"], _ = budgets(hist_host.numpy(), T_total, C * L)
            state["hist_pending"] = False

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(warmup):
        step(x)
    barrier()

    clocks = ClockSampler(os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out"))
                                       else "/tmp", f"clocks_rank{rank}.csv"))
    if rank == 0 and not os.environ.get("FLUX_BENCH_NO_CLOCKS"):  # diagnostics only: the line then has no clocks
        clocks.start()
    F.timing_read(reset=True)
    F.timing_enable(True)
    F.timing_clocks(reset=True)
    launches0 = F.launch_count()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    h0 = time.perf_counter()
    host_ms = []  # host time to enqueue each step (diagnostic: a step whose host time reaches the GPU's starves it)
    for _ in range(steps):
        step(x)
        host_ms.append(1e3 * (time.perf_counter() - h0))
    ev1.record(stream)
    barrier()
    F.timing_enable(False)
    launches = F.launch_count() - launches0
    kern = F.timing_read(reset=True)
    gemm_mhz = F.timing_clocks(reset=True)  # average SM clock measured inside the expert GEMMs
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clk = clocks.stop(gpus=set(range(world))) if rank == 0 else None

    # ---- e2e: the same step through the public API with host buffers: every step copies its tokens H2D
    #      from pinned memory and its profiling result (reduced histogram + the D_e CSR of every layer of
    #      every chunk) D2H.  Copies run on a copy stream, pipelined like a serving loop: step i+1's tokens
    #      go up while step i profiles (double-buffered x), each chunk's D_e comes down while the next
    #      chunk profiles (its first layer waits for that copy).
    x_host = x.cpu().pin_memory()
    off_host = torch.empty((n_chunks,) + tuple(prof.offsets.shape), dtype=torch.int32).pin_memory()
    ti_host = torch.empty((n_chunks,) + tuple(prof.token_index.shape), dtype=torch.int32).pin_memory()
    x_dev = [torch.empty_like(x), torch.empty_like(x)]
    h2d = x_host.numel() * x_host.element_size()
    d2h = hist_host.numel() * 8 + off_host.numel() * 4 + ti_host.numel() * 4
    cstream = torch.cuda.Stream()
    ev_h2d = [torch.cuda.Event(), torch.cuda.Event()]
    ev_prof, ev_d2h = torch.cuda.Event(), torch.cuda.Event()
    st = {"i": 0, "n": 1, "d2h_pending": False}

    def h2d_into(buf):
        with torch.cuda.stream(cstream):
            x_dev[buf].copy_(x_host, non_blocking=True)
            ev_h2d[buf].record(cstream)

    def before_chunk(c):
        if c == 0:
            stream.wait_event(ev_h2d[st["i"] % 2])  # this step's tokens are on the device
        if st["d2h_pending"]:
            stream.wait_event(ev_d2h)  # the previous chunk's D_e has left the device

    def after_chunk(c):
        ev_prof.record(stream)
        with torch.cuda.stream(cstream):
            cstream.wait_event(ev_prof)
            off_host[c].copy_(prof.offsets, non_blocking=True)
            ti_host[c].copy_(prof.token_index, non_blocking=True)
            ev_d2h.record(cstream)
        st["d2h_pending"] = True
        if c == n_chunks - 1 and st["i"] + 1 < st["n"]:
            h2d_into((st["i"] + 1) % 2)  # the next step's tokens (that buffer's reader is done)

    def e2e_step():
        step(x_dev[st["i"] % 2], before_chunk, after_chunk)
        st["i"] += 1

    def e2e_drain():
        ev_d2h.synchronize()  # the last chunk's D_e is on the host
        cstream.synchronize()

    st["n"] = 1
    h2d_into(0)
    e2e_step()
    e2e_drain()
    barrier()
    st.update(i=0, n=steps, d2h_pending=False)
    ev0.record(stream)
    cstream.wait_event(ev0)
    h2d_into(0)  # the first timed step's tokens: inside the timed region
    for _ in range(steps):
        e2e_step()
    e2e_drain()
    ev1.record(stream)
    barrier()
    ms_e2e = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    del x_dev, x_host, off_host, ti_host

    report_budgets()
    out = {"ms": ms, "ms_e2e": ms_e2e, "h2d": h2d, "d2h": d2h, "launches": launches, "kern": kern, "clk": clk,
           "host_ms": host_ms,
           "gemm_mhz": gemm_mhz,
           "T_rank": T_rank, "Tc": Tc, "n_chunks": n_chunks, "fused_bops": qm.bops is not None, "C": C, "budget_C": [int(c) for c in state["C"]],
           "steps": steps}

    # ---- merge quality of the round's merged model (not timed): the paper's output error —
    #      mean cosine distance between the final outputs of the compact model (tuning experts + the
    #      eq.(2) merges, gate re-routed, bf16) and of the original bf16 model on the first tokens of x
    if stream_extras and args.error_tokens > 0 and rank == 0:
        from paper_2508_19078_b200.driver import compact_model, dense_model
        n_err = min(args.error_tokens, T_rank)
        n_cl = [int(c) for c in state["C"]] if args.budget == "adaptive" else C
        dense = dense_model(masters)
        comp = compact_model(masters, alpha, state["cluster_of"], n_cl, 0)
        outs = []
        for mdl in (dense, comp):
            pr = Profiler(mdl.shape, n_err, with_de=False)
            outs.append(pr.run(mdl, x[:n_err]).clone())
            del pr
        out["merge_output_error"] = {
            "value": float(F.output_error(outs[1], outs[0]).item()), "tokens": n_err, "clusters_per_layer": n_cl,
            "alpha": args.alpha, "clustering": args.clustering, "budget": args.budget,
            "what": "mean cosine distance of final token outputs, merged vs original bf16 model (P:686-689)"}
        del comp, outs

    # ---- NEXT-4 stale profiling (not part of the timed step): participant rounds, serial (Fig. 7a) vs
    #      stale (Fig. 7b), each round = profile + merge into the compact model + its forward over the
    #      local fine-tuning tokens (the first quarter of x) + the modelled server-aggregation wait
    if stream_extras and args.rounds > 0 and world == 1 and n_chunks == 1:
        from paper_2508_19078_b200.rounds import Participant
        del prof
        torch.cuda.empty_cache()
        # modelled wait: upload the round's update + download the aggregated model over the
        # participant's link; the paper gives no number: the compact model's merged experts (bf16) at
        # --agg-gbps (default 25 Gb/s), both directions
        merged_bytes = L * 3 * cfg.ffn * cfg.hidden * 2 * C
        wait_s = args.agg_wait if args.agg_wait >= 0 else 2 * merged_bytes * 8 / (args.agg_gbps * 1e9)
        part = Participant(masters, x, x[: max(1, T_rank // 4)], comm, C, T_total, clustering=args.clustering,
                           seeded_cluster_of=cluster_of, agg_wait_s=wait_s)
        part.round_serial()  # warm-up; leaves f^r for the first stale round
        ser = [part.round_serial() for _ in range(args.rounds)]
        stl = [part.round_stale() for _ in range(args.rounds)]
        med = lambda rs, k: statistics.median(r[k] for r in rs)  # noqa: E731
        out["stale_profiling"] = {
            "serial_makespan_ms": med(ser, "makespan_ms"), "stale_makespan_ms": med(stl, "makespan_ms"),
            "makespan_cut": 1.0 - med(stl, "makespan_ms") / med(ser, "makespan_ms"),
            "agg_wait_ms": 1e3 * wait_s,
            "serial_gpu_ms": med(ser, "round_ms"), "serial_ft_start_ms": med(ser, "ft_start_ms"),
            "stale_gpu_ms": med(stl, "round_ms"), "stale_ft_start_ms": med(stl, "ft_start_ms"),
            "stale_profile_done_ms": med(stl, "profile_done_ms"), "rounds": args.rounds,
            "finetune_tokens": int(max(1, T_rank // 4)),
            "what": "participant round = profile + merge (compact model) + compact-model forward over the "
                    "fine-tuning tokens + modelled aggregation wait (host idle: 2 x merged-expert bytes at "
                    f"{args.agg_gbps} Gb/s); stale = merge with f^(r-1) at once, profile on a low-priority stream "
                    "during fine-tuning and the wait (Fig. 7b, P:619-631); makespan = host wall clock"}
        del part
    comm.destroy()
    return out


def roofline_gemm(cfg, T_rank, res, peaks, peak_src):
    """The dominant kernel: the gate/up grouped GEMM (routed + shared, one launch per layer per chunk)."""
    H, k = cfg.hidden, cfg.top_k
    flop_gu = 2.0 * res["Tc"] * (k * H * 2 * cfg.ffn + H * 2 * cfg.shared_ffn)  # per launch
    kname = "gemm_gate_up (K3+K5)"
    gu_ms, gu_n = res["kern"].get("gemm_gate_up", (0.0, 0))
    if not gu_n and res["kern"].get("gemm_chain", (0.0, 0))[1]:  # gate/up + down chained in one launch
        gu_ms, gu_n = res["kern"]["gemm_chain"]
        flop_gu += 2.0 * res["Tc"] * (k * cfg.ffn * H + cfg.shared_ffn * H)
        kname = "gemm_chain (K3+K4+K5: gate/up and down in one launch)"
    achieved = flop_gu / (gu_ms / gu_n / 1000.0) / 1e12 if gu_n else None
    peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        # dram read+write bytes per launch from the committed `ncu --set full` capture (profiles/)
        traffic = json.load(open(tp)).get(f"{cfg_key(cfg)}:{res['Tc']}:K3/K5 gate/up GEMM (pair)")
    clk = res["clk"]
    return {"bound": "tensor", "kernel": kname, "achieved": achieved, "peak": peak,
            "unit": "TFLOP/s", "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "peak_source": peak_src + ", bf16 sustained", "flop_per_launch": flop_gu,
            "share_of_step": (gu_ms / res["steps"]) / (res["ms"] / res["steps"]) if gu_n else None,
            # context for power-capped runs: the dense bf16 MMA peak at the median SM clock seen under load
            # (148 SMs x 8192 FLOP/clk/SM = 2.25 PFLOP/s at 1.856 GHz)
            "peak_at_clock": (148 * 8192 * clk["sm_mhz"] * 1e6 / 1e12) if clk else None,
            "frac_at_clock": (achieved / (148 * 8192 * clk["sm_mhz"] * 1e6 / 1e12)) if (clk and achieved) else None,
            # the same against the clock measured inside the GEMM itself (%clock64 / %globaltimer, libflux)
            "kernel_mhz": res.get("gemm_mhz", {}).get("gemm_gate_up"),
            "frac_at_kernel_clock": (achieved / (148 * 8192 * res["gemm_mhz"]["gemm_gate_up"] * 1e6 / 1e12))
            if (achieved and res.get("gemm_mhz", {}).get("gemm_gate_up")) else None}


def cfg_key(cfg):
    return {"deepseek_moe_16b": "deepseek_moe", "llama_moe_3.5b": "llama_moe"}.get(cfg.name, cfg.name)


def kernel_table(cfg, res, peaks):
    """Per-kernel time per step, and for the HBM-bound kernels algorithmic GB/s against the measured copy
    peak and the north star's ~8 TB/s."""
    hbm = peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"])
    steps = res["steps"]
    by = kernel_bytes(cfg, res["T_rank"], res["C"], res["n_chunks"], res.get("fused_bops", False))
    # DRAM read + write bytes per launch from the committed `ncu --set full` captures (profiles/traffic.json)
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    ncu_label = {"router": "K1 router", "permute": "K2 permute (one kernel)", "gemm_gate_up": "K3/K5 gate/up GEMM (pair)",
                 "gemm_down": "K4/K5 down GEMM (pair)", "combine": "K6 combine"}
    out = {}
    for n, (ms_tot, cnt) in res["kern"].items():
        if not cnt:
            continue
        d = {"ms_per_step": ms_tot / steps, "launches_per_step": cnt / steps}
        if n in by and ms_tot > 0:
            gbs = by[n] / (ms_tot / steps / 1e3) / 1e9
            d.update(bytes_per_step=by[n], gbs=gbs, frac_hbm_measured=gbs / hbm, frac_hbm_8tbs=gbs / SPEC_HBM_GBS)
        t = traffic.get(f"{cfg_key(cfg)}:{res['Tc']}:{ncu_label.get(n, '')}")
        if t:
            d["ncu_dram_bytes_per_launch"] = t
            if n in by:
                d["ncu_dram_vs_algorithmic"] = t / (by[n] / (cnt / steps))
        out[n] = d
    return out


# ------------------------------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="flux", choices=["flux", "reference"])
    ap.add_argument("--config", default="deepseek_moe")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--tokens", type=int, default=0, help="tokens per GPU (weak) or in total (strong)")
    ap.add_argument("--chunk", type=int, default=0, help="tokens per flux_profile_layer call (default: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-tokens", type=int, default=128)  # oracle sample (~20-30 s of host CPU work)
    ap.add_argument("--ref-layers", type=int, default=2)
    ap.add_argument("--clusters", type=int, default=0)
    ap.add_argument("--budget", default="uniform", choices=["uniform", "adaptive"],
                    help="uniform: C clusters in every layer (BASELINE configs[3]); adaptive: eq.(1) B(l)")
    ap.add_argument("--rounds", type=int, default=2,
                    help="NEXT-4: serial vs stale-profiling participant rounds measured after the run (0 = skip)")
    ap.add_argument("--agg-gbps", type=float, default=25.0, help="NEXT-4: participant link for the modelled wait")
    ap.add_argument("--agg-wait", type=float, default=-1.0, help="NEXT-4: modelled wait in s (overrides --agg-gbps)")
    ap.add_argument("--alpha", default="f", choices=["f", "attn"],
                    help="merge importance: activation frequency (BASELINE config) or f·ā with synthetic attention")
    ap.add_argument("--wbits", type=int, default=0, choices=[0, 2, 4, 8],
                    help="override the config's bit level (2 = the paper's bit-2 ablation, NEXT-3)")
    ap.add_argument("--error-tokens", type=int, default=8192,
                    help="tokens for the merged model's output error after the timed run (0 = skip)")
    ap.add_argument("--clustering", default="pca", choices=["pca", "seeded"],
                    help="pca: §5.2 PCA + K-Means on the GPU inside the step; seeded: a fixed balanced partition")
    ap.add_argument("--other-configs", default="llama_moe",
                    help="comma-separated extra workloads measured in the same run (N = 1 only; '' = none)")
    ap.add_argument("--chain", default="auto", choices=["auto", "on", "off"],
                    help="flux_policy.gemm_chain: gate/up + down GEMMs in one launch (on) or two (off)")
    ap.add_argument("--fused-dequant", default="on", choices=["on", "off"],
                    help="on: the quantizer writes every layer's bf16 B operands in the same pass "
                         "(flux_quantize_weights_bops, ~1.1 GB per DeepSeek-shape layer of HBM); off: one "
                         "dequantization pass per flux_profile_layer call")
    ap.add_argument("--selftest-launcher", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    maybe_relaunch(args)
    if args.selftest_launcher:
        launcher_selftest(args)
        return

    import synth
    cfg = synth.CONFIGS[args.config]
    if args.wbits:
        cfg = cfg.with_(wbits=args.wbits, name=f"{cfg.name}_int{args.wbits}")
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))

    def rank_tokens(c, key):
        if args.scaling == "strong":
            total = args.tokens or STRONG_TOKENS.get(key, c.tokens * 8)
            if total % world:
                raise SystemExit(f"{total} tokens do not split over {world} ranks")
            return total // world
        return args.tokens or c.tokens

    T_rank = rank_tokens(cfg, args.config)
    if args.impl == "reference":
        run_reference(args, cfg, rank, world, T_rank)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    res = measure(args, cfg, T_rank, rank, world)
    import gc
    gc.collect()
    torch.cuda.empty_cache()

    others = {}
    if world == 1 and args.other_configs:
        for key in [c for c in args.other_configs.split(",") if c and c != args.config]:
            ocfg = synth.CONFIGS[key]
            oT = rank_tokens(ocfg, key)
            r = measure(args, ocfg, oT, rank, world, stream_extras=False, steps=max(1, min(args.steps, 3)),
                        warmup=max(args.warmup, 3))
            gc.collect()
            torch.cuda.empty_cache()
            others[key] = r

    if rank == 0:
        peaks, peak_src = load_peaks()
        T_total = T_rank * world
        line = {
            "metric": METRIC, "value": T_total * args.steps / (res["ms"] / 1000.0), "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["ms"] / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": dict(workload_config(cfg, T_rank, world, args.scaling, res["Tc"]),
                           dequant="fused into the quantizer" if res["fused_bops"] else "one pass per profiling call"),
            "roofline": roofline_gemm(cfg, T_rank, res, peaks, peak_src),
            "e2e": {"value": T_total * args.steps / (res["ms_e2e"] / 1000.0), "unit": "tokens/s",
                    "h2d_bytes_per_step": res["h2d"], "d2h_bytes_per_step": res["d2h"]},
            "gpu_launches": res["launches"],
            "clocks": res["clk"],
            "kernels": kernel_table(cfg, res, peaks),
            "host_enqueue_ms": [round(t, 1) for t in res["host_ms"]],  # cumulative, per timed step (diagnostic)
            "budget": args.budget,
            "budget_C": res["budget_C"],
            "merge_output_error": res.get("merge_output_error"),
            "stale_profiling": res.get("stale_profiling"),
        }
        if others:
            line["other_configs"] = {}
            for key, r in others.items():
                ocfg = synth.CONFIGS[key]
                line["other_configs"][key] = {
                    "value": r["T_rank"] * r["steps"] / (r["ms"] / 1000.0), "unit": "tokens/s",
                    "ms_per_step": r["ms"] / r["steps"], "steps": r["steps"],
                    "e2e": {"value": r["T_rank"] * r["steps"] / (r["ms_e2e"] / 1000.0), "unit": "tokens/s",
                            "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"]},
                    "config": workload_config(ocfg, r["T_rank"], 1, args.scaling, r["Tc"]),
                    "roofline": roofline_gemm(ocfg, r["T_rank"], r, peaks, peak_src),
                    "kernels": kernel_table(ocfg, r, peaks), "clocks": r["clk"], "gpu_launches": r["launches"]}
        if world == 1 and not args.no_cpu_baseline:
            v, det = oracle_costs(cfg, args.ref_tokens, args.ref_layers, T_total)
            line["cpu_baseline"] = {"value": v, "unit": "tokens/s", "kind": "oracle", **det}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
