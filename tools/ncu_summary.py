"""Summarise ncu captures into profiles/ (tracked): per-kernel launch shares from a
--metrics gpu__time_duration.sum launch list, and key counters of a --set full capture.

usage: python tools/ncu_summary.py launches <launches.csv> <out.md>
       python tools/ncu_summary.py full <report.ncu-rep> <out.md> [traffic.json key-prefix]
       python tools/ncu_summary.py conflicts <out.md> <report.ncu-rep>...
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys

NAMES = [("grouped_gemm_pair_kernel<0>", "K3/K5 gate/up GEMM (pair)"), ("grouped_gemm_pair_kernel<1>", "K4/K5 down GEMM (pair)"),
         ("grouped_gemm_kernel<0>", "K3/K5 gate/up GEMM (1-CTA)"), ("grouped_gemm_kernel<1>", "K4/K5 down GEMM (1-CTA)"),
         ("router_kernel", "K1 router"), ("permute_kernel", "K2 permute (one kernel)"), ("scatter_kernel", "K2 x_perm copy"),
         ("grouped_gemm_pair_kernel<(int)0>", "K3/K5 gate/up GEMM (pair)"),
         ("grouped_gemm_pair_kernel<(int)1>", "K4/K5 down GEMM (pair)"),
         ("grouped_gemm_pair_q_kernel<(int)0", "K3/K5 gate/up GEMM (fused dequant)"),
         ("grouped_gemm_pair_q_kernel<(int)1", "K4/K5 down GEMM (fused dequant)"),
         ("grouped_gemm_kernel<(int)0>", "K3/K5 gate/up GEMM (1-CTA)"), ("grouped_gemm_kernel<(int)1>", "K4/K5 down GEMM (1-CTA)"),
         ("combine_kernel", "K6 combine"), ("quantize_kernel", "K0 quantize"), ("dequant_kernel", "K3/K4 dequant pass"),
         ("merge_tma_kernel", "K7 merge (batched, TMA)"), ("merge_kernel", "K7 merge"), ("gram_reduce_kernel", "K8b Gram reduce"), ("gram_kernel", "K8 Gram (PCA)"),
         ("eig_kernel", "K8c Jacobi eigen"), ("frequencies_kernel", "alpha = f (frequencies)"), ("kmeans_kernel", "K9 K-Means"), ("cosine_distance_kernel", "output error")]


def label(name):
    for key, lab in NAMES:
        if key in name:
            return lab
    return name[:60]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
    agg = collections.OrderedDict()
    setup = collections.Counter()
    for r in rows[i + 1:]:
        if "synth_kernel" in r[ki]:  # input generation during setup (not part of a step)
            setup[r[ki][:40]] += 1
            continue
        ms = float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        agg.setdefault(label(r[ki]), []).append(ms)
    total = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list — {path.split('/')[-1]}", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` over `bench.py --steps 1 --warmup 1`"
             " (warm-up + timed + e2e steps, `--rounds 0 --error-tokens 0`). Launches are serialised and cold-cache: compare"
             " SHARES with bench.py's live per-kernel CUDA-event times, not absolutes.", "",
             "| kernel | launches | mean ms | total ms | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.3f} | {sum(v):.1f} | {100 * sum(v) / total:.1f}% |")
    lines.append(f"| **all** | {sum(len(v) for v in agg.values())} | | {total:.1f} | 100% |")
    if setup:
        lines += ["", f"Excluded (setup, not in a step): {dict(setup)}. `FillFunctor` = the per-round "
                      "histogram zeroing (`hist.zero_()`, the caller's duty per include/flux.h)."]
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_op_read_hit_rate.pct",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def full(path, out, traffic_prefix=None):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full — {path.split('/')[-1]}", ""]
    traffic = {}
    for r in rows[2:]:
        d = {h: (u, v) for h, u, v in zip(hdr, units, r)}
        name = d.get("Kernel Name", ("", "?"))[1]
        lines += [f"## {label(name)}", f"`{name[:150]}`", "", "| metric | unit | value |", "|---|---|---:|"]
        for k in KEYS:
            # ncu prefixes some section metrics; match by suffix
            hit = [h for h in d if h == k or h.endswith("." + k)]
            if hit:
                u, v = d[hit[0]]
                lines.append(f"| {k} | {u} | {v} |")
        rd = d.get("dram__bytes_read.sum")
        wr = d.get("dram__bytes_write.sum")
        if rd and wr:
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tb = float(rd[1].replace(",", "")) * mult.get(rd[0], 1) + float(wr[1].replace(",", "")) * mult.get(wr[0], 1)
            lines.append(f"| dram read+write per launch | byte | {tb:.4g} |")
            traffic[label(name)] = tb
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    return traffic


def conflicts(out, paths):
    """Per-kernel shared-memory wavefronts attributed to SASS instructions (source page: actual vs
    ideal per instruction) beside the kernel-level l1tex bank-conflict counter, which also counts
    LSU accesses delayed by the async proxy (TMA writes, tcgen05.mma operand reads) on the same banks."""
    lines = ["# Shared-memory bank conflicts — per instruction vs kernel counter", "",
             "`ncu --page source --print-source sass`: for every SASS instruction with shared wavefronts, "
             "`L1 Wavefronts Shared` (actual) vs `L1 Wavefronts Shared Ideal`; excess = actual − ideal is "
             "what the instruction's own address pattern costs. The kernel-level "
             "`l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum` is from the raw page of the same report.", ""]
    for path in paths:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(io.StringIO(raw)))
        counters = {}
        for r in rr[2:]:
            d = dict(zip(rr[0], r))
            get = lambda k: next((v for h, v in d.items() if h == k or h.endswith("." + k)), "?")
            counters.setdefault(label(d.get("Kernel Name", "?")), (get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
                                                                  get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")))
        src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        kern, hdr, per = None, None, collections.OrderedDict()
        for row in csv.reader(io.StringIO(src)):
            if row and row[0] == "Kernel Name":
                kern, hdr = row[1], None
                continue
            if row and row[0] == "Address":
                hdr = row
                continue
            if hdr is None or len(row) < len(hdr):
                continue
            d = dict(zip(hdr, row))
            try:
                w = float(d["L1 Wavefronts Shared"] or 0)
                ideal = float(d["L1 Wavefronts Shared Ideal"] or 0)
            except (KeyError, ValueError):
                continue
            if w > 0:  # one launch per kernel name: later duplicates of an address are other launches
                per.setdefault(kern, {}).setdefault(d["Address"], (w, ideal, d["Source"].strip()))
        lines += [f"## {path.split('/')[-1]}", "", "| kernel | counter conflicts / wavefronts | instr. wavefronts | ideal | excess | top excess instruction |",
                  "|---|---|---:|---:|---:|---|"]
        for k, v in per.items():
            v = list(v.values())
            w, ideal = sum(x[0] for x in v), sum(x[1] for x in v)
            top = max(v, key=lambda x: x[0] - x[1])
            c = counters.get(label(k), ("?", "?"))
            top_s = f"`{top[2][:48]}` ({top[0] - top[1]:.0f})" if top[0] > top[1] else "—"
            lines.append(f"| {label(k)} | {c[0]} / {c[1]} | {w:.4g} | {ideal:.4g} | {w - ideal:.4g} | {top_s} |")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "conflicts":
        conflicts(sys.argv[2], sys.argv[3:])
    elif sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        tr = full(sys.argv[2], sys.argv[3])
        if len(sys.argv) > 4:
            p = "profiles/traffic.json"
            try:
                cur = json.load(open(p))
            except Exception:
                cur = {}
            for k, v in tr.items():
                cur[f"{sys.argv[4]}:{k}"] = v
            json.dump(cur, open(p, "w"), indent=1)
