"""rounds — one participant round of Flux on one GPU, with and without stale profiling (NEXT-4).

Paper §4.2 (Fig. 7): profiling the latest model w_r at the start of every round (Fig. 7a)
delays local fine-tuning; Flux instead merges with the STALE statistics f^{r-1} of the previous
round and quantizes + profiles w_r concurrently (Fig. 7b, "Mer. x_r, f_{r-1}"), so the next round
merges with f^r.

Here a round is:
  profile(w_r)  = a0 quantize + a1-a6 profile + a7 NCCL reduce + §5.2 clustering  -> f^r, cluster_of^r
  merge(w_r, f) = eq.(2) into the compact model (flux_compact_experts, NEXT-2)
  fine-tune     = the compact model's forward over the local fine-tuning tokens (flux_profile_layer,
                  wbits 16, gate re-routing) — the forward half of local fine-tuning; the backward
                  pass and the optimizer are outside this path, as is the server's
                  aggregation, whose waiting time is what stale profiling hides on a participant.
  serial (Fig. 7a): profile -> merge(f^r) -> fine-tune, one stream.
  stale  (Fig. 7b): foreground stream: merge(f^{r-1}) -> fine-tune;
                    background stream: profile -> f^r for the next round, once fine-tuning is done
                    (during the aggregation wait).
Both are measured with CUDA events on their streams: the fine-tuning start latency (round start ->
merged model ready) and the GPU span of the round.

Round makespan with the server's aggregation (Fig. 7: "the latency of model aggregation on
the server ... the participant is idle"): after fine-tuning, the participant uploads its update and waits
for the aggregated model; that wait W is modelled (agg_wait_s, an input — the paper gives no number) as
an idle period on the host.  Serial: profile -> merge -> fine-tune -> wait W.  Stale: merge(f^{r-1}) ->
fine-tune -> wait W on the foreground while the background profile of w_r runs on the GPU, so the
profile hides inside the wait (makespan = fine-tune + W when the profile is shorter than W).  The makespan is host wall-clock from the round start until both the
wait and every GPU stream are done.  Buffers and sequencing only; all arithmetic is in libflux.
"""
from __future__ import annotations

import time

import numpy as np
import torch

from .driver import (MasterWeights, ModelShape, Profiler, QuantizedModel, cluster_model, compact_model,
                     expert_features_model, feature_dim)


class Participant:
    def __init__(self, masters: MasterWeights, x_prof: torch.Tensor, x_ft: torch.Tensor, comm, n_clusters: int,
                 T_total: int, clustering: str = "pca", seeded_cluster_of: torch.Tensor | None = None,
                 agg_wait_s: float = 0.0):
        s = masters.shape
        self.m = masters
        self.shape = s
        self.comm = comm
        self.C = n_clusters
        self.T_total = T_total
        self.clustering = clustering
        self.agg_wait_s = agg_wait_s  # modelled server-aggregation wait after fine-tuning
        self.x_prof, self.x_ft = x_prof, x_ft
        self.qm = QuantizedModel(s)
        self.prof = Profiler(s, x_prof.shape[0], with_de=True)
        dev = masters.gate.device
        self.alpha = torch.empty(s.n_layers, s.n_experts, dtype=torch.float32, device=dev)
        self.cluster_of = (seeded_cluster_of.clone() if seeded_cluster_of is not None
                           else torch.empty(s.n_layers, s.n_experts, dtype=torch.int32, device=dev))
        self.next_cluster_of = self.cluster_of.clone()
        self.hist_host = torch.empty(s.n_layers, s.n_experts, dtype=torch.int64).pin_memory()
        self.alpha_host = torch.empty(s.n_layers, s.n_experts, dtype=torch.float32).pin_memory()
        self.fg = torch.cuda.Stream(priority=-1)  # fine-tuning path
        self.bg = torch.cuda.Stream(priority=0)   # stale profiling
        self.ft_prof = None
        self.compact = None
        self.profiled = torch.cuda.Event()

    # ------------------------------------------------------------------ pieces
    def profile(self, stream):
        """quantize + profile + reduce (+ clustering) of the current model on `stream` -> device hist, next
        cluster assignment; records self.profiled."""
        with torch.cuda.stream(stream):
            if self.clustering == "pca":
                feats, _, _ = expert_features_model(self.m, feature_dim(self.shape.n_experts), stream=stream)
            self.qm.quantize_from(self.m, stream)
            self.prof.run(self.qm, self.x_prof, stream=stream)
            self.comm.reduce_stats(self.prof.hist, stream)
            if self.clustering == "pca":
                self.next_cluster_of.copy_(cluster_model(feats, self.prof.hist, self.C, stream=stream))
            self.hist_host.copy_(self.prof.hist, non_blocking=True)
            self.profiled.record(stream)

    def absorb_statistics(self):
        """Host: wait for the profile, f = hist / T -> α for the next merge."""
        self.profiled.synchronize()
        f = self.hist_host.numpy() / float(self.T_total)
        self.alpha_host.copy_(torch.from_numpy(f.astype(np.float32)))
        with torch.cuda.stream(self.fg):  # ordered before the foreground's next merge
            self.alpha.copy_(self.alpha_host, non_blocking=True)
            self.cluster_of.copy_(self.next_cluster_of, non_blocking=True)

    def merge_and_finetune(self, stream, ev_merged=None):
        with torch.cuda.stream(stream):
            self.compact = compact_model(self.m, self.alpha, self.cluster_of, self.C, 0, stream=stream,
                                         out=self.compact)
            if ev_merged is not None:
                ev_merged.record(stream)
            if self.ft_prof is None:
                self.ft_prof = Profiler(self.compact.shape, self.x_ft.shape[0], with_de=False)
            self.ft_prof.run(self.compact, self.x_ft, stream=stream)

    # ------------------------------------------------------------------ rounds
    def round_serial(self):
        """Fig. 7a: profile w_r, then merge with f^r, then fine-tune (one stream), then wait for aggregation."""
        st = self.fg
        e0, em, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        e0.record(st)
        self.profile(st)
        self.absorb_statistics()  # host waits: the merge needs f^r
        self.merge_and_finetune(st, em)
        e1.record(st)
        e1.synchronize()
        time.sleep(self.agg_wait_s)  # upload + server aggregation + download: the participant idles
        makespan = time.perf_counter() - h0
        return {"ft_start_ms": e0.elapsed_time(em), "round_ms": e0.elapsed_time(e1), "makespan_ms": 1e3 * makespan}

    def round_stale(self):
        """Fig. 7b: merge with the stale f^{r-1} and fine-tune at once; profile w_r in the background, hidden
        behind the aggregation wait."""
        e0, em, efg, ebg = (torch.cuda.Event(enable_timing=True) for _ in range(4))
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        e0.record(self.fg)
        self.merge_and_finetune(self.fg, em)  # foreground first: uses f^{r-1} (self.alpha, self.cluster_of)
        efg.record(self.fg)
        # background: f^r for the next round, started once fine-tuning is done, i.e. inside the wait.  The
        # expert GEMMs and K1 are persistent kernels that hold every SM until they finish, so a stream
        # priority cannot keep a concurrent profile from stretching the fine-tuning (measured: fine-tuning
        # done 0.25-0.65 s after the round start depending on the interleaving, vs ~0.2 s alone)
        self.bg.wait_event(efg)
        self.profile(self.bg)
        ebg.record(self.bg)
        efg.synchronize()                     # fine-tuning done: upload, wait for the aggregated model
        time.sleep(self.agg_wait_s)
        ebg.synchronize()
        makespan = time.perf_counter() - h0
        self.fg.wait_event(ebg)
        e_end = torch.cuda.Event(enable_timing=True)
        e_end.record(self.fg)
        e_end.synchronize()
        out = {"ft_start_ms": e0.elapsed_time(em), "round_ms": e0.elapsed_time(e_end),
               "finetune_done_ms": e0.elapsed_time(efg), "profile_done_ms": e0.elapsed_time(ebg),
               "makespan_ms": 1e3 * makespan}
        self.absorb_statistics()  # f^r becomes the next round's stale statistics
        return out
