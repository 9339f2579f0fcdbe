/* include/flux.h — C ABI of libflux.so, the B200 (sm_100a) hot path of Flux
 * (arXiv 2508.19078): quantization-based local expert-activation profiling,
 * the statistics all-reduce, and the activation-frequency-weighted merge of
 * non-tuning experts.
 *
 * Citations: "P:N" = line N of the paper text; "R#" = a reading of
 * a passage the paper leaves open, listed in DESIGN.md §2.
 *
 * Conventions (all entry points):
 *  - Plain C types only.  Device pointers are CUDA device addresses; `stream`
 *    is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Ownership: the caller owns every buffer.  Hot calls allocate nothing;
 *    scratch comes from the caller's workspace.  Only flux_comm is owned by
 *    the library (flux_comm_init / flux_comm_destroy).
 *  - Stream-ordered and asynchronous.  Argument / shape validation happens on
 *    the host before any launch; on error nothing is launched and a status is
 *    returned.  Launch failures return FLUX_E_CUDA; asynchronous device faults
 *    surface at the caller's next synchronisation.
 *  - No CPU fallback: unsupported shapes return FLUX_E_UNSUPPORTED, and a host
 *    without an sm_100 device gets FLUX_E_CUDA.
 *  - Deterministic: outputs are bitwise reproducible and independent of how
 *    tokens are split across calls (chunking) or GPUs (data parallelism).
 *  - Layouts are row-major with the contraction dimension contiguous.  bf16
 *    is IEEE bfloat16 (uint16 storage).  INT4 is packed two per byte, even k
 *    in the low nibble, two's complement.
 */
#ifndef FLUX_H_
#define FLUX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FLUX_OK = 0,
  FLUX_E_INVALID = 1,     /* bad pointer / size / alignment / value              */
  FLUX_E_UNSUPPORTED = 2, /* shape or dtype outside the supported set            */
  FLUX_E_WORKSPACE = 3,   /* workspace smaller than flux_profile_layer_workspace  */
  FLUX_E_CUDA = 4,        /* CUDA runtime / driver error (incl. no sm_100 device) */
  FLUX_E_NCCL = 5         /* NCCL error, or libnccl.so.2 could not be loaded      */
} flux_status;

typedef enum { FLUX_BF16 = 0, FLUX_FP32 = 1 } flux_dtype;

const char* flux_status_string(flux_status s);

/* ============================================================================
 * Model shape of one MoE layer (Table 1).
 * Supported: hidden % 64 == 0; ffn % 16 == 0 (and shared_ffn); 1 <= top_k <= 8,
 * top_k <= n_experts <= 128; wbits in {2, 4, 8, 16}; group_size == 0 (per output channel)
 * or a multiple of 64 dividing both hidden and ffn (and shared_ffn); INT4 needs every
 * packed row to be a multiple of 16 B (hidden % 32 == 0, ffn % 32 == 0), INT2 hidden, ffn
 * and shared_ffn % 64 == 0.  (SURVEY §8(b) allowed E <= 256; the BASELINE configs need <= 64.)
 * ========================================================================== */
typedef struct {
  int32_t hidden;     /* H                                                    */
  int32_t ffn;        /* F, width of one routed expert                        */
  int32_t n_experts;  /* E, routed experts                                    */
  int32_t top_k;      /* k, experts per token                                 */
  int32_t shared_ffn; /* F_s of the always-on shared experts (0 = none), R5   */
  int32_t wbits;      /* 8, 4 or 2 (bit level chosen per participant; 2 = the "2-bit"
                         of P:1516-1517, NEXT-3: four codes per byte, needs H, F, F_s % 64); 16 = bf16
                         weights, not quantized (the compact model after merging, NEXT-2) */
  int32_t group_size; /* 0 = per output channel, else g along the contraction (0 for wbits 16) */
  int32_t norm_topk;  /* 0: w = softmax prob; 1: renormalised over top-k (R2) */
  int32_t n_router;   /* 0: the router scores the n_experts experts.  > 0 (NEXT-2, gate
                         re-routing after merging, §7, reading R14): the router
                         keeps the ORIGINAL n_router experts and flux_qlayer.remap sends each
                         pick to one of the n_experts slots of the compact model; requires
                         n_experts <= n_router <= 128 and top_k <= n_router */
} flux_moe_cfg;

/* Quantized weights of one layer, canonical layout (device pointers):
 *   router_w  bf16 [E_r][H]             (not quantized, R1; E_r = n_router or n_experts)
 *   gate_q    [E][F][H']   up_q [E][F][H']   H' = H (int8), H/2 (int4) or H/4 bytes (int2)
 *   gate_s    fp32 [E][F][H/g]          (g = H when group_size == 0)
 *   down_q    [E][H][F']                F' = F, F/2 or F/4
 *   down_s    fp32 [E][H][F/g]
 *   sh_*      same for the shared MLP with F_s instead of F (NULL if F_s == 0)
 *   wbits 16: *_q are bf16 [E][F][H] / [E][H][F] weights and the scales are ignored (may be NULL)
 *   remap     int32 [n_router], slot in [0, n_experts) of every original expert (flux_merge_experts'
 *             remap); required iff cfg.n_router > 0, else ignored
 * All pointers 16-byte aligned. */
typedef struct {
  const void* router_w;
  const void *gate_q, *up_q, *down_q;
  const float *gate_s, *up_s, *down_s;
  const void *sh_gate_q, *sh_up_q, *sh_down_q;
  const float *sh_gate_s, *sh_up_s, *sh_down_s;
  const int32_t* remap;
} flux_qlayer;

/* Per-layer outputs (device pointers, caller-owned; optional ones may be NULL):
 *   y              bf16 [T][H]   y_t = bf16(r_t + sh_t + Σ_j w_tj · o_{t,S_tj})   (R6) — required
 *   topk_ids       int32 [T][k]  S_t, descending logit, lower index on ties (R2)  — required.
 *                                With re-routing (n_router > 0): the slot of every pick; a pick
 *                                whose slot repeats an earlier pick's is folded into it (its
 *                                weight added there) and reads -1
 *   topk_w         fp32 [T][k]   gate weights w_tj (R2), 0 for a folded pick      — required
 *   hist           int64 [E]     ACCUMULATED (+=) activation counts, P:296-298    — required;
 *                                the caller zeroes it once per profiling round
 *   expert_offsets int32 [E+1]   D_e segment bounds into token_index  — optional
 *   token_index    int32 [T*k]   D_e members, ascending chunk-local token id (R3)  — optional
 *   router_logits  fp32 [T][E]   z = x·W_rᵀ, for parity checks only               — optional */
typedef struct {
  void* y;
  int32_t* topk_ids;
  float* topk_w;
  int64_t* hist;
  int32_t* expert_offsets;
  int32_t* token_index;
  float* router_logits;
} flux_layer_out;

/* Performance policy of flux_profile_layer_ex (NULL or all-zero = the library's measured defaults).
 * Every value produces bit-identical outputs (tests/test_gpu_parity.py::test_weight_paths_bit_identical);
 * values marked TEST-ONLY were measured slower on B200 and exist so that the bit-identity
 * test can pin them against the defaults. */
enum {
  FLUX_WEIGHTS_AUTO = 0,          /* dequant pass when T·k >= 2048·E (B tiles reused by many m-tiles), else in-GEMM */
  FLUX_WEIGHTS_DEQUANT_PASS = 1,  /* one dequantization pass per layer into bf16 B operands, TMA-fed GEMMs */
  FLUX_WEIGHTS_IN_GEMM = 2        /* dequant warps inside the GEMM convert the raw codes per B tile (INT4/INT8) */
};
enum {
  FLUX_ROWS_AUTO = 0,             /* in-GEMM cp.async gather of the routed rows from x on the pass path, else
                                     materialised */
  FLUX_ROWS_MATERIALISED = 1,     /* K2 writes x_perm (k·H·2 bytes per token) */
  FLUX_ROWS_TMA_GATHER4 = 2       /* TEST-ONLY: TMA tile::gather4 (~2.5x slower gate/up GEMM) */
};
#define FLUX_L2_SET 0x100         /* l2_hints = FLUX_L2_SET | bits overrides the default (bits 1) */
enum {
  FLUX_CHAIN_AUTO = 0,            /* the measured default: two launches               */
  FLUX_CHAIN_OFF = 1,             /* gate/up and down GEMMs as two launches (act round-trips through HBM) */
  FLUX_CHAIN_ON = 2               /* TEST-ONLY: one persistent launch, each m-tile's down tiles 24 m-tiles
                                     behind its gate/up tiles (dequant-pass path with the in-GEMM gather,
                                     claimed tiles, standalone combine; ignored otherwise).  Measured no
                                     faster: act leaves L2 before it is read back */
};
typedef struct {
  int32_t weight_path;    /* FLUX_WEIGHTS_*                                                      */
  int32_t routed_rows;    /* FLUX_ROWS_*                                                         */
  int32_t fused_combine;  /* 1 = TEST-ONLY: K6 in the shared-MLP down-GEMM epilogue (needs F_s > 0) */
  int32_t static_tiles;   /* 1 = TEST-ONLY: static round-robin GEMM tile order instead of claimed tiles */
  int32_t l2_hints;       /* 0 = default (evict_first on the act / y_perm stores); FLUX_L2_SET | bits:
                             bit 0 evict_first on output stores, bit 1 evict_last on B, bit 2 evict_first on A */
  int32_t gemm_chain;     /* FLUX_CHAIN_*                                                        */
} flux_policy;

/* Workspace bytes flux_profile_layer needs for T tokens (host function); it depends on the policy
 * (default policy for flux_profile_layer_workspace).  0 on invalid arguments.
 * The environment variable FLUX_DEBUG_SYNC=1 synchronises after every launch (see flux_last_error). */
size_t flux_profile_layer_workspace_ex(const flux_moe_cfg* cfg, const flux_policy* policy, int64_t T);
size_t flux_profile_layer_workspace(const flux_moe_cfg* cfg, int64_t T);

/* One quantized MoE layer forward over T tokens that also emits the expert
 * activation statistics — the profiling step of §4.1:
 *   z = x·W_rᵀ; S_t = top-k(z_t); w_t from softmax(z_t)            (R2)
 *   hist[e] += #{t : e ∈ S_t}; D_e = {t : e ∈ S_t}
 *   o_{t,e} = bf16(bf16(SiLU(x_t·ŵgᵀ)⊙(x_t·ŵuᵀ))·ŵdᵀ)                 (R4)
 *   ŵ = q·s for per-channel codes (the scale multiplies the fp32 dot product in the
 *   epilogue); ŵ = bf16(q·bf16(s)) for grouped codes (reading R1b, the W4A16 convention)
 *   sh_t = shared SwiGLU(x_t) (R5);  y_t = bf16(r_t + sh_t + Σ_j w_tj o_{t,S_tj})
 * x: bf16 [T][H] device; residual: bf16 [T][H] device or NULL (NULL = x, R6; an all-zero
 * buffer gives the MoE branch alone, y = bf16(sh + Σ_j w_j o_j)).
 * T may be 0 (no-op) or any positive count up to 2^31/k. Tokens are
 * independent; results do not depend on T or on how a batch is split. */
flux_status flux_profile_layer(const flux_moe_cfg* cfg, const flux_qlayer* w, const void* x, const void* residual,
                               int64_t T, const flux_layer_out* out, void* ws, size_t ws_bytes, void* stream);
/* The same with an explicit performance policy (NULL = defaults); ws sized by
 * flux_profile_layer_workspace_ex with the same policy. */
flux_status flux_profile_layer_ex(const flux_moe_cfg* cfg, const flux_policy* policy, const flux_qlayer* w,
                                  const void* x, const void* residual, int64_t T, const flux_layer_out* out, void* ws,
                                  size_t ws_bytes, void* stream);

/* Activation-frequency-weighted merge of non-tuning experts, eq.(2):
 *   W_c = Σ_{e∈E_c} α_e / Σ_{e'∈E_c} α_e' · W_e  (Σα = 0 -> plain mean, R10)
 * One weight family of one layer per call (or all families if the caller
 * stores them concatenated):
 *   experts     [E][numel] dtype, device       cluster_of int32 [E] device, -1 = tuning expert (kept)
 *   alpha       fp32 [E] device, >= 0 (α = f, or f·ā)
 *   merged      [n_clusters][numel] dtype, device; fp32 accumulation, one rounding
 *   remap       int32 [E] device or NULL: compact slot of e — tuning experts
 *               first in ascending id, then clusters 0..C-1
 * numel % 8 == 0, pointers 16-byte aligned, 1 <= n_clusters <= E <= 1024.
 * A cluster id in [0, n_clusters) with no member produces an all-zero output (no
 * error is reported: K-Means may legitimately leave a cluster empty); an expert
 * whose id is < -1 or >= n_clusters belongs to no output (its remap is -1). */
flux_status flux_merge_experts(flux_dtype dtype, int32_t n_experts, int64_t numel, const void* experts,
                               const int32_t* cluster_of, const float* alpha, int32_t n_clusters, void* merged,
                               int32_t* remap, void* stream);

/* The same eq.(2) merge for a BATCH of jobs in ONE persistent launch (a job = one weight family
 * of one layer; the whole model's L x 3 families in one call).  All jobs share n_experts and numel;
 * each has its own cluster_of / alpha / n_clusters (per-layer budgets B(l) of eq.(1)),
 * output and remap.  compact = 0: out = [n_clusters][numel] as flux_merge_experts; compact = 1: out =
 * the compact model's slots [n_tuning + n_clusters][numel] as flux_compact_experts, where n_tuning must
 * be the number of -1 entries of cluster_of.  Results are bit-identical to one flux_merge_experts /
 * flux_compact_experts call per job.  jobs: HOST array of n_jobs <= FLUX_MERGE_MAX_JOBS entries (read
 * before the call returns); device pointers 16-byte aligned; numel % 8 == 0. */
#define FLUX_MERGE_MAX_JOBS 256
typedef struct {
  const void* experts;       /* [E][numel] dtype, device                                      */
  const int32_t* cluster_of; /* [E] device, -1 = tuning expert                                */
  const float* alpha;        /* [E] device, >= 0                                              */
  int32_t n_clusters;        /* C of this job                                                 */
  int32_t n_tuning;          /* compact = 1 only: tuning experts of this job (slots = n_tuning + C) */
  void* out;                 /* [C][numel] or [n_tuning + C][numel] dtype, device             */
  int32_t* remap;            /* [E] device or NULL: compact slot of every expert             */
} flux_merge_job;
flux_status flux_merge_experts_batch(flux_dtype dtype, int32_t n_experts, int64_t numel, int32_t n_jobs,
                                     const flux_merge_job* jobs, int32_t compact, void* stream);

/* ---------------------------------------------------------------------------
 * NEXT-2: the compact model after merging (§5.3 + §7 "Customized MoE construction",
 * "Gate re-routing") and its quality measure.
 * ------------------------------------------------------------------------- */
/* eq.(2) as flux_merge_experts, but the output holds every slot of the compact model in
 * remap order: compact[remap[e]] for all e — each tuning expert copied bit for bit (a
 * singleton with weight α/α = 1), then the C merged clusters.  compact: [n_tun + C][numel]
 * (n_tun = the number of -1 entries; slots at index >= n_experts are never written, which
 * only concerns n_tun + C > E, where some clusters are necessarily empty).
 * Feed the slots to flux_profile_layer with wbits = 16, n_experts = n_tun + C,
 * n_router = E and flux_qlayer.remap = remap (the gate keeps scoring the original experts). */
flux_status flux_compact_experts(flux_dtype dtype, int32_t n_experts, int64_t numel, const void* experts,
                                 const int32_t* cluster_of, const float* alpha, int32_t n_clusters, void* compact,
                                 int32_t* remap, void* stream);
/* The paper's merge output error: the average over T tokens of the
 * cosine distance 1 - a_t·b_t/(|a_t||b_t|) between two bf16 [T][H] outputs (the merged and the
 * original model's final token outputs); fp64 accumulation, fixed order (deterministic).
 * result: device double [1]; ws: device, >= flux_output_error_workspace() bytes. */
size_t flux_output_error_workspace(void);
flux_status flux_output_error(int64_t T, int32_t hidden, const void* a, const void* b, double* result, void* ws,
                              size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * NEXT-1: similarity-based expert clustering, §5.2.
 * ------------------------------------------------------------------------- */
/* Bytes of device workspace flux_expert_features needs (16-byte aligned); fam_numel: HOST
 * int64 [n_fam] (per-expert element count of each family).  0 on invalid arguments. */
size_t flux_expert_features_workspace(int32_t n_layers, int32_t n_experts, int32_t n_fam, const int64_t* fam_numel);
/* C1, reading R12: PCA features of the experts of each layer.  Expert e is
 * the concatenation of its parameter families (e.g. gate|up, down); family f of layer l
 * is fam[l*n_fam + f], a bf16 device array [E][fam_numel[f]] (expert-major, contiguous;
 * fam: HOST array of device pointers).  Per layer: raw Gram G = Σ_f X_f X_fᵀ (tensor
 * cores, fp32 accumulation over 2048-column sub-chunks, 4096-column chunks claimed
 * dynamically by the CTAs, chunk partials summed in fp64 in chunk order: deterministic),
 * centred H G H, fp64 Jacobi
 * eigendecomposition, scores features[l][e][j] = V[e][j]·sqrt(max(λ_j,0)) for the top-d
 * eigenvalues (descending).  Each score column is defined up to sign.
 * Outputs (device, fp32): features [L][E][d]; gram [L][E][E] raw Gram (NULL = skip);
 * eigvals [L][d] (NULL = skip).  2 <= E <= 128, 1 <= d <= min(E, 32), 1 <= n_fam <= 4, fam_numel % 8 == 0,
 * pointers 16-byte aligned.  Asynchronous on `stream`. */
flux_status flux_expert_features(int32_t n_layers, int32_t n_experts, int32_t n_fam, const void* const* fam,
                                 const int64_t* fam_numel, int32_t d, float* features, float* gram, float* eigvals,
                                 void* ws, size_t ws_bytes, void* stream);
/* C2, reading R13: fused, layer-masked cosine K-Means over all layers (one
 * CTA per layer; masking cross-layer distances decouples the layers exactly).  Init: the
 * n_clusters[l] non-tuning experts with the highest count (ties: lower id); assignment
 * argmin of 1 - cos (ties: lower centroid); update: member mean (empty: unchanged);
 * stop when no assignment changes or after max_iter iterations.  fp64 arithmetic.
 * features: device fp32 [L][E][d]; counts: device int64 [L][E] (the profiled
 * histograms, frequency = count / T); n_clusters: HOST int32 [L], 1 <= B(l) <= number of
 * non-tuning experts; tuning: HOST uint8 [L][E] (non-zero = tuning expert, NULL = none).
 * cluster_of: device int32 [L][E] (-1 for tuning experts, ready for flux_merge_experts);
 * iterations: device int32 [L] (NULL = skip).  L <= 128, E <= 128, d <= 32. */
flux_status flux_cluster_experts(int32_t n_layers, int32_t n_experts, int32_t d, const float* features,
                                 const int64_t* counts, const int32_t* n_clusters, const uint8_t* tuning,
                                 int32_t max_iter, int32_t* cluster_of, int32_t* iterations, void* stream);

/* ---------------------------------------------------------------------------
 * NEXT-3: attention-weighted importance α_e = f_e·ā_e of eq.(2), reading R15.
 * ------------------------------------------------------------------------- */
/* attn_hist[e] += Σ over live picks (t, j) with ids[t][j] == e of RNE(attn[t]·2^24), int64.
 * ā_e = the average attention value of the tokens assigned to e, f_e = count_e / T, so
 * α_e = f_e·ā_e = attn_hist[e] / (2^24·T): an integer statistic, exact, order-free and
 * additive over ranks (reduce it with flux_reduce_stats like the histogram).
 * ids: device int32 [T][top_k] (flux_profile_layer's topk_ids; -1 = folded pick, skipped);
 * attn: device fp32 [T], 0 <= a_t < 2^30 (the per-token attention value of the model's
 * attention layer — outside this path); attn_hist: device int64 [n_experts], accumulated. */
flux_status flux_attention_hist(int64_t T, int32_t top_k, int32_t n_experts, const int32_t* ids, const float* attn,
                                int64_t* attn_hist, void* stream);

/* The merge importance on the device: alpha[i] = fl32(counts[i] / denom) (fp64 quotient, one rounding)
 * — the activation frequency f = count / T (denom = T_total) or α = f·ā = A / (2^24·T)
 * (denom = 2^24·T_total, reading R15).  counts: device int64 [n]; alpha: device fp32 [n]; denom > 0.
 * Lets a round go from the reduced statistics to the merge without a host round trip. */
flux_status flux_frequencies(int64_t n, const int64_t* counts, double denom, float* alpha, void* stream);

/* ---------------------------------------------------------------------------
 * Statistics all-reduce over the GPUs of one box (NCCL over NVLink/NVSwitch).
 * The counts are additive integers, so the reduced histogram equals the
 * single-GPU histogram of the union of the shards bit for bit.
 * ------------------------------------------------------------------------- */
typedef struct flux_comm flux_comm;
/* Rank 0 creates the 128-byte NCCL unique id; the caller distributes it. */
flux_status flux_comm_unique_id(void* out_128_bytes);
/* Collective over all ranks; binds to the current CUDA device. */
flux_status flux_comm_init(flux_comm** out, const void* unique_id_128_bytes, int32_t nranks, int32_t rank);
/* In-place sum of `count` int64 counters (device pointer) on `stream`. */
flux_status flux_reduce_stats(flux_comm* comm, int64_t* hist, size_t count, void* stream);
flux_status flux_comm_destroy(flux_comm* comm);

/* ---------------------------------------------------------------------------
 * Helpers (not per-token hot).
 * ------------------------------------------------------------------------- */
/* Weight quantizer, reading R1: symmetric, per row,
 * groups of g along K (g = K if group_size == 0):
 *   s = fl32(max|w| / qmax), q = clamp(RNE(fl32(w/s)), -qmax-1, qmax), s = 0 -> q = 0
 * w: [R][K] bf16 or fp32 device; q: [R][K] int8, [R][K/2] packed int4 or [R][K/4] packed int2
 * (element k in bits 2(k mod 4)); s: fp32 [R][K/g].  wbits 8, 4 or 2 (qmax = 2^(b-1) - 1).
 * Bit-exact (IEEE division, no fast-math).  Needs K % 8 == 0 for INT2. */
flux_status flux_quantize_weights(int32_t wbits, int32_t group_size, flux_dtype in_dtype, const void* w, int64_t R,
                                  int64_t K, void* q, float* s, void* stream);

/* The quantized model's bf16 B operands ("bops"): on the dequant-pass path
 * (flux_profile_layer_uses_bops == 1) the expert GEMMs stream a layer's weights as bf16,
 * ŵ = bf16(q·bf16(s)) for grouped codes and bf16(q) per channel (scale in the GEMM epilogue) —
 * reading R1b.  flux_profile_layer materialises them in its workspace with one dequantization
 * pass per call; a caller that quantizes once and profiles many times (every chunk of a round) can
 * instead produce them with the quantizer and hand them in.  A layer's bops buffer is
 * flux_layer_bops_bytes(cfg) bytes, 16-byte aligned, layout private to the library; rows that pad
 * F to a multiple of 128 are never written or read as data (zero the buffer once if it must be
 * deterministic bytewise).
 *   flux_quantize_weights_bops   one weight family of n_layers consecutive layers, quantized exactly
 *       as flux_quantize_weights does (w, q, s: the family's [n_layers·rows][K] matrices) AND written
 *       into bops + l·bops_stride as B operands in the same pass (the bytes flux_dequantize_layer
 *       would write from q and s).  family: FLUX_FAM_*; rows x K = [E·F][H] (gate, up), [E·H][F]
 *       (down), [F_s][H] / [H][F_s] (shared).  wbits 2, 4 or 8.
 *   flux_dequantize_layer         the dequantization pass alone: w's q, s -> bops.
 *   flux_profile_layer_bops       flux_profile_layer_ex with this layer's bops (NULL = dequantize in
 *       the workspace as usual); bit-identical outputs.  ws >= flux_profile_layer_workspace_bops.
 *   flux_profile_layer_uses_bops  1 / 0: whether T tokens take the dequant-pass path; -1 invalid. */
enum { FLUX_FAM_GATE = 0, FLUX_FAM_UP = 1, FLUX_FAM_DOWN = 2, FLUX_FAM_SH_GATE = 3, FLUX_FAM_SH_UP = 4, FLUX_FAM_SH_DOWN = 5 };
size_t flux_layer_bops_bytes(const flux_moe_cfg* cfg);
flux_status flux_quantize_weights_bops(const flux_moe_cfg* cfg, int32_t family, flux_dtype in_dtype, const void* w,
                                       int32_t n_layers, void* q, float* s, void* bops, size_t bops_stride,
                                       void* stream);
flux_status flux_dequantize_layer(const flux_moe_cfg* cfg, const flux_qlayer* w, void* bops, void* stream);
int32_t flux_profile_layer_uses_bops(const flux_moe_cfg* cfg, const flux_policy* policy, int64_t T);
size_t flux_profile_layer_workspace_bops(const flux_moe_cfg* cfg, const flux_policy* policy, int64_t T);
flux_status flux_profile_layer_bops(const flux_moe_cfg* cfg, const flux_policy* policy, const flux_qlayer* w,
                                    const void* bops, const void* x, const void* residual, int64_t T,
                                    const flux_layer_out* out, void* ws, size_t ws_bytes, void* stream);

/* Adaptive expert layer size, eq.(1), reading R9 (host function):
 *   f_l = hist[l][·]/T, v_l = population variance of f_l, b_l = (L-l+1)/max(v_l,1e-12) (l = 1..L),
 *   C_l = clamp(floor(b_l/Σ_k b_k · B_non), 1, n_non[l]).
 * hist: host int64 [L][E]; n_non: host int32 [L] (NULL = E); C_out: host int32 [L].
 * *overrun (may be NULL) = Σ C_l - B_non. */
flux_status flux_layer_budget(int32_t L, int32_t E, const int64_t* hist, int64_t T, int64_t B_non,
                              const int32_t* n_non, int32_t* C_out, int64_t* overrun);

/* ---------------------------------------------------------------------------
 * Diagnostics (benchmarking only).
 * ------------------------------------------------------------------------- */
/* Opt-in: while on, every hot launch records a CUDA event pair on its own stream. */
void flux_timing_enable(int on);
/* Synchronises pending events and returns per-kernel totals: ms_out[i] (milliseconds) and
 * count_out[i] (launches) for kernel kind i (names: flux_kernel_name); reset != 0 clears them.
 * Returns the number of kernel kinds. */
int flux_timing_read(double* ms_out, long long* count_out, int n, int reset);
const char* flux_kernel_name(int kind);
/* Average SM clock in MHz measured INSIDE the probed kernels (the CTA-pair expert GEMMs: one thread
 * reads %clock64 and %globaltimer at the kernel's start and end) while timing is enabled, per kernel
 * kind; 0 where nothing was probed.  Synchronises the device.  Returns the number of kernel kinds. */
int flux_timing_clocks(double* mhz_out, int n, int reset);
/* Text of the last CUDA error this thread's calls saw ("" if none).  With the
 * environment variable FLUX_DEBUG_SYNC=1 every launch is synchronised and a
 * failure names the kernel that raised it. */
const char* flux_last_error(void);
/* Total kernels this library has launched in the process (monotonic). */
long long flux_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* FLUX_H_ */
