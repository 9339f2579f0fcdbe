// internal.h — host-side declarations shared by the libflux translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/flux.h"

namespace flux {

constexpr int kNumSMs = 148;
constexpr int kRouterTile = 256;  // tokens per router tile: the unit of tile_counts / tile_base / rank

// TMA descriptor for a row-major 2D tensor [rows][cols] of `elem_bytes` elements,
// box = box_cols x box_rows, 128-byte swizzle (box_cols * elem_bytes must be 128 or
// the swizzle must be NONE), out-of-bounds elements read as zero.
bool make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, uint32_t elem_bytes, uint64_t rows,
                  uint64_t cols, uint64_t row_stride_bytes, uint32_t box_cols, uint32_t box_rows,
                  CUtensorMapSwizzle swizzle);
bool make_tmap_gram_blocks(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                           uint32_t n_blocks);

inline flux_status cuda_status(cudaError_t e) { return e == cudaSuccess ? FLUX_OK : FLUX_E_CUDA; }

// ---------------------------------------------------------------- per-kernel timing (timing.cpp)
enum KernelKind {
  K_QUANTIZE = 0, K_DEQUANT, K_ROUTER, K_PERMUTE, K_SCATTER, K_GEMM_GU, K_GEMM_DN, K_COMBINE, K_MERGE,
  K_GEMM_DN_SH_COMBINE, K_GEMM_CHAIN, K_GRAM, K_GRAM_REDUCE, K_EIG, K_KMEANS, K_COSINE, K_ATTN_HIST, K_FREQ, FLUX_NUM_KERNELS
};
// RAII: counts one launch; when timing is enabled records CUDA events around it on `st`.
class KernelTimer {
 public:
  KernelTimer(int kind, cudaStream_t st);
  ~KernelTimer();
  KernelTimer(const KernelTimer&) = delete;
  KernelTimer& operator=(const KernelTimer&) = delete;

 private:
  int kind_;
  cudaStream_t st_;
  cudaEvent_t a_ = nullptr, b_ = nullptr;
};

void set_last_error(const char* what, cudaError_t e);
// Device slots [Σ clocks, Σ ns] of kernel kind `kind` while timing is enabled, else null (timing.cpp).
unsigned long long* clock_probe(int kind);
const char* last_error();

// ---------------------------------------------------------------- launchers
// K0 (quantize.cu)
// Optional fused output of the quantizer: the family's bf16 B operands exactly as launch_dequant writes
// them (ŵ = bf16(q·bf16(s)) grouped, bf16(q) per channel), for the rows of n consecutive layers.
// Unsigned division by a run-time constant d >= 1 for n < 2^31 (Granlund-Montgomery): q = (umulhi(n, m) + n) >> l.
struct FastDiv {
  uint32_t d, m, l;
};
inline FastDiv make_fastdiv(uint32_t d) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  const uint64_t m = ((1ull << 32) * ((1ull << l) - d)) / d + 1;
  return {d, (uint32_t)m, l};
}
struct BopsOut {
  void* out;              // this family's B-operand region in layer 0's buffer (null = no fused output)
  int64_t layer_stride;   // bytes between consecutive layers' buffers
  FastDiv ipr;            // quantization groups per row (K / g)
  FastDiv layer_rows;     // rows of this family per layer (G·N)
  FastDiv n;              // N, rows per expert
  int Fp, interleave, up, ldo, per_channel;  // launch_dequant's row mapping; up: the up half of gate/up
};
cudaError_t launch_quantize(int wbits, int64_t g, bool in_fp32, const void* w, int64_t R, int64_t K, void* q, float* s,
                            cudaStream_t st, const BopsOut* bo = nullptr);
// K7 (merge.cu)
constexpr int kMergeMaxJobs = 256;
struct MergeJob {           // one weight family of one layer
  const void* experts;      // [E][numel]
  const int32_t* cluster_of;// [E]
  const float* alpha;       // [E]
  void* merged;             // [n_out][numel]
  int32_t* remap;           // [E] or null
  int n_clusters;
  int n_slots;              // compact mode: n_tun + n_clusters (0 = unknown, E used as the bound)
};
struct MergeBatch {
  int n_jobs, E, compact;
  int64_t numel;
  MergeJob jobs[kMergeMaxJobs];
  int64_t chunk_prefix[kMergeMaxJobs + 1];  // filled by launch_merge_batch
};
cudaError_t launch_merge_batch(bool fp32, const MergeBatch& b, cudaStream_t st);
cudaError_t launch_merge(bool fp32, int E, int64_t numel, const void* experts, const int32_t* cluster_of,
                         const float* alpha, int C, void* merged, int32_t* remap, cudaStream_t st, int compact = 0);
// output error of a merged model: mean over tokens of 1 - cos(a_t, b_t)
cudaError_t launch_attention_hist(int64_t T, int k, int E, const int32_t* ids, const float* attn, int64_t* A,
                                  cudaStream_t st);
size_t cosine_workspace();
cudaError_t launch_frequencies(int64_t n, const int64_t* counts, double denom, float* alpha, cudaStream_t st);
cudaError_t launch_cosine_distance(int64_t T, int H, const void* a, const void* b, double* ws, double* out,
                                   cudaStream_t st);

// NEXT-1 expert clustering (cluster.cu), §5.2
constexpr int kClusterMaxE = 128, kClusterMaxD = 32, kClusterMaxL = 128;
struct KMeansArgs {
  int32_t n_clusters[kClusterMaxL];  // B(l)
  uint64_t tuning[kClusterMaxL][2];  // bit e set: expert e of layer l is a tuning expert (not clustered)
};
size_t features_workspace(int L, int E, int n_fam, const int64_t* P);
float* features_gram_slot(void* ws, int E, int n_fam, const int64_t* P, int l);
int* features_counter(void* ws, int L, int E, int n_fam, const int64_t* P);
constexpr int kClusterMaxFam = 4;
cudaError_t launch_gram(int E, int n_fam, const void* const* X, const int64_t* P, float* partial, int* counter,
                        int* n_slots, cudaStream_t st);
cudaError_t launch_gram_reduce(int E, const float* partial, int n_slots, float* G, float* G_user, int* counter,
                               cudaStream_t st);
cudaError_t launch_eig(int L, int E, int d, const float* G, float* features, float* eigvals, cudaStream_t st);
cudaError_t launch_kmeans(int L, int E, int d, const float* features, const int64_t* counts, const KMeansArgs& ka,
                          int max_iter, int32_t* cluster_of, int32_t* iters, cudaStream_t st);

// K1 (router.cu)
struct RouterArgs {
  int64_t T;
  int H, E, k, norm;
  int32_t* ids;         // [T][k]
  float* w;             // [T][k]
  float* logits;        // [T][E] or null
  int64_t* hist;        // [E] (+=)
  int32_t* tile_counts; // [n_tiles][E]
  int32_t* rank;        // [T][k] rank of t inside its router tile among tokens choosing the same expert
  int E_slots;           // experts of the weights (hist, tile counts); == E unless re-routing
  const int32_t* remap;  // [E] pick -> slot (NEXT-2 gate re-routing) or null
  int32_t* zero4;        // 4 ints zeroed by the router (the K2 grid barrier + the pair-GEMM tile counters)
};
cudaError_t launch_router(const CUtensorMap& tmap_x, const CUtensorMap& tmap_wr, int npad, const RouterArgs& a,
                          cudaStream_t st);

// K2 (permute.cu)
struct ScheduleArgs {
  int E, k;
  int64_t T;
  int n_tiles;              // router tiles (kRouterTile tokens)
  const int32_t* tile_counts;
  int32_t* tile_base;       // [n_tiles][E]
  int32_t* offsets;         // [E+1] internal
  int32_t* user_offsets;    // [E+1] or null
  int32_t* done_counter;    // 4 ints: [0] K2 ticket / grid barrier, [1..3] pair-GEMM tile counters
  int has_shared;
  int n_tiles_gu, n_tiles_gu_sh;  // n-tiles of the gate/up GEMM (routed, shared)
  int n_tiles_dn, n_tiles_dn_sh;  // n-tiles of the down GEMM
  int32_t* sched_gu;        // [n_groups+1] tile prefix of the gate/up GEMM
  int32_t* sched_dn;        // [n_groups+1]
  int32_t* grp_row0;        // [n_groups] first A row of each group
  int32_t* grp_rows;        // [n_groups] rows of each group
  int gemm_bm;              // GEMM tile rows (128 or 256)
  int32_t* sched_c;         // [n_groups+1] chained gate/up + down tile prefix (null = not chained)
  int32_t* mt_base;         // [n_groups] first global m-tile of each group (chained)
  int32_t* ready;           // [M_total] per-m-tile act completion counters, zeroed by K2 (chained)
  int32_t* sched_sh;        // [2] tile prefix of the shared-MLP-only down GEMM (fused combine)
  int32_t* grp_row0_sh;     // [1] = 0
  int32_t* grp_rows_sh;     // [1] = T
};
// K2 as ONE kernel (schedule + index scatter; the counters are zeroed by the router): ids, rank from K1
// -> tile_base, offsets, GEMM schedules, inv_pos [T][k], token_index [T*k]
cudaError_t launch_permute(const ScheduleArgs& a, const int32_t* ids, const int32_t* rank, int32_t* inv_pos,
                           int32_t* token_index, cudaStream_t st);
cudaError_t launch_scatter(const void* x, int64_t T, int H, int E, int k, const int32_t* ids, const int32_t* rank,
                           const int32_t* tile_base, const int32_t* offsets, int32_t* inv_pos, int32_t* token_index,
                           void* x_perm, cudaStream_t st);

// K6 (combine.cu)
cudaError_t launch_combine(int64_t T, int H, int k, const void* residual, const void* y_sh, const void* y_perm,
                           const float* w, const int32_t* inv_pos, void* y, cudaStream_t st,
                           bool empty_picks = false);

// K3/K4/K5 (gemm_pair.cu, gemm_chain.cu; the dequant pass in dequant.cu)
enum GemmEpi { EPI_SWIGLU = 0, EPI_STORE = 1, EPI_COMBINE = 2 };
struct GemmArgs {
  // groups 0..E-1: routed experts (A = tm_a_r rows grp_row0.., B = tm_b_r rows g*b_rows_r..);
  // group E (if n_groups > E): the shared MLP (A = tm_a_s, B = tm_b_s)
  int n_groups, E;
  const int32_t* sched;     // [n_groups+1] tile prefix (device, written by K2)
  const int32_t* grp_row0;  // [n_groups] first A row per group (device)
  const int32_t* grp_rows;  // [n_groups] rows per group (device)
  int n_tiles_r, n_tiles_s; // n-tiles per group (routed, shared)
  int K_r, K_s;             // contraction length (routed, shared)
  int N_r, N_s;             // output features per group
  int b_rows_r;             // rows of one routed group in the B tensor
  const float *cs0_r, *cs1_r, *cs0_s, *cs1_s;  // per-channel scales [group][N] or null
  void *out_r, *out_s;      // bf16 [rows][ld]
  int64_t ld_r, ld_s;
  int64_t rows_r, rows_s;   // rows of out_r / out_s (TMA-store tensor maps of the CTA-pair kernel)
  int grid;
  int bm;                   // rows per tile: 256 (CTA-pair kernel)
  // EPI_COMBINE only (shared-MLP down GEMM whose epilogue writes the layer output)
  const void* resid;        // bf16 [T][H]
  const void* y_perm;       // bf16 [T*k][H] routed expert outputs
  const float* topk_w;      // [T][k]
  const int32_t* inv_pos;   // [T][k]
  int k;
  // routed A rows gathered from x (tm_a_r = gather map over x, box {64,1}) by token_index; null =
  // rows read contiguously from a materialised x_perm / act
  const int32_t* gather_idx;
  // CTA-pair pass-path kernel only: gather the rows with per-lane 16-byte cp.async (LDGSTS) from
  // a_src (bf16 [T][a_ld]) instead of TMA tile::gather4 (tm_a_r unused for routed tiles then)
  int gather_cp;
  const void* a_src;
  int a_ld;
  int32_t* tile_ctr;  // CTA-pair kernels: zeroed int the pair leaders claim tiles from (null = static)
  int l2_hints;  // L2 cache policies of the CTA-pair pass kernel: bit 0 = evict_first on the output
                 // stores, bit 1 = evict_last on the B loads, bit 2 = evict_first on the A loads
  unsigned long long* clk_probe;  // diagnostics: [Σ SM clocks, Σ ns] of this launch added by CTA 0 (or null)
};
cudaError_t launch_gemm(GemmEpi epi, const CUtensorMap& a_r, const CUtensorMap& a_s, const CUtensorMap& b_r,
                        const CUtensorMap& b_s, const GemmArgs& a, cudaStream_t st);
// K3 + K4 chained in one persistent launch (gemm_chain.cu): gate/up (args g0, maps *0) and down (g1, *1)
struct ChainArgs {
  const int32_t* sched_c;  // [n_groups+1] (K2)
  const int32_t* mt_base;  // [n_groups] (K2)
  int32_t* ready;          // [M_total], zeroed by K2
  int D;                   // lag of a group's down tiles behind its gate/up tiles, in m-tiles
  int32_t* tile_ctr;       // zeroed int
};
cudaError_t launch_gemm_chain(const CUtensorMap& a_r0, const CUtensorMap& a_s0, const CUtensorMap& b_r0,
                              const CUtensorMap& b_s0, const CUtensorMap& a_r1, const CUtensorMap& a_s1,
                              const CUtensorMap& b_r1, const CUtensorMap& b_s1, const GemmArgs& g0,
                              const GemmArgs& g1, const ChainArgs& ca, cudaStream_t st);

// Fused-dequant variant (CTA pairs): B comes straight from the quantized weights.
struct QGemmArgs {
  GemmArgs base;                 // bm must be 256
  int wbits;                     // 4 or 8
  int gsz;                       // group size along K; 0 = per output channel (scale in the epilogue)
  int gate_up;                   // 1: CTA rank 0 dequantizes gate rows, rank 1 the matching up rows
                                 // 0: rank r dequantizes rows [128r, 128r+128) of the 256-row tile
  int qrows_r, qrows_s;          // rows of one group in the quantized tensor (routed, shared)
  int64_t qtotal_r, qtotal_s;    // total rows of the quantized tensors
  const float *gs_r0, *gs_r1, *gs_s0, *gs_s1;  // group scales [rows][K/gsz] of the rank-0 / rank-1 sources
};
cudaError_t launch_gemm_q(GemmEpi epi, const CUtensorMap& a_r, const CUtensorMap& a_s, const CUtensorMap& q_r0,
                          const CUtensorMap& q_r1, const CUtensorMap& q_s0, const CUtensorMap& q_s1,
                          const QGemmArgs& a, cudaStream_t st);
cudaError_t launch_dequant(int wbits, const uint8_t* q0, const float* s0, const uint8_t* q1, const float* s1, int G,
                           int N, int K, int Fp, int interleave, int gsz, int per_channel, int ldo, void* out,
                           cudaStream_t st);

}  // namespace flux
