// api.cu — the C ABI of libflux.so (include/flux.h): argument validation,
// workspace carving, TMA descriptors and the launch sequence of one profiled
// MoE layer.  Every step of the computation runs in the kernels of this
// library; there is no host or CPU fallback path.
#include <algorithm>
#include <mutex>

#include "internal.h"

namespace flux {

// ---------------------------------------------------------------- TMA descriptor creation
namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
std::once_flag g_encode_once;

EncodeTiledFn encode_fn() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  });
  return g_encode;
}
}  // namespace

bool make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, uint32_t elem_bytes, uint64_t rows,
                  uint64_t cols, uint64_t row_stride_bytes, uint32_t box_cols, uint32_t box_rows,
                  CUtensorMapSwizzle swizzle) {
  EncodeTiledFn f = encode_fn();
  if (!f) return false;
  cuuint64_t dims[2] = {cols, std::max<uint64_t>(rows, 1)};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  (void)elem_bytes;
  CUresult r = f(map, dtype, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// X bf16 [rows][cols] seen as [cols/64 blocks][rows][64]: element (c, r, b) at r·cols + 64·b + c.  One
// box {64, box_rows, n_blocks} lands in shared memory as n_blocks consecutive [box_rows][128 B] tiles
// (128B-swizzled: the K-major operand layout of the Gram MMA).
bool make_tmap_gram_blocks(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                           uint32_t n_blocks) {
  EncodeTiledFn f = encode_fn();
  if (!f) return false;
  cuuint64_t dims[3] = {64, std::max<uint64_t>(rows, 1), cols / 64};
  cuuint64_t strides[2] = {cols * 2, 128};
  cuuint32_t box[3] = {64, box_rows, n_blocks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = f(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static bool tmap_bf16(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                      uint64_t ld = 0 /* row length in elements, default cols */) {
  return make_tmap_2d(m, base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rows, cols, (ld ? ld : cols) * 2, 64, box_rows,
                      CU_TENSOR_MAP_SWIZZLE_128B);
}

// ---------------------------------------------------------------- device check
static flux_status check_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FLUX_E_CUDA;
  int major = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return FLUX_E_CUDA;
  return major == 10 ? FLUX_OK : FLUX_E_CUDA;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ---------------------------------------------------------------- performance policy (flux_policy)
// Every choice produces bit-identical outputs (tests/test_gpu_parity.py::test_weight_paths_bit_identical);
// the defaults are the measured winners on B200.  Paths measured slower are kept only as
// test-only values of the policy, so the bit-identity test can pin them against the defaults.
//  * weight path — where the bf16 B operand of the expert GEMMs comes from (bf16(q·bf16(s)) or exact q):
//    in-GEMM dequant warps convert each B tile per m-tile (best when few tokens reach each expert); one
//    dequantization pass per layer feeds TMA-loaded bf16 tiles (best when every B tile is reused by many
//    m-tiles: 262,144 tokens = ~96 m-tiles per expert).  Auto: the pass when the average routed rows per
//    expert reach 8 tile rows (T·k >= 2048·E).
//  * routed A rows of the gate/up GEMM: gathered from x inside the GEMM by two producer warps with per-lane
//    16-byte cp.async (default on the pass path: K2 then writes only the D_e indices; measured +5% tokens/s
//    in the bench step on both BASELINE shapes, the lower HBM power raises the capped clocks), materialised
//    by K2 as x_perm (the in-GEMM-dequant kernel always), or TMA tile::gather4 (test-only: ~2.5x slower GEMM).
//  * K6 placement: standalone (default) or fused into the shared-MLP down-GEMM epilogue (test-only: ties
//    the standalone kernel in isolation, 0.6% behind in the bench step with claimed tiles).
//  * tile order of the CTA-pair GEMMs: claimed in global order from a counter (default: the n-tiles of an
//    m-tile run together and share their A rows in L2; gate/up and down read 8.3 / 6.3 GB per DeepSeek
//    layer from DRAM instead of 8-12 / 10-17 GB) or static round-robin over the 74 pairs (test-only).
//  * L2 hints (bits): 1 = evict_first on the act / y_perm TMA stores (default; the down GEMM's DRAM reads
//    12.1 -> 10.7 GB per layer), 2 = evict_last on B, 4 = evict_first on A (both measured worse).
enum GatherMode { GATHER_NONE = 0, GATHER_TMA = 1, GATHER_CP = 2 };
struct Policy {
  bool pass;
  GatherMode gmode;
  bool fused_combine;
  bool dynamic_tiles;
  int l2_hints;
  bool chain;  // gate/up + down in one launch (gemm_chain.cu)
};
static Policy resolve_policy(const flux_moe_cfg& c, const flux_policy* up, int64_t T) {
  flux_policy d{};
  const flux_policy& u = up ? *up : d;
  Policy p;
  if (c.wbits == 16 || c.wbits == 2) p.pass = true;  // bf16 copy / INT2 codes: the in-GEMM kernel does INT4/INT8
  else if (u.weight_path == FLUX_WEIGHTS_DEQUANT_PASS) p.pass = true;
  else if (u.weight_path == FLUX_WEIGHTS_IN_GEMM) p.pass = false;
  else p.pass = T * c.top_k >= (int64_t)2048 * c.n_experts;
  if (u.routed_rows == FLUX_ROWS_MATERIALISED) p.gmode = GATHER_NONE;
  else if (u.routed_rows == FLUX_ROWS_TMA_GATHER4) p.gmode = GATHER_TMA;
  else p.gmode = p.pass ? GATHER_CP : GATHER_NONE;
  p.fused_combine = u.fused_combine != 0 && c.shared_ffn > 0;
  p.dynamic_tiles = u.static_tiles == 0;
  p.l2_hints = (u.l2_hints & FLUX_L2_SET) ? (u.l2_hints & 7) : 1;
  // chained GEMMs need the dequant-pass kernels with the cp.async gather, claimed tiles and the standalone
  // combine, and at most 128 routed groups (+ the shared MLP); auto = off until measured faster
  p.chain = u.gemm_chain == FLUX_CHAIN_ON && p.pass && p.gmode == GATHER_CP && p.dynamic_tiles && !p.fused_combine &&
            c.n_experts <= 128;
  return p;
}
static flux_status validate_policy(const flux_policy* u) {
  if (!u) return FLUX_OK;
  if (u->weight_path < 0 || u->weight_path > 2 || u->routed_rows < 0 || u->routed_rows > 2 ||
      (u->fused_combine != 0 && u->fused_combine != 1) || (u->static_tiles != 0 && u->static_tiles != 1) ||
      (u->l2_hints != 0 && (!(u->l2_hints & FLUX_L2_SET) || (u->l2_hints & ~(FLUX_L2_SET | 7)) != 0)) ||
      u->gemm_chain < 0 || u->gemm_chain > 2)
    return FLUX_E_INVALID;
  return FLUX_OK;
}

static bool tmap_u8(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols_bytes, uint32_t box_cols) {
  return make_tmap_2d(m, base, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, rows, cols_bytes, cols_bytes, box_cols, 128,
                      CU_TENSOR_MAP_SWIZZLE_NONE);
}
// A operand of the routed gate/up GEMM: a gather map over x (box {64 cols, 1 row}, rows picked by
// token_index with tile::gather4) for the CTA-pair kernels, else the materialised x_perm.
static bool tmap_a_routed(CUtensorMap* m, bool gather, const void* x, const void* x_perm, int64_t T, int64_t Tk,
                          int H) {
  if (gather) return tmap_bf16(m, x, T, H, 1);
  return tmap_bf16(m, x_perm, Tk, H, 128);
}

// ---------------------------------------------------------------- workspace layout
namespace {
struct Layout {
  size_t off = 0;
  size_t take(size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  }
};
struct WsPlan {
  size_t tile_counts, tile_base, rank, offsets, token_index, inv_pos, counter, sched_gu, sched_dn, row0, rows;
  size_t x_perm, y_perm, act, act_sh, sh_sched, y_sh, wgu_r, wdn_r, wgu_s, wdn_s, sched_c, mt_base, ready;
  size_t total;
};
int pad128(int v) { return (v + 127) / 128 * 128; }
// Row length (elements) of the bf16 buffers whose K is F or F_s (act, act_sh, the down-projection B
// operands): padded to 64 elements so every row starts on a 128-byte line.  F = 688 (LLaMA shape)
// has 1376-byte rows, and every 128-byte TMA row segment of an unpadded buffer straddles two lines.
// The tensor maps keep the logical width F, so the pad columns are never read (no zeroing needed).
int pad64(int v) { return (v + 63) / 64 * 64; }

// The bf16 B operands of one layer (the dequantization pass's output).  The caller-owned buffer of
// flux_quantize_weights_bops / flux_dequantize_layer / flux_profile_layer_bops has this layout,
// sized by flux_layer_bops_bytes.
struct BopsPlan {
  size_t gu_r, dn_r, gu_s, dn_s, total;
};
BopsPlan bops_plan(const flux_moe_cfg& c, bool present = true) {
  Layout L;
  BopsPlan b;
  const size_t on = present ? 1 : 0;
  b.gu_r = L.take(on * 2ull * c.n_experts * 2 * pad128(c.ffn) * c.hidden);
  b.dn_r = L.take(on * 2ull * c.n_experts * c.hidden * pad64(c.ffn));
  b.gu_s = L.take(on * 2ull * 2 * pad128(c.shared_ffn) * c.hidden);
  b.dn_s = L.take(on * 2ull * c.hidden * pad64(c.shared_ffn));
  b.total = L.off;
  return b;
}

// ext_bops: the caller supplies the B operands (flux_profile_layer_bops): none in the workspace
WsPlan plan(const flux_moe_cfg& c, const Policy& pol, int64_t T, bool ext_bops = false) {
  Layout L;
  WsPlan p;
  const int64_t n_rt = (T + kRouterTile - 1) / kRouterTile;
  const int64_t Tk = T * c.top_k;
  const int n_groups = c.n_experts + (c.shared_ffn > 0);
  p.tile_counts = L.take(sizeof(int32_t) * n_rt * c.n_experts);
  p.tile_base = L.take(sizeof(int32_t) * n_rt * c.n_experts);
  p.rank = L.take(sizeof(int32_t) * Tk);
  p.offsets = L.take(sizeof(int32_t) * (c.n_experts + 1));
  p.token_index = L.take(sizeof(int32_t) * Tk);
  p.inv_pos = L.take(sizeof(int32_t) * Tk);
  p.counter = L.take(4 * sizeof(int32_t));  // K2's ticket + the tile counters of the three pair GEMM launches
  p.sched_gu = L.take(sizeof(int32_t) * (n_groups + 1));
  p.sched_dn = L.take(sizeof(int32_t) * (n_groups + 1));
  p.row0 = L.take(sizeof(int32_t) * n_groups);
  p.rows = L.take(sizeof(int32_t) * n_groups);
  // x_perm (routed A rows materialised by K2) unless the GEMM gathers them; y_perm always.
  p.x_perm = L.take(pol.gmode != GATHER_NONE ? 0 : 2ull * Tk * c.hidden);
  p.y_perm = L.take(2ull * Tk * c.hidden);
  p.act = L.take(2ull * Tk * pad64(c.ffn));
  p.act_sh = L.take(2ull * T * pad64(c.shared_ffn));
  p.sh_sched = L.take(4 * sizeof(int32_t));  // sched_sh[2], row0_sh[1], rows_sh[1]
  p.y_sh = L.take(c.shared_ffn && !pol.fused_combine ? 2ull * T * c.hidden : 0);
  // bf16 B operands only for the separate-pass path, unless the caller supplies them
  const BopsPlan b = bops_plan(c, pol.pass && !ext_bops);
  const size_t b0 = L.take(b.total);
  p.wgu_r = b0 + b.gu_r;
  p.wdn_r = b0 + b.dn_r;
  p.wgu_s = b0 + b.gu_s;
  p.wdn_s = b0 + b.dn_s;
  const size_t ch = pol.chain ? 1 : 0;  // chained GEMMs: tile / m-tile prefixes and the act ready flags
  p.sched_c = L.take(ch * sizeof(int32_t) * (n_groups + 1));
  p.mt_base = L.take(ch * sizeof(int32_t) * n_groups);
  p.ready = L.take(ch * sizeof(int32_t) * (Tk / 256 + T / 256 + n_groups + 2));
  p.total = L.off;
  return p;
}

flux_status validate_cfg(const flux_moe_cfg* c) {
  if (!c) return FLUX_E_INVALID;
  if (c->hidden <= 0 || c->ffn <= 0 || c->n_experts <= 0 || c->top_k <= 0 || c->shared_ffn < 0)
    return FLUX_E_INVALID;
  if (c->wbits != 2 && c->wbits != 4 && c->wbits != 8 && c->wbits != 16) return FLUX_E_UNSUPPORTED;
  if (c->wbits == 16 && c->group_size != 0) return FLUX_E_UNSUPPORTED;
  if (c->n_router < 0) return FLUX_E_INVALID;
  if (c->n_router > 0 && (c->n_router > 128 || c->n_experts > c->n_router || c->top_k > c->n_router))
    return FLUX_E_UNSUPPORTED;
  if (c->hidden % 64 || c->ffn % 16 || c->shared_ffn % 16) return FLUX_E_UNSUPPORTED;
  if (c->n_experts > 128 || c->top_k > 8 || (c->n_router == 0 && c->top_k > c->n_experts)) return FLUX_E_UNSUPPORTED;
  if (c->norm_topk != 0 && c->norm_topk != 1) return FLUX_E_INVALID;
  if (c->group_size < 0) return FLUX_E_INVALID;
  if (c->group_size > 0) {
    if (c->group_size % 64 || c->hidden % c->group_size || c->ffn % c->group_size ||
        (c->shared_ffn && c->shared_ffn % c->group_size))
      return FLUX_E_UNSUPPORTED;
  }
  if (c->wbits == 4 && (c->hidden % 32 || c->ffn % 32 || c->shared_ffn % 32)) return FLUX_E_UNSUPPORTED;
  if (c->wbits == 2 && (c->hidden % 64 || c->ffn % 64 || c->shared_ffn % 64)) return FLUX_E_UNSUPPORTED;
  return FLUX_OK;
}

// The dequantization pass of one layer (R1b; launch_dequant) into B-operand buffers.
struct Bops {
  void *gu_r, *dn_r, *gu_s, *dn_s;
};
Bops bops_at(const flux_moe_cfg& c, void* base) {
  const BopsPlan b = bops_plan(c);
  uint8_t* p = (uint8_t*)base;
  return {p + b.gu_r, p + b.dn_r, p + b.gu_s, p + b.dn_s};
}
cudaError_t dequant_layer(const flux_moe_cfg& c, const flux_qlayer* w, const Bops& b, cudaStream_t s) {
  const bool per_channel = c.group_size == 0 && c.wbits != 16;
  const int H = c.hidden, F = c.ffn, Fs = c.shared_ffn, E = c.n_experts;
  const int g_h = per_channel ? H : c.group_size, g_f = per_channel ? F : c.group_size,
            g_fs = per_channel ? Fs : c.group_size;
  const int pc = per_channel ? 1 : 0;
  KernelTimer kt(K_DEQUANT, s);
  cudaError_t e = launch_dequant(c.wbits, (const uint8_t*)w->gate_q, w->gate_s, (const uint8_t*)w->up_q, w->up_s, E, F,
                                 H, pad128(F), 1, g_h, pc, H, b.gu_r, s);
  if (e == cudaSuccess)
    e = launch_dequant(c.wbits, (const uint8_t*)w->down_q, w->down_s, nullptr, nullptr, E, H, F, 0, 0, g_f, pc,
                       pad64(F), b.dn_r, s);
  if (e == cudaSuccess && Fs > 0)
    e = launch_dequant(c.wbits, (const uint8_t*)w->sh_gate_q, w->sh_gate_s, (const uint8_t*)w->sh_up_q, w->sh_up_s, 1,
                       Fs, H, pad128(Fs), 1, g_h, pc, H, b.gu_s, s);
  if (e == cudaSuccess && Fs > 0)
    e = launch_dequant(c.wbits, (const uint8_t*)w->sh_down_q, w->sh_down_s, nullptr, nullptr, 1, H, Fs, 0, 0, g_fs, pc,
                       pad64(Fs), b.dn_s, s);
  return e;
}
// the weight pointers flux_profile_layer requires of a layer
flux_status check_qlayer(const flux_moe_cfg& c, const flux_qlayer* w) {
  const bool quantized = c.wbits != 16;
  if (!w || !w->router_w || !w->gate_q || !w->up_q || !w->down_q ||
      (quantized && (!w->gate_s || !w->up_s || !w->down_s)))
    return FLUX_E_INVALID;
  if (c.shared_ffn > 0 && (!w->sh_gate_q || !w->sh_up_q || !w->sh_down_q ||
                           (quantized && (!w->sh_gate_s || !w->sh_up_s || !w->sh_down_s))))
    return FLUX_E_INVALID;
  if (c.n_router > 0 && !w->remap) return FLUX_E_INVALID;
  const void* ptrs16[] = {w->router_w, w->gate_q, w->up_q, w->down_q, w->sh_gate_q, w->sh_up_q, w->sh_down_q};
  for (const void* p : ptrs16)
    if (p && !aligned16(p)) return FLUX_E_INVALID;
  return FLUX_OK;
}
}  // namespace

}  // namespace flux

using namespace flux;

extern "C" {

const char* flux_status_string(flux_status s) {
  switch (s) {
    case FLUX_OK: return "ok";
    case FLUX_E_INVALID: return "invalid argument";
    case FLUX_E_UNSUPPORTED: return "unsupported shape or dtype";
    case FLUX_E_WORKSPACE: return "workspace too small";
    case FLUX_E_CUDA: return "CUDA error (or no sm_100 device)";
    case FLUX_E_NCCL: return "NCCL error";
  }
  return "unknown status";
}

size_t flux_profile_layer_workspace_ex(const flux_moe_cfg* cfg, const flux_policy* policy, int64_t T) {
  if (validate_cfg(cfg) != FLUX_OK || validate_policy(policy) != FLUX_OK || T < 0) return 0;
  return plan(*cfg, resolve_policy(*cfg, policy, T), T).total;
}

size_t flux_profile_layer_workspace(const flux_moe_cfg* cfg, int64_t T) {
  return flux_profile_layer_workspace_ex(cfg, nullptr, T);
}

flux_status flux_profile_layer(const flux_moe_cfg* cfg, const flux_qlayer* w, const void* x, const void* residual,
                               int64_t T, const flux_layer_out* out, void* ws, size_t ws_bytes, void* stream) {
  return flux_profile_layer_ex(cfg, nullptr, w, x, residual, T, out, ws, ws_bytes, stream);
}

// flux_profile_layer_ex / flux_profile_layer_bops.  bops: this layer's B operands already
// dequantized (used on the dequant-pass path, ignored otherwise).
static flux_status profile_impl(const flux_moe_cfg* cfg, const flux_policy* policy, const flux_qlayer* w,
                                const void* bops, const void* x, const void* residual, int64_t T,
                                const flux_layer_out* out, void* ws, size_t ws_bytes, void* stream) {
  flux_status st = validate_cfg(cfg);
  if (st != FLUX_OK) return st;
  if ((st = validate_policy(policy)) != FLUX_OK) return st;
  if (!w || !out || T < 0) return FLUX_E_INVALID;
  if (bops && !aligned16(bops)) return FLUX_E_INVALID;
  if (T == 0) return FLUX_OK;
  if (T * cfg->top_k >= (int64_t)1 << 31) return FLUX_E_UNSUPPORTED;
  const flux_moe_cfg& c = *cfg;
  const bool sh = c.shared_ffn > 0;
  const bool quantized = c.wbits != 16;
  if (!x || !out->y || !out->topk_ids || !out->topk_w || !out->hist) return FLUX_E_INVALID;
  if ((st = check_qlayer(c, w)) != FLUX_OK) return st;
  const void* ptrs16[] = {x, residual, out->y, ws};
  for (const void* p : ptrs16)
    if (p && !aligned16(p)) return FLUX_E_INVALID;
  const Policy pol = resolve_policy(c, policy, T);
  const bool ext_bops = bops != nullptr && pol.pass;
  const WsPlan P = plan(c, pol, T, ext_bops);
  if (!ws || ws_bytes < P.total) return FLUX_E_WORKSPACE;
  if ((st = check_device()) != FLUX_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* W = (uint8_t*)ws;
  const int H = c.hidden, F = c.ffn, Fs = c.shared_ffn, E = c.n_experts, k = c.top_k;
  const int Fp = pad128(F), Fsp = pad128(Fs);
  const int Fld = pad64(F), Fsld = pad64(Fs);  // row lengths of act / act_sh / the down B operands
  const bool per_channel = c.group_size == 0 && quantized;  // per-channel scales applied in the epilogue
  const int E_r = c.n_router > 0 ? c.n_router : E;           // experts the router scores
  const int g_h = per_channel ? H : c.group_size, g_f = per_channel ? F : c.group_size,
            g_fs = per_channel ? Fs : c.group_size;
  const int64_t n_rt = (T + kRouterTile - 1) / kRouterTile;
  const int64_t Tk = T * k;
  const int n_groups = E + (sh ? 1 : 0);

  int32_t* tile_counts = (int32_t*)(W + P.tile_counts);
  int32_t* tile_base = (int32_t*)(W + P.tile_base);
  int32_t* rank = (int32_t*)(W + P.rank);
  int32_t* offsets = (int32_t*)(W + P.offsets);
  int32_t* token_index = out->token_index ? out->token_index : (int32_t*)(W + P.token_index);
  int32_t* inv_pos = (int32_t*)(W + P.inv_pos);
  const GatherMode gmode = pol.gmode;
  const bool gather_a = gmode != GATHER_NONE;
  void* x_perm = gather_a ? nullptr : W + P.x_perm;
  void* y_perm = W + P.y_perm;
  void* act = W + P.act;
  void* act_sh = W + P.act_sh;
  int32_t* sh_sched = (int32_t*)(W + P.sh_sched);
  const bool fuse_combine = sh && pol.fused_combine;
  void* y_sh = W + P.y_sh;  // shared-MLP output (unused when the combine is fused into its down GEMM)
  const Bops ob = ext_bops ? bops_at(c, const_cast<void*>(bops)) : Bops{W + P.wgu_r, W + P.wdn_r, W + P.wgu_s, W + P.wdn_s};
  void* wgu_r = ob.gu_r;
  void* wdn_r = ob.dn_r;
  void* wgu_s = ob.gu_s;
  void* wdn_s = ob.dn_s;

  // ---- (a) weights -> bf16 B operands (scale folded for grouped quantization)
  cudaError_t e = cudaSuccess;
  const bool pass = pol.pass;
  if (pass && !ext_bops) e = dequant_layer(c, w, ob, s);
  if (e != cudaSuccess) { set_last_error("dequant", e); return FLUX_E_CUDA; }

  // ---- (b) K1 router + top-k + histogram
  const int npad = E_r <= 16 ? 16 : E_r <= 32 ? 32 : E_r <= 64 ? 64 : 128;
  CUtensorMap tm_x, tm_wr;
  if (!tmap_bf16(&tm_x, x, T, H, kRouterTile) || !tmap_bf16(&tm_wr, w->router_w, E_r, H, npad)) { set_last_error("router tensor map", cudaErrorInvalidValue); return FLUX_E_CUDA; }
  RouterArgs ra{T, H, E_r, k, c.norm_topk, out->topk_ids, out->topk_w, out->router_logits, out->hist, tile_counts, rank,
                E, c.n_router > 0 ? w->remap : nullptr, (int32_t*)(W + P.counter)};
  {
    KernelTimer kt(K_ROUTER, s);
    if ((e = launch_router(tm_x, tm_wr, npad, ra, s)) != cudaSuccess) { set_last_error("router", e); return FLUX_E_CUDA; }
  }

  // ---- (c) K2 schedule + scatter/gather (D_e)
  ScheduleArgs sa;
  sa.E = E;
  sa.k = k;
  sa.T = T;
  sa.n_tiles = (int)n_rt;
  sa.tile_counts = tile_counts;
  sa.tile_base = tile_base;
  sa.offsets = offsets;
  sa.user_offsets = out->expert_offsets;
  sa.done_counter = (int32_t*)(W + P.counter);
  sa.has_shared = sh;
  sa.n_tiles_gu = Fp / 128;
  sa.n_tiles_gu_sh = Fsp / 128;
  sa.n_tiles_dn = (H + 255) / 256;
  sa.n_tiles_dn_sh = (H + 255) / 256;
  sa.sched_gu = (int32_t*)(W + P.sched_gu);
  sa.sched_dn = (int32_t*)(W + P.sched_dn);
  sa.grp_row0 = (int32_t*)(W + P.row0);
  sa.grp_rows = (int32_t*)(W + P.rows);
  sa.gemm_bm = 256;  // CTA pairs
  sa.sched_sh = sh ? sh_sched : nullptr;
  sa.sched_c = pol.chain ? (int32_t*)(W + P.sched_c) : nullptr;
  sa.mt_base = pol.chain ? (int32_t*)(W + P.mt_base) : nullptr;
  sa.ready = pol.chain ? (int32_t*)(W + P.ready) : nullptr;
  sa.grp_row0_sh = sh_sched + 2;
  sa.grp_rows_sh = sh_sched + 3;
  {  // indices in one kernel; the routed rows are copied to x_perm only when the GEMM does not gather them
    KernelTimer kt(K_PERMUTE, s);
    if ((e = launch_permute(sa, out->topk_ids, rank, inv_pos, token_index, s)) != cudaSuccess) { set_last_error("permute", e); return FLUX_E_CUDA; }
  }
  if (x_perm) {
    KernelTimer kt(K_SCATTER, s);
    if ((e = launch_scatter(x, T, H, E, k, out->topk_ids, rank, tile_base, offsets, inv_pos, token_index, x_perm,
                            s)) != cudaSuccess) { set_last_error("scatter", e); return FLUX_E_CUDA; }
  }

  // ---- (d) K3 + K5: gate/up grouped GEMM with SwiGLU epilogue (routed + shared in one launch)
  // ---- (e) K4 + K5: down grouped GEMM -> y_perm (aliases x_perm) and y_sh
  GemmArgs ga{};
  ga.n_groups = n_groups;
  ga.E = E;
  ga.sched = sa.sched_gu;
  ga.grp_row0 = sa.grp_row0;
  ga.grp_rows = sa.grp_rows;
  ga.n_tiles_r = sa.n_tiles_gu;
  ga.n_tiles_s = sa.n_tiles_gu_sh;
  ga.K_r = H;
  ga.K_s = H;
  ga.N_r = F;
  ga.N_s = Fs;
  ga.b_rows_r = 2 * Fp;
  ga.cs0_r = per_channel ? w->gate_s : nullptr;
  ga.cs1_r = per_channel ? w->up_s : nullptr;
  ga.cs0_s = per_channel ? w->sh_gate_s : nullptr;
  ga.cs1_s = per_channel ? w->sh_up_s : nullptr;
  ga.out_r = act;
  ga.out_s = act_sh;
  ga.ld_r = Fld;
  ga.ld_s = Fsld;
  ga.rows_r = Tk;
  ga.rows_s = T;
  ga.grid = kNumSMs;
  ga.bm = sa.gemm_bm;
  ga.gather_idx = gather_a ? token_index : nullptr;
  ga.gather_cp = gmode == GATHER_CP ? 1 : 0;
  ga.l2_hints = pol.l2_hints;
  ga.clk_probe = clock_probe(K_GEMM_GU);  // null unless flux_timing_enable(1)
  ga.tile_ctr = pol.dynamic_tiles ? sa.done_counter + 1 : nullptr;  // zeroed by K1
  ga.a_src = x;
  ga.a_ld = H;
  GemmArgs gd = ga;
  gd.gather_idx = nullptr;  // the down GEMM reads act, materialised in permuted order by K3
  gd.gather_cp = 0;
  gd.tile_ctr = ga.tile_ctr ? sa.done_counter + 2 : nullptr;
  gd.clk_probe = clock_probe(K_GEMM_DN);
  gd.sched = sa.sched_dn;
  gd.n_tiles_r = sa.n_tiles_dn;
  gd.n_tiles_s = sa.n_tiles_dn_sh;
  gd.K_r = F;
  gd.K_s = Fs;
  gd.N_r = H;
  gd.N_s = H;
  gd.b_rows_r = H;
  gd.cs0_r = per_channel ? w->down_s : nullptr;
  gd.cs1_r = nullptr;
  gd.cs0_s = per_channel ? w->sh_down_s : nullptr;
  gd.cs1_s = nullptr;
  gd.out_r = y_perm;
  gd.out_s = y_sh;
  gd.ld_r = H;
  gd.ld_s = H;
  if (fuse_combine) gd.n_groups = E;  // routed experts only; the shared MLP's down GEMM carries K6
  const void* resid = residual ? residual : x;
  // the shared MLP's down GEMM alone, epilogue = the layer output (K6 fused): one group, E = 0
  GemmArgs gsc = gd;
  gsc.n_groups = 1;
  gsc.E = 0;
  gsc.sched = sa.sched_sh;
  gsc.grp_row0 = sa.grp_row0_sh;
  gsc.grp_rows = sa.grp_rows_sh;
  gsc.out_s = out->y;
  gsc.resid = resid;
  gsc.y_perm = y_perm;
  gsc.topk_w = out->topk_w;
  gsc.inv_pos = inv_pos;
  gsc.k = k;
  gsc.tile_ctr = ga.tile_ctr ? sa.done_counter + 3 : nullptr;

  CUtensorMap a_r, a_s, b_r, b_s;
  if (pass) {
    const uint32_t bbox = 128;  // B rows per TMA box: half the 256-row tile of a CTA pair
    if (!tmap_a_routed(&a_r, gather_a, x, x_perm, T, Tk, H) || !tmap_bf16(&b_r, wgu_r, (uint64_t)E * 2 * Fp, H, bbox) ||
        (sh && (!tmap_bf16(&a_s, x, T, H, 128) || !tmap_bf16(&b_s, wgu_s, 2ull * Fsp, H, bbox)))) {
      set_last_error("gate/up tensor maps", cudaErrorInvalidValue);
      return FLUX_E_CUDA;
    }
    if (!sh) { a_s = a_r; b_s = b_r; }
    if (pol.chain) {  // K3 + K4 in one persistent launch
      CUtensorMap a_r1, a_s1, b_r1, b_s1;
      if (!tmap_bf16(&a_r1, act, Tk, F, 128, Fld) || !tmap_bf16(&b_r1, wdn_r, (uint64_t)E * H, F, bbox, Fld) ||
          (sh && (!tmap_bf16(&a_s1, act_sh, T, Fs, 128, Fsld) || !tmap_bf16(&b_s1, wdn_s, H, Fs, bbox, Fsld)))) {
        set_last_error("chain tensor maps", cudaErrorInvalidValue);
        return FLUX_E_CUDA;
      }
      if (!sh) { a_s1 = a_r1; b_s1 = b_r1; }
      ChainArgs ca{sa.sched_c, sa.mt_base, sa.ready, 24, sa.done_counter + 1};
      KernelTimer kt(K_GEMM_CHAIN, s);
      if ((e = launch_gemm_chain(a_r, a_s, b_r, b_s, a_r1, a_s1, b_r1, b_s1, ga, gd, ca, s)) != cudaSuccess) {
        set_last_error("gemm_chain", e);
        return FLUX_E_CUDA;
      }
    } else {
    {
      KernelTimer kt(K_GEMM_GU, s);
      if ((e = launch_gemm(EPI_SWIGLU, a_r, a_s, b_r, b_s, ga, s)) != cudaSuccess) { set_last_error("gemm_gate_up", e); return FLUX_E_CUDA; }
    }
    if (!tmap_bf16(&a_r, act, Tk, F, 128, Fld) || !tmap_bf16(&b_r, wdn_r, (uint64_t)E * H, F, bbox, Fld) ||
        (sh && (!tmap_bf16(&a_s, act_sh, T, Fs, 128, Fsld) || !tmap_bf16(&b_s, wdn_s, H, Fs, bbox, Fsld)))) {
      set_last_error("down tensor maps", cudaErrorInvalidValue);
      return FLUX_E_CUDA;
    }
    {
      KernelTimer kt(K_GEMM_DN, s);
      if ((e = launch_gemm(EPI_STORE, a_r, sh ? a_s : a_r, b_r, sh ? b_s : b_r, gd, s)) != cudaSuccess) { set_last_error("gemm_down", e); return FLUX_E_CUDA; }
    }
    if (fuse_combine) {
      KernelTimer kt(K_GEMM_DN_SH_COMBINE, s);
      if ((e = launch_gemm(EPI_COMBINE, a_s, a_s, b_s, b_s, gsc, s)) != cudaSuccess) { set_last_error("gemm_down_shared_combine", e); return FLUX_E_CUDA; }
    }
    }
  } else {
    // fused dequant: B tiles are built on chip from the canonical quantized weights
    const uint32_t qb = c.wbits == 4 ? 32 : 64;       // raw bytes per row per 64-wide K slice
    const uint64_t Hq = c.wbits == 4 ? H / 2 : H, Fq = c.wbits == 4 ? F / 2 : F, Fsq = c.wbits == 4 ? Fs / 2 : Fs;
    CUtensorMap q_r0, q_r1, q_s0, q_s1;
    QGemmArgs qa{};
    qa.wbits = c.wbits;
    qa.gsz = c.group_size;
    // gate/up
    if (!tmap_a_routed(&a_r, gather_a, x, x_perm, T, Tk, H) || !tmap_u8(&q_r0, w->gate_q, (uint64_t)E * F, Hq, qb) ||
        !tmap_u8(&q_r1, w->up_q, (uint64_t)E * F, Hq, qb) ||
        (sh && (!tmap_bf16(&a_s, x, T, H, 128) || !tmap_u8(&q_s0, w->sh_gate_q, Fs, Hq, qb) ||
                !tmap_u8(&q_s1, w->sh_up_q, Fs, Hq, qb)))) {
      set_last_error("gate/up tensor maps", cudaErrorInvalidValue);
      return FLUX_E_CUDA;
    }
    if (!sh) { a_s = a_r; q_s0 = q_r0; q_s1 = q_r1; }
    qa.base = ga;
    qa.gate_up = 1;
    qa.qrows_r = F;
    qa.qrows_s = Fs;
    qa.qtotal_r = (int64_t)E * F;
    qa.qtotal_s = Fs;
    qa.gs_r0 = w->gate_s;
    qa.gs_r1 = w->up_s;
    qa.gs_s0 = w->sh_gate_s;
    qa.gs_s1 = w->sh_up_s;
    {
      KernelTimer kt(K_GEMM_GU, s);
      if ((e = launch_gemm_q(EPI_SWIGLU, a_r, a_s, q_r0, q_r1, q_s0, q_s1, qa, s)) != cudaSuccess) { set_last_error("gemm_gate_up", e); return FLUX_E_CUDA; }
    }
    // down
    if (!tmap_bf16(&a_r, act, Tk, F, 128, Fld) || !tmap_u8(&q_r0, w->down_q, (uint64_t)E * H, Fq, qb) ||
        (sh && (!tmap_bf16(&a_s, act_sh, T, Fs, 128, Fsld) || !tmap_u8(&q_s0, w->sh_down_q, H, Fsq, qb)))) {
      set_last_error("down tensor maps", cudaErrorInvalidValue);
      return FLUX_E_CUDA;
    }
    q_r1 = q_r0;
    q_s1 = q_s0;
    qa.base = gd;
    qa.gate_up = 0;
    qa.qrows_r = H;
    qa.qrows_s = H;
    qa.qtotal_r = (int64_t)E * H;
    qa.qtotal_s = H;
    qa.gs_r0 = qa.gs_r1 = w->down_s;
    qa.gs_s0 = qa.gs_s1 = w->sh_down_s;
    {
      KernelTimer kt(K_GEMM_DN, s);
      if ((e = launch_gemm_q(EPI_STORE, a_r, sh ? a_s : a_r, q_r0, q_r1, sh ? q_s0 : q_r0, sh ? q_s1 : q_r1, qa,
                             s)) != cudaSuccess) { set_last_error("gemm_down", e); return FLUX_E_CUDA; }
    }
    if (fuse_combine) {
      qa.base = gsc;
      KernelTimer kt(K_GEMM_DN_SH_COMBINE, s);
      if ((e = launch_gemm_q(EPI_COMBINE, a_s, a_s, q_s0, q_s1, q_s0, q_s1, qa, s)) != cudaSuccess) { set_last_error("gemm_down_shared_combine", e); return FLUX_E_CUDA; }
    }
  }

  // ---- (f) K6 combine: fused into the shared-MLP down GEMM when there is one, else standalone
  if (!fuse_combine) {
    KernelTimer kt(K_COMBINE, s);
    if ((e = launch_combine(T, H, k, resid, sh ? y_sh : nullptr, y_perm, out->topk_w, inv_pos, out->y, s,
                            c.n_router > 0)) != cudaSuccess) {
      set_last_error("combine", e);
      return FLUX_E_CUDA;
    }
  }
  return FLUX_OK;
}

flux_status flux_profile_layer_ex(const flux_moe_cfg* cfg, const flux_policy* policy, const flux_qlayer* w,
                                  const void* x, const void* residual, int64_t T, const flux_layer_out* out, void* ws,
                                  size_t ws_bytes, void* stream) {
  return profile_impl(cfg, policy, w, nullptr, x, residual, T, out, ws, ws_bytes, stream);
}

flux_status flux_profile_layer_bops(const flux_moe_cfg* cfg, const flux_policy* policy, const flux_qlayer* w,
                                    const void* bops, const void* x, const void* residual, int64_t T,
                                    const flux_layer_out* out, void* ws, size_t ws_bytes, void* stream) {
  return profile_impl(cfg, policy, w, bops, x, residual, T, out, ws, ws_bytes, stream);
}

size_t flux_profile_layer_workspace_bops(const flux_moe_cfg* cfg, const flux_policy* policy, int64_t T) {
  if (validate_cfg(cfg) != FLUX_OK || validate_policy(policy) != FLUX_OK || T < 0) return 0;
  return plan(*cfg, resolve_policy(*cfg, policy, T), T, true).total;
}

int32_t flux_profile_layer_uses_bops(const flux_moe_cfg* cfg, const flux_policy* policy, int64_t T) {
  if (validate_cfg(cfg) != FLUX_OK || validate_policy(policy) != FLUX_OK || T < 0) return -1;
  return resolve_policy(*cfg, policy, T).pass ? 1 : 0;
}

size_t flux_layer_bops_bytes(const flux_moe_cfg* cfg) {
  if (validate_cfg(cfg) != FLUX_OK) return 0;
  return bops_plan(*cfg).total;
}

flux_status flux_dequantize_layer(const flux_moe_cfg* cfg, const flux_qlayer* w, void* bops, void* stream) {
  flux_status st = validate_cfg(cfg);
  if (st != FLUX_OK) return st;
  if ((st = check_qlayer(*cfg, w)) != FLUX_OK) return st;
  if (!bops || !aligned16(bops)) return FLUX_E_INVALID;
  if ((st = check_device()) != FLUX_OK) return st;
  const cudaError_t e = dequant_layer(*cfg, w, bops_at(*cfg, bops), (cudaStream_t)stream);
  if (e != cudaSuccess) set_last_error("dequant", e);
  return cuda_status(e);
}

flux_status flux_quantize_weights(int32_t wbits, int32_t group_size, flux_dtype in_dtype, const void* w, int64_t R,
                                  int64_t K, void* q, float* s, void* stream) {
  if (wbits != 2 && wbits != 4 && wbits != 8) return FLUX_E_UNSUPPORTED;
  if (in_dtype != FLUX_BF16 && in_dtype != FLUX_FP32) return FLUX_E_INVALID;
  if (wbits == 2 && K % 8) return FLUX_E_UNSUPPORTED;
  if (R < 0 || K <= 0 || group_size < 0) return FLUX_E_INVALID;
  const int64_t g = group_size ? group_size : K;
  if (K % g || g % 8 || g > 4096) return FLUX_E_UNSUPPORTED;
  if (R == 0) return FLUX_OK;
  if (!w || !q || !s || !aligned16(w) || !aligned16(q) || (reinterpret_cast<uintptr_t>(s) & 3)) return FLUX_E_INVALID;
  flux_status st = check_device();
  if (st != FLUX_OK) return st;
  KernelTimer kt(K_QUANTIZE, (cudaStream_t)stream);
  return cuda_status(launch_quantize(wbits, g, in_dtype == FLUX_FP32, w, R, K, q, s, (cudaStream_t)stream));
}

flux_status flux_quantize_weights_bops(const flux_moe_cfg* cfg, int32_t family, flux_dtype in_dtype, const void* w,
                                       int32_t n_layers, void* q, float* s, void* bops, size_t bops_stride,
                                       void* stream) {
  flux_status st = validate_cfg(cfg);
  if (st != FLUX_OK) return st;
  const flux_moe_cfg& c = *cfg;
  if (c.wbits == 16) return FLUX_E_UNSUPPORTED;
  if (family < FLUX_FAM_GATE || family > FLUX_FAM_SH_DOWN || n_layers < 0) return FLUX_E_INVALID;
  const bool shared = family >= FLUX_FAM_SH_GATE;
  if (shared && c.shared_ffn == 0) return FLUX_E_INVALID;
  if (in_dtype != FLUX_BF16 && in_dtype != FLUX_FP32) return FLUX_E_INVALID;
  if (!bops || !aligned16(bops) || bops_stride % 16 || bops_stride < bops_plan(c).total) return FLUX_E_INVALID;
  const int H = c.hidden, F = shared ? c.shared_ffn : c.ffn, G = shared ? 1 : c.n_experts;
  const bool down = family == FLUX_FAM_DOWN || family == FLUX_FAM_SH_DOWN;
  const int N = down ? H : F, K = down ? F : H;  // rows and contraction of this family's matrices
  const int64_t rows = (int64_t)G * N;
  const int64_t g = c.group_size ? c.group_size : K;
  if (K % g || g % 8 || g > 4096) return FLUX_E_UNSUPPORTED;  // the quantizer's team shapes (as flux_quantize_weights)
  if (n_layers == 0) return FLUX_OK;
  if (!w || !q || !s || !aligned16(w) || !aligned16(q) || (reinterpret_cast<uintptr_t>(s) & 3)) return FLUX_E_INVALID;
  if ((st = check_device()) != FLUX_OK) return st;
  const BopsPlan b = bops_plan(c);
  BopsOut bo{};
  const size_t off = family == FLUX_FAM_GATE || family == FLUX_FAM_UP ? b.gu_r
                     : family == FLUX_FAM_DOWN                        ? b.dn_r
                     : family == FLUX_FAM_SH_DOWN                     ? b.dn_s
                                                                      : b.gu_s;
  bo.out = (uint8_t*)bops + off;
  bo.layer_stride = (int64_t)bops_stride;
  if (rows * n_layers * (K / g) >= (int64_t)1 << 31) return FLUX_E_UNSUPPORTED;  // 32-bit item arithmetic in the kernel
  bo.ipr = make_fastdiv((uint32_t)(K / g));
  bo.layer_rows = make_fastdiv((uint32_t)rows);
  bo.n = make_fastdiv((uint32_t)N);
  bo.Fp = pad128(F);
  bo.interleave = down ? 0 : 1;
  bo.up = family == FLUX_FAM_UP || family == FLUX_FAM_SH_UP;
  bo.ldo = down ? pad64(F) : H;
  bo.per_channel = c.group_size == 0;
  KernelTimer kt(K_QUANTIZE, (cudaStream_t)stream);
  return cuda_status(
      launch_quantize(c.wbits, g, in_dtype == FLUX_FP32, w, rows * n_layers, K, q, s, (cudaStream_t)stream, &bo));
}

flux_status flux_merge_experts(flux_dtype dtype, int32_t n_experts, int64_t numel, const void* experts,
                               const int32_t* cluster_of, const float* alpha, int32_t n_clusters, void* merged,
                               int32_t* remap, void* stream) {
  if (dtype != FLUX_BF16 && dtype != FLUX_FP32) return FLUX_E_INVALID;
  if (n_experts < 1 || n_experts > 1024 || n_clusters < 1 || n_clusters > n_experts || numel < 0)
    return FLUX_E_INVALID;
  if (numel % 8) return FLUX_E_UNSUPPORTED;
  if (!experts || !cluster_of || !alpha || !merged || !aligned16(experts) || !aligned16(merged)) return FLUX_E_INVALID;
  flux_status st = check_device();
  if (st != FLUX_OK) return st;
  KernelTimer kt(K_MERGE, (cudaStream_t)stream);
  return cuda_status(launch_merge(dtype == FLUX_FP32, n_experts, numel, experts, cluster_of, alpha, n_clusters, merged,
                                  remap, (cudaStream_t)stream));
}

flux_status flux_merge_experts_batch(flux_dtype dtype, int32_t n_experts, int64_t numel, int32_t n_jobs,
                                     const flux_merge_job* jobs, int32_t compact, void* stream) {
  if (dtype != FLUX_BF16 && dtype != FLUX_FP32) return FLUX_E_INVALID;
  if (n_experts < 1 || n_experts > 1024 || numel < 0 || n_jobs < 0 || n_jobs > FLUX_MERGE_MAX_JOBS ||
      (compact != 0 && compact != 1))
    return FLUX_E_INVALID;
  if (numel % 8) return FLUX_E_UNSUPPORTED;
  if (n_jobs == 0) return FLUX_OK;
  if (!jobs) return FLUX_E_INVALID;
  MergeBatch b{};
  b.n_jobs = n_jobs;
  b.E = n_experts;
  b.numel = numel;
  b.compact = compact;
  for (int j = 0; j < n_jobs; ++j) {
    const flux_merge_job& J = jobs[j];
    if (!J.experts || !J.cluster_of || !J.alpha || !J.out || !aligned16(J.experts) || !aligned16(J.out))
      return FLUX_E_INVALID;
    if (J.n_clusters < (compact ? 0 : 1) || J.n_clusters > n_experts) return FLUX_E_INVALID;
    if (compact && (J.n_tuning < 0 || J.n_tuning + J.n_clusters > n_experts || J.n_tuning + J.n_clusters < 1))
      return FLUX_E_INVALID;
    b.jobs[j] = MergeJob{J.experts, J.cluster_of, J.alpha, J.out, J.remap, J.n_clusters,
                         compact ? J.n_tuning + J.n_clusters : 0};
  }
  flux_status st = check_device();
  if (st != FLUX_OK) return st;
  KernelTimer kt(K_MERGE, (cudaStream_t)stream);
  cudaError_t e = launch_merge_batch(dtype == FLUX_FP32, b, (cudaStream_t)stream);
  if (e != cudaSuccess) set_last_error("merge_batch", e);
  return cuda_status(e);
}

/* ---------------------------------------------------------------- NEXT-2: compact model + output error */
flux_status flux_compact_experts(flux_dtype dtype, int32_t n_experts, int64_t numel, const void* experts,
                                 const int32_t* cluster_of, const float* alpha, int32_t n_clusters, void* compact,
                                 int32_t* remap, void* stream) {
  if (dtype != FLUX_BF16 && dtype != FLUX_FP32) return FLUX_E_INVALID;
  if (n_experts < 1 || n_experts > 1024 || n_clusters < 0 || n_clusters > n_experts || numel < 0)
    return FLUX_E_INVALID;
  if (numel % 8) return FLUX_E_UNSUPPORTED;
  if (!experts || !cluster_of || !alpha || !compact || !aligned16(experts) || !aligned16(compact))
    return FLUX_E_INVALID;
  flux_status st = check_device();
  if (st != FLUX_OK) return st;
  KernelTimer kt(K_MERGE, (cudaStream_t)stream);
  return cuda_status(launch_merge(dtype == FLUX_FP32, n_experts, numel, experts, cluster_of, alpha, n_clusters,
                                  compact, remap, (cudaStream_t)stream, 1));
}

flux_status flux_attention_hist(int64_t T, int32_t top_k, int32_t n_experts, const int32_t* ids, const float* attn,
                                int64_t* attn_hist, void* stream) {
  if (T < 0 || top_k < 1 || top_k > 8 || n_experts < 1 || n_experts > 1024) return FLUX_E_INVALID;
  if (T == 0) return FLUX_OK;
  if (!ids || !attn || !attn_hist) return FLUX_E_INVALID;
  flux_status st = check_device();
  if (st != FLUX_OK) return st;
  KernelTimer kt(K_ATTN_HIST, (cudaStream_t)stream);
  cudaError_t e = launch_attention_hist(T, top_k, n_experts, ids, attn, attn_hist, (cudaStream_t)stream);
  if (e != cudaSuccess) set_last_error("attention_hist", e);
  return cuda_status(e);
}

flux_status flux_frequencies(int64_t n, const int64_t* counts, double denom, float* alpha, void* stream) {
  if (n < 0 || !(denom > 0.0)) return FLUX_E_INVALID;
  if (n == 0) return FLUX_OK;
  if (!counts || !alpha) return FLUX_E_INVALID;
  flux_status st = check_device();
  if (st != FLUX_OK) return st;
  KernelTimer kt(K_FREQ, (cudaStream_t)stream);
  cudaError_t e = launch_frequencies(n, counts, denom, alpha, (cudaStream_t)stream);
  if (e != cudaSuccess) set_last_error("frequencies", e);
  return cuda_status(e);
}

size_t flux_output_error_workspace(void) { return cosine_workspace(); }

flux_status flux_output_error(int64_t T, int32_t hidden, const void* a, const void* b, double* result, void* ws,
                              size_t ws_bytes, void* stream) {
  if (T < 0 || hidden <= 0 || hidden % 8) return FLUX_E_INVALID;
  if (!a || !b || !result || !ws || !aligned16(a) || !aligned16(b) || !aligned16(ws)) return FLUX_E_INVALID;
  if (ws_bytes < cosine_workspace()) return FLUX_E_WORKSPACE;
  flux_status st = check_device();
  if (st != FLUX_OK) return st;
  KernelTimer kt(K_COSINE, (cudaStream_t)stream);
  cudaError_t e = launch_cosine_distance(T, hidden, a, b, (double*)ws, result, (cudaStream_t)stream);
  if (e != cudaSuccess) set_last_error("cosine_distance", e);
  return cuda_status(e);
}

/* ---------------------------------------------------------------- NEXT-1: expert clustering (§5.2) */
size_t flux_expert_features_workspace(int32_t n_layers, int32_t n_experts, int32_t n_fam, const int64_t* fam_numel) {
  if (n_layers < 1 || n_experts < 2 || n_experts > kClusterMaxE || n_fam < 1 || n_fam > kClusterMaxFam || !fam_numel)
    return 0;
  for (int f = 0; f < n_fam; ++f)
    if (fam_numel[f] < 1) return 0;
  return features_workspace(n_layers, n_experts, n_fam, fam_numel);
}

flux_status flux_expert_features(int32_t n_layers, int32_t n_experts, int32_t n_fam, const void* const* fam,
                                 const int64_t* fam_numel, int32_t d, float* features, float* gram,
                                 float* eigvals, void* ws, size_t ws_bytes, void* stream) {
  const int L = n_layers, E = n_experts;
  if (L < 1 || n_fam < 1 || n_fam > kClusterMaxFam || E < 2 || E > kClusterMaxE || d < 1 || d > E ||
      d > kClusterMaxD)
    return FLUX_E_INVALID;
  if (!fam || !fam_numel || !features || !ws) return FLUX_E_INVALID;
  for (int f = 0; f < n_fam; ++f)
    if (fam_numel[f] < 1 || fam_numel[f] % 8) return FLUX_E_UNSUPPORTED;
  if (ws_bytes < features_workspace(L, E, n_fam, fam_numel) || !aligned16(ws)) return FLUX_E_INVALID;
  for (int i = 0; i < L * n_fam; ++i)
    if (!fam[i] || !aligned16(fam[i])) return FLUX_E_INVALID;
  flux_status st = check_device();
  if (st != FLUX_OK) return st;
  cudaStream_t s = (cudaStream_t)stream;
  float* partial = reinterpret_cast<float*>(ws);
  float* G = features_gram_slot(ws, E, n_fam, fam_numel, 0);
  int* counter = features_counter(ws, L, E, n_fam, fam_numel);
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(int), s);
  if (e != cudaSuccess) return FLUX_E_CUDA;
  for (int l = 0; l < L; ++l) {
    int slots = 0;
    {
      KernelTimer kt(K_GRAM, s);
      e = launch_gram(E, n_fam, fam + (size_t)l * n_fam, fam_numel, partial, counter, &slots, s);
      if (e != cudaSuccess) {
        set_last_error("gram", e);
        return FLUX_E_CUDA;
      }
    }
    KernelTimer kt(K_GRAM_REDUCE, s);
    e = launch_gram_reduce(E, partial, slots, G + (size_t)l * E * E,
                           gram ? gram + (size_t)l * E * E : nullptr, counter, s);
    if (e != cudaSuccess) {
      set_last_error("gram_reduce", e);
      return FLUX_E_CUDA;
    }
  }
  KernelTimer kt(K_EIG, s);
  e = launch_eig(L, E, d, G, features, eigvals, s);
  if (e != cudaSuccess) set_last_error("eig", e);
  return cuda_status(e);
}

flux_status flux_cluster_experts(int32_t n_layers, int32_t n_experts, int32_t d, const float* features,
                                 const int64_t* counts, const int32_t* n_clusters, const uint8_t* tuning,
                                 int32_t max_iter, int32_t* cluster_of, int32_t* iterations, void* stream) {
  const int L = n_layers, E = n_experts;
  if (L < 1 || L > kClusterMaxL || E < 1 || E > kClusterMaxE || d < 1 || d > kClusterMaxD || max_iter < 1)
    return FLUX_E_INVALID;
  if (!features || !counts || !n_clusters || !cluster_of) return FLUX_E_INVALID;
  KMeansArgs ka;
  for (int l = 0; l < L; ++l) {
    uint64_t m[2] = {0, 0};
    int n_non = E;
    if (tuning)
      for (int e = 0; e < E; ++e)
        if (tuning[l * E + e]) {
          m[e >> 6] |= 1ull << (e & 63);
          --n_non;
        }
    if (n_clusters[l] < 1 || n_clusters[l] > n_non) return FLUX_E_INVALID;
    ka.n_clusters[l] = n_clusters[l];
    ka.tuning[l][0] = m[0];
    ka.tuning[l][1] = m[1];
  }
  flux_status st = check_device();
  if (st != FLUX_OK) return st;
  KernelTimer kt(K_KMEANS, (cudaStream_t)stream);
  cudaError_t e = launch_kmeans(L, E, d, features, counts, ka, max_iter, cluster_of, iterations, (cudaStream_t)stream);
  if (e != cudaSuccess) set_last_error("kmeans", e);
  return cuda_status(e);
}

}  // extern "C"
