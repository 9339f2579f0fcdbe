// gemm_common.cuh — pieces shared by the grouped expert GEMMs (K3/K4/K5):
// parameters, tile decoding and the epilogues (SwiGLU / store) that turn one
// 128-row x 256-column fp32 TMEM accumulator slice into bf16 rows.
#pragma once
#include "internal.h"
#include "ptx.cuh"

namespace flux {
namespace gemm {

constexpr int kBN = 256, kBK = 64;
constexpr int kMaxGroups = 257;

struct Params {
  int n_groups, E;
  const int32_t* sched;     // [n_groups+1] tile prefix
  const int32_t* grp_row0;  // [n_groups]
  const int32_t* grp_rows;  // [n_groups]
  int n_tiles_r, n_tiles_s;
  int K_r, K_s;
  int N_r, N_s;
  int b_rows_r;                                // B rows per routed group in the B tensor
  const float *cs0_r, *cs1_r, *cs0_s, *cs1_s;  // per-channel scales [group][N] or null
  void *out_r, *out_s;
  int64_t ld_r, ld_s;
  // EPI_COMBINE (shared-MLP down GEMM only): y = bf16(resid + bf16(acc) + Σ_j w_j · y_perm[inv_pos_j])
  const __nv_bfloat16* resid;
  const __nv_bfloat16* y_perm;
  const float* topk_w;
  const int32_t* inv_pos;
  int k;
  // routed A rows gathered from x by token id (TMA tile::gather4) instead of a materialised x_perm
  const int32_t* gather_idx;  // token_index [T*k] or null
  int gather_cp;               // 1: gather with cp.async (CTA-pair pass kernel) instead of TMA gather4
  const __nv_bfloat16* a_src;  // gather source rows (x) and their stride in elements
  int a_ld;
  int l2_hints;                // GemmArgs::l2_hints
  int32_t* tile_ctr;           // GemmArgs::tile_ctr
  unsigned long long* clk_probe;  // GemmArgs::clk_probe
};

struct TileInfo {
  int g, m, n;
};

__device__ __forceinline__ TileInfo decode(int tile, const int32_t* s_sched, int n_groups, int nt_r, int nt_s, int E) {
  int lo = 0, hi = n_groups - 1;  // largest g with sched[g] <= tile
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_sched[mid] <= tile) lo = mid;
    else hi = mid - 1;
  }
  const int nt = lo < E ? nt_r : nt_s;
  const int local = tile - s_sched[lo];
  return {lo, local / nt, local % nt};
}

// Output columns one MMA of tile ti must produce (CTA-pair kernels).  The last n-tile of a group
// whose width is not a multiple of the tile issues only its valid columns: for gate/up the pair's
// B halves hold gate features [0, f) (CTA 0) and up features [0, f) (CTA 1) of the tile, so an
// N = 2f MMA reads the first f rows of each half and leaves gate in accumulator columns [0, f) and
// up in [f, 2f) (e.g. F = 688: the sixth tile runs N = 96 instead of 256).  N % 16 == 0 and
// F % 16 == 0 (validate_cfg) keep every N a legal M=256 MMA width.
template <int EPI>
__device__ __forceinline__ int pair_tile_cols(const Params& p, const TileInfo& ti) {
  const int N = ti.g < p.E ? p.N_r : p.N_s;
  if constexpr (EPI == EPI_SWIGLU) return 2 * min(kBN / 2, N - ti.n * (kBN / 2));
  else return min(kBN, N - ti.n * kBN);
}
// K=16 MMAs of K slice kb (the last slice of a K that is not a multiple of 64 is partly empty)
__device__ __forceinline__ int slice_k16(int K, int kb) { return min(kBK / 16, (K - kb * kBK) / 16); }

// Per-channel scales (INT8/INT4/INT2 with group_size 0, reading R1b: the fp32 scale multiplies the
// accumulator) of one tile, staged once per tile in shared memory by the 128 epilogue threads
// instead of one dependent global load per 16 columns per thread (those loads serialised ~16 L2
// round trips into every tile's epilogue: 34% tensor-pipe activity on the LLaMA-shape down GEMM).
// Layout per tile: [0, 256) = cs0 of the tile's local columns (STORE) or gate features (SWIGLU),
// [256, 384) = cs1 of the up features; two buffers alternate by tile parity (a buffer is rewritten
// two tiles later, after every epilogue thread passed the next tile's barrier).
constexpr int kScaleFloats = 512;
constexpr int kScaleSmemBytes = 2 * kScaleFloats * 4;
template <int EPI>
__device__ __forceinline__ const float* stage_tile_scales(const Params& p, const TileInfo& ti, float* s_scales,
                                                          uint32_t tc, int et /* epilogue thread 0..127 */) {
  const bool routed = ti.g < p.E;
  const float* cs0 = routed ? p.cs0_r : p.cs0_s;
  if (!cs0) return nullptr;  // uniform per launch (grouped scales are folded into the B operand)
  const float* cs1 = routed ? p.cs1_r : p.cs1_s;
  const int N = routed ? p.N_r : p.N_s;
  const int64_t base = routed ? (int64_t)ti.g * N : 0;
  float* sc = s_scales + (tc & 1) * kScaleFloats;
  if constexpr (EPI == EPI_SWIGLU) {
    const int f = ti.n * (kBN / 2) + et;  // 128 threads: one gate and one up feature each
    sc[et] = f < N ? __ldg(&cs0[base + f]) : 0.f;
    sc[256 + et] = f < N ? __ldg(&cs1[base + f]) : 0.f;
  } else {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int c = ti.n * kBN + et + 128 * i;
      sc[et + 128 * i] = c < N ? __ldg(&cs0[base + c]) : 0.f;
    }
  }
  named_bar_sync(2, 128);
  return sc;
}
__device__ __forceinline__ void lds16(const float* sc, float (&v)[16]) {
  const float4* q = reinterpret_cast<const float4*>(sc);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 t = q[i];
    v[4 * i] = t.x;
    v[4 * i + 1] = t.y;
    v[4 * i + 2] = t.z;
    v[4 * i + 3] = t.w;
  }
}

// SiLU(v) = v / (1 + e^-v) with the SFU exp and the fast reciprocal-divide: ~2 ulp fp32 (far below
// the bf16 rounding of a that follows), and ~5x fewer issue slots than expf + IEEE division, which
// matters because the epilogue shares the SM's issue bandwidth with the next tile's producers.
// For v << 0, e^-v = inf and __fdividef(v, inf) = 0 = SiLU's limit.
__device__ __forceinline__ float silu(float v) { return __fdividef(v, 1.0f + __expf(-v)); }

// Epilogue of one accumulator slice: this thread owns TMEM lane (row) `taddr`'s lane, i.e. output
// row `orow` (valid = inside the group).  EPI_SWIGLU: columns [0,128) = gate, [128,256) = up of
// features n*128 + j; EPI_STORE: columns = output features n*256 + j.
template <int EPI>
__device__ __forceinline__ void epilogue_slice(const Params& p, uint32_t taddr, const TileInfo& ti, bool valid,
                                               int64_t orow, int up_col, const float* sc) {
  const bool routed = ti.g < p.E;
  const int N = routed ? p.N_r : p.N_s;
  const int64_t ld = routed ? p.ld_r : p.ld_s;
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(routed ? p.out_r : p.out_s) + orow * ld;
  if constexpr (EPI == EPI_SWIGLU) {
    // gate in accumulator columns [0, up_col), up in [up_col, 2·up_col) (pair_tile_cols)
    for (int j = 0; j < kBN / 2; j += 16) {
      const int f0 = ti.n * (kBN / 2) + j;
      if (j >= up_col || f0 >= N) break;  // warp-uniform (N % 16 == 0)
      float gv[16], uv[16];
      tmem_ld16(taddr + j, gv);
      tmem_ld16(taddr + up_col + j, uv);
      tmem_ld_wait();
      if (sc) {
        float gs[16], us[16];
        lds16(sc + j, gs);
        lds16(sc + 256 + j, us);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          gv[i] *= gs[i];
          uv[i] *= us[i];
        }
      }
      uint32_t pk[8];
#pragma unroll
      for (int i = 0; i < 16; i += 2) pk[i / 2] = pack_bf16x2(silu(gv[i]) * uv[i], silu(gv[i + 1]) * uv[i + 1]);
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(out + f0);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
  } else if constexpr (EPI == EPI_COMBINE) {
    // The layer output for token row `orow` (K6 fused here, reading R6): identical order and
    // roundings to combine.cu — acc = r; acc += bf16(sh); acc = fma(w_j, o_j, acc) for j = 0..k-1.
    int pos[8];
    float wt[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      pos[jj] = 0;
      wt[jj] = 0.f;
      if (valid && jj < p.k) {
        pos[jj] = __ldg(&p.inv_pos[orow * p.k + jj]);
        wt[jj] = __ldg(&p.topk_w[orow * p.k + jj]);
      }
    }
    const int H = N;
    for (int j = 0; j < kBN; j += 16) {
      const int c0 = ti.n * kBN + j;
      float v[16];
      tmem_ld16(taddr + j, v);
      tmem_ld_wait();
      if (c0 >= N || !valid) continue;
      // issue every load of this 16-column chunk before using any of them
      uint4 rr[2], oo[8][2];
      const uint4* rp = reinterpret_cast<const uint4*>(p.resid + orow * H + c0);
      rr[0] = __ldg(rp);
      rr[1] = __ldg(rp + 1);
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
        if (jj < p.k && pos[jj] >= 0) {  // pos -1: a pick folded by gate re-routing (NEXT-2)
          const uint4* op = reinterpret_cast<const uint4*>(p.y_perm + (int64_t)pos[jj] * H + c0);
          oo[jj][0] = __ldg(op);
          oo[jj][1] = __ldg(op + 1);
        }
      float acc[16];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&rr[h]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(b[i]);
          acc[8 * h + 2 * i] = f.x;
          acc[8 * h + 2 * i + 1] = f.y;
        }
      }
      if (sc) {  // per-channel scale of the shared MLP's down projection (reading R1b)
        float cs[16];
        lds16(sc + j, cs);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] *= cs[i];
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] += __bfloat162float(__float2bfloat16_rn(v[i]));  // o_sh = bf16(a·ŵ)
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
        if (jj < p.k && pos[jj] >= 0) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&oo[jj][h]);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 f = __bfloat1622float2(b[i]);
              acc[8 * h + 2 * i] = fmaf(wt[jj], f.x, acc[8 * h + 2 * i]);
              acc[8 * h + 2 * i + 1] = fmaf(wt[jj], f.y, acc[8 * h + 2 * i + 1]);
            }
          }
        }
      uint4* dst = reinterpret_cast<uint4*>(out + c0);
      dst[0] = make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]), pack_bf16x2(acc[4], acc[5]),
                          pack_bf16x2(acc[6], acc[7]));
      dst[1] = make_uint4(pack_bf16x2(acc[8], acc[9]), pack_bf16x2(acc[10], acc[11]),
                          pack_bf16x2(acc[12], acc[13]), pack_bf16x2(acc[14], acc[15]));
    }
  } else {
    for (int j = 0; j < kBN; j += 16) {
      const int c0 = ti.n * kBN + j;
      float v[16];
      tmem_ld16(taddr + j, v);
      tmem_ld_wait();
      if (c0 >= N) continue;
      if (sc) {
        float cs[16];
        lds16(sc + j, cs);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] *= cs[i];
      }
      uint32_t pk[8];
#pragma unroll
      for (int i = 0; i < 16; i += 2) pk[i / 2] = pack_bf16x2(v[i], v[i + 1]);
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(out + c0);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// A operand producer of the CTA-pair kernels, run by all 32 lanes of the producer warp.
// Per tile: if rows come from a gather (routed groups with gather_idx), the warp stages the 128
// token ids of this CTA's rows in shared memory (rows past the group end read token 0; they are
// masked in the epilogue).  Per K slice, lane 0 issues one 128-row box, or 32 tile::gather4.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void stage_gather_rows(int32_t* s_idx, const Params& p, int row0, int rows_in_grp,
                                                  int first_local_row) {
  const int lane = (int)lane_id();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int r = lane * 4 + j, rl = first_local_row + r;
    s_idx[r] = rl < rows_in_grp ? __ldg(&p.gather_idx[row0 + rl]) : 0;
  }
  __syncwarp();
}
// Called by all 32 lanes of the producer warp: lane 0 issues the plain 128-row box; for gathers
// every lane issues one tile::gather4 (rows 4·lane .. 4·lane+3), i.e. one warp-wide instruction.
__device__ __forceinline__ void load_a_pair(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int kb, int arow,
                                            bool gather, const int32_t* s_idx) {
  const int lane = (int)lane_id();
  if (!gather) {
    if (lane == 0) tma_load_2d_pair(dst, map, bar, kb * kBK, arow);
    return;
  }
  const int4 r = *reinterpret_cast<const int4*>(s_idx + 4 * lane);
  tma_gather4_pair(dst + lane * 512, map, bar, kb * kBK, r.x, r.y, r.z, r.w);
}

// ---------------------------------------------------------------------------
// In-register weight dequantization (reading R1b): exact codes, one rounding.
// ---------------------------------------------------------------------------
// 8 INT4 codes (one 32-bit word, even k in the low nibble) -> 8 bf16 in k order.
template <bool GROUPED>
__device__ __forceinline__ uint4 deq_int4x8(uint32_t w, __nv_bfloat162 s2) {
  const uint32_t x = w ^ 0x88888888u;  // two's complement -> offset binary (q + 8)
  uint32_t p[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) p[i] = ((x >> (4 * i)) & 0x000F000Fu) | 0x43004300u;  // bf16 {136+q_i, 136+q_{i+4}}
  const __nv_bfloat162 off = __floats2bfloat162_rn(136.0f, 136.0f);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&p[i]);
    v = __hsub2(v, off);               // exact q
    if (GROUPED) v = __hmul2(v, s2);   // bf16(q * bf16(s)): exact product, one rounding
    p[i] = *reinterpret_cast<uint32_t*>(&v);
  }
  uint4 o;
  o.x = __byte_perm(p[0], p[1], 0x5410);  // (k0, k1)
  o.y = __byte_perm(p[2], p[3], 0x5410);  // (k2, k3)
  o.z = __byte_perm(p[0], p[1], 0x7632);  // (k4, k5)
  o.w = __byte_perm(p[2], p[3], 0x7632);  // (k6, k7)
  return o;
}

// 8 INT2 codes (16 bits, element k in bits 2k) -> 8 bf16 (16 bytes), same scheme as INT4: offset
// binary q + 2 in the mantissa of bf16 128, minus 130 exactly.
template <bool GROUPED>
__device__ __forceinline__ uint4 deq_int2x8(uint32_t w16, __nv_bfloat162 s2) {
  const uint32_t x = (w16 ^ 0xAAAAu) & 0xFFFFu;          // two's complement -> offset binary (q + 2)
  const uint32_t x2 = (x & 0xFFu) | ((x & 0xFF00u) << 8);  // codes 0-3 in bits 0-7, codes 4-7 in bits 16-23
  uint32_t p[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) p[i] = ((x2 >> (2 * i)) & 0x00030003u) | 0x43004300u;  // bf16 {130+q_i, 130+q_{i+4}}
  const __nv_bfloat162 off = __floats2bfloat162_rn(130.0f, 130.0f);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&p[i]);
    v = __hsub2(v, off);               // exact q
    if (GROUPED) v = __hmul2(v, s2);   // bf16(q * bf16(s)): exact product, one rounding
    p[i] = *reinterpret_cast<uint32_t*>(&v);
  }
  uint4 o;
  o.x = __byte_perm(p[0], p[1], 0x5410);
  o.y = __byte_perm(p[2], p[3], 0x5410);
  o.z = __byte_perm(p[0], p[1], 0x7632);
  o.w = __byte_perm(p[2], p[3], 0x7632);
  return o;
}

// 4 INT8 codes (one word, k order) -> 2 bf16x2 words; q exact via the fp32 2^23 magic.
template <bool GROUPED>
__device__ __forceinline__ uint2 deq_int8x4(uint32_t w, float s) {
  const uint32_t x = w ^ 0x80808080u;
  float f[4];
  f[0] = __uint_as_float(__byte_perm(x, 0x4B000000u, 0x7650)) - 8388736.0f;
  f[1] = __uint_as_float(__byte_perm(x, 0x4B000000u, 0x7651)) - 8388736.0f;
  f[2] = __uint_as_float(__byte_perm(x, 0x4B000000u, 0x7652)) - 8388736.0f;
  f[3] = __uint_as_float(__byte_perm(x, 0x4B000000u, 0x7653)) - 8388736.0f;
  if (GROUPED) {
#pragma unroll
    for (int i = 0; i < 4; ++i) f[i] *= s;  // q·bf16(s) exact in fp32 (8 x 8 bits)
  }
  return make_uint2(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]));
}

inline Params make_params(const GemmArgs& g) {
  Params p;
  p.n_groups = g.n_groups;
  p.E = g.E;
  p.sched = g.sched;
  p.grp_row0 = g.grp_row0;
  p.grp_rows = g.grp_rows;
  p.n_tiles_r = g.n_tiles_r;
  p.n_tiles_s = g.n_tiles_s;
  p.K_r = g.K_r;
  p.K_s = g.K_s;
  p.N_r = g.N_r;
  p.N_s = g.N_s;
  p.b_rows_r = g.b_rows_r;
  p.cs0_r = g.cs0_r;
  p.cs1_r = g.cs1_r;
  p.cs0_s = g.cs0_s;
  p.cs1_s = g.cs1_s;
  p.out_r = g.out_r;
  p.out_s = g.out_s;
  p.ld_r = g.ld_r;
  p.ld_s = g.ld_s;
  p.resid = reinterpret_cast<const __nv_bfloat16*>(g.resid);
  p.y_perm = reinterpret_cast<const __nv_bfloat16*>(g.y_perm);
  p.topk_w = g.topk_w;
  p.inv_pos = g.inv_pos;
  p.k = g.k;
  p.gather_idx = g.gather_idx;
  p.gather_cp = g.gather_cp;
  p.a_src = reinterpret_cast<const __nv_bfloat16*>(g.a_src);
  p.a_ld = g.a_ld;
  p.clk_probe = g.clk_probe;
  p.l2_hints = g.l2_hints;
  p.tile_ctr = g.tile_ctr;
  return p;
}

}  // namespace gemm
}  // namespace flux
