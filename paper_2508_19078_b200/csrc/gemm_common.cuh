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

__device__ __forceinline__ float silu(float v) { return v / (1.0f + expf(-v)); }

// Epilogue of one accumulator slice: this thread owns TMEM lane (row) `taddr`'s lane, i.e. output
// row `orow` (valid = inside the group).  EPI_SWIGLU: columns [0,128) = gate, [128,256) = up of
// features n*128 + j; EPI_STORE: columns = output features n*256 + j.
template <int EPI>
__device__ __forceinline__ void epilogue_slice(const Params& p, uint32_t taddr, const TileInfo& ti, bool valid,
                                               int64_t orow) {
  const bool routed = ti.g < p.E;
  const int N = routed ? p.N_r : p.N_s;
  const int64_t ld = routed ? p.ld_r : p.ld_s;
  __nv_bfloat16* out = reinterpret_cast<__nv_bfloat16*>(routed ? p.out_r : p.out_s) + orow * ld;
  const float* cs0 = routed ? p.cs0_r : p.cs0_s;
  const float* cs1 = routed ? p.cs1_r : p.cs1_s;
  const int64_t cs_base = routed ? (int64_t)ti.g * N : 0;
  if constexpr (EPI == EPI_SWIGLU) {
    for (int j = 0; j < kBN / 2; j += 16) {
      const int f0 = ti.n * (kBN / 2) + j;
      float gv[16], uv[16];
      tmem_ld16(taddr + j, gv);
      tmem_ld16(taddr + kBN / 2 + j, uv);
      tmem_ld_wait();
      if (f0 >= N) continue;  // warp-uniform (N % 16 == 0)
      uint32_t pk[8];
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        float g0 = gv[i], g1 = gv[i + 1], u0 = uv[i], u1 = uv[i + 1];
        if (cs0) {
          g0 *= __ldg(&cs0[cs_base + f0 + i]);
          g1 *= __ldg(&cs0[cs_base + f0 + i + 1]);
          u0 *= __ldg(&cs1[cs_base + f0 + i]);
          u1 *= __ldg(&cs1[cs_base + f0 + i + 1]);
        }
        pk[i / 2] = pack_bf16x2(silu(g0) * u0, silu(g1) * u1);
      }
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(out + f0);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
  } else {
    for (int j = 0; j < kBN; j += 16) {
      const int c0 = ti.n * kBN + j;
      float v[16];
      tmem_ld16(taddr + j, v);
      tmem_ld_wait();
      if (c0 >= N) continue;
      uint32_t pk[8];
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        float a0 = v[i], a1 = v[i + 1];
        if (cs0) {
          a0 *= __ldg(&cs0[cs_base + c0 + i]);
          a1 *= __ldg(&cs0[cs_base + c0 + i + 1]);
        }
        pk[i / 2] = pack_bf16x2(a0, a1);
      }
      if (valid) {
        uint4* dst = reinterpret_cast<uint4*>(out + c0);
        dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
      }
    }
  }
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
  return p;
}

}  // namespace gemm
}  // namespace flux
