// combine.cu — K6: the MoE layer output (reading R6):
//   y_t = bf16( r_t + sh_t + Σ_j w_tj · o_{t,S_tj} )
// gather-based (inv_pos from K2), fp32 accumulation in the fixed order
// residual, shared, j = 0..k-1, one rounding.  One warp per token, 16-byte
// vectors; every byte is read or written exactly once.
#include "internal.h"
#include "ptx.cuh"

namespace flux {
namespace {

__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 p = __bfloat1622float2(h[i]);
    f[2 * i] = p.x;
    f[2 * i + 1] = p.y;
  }
}

// EMPTY: picks may be empty (pos -1, folded by gate re-routing, NEXT-2).  The plain path keeps
// every load unconditional so all (k + 2) x U loads issue before any is used.  U = 16-byte chunks per
// lane per iteration: 2, or 4 when a token has few source rows (k <= 4 and k + residual + shared <= 6,
// e.g. the LLaMA shape's k = 4 without shared experts), so a warp keeps about the same bytes in flight;
// KMAX sizes the per-pick arrays (registers).
template <bool EMPTY, int U, int KMAX>
__global__ void __launch_bounds__(256) combine_kernel(int64_t T, int H, int k, const uint4* __restrict__ residual,
                                                      const uint4* __restrict__ y_sh, const uint4* __restrict__ y_perm,
                                                      const float* __restrict__ w, const int32_t* __restrict__ inv_pos,
                                                      uint4* __restrict__ y) {
  const int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= T) return;
  const int lane = threadIdx.x & 31;
  const int nvec = H / 8;
  int pos[KMAX];
  float wt[KMAX];
#pragma unroll
  for (int j = 0; j < KMAX; ++j) {
    pos[j] = 0;
    wt[j] = 0.f;
    if (j < k) {
      pos[j] = __ldg(&inv_pos[t * k + j]);
      wt[j] = __ldg(&w[t * k + j]);
    }
  }
  // U 16-byte chunks per lane per iteration: all loads are issued before any is used
  for (int c0 = lane; c0 < nvec; c0 += 32 * U) {
    uint4 rv[U], sv[U], ov[KMAX][U];
    bool has[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + 32 * u;
      has[u] = c < nvec;
      if (!has[u]) continue;
      rv[u] = __ldg(&residual[t * nvec + c]);
      if (y_sh) sv[u] = __ldg(&y_sh[t * nvec + c]);
#pragma unroll
      for (int j = 0; j < KMAX; ++j)
        if (j < k && (!EMPTY || pos[j] >= 0)) ov[j][u] = __ldcs(&y_perm[(int64_t)pos[j] * nvec + c]);  // streaming
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!has[u]) continue;
      float acc[8], f[8];
      unpack8(rv[u], acc);
      if (y_sh) {
        unpack8(sv[u], f);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += f[i];
      }
#pragma unroll
      for (int j = 0; j < KMAX; ++j) {
        if (j < k && (!EMPTY || pos[j] >= 0)) {  // pos -1: a pick folded by gate re-routing
          unpack8(ov[j][u], f);
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = fmaf(wt[j], f[i], acc[i]);
        }
      }
      uint4 o;
      o.x = pack_bf16x2(acc[0], acc[1]);
      o.y = pack_bf16x2(acc[2], acc[3]);
      o.z = pack_bf16x2(acc[4], acc[5]);
      o.w = pack_bf16x2(acc[6], acc[7]);
      y[t * nvec + c0 + 32 * u] = o;
    }
  }
}
}  // namespace

cudaError_t launch_combine(int64_t T, int H, int k, const void* residual, const void* y_sh, const void* y_perm,
                           const float* w, const int32_t* inv_pos, void* y, cudaStream_t st, bool empty_picks) {
  if (T == 0) return cudaSuccess;
  const unsigned grid = (unsigned)((T + 7) / 8);
  const bool wide = k <= 4 && k + 1 + (y_sh ? 1 : 0) <= 6;
  auto kern = empty_picks ? (wide ? combine_kernel<true, 4, 4> : combine_kernel<true, 2, 8>)
                          : (wide ? combine_kernel<false, 4, 4> : combine_kernel<false, 2, 8>);
  kern<<<grid, 256, 0, st>>>(T, H, k, (const uint4*)residual, (const uint4*)y_sh, (const uint4*)y_perm, w, inv_pos,
                             (uint4*)y);
  return cudaGetLastError();
}

}  // namespace flux
