// dequant.cu — the dequantization pass of the expert GEMMs (DESIGN.md §5.1 "Where the bf16 B operand
// comes from"): the quantized weights of one layer (reading R1/R1b) become the bf16 B
// operands the CTA-pair GEMMs stream with TMA, once per layer, when every B tile is reused by many
// m-tiles (262,144 tokens: ~96 m-tiles per expert).  HBM-bound: read 0.5 B (INT4) + write 2 B per weight.
#include "internal.h"
#include "ptx.cuh"
#include "gemm_common.cuh"

namespace flux {
namespace {
using namespace gemm;
// ---------------------------------------------------------------------------
// Dequantization of one weight family into the bf16 B operand layout.
//   interleave == 1 (gate/up): out[g][2*Fp][K], rows [256n, 256n+128) = gate
//     features [128n, 128n+128), rows [256n+128, 256n+256) = up features; rows
//     of features >= F are zero.
//   interleave == 0: out[g][N][K] = the family as stored.
//   value = bf16(q) when per_channel (the scale is applied in the GEMM
//   epilogue, exact), else bf16(q · s[group]).
// ---------------------------------------------------------------------------
template <int WBITS>
__global__ void __launch_bounds__(256) dequant_kernel(const uint8_t* __restrict__ q0, const float* __restrict__ s0,
                                                      const uint8_t* __restrict__ q1, const float* __restrict__ s1,
                                                      int G, int N, int K, int Fp, int interleave, int gsz,
                                                      int per_channel, int ldo, uint4* __restrict__ out) {
  // one warp per output row; lanes walk the row in 8-element (16-byte) vectors
  const int64_t rows_out = interleave ? 2LL * Fp : N;
  const int64_t n_rows = (int64_t)G * rows_out;
  const int lane = threadIdx.x & 31;
  const int vec_per_row = K / 8;
  const int64_t wid0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t orow = wid0; orow < n_rows; orow += nw) {
    const int g = (int)(orow / rows_out);
    const int r = (int)(orow - (int64_t)g * rows_out);
    const uint8_t* q = q0;
    const float* s = s0;
    int src_row = r;
    if (interleave) {
      const int blk = r >> 8, w = r & 255;
      src_row = blk * 128 + (w & 127);
      if (w >= 128) { q = q1; s = s1; }
    }
    uint4* dst = out + orow * (ldo / 8);  // output rows padded to ldo elements (128-B aligned rows)
    if (src_row >= N) {  // padding rows of the interleaved layout
      for (int v = lane; v < vec_per_row; v += 32) dst[v] = make_uint4(0, 0, 0, 0);
      continue;
    }
    const int64_t srow = (int64_t)g * N + src_row;
    if constexpr (WBITS == 16) {  // bf16 weights (compact model, NEXT-2): layout copy only
      const uint4* src = reinterpret_cast<const uint4*>(q) + srow * vec_per_row;
      for (int v0 = lane; v0 < vec_per_row; v0 += 128) {
        uint4 r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (v0 + 32 * u < vec_per_row) r[u] = __ldg(&src[v0 + 32 * u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (v0 + 32 * u < vec_per_row) dst[v0 + 32 * u] = r[u];
      }
      continue;
    }
    const float* srow_s = s + (per_channel ? 0 : srow * (K / gsz));
    const int vec_per_grp = per_channel ? vec_per_row : gsz / 8;
    // four output vectors per lane per iteration: all raw loads in flight before converting
    for (int v0 = lane; v0 < vec_per_row; v0 += 128) {
      uint32_t r4[4];
      uint2 r8[4];
      uint32_t r2[4];
      float sc[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int v = v0 + 32 * u;
        if (v >= vec_per_row) continue;
        sc[u] = per_channel ? 0.f : __ldg(&srow_s[v / vec_per_grp]);
        if (WBITS == 2) r2[u] = __ldg(reinterpret_cast<const uint16_t*>(q + srow * (K / 4)) + v);
        else if (WBITS == 4) r4[u] = __ldg(reinterpret_cast<const uint32_t*>(q + srow * (K / 2)) + v);
        else r8[u] = __ldg(reinterpret_cast<const uint2*>(q + srow * K) + v);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int v = v0 + 32 * u;
        if (v >= vec_per_row) continue;
        const float s = __bfloat162float(__float2bfloat16_rn(sc[u]));
        if (WBITS == 2) {
          dst[v] = per_channel ? deq_int2x8<false>(r2[u], __floats2bfloat162_rn(0.f, 0.f))
                               : deq_int2x8<true>(r2[u], __floats2bfloat162_rn(s, s));
        } else if (WBITS == 4) {
          dst[v] = per_channel ? deq_int4x8<false>(r4[u], __floats2bfloat162_rn(0.f, 0.f))
                               : deq_int4x8<true>(r4[u], __floats2bfloat162_rn(s, s));
        } else {
          const uint2 a = per_channel ? deq_int8x4<false>(r8[u].x, 0.f) : deq_int8x4<true>(r8[u].x, s);
          const uint2 b = per_channel ? deq_int8x4<false>(r8[u].y, 0.f) : deq_int8x4<true>(r8[u].y, s);
          dst[v] = make_uint4(a.x, a.y, b.x, b.y);
        }
      }
    }
  }
}
}  // namespace

cudaError_t launch_dequant(int wbits, const uint8_t* q0, const float* s0, const uint8_t* q1, const float* s1, int G,
                           int N, int K, int Fp, int interleave, int gsz, int per_channel, int ldo, void* out,
                           cudaStream_t st) {
  const int64_t rows_out = interleave ? 2LL * Fp : N;
  const int64_t n_rows = (int64_t)G * rows_out;
  if (n_rows == 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<int64_t>((n_rows + 7) / 8, (int64_t)kNumSMs * 16);
  if (wbits == 16)
    dequant_kernel<16><<<grid, 256, 0, st>>>(q0, s0, q1, s1, G, N, K, Fp, interleave, gsz, per_channel, ldo, (uint4*)out);
  else if (wbits == 8)
    dequant_kernel<8><<<grid, 256, 0, st>>>(q0, s0, q1, s1, G, N, K, Fp, interleave, gsz, per_channel, ldo, (uint4*)out);
  else if (wbits == 2)
    dequant_kernel<2><<<grid, 256, 0, st>>>(q0, s0, q1, s1, G, N, K, Fp, interleave, gsz, per_channel, ldo, (uint4*)out);
  else
    dequant_kernel<4><<<grid, 256, 0, st>>>(q0, s0, q1, s1, G, N, K, Fp, interleave, gsz, per_channel, ldo, (uint4*)out);
  return cudaGetLastError();
}

}  // namespace flux
