// quantize.cu — K0: the participant's low-bit copy of the model (P:556-565,
// "quantize and profile the latest MoE model ... in each round" P:613-615),
// bit level chosen per participant.  Reading R1: symmetric, per
// row, groups of g along K:
//   s = fl32(max|w| / qmax),  q = clamp(RNE(fl32(w / s)), -qmax-1, qmax),  s == 0 -> q = 0
// IEEE division (__fdiv_rn) and round-to-nearest-even conversion, so the
// result is bit-identical to any correct implementation of that definition.
// INT4 output is packed two per byte, even k in the low nibble; INT2 (NEXT-3) four per byte.
//
// HBM-bound: a team of lanes owns one (row, group); every lane loads 16 B
// vectors of the group once into registers, the team max-reduces with
// shuffles, then each lane writes its 4 (INT4) or 8 (INT8) output bytes.
#include "internal.h"
#include "ptx.cuh"

namespace flux {
namespace {

template <bool F32IN>
__device__ __forceinline__ void load8(const void* w, int64_t elem, float (&f)[8]) {
  if constexpr (F32IN) {
    const float4* p = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(w) + elem);
    float4 a = __ldg(p), b = __ldg(p + 1);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  } else {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(w) + elem));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 p = __bfloat1622float2(h[i]);
      f[2 * i] = p.x;
      f[2 * i + 1] = p.y;
    }
  }
}

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// TS lanes per (row, group), CPL 8-element chunks per lane.
template <int WBITS, bool F32IN, int TS, int CPL>
__global__ void __launch_bounds__(256) quantize_kernel(const void* __restrict__ w, int64_t R, int64_t K, int64_t g,
                                                       uint8_t* __restrict__ q, float* __restrict__ s) {
  constexpr int qmax = (1 << (WBITS - 1)) - 1;
  const int64_t G = K / g;
  const int64_t n_items = R * G;
  const int nchunks = (int)(g / 8);
  const int lane_t = threadIdx.x % TS;
  const int64_t team0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / TS;
  const int64_t nteams = ((int64_t)gridDim.x * blockDim.x) / TS;
  // (row, grp) advanced incrementally: no 64-bit division per item
  int64_t row = team0 / G, grp = team0 - row * G;
  const int64_t drow = nteams / G, dgrp = nteams - drow * G;
  // Items are consecutive (row, group) pairs, i.e. consecutive g-element slices of w: a warp's
  // teams read one contiguous span per iteration.  Lane 0 prefetches the span kAhead iterations
  // ahead into L2, which keeps ~4x more HBM bytes in flight than the registers alone can (80
  // registers/thread cap residency at 24 warps/SM, each holding one 2 KB span).
  constexpr int kAhead = 4;
  const uint32_t span_bytes = (uint32_t)((32 / TS) * g * (F32IN ? 4 : 2));
  const int64_t warp_item0 = team0 - (threadIdx.x % 32) / TS;
  for (int64_t item = team0; item < n_items; item += nteams) {
    const int64_t base = row * K + grp * g;
    if ((threadIdx.x & 31) == 0) {
      const int64_t pf = warp_item0 + (item - team0) + kAhead * nteams;  // first item of the span
      if (pf + 32 / TS <= n_items)
        bulk_prefetch_l2(reinterpret_cast<const uint8_t*>(w) + pf * g * (F32IN ? 4 : 2), span_bytes);
    }
    float v[CPL][8];
    float amax = 0.f;
    // chunk i of this lane is c = lane_t + i*TS: a team reads TS consecutive 16-byte vectors per load
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int c = lane_t + i * TS;
      if (c < nchunks) {
        load8<F32IN>(w, base + c * 8, v[i]);
#pragma unroll
        for (int j = 0; j < 8; ++j) amax = fmaxf(amax, fabsf(v[i][j]));
      }
    }
#pragma unroll
    for (int o = TS / 2; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o, TS));
    const float sc = __fdiv_rn(amax, (float)qmax);
    if (lane_t == 0) s[item] = sc;
    const float rcp = __frcp_rn(sc);
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int c = lane_t + i * TS;
      if (c >= nchunks) continue;
      // RNE(fl32(w/s)) without a division or a float->int conversion on the common path (the
      // conversion pipe runs at a quarter of the FMA rate and bounded the previous version):
      //   t = fma(w, fl32(1/s), 1.5·2^23) rounds the exact product w·fl32(1/s) to an integer, and
      //   the low byte of t's bit pattern is that integer in two's complement (|q| <= 127);
      //   d = fma(w, fl32(1/s), -(t - 1.5·2^23)) is the product's distance to it.
      // w·fl32(1/s) differs from fl32(w/s) by < 2^-16 (|quotient| <= 127.5, two 2^-24 relative
      // errors), so both round to the same integer unless |d| >= 1/2 - 2^-14; those (rare) chunks
      // redo the IEEE division per element.  |fl32(w/s)| <= qmax·(1 + 2^-23) < qmax + 1/2 (s is
      // max|w|/qmax rounded), so the fast path never needs the clamp.  s == 0 (1/s = inf) and
      // non-finite inputs (d = NaN, kept by the NaN-propagating max) take the slow path.
      constexpr float kMagic = 12582912.0f;  // 1.5·2^23
      uint32_t tb[8];
      float dmax = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float t = fmaf(v[i][j], rcp, kMagic);
        const float d = fmaf(v[i][j], rcp, kMagic - t);
        dmax = fmax_nan(dmax, fabsf(d));
        tb[j] = __float_as_uint(t);
      }
      if (!(dmax < 0.5f - 6.103515625e-05f) || !(rcp < INFINITY)) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int qi = sc == 0.f ? 0 : max(-qmax - 1, min(qmax, __float2int_rn(__fdiv_rn(v[i][j], sc))));
          tb[j] = (uint32_t)qi;  // only the low byte is used below
        }
      }
      // gather the low bytes: bl = codes 0-3, bh = codes 4-7 (one byte each, two's complement)
      const uint32_t bl = __byte_perm(__byte_perm(tb[0], tb[1], 0x0040), __byte_perm(tb[2], tb[3], 0x0040), 0x5410);
      const uint32_t bh = __byte_perm(__byte_perm(tb[4], tb[5], 0x0040), __byte_perm(tb[6], tb[7], 0x0040), 0x5410);
      if constexpr (WBITS == 2) {  // four codes per byte, element k in bits 2(k mod 4)
        uint32_t o = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) o |= (tb[j] & 0x3u) << (2 * j);
        *reinterpret_cast<uint16_t*>(q + (base + c * 8) / 4) = (uint16_t)o;
      } else if constexpr (WBITS == 8) {
        *reinterpret_cast<uint2*>(q + base + c * 8) = make_uint2(bl, bh);
      } else {
        // byte i of (b >> 4) carries byte i+1's low nibble in its high nibble: one bitwise mux
        // per word puts codes (0,1) in byte 0 and (2,3) in byte 2; a final permute packs them
        const uint32_t xl = (bl & 0x0F0F0F0Fu) | ((bl >> 4) & 0xF0F0F0F0u);
        const uint32_t xh = (bh & 0x0F0F0F0Fu) | ((bh >> 4) & 0xF0F0F0F0u);
        *reinterpret_cast<uint32_t*>(q + (base + c * 8) / 2) = __byte_perm(xl, xh, 0x6420);
      }
    }
    row += drow;
    grp += dgrp;
    if (grp >= G) {
      grp -= G;
      ++row;
    }
  }
}

template <int WBITS, bool F32IN>
cudaError_t dispatch(int64_t g, const void* w, int64_t R, int64_t K, void* q, float* s, cudaStream_t st) {
  const int64_t nch = g / 8;
  const int64_t items = R * (K / g);
  auto grid_for = [&](int ts) {
    int64_t teams_per_block = 256 / ts;
    int64_t b = (items + teams_per_block - 1) / teams_per_block;
    return (unsigned)std::min<int64_t>(b, (int64_t)kNumSMs * 16);
  };
  uint8_t* qq = (uint8_t*)q;
#define QLAUNCH(TS, CPL) \
  quantize_kernel<WBITS, F32IN, TS, CPL><<<grid_for(TS), 256, 0, st>>>(w, R, K, g, qq, s)
  // several 16-byte chunks per lane: enough loads in flight per warp to cover HBM latency
  // (measured on B200 for g = 128: teams of 16/8/4/2/1 lanes -> 0.36/0.43/0.44/0.34/0.18 of HBM peak)
  if (nch == 8) QLAUNCH(4, 2);
  else if (nch == 16) QLAUNCH(4, 4);
  else if (nch == 32) QLAUNCH(8, 4);
  else if (nch <= 32) QLAUNCH(32, 1);
  else if (nch <= 64) QLAUNCH(32, 2);
  else if (nch <= 128) QLAUNCH(32, 4);
  else if (nch <= 256) QLAUNCH(32, 8);
  else if (nch <= 512) QLAUNCH(32, 16);
  else return cudaErrorInvalidValue;
#undef QLAUNCH
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_quantize(int wbits, int64_t g, bool in_fp32, const void* w, int64_t R, int64_t K, void* q, float* s,
                            cudaStream_t st) {
  if (R == 0) return cudaSuccess;
  if (wbits == 8)
    return in_fp32 ? dispatch<8, true>(g, w, R, K, q, s, st) : dispatch<8, false>(g, w, R, K, q, s, st);
  if (wbits == 2)
    return in_fp32 ? dispatch<2, true>(g, w, R, K, q, s, st) : dispatch<2, false>(g, w, R, K, q, s, st);
  return in_fp32 ? dispatch<4, true>(g, w, R, K, q, s, st) : dispatch<4, false>(g, w, R, K, q, s, st);
}

}  // namespace flux
