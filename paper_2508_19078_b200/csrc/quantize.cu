// quantize.cu — K0: the participant's low-bit copy of the model (P:556-565,
// "quantize and profile the latest MoE model ... in each round" P:613-615),
// bit level chosen per participant.  Reading R1: symmetric, per
// row, groups of g along K:
//   s = fl32(max|w| / qmax),  q = clamp(RNE(fl32(w / s)), -qmax-1, qmax),  s == 0 -> q = 0
// IEEE division (__fdiv_rn) and round-to-nearest-even conversion, so the
// result is bit-identical to any correct implementation of that definition.
// INT4 output is packed two per byte, even k in the low nibble; INT2 (NEXT-3) four per byte.
//
// HBM-bound: a team of TS lanes owns one (row, group) = one g-element slice of w (items are
// consecutive slices, item i starts at element i·g); every lane holds CPL 16-byte chunks of it in
// registers, the team max-reduces with shuffles, then each lane writes its packed codes.  The
// common path computes fl32(w/s) exactly with three FMA-pipe operations per element pair (packed
// f32x2; no division, no float->int conversion, no branch).
#include "internal.h"
#include "ptx.cuh"
#include "gemm_common.cuh"

namespace flux {
namespace {

template <bool F32IN>
struct Chunk {  // 8 consecutive input elements as loaded (bf16: one uint4, fp32: two float4)
  uint4 a, b;
};

template <bool F32IN>
__device__ __forceinline__ Chunk<F32IN> load_chunk(const void* w, int64_t elem) {
  Chunk<F32IN> c;
  if constexpr (F32IN) {
    const uint4* p = reinterpret_cast<const uint4*>(reinterpret_cast<const float*>(w) + elem);
    c.a = __ldg(p);
    c.b = __ldg(p + 1);
  } else {
    c.a = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(w) + elem));
  }
  return c;
}

template <bool F32IN>
__device__ __forceinline__ float elem(const Chunk<F32IN>& c, int j) {  // j is a compile-time index
  if constexpr (F32IN) {
    const uint32_t u = j < 4 ? (&c.a.x)[j] : (&c.b.x)[j - 4];
    return __uint_as_float(u);
  } else {
    const uint32_t u = (&c.a.x)[j >> 1];
    return __uint_as_float((j & 1) ? (u & 0xFFFF0000u) : (u << 16));  // bf16 -> fp32 is exact
  }
}

template <int WBITS>
__device__ __forceinline__ uint2 store_codes(uint8_t* q, int64_t e0, const uint32_t (&tb)[8]) {
  // tb[j]'s low byte = code j in two's complement; e0 = index of the chunk's first element.
  // Returns the packed codes as stored (INT2: 16 bits in .x; INT4: .x; INT8: .x, .y).
  if constexpr (WBITS == 2) {  // four codes per byte, element k in bits 2(k mod 4)
    uint32_t o = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) o |= (tb[j] & 0x3u) << (2 * j);
    *reinterpret_cast<uint16_t*>(q + e0 / 4) = (uint16_t)o;
    return make_uint2(o & 0xFFFFu, 0u);
  } else {
    // gather the low bytes: bl = codes 0-3, bh = codes 4-7
    const uint32_t bl = __byte_perm(__byte_perm(tb[0], tb[1], 0x0040), __byte_perm(tb[2], tb[3], 0x0040), 0x5410);
    const uint32_t bh = __byte_perm(__byte_perm(tb[4], tb[5], 0x0040), __byte_perm(tb[6], tb[7], 0x0040), 0x5410);
    if constexpr (WBITS == 8) {
      *reinterpret_cast<uint2*>(q + e0) = make_uint2(bl, bh);
      return make_uint2(bl, bh);
    } else {
      // byte i of (b >> 4) carries byte i+1's low nibble in its high nibble: one bitwise mux per
      // word puts codes (0,1) in byte 0 and (2,3) in byte 2; a final permute packs the four bytes
      const uint32_t xl = (bl & 0x0F0F0F0Fu) | ((bl >> 4) & 0xF0F0F0F0u);
      const uint32_t xh = (bh & 0x0F0F0F0Fu) | ((bh >> 4) & 0xF0F0F0F0u);
      const uint32_t o = __byte_perm(xl, xh, 0x6420);
      *reinterpret_cast<uint32_t*>(q + e0 / 2) = o;
      return make_uint2(o, 0u);
    }
  }
}

// The fused dequantization output (BopsOut): the packed codes just stored, converted by the dequant
// pass's own functions (gemm_common.cuh) with the same scale rounding, so the bytes equal
// launch_dequant's.  bops_row: the output row of quantization group `item` (once per item: three
// multiply-shift divisions) and the group's first 16-byte vector in it.
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
  return (__umulhi(n, f.m) + n) >> f.l;
}
__device__ __forceinline__ uint4* bops_row(const BopsOut& bo, int64_t item, int g) {
  const uint32_t it = (uint32_t)item;
  const uint32_t row = fdiv(it, bo.ipr);
  const uint32_t gi = it - row * bo.ipr.d;
  const uint32_t layer = fdiv(row, bo.layer_rows);
  const uint32_t gr = row - layer * bo.layer_rows.d;
  int64_t orow = gr;
  if (bo.interleave) {
    const uint32_t ge = fdiv(gr, bo.n);
    const uint32_t f = gr - ge * bo.n.d;
    orow = (int64_t)ge * 2 * bo.Fp + (f >> 7) * 256 + bo.up * 128 + (f & 127);
  }
  return reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(bo.out) + (int64_t)layer * bo.layer_stride) +
         orow * (bo.ldo / 8) + gi * (uint32_t)(g / 8);
}
template <int WBITS>
__device__ __forceinline__ void store_bops(const BopsOut& bo, uint4* dst, uint2 packed, float sc) {
  const float sb = __bfloat162float(__float2bfloat16_rn(sc));
  const __nv_bfloat162 s2 = __floats2bfloat162_rn(bo.per_channel ? 0.f : sb, bo.per_channel ? 0.f : sb);
  if constexpr (WBITS == 2) {
    *dst = bo.per_channel ? gemm::deq_int2x8<false>(packed.x, s2) : gemm::deq_int2x8<true>(packed.x, s2);
  } else if constexpr (WBITS == 4) {
    *dst = bo.per_channel ? gemm::deq_int4x8<false>(packed.x, s2) : gemm::deq_int4x8<true>(packed.x, s2);
  } else {
    const uint2 a = bo.per_channel ? gemm::deq_int8x4<false>(packed.x, 0.f) : gemm::deq_int8x4<true>(packed.x, sb);
    const uint2 b = bo.per_channel ? gemm::deq_int8x4<false>(packed.y, 0.f) : gemm::deq_int8x4<true>(packed.y, sb);
    *dst = make_uint4(a.x, a.y, b.x, b.y);
  }
}

// The definition itself, per element (IEEE division, RNE conversion, clamp): groups with a zero,
// tiny or non-finite scale.  Out of line so the common path keeps its registers.
template <int WBITS, bool F32IN, bool BOPS>
__device__ __noinline__ void quantize_chunk_exact(const void* w, int64_t e0, float sc, uint8_t* q, const BopsOut& bo,
                                                  uint4* dst) {
  constexpr int qmax = (1 << (WBITS - 1)) - 1;
  const Chunk<F32IN> c = load_chunk<F32IN>(w, e0);
  uint32_t tb[8];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    tb[j] = sc == 0.f ? 0u : (uint32_t)max(-qmax - 1, min(qmax, __float2int_rn(__fdiv_rn(elem(c, j), sc))));
  const uint2 packed = store_codes<WBITS>(q, e0, tb);
  if constexpr (BOPS) store_bops<WBITS>(bo, dst, packed, sc);
}

// TS lanes per item, CPL chunks of 8 elements per lane; GUARD: the item has fewer than TS·CPL
// chunks (nch, runtime), else exactly TS·CPL.
template <int WBITS, bool F32IN, int TS, int CPL, bool GUARD, bool BOPS>
__global__ void __launch_bounds__(256) quantize_kernel(const void* __restrict__ w, int64_t n_items, int g, int nch,
                                                       uint8_t* __restrict__ q, float* __restrict__ s,
                                                       const __grid_constant__ BopsOut bo) {
  constexpr int qmax = (1 << (WBITS - 1)) - 1;
  constexpr int kEsize = F32IN ? 4 : 2;
  const int lane_t = threadIdx.x % TS;
  const int64_t team0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / TS;
  const int64_t nteams = ((int64_t)gridDim.x * blockDim.x) / TS;
  // A warp's teams read one contiguous span per iteration; lane 0 prefetches the span kAhead
  // iterations ahead into L2 (HBM bytes in flight without holding registers).
  constexpr int kAhead = 4;
  const uint32_t span_bytes = (uint32_t)((32 / TS) * g * kEsize);
  const int64_t warp_item0 = team0 - (threadIdx.x % 32) / TS;
  for (int64_t item = team0; item < n_items; item += nteams) {
    const int64_t base = item * g;
    uint4* brow = nullptr;  // fused output: this group's first 16-byte vector
    if constexpr (BOPS) brow = bops_row(bo, item, g);
    if ((threadIdx.x & 31) == 0) {
      const int64_t pf = warp_item0 + (item - team0) + kAhead * nteams;
      if (pf + 32 / TS <= n_items) bulk_prefetch_l2(reinterpret_cast<const uint8_t*>(w) + pf * g * kEsize, span_bytes);
    }
    // chunk i of this lane is c = lane_t + i·TS: a team reads TS consecutive 16-byte vectors per load
    Chunk<F32IN> ch[CPL];
#pragma unroll
    for (int i = 0; i < CPL; ++i)
      if (!GUARD || lane_t + i * TS < nch) ch[i] = load_chunk<F32IN>(w, base + (lane_t + i * TS) * 8);
    float amax = 0.f;
#pragma unroll
    for (int i = 0; i < CPL; ++i)
      if (!GUARD || lane_t + i * TS < nch) {
#pragma unroll
        for (int j = 0; j < 8; ++j) amax = fmaxf(amax, fabsf(elem(ch[i], j)));
      }
#pragma unroll
    for (int o = TS / 2; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o, TS));
    const float sc = __fdiv_rn(amax, (float)qmax);
    if (lane_t == 0) s[item] = sc;
    const float rcp = __frcp_rn(sc);
    // RNE(fl32(w/s)) without a division per element and without a float->int conversion (the
    // conversion pipe runs at a quarter of the FMA rate):
    //   q0 = fl32(w·y), y = fl32(1/s) (correctly rounded, __frcp_rn); r = w - q0·s (exact, FMA);
    //   q1 = fl32(q0 + r·y) = fl32(w/s) exactly (Markstein's correction theorem: y correctly
    //   rounded and q0 within one ulp of w/s give the correctly rounded quotient; pinned for every
    //   bf16 (w, s) pair by tests/test_gpu_parity.py::test_quantizer_exhaustive_bf16);
    //   t = fl32(q1 + 1.5·2^23) rounds q1 to an integer, ties to even, and the low byte of t's bit
    //   pattern is that integer in two's complement.
    // |fl32(w/s)| <= qmax·(1 + 2^-23) < qmax + 1/2 (s is max|w|/qmax rounded), so no clamp is
    // needed.  Groups whose scale is 0, tiny (r could underflow) or non-finite take the definition
    // itself (IEEE division per element), a branch uniform per team.
    constexpr float kMagic = 12582912.0f;  // 1.5·2^23
    const bool fast = sc >= 0x1p-90f && sc <= 0x1p100f;
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int c = lane_t + i * TS;
      if (GUARD && c >= nch) continue;
      if (!fast) {
        quantize_chunk_exact<WBITS, F32IN, BOPS>(w, base + c * 8, sc, q, bo, brow + c);
        continue;
      }
      uint32_t tb[8];
      // two elements per packed op: q0 = w·y, r = q0·(−s) + w (= −q0·s + w exactly), q1 = r·y + q0,
      // t = q1 + 1.5·2^23 — the same per-lane roundings as the scalar sequence
      const float2 y2 = make_float2(rcp, rcp), ns2 = make_float2(-sc, -sc), m2 = make_float2(kMagic, kMagic);
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const float2 x = make_float2(elem(ch[i], j), elem(ch[i], j + 1));
        const float2 q0 = mul2_rn(x, y2);
        const float2 r = fma2_rn(q0, ns2, x);
        const float2 q1 = fma2_rn(r, y2, q0);
        const float2 t = add2_rn(q1, m2);
        tb[j] = __float_as_uint(t.x);
        tb[j + 1] = __float_as_uint(t.y);
      }
      const uint2 packed = store_codes<WBITS>(q, base + c * 8, tb);
      if constexpr (BOPS) store_bops<WBITS>(bo, brow + c, packed, sc);
    }
  }
}

template <int WBITS, bool F32IN, bool BOPS>
cudaError_t dispatch(int64_t g, const void* w, int64_t R, int64_t K, void* q, float* s, cudaStream_t st,
                     const BopsOut& bo) {
  const int nch = (int)(g / 8);
  const int64_t items = R * (K / g);
  auto grid_for = [&](int ts) {
    int64_t teams_per_block = 256 / ts;
    int64_t b = (items + teams_per_block - 1) / teams_per_block;
    return (unsigned)std::min<int64_t>(b, (int64_t)kNumSMs * 16);
  };
  uint8_t* qq = (uint8_t*)q;
#define QLAUNCH(TS, CPL, GUARD) \
  quantize_kernel<WBITS, F32IN, TS, CPL, GUARD, BOPS><<<grid_for(TS), 256, 0, st>>>(w, items, (int)g, nch, qq, s, bo)
  // exact team shapes for the common group sizes (g = 64, 128, 256 and per-channel K = 2048/4096),
  // guarded whole-warp teams for the rest
  if (nch == 8) QLAUNCH(4, 2, false);
  else if (nch == 16) QLAUNCH(4, 4, false);
  else if (nch == 32) QLAUNCH(8, 4, false);
  else if (nch == 256) QLAUNCH(32, 8, false);
  else if (nch == 512) QLAUNCH(32, 16, false);
  else if (nch <= 32) QLAUNCH(32, 1, true);
  else if (nch <= 64) QLAUNCH(32, 2, true);
  else if (nch <= 128) QLAUNCH(32, 4, true);
  else if (nch <= 256) QLAUNCH(32, 8, true);
  else if (nch <= 512) QLAUNCH(32, 16, true);
  else return cudaErrorInvalidValue;
#undef QLAUNCH
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_quantize(int wbits, int64_t g, bool in_fp32, const void* w, int64_t R, int64_t K, void* q, float* s,
                            cudaStream_t st, const BopsOut* bo) {
  if (R == 0) return cudaSuccess;
  BopsOut none{};
  const BopsOut& b = bo ? *bo : none;
#define QDISPATCH(WB, F32)                                                          \
  (bo && bo->out ? dispatch<WB, F32, true>(g, w, R, K, q, s, st, b) : dispatch<WB, F32, false>(g, w, R, K, q, s, st, b))
  if (wbits == 8) return in_fp32 ? QDISPATCH(8, true) : QDISPATCH(8, false);
  if (wbits == 2) return in_fp32 ? QDISPATCH(2, true) : QDISPATCH(2, false);
  return in_fp32 ? QDISPATCH(4, true) : QDISPATCH(4, false);
#undef QDISPATCH
}

}  // namespace flux
