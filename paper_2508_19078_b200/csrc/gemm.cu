// gemm.cu — K3/K4/K5: the expert FFNs of the quantized MoE model
// as grouped GEMMs on the 5th-generation tensor cores.
//
//   gate/up (EPI_SWIGLU):  act[r][f] = bf16( SiLU(x_r·ŵg_fᵀ) · (x_r·ŵu_fᵀ) )     (R4)
//   down    (EPI_STORE):   o[r][h]   = bf16( act_r·ŵd_hᵀ )
// Groups 0..E-1 are the routed experts (A rows = the expert's D_e segment of
// x_perm / act, K2), group E the shared MLP (A rows = every token, R5), all in
// ONE persistent launch per GEMM.  Tile = 128 rows x 256 output columns x 64-K
// slices; for gate/up the 256 B-rows of a tile are 128 gate rows followed by
// the 128 matching up rows, so one accumulator holds g and u of the same
// (row, feature) and SwiGLU is applied in the epilogue.
//
// Warp roles (256 threads, 1 CTA/SM, grid = #SMs, static round-robin tiles):
//   warp 0: TMA producer — A and B 64-wide K slices, 128-byte swizzle, 4-stage ring
//   warp 1: MMA issuer   — tcgen05.mma M=128 N=256 K=16, fp32 accumulator in TMEM
//   warp 2: TMEM allocator (512 columns = 2 accumulator stages)
//   warps 4-7: epilogue  — tcgen05.ld, per-channel scale (INT8), SwiGLU, bf16 store
// The accumulator is double-buffered so the epilogue of tile i overlaps the
// MMAs of tile i+1.  Tile shape and K order never depend on the number of
// tokens, so every output row is computed identically however the batch is
// split (batch invariance).
#include "gemm_common.cuh"

namespace flux {
namespace {

using namespace gemm;
constexpr int kBM = 128, kStages = 4;
constexpr int kABytes = kBM * kBK * 2;   // 16 KB
constexpr int kBBytes = kBN * kBK * 2;   // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kThreads = 256;
constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256 + 3 * kMaxGroups * 4 + 64 + 16 + kScaleSmemBytes;

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tm_a_r, const __grid_constant__ CUtensorMap tm_a_s,
                        const __grid_constant__ CUtensorMap tm_b_r, const __grid_constant__ CUtensorMap tm_b_s,
                        Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;   // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int32_t* s_sched = reinterpret_cast<int32_t*>(smem + kStages * kStageBytes + 256);
  int32_t* s_row0 = s_sched + kMaxGroups;
  int32_t* s_rows = s_row0 + kMaxGroups;
  float* s_scales =  // [2][kScaleFloats] (stage_tile_scales), 16-byte aligned
      reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(s_rows + kMaxGroups) + 15) & ~uintptr_t(15));

  const int warp = warp_id();
  for (int i = threadIdx.x; i <= p.n_groups; i += kThreads) s_sched[i] = p.sched[i];
  for (int i = threadIdx.x; i < p.n_groups; i += kThreads) {
    s_row0[i] = p.grp_row0[i];
    s_rows[i] = p.grp_rows[i];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total = s_sched[p.n_groups];
  const int nkb_r = (p.K_r + kBK - 1) / kBK, nkb_s = (p.K_s + kBK - 1) / kBK;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&tm_a_r);
      tma_prefetch(&tm_b_r);
      tma_prefetch(&tm_a_s);
      tma_prefetch(&tm_b_s);
      uint32_t it = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const TileInfo ti = decode(tile, s_sched, p.n_groups, p.n_tiles_r, p.n_tiles_s, p.E);
        const bool routed = ti.g < p.E;
        const int arow = s_row0[ti.g] + ti.m * kBM;
        const int brow = (routed ? ti.g * p.b_rows_r : 0) + ti.n * kBN;
        const CUtensorMap* ta = routed ? &tm_a_r : &tm_a_s;
        const CUtensorMap* tb = routed ? &tm_b_r : &tm_b_s;
        const int nkb = routed ? nkb_r : nkb_s;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * kStageBytes;
          mbar_arrive_expect_tx(&full[s], kStageBytes);
          tma_load_2d(st, ta, &full[s], kb * kBK, arow);
          tma_load_2d(st + kABytes, tb, &full[s], kb * kBK, brow);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = umma_idesc_bf16(kBM, kBN);
    uint32_t it = 0, tc = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++tc) {
      const TileInfo ti = decode(tile, s_sched, p.n_groups, p.n_tiles_r, p.n_tiles_s, p.E);
      const int nkb = ti.g < p.E ? nkb_r : nkb_s;
      const uint32_t acc = tc & 1, aph = (tc >> 1) & 1;
      mbar_wait(&tempty[acc], aph ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + acc * kBN;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % kStages;
        const uint32_t ph = (it / kStages) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(smem + s * kStageBytes);
          const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + kABytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) umma_bf16(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          umma_commit(&empty[s]);
          if (kb == nkb - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    uint32_t tc = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++tc) {
      const TileInfo ti = decode(tile, s_sched, p.n_groups, p.n_tiles_r, p.n_tiles_s, p.E);
      const uint32_t acc = tc & 1, aph = (tc >> 1) & 1;
      const float* sc = stage_tile_scales<EPI>(p, ti, s_scales, tc, (int)threadIdx.x - 128);
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int r_local = ti.m * kBM + q * 32 + (int)lane_id();
      epilogue_slice<EPI>(p, tmem + acc * kBN + lane_base, ti, r_local < s_rows[ti.g],
                          (int64_t)s_row0[ti.g] + r_local, kBN / 2, sc);
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

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

cudaError_t launch_gemm_1sm(GemmEpi epi, const CUtensorMap& a_r, const CUtensorMap& a_s, const CUtensorMap& b_r,
                            const CUtensorMap& b_s, const GemmArgs& g, cudaStream_t st) {
  const Params p = make_params(g);
  if (g.n_groups > kMaxGroups - 1) return cudaErrorInvalidValue;
  auto kern = epi == EPI_SWIGLU  ? grouped_gemm_kernel<EPI_SWIGLU>
              : epi == EPI_STORE ? grouped_gemm_kernel<EPI_STORE>
                                 : grouped_gemm_kernel<EPI_COMBINE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  if (e != cudaSuccess) return e;
  kern<<<g.grid, kThreads, kSmemBytes, st>>>(a_r, a_s, b_r, b_s, p);
  return cudaGetLastError();
}

}  // namespace flux
