// router.cu — K1: gating network + top-k + activation histogram, fused.
//
// Paper: tokens "first pass through a gating network, which determines their
// assignment to different experts"; activation frequency =
// activated tokens / total tokens.  Reading R2:
// z = x·W_rᵀ, p = softmax(z), S = top-k(z) (lower expert index on ties,
// listed by descending z), w = p_S (norm 0) or p_S/Σp_S (norm 1).
//
// One CTA = 128 tokens.  The logits are a real (if skinny) GEMM,
// [128 × H]·[H × N] with N = E padded to a multiple of 16, so they run on the
// tensor cores: TMA streams 64-wide K slices of x and W_r (128-byte swizzle)
// through a 4-stage mbarrier ring, one thread issues tcgen05.mma (M=128, N,
// K=16) into a TMEM accumulator, and 4 epilogue warps read one token row each
// with tcgen05.ld.  The epilogue keeps the row in registers: max, softmax
// denominator, k argmax passes, weights.  The histogram is CTA-aggregated:
// each token sets its bit in a per-expert 128-bit mask in shared memory; one
// popcount per expert gives this tile's count (one global atomic per expert
// per CTA) and the stable within-tile rank of every (token, expert) pair that
// the permutation (K2) needs.  NEXT-2 gate re-routing (§7, R14): with a remap table
// the picks are sent to the compact model's slots in the same epilogue, repeated slots folded.
#include "internal.h"
#include "ptx.cuh"

namespace flux {

namespace {
constexpr int kStages = 4;  // (3 stages / 3 CTAs per SM measured slower: 0.38 vs 0.32 ms per layer)
constexpr int kBM = 128, kBK = 64;
constexpr int kThreads = 192;  // warp 0: TMA, warp 1: MMA + TMEM, warps 2..5: epilogue

template <int NPAD>
struct RouterSmem {
  static constexpr int kA = kBM * kBK * 2;    // 16 KB
  static constexpr int kB = NPAD * kBK * 2;   // <= 16 KB
  static constexpr int kStage = kA + kB;
  static constexpr int kBytes = kStages * kStage + 1024 /*align*/ + 256 /*barriers*/ + NPAD * 4 * 4 /*masks*/;
};

template <int NPAD>
__global__ void __launch_bounds__(kThreads, 1)
    router_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_wr,
                  RouterArgs a) {
  using S = RouterSmem<NPAD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * S::kStage);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  uint32_t* masks = reinterpret_cast<uint32_t*>(smem + kStages * S::kStage + 256);  // [NPAD][4]

  constexpr uint32_t kTmemCols = NPAD <= 32 ? 32 : (NPAD <= 64 ? 64 : 128);
  const int warp = warp_id();
  const int tile = blockIdx.x;
  const int nkb = a.H / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&tmap_x);
      tma_prefetch(&tmap_wr);
      const uint64_t pol_x = policy_evict_first();
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % kStages;
        const uint32_t ph = (kb / kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * S::kStage;
        mbar_arrive_expect_tx(&full[s], S::kStage);
        tma_load_2d_hint(sa, &tmap_x, &full[s], kb * kBK, tile * kBM, pol_x);
        tma_load_2d(sa + S::kA, &tmap_wr, &full[s], kb * kBK, 0);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = umma_idesc_bf16(kBM, NPAD);
    for (int kb = 0; kb < nkb; ++kb) {
      const int s = kb % kStages;
      const uint32_t ph = (kb / kStages) & 1;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t sa = smem_u32(smem + s * S::kStage);
        const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + S::kA);
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)  // +32 bytes along K inside the swizzle atom = +2 in addr>>4
          umma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
        umma_commit(&empty[s]);
        if (kb == nkb - 1) umma_commit(acc_full);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int row = q * 32 + lane_id();     // token row inside the tile == TMEM lane
    const int64_t t = (int64_t)tile * kBM + row;
    const bool valid = t < a.T;
    const int E = a.E, k = a.k;
    const int et = threadIdx.x - 64;        // 0..127
    for (int i = et; i < NPAD * 4; i += 128) masks[i] = 0;

    mbar_wait(acc_full, 0);
    tc_fence_after();
    float z[NPAD];
#pragma unroll
    for (int c = 0; c < NPAD; c += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c, v);
#pragma unroll
      for (int i = 0; i < 16; ++i) z[c + i] = v[i];
    }
    tmem_ld_wait();

    // softmax statistics over the E real experts (padded columns excluded)
    float zmax = -INFINITY;
#pragma unroll
    for (int e = 0; e < NPAD; ++e)
      if (e < E) zmax = fmaxf(zmax, z[e]);
    float denom = 0.f;
#pragma unroll
    for (int e = 0; e < NPAD; ++e)
      if (e < E) denom += expf(z[e] - zmax);

    // top-k: k passes of "largest unselected, lowest index on ties"
    uint32_t sel[(NPAD + 31) / 32];
#pragma unroll
    for (int i = 0; i < (NPAD + 31) / 32; ++i) sel[i] = 0;
    int ids[8];
    float ps[8];
    float psum = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      ids[j] = 0;
      ps[j] = 0.f;
      if (j >= k) continue;
      int best = -1;
      float bz = 0.f;
#pragma unroll
      for (int e = 0; e < NPAD; ++e) {
        const bool free_e = e < E && !((sel[e >> 5] >> (e & 31)) & 1u);
        if (free_e && (best < 0 || z[e] > bz)) {
          best = e;
          bz = z[e];
        }
      }
#pragma unroll
      for (int i = 0; i < (NPAD + 31) / 32; ++i)
        if ((best >> 5) == i) sel[i] |= 1u << (best & 31);
      ids[j] = best;
      ps[j] = expf(bz - zmax) / denom;
      psum += ps[j];
    }

    // gate weights; with re-routing (NEXT-2, R14) every pick goes to remap[id] and a pick whose slot
    // repeats an earlier (higher-logit) pick's is folded into it: weight added, pick emptied (-1)
    float wt[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) wt[j] = j < k ? (a.norm ? ps[j] / psum : ps[j]) : 0.f;
    if (a.remap) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < k) ids[j] = __ldg(&a.remap[ids[j]]);
#pragma unroll
      for (int j = 1; j < 8; ++j) {
        if (j >= k) continue;
        bool done = false;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if (i < j && !done && ids[i] >= 0 && ids[i] == ids[j]) {
            wt[i] += wt[j];
            wt[j] = 0.f;
            ids[j] = -1;
            done = true;
          }
      }
    }

    named_bar_sync(1, 128);  // masks zeroed
    if (valid) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < k && ids[j] >= 0) atomicOr(&masks[ids[j] * 4 + (row >> 5)], 1u << (row & 31));
    }
    named_bar_sync(1, 128);

    if (valid) {
      int32_t* gid = a.ids + t * k;
      float* gw = a.w + t * k;
      int32_t* grk = a.rank + t * k;
      const uint32_t below = (1u << (row & 31)) - 1u;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j >= k) continue;
        int r = 0;
        if (ids[j] >= 0) {
          const uint32_t* m = &masks[ids[j] * 4];
          r = __popc(m[row >> 5] & below);
          for (int wd = 0; wd < (row >> 5); ++wd) r += __popc(m[wd]);
        }
        gid[j] = ids[j];
        gw[j] = wt[j];
        grk[j] = r;
      }
      if (a.logits) {
        float* gl = a.logits + t * E;
#pragma unroll
        for (int e = 0; e < NPAD; ++e)
          if (e < E) gl[e] = z[e];
      }
    }
    if (et < a.E_slots) {
      const uint32_t* m = &masks[et * 4];
      const int cnt = __popc(m[0]) + __popc(m[1]) + __popc(m[2]) + __popc(m[3]);
      a.tile_counts[(int64_t)tile * a.E_slots + et] = cnt;
      if (cnt) atomicAdd(reinterpret_cast<unsigned long long*>(a.hist + et), (unsigned long long)cnt);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kTmemCols>(tmem);
}
}  // namespace

template <int NPAD>
static cudaError_t launch_router_n(const CUtensorMap& tx, const CUtensorMap& tw, const RouterArgs& a,
                                   cudaStream_t st) {
  const int smem = RouterSmem<NPAD>::kBytes;
  cudaError_t e = cudaFuncSetAttribute(router_kernel<NPAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const unsigned grid = (unsigned)((a.T + kBM - 1) / kBM);
  router_kernel<NPAD><<<grid, kThreads, smem, st>>>(tx, tw, a);
  return cudaGetLastError();
}

cudaError_t launch_router(const CUtensorMap& tx, const CUtensorMap& tw, int npad, const RouterArgs& a,
                          cudaStream_t st) {
  switch (npad) {
    case 16: return launch_router_n<16>(tx, tw, a, st);
    case 32: return launch_router_n<32>(tx, tw, a, st);
    case 64: return launch_router_n<64>(tx, tw, a, st);
    case 128: return launch_router_n<128>(tx, tw, a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace flux
