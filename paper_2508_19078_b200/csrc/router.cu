// router.cu — K1: gating network + top-k + activation histogram, fused.
//
// Paper: tokens "first pass through a gating network, which determines their
// assignment to different experts"; activation frequency =
// activated tokens / total tokens.  Reading R2:
// z = x·W_rᵀ, p = softmax(z), S = top-k(z) (lower expert index on ties,
// listed by descending z), w = p_S (norm 0) or p_S/Σp_S (norm 1).
//
// One router tile = 256 tokens; persistent CTAs (one per SM) walk the tiles.  The logits are a real (if skinny) GEMM,
// [128 × H]·[H × N] with N = E padded to a multiple of 16, so they run on the
// tensor cores: TMA streams 64-wide K slices of x and W_r (128-byte swizzle)
// through a 4-stage mbarrier ring, one thread issues tcgen05.mma (M=128, N,
// K=16) into a TMEM accumulator, and 4 epilogue warps read one token row each
// with tcgen05.ld.  The epilogue keeps the row in registers: max, softmax
// denominator, k argmax passes, weights.  The histogram is CTA-aggregated:
// every epilogue warp builds, with one ballot per expert, the 32-bit mask of
// its 32 tokens that picked that expert (a 256-bit mask per expert per tile in
// shared memory, each word written by exactly one warp: no shared atomics);
// popcounts give this tile's count (one global atomic per expert per CTA) and
// the stable within-tile rank of every (token, expert) pair that the
// permutation (K2) needs.  NEXT-2 gate re-routing (§7, R14): with a remap table
// the picks are sent to the compact model's slots in the same epilogue, repeated slots folded.
#include <algorithm>

#include "internal.h"
#include "ptx.cuh"

namespace flux {

namespace {
constexpr int kBM = kRouterTile, kBK = 64;  // 256 tokens per tile: two M=128 MMAs share each W_r slice
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;  // warp 0: TMA, warp 1: MMA + TMEM, warps 2..9: epilogue

template <int NPAD>
struct RouterSmem {
  static constexpr int kA = kBM * kBK * 2;    // 32 KB of x (256 rows x 128 B)
  static constexpr int kB = NPAD * kBK * 2;   // <= 16 KB of W_r
  static constexpr int kStage = kA + kB;
  static constexpr int kStages = NPAD <= 64 ? 5 : 4;  // ~160 / 128 KB of x in flight per SM
  static constexpr int kBytes = kStages * kStage + 1024 /*align*/ + 256 /*barriers*/ + NPAD * 8 * 4 /*masks*/;
};

// Persistent: CTA b handles router tiles b, b + gridDim.x, ...  The TMEM accumulators are double
// buffered, so the epilogue (softmax, top-k, histogram) of tile i overlaps the loads and MMAs of
// tile i + 1 and the x stream never stops.  A 256-token tile halves the W_r re-reads from L2
// (W_r is 256 KB for the DeepSeek shape: re-read per 128 tokens it cost half the x traffic again).
template <int NPAD>
__global__ void __launch_bounds__(kThreads, 1)
    router_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_wr,
                  RouterArgs a) {
  using S = RouterSmem<NPAD>;
  constexpr int kStages = S::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, still a shared-space pointer
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * S::kStage);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  uint32_t* masks = reinterpret_cast<uint32_t*>(smem + kStages * S::kStage + 256);  // [8 row groups][NPAD]

  // two buffers x two 128-row halves x NPAD columns
  constexpr uint32_t kTmemCols = NPAD <= 16 ? 64 : (NPAD <= 32 ? 128 : (NPAD <= 64 ? 256 : 512));
  const int warp = warp_id();
  const int n_tiles = (int)((a.T + kBM - 1) / kBM);
  const int nkb = a.H / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kEpiWarps);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (a.zero4 && blockIdx.x == 0 && threadIdx.x < 4) a.zero4[threadIdx.x] = 0;  // for K2 and the GEMMs

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&tmap_x);
      tma_prefetch(&tmap_wr);
      const uint64_t pol_x = policy_evict_first();
      int g = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x)
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % kStages;
          const uint32_t ph = (g / kStages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * S::kStage;
          mbar_arrive_expect_tx(&full[s], S::kStage);
          tma_load_2d_hint(sa, &tmap_x, &full[s], kb * kBK, tile * kBM, pol_x);
          tma_load_2d(sa + S::kA, &tmap_wr, &full[s], kb * kBK, 0);
        }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = umma_idesc_bf16(128, NPAD);
    int g = 0, i = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++i) {
      const int b = i & 1;
      mbar_wait(&acc_empty[b], ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % kStages;
        const uint32_t ph = (g / kStages) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = smem_u32(smem + s * S::kStage);
          const uint64_t da0 = umma_desc_sw128(sa), da1 = umma_desc_sw128(sa + S::kA / 2),
                         db = umma_desc_sw128(sa + S::kA);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {  // +32 bytes along K inside the swizzle atom = +2 in addr>>4
            umma_bf16(tmem + (2 * b) * NPAD, da0 + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
            umma_bf16(tmem + (2 * b + 1) * NPAD, da1 + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[s]);
          if (kb == nkb - 1) umma_commit(&acc_full[b]);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2..9)
    const int q = warp & 3;                   // TMEM lane quarter this warp may access
    const int half = (warp - 2) >> 2;         // which 128-row half of the tile
    const int row = half * 128 + q * 32 + lane_id();  // token row inside the tile
    const int E = a.E, k = a.k;
    const int et = threadIdx.x - 64;          // 0..255
    int i = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++i) {
      const int b = i & 1;
      const int64_t t = (int64_t)tile * kBM + row;
      const bool valid = t < a.T;
      mbar_wait(&acc_full[b], (i >> 1) & 1);
      tc_fence_after();
      float z[NPAD];
#pragma unroll
      for (int c = 0; c < NPAD; c += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + (2 * b + half) * NPAD + c, v);
#pragma unroll
        for (int j = 0; j < 16; ++j) z[c + j] = v[j];
      }
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&acc_empty[b]);  // the MMA warp may reuse this accumulator

      // softmax statistics over the E real experts (padded columns excluded)
      float zmax = -INFINITY;
#pragma unroll
      for (int e = 0; e < NPAD; ++e)
        if (e < E) zmax = fmaxf(zmax, z[e]);
      float denom = 0.f;
#pragma unroll
      for (int e = 0; e < NPAD; ++e)
        if (e < E) denom += expf(z[e] - zmax);

      if (a.logits && valid) {  // parity/debug output, before the selection below consumes z
        float* gl = a.logits + t * E;
#pragma unroll
        for (int e = 0; e < NPAD; ++e)
          if (e < E) gl[e] = z[e];
      }
      // top-k: k passes of "largest remaining, lowest index on ties" (strict > while scanning e upwards);
      // a picked logit is replaced by -inf, padded columns never qualify: ~5 instructions per element
      // and pass instead of ~7.5 with a selected-bit mask (the epilogue is the router's issue budget at
      // the power-capped clock)
#pragma unroll
      for (int e = 0; e < NPAD; ++e)
        if (e >= E) z[e] = -INFINITY;
      int ids[8];
      float ps[8];
      float psum = 0.f;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        ids[j] = 0;
        ps[j] = 0.f;
        if (j >= k) continue;
        int best = 0;
        float bz = -INFINITY;
#pragma unroll
        for (int e = 0; e < NPAD; ++e) {
          const bool gt = z[e] > bz;
          bz = gt ? z[e] : bz;
          best = gt ? e : best;
        }
#pragma unroll
        for (int e = 0; e < NPAD; ++e) z[e] = e == best ? -INFINITY : z[e];
        ids[j] = best;
        ps[j] = expf(bz - zmax) / denom;
        psum += ps[j];
      }

      // gate weights; with re-routing (NEXT-2, R14) every pick goes to remap[id] and a pick whose
      // slot repeats an earlier (higher-logit) pick's is folded into it: weight added, pick emptied
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
          for (int m = 0; m < 8; ++m)
            if (m < j && !done && ids[m] >= 0 && ids[m] == ids[j]) {
              wt[m] += wt[j];
              wt[j] = 0.f;
              ids[j] = -1;
              done = true;
            }
        }
      }

      // per-expert token masks of this warp's 32 rows: one ballot per expert column (no shared-memory
      // atomics: every mask word has exactly one writer), masks[wr][e] with wr = row >> 5
      uint32_t pk[(NPAD + 31) / 32];
#pragma unroll
      for (int w = 0; w < (NPAD + 31) / 32; ++w) pk[w] = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (valid && j < k && ids[j] >= 0) {
#pragma unroll
          for (int w = 0; w < (NPAD + 31) / 32; ++w)
            if ((ids[j] >> 5) == w) pk[w] |= 1u << (ids[j] & 31);
        }
      uint32_t word[(NPAD + 31) / 32] = {};
#pragma unroll
      for (int e = 0; e < NPAD; ++e) {
        const uint32_t bal = __ballot_sync(0xffffffffu, (pk[e >> 5] >> (e & 31)) & 1u);
        if ((e & 31) == lane_id()) word[e >> 5] = bal;
      }
      named_bar_sync(1, 32 * kEpiWarps);  // the previous tile's mask readers are done
#pragma unroll
      for (int w = 0; w < (NPAD + 31) / 32; ++w)
        if (w * 32 + lane_id() < NPAD) masks[(row >> 5) * NPAD + w * 32 + lane_id()] = word[w];
      named_bar_sync(1, 32 * kEpiWarps);

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
            const uint32_t* m = &masks[ids[j]];
            r = __popc(m[(row >> 5) * NPAD] & below);
            for (int wd = 0; wd < (row >> 5); ++wd) r += __popc(m[wd * NPAD]);
          }
          gid[j] = ids[j];
          gw[j] = wt[j];
          grk[j] = r;
        }
      }
      if (et < a.E_slots) {
        const uint32_t* m = &masks[et];
        int cnt = 0;
#pragma unroll
        for (int wd = 0; wd < 8; ++wd) cnt += __popc(m[wd * NPAD]);
        a.tile_counts[(int64_t)tile * a.E_slots + et] = cnt;
        if (cnt) atomicAdd(reinterpret_cast<unsigned long long*>(a.hist + et), (unsigned long long)cnt);
      }
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
  const int64_t n_tiles = (a.T + kBM - 1) / kBM;
  const unsigned grid = (unsigned)std::min<int64_t>(n_tiles, kNumSMs);
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
