// permute.cu — K2: D_e (the tokens routed to each expert) as a
// deterministic, stable permutation, plus the grouped-GEMM tile schedule.
//
//  permute_kernel   ONE cooperative launch: per-expert exclusive scans over the
//                   router's per-tile counts -> tile_base[tile][e]; a grid
//                   barrier; every CTA scans the per-expert totals -> offsets
//                   (CTA 0 publishes them with the tile prefix of both grouped
//                   GEMMs); then one thread per pick (t, j):
//                   pos = offsets[e] + tile_base[tile][e] + rank (rank from K1)
//                   -> token_index[pos] = t (ascending t inside every segment:
//                   reading R3), inv_pos[t][j] = pos.  k·16 bytes per token.
//  scatter_kernel   (one warp per token; only when x_perm is materialised): the
//                   gather x[t] -> x_perm[pos] (16-byte vectors, x read once,
//                   written k times), rewriting the same indices.
// No atomics decide positions, so D_e is bitwise reproducible.
#include <algorithm>

#include "internal.h"
#include "ptx.cuh"

namespace flux {

namespace {


// Exclusive scan over the CTA (NW warps); sh: NW ints of shared memory.
template <int NW>
__device__ __forceinline__ int block_exclusive_scan(int v, int* sh, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < NW ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < NW; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NW) sh[lane] = s;
  }
  __syncthreads();
  const int warp_prefix = wid ? sh[wid - 1] : 0;
  total = sh[NW - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

__global__ void __launch_bounds__(256) scatter_kernel(const uint4* __restrict__ x, int64_t T, int H, int E, int k,
                                                      const int32_t* __restrict__ ids, const int32_t* __restrict__ rank,
                                                      const int32_t* __restrict__ tile_base,
                                                      const int32_t* __restrict__ offsets, int32_t* __restrict__ inv_pos,
                                                      int32_t* __restrict__ token_index, uint4* __restrict__ x_perm) {
  const int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= T) return;
  const int lane = threadIdx.x & 31;
  const int tile = (int)(t / kRouterTile);
  int pos[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    pos[j] = -1;
    if (j < k) {
      const int e = __ldg(&ids[t * k + j]);
      if (e >= 0)  // -1: a pick folded by gate re-routing (NEXT-2) owns no row
        pos[j] = __ldg(&offsets[e]) + __ldg(&tile_base[(int64_t)tile * E + e]) + __ldg(&rank[t * k + j]);
    }
  }
  if (lane < k) {
    int p = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (j == lane) p = pos[j];
    inv_pos[t * k + lane] = p;
    if (p >= 0) token_index[p] = (int32_t)t;
  }
  const int nvec = H / 8;  // 16-byte vectors per row
  const uint4* src = x + t * nvec;
  // four 16-byte vectors per lane in flight before the k copies are written
  for (int c0 = lane; c0 < nvec; c0 += 128) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c0 + 32 * u < nvec) v[u] = __ldg(&src[c0 + 32 * u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (c0 + 32 * u >= nvec) continue;
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < k && pos[j] >= 0) x_perm[(int64_t)pos[j] * nvec + c0 + 32 * u] = v[u];
    }
  }
}
// K2 in one launch.  Phase 1: CTA e (strided) scans expert e's per-tile counts -> tile_base[tile][e]
// and grp_rows[e] = its row count.  Grid barrier (counter zeroed by K1; the launch is cooperative, so
// every CTA is resident).  Phase 2: every CTA scans the E counts into its own shared offsets table; CTA 0
// also publishes offsets, the user's D_e bounds and both GEMM tile schedules.  Phase 3: one thread per
// pick (t, j): pos = offsets[e] + tile_base[tile][e] + rank -> token_index[pos] = t, inv_pos = pos.
constexpr int kMaxE2 = 1024;
__global__ void __launch_bounds__(512) permute_kernel(ScheduleArgs a, const int32_t* __restrict__ ids,
                                                      const int32_t* __restrict__ rank, int32_t* __restrict__ inv_pos,
                                                      int32_t* __restrict__ token_index) {
  __shared__ int sh[16];
  __shared__ int s_off[kMaxE2 + 1];
  const int E = a.E;
  // ---- phase 1: per-expert scans
  for (int e = blockIdx.x; e < E; e += gridDim.x) {
    int carry = 0;
    for (int base = 0; base < a.n_tiles; base += 512) {
      const int tile = base + threadIdx.x;
      const int v = tile < a.n_tiles ? __ldcg(&a.tile_counts[(int64_t)tile * E + e]) : 0;
      int tot;
      const int ex = block_exclusive_scan<16>(v, sh, tot);
      if (tile < a.n_tiles) a.tile_base[(int64_t)tile * E + e] = carry + ex;
      carry += tot;
    }
    if (threadIdx.x == 0) a.grp_rows[e] = carry;
  }
  // ---- grid barrier
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(a.done_counter, 1);
    int seen;
    for (;;) {  // back off between polls: ~300 CTAs polling one line slow the arrivals down
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(seen) : "l"(a.done_counter) : "memory");
      if (seen >= (int)gridDim.x) break;
      __nanosleep(64);
    }
  }
  __syncthreads();
  // ---- phase 2: offsets (every CTA, in shared memory); CTA 0 publishes offsets + GEMM schedules
  const int n_groups = E + (a.has_shared ? 1 : 0);
  int carry_rows = 0, carry_gu = 0, carry_dn = 0;
  for (int base = 0; base < n_groups; base += 512) {
    const int g = base + threadIdx.x;
    int rows = 0;
    if (g < E) rows = __ldcg(&a.grp_rows[g]);
    else if (g < n_groups) rows = (int)a.T;
    int tot_rows;
    const int ex_rows = block_exclusive_scan<16>(g < E ? rows : 0, sh, tot_rows);
    const int row0 = g < E ? carry_rows + ex_rows : 0;
    if (g < E) s_off[g] = row0;
    if (blockIdx.x == 0) {
      const int mt = (rows + a.gemm_bm - 1) / a.gemm_bm;
      const int ngu = mt * (g < E ? a.n_tiles_gu : a.n_tiles_gu_sh);
      const int ndn = mt * (g < E ? a.n_tiles_dn : a.n_tiles_dn_sh);
      int tot_gu, tot_dn;
      const int ex_gu = block_exclusive_scan<16>(g < n_groups ? ngu : 0, sh, tot_gu);
      const int ex_dn = block_exclusive_scan<16>(g < n_groups ? ndn : 0, sh, tot_dn);
      if (g < n_groups) {
        a.grp_row0[g] = row0;
        if (g >= E) a.grp_rows[g] = rows;
        a.sched_gu[g] = carry_gu + ex_gu;
        a.sched_dn[g] = carry_dn + ex_dn;
      }
      carry_gu += tot_gu;
      carry_dn += tot_dn;
    }
    carry_rows += tot_rows;
  }
  if (threadIdx.x == 0) s_off[E] = carry_rows;
  __syncthreads();
  if (blockIdx.x == 0 && a.sched_c) {  // chained GEMM (gemm_chain.cu): per-group tile and m-tile prefixes
    int carry_c = 0, carry_mt = 0;
    for (int base = 0; base < n_groups; base += 512) {
      const int g = base + threadIdx.x;
      int mt = 0, nc = 0;
      if (g < n_groups) {
        const int rows = g < E ? __ldcg(&a.grp_rows[g]) : (int)a.T;
        mt = (rows + a.gemm_bm - 1) / a.gemm_bm;
        nc = mt * (g < E ? a.n_tiles_gu + a.n_tiles_dn : a.n_tiles_gu_sh + a.n_tiles_dn_sh);
      }
      int tot_c, tot_mt;
      const int ex_c = block_exclusive_scan<16>(nc, sh, tot_c);
      const int ex_mt = block_exclusive_scan<16>(mt, sh, tot_mt);
      if (g < n_groups) {
        a.sched_c[g] = carry_c + ex_c;
        a.mt_base[g] = carry_mt + ex_mt;
      }
      carry_c += tot_c;
      carry_mt += tot_mt;
    }
    if (threadIdx.x == 0) a.sched_c[n_groups] = carry_c;
    for (int i = threadIdx.x; i < carry_mt; i += 512) a.ready[i] = 0;
  }
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) {
      a.sched_gu[n_groups] = carry_gu;
      a.sched_dn[n_groups] = carry_dn;
      if (a.sched_sh) {  // the shared MLP alone (down GEMM with the fused combine epilogue)
        a.sched_sh[0] = 0;
        a.sched_sh[1] = (int)((a.T + a.gemm_bm - 1) / a.gemm_bm) * a.n_tiles_dn_sh;
        a.grp_row0_sh[0] = 0;
        a.grp_rows_sh[0] = (int)a.T;
      }
    }
    for (int g = threadIdx.x; g <= E; g += 512) {
      a.offsets[g] = s_off[g];
      if (a.user_offsets) a.user_offsets[g] = s_off[g];
    }
  }
  // ---- phase 3: one thread per pick; four independent picks per thread in flight (their ids / rank /
  // tile_base loads are issued before the first store)
  const int64_t Tk = a.T * a.k;
  const int k = a.k;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < Tk; i0 += 4 * stride) {
    int e[4], r[4], tb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      e[u] = i < Tk ? __ldcs(&ids[i]) : -2;
      r[u] = i < Tk ? __ldcs(&rank[i]) : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      tb[u] = e[u] >= 0 ? __ldcg(&a.tile_base[((i / k) / kRouterTile) * E + e[u]]) : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      if (e[u] == -2) continue;
      int p = -1;
      if (e[u] >= 0) {  // -1: a pick folded by gate re-routing (NEXT-2) owns no row
        p = s_off[e[u]] + tb[u] + r[u];
        token_index[p] = (int32_t)(i / k);
      }
      inv_pos[i] = p;
    }
  }
}
}  // namespace

cudaError_t launch_permute(const ScheduleArgs& a0, const int32_t* ids, const int32_t* rank, int32_t* inv_pos,
                           int32_t* token_index, cudaStream_t st) {
  if (a0.E > kMaxE2) return cudaErrorInvalidValue;
  static int max_blocks = -1;  // co-resident CTAs per SM (cooperative launch bound)
  if (max_blocks < 0) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, permute_kernel, 512, 0) != cudaSuccess) return cudaErrorUnknown;
    max_blocks = n;
  }
  const int64_t Tk = a0.T * a0.k;
  const int64_t want = std::max<int64_t>((int64_t)a0.E, (Tk + 2047) / 2048);  // 4 picks per thread
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)kNumSMs * std::min(max_blocks, 2)));
  ScheduleArgs a = a0;
  void* args[] = {&a, &ids, &rank, &inv_pos, &token_index};
  return cudaLaunchCooperativeKernel((const void*)permute_kernel, dim3(grid), dim3(512), args, 0, st);
}

cudaError_t launch_scatter(const void* x, int64_t T, int H, int E, int k, const int32_t* ids, const int32_t* rank,
                           const int32_t* tile_base, const int32_t* offsets, int32_t* inv_pos, int32_t* token_index,
                           void* x_perm, cudaStream_t st) {
  if (T == 0 || !x_perm) return cudaSuccess;
  const unsigned grid = (unsigned)((T + 7) / 8);
  scatter_kernel<<<grid, 256, 0, st>>>((const uint4*)x, T, H, E, k, ids, rank, tile_base, offsets, inv_pos,
                                       token_index, (uint4*)x_perm);
  return cudaGetLastError();
}

}  // namespace flux
