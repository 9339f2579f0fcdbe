// gemm_chain.cu — K3+K4 chained: the gate/up GEMM (SwiGLU epilogue -> act) and the down GEMM
// (act -> y_perm) of every expert group in ONE persistent CTA-pair launch, so that each m-tile's act
// rows are consumed by the down GEMM while they are still in L2 instead of a round trip through HBM
// (act is T·k·F·2 bytes: 4.4 GB per DeepSeek-shape layer written and read back, plus the shared
// MLP's 1.5 GB).
//
// Tile order (claimed in global order from one counter, as the two-launch kernels): group by group;
// inside group g with M m-tiles, a gate/up n-tiles and b down n-tiles, a lag of D m-tiles:
//   gu(0..D-1) | gu(D) dn(0) | gu(D+1) dn(1) | ... | gu(M-1) dn(M-1-D) | dn(M-D..M-1)
// A down tile of m-tile m waits (its producer polls a per-m-tile counter) until every gate/up
// epilogue warp of both CTAs of every gate/up tile of m-tile m has stored its act rows: 8 arrivals
// per gate/up tile.  Every gate/up tile of m-tile m is claimed before any of its down tiles and never
// waits itself, and a pair's producer waits only after it issued all loads of its earlier tiles, so
// the wait always ends.  With D m-tiles of lag the act working set is ~D·(rows x F x 2 B) — a few MB
// — and the awaited tiles have finished long before (D = 8: ~150 tiles claimed in between, 74 pairs).
//
// Everything else (tile shape 256 x 256 x 64-K, the 6-stage ring, cp.async gather of the routed A rows
// of gate/up tiles, TMEM double buffering, TMA-store epilogues, MMA instruction order per tile) is the
// gemm_pair.cu kernel's, so every output is bit-identical to the two-launch path.
//
// Measured (B200): NOT faster.  The lag must be ~24 m-tiles or the down tiles wait
// (D = 2: 1.7x slower; D = 8 still waits on the LLaMA shape), and at that distance the act lines have
// left L2 under the gathered x rows and the B tiles (ncu: 27.6 GB of DRAM traffic per DeepSeek layer
// vs 27.9 GB for the two launches; the dirty act lines are written back either way).  In the bench step
// DeepSeek ties (781 vs 780 ms of GEMM per step) and LLaMA loses 3%, so the policy default keeps the
// two launches and this kernel is reachable as FLUX_CHAIN_ON (covered by the bit-identity tests).
#include "gemm_pair.cuh"

namespace flux {
namespace {
using namespace gemm;

struct ChainMaps {  // [0] = gate/up, [1] = down
  CUtensorMap a_r[2], a_s[2], b_r[2], b_s[2], o_r[2], o_s[2];
};
struct ChainParams {
  Params p[2];
  const int32_t* sched_c;  // [n_groups+1] prefix of M_g·(a_g + b_g)
  const int32_t* mt_base;  // [n_groups] first global m-tile index of each group
  int32_t* ready;          // [M_total] act slices stored per m-tile (8 per gate/up tile)
  int D;
  int act_hint;            // 1: act stored with the default L2 policy, read with evict_first; 2: stored evict_first
};

struct CTile {
  int type;  // 0 = gate/up, 1 = down
  TileInfo ti;
};

__device__ __forceinline__ CTile decode_chain(int tile, const int32_t* s_sched_c, const int32_t* s_rows,
                                              const ChainParams& c, int n_groups, int E) {
  int lo = 0, hi = n_groups - 1;  // largest g with sched_c[g] <= tile
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_sched_c[mid] <= tile) lo = mid;
    else hi = mid - 1;
  }
  const int g = lo;
  int local = tile - s_sched_c[g];
  const int M = (s_rows[g] + kPairM - 1) / kPairM;
  const int a = g < E ? c.p[0].n_tiles_r : c.p[0].n_tiles_s;
  const int b = g < E ? c.p[1].n_tiles_r : c.p[1].n_tiles_s;
  const int Dg = min(c.D, M);
  if (local < Dg * a) return {0, {g, local / a, local % a}};
  local -= Dg * a;
  const int mid = (M - Dg) * (a + b);
  if (local < mid) {
    const int s = local / (a + b), r = local - s * (a + b);
    return r < a ? CTile{0, {g, Dg + s, r}} : CTile{1, {g, s, r - a}};
  }
  local -= mid;
  return {1, {g, M - Dg + local / b, local % b}};
}

__device__ __forceinline__ int ld_acquire_gpu(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

constexpr int kChainThreads = 288;  // TMA, MMA, 2 gather producers, 4 epilogue, gather relay

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kChainThreads, 1)
    chained_gemm_pair_kernel(const __grid_constant__ ChainMaps mp, const __grid_constant__ ChainParams c,
                             int32_t* tile_ctr) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, shared space
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* afull = full + 24;        // [kStages] (byte 192)
  int32_t* s_sched = reinterpret_cast<int32_t*>(smem + kStages * kStageBytes + 256);
  int32_t* s_row0 = s_sched + kMaxGroups;
  int32_t* s_rows = s_row0 + kMaxGroups;
  int32_t* s_mtb = s_rows + kMaxGroups;  // [n_groups <= 129] first m-tile of every group (the gather-id slot)
  float* s_scales = reinterpret_cast<float*>(smem + kStages * kStageBytes + kMiscBytes - kScaleSmemBytes);
  uint8_t* s_out = smem + kStages * kStageBytes + kMiscBytes;  // [4 warps][kStageOutBytes]
  uint64_t* tid_full = reinterpret_cast<uint64_t*>(s_out + 4 * kStageOutBytes + 4 * kPickBytes);
  uint64_t* tid_empty = tid_full + kTileSlots;
  int32_t* s_tid = reinterpret_cast<int32_t*>(tid_empty + kTileSlots);

  const Params& p0 = c.p[0];
  const int n_groups = p0.n_groups, E = p0.E;
  const int warp = warp_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  for (int i = threadIdx.x; i <= n_groups; i += kChainThreads) s_sched[i] = c.sched_c[i];
  for (int i = threadIdx.x; i < n_groups; i += kChainThreads) {
    s_row0[i] = p0.grp_row0[i];
    s_rows[i] = p0.grp_rows[i];
    s_mtb[i] = c.mt_base[i];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 3);  // leader expect_tx + one gather-relay arrive per CTA
      mbar_init(&empty[s], 1);
      mbar_init(&afull[s], 32 * kGatherParts);
    }
    for (int s = 0; s < kTileSlots; ++s) {
      mbar_init(&tid_full[s], 1);
      mbar_init(&tid_empty[s], 16);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int total = s_sched[n_groups];
  auto decode = [&](int tile) { return decode_chain(tile, s_sched, s_rows, c, n_groups, E); };
  auto nkb_of = [&](const CTile& t) {
    const Params& p = c.p[t.type];
    return ((t.ti.g < E ? p.K_r : p.K_s) + kBK - 1) / kBK;
  };

  // ---- tile ids: claimed in global order by the leader's producer, published through a ring
  auto read_tile = [&](int i) -> int {
    const int slot = i % kTileSlots;
    mbar_wait(&tid_full[slot], (i / kTileSlots) & 1);
    return *reinterpret_cast<volatile int32_t*>(&s_tid[slot]);
  };
  auto release_tile = [&](int i) {
    const int slot = i % kTileSlots;
    if (leader)
      mbar_arrive(&tid_empty[slot]);
    else
      mbar_arrive_cluster(mapa(smem_u32(&tid_empty[slot]), 0));
  };
  auto next_tile = [&](int i) -> int {  // whole warp; -1 = done
    int t = 0;
    if (lane_id() == 0) t = read_tile(i);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (lane_id() == 0) release_tile(i);
    return t;
  };
  int cur = 0, pending = 0;
  auto claim = [&]() -> int {
    const int v = atomicAdd(tile_ctr, 1);
    return v < total ? v : -1;
  };
  auto publish = [&](int i, int t) {
    const int slot = i % kTileSlots;
    mbar_wait(&tid_empty[slot], ((i / kTileSlots) & 1) ^ 1);
    s_tid[slot] = t;
    mbar_arrive(&tid_full[slot]);
    const uint32_t peer_full = mapa(smem_u32(&tid_full[slot]), 1);
    mbar_arrive_expect_tx_cluster(peer_full, 4);
    st_async_u32(mapa(smem_u32(&s_tid[slot]), 1), (uint32_t)t, peer_full);
  };
  if (leader && warp == 0 && lane_id() == 0) {
    cur = claim();
    publish(0, cur);
    pending = cur >= 0 ? claim() : -1;
  }
  auto claim_tile = [&](int i) -> int {
    int t = 0;
    if (lane_id() == 0) {
      t = cur;
      if (t >= 0) {
        publish(i + 1, pending);
        cur = pending;
        if (pending >= 0) pending = claim();
      }
    }
    return __shfl_sync(0xffffffffu, t, 0);
  };

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane_id() == 0)
      for (int t = 0; t < 2; ++t) {
        tma_prefetch(&mp.a_r[t]);
        tma_prefetch(&mp.b_r[t]);
        tma_prefetch(&mp.a_s[t]);
        tma_prefetch(&mp.b_s[t]);
      }
    const uint64_t pol_first = policy_evict_first();
    uint32_t it = 0;
    for (int i = 0;; ++i) {
      const int tile = leader ? claim_tile(i) : next_tile(i);
      if (tile < 0) break;
      const CTile ct = decode(tile);
      const TileInfo& ti = ct.ti;
      const Params& p = c.p[ct.type];
      const bool routed = ti.g < E;
      const bool gather = ct.type == 0 && routed;  // A rows by the cp.async gather warps
      if (ct.type == 1) {
        // the act rows of this m-tile: every gate/up epilogue warp of both CTAs of all a_g tiles
        const int want = 8 * (routed ? p0.n_tiles_r : p0.n_tiles_s);
        const int32_t* flag = c.ready + s_mtb[ti.g] + ti.m;
        if (lane_id() == 0 && ld_acquire_gpu(flag) < want) {
          const uint64_t t0 = globaltimer_ns();
          while (ld_acquire_gpu(flag) < want) {  // a wait past 10 s can only be a deadlock: fail loudly
            __nanosleep(128);
            if (globaltimer_ns() - t0 > 10000000000ull) __trap();
          }
        }
        if (lane_id() == 0) {
          asm volatile("fence.proxy.async.global;" ::: "memory");  // order the acquire before the TMA reads
        }
        __syncwarp();
      }
      const int first = ti.m * kPairM + (int)rank * kHalfM;
      const int arow = s_row0[ti.g] + first;
      const int half = ct.type == 0 ? kBN / 2 : pair_tile_cols<EPI_STORE>(p, ti) / 2;
      const int brow = (routed ? ti.g * p.b_rows_r : 0) + ti.n * kBN + (int)rank * half;
      const CUtensorMap* ta = routed ? &mp.a_r[ct.type] : &mp.a_s[ct.type];
      const CUtensorMap* tb = routed ? &mp.b_r[ct.type] : &mp.b_s[ct.type];
      const int nkb = nkb_of(ct);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = (it + kb) % kStages;
        const uint32_t ph = ((it + kb) / kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * kStageBytes;
        if (leader && lane_id() == 0) mbar_arrive_expect_tx(&full[s], gather ? 2 * kBBytes : 2 * kStageBytes);
        __syncwarp();
        if (lane_id() == 0) {
          if (ct.type == 1 && c.act_hint)  // act is dead once the m-tile's down tiles read it
            tma_load_2d_pair_hint(st, ta, &full[s], kb * kBK, arow, pol_first);
          else if (!gather)
            tma_load_2d_pair(st, ta, &full[s], kb * kBK, arow);
          tma_load_2d_pair(st + kABytes, tb, &full[s], kb * kBK, brow);
        }
      }
      it += nkb;
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader CTA)
    if (leader) {
      uint32_t it = 0, tc = 0;
      for (int i = 0;; ++i, ++tc) {
        const int tile = next_tile(i);
        if (tile < 0) break;
        const CTile ct = decode(tile);
        const Params& p = c.p[ct.type];
        const int nkb = nkb_of(ct);
        const int K = ct.ti.g < E ? p.K_r : p.K_s;
        const int cols = ct.type == 0 ? pair_tile_cols<EPI_SWIGLU>(p, ct.ti) : pair_tile_cols<EPI_STORE>(p, ct.ti);
        const uint32_t idesc = umma_idesc_bf16(kPairM, (uint32_t)cols);
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
            const int nk = slice_k16(K, kb);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              if (k < nk) umma_bf16_pair(d, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
            umma_commit_pair_mc(&empty[s], 0x3);
            if (kb == nkb - 1) umma_commit_pair_mc(&tfull[acc], 0x3);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 2 || warp == 3) {
    // ---------------------------------------------------------------- cp.async gather (gate/up, routed)
    const int part = warp - 2;
    uint32_t it = 0;
    for (int i = 0;; ++i) {
      const int tile = next_tile(i);
      if (tile < 0) break;
      const CTile ct = decode(tile);
      const bool gather = ct.type == 0 && ct.ti.g < E;
      const int nkb = nkb_of(ct);
      int tok[kGatherRows];
      if (gather) gather_ids(p0, s_row0[ct.ti.g], s_rows[ct.ti.g], ct.ti.m * kPairM + (int)rank * kHalfM, part, tok);
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % kStages;
        mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
        if (gather) gather_a_cp(smem + s * kStageBytes, p0, tok, kb, part);
        cp_async_mbar_arrive_noinc(&afull[s]);
      }
    }
  } else if (warp == 8) {
    // ---------------------------------------------------------------- gather relay
    if (lane_id() == 0) {
      const uint32_t full_leader0 = mapa(smem_u32(&full[0]), 0);
      uint32_t it = 0;
      for (int i = 0;; ++i) {
        const int tile = read_tile(i);
        if (tile >= -1) release_tile(i);
        if (tile < 0) break;
        const int nkb = nkb_of(decode(tile));
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kStages;
          mbar_wait(&afull[s], (it / kStages) & 1);
          fence_proxy_async_smem();
          mbar_arrive_cluster(full_leader0 + s * 8);
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const uint32_t tempty_leader0 = mapa(smem_u32(&tempty[0]), 0);
    const uint32_t stage_out = smem_u32(s_out) + q * kStageOutBytes;
    const uint64_t pol_store = policy_evict_first();
    uint32_t tc = 0;
    for (int i = 0;; ++i, ++tc) {
      const int tile = next_tile(i);
      if (tile < 0) break;
      const CTile ct = decode(tile);
      const TileInfo& ti = ct.ti;
      const Params& p = c.p[ct.type];
      const uint32_t acc = tc & 1, aph = (tc >> 1) & 1;
      const float* sc = ct.type == 0
                            ? stage_tile_scales<EPI_SWIGLU>(p, ti, s_scales, tc, (int)threadIdx.x - 128)
                            : stage_tile_scales<EPI_STORE>(p, ti, s_scales, tc, (int)threadIdx.x - 128);
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int r_warp = ti.m * kPairM + (int)rank * kHalfM + q * 32;
      const bool routed = ti.g < E;
      const CUtensorMap* tmo = routed ? &mp.o_r[ct.type] : &mp.o_s[ct.type];
      const uint32_t taddr = tmem + acc * kBN + lane_base;
      if (ct.type == 0) {
        const int half = pair_tile_cols<EPI_SWIGLU>(p, ti) / 2;
        if (r_warp + 32 <= s_rows[ti.g]) {
          epilogue_tma<EPI_SWIGLU>(p, taddr, ti, half, sc, tmo, stage_out, s_row0[ti.g] + r_warp, c.act_hint == 2,
                                   pol_store);
        } else {
          const int r_local = r_warp + (int)lane_id();
          epilogue_slice<EPI_SWIGLU>(p, taddr, ti, r_local < s_rows[ti.g], (int64_t)s_row0[ti.g] + r_local, half,
                                     sc);
        }
      } else {
        const int half = pair_tile_cols<EPI_STORE>(p, ti) / 2;
        if (r_warp + 32 <= s_rows[ti.g]) {
          epilogue_tma<EPI_STORE, 2>(p, taddr, ti, half, sc, tmo, stage_out, s_row0[ti.g] + r_warp, true, pol_store);
        } else {
          const int r_local = r_warp + (int)lane_id();
          epilogue_slice<EPI_STORE>(p, taddr, ti, r_local < s_rows[ti.g], (int64_t)s_row0[ti.g] + r_local, half,
                                    sc);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive_cluster(tempty_leader0 + acc * 8);
      if (ct.type == 0) {
        // publish this warp's act rows of the m-tile: its TMA stores complete, then every lane's own
        // stores (the per-thread tail path) ordered before the release
        if (lane_id() == 0) {
          bulk_wait_group0();
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        __threadfence();
        __syncwarp();
        if (lane_id() == 0) atomicAdd(c.ready + s_mtb[ti.g] + ti.m, 1);
      }
    }
    if (lane_id() == 0) bulk_wait_group0();
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) tmem_dealloc_pair<512>(tmem);
}
}  // namespace

cudaError_t launch_gemm_chain(const CUtensorMap& a_r0, const CUtensorMap& a_s0, const CUtensorMap& b_r0,
                              const CUtensorMap& b_s0, const CUtensorMap& a_r1, const CUtensorMap& a_s1,
                              const CUtensorMap& b_r1, const CUtensorMap& b_s1, const GemmArgs& g0,
                              const GemmArgs& g1, const ChainArgs& ca, cudaStream_t st) {
  if (g0.bm != 256 || g0.n_groups > kMaxGroups - 1 || !ca.tile_ctr || !g0.gather_idx || !g0.gather_cp)
    return cudaErrorInvalidValue;
  ChainMaps mp;
  ChainParams c;
  c.p[0] = make_params(g0);
  c.p[1] = make_params(g1);
  c.sched_c = ca.sched_c;
  c.mt_base = ca.mt_base;
  c.ready = ca.ready;
  c.D = ca.D;
  c.act_hint = 1;
  auto omap = [](CUtensorMap* m, void* base, int64_t rows, int N, int64_t ld) {
    return make_tmap_2d(m, base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)rows, (uint64_t)N, (uint64_t)ld * 2, 64,
                        32, CU_TENSOR_MAP_SWIZZLE_128B);
  };
  const GemmArgs* gs[2] = {&g0, &g1};
  for (int t = 0; t < 2; ++t) {
    const GemmArgs& g = *gs[t];
    if (!omap(&mp.o_r[t], g.out_r, g.rows_r, g.N_r, g.ld_r)) return cudaErrorInvalidValue;
    mp.o_s[t] = mp.o_r[t];
    if (g.n_groups > g.E && !omap(&mp.o_s[t], g.out_s, g.rows_s, g.N_s, g.ld_s)) return cudaErrorInvalidValue;
  }
  mp.a_r[0] = a_r0;
  mp.a_s[0] = a_s0;
  mp.b_r[0] = b_r0;
  mp.b_s[0] = b_s0;
  mp.a_r[1] = a_r1;
  mp.a_s[1] = a_s1;
  mp.b_r[1] = b_r1;
  mp.b_s[1] = b_s1;
  cudaError_t e = cudaFuncSetAttribute(chained_gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kSmemBytes);
  if (e != cudaSuccess) return e;
  chained_gemm_pair_kernel<<<(g0.grid / 2) * 2, kChainThreads, kSmemBytes, st>>>(mp, c, ca.tile_ctr);
  return cudaGetLastError();
}

}  // namespace flux
