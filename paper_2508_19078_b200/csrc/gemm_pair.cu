// gemm_pair.cu — K3/K4/K5 grouped expert GEMMs on CTA pairs (tcgen05 cta_group::2).
//
// The expert FFNs of the quantized MoE model as grouped GEMMs: gate/up with the SwiGLU
// epilogue (act = bf16(SiLU(x·ŵgᵀ)·(x·ŵuᵀ)), R4) and down (o = bf16(act·ŵdᵀ)); groups 0..E-1 are the
// routed experts (A rows = the expert's D_e segment), group E the shared MLP (R5).  Each tile is 256 rows
// x 256 output columns computed by a cluster of two CTAs on the two SMs of a
// TPC: every CTA TMA-loads its own 128 A rows and its half (128 rows) of the
// 256-row B tile per 64-wide K slice; the leader CTA issues
// tcgen05.mma.cta_group::2 (M=256, N=256, K=16), which reads A and B from both
// CTAs' shared memory and writes each CTA's 128 accumulator rows to its own
// TMEM.  Versus a 1-CTA M=128 kernel (round 1, removed) this cuts the shared-memory operand traffic
// per MMA FLOP by a third (each SM stages 32 KB per K slice instead of 48 KB).
//
// Warp roles (per CTA): 0 = TMA producer (B halves; A when it comes by TMA), 1 = MMA issuer
// (leader CTA only), 2-3 = cp.async gather producers of the routed A rows (gate/up only; warp 2
// also allocates TMEM), 4-7 = epilogue (TMEM lane quadrant warp % 4), 8 = gather relay (gate/up
// only: the other epilogues launch 8 warps and keep 255 registers per thread).
//
// Synchronisation: full[s] lives in the leader (TMA bytes of both CTAs complete
// on it; the leader's producer arms it with the pair's byte count; with the
// cp.async gather it also takes one relay arrive per CTA); empty[s] and
// tfull[a] exist in both CTAs and are signalled by a multicast tcgen05.commit;
// afull[s] is CTA-local (64 cp.async noinc arrivals of the gather warps);
// tempty[a] lives in the leader and collects one arrive per epilogue warp of
// both CTAs.  The tile loop runs per cluster: tiles claimed in global order from an atomic counter
// (tid_full / tid_empty ring of claimed ids, see claim_tile / next_tile) or, with a null counter, the static
// round-robin over the 74 pairs.
#include "gemm_pair.cuh"

namespace flux {
namespace {
using namespace gemm;

__device__ __forceinline__ void unpack_bf16x8(const uint4& v, float (&f)[8]) {
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 x = __bfloat1622float2(b[i]);
    f[2 * i] = x.x;
    f[2 * i + 1] = x.y;
  }
}

// Fused K6 (EPI_COMBINE, the shared MLP's down GEMM; reading R6, same order and roundings as
// combine.cu): y[t] = bf16(r_t + bf16(acc_t) + Σ_j w_tj·y_perm[inv_pos_tj]) for this warp's 32 token
// rows x the tile's 256 columns.  Per tile each thread puts its row's picks (inv_pos, w) in the
// warp's 2 KB pick table; per 64-column chunk the warp writes o_sh = bf16(acc·scale) of its rows
// (one TMEM lane = one row per thread) into its 4 KB staging buffer (128-byte swizzle), then
// switches to 8 lanes per row: 4 rows per warp instruction, every load of y_perm and of the residual
// and every store of y a full 128-byte line, four row groups' loads in flight before the first FMA.
__device__ __forceinline__ void epilogue_combine(const Params& p, uint32_t taddr, const TileInfo& ti, const float* sc,
                                                 uint32_t stage, uint32_t picks, int r_warp, int rows_in_grp) {
  const int lane = (int)lane_id();
  const int H = p.N_s;
  const int k = p.k;
  {
    const int t = r_warp + lane;
    uint32_t pv[8], wv[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
      int pos = -1;
      float wt = 0.f;
      if (t < rows_in_grp && jj < k) {
        pos = __ldg(&p.inv_pos[(int64_t)t * k + jj]);  // -1: a pick folded by gate re-routing (NEXT-2)
        wt = __ldg(&p.topk_w[(int64_t)t * k + jj]);
      }
      pv[jj] = (uint32_t)pos;
      wv[jj] = __float_as_uint(wt);
    }
    const uint32_t row = picks + lane * 64;
    st_shared_v4(row, make_uint4(pv[0], pv[1], pv[2], pv[3]));
    st_shared_v4(row + 16, make_uint4(pv[4], pv[5], pv[6], pv[7]));
    st_shared_v4(row + 32, make_uint4(wv[0], wv[1], wv[2], wv[3]));
    st_shared_v4(row + 48, make_uint4(wv[4], wv[5], wv[6], wv[7]));
  }
  __nv_bfloat16* y = reinterpret_cast<__nv_bfloat16*>(p.out_s);
  const int chunk = lane & 7, sub = lane >> 3;
  const int n_chunks = min(kBN / 64, (H - ti.n * kBN) / 64);  // H % 64 == 0
  // phase 1 of chunk cc: o_sh of this thread's row -> staging row `lane`
  auto stage_chunk = [&](int cc) {
    float v0[16], v1[16], v2[16], v3[16];
    tmem_ld16(taddr + cc * 64, v0);
    tmem_ld16(taddr + cc * 64 + 16, v1);
    tmem_ld16(taddr + cc * 64 + 32, v2);
    tmem_ld16(taddr + cc * 64 + 48, v3);
    tmem_ld_wait();
    const uint32_t row_addr = stage + lane * 128;
    auto put = [&](float (&v)[16], int h) {
      if (sc) {
        float cs[16];
        lds16(sc + cc * 64 + 16 * h, cs);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] *= cs[i];
      }
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int c16 = 2 * h + c;
        st_shared_v4(row_addr + ((c16 ^ (lane & 7)) << 4),
                     make_uint4(pack_bf16x2(v[8 * c], v[8 * c + 1]), pack_bf16x2(v[8 * c + 2], v[8 * c + 3]),
                                pack_bf16x2(v[8 * c + 4], v[8 * c + 5]), pack_bf16x2(v[8 * c + 6], v[8 * c + 7])));
      }
    };
    put(v0, 0);
    put(v1, 1);
    put(v2, 2);
    put(v3, 3);
  };
  // phase 2 per chunk: 8 lanes per row, rows rr = 4·group + sub, 16-byte column chunk `chunk`; four
  // row groups' loads are issued before the first FMA (measured: 4.1 ms/layer for the fused shared
  // down + combine; two groups 4.3; two groups software-pipelined across chunks 4.9)
  __syncwarp();  // the pick table is visible to the whole warp
  constexpr int kRowsInFlight = 4;
  for (int cc = 0; cc < n_chunks; ++cc) {
    const int c0 = ti.n * kBN + cc * 64;
    stage_chunk(cc);
    __syncwarp();  // staging rows are visible to the whole warp
#pragma unroll 1
    for (int it = 0; it < 8; it += kRowsInFlight) {
      uint4 rv[kRowsInFlight], ov[kRowsInFlight][8];
      uint32_t live[kRowsInFlight];  // bit jj: pick jj has a y_perm row
#pragma unroll
      for (int u = 0; u < kRowsInFlight; ++u) {
        const int rr = 4 * (it + u) + sub;
        const int t = r_warp + rr;
        live[u] = 0;
        if (t < rows_in_grp) {
          rv[u] = __ldg(reinterpret_cast<const uint4*>(p.resid + (int64_t)t * H + c0) + chunk);
          const uint4 pa = ld_shared_v4(picks + rr * 64), pb = ld_shared_v4(picks + rr * 64 + 16);
          const int pj[8] = {(int)pa.x, (int)pa.y, (int)pa.z, (int)pa.w, (int)pb.x, (int)pb.y, (int)pb.z, (int)pb.w};
#pragma unroll
          for (int jj = 0; jj < 8; ++jj)
            if (jj < k && pj[jj] >= 0) {  // -1: a pick folded by gate re-routing (NEXT-2)
              ov[u][jj] = __ldg(reinterpret_cast<const uint4*>(p.y_perm + (int64_t)pj[jj] * H + c0) + chunk);
              live[u] |= 1u << jj;
            }
        }
      }
#pragma unroll
      for (int u = 0; u < kRowsInFlight; ++u) {
        const int rr = 4 * (it + u) + sub;
        const int t = r_warp + rr;
        if (t >= rows_in_grp) continue;
        const uint4 sv = ld_shared_v4(stage + rr * 128 + ((chunk ^ (rr & 7)) << 4));
        const uint4 wa = ld_shared_v4(picks + rr * 64 + 32), wb = ld_shared_v4(picks + rr * 64 + 48);
        const float wj[8] = {__uint_as_float(wa.x), __uint_as_float(wa.y), __uint_as_float(wa.z),
                             __uint_as_float(wa.w), __uint_as_float(wb.x), __uint_as_float(wb.y),
                             __uint_as_float(wb.z), __uint_as_float(wb.w)};
        float acc[8], f[8];
        unpack_bf16x8(rv[u], acc);
        unpack_bf16x8(sv, f);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += f[i];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
          if (live[u] & (1u << jj)) {
            unpack_bf16x8(ov[u][jj], f);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] = fmaf(wj[jj], f[i], acc[i]);
          }
        *(reinterpret_cast<uint4*>(y + (int64_t)t * H + c0) + chunk) =
            make_uint4(pack_bf16x2(acc[0], acc[1]), pack_bf16x2(acc[2], acc[3]), pack_bf16x2(acc[4], acc[5]),
                       pack_bf16x2(acc[6], acc[7]));
      }
    }
    __syncwarp();  // the staging buffer is rewritten by the next chunk
  }
}

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsOf<EPI>, 1)
    grouped_gemm_pair_kernel(const __grid_constant__ CUtensorMap tm_a_r, const __grid_constant__ CUtensorMap tm_a_s,
                             const __grid_constant__ CUtensorMap tm_b_r, const __grid_constant__ CUtensorMap tm_b_s,
                             const __grid_constant__ CUtensorMap tm_o_r, const __grid_constant__ CUtensorMap tm_o_s,
                             Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, still a shared-space pointer
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;  // [2]
  uint64_t* tempty = tfull + 2;       // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  uint64_t* afull = full + 24;        // [kStages] (byte 192): this CTA's cp.async-gathered A rows landed
  int32_t* s_sched = reinterpret_cast<int32_t*>(smem + kStages * kStageBytes + 256);
  int32_t* s_row0 = s_sched + kMaxGroups;
  int32_t* s_rows = s_row0 + kMaxGroups;
  // [128] gathered token ids, 16-byte aligned: byte 256 + 4·(3·kMaxGroups + 1) = 3344 past the 1 KB-aligned
  // ring end (pointer arithmetic on the shared array keeps LDS/STS instead of generic accesses)
  static_assert((256 + 4 * (3 * kMaxGroups + 1)) % 16 == 0, "s_idx alignment");
  int32_t* s_idx = s_rows + kMaxGroups + 1;
  float* s_scales = reinterpret_cast<float*>(s_idx + 128);  // [2][kScaleFloats] (stage_tile_scales)
  uint8_t* s_out = smem + kStages * kStageBytes + kMiscBytes;  // [4 warps][kStageOutBytes]
  uint64_t* tid_full = reinterpret_cast<uint64_t*>(s_out + 4 * kStageOutBytes + 4 * kPickBytes);  // [kTileSlots]
  uint64_t* tid_empty = tid_full + kTileSlots;  // [kTileSlots], the leader's are the ones used
  int32_t* s_tid = reinterpret_cast<int32_t*>(tid_empty + kTileSlots);  // [kTileSlots]

  ClockProbe probe;
  probe.start(p.clk_probe);
  const int warp = warp_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  constexpr int kThreads = kThreadsOf<EPI>;
  for (int i = threadIdx.x; i <= p.n_groups; i += kThreads) s_sched[i] = p.sched[i];
  for (int i = threadIdx.x; i < p.n_groups; i += kThreads) {
    s_row0[i] = p.grp_row0[i];
    s_rows[i] = p.grp_rows[i];
  }
  // cp.async gather: full[s] also waits for one relay arrive per CTA (its A rows landed and were
  // made visible to the async proxy), on top of the leader's expect_tx arrive
  const bool cpg = EPI == EPI_SWIGLU && p.gather_idx != nullptr && p.gather_cp;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], cpg ? 3 : 1);
      mbar_init(&empty[s], 1);
      mbar_init(&afull[s], 32 * kGatherParts);
    }
    // tile-id consumers per slot, both CTAs: warp 0 of CTA 1, the MMA warp of CTA 0, 4 + 4 epilogue
    // warps, and with the cp.async gather 2 + 2 gather warps and 2 relays
    for (int s = 0; s < kTileSlots; ++s) {
      mbar_init(&tid_full[s], 1);
      mbar_init(&tid_empty[s], 10 + (cpg ? 6 : 0));
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
  const int total = s_sched[p.n_groups];
  const int nkb_r = (p.K_r + kBK - 1) / kBK, nkb_s = (p.K_s + kBK - 1) / kBK;
  const int cid = (int)cluster_id_x(), ncl = (int)ncluster_x();
  // The pair's tile sequence: static round-robin (tile i of this pair = cid + i·ncl), or, with
  // p.tile_ctr, claimed in global order by the leader's producer warp (atomicAdd) and published to
  // every role of both CTAs through a ring of tile ids — concurrent pairs then always work on
  // neighbouring tiles (the n-tiles of one m-tile together), however far their speeds drift.
  const bool dyn = p.tile_ctr != nullptr;
  // Publishing: the leader writes the id into its ring and arrives on its tid_full, and st.async's
  // it into CTA 1's ring, completing 4 transaction bytes on CTA 1's tid_full (no memory barrier on
  // the publishing warp, which also issues the TMA loads).
  auto read_tile = [&](int i) -> int {  // one lane: the i-th tile id published to this CTA
    const int slot = i % kTileSlots;
    mbar_wait(&tid_full[slot], (i / kTileSlots) & 1);  // CTA 1: completed by the peer's st.async
    return *reinterpret_cast<volatile int32_t*>(&s_tid[slot]);
  };
  // Called once the id read by read_tile(i) has been consumed (so the load has completed): frees the
  // slot.  A plain arrive (no cluster-scope release: that would be a MEMBAR draining every in-flight
  // cp.async of the gather warps at each tile boundary).
  auto release_tile = [&](int i) {
    const int slot = i % kTileSlots;
    if (leader)
      mbar_arrive(&tid_empty[slot]);
    else
      mbar_arrive_cluster(mapa(smem_u32(&tid_empty[slot]), 0));
  };
  auto next_tile = [&](int i) -> int {  // whole warp; -1 = done
    if (!dyn) {
      const int t = cid + i * ncl;
      return t < total ? t : -1;
    }
    int t = 0;
    if (lane_id() == 0) t = read_tile(i);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (lane_id() == 0) release_tile(i);
    return t;
  };
  // Leader's warp 0 (lane 0) publishes one tile ahead: at iteration i it publishes tile i + 1 (so
  // CTA 1's producer learns it while both CTAs still load tile i — publishing at the tile boundary
  // cost ~7%) and claims tile i + 2, whose atomic round trip overlaps this tile's loads.
  int cur = 0, pending = 0;
  auto claim = [&]() -> int {
    const int c = atomicAdd(p.tile_ctr, 1);
    return c < total ? c : -1;
  };
  auto publish = [&](int i, int t) {
    const int slot = i % kTileSlots;
    mbar_wait(&tid_empty[slot], ((i / kTileSlots) & 1) ^ 1);  // every consumer has read slot's last id
    s_tid[slot] = t;
    mbar_arrive(&tid_full[slot]);
    const uint32_t peer_full = mapa(smem_u32(&tid_full[slot]), 1);
    mbar_arrive_expect_tx_cluster(peer_full, 4);
    st_async_u32(mapa(smem_u32(&s_tid[slot]), 1), (uint32_t)t, peer_full);
  };
  if (dyn && leader && warp == 0 && lane_id() == 0) {
    cur = claim();
    publish(0, cur);
    pending = cur >= 0 ? claim() : -1;
  }
  auto claim_tile = [&](int i) -> int {  // whole warp 0 of the leader: the i-th tile of this pair
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
    // whole warp: it stages gathered row ids; lane 0 issues the TMA
    if (lane_id() == 0) {
      tma_prefetch(&tm_a_r);
      tma_prefetch(&tm_b_r);
      tma_prefetch(&tm_a_s);
      tma_prefetch(&tm_b_s);
    }
    const uint64_t pol_a = policy_evict_first(), pol_b = policy_evict_last();
    uint32_t it = 0;
    for (int i = 0;; ++i) {
      const int tile = dyn && leader ? claim_tile(i) : next_tile(i);
      if (tile < 0) break;
      const TileInfo ti = decode(tile, s_sched, p.n_groups, p.n_tiles_r, p.n_tiles_s, p.E);
      const bool routed = ti.g < p.E;
      const bool gather = routed && p.gather_idx != nullptr;
      const int first = ti.m * kPairM + (int)rank * kHalfM;
      const int arow = s_row0[ti.g] + first;
      // CTA 1's half starts at the tile's second half of B rows: the up features (gate/up layout)
      // or output column cols/2 (a trimmed last tile reads cols/2 rows from each CTA)
      const int half = EPI == EPI_SWIGLU ? kBN / 2 : pair_tile_cols<EPI>(p, ti) / 2;
      const int brow = (routed ? ti.g * p.b_rows_r : 0) + ti.n * kBN + (int)rank * half;
      const CUtensorMap* ta = routed ? &tm_a_r : &tm_a_s;
      const CUtensorMap* tb = routed ? &tm_b_r : &tm_b_s;
      const int nkb = routed ? nkb_r : nkb_s;
      if (gather && !cpg) stage_gather_rows(s_idx, p, s_row0[ti.g], s_rows[ti.g], first);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = (it + kb) % kStages;
        const uint32_t ph = ((it + kb) / kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * kStageBytes;
        const bool a_cp = cpg && gather;  // A rows by cp.async: only the B halves are TMA bytes
        if (leader && lane_id() == 0) mbar_arrive_expect_tx(&full[s], a_cp ? 2 * kBBytes : 2 * kStageBytes);
        __syncwarp();  // the transaction count is armed before any of this warp's copies can land
        if (!a_cp) {
          if ((p.l2_hints & 4) && !gather) {
            if (lane_id() == 0) tma_load_2d_pair_hint(st, ta, &full[s], kb * kBK, arow, pol_a);
          } else {
            load_a_pair(st, ta, &full[s], kb, arow, gather, s_idx);  // else: warps 2 and 3
          }
        }
        if (lane_id() == 0) {
          if (p.l2_hints & 2)
            tma_load_2d_pair_hint(st + kABytes, tb, &full[s], kb * kBK, brow, pol_b);
          else
            tma_load_2d_pair(st + kABytes, tb, &full[s], kb * kBK, brow);
        }
      }
      it += nkb;
      __syncwarp();  // s_idx is rewritten for the next tile only after this one was issued
    }
  } else if (warp == 1) {
    if (leader) {
      uint32_t it = 0, tc = 0;
      for (int i = 0;; ++i, ++tc) {
        const int tile = next_tile(i);
        if (tile < 0) break;
        const TileInfo ti = decode(tile, s_sched, p.n_groups, p.n_tiles_r, p.n_tiles_s, p.E);
        const int nkb = ti.g < p.E ? nkb_r : nkb_s;
        const int K = ti.g < p.E ? p.K_r : p.K_s;
        const uint32_t idesc = umma_idesc_bf16(kPairM, (uint32_t)pair_tile_cols<EPI>(p, ti));
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
    // cp.async gather producers (warp 2: rows 0..63 of this CTA's half, warp 3: rows 64..127);
    // every lane arrives on afull every stage (at once for stages whose A comes by TMA)
    if (cpg) {
      const int part = warp - 2;
      uint32_t it = 0;
      for (int i = 0;; ++i) {
        const int tile = next_tile(i);
        if (tile < 0) break;
        const TileInfo ti = decode(tile, s_sched, p.n_groups, p.n_tiles_r, p.n_tiles_s, p.E);
        const bool gather = ti.g < p.E;
        const int nkb = gather ? nkb_r : nkb_s;
        int tok[kGatherRows];
        if (gather) gather_ids(p, s_row0[ti.g], s_rows[ti.g], ti.m * kPairM + (int)rank * kHalfM, part, tok);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kStages;
          mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
          if (gather) gather_a_cp(smem + s * kStageBytes, p, tok, kb, part);
          cp_async_mbar_arrive_noinc(&afull[s]);
        }
      }
    }
  } else if (warp == 8) {
    // cp.async gather relay: once this CTA's gathered rows of stage s have landed, make them visible
    // to the async proxy (tcgen05.mma reads them) and arrive on the leader's full[s]
    if (cpg && lane_id() == 0) {
      const uint32_t full_leader0 = mapa(smem_u32(&full[0]), 0);
      uint32_t it = 0;
      for (int i = 0;; ++i) {
        int tile = cid + i * ncl < total ? cid + i * ncl : -1;
        if (dyn) {
          tile = read_tile(i);
          if (tile >= -1) release_tile(i);  // (always true: makes the release depend on the loaded id)
        }
        if (tile < 0) break;
        const TileInfo ti = decode(tile, s_sched, p.n_groups, p.n_tiles_r, p.n_tiles_s, p.E);
        const int nkb = ti.g < p.E ? nkb_r : nkb_s;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kStages;
          mbar_wait(&afull[s], (it / kStages) & 1);
          fence_proxy_async_smem();
          mbar_arrive_cluster(full_leader0 + s * 8);
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const uint32_t tempty_leader0 = mapa(smem_u32(&tempty[0]), 0);
    const uint32_t stage_out = smem_u32(s_out) + q * kStageOutBytes;
    const uint64_t pol_store = policy_evict_first();
    uint32_t tc = 0;
    for (int i = 0;; ++i, ++tc) {
      const int tile = next_tile(i);
      if (tile < 0) break;
      const TileInfo ti = decode(tile, s_sched, p.n_groups, p.n_tiles_r, p.n_tiles_s, p.E);
      const uint32_t acc = tc & 1, aph = (tc >> 1) & 1;
      const float* sc = stage_tile_scales<EPI>(p, ti, s_scales, tc, (int)threadIdx.x - 128);
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int r_warp = ti.m * kPairM + (int)rank * kHalfM + q * 32;  // this warp's first row in the group
      const int half = pair_tile_cols<EPI>(p, ti) / 2;
      if constexpr (EPI == EPI_COMBINE) {
        epilogue_combine(p, tmem + acc * kBN + lane_base, ti, sc, stage_out,
                         smem_u32(s_out) + 4 * kStageOutBytes + q * kPickBytes, r_warp, s_rows[ti.g]);
      } else if (r_warp + 32 <= s_rows[ti.g]) {
        epilogue_tma<EPI>(p, tmem + acc * kBN + lane_base, ti, half, sc, ti.g < p.E ? &tm_o_r : &tm_o_s,
                          stage_out, s_row0[ti.g] + r_warp, (p.l2_hints & 1) != 0, pol_store);
      } else {  // a group's last rows (masked per thread) and the fused combine
        const int r_local = r_warp + (int)lane_id();
        epilogue_slice<EPI>(p, tmem + acc * kBN + lane_base, ti, r_local < s_rows[ti.g],
                            (int64_t)s_row0[ti.g] + r_local, half, sc);
      }
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive_cluster(tempty_leader0 + acc * 8);
    }
    if (lane_id() == 0) bulk_wait_group0();  // every TMA store of this warp is complete
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) tmem_dealloc_pair<512>(tmem);
  probe.stop(p.clk_probe);
}
}  // namespace

cudaError_t launch_gemm(GemmEpi epi, const CUtensorMap& a_r, const CUtensorMap& a_s, const CUtensorMap& b_r,
                        const CUtensorMap& b_s, const GemmArgs& g, cudaStream_t st) {
  if (g.bm != 256 || g.n_groups > kMaxGroups - 1) return cudaErrorInvalidValue;
  const Params p = make_params(g);
  // output tensor maps of the TMA-store epilogue: bf16 [rows][N], row stride ld, 32x64 boxes
  CUtensorMap o_r, o_s;
  auto omap = [](CUtensorMap* m, void* base, int64_t rows, int N, int64_t ld) {
    return make_tmap_2d(m, base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)rows, (uint64_t)N, (uint64_t)ld * 2, 64,
                        32, CU_TENSOR_MAP_SWIZZLE_128B);
  };
  if (epi != EPI_COMBINE) {
    if (!omap(&o_r, g.out_r, g.rows_r, g.N_r, g.ld_r)) return cudaErrorInvalidValue;
    o_s = o_r;
    if (g.n_groups > g.E && !omap(&o_s, g.out_s, g.rows_s, g.N_s, g.ld_s)) return cudaErrorInvalidValue;
  } else {
    o_r = a_r;  // unused by the fused-combine epilogue
    o_s = a_r;
  }
  auto kern = epi == EPI_SWIGLU  ? grouped_gemm_pair_kernel<EPI_SWIGLU>
              : epi == EPI_STORE ? grouped_gemm_pair_kernel<EPI_STORE>
                                 : grouped_gemm_pair_kernel<EPI_COMBINE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  if (e != cudaSuccess) return e;
  const int threads = epi == EPI_SWIGLU ? kThreadsOf<EPI_SWIGLU> : kThreadsOf<EPI_STORE>;
  kern<<<(g.grid / 2) * 2, threads, kSmemBytes, st>>>(a_r, a_s, b_r, b_s, o_r, o_s, p);
  return cudaGetLastError();
}

}  // namespace flux
