// gemm_pair_q.cu — K3/K4/K5 with the weight dequantization fused into the
// GEMM (the quantized expert FFNs of the profiling model; weight
// format R1, dequantized value R1b).
//
// CTA-pair tiles of 256 rows x 256 output columns as in gemm_pair.cu, but the
// B operand is produced on chip from the quantized weights:
//   * the producer warp TMA-loads this CTA's 128 A rows (bf16, SW128) and the
//     raw quantized bytes of its 128 B rows for the K slice (INT4: 32 B/row,
//     INT8: 64 B/row) into the same ring stage;
//   * eight dequant warps (two threads per B row) read the raw codes, convert in
//     registers — INT4: XOR 0x8 to offset binary, OR into the mantissa of the
//     bf16 128.0 (exact 136+q), subtract 136 (exact q), multiply by bf16(s)
//     with a single rounding = bf16(q·bf16(s)) (R1b); INT8: the same through
//     the fp32 2^23 magic; per-channel codes stay exact and the scale is
//     applied to the fp32 accumulator in the epilogue — and write the
//     128-byte-swizzled K-major B rows the MMA descriptor expects;
//   * they fence the generic->async proxy and arrive on the leader's full
//     barrier, which also counts the A bytes of both CTAs;
//   * the leader issues tcgen05.mma.cta_group::2 M=256 N=256 K=16.
// For gate/up, CTA 0 dequantizes the 128 gate rows and CTA 1 the matching 128
// up rows, so each accumulator row holds g and u of the same features and the
// SwiGLU epilogue is unchanged.
#include "gemm_common.cuh"

namespace flux {
namespace {
using namespace gemm;

constexpr int kHalfM = 128, kPairM = 256;
constexpr int kABytes = kHalfM * kBK * 2;     // 16 KB
constexpr int kBBytes = (kBN / 2) * kBK * 2;  // 16 KB (bf16 B half, written by the dequant warps)
constexpr int kThreads = 512;  // 0 TMA, 1 MMA, 2 TMEM, 3 idle, 4-7 epilogue, 8-15 dequant
template <int WB>
struct Cfg {
  static constexpr int kRawRow = WB == 4 ? 32 : 64;  // raw bytes of one B row per K slice
  static constexpr int kRawBytes = 128 * kRawRow;
  static constexpr int kStageBytes = kABytes + kBBytes;  // A/B ring (consumed by the MMA)
  static constexpr int kStages = 5;
  static constexpr int kRawStages = WB == 4 ? 10 : 5;   // raw-code ring (consumed by the dequant warps)
  static constexpr int kSmemBytes =
      kStages * kStageBytes + kRawStages * kRawBytes + 1024 + 512 + 3 * kMaxGroups * 4 + 64 + 128 * 4 + 16 + kScaleSmemBytes;
};
constexpr int kScalePrefetch = 4;  // K slices of group scales kept in flight per dequant thread

struct QParams {
  Params p;
  int wbits, gsz, gate_up;
  int qrows_r, qrows_s;
  long long qtotal_r, qtotal_s;
  const float *gs_r0, *gs_r1, *gs_s0, *gs_s1;
};

template <int EPI, int WB, bool GROUPED>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    grouped_gemm_pair_q_kernel(const __grid_constant__ CUtensorMap tm_a_r, const __grid_constant__ CUtensorMap tm_a_s,
                               const __grid_constant__ CUtensorMap tm_q_r0,
                               const __grid_constant__ CUtensorMap tm_q_r1,
                               const __grid_constant__ CUtensorMap tm_q_s0,
                               const __grid_constant__ CUtensorMap tm_q_s1, QParams qp) {
  const Params& p = qp.p;
  constexpr int kRawRow = Cfg<WB>::kRawRow;
  constexpr int kRawTx = Cfg<WB>::kRawBytes;
  constexpr int kStages = Cfg<WB>::kStages;
  constexpr int kRawStages = Cfg<WB>::kRawStages;
  constexpr int kStageBytes = Cfg<WB>::kStageBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, still a shared-space pointer
  uint8_t* raw_ring = smem + kStages * kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(raw_ring + kRawStages * kRawTx);  // leader: A bytes + dequant arrivals
  uint64_t* empty = full + kStages;                                             // both: MMA done with A/B stage
  uint64_t* rawf = empty + kStages;                                             // local: raw codes landed
  uint64_t* rawe = rawf + kRawStages;                                           // local: dequant warps read them
  uint64_t* tfull = rawe + kRawStages;                                          // [2]
  uint64_t* tempty = tfull + 2;                                                 // [2] leader
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int32_t* s_sched = reinterpret_cast<int32_t*>(raw_ring + kRawStages * kRawTx + 512);
  int32_t* s_row0 = s_sched + kMaxGroups;
  int32_t* s_rows = s_row0 + kMaxGroups;
  // [128] gathered token ids, 16-byte aligned: byte 256 + 4·(3·kMaxGroups + 1) = 3344 past the 1 KB-aligned
  // ring end (pointer arithmetic on the shared array keeps LDS/STS instead of generic accesses)
  static_assert((256 + 4 * (3 * kMaxGroups + 1)) % 16 == 0, "s_idx alignment");
  int32_t* s_idx = s_rows + kMaxGroups + 1;
  float* s_scales = reinterpret_cast<float*>(s_idx + 128);  // [2][kScaleFloats] (stage_tile_scales)

  const int warp = warp_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  for (int i = threadIdx.x; i <= p.n_groups; i += kThreads) s_sched[i] = p.sched[i];
  for (int i = threadIdx.x; i < p.n_groups; i += kThreads) {
    s_row0[i] = p.grp_row0[i];
    s_rows[i] = p.grp_rows[i];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1 + 16);  // leader producer + 8 dequant warps x 2 CTAs
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < kRawStages; ++s) {
      mbar_init(&rawf[s], 1);
      mbar_init(&rawe[s], 8);  // the 8 dequant warps of this CTA
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
  // Tile order: n fastest inside a group.  An m-fastest order (consecutive pairs share the B n-tile, so
  // its raw codes come from L2) measured no faster (42.9 / 43.1 vs 42.4 / 41.8 ms per
  // DeepSeek layer): every tile still dequantizes its own B tile in shared memory.
  auto decode_q = [&](int tile) -> TileInfo {
    return decode(tile, s_sched, p.n_groups, p.n_tiles_r, p.n_tiles_s, p.E);
  };

  // B row (in the quantized tensor of this CTA's source) of a tile's first row
  auto qrow_of = [&](const TileInfo& ti) -> int {
    const bool routed = ti.g < p.E;
    const int grp_base = routed ? ti.g * qp.qrows_r : 0;
    // STORE: CTA 1 holds output columns [cols/2, cols) of the tile (pair_tile_cols)
    return qp.gate_up ? grp_base + ti.n * (kBN / 2)
                      : grp_base + ti.n * kBN + (int)rank * (pair_tile_cols<EPI>(p, ti) / 2);
  };

  if (warp == 0) {
    // ------------------------------------------------------------ A producer (ring freed by the MMA)
    if (lane_id() == 0) {
      tma_prefetch(&tm_a_r);
      tma_prefetch(&tm_a_s);
    }
    uint32_t it = 0;
    for (int tile = cid; tile < total; tile += ncl) {
      const TileInfo ti = decode_q(tile);
      const bool routed = ti.g < p.E;
      const bool gather = routed && p.gather_idx != nullptr;
      const int first = ti.m * kPairM + (int)rank * kHalfM;
      const int arow = s_row0[ti.g] + first;
      const CUtensorMap* ta = routed ? &tm_a_r : &tm_a_s;
      const int nkb = routed ? nkb_r : nkb_s;
      if (gather) stage_gather_rows(s_idx, p, s_row0[ti.g], s_rows[ti.g], first);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = (it + kb) % kStages;
        const uint32_t ph = ((it + kb) / kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        if (leader && lane_id() == 0) mbar_arrive_expect_tx(&full[s], 2 * kABytes);
        __syncwarp();
        load_a_pair(smem + s * kStageBytes, ta, &full[s], kb, arow, gather, s_idx);
      }
      it += nkb;
      __syncwarp();
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ raw-code producer (ring freed by dequant)
    if (elect_one()) {
      const CUtensorMap* q_r = rank == 0 || !qp.gate_up ? &tm_q_r0 : &tm_q_r1;
      const CUtensorMap* q_s = rank == 0 || !qp.gate_up ? &tm_q_s0 : &tm_q_s1;
      tma_prefetch(q_r);
      tma_prefetch(q_s);
      uint32_t it = 0;
      for (int tile = cid; tile < total; tile += ncl) {
        const TileInfo ti = decode_q(tile);
        const bool routed = ti.g < p.E;
        const int qrow = qrow_of(ti);
        const CUtensorMap* tq = routed ? q_r : q_s;
        const int nkb = routed ? nkb_r : nkb_s;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kRawStages;
          const uint32_t ph = (it / kRawStages) & 1;
          mbar_wait(&rawe[s], ph ^ 1);
          mbar_arrive_expect_tx(&rawf[s], kRawTx);
          tma_load_2d(raw_ring + s * kRawTx, tq, &rawf[s], kb * kRawRow, qrow);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader)
    if (leader) {
      uint32_t it = 0, tc = 0;
      for (int tile = cid; tile < total; tile += ncl, ++tc) {
        const TileInfo ti = decode_q(tile);
        const int nkb = ti.g < p.E ? nkb_r : nkb_s;
        const int K = ti.g < p.E ? p.K_r : p.K_s;
        const uint32_t idesc = umma_idesc_bf16(kPairM, (uint32_t)pair_tile_cols<EPI>(p, ti));
        const uint32_t acc = tc & 1, aph = (tc >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);  // CTA-scope acquire: a cluster-scope one invalidates L1
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
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const uint32_t tempty_leader0 = mapa(smem_u32(&tempty[0]), 0);
    uint32_t tc = 0;
    for (int tile = cid; tile < total; tile += ncl, ++tc) {
      const TileInfo ti = decode_q(tile);
      const uint32_t acc = tc & 1, aph = (tc >> 1) & 1;
      const float* sc = stage_tile_scales<EPI>(p, ti, s_scales, tc, (int)threadIdx.x - 128);
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int r_local = ti.m * kPairM + (int)rank * kHalfM + q * 32 + (int)lane_id();
      epilogue_slice<EPI>(p, tmem + acc * kBN + lane_base, ti, r_local < s_rows[ti.g],
                          (int64_t)s_row0[ti.g] + r_local, pair_tile_cols<EPI>(p, ti) / 2, sc);
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive_cluster(tempty_leader0 + acc * 8);
    }
  } else if (warp >= 8) {
    // ------------------------------------------------------------ dequant (both CTAs)
    // 8 warps, two threads per B row: thread dt owns half `hf` (32 K values) of row `r`, so raw
    // loads are contiguous across the warp and the swizzled 16-byte stores of 8 consecutive
    // threads hit 8 distinct bank groups (conflict-free).
    const int dt = threadIdx.x - 256;  // 0..255
    const int r = dt >> 1, hf = dt & 1;
    const uint32_t full_leader0 = mapa(smem_u32(&full[0]), 0);
    const float* gs_r = rank == 0 || !qp.gate_up ? qp.gs_r0 : qp.gs_r1;
    const float* gs_s = rank == 0 || !qp.gate_up ? qp.gs_s0 : qp.gs_s1;
    const int kb_per_group = GROUPED ? qp.gsz / kBK : 1;
    const uint32_t sw = r & 7;
    const uint32_t smem_base = smem_u32(smem);
    const uint32_t raw_base = smem_u32(raw_ring);
    uint32_t it = 0;
    for (int tile = cid; tile < total; tile += ncl) {
      const TileInfo ti = decode_q(tile);
      const bool routed = ti.g < p.E;
      const int nkb = routed ? nkb_r : nkb_s;
      const int K = routed ? p.K_r : p.K_s;
      const long long row = (long long)qrow_of(ti) + r;
      const bool row_ok = row < (routed ? qp.qtotal_r : qp.qtotal_s);
      const int n_grp = GROUPED ? K / qp.gsz : 1;
      const float* srow = (routed ? gs_r : gs_s) + (GROUPED && row_ok ? row * n_grp : 0);
      // group scales: the next kScalePrefetch groups stay in flight (L1 is mostly shared memory here)
      float pre[kScalePrefetch];
#pragma unroll
      for (int i = 0; i < kScalePrefetch; ++i) pre[i] = (GROUPED && row_ok && i < n_grp) ? __ldg(&srow[i]) : 0.f;
      int in_grp = 0, next_grp = kScalePrefetch;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % kStages;
        const uint32_t ph = (it / kStages) & 1;
        const int rs = it % kRawStages;
        const uint32_t rph = (it / kRawStages) & 1;
        const float sc = GROUPED ? __bfloat162float(__float2bfloat16_rn(pre[0])) : 0.f;
        if (GROUPED && ++in_grp == kb_per_group) {  // advance to the next group after its last K slice
          in_grp = 0;
#pragma unroll
          for (int i = 0; i < kScalePrefetch - 1; ++i) pre[i] = pre[i + 1];
          pre[kScalePrefetch - 1] = (row_ok && next_grp < n_grp) ? __ldg(&srow[next_grp]) : 0.f;
          ++next_grp;
        }
        // 1) raw codes of this K slice -> registers (converted), then release the raw slot
        mbar_wait(&rawf[rs], rph);
        const uint32_t rbase = raw_base + rs * kRawTx;
        uint4 outv[4];
        if constexpr (WB == 4) {
          const uint4 v = ld_shared_v4(rbase + dt * 16);
          const uint32_t wds[4] = {v.x, v.y, v.z, v.w};
          const __nv_bfloat162 s2 = __floats2bfloat162_rn(sc, sc);
#pragma unroll
          for (int i = 0; i < 4; ++i) outv[i] = deq_int4x8<GROUPED>(wds[i], s2);
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint4 v = ld_shared_v4(rbase + dt * 32 + 16 * h);
            const uint2 a0 = deq_int8x4<GROUPED>(v.x, sc), a1 = deq_int8x4<GROUPED>(v.y, sc);
            const uint2 a2 = deq_int8x4<GROUPED>(v.z, sc), a3 = deq_int8x4<GROUPED>(v.w, sc);
            outv[2 * h] = make_uint4(a0.x, a0.y, a1.x, a1.y);
            outv[2 * h + 1] = make_uint4(a2.x, a2.y, a3.x, a3.y);
          }
        }
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&rawe[rs]);
        // 2) the B slot is free once the MMA has consumed it (same phase the A producer waits for)
        mbar_wait(&empty[s], ph ^ 1);
        const uint32_t brow = smem_base + s * kStageBytes + kABytes + r * 128;
#pragma unroll
        for (int i = 0; i < 4; ++i) st_shared_v4(brow + (((uint32_t)(hf * 4 + i) ^ sw) << 4), outv[i]);
        fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the tensor core (async proxy)
        __syncwarp();
        if (lane_id() == 0) mbar_arrive_cluster(full_leader0 + s * 8);
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) tmem_dealloc_pair<512>(tmem);
}
}  // namespace

cudaError_t launch_gemm_q(GemmEpi epi, const CUtensorMap& a_r, const CUtensorMap& a_s, const CUtensorMap& q_r0,
                          const CUtensorMap& q_r1, const CUtensorMap& q_s0, const CUtensorMap& q_s1,
                          const QGemmArgs& g, cudaStream_t st) {
  if (g.base.bm != 256 || g.base.n_groups > kMaxGroups - 1) return cudaErrorInvalidValue;
  QParams qp;
  qp.p = make_params(g.base);
  qp.wbits = g.wbits;
  qp.gsz = g.gsz;
  qp.gate_up = g.gate_up;
  qp.qrows_r = g.qrows_r;
  qp.qrows_s = g.qrows_s;
  qp.qtotal_r = g.qtotal_r;
  qp.qtotal_s = g.qtotal_s;
  qp.gs_r0 = g.gs_r0;
  qp.gs_r1 = g.gs_r1;
  qp.gs_s0 = g.gs_s0;
  qp.gs_s1 = g.gs_s1;
  const bool grouped = g.gsz > 0;
  void (*kern)(CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, CUtensorMap, QParams) = nullptr;
#define PICK(E_, W_, G_) \
  if (epi == E_ && g.wbits == W_ && grouped == G_) kern = grouped_gemm_pair_q_kernel<E_, W_, G_>;
  PICK(EPI_SWIGLU, 4, true) PICK(EPI_SWIGLU, 4, false) PICK(EPI_SWIGLU, 8, true) PICK(EPI_SWIGLU, 8, false)
  PICK(EPI_STORE, 4, true) PICK(EPI_STORE, 4, false) PICK(EPI_STORE, 8, true) PICK(EPI_STORE, 8, false)
  PICK(EPI_COMBINE, 4, true) PICK(EPI_COMBINE, 4, false) PICK(EPI_COMBINE, 8, true) PICK(EPI_COMBINE, 8, false)
#undef PICK
  if (!kern) return cudaErrorInvalidValue;
  const int smem = g.wbits == 4 ? Cfg<4>::kSmemBytes : Cfg<8>::kSmemBytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<(g.base.grid / 2) * 2, kThreads, smem, st>>>(a_r, a_s, q_r0, q_r1, q_s0, q_s1, qp);
  return cudaGetLastError();
}

}  // namespace flux
