// gemm_pair.cuh — pieces shared by the CTA-pair grouped GEMM kernels (gemm_pair.cu: one GEMM per
// launch; gemm_chain.cu: gate/up and down chained in one persistent launch): the tile / stage
// geometry, the TMA-store epilogue and the cp.async gather of the routed A rows.
#pragma once
#include "gemm_common.cuh"

namespace flux {
namespace {
using namespace gemm;

constexpr int kHalfM = 128, kPairM = 256, kStages = 6;
constexpr int kABytes = kHalfM * kBK * 2;     // 16 KB: this CTA's A rows
constexpr int kBBytes = (kBN / 2) * kBK * 2;  // 16 KB: this CTA's half of B
constexpr int kStageBytes = kABytes + kBBytes;
// 9 warps for gate/up (TMA, MMA, 2 gather producers, 4 epilogue, gather relay); the other epilogues
// run without the gather warps' relay: 8 warps, i.e. 2 per SM sub-partition, so each thread may use
// up to 255 registers (a 9th warp puts 3 warps on one sub-partition and caps them at 168)
template <int EPI>
constexpr int kThreadsOf = EPI == EPI_SWIGLU ? 288 : 256;
// after the ring: barriers, schedule copies, gather ids and scales (< 8 KB), then one 4 KB TMA-store
// staging buffer per epilogue warp (1024-byte aligned: 128-byte swizzle atoms)
constexpr int kMiscBytes = 8192;
static_assert(256 + 3 * kMaxGroups * 4 + 16 + 128 * 4 + kScaleSmemBytes <= kMiscBytes, "smem layout");
constexpr int kStageOutBytes = 4096;  // 32 rows x 64 bf16 columns
constexpr int kPickBytes = 32 * 64;  // per epilogue warp: 32 rows x (8 inv_pos + 8 gate weights), fused combine
// dynamic tile claiming: a ring of claimed tile ids with full/empty barriers (after the pick tables)
constexpr int kTileSlots = 8;
constexpr int kTileRingBytes = 256;
static_assert(2 * kTileSlots * 8 + kTileSlots * 4 <= kTileRingBytes, "tile ring");
constexpr int kSmemBytes =
    1024 + kStages * kStageBytes + kMiscBytes + 4 * kStageOutBytes + 4 * kPickBytes + kTileRingBytes;

// TMA-store epilogue of one 32-row slice (a warp's TMEM lanes) whose rows all lie inside the group:
// per 64-column chunk the warp converts its accumulator columns to bf16, writes them to its staging
// buffer in the 128-byte-swizzled layout of the output tensor map (conflict-free: the 16-byte chunk
// index is XORed with row % 8), and one lane issues a TMA store of the 32x64 box.  Versus one STG
// per thread-row (32 scattered rows per instruction) this keeps the LSU out of the epilogue, which
// bounded the LLaMA-shape down GEMM.  Same values and roundings as epilogue_slice.
template <int EPI, int kBatch = (EPI == EPI_SWIGLU ? 2 : 4)>
__device__ __forceinline__ void epilogue_tma(const Params& p, uint32_t taddr, const TileInfo& ti, int up_col,
                                             const float* sc, const CUtensorMap* tmo, uint32_t stage, int out_row,
                                             bool hint, uint64_t pol) {
  const int N = ti.g < p.E ? p.N_r : p.N_s;
  const uint32_t lane = lane_id();
  constexpr int kChunks = EPI == EPI_SWIGLU ? 2 : 4;  // 64-column output chunks per tile
  for (int cc = 0; cc < kChunks; ++cc) {
    const int j0 = cc * 64;
    const int col0 = (EPI == EPI_SWIGLU ? ti.n * (kBN / 2) : ti.n * kBN) + j0;
    if ((EPI == EPI_SWIGLU && j0 >= up_col) || col0 >= N) break;  // warp-uniform
    uint32_t pk[32];
    // TMEM loads are batched before one wait: all four 16-column groups of the chunk (STORE) or two
    // gate + two up groups (SWIGLU, whose 9-warp kernel is capped at 168 registers; the chained kernel
    // runs its STORE epilogue with batches of two as well)
#pragma unroll
    for (int h0 = 0; h0 < 4; h0 += kBatch) {
      float gv[kBatch][16], uv[kBatch][16];
      bool live[kBatch];
#pragma unroll
      for (int b = 0; b < kBatch; ++b) {
        const int j = j0 + 16 * (h0 + b);
        live[b] = (EPI != EPI_SWIGLU || j < up_col) && col0 + 16 * (h0 + b) < N;  // warp-uniform
        if (live[b]) {
          tmem_ld16(taddr + j, gv[b]);
          if constexpr (EPI == EPI_SWIGLU) tmem_ld16(taddr + up_col + j, uv[b]);
        }
      }
      tmem_ld_wait();
#pragma unroll
      for (int b = 0; b < kBatch; ++b) {
        const int h = h0 + b;
        const int j = j0 + 16 * h;
        if (!live[b]) {
#pragma unroll
          for (int i = 0; i < 8; ++i) pk[8 * h + i] = 0u;
          continue;
        }
        if constexpr (EPI == EPI_SWIGLU) {
          if (sc) {
            float gs[16], us[16];
            lds16(sc + j, gs);
            lds16(sc + 256 + j, us);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              gv[b][i] *= gs[i];
              uv[b][i] *= us[i];
            }
          }
#pragma unroll
          for (int i = 0; i < 16; i += 2)
            pk[8 * h + i / 2] = pack_bf16x2(silu(gv[b][i]) * uv[b][i], silu(gv[b][i + 1]) * uv[b][i + 1]);
        } else {
          if (sc) {
            float cs[16];
            lds16(sc + j, cs);
#pragma unroll
            for (int i = 0; i < 16; ++i) gv[b][i] *= cs[i];
          }
#pragma unroll
          for (int i = 0; i < 16; i += 2) pk[8 * h + i / 2] = pack_bf16x2(gv[b][i], gv[b][i + 1]);
        }
      }
    }
    if (lane == 0) bulk_wait_group_read0();  // the previous chunk's store has read the buffer
    __syncwarp();
    const uint32_t row_addr = stage + lane * 128;
#pragma unroll
    for (int c16 = 0; c16 < 8; ++c16)
      st_shared_v4(row_addr + ((c16 ^ (lane & 7)) << 4),
                   make_uint4(pk[4 * c16], pk[4 * c16 + 1], pk[4 * c16 + 2], pk[4 * c16 + 3]));
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (hint)
        tma_store_2d_hint(tmo, stage, col0, out_row, pol);
      else
        tma_store_2d(tmo, stage, col0, out_row);
      bulk_commit_group();
    }
  }
}

// Routed A rows gathered from x with per-lane 16-byte cp.async (LDGSTS) instead of a materialised
// x_perm: per 64-wide K slice this CTA's 128 rows x 128 bytes are copied by two producer warps
// (warps 2 and 3, 64 rows each; one warp is issue-bound, and warp 0 keeps the TMA loads of B and
// of the shared MLP's A), one warp instruction per 4 rows
// (8 lanes per row, 16-byte chunk c of row r to r·128 + ((c ^ r%8)·16): the 128-byte swizzle a TMA
// box would produce, conflict-free).  A lane's 16 row sources (token ids; rows past the group end
// read token 0 and are masked in the epilogue) are loaded into registers once per tile, so a slice
// is 16 independent address + LDGSTS pairs per lane.  H % 64 == 0: no K tail.
constexpr int kGatherParts = 2;
constexpr int kGatherRows = kHalfM / 4 / kGatherParts;  // row groups of 4 per warp
__device__ __forceinline__ void gather_ids(const Params& p, int row0, int rows_in_grp, int first, int part,
                                           int (&tok)[kGatherRows]) {
  const int lane = (int)lane_id();
#pragma unroll
  for (int i = 0; i < kGatherRows; ++i) {
    const int rl = first + part * (kHalfM / kGatherParts) + 4 * i + (lane >> 3);
    tok[i] = rl < rows_in_grp ? __ldg(&p.gather_idx[row0 + rl]) : 0;
  }
}
__device__ __forceinline__ void gather_a_cp(uint8_t* dst, const Params& p, const int (&tok)[kGatherRows], int kb,
                                            int part) {
  const int lane = (int)lane_id();
  const int chunk = lane & 7;
  const uint32_t base = smem_u32(dst);
  const __nv_bfloat16* src0 = p.a_src + kb * kBK + chunk * 8;
#pragma unroll
  for (int i = 0; i < kGatherRows; ++i) {
    const int row = part * (kHalfM / kGatherParts) + 4 * i + (lane >> 3);
    cp_async16(base + row * 128 + ((chunk ^ (row & 7)) << 4), src0 + (int64_t)tok[i] * p.a_ld);
  }
}

}  // namespace
}  // namespace flux
