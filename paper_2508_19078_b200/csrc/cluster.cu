// cluster.cu — NEXT-1: similarity-based expert clustering, §5.2.
//
//  C1 features: PCA of a layer's experts (each expert = all of its
//     parameters), via the E x E Gram matrix G = X Xᵀ of the raw vectors:
//     gram_kernel   — split-K tcgen05 GEMM: every CTA streams a contiguous K range
//                     of X [E][P] with TMA (64-column slices, rows >= E zero-filled)
//                     and computes X_k X_kᵀ with M=128, N=E_pad; A and B are the
//                     SAME shared-memory tile.  fp32 partials per CTA.
//     gram_reduce   — sums the partials in a fixed order (deterministic).
//     eig_kernel    — one CTA: centre G (H G H), parallel cyclic Jacobi in fp64
//                     (round-robin pairing, E/2 disjoint rotations per round), sort
//                     eigenvalues, scores F = V_d Λ_d^(1/2).
//  C2 fused K-Means (reading R13): layers are independent once
//     cross-layer distances are masked, so the fused problem is one CTA per layer
//     in one launch: init from the most frequent non-tuning experts, cosine
//     assignment (ties -> lower centroid), mean update (fixed member order), stop
//     when no assignment changes.  fp64.
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "internal.h"
#include "ptx.cuh"

namespace flux {
namespace {

constexpr int kBM = 128, kBK = 64, kMaxE = 128;
constexpr int kMaxFam = 4;
constexpr int kGramInflight = 128 * 1024;  // bytes of expert data in flight per SM (HBM latency x bandwidth / SM)
// 64-column slices per stage: each row streams 512 contiguous bytes (1 KB for 16 experts, whose eight
// slices make one 128-row MMA operand)
constexpr int slices_of(int npad) { return npad <= 16 ? 8 : 4; }
constexpr int kSubStages = 8;              // TMEM accumulation sub-chunk (32 slices = 128 MMAs), then drained
constexpr int kChunkSlices = 64;           // work unit claimed dynamically; one partial slot each
constexpr int kRing = 8;                   // claimed-chunk ring (producer -> MMA, epilogue)

struct GramMaps {
  CUtensorMap map[kMaxFam];   // family f of this layer: bf16 [E][P_f], box {64 cols, NPAD rows}
  CUtensorMap map4[kMaxFam];  // the same family as [P_f/64 blocks][E][64]: box {64, NPAD, slices} = one stage
  int64_t kb_end[kMaxFam];    // cumulative 64-column slice counts
  int64_t nblk[kMaxFam];      // whole 64-column blocks of family f (map4's outer extent)
  int n_fam;
};

// GRP = slices per MMA (1, or 128 / NPAD when consecutive slices are paired, see gram_kernel)
template <int NPAD, int INFL, int GRP>
struct GramCfg {
  static constexpr int kSlice = NPAD * kBK * 2;  // NPAD expert rows x 64 columns (128 B rows)
  static constexpr int kSl = slices_of(NPAD);
  static constexpr int kTile = kSl * kSlice;
  static constexpr int kStages = INFL / kTile < 3 ? 3 : (INFL / kTile < 16 ? INFL / kTile : 16);
  // The MMA reads M=128 rows from a slice; rows >= NPAD only feed accumulator rows that are never
  // stored, but they must be readable shared memory: pad the ring by the overhang.
  static constexpr int kPad = (kBM - NPAD) * 128;
  static constexpr int kBarriers = 2 * kStages + 4 + 2 * kRing;
  static constexpr int kAccCols = GRP > 1 ? kBM : NPAD;  // accumulator columns (N of the MMA)
  static constexpr int kXBytes = (GRP - 1) * NPAD * (NPAD + 1) * 4;  // cross-block sums of the epilogue
  static constexpr int kBytes = kStages * kTile + kPad + 1024 + kBarriers * 8 + kRing * 4 + 64 + kXBytes;
};

// Split-K Gram of one layer.  The concatenated 64-column slices of every family form chunks of
// kChunkSlices; CTAs claim chunks from a global counter (SMs stream HBM at different rates, so a
// static split leaves the fast ones idle) and store each chunk's fp32 X_k X_kᵀ [E][E] to its own
// slot partial[chunk] — the slot depends only on the chunk, so the reduction below is deterministic.
// A and B are the same shared-memory tile.  Precision: the tensor-core fp32 accumulator loses
// ~2^-24 (relative) per accumulating MMA, a bias that grows with the accumulation length; TMEM
// therefore accumulates sub-chunks of 128 MMAs (two buffers: the MMAs of sub-chunk c+1 overlap the
// drain of c) and the epilogue sums the sub-chunks of a chunk in registers.
// The counter is reset by gram_reduce_kernel, which runs after this kernel on the same stream.
//
// Paired slices (GRP = 128/NPAD > 1, NPAD 64, 32 or 16): a stage holds kSlices consecutive [NPAD][64]
// slices, so GRP of them form one 128-row K-major operand.  One M=128, N=128 MMA with that operand as
// both A and B computes all GRP x GRP slice products; the GRP diagonal NPAD x NPAD blocks are the
// wanted X_s X_sᵀ (the rest is never read).  Versus one M=128, N=NPAD MMA per slice (whose A rows
// beyond NPAD are the next slice's, read for nothing) this halves the MMAs' shared-memory operand reads
// per byte of X (the kernel's bound, ~18 B per SM clock), and the epilogue sums the GRP blocks of
// a chunk in a fixed order (deterministic).  Needs every stage's slice count to be a multiple of GRP
// (the launcher checks the layer's total).
template <int NPAD, int INFL, int GRP>
__global__ void __launch_bounds__(192, 1)
    gram_kernel(const __grid_constant__ GramMaps gm, int E, float* __restrict__ partial, int* __restrict__ counter) {
  using C = GramCfg<NPAD, INFL, GRP>;
  constexpr int kSlices = C::kSl;
  static_assert(kSlices % GRP == 0 && kChunkSlices % kSlices == 0 && GRP * NPAD <= kBM, "slice pairing");
  constexpr int kStages = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, still a shared-space pointer
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * C::kTile + C::kPad);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;    // [2]
  uint64_t* acc_empty = acc_full + 2;      // [2]
  uint64_t* chunk_full = acc_empty + 2;    // [kRing]
  uint64_t* chunk_empty = chunk_full + kRing;
  int* ring = reinterpret_cast<int*>(chunk_empty + kRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ring + kRing);
  constexpr uint32_t kCols = 2 * C::kAccCols <= 32 ? 32 : 2 * C::kAccCols;  // two accumulators
  float* xbuf = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(tmem_slot) + 64);  // [GRP-1][NPAD][NPAD+1]
  const int warp = warp_id();
  const int64_t n_kb = gm.kb_end[gm.n_fam - 1];
  const int n_chunks = (int)((n_kb + kChunkSlices - 1) / kChunkSlices);
  auto chunk_stages = [&](int id) {
    const int64_t left = n_kb - (int64_t)id * kChunkSlices;
    const int sl = left < kChunkSlices ? (int)left : kChunkSlices;
    return (sl + kSlices - 1) / kSlices;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 4);  // one arrive per epilogue warp
    }
    for (int r = 0; r < kRing; ++r) {
      mbar_init(&chunk_full[r], 1);
      mbar_init(&chunk_empty[r], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      for (int i = 0; i < gm.n_fam; ++i) tma_prefetch(&gm.map[i]);
      const uint64_t pol = policy_evict_first();
      int gs = 0;  // stages issued by this CTA
      for (int j = 0;; ++j) {
        const int r = j % kRing;
        mbar_wait(&chunk_empty[r], ((j / kRing) & 1) ^ 1);
        int id = atomicAdd(counter, 1);
        if (id >= n_chunks) id = -1;
        ring[r] = id;
        mbar_arrive(&chunk_full[r]);
        if (id < 0) break;
        const int64_t kb0 = (int64_t)id * kChunkSlices;
        const int64_t kb1 = kb0 + kChunkSlices < n_kb ? kb0 + kChunkSlices : n_kb;
        int f = 0;
        while (kb0 >= gm.kb_end[f]) ++f;
        for (int64_t kb = kb0; kb < kb1; kb += kSlices, ++gs) {
          const int s = gs % kStages;
          const uint32_t ph = (gs / kStages) & 1;
          const int n_sl = kb1 - kb < kSlices ? (int)(kb1 - kb) : kSlices;
          while (kb >= gm.kb_end[f]) ++f;
          const int64_t local = kb - (f ? gm.kb_end[f - 1] : 0);
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], n_sl * C::kSlice);
          if (n_sl == kSlices && local + kSlices <= gm.nblk[f]) {
            // the whole stage in one 3D box: kSlices blocks of 64 columns x NPAD rows, written as kSlices
            // consecutive [NPAD][128 B] slices (a quarter of the producer's instructions per byte)
            tma_load_3d_hint(smem + s * C::kTile, &gm.map4[f], &full[s], 0, 0, (int32_t)local, pol);
          } else {
            int ft = f;
            for (int t = 0; t < n_sl; ++t) {
              while (kb + t >= gm.kb_end[ft]) ++ft;
              const int64_t lt = kb + t - (ft ? gm.kb_end[ft - 1] : 0);
              tma_load_2d_hint(smem + s * C::kTile + t * C::kSlice, &gm.map[ft], &full[s], (int32_t)(lt * kBK), 0,
                               pol);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = umma_idesc_bf16(kBM, C::kAccCols);
    int gs = 0, gc = 0;  // stages consumed, sub-chunks accumulated
    for (int j = 0;; ++j) {
      const int r = j % kRing;
      mbar_wait(&chunk_full[r], (j / kRing) & 1);
      const int id = ring[r];
      if (id < 0) break;
      const int n_st = chunk_stages(id);
      const int64_t kb_base = (int64_t)id * kChunkSlices;
      for (int st = 0; st < n_st; ++st, ++gs) {
        const int s = gs % kStages;
        const uint32_t ph = (gs / kStages) & 1;
        const int b = gc & 1;
        const bool first = st % kSubStages == 0;
        const bool last = (st + 1) % kSubStages == 0 || st == n_st - 1;
        if (first) mbar_wait(&acc_empty[b], ((gc >> 1) & 1) ^ 1);
        mbar_wait(&full[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const int64_t left = n_kb - kb_base - (int64_t)st * kSlices;
          const int n_sl = left < kSlices ? (int)left : kSlices;
          const uint32_t d = tmem + b * C::kAccCols;
          for (int t = 0; t < n_sl; t += GRP) {
            const uint64_t desc = umma_desc_sw128(smem_u32(smem + s * C::kTile + t * C::kSlice));
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              umma_bf16(d, desc + 2 * k, desc + 2 * k, idesc, !(first && t == 0 && k == 0));
          }
          umma_commit(&empty[s]);
          if (last) umma_commit(&acc_full[b]);
        }
        __syncwarp();
        if (last) ++gc;
      }
    }
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane_id();
    const int blk = row / NPAD, er = row % NPAD;  // paired slices: diagonal block and its expert row
    const bool live = GRP > 1 ? (q * 32) % NPAD < E : q * 32 < E;  // warp-uniform
    int gc = 0;
    for (int j = 0;; ++j) {
      const int r = j % kRing;
      mbar_wait(&chunk_full[r], (j / kRing) & 1);
      const int id = ring[r];
      if (id < 0) break;
      const int n_sub = (chunk_stages(id) + kSubStages - 1) / kSubStages;
      float acc[NPAD];
#pragma unroll
      for (int i = 0; i < NPAD; ++i) acc[i] = 0.f;
      for (int sub = 0; sub < n_sub; ++sub, ++gc) {
        const int b = gc & 1;
        mbar_wait(&acc_full[b], (gc >> 1) & 1);
        tc_fence_after();
        if constexpr (GRP > 1 && NPAD < 32) {
          // 16-row blocks: lanes 0-15 and 16-31 of a warp are rows of two blocks (columns must be
          // warp-uniform in tcgen05.ld): load both blocks' columns, each lane keeps its own
          float v[16], w[16];
          const uint32_t a = tmem + ((uint32_t)(q * 32) << 16) + b * C::kAccCols + (q * 32 / NPAD) * NPAD;
          tmem_ld16(a, v);
          tmem_ld16(a + 16, w);
          tmem_ld_wait();
          const bool hi = lane_id() >= 16;
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[i] += hi ? w[i] : v[i];
        } else if (live) {
#pragma unroll
          for (int col = 0; col < NPAD; col += 16) {
            float v[16];
            tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + b * C::kAccCols + (GRP > 1 ? blk * NPAD : 0) + col, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[col + i] += v[i];
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&acc_empty[b]);
      }
      float* out = partial + (int64_t)id * E * E;
      if constexpr (GRP > 1) {
        // block sums in a fixed order: block 0's rows add blocks 1..GRP-1 (row stride NPAD+1: no conflicts)
        if (blk > 0 && live)
#pragma unroll
          for (int i = 0; i < NPAD; ++i) xbuf[((blk - 1) * NPAD + er) * (NPAD + 1) + i] = acc[i];
        named_bar_sync(1, 128);
        if (blk == 0 && er < E) {
#pragma unroll
          for (int gb = 1; gb < GRP; ++gb)
#pragma unroll
            for (int i = 0; i < NPAD; ++i) acc[i] += xbuf[((gb - 1) * NPAD + er) * (NPAD + 1) + i];
#pragma unroll
          for (int i = 0; i < NPAD; ++i)
            if (i < E) out[er * E + i] = acc[i];
        }
        named_bar_sync(1, 128);  // xbuf is rewritten by the next chunk
      } else if (row < E) {
#pragma unroll
        for (int i = 0; i < NPAD; ++i)
          if (i < E) out[row * E + i] = acc[i];
      }
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&chunk_empty[r]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kCols>(tmem);
}

// G[i][j] = Σ_p partial[p][i][j]: NG = 1024/EP groups of partials per (i, j), each summed in
// ascending p, then the group sums in ascending order (fixed order: deterministic).  One CTA per row.
template <int EP>
__global__ void __launch_bounds__(1024) gram_reduce_kernel(const float* __restrict__ partial, int n_partial, int E,
                                                           float* __restrict__ G, float* __restrict__ G_user,
                                                           int* __restrict__ counter) {
  constexpr int NG = 1024 / EP;
  __shared__ double part[NG][EP];
  const int i = blockIdx.x, j = threadIdx.x % EP, g = threadIdx.x / EP;
  if (i == 0 && threadIdx.x == 0) *counter = 0;  // the Gram kernel that claimed from it has completed
  double acc = 0.0;
  if (j < E) {  // ascending p; eight loads in flight before their (in-order) additions
    const float* src = partial + i * E + j;
    const int64_t ee = (int64_t)E * E;
    int p = g;
    for (; p + 7 * NG < n_partial; p += 8 * NG) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + (int64_t)(p + u * NG) * ee);
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += v[u];
    }
    for (; p < n_partial; p += NG) acc += __ldcg(src + (int64_t)p * ee);
  }
  part[g][j] = acc;
  __syncthreads();
  if (g == 0 && j < E) {
    double t = 0.0;
#pragma unroll
    for (int h = 0; h < NG; ++h) t += part[h][j];
    G[i * E + j] = (float)t;
    if (G_user) G_user[i * E + j] = (float)t;
  }
}

// One CTA per layer.  A = H G H in fp64 shared memory; parallel cyclic Jacobi (round-robin
// pairing: n/2 disjoint rotations per round applied to rows, then to columns and to V).
// V is fp64 for E <= 64 and fp32 for E <= 128 (A fp64 + V fp64 would not fit in 227 KB).
constexpr int kEigThreads = 512;
template <typename VT>
__global__ void __launch_bounds__(kEigThreads) eig_kernel(const float* __restrict__ G, int E, int d,
                                                          float* __restrict__ features, float* __restrict__ eigvals) {
  const int n = E + (E & 1);  // even count for the round-robin pairing (dummy index n-1 if E is odd)
  const int ld = n + 1;
  extern __shared__ double eig_smem[];  // A [n][ld] fp64, then V [n][ld] VT
  double* A = eig_smem;
  VT* V = reinterpret_cast<VT*>(eig_smem + n * ld);
  G += (size_t)blockIdx.x * E * E;
  features += (size_t)blockIdx.x * E * d;
  if (eigvals) eigvals += (size_t)blockIdx.x * d;
  __shared__ double rc[kMaxE / 2], rs[kMaxE / 2];
  __shared__ int rp[kMaxE / 2], rq[kMaxE / 2];
  __shared__ double red[kEigThreads];
  __shared__ int order[kMaxE];
  __shared__ double rsum[kMaxE];
  __shared__ double tot;
  const int tid = threadIdx.x;
  // centring: A = G - r/E 1ᵀ - 1 r/Eᵀ + s/E², r_i = Σ_j G_ij, s = Σ r_i
  for (int i = tid; i < E; i += kEigThreads) {
    double r = 0.0;
    for (int j = 0; j < E; ++j) r += (double)G[i * E + j];
    rsum[i] = r;
  }
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int i = 0; i < E; ++i) t += rsum[i];
    tot = t;
  }
  __syncthreads();
  for (int idx = tid; idx < n * n; idx += kEigThreads) {
    const int i = idx / n, j = idx % n;
    double a = 0.0;
    if (i < E && j < E) a = (double)G[i * E + j] - rsum[i] / E - rsum[j] / E + tot / ((double)E * E);
    A[i * ld + j] = a;
    V[i * ld + j] = i == j ? VT(1) : VT(0);
  }
  __syncthreads();
  auto block_sum = [&](double v) {
    red[tid] = v;
    __syncthreads();
    for (int st = kEigThreads / 2; st > 0; st >>= 1) {
      if (tid < st) red[tid] += red[tid + st];
      __syncthreads();
    }
    const double r = red[0];
    __syncthreads();
    return r;
  };
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, all = 0.0;
    for (int idx = tid; idx < n * n; idx += kEigThreads) {
      const int i = idx / n, j = idx % n;
      const double a2 = A[i * ld + j] * A[i * ld + j];
      all += a2;
      if (i != j) off += a2;
    }
    const double off_t = block_sum(off), all_t = block_sum(all);
    if (off_t <= 1e-24 * all_t || all_t == 0.0) break;  // off-diagonal norm <= 1e-12 of the total
    for (int round = 0; round < n - 1; ++round) {
      if (tid < n / 2) {  // circle method: position 0 fixed, the others rotate
        auto player = [&](int pos) { return pos == 0 ? 0 : 1 + ((pos - 1 + round) % (n - 1)); };
        int p = player(tid), q = player(n - 1 - tid);
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        const double apq = A[p * ld + q];
        double c = 1.0, sn = 0.0;
        if (fabs(apq) > 1e-300) {
          const double theta = (A[q * ld + q] - A[p * ld + p]) / (2.0 * apq);
          const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          c = 1.0 / sqrt(t * t + 1.0);
          sn = t * c;
        }
        rp[tid] = p;
        rq[tid] = q;
        rc[tid] = c;
        rs[tid] = sn;
      }
      __syncthreads();
      for (int idx = tid; idx < (n / 2) * n; idx += kEigThreads) {  // A <- Jᵀ A
        const int r = idx / n, k = idx % n;
        const int p = rp[r], q = rq[r];
        const double c = rc[r], sn = rs[r];
        const double ap = A[p * ld + k], aq = A[q * ld + k];
        A[p * ld + k] = c * ap - sn * aq;
        A[q * ld + k] = sn * ap + c * aq;
      }
      __syncthreads();
      for (int idx = tid; idx < (n / 2) * n; idx += kEigThreads) {  // A <- A J, V <- V J
        const int r = idx / n, k = idx % n;
        const int p = rp[r], q = rq[r];
        const double c = rc[r], sn = rs[r];
        const double ap = A[k * ld + p], aq = A[k * ld + q];
        A[k * ld + p] = c * ap - sn * aq;
        A[k * ld + q] = sn * ap + c * aq;
        const double vp = V[k * ld + p], vq = V[k * ld + q];
        V[k * ld + p] = VT(c * vp - sn * vq);
        V[k * ld + q] = VT(sn * vp + c * vq);
      }
      __syncthreads();
    }
  }
  if (tid == 0) {  // eigenvalues descending (stable: lower index first on ties)
    for (int i = 0; i < E; ++i) order[i] = i;
    for (int i = 0; i < E; ++i)
      for (int j = i + 1; j < E; ++j)
        if (A[order[j] * ld + order[j]] > A[order[i] * ld + order[i]]) {
          const int t = order[i];
          order[i] = order[j];
          order[j] = t;
        }
  }
  __syncthreads();
  for (int idx = tid; idx < E * d; idx += kEigThreads) {
    const int e = idx / d, j = idx % d;
    const int col = order[j];
    const double lam = A[col * ld + col] > 0.0 ? A[col * ld + col] : 0.0;
    features[e * d + j] = (float)((double)V[e * ld + col] * sqrt(lam));
  }
  if (eigvals)
    for (int j = tid; j < d; j += kEigThreads) eigvals[j] = (float)A[order[j] * ld + order[j]];
}

// One CTA per layer; thread e = expert e.  Frequencies enter as the profiled counts (f = count / T
// is monotone in the count, so the initial ranking is the same).
__global__ void __launch_bounds__(kMaxE) kmeans_kernel(int E, int d, const float* __restrict__ features,
                                                       const int64_t* __restrict__ counts,
                                                       const __grid_constant__ KMeansArgs ka, int max_iter,
                                                       int32_t* __restrict__ cluster_of, int32_t* __restrict__ iters) {
  constexpr int kMaxD = 32;
  extern __shared__ double km_smem[];  // F [E][d], mu [E][d]
  double* F = km_smem;
  double* mu = km_smem + E * d;
  __shared__ int init_rank[kMaxE];
  __shared__ int assign[kMaxE];
  const int l = blockIdx.x, e = threadIdx.x;
  const int B = ka.n_clusters[l];
  auto is_tuning = [&](int x) { return (ka.tuning[l][x >> 6] >> (x & 63)) & 1; };
  const bool valid = e < E;
  const bool tun = valid && is_tuning(e);
  if (valid)
    for (int j = 0; j < d; ++j) F[e * d + j] = (double)features[((int64_t)l * E + e) * d + j];
  // rank among non-tuning experts by (-count, id)
  if (valid && !tun) {
    const int64_t fe = counts[l * E + e];
    int r = 0;
    for (int o = 0; o < E; ++o) {
      if (is_tuning(o)) continue;
      const int64_t fo = counts[l * E + o];
      r += (fo > fe) || (fo == fe && o < e);
    }
    init_rank[e] = r;
  } else if (valid) {
    init_rank[e] = -1;
  }
  __syncthreads();
  if (valid && !tun && init_rank[e] < B)
    for (int j = 0; j < d; ++j) mu[init_rank[e] * d + j] = F[e * d + j];
  if (valid) assign[e] = -1;
  __syncthreads();
  int it = 0;
  for (it = 1; it <= max_iter; ++it) {
    int mine = -1;
    if (valid && !tun) {
      double nf = 0.0;
      for (int j = 0; j < d; ++j) nf += F[e * d + j] * F[e * d + j];
      nf = sqrt(nf);
      double best = INFINITY;
      for (int c = 0; c < B; ++c) {
        double dot = 0.0, nm = 0.0;
        for (int j = 0; j < d; ++j) {
          dot += F[e * d + j] * mu[c * d + j];
          nm += mu[c * d + j] * mu[c * d + j];
        }
        nm = sqrt(nm);
        const double dist = (nf == 0.0 || nm == 0.0) ? 1.0 : 1.0 - dot / (nf * nm);
        if (dist < best) {
          best = dist;
          mine = c;
        }
      }
    }
    const int changed = __syncthreads_or(valid && mine != assign[e]);
    if (valid) assign[e] = mine;
    __syncthreads();
    if (e < B) {  // centroid e: mean of its members in ascending expert order
      int cnt = 0;
      double acc[kMaxD];
      for (int j = 0; j < d; ++j) acc[j] = 0.0;
      for (int o = 0; o < E; ++o)
        if (assign[o] == e) {
          ++cnt;
          for (int j = 0; j < d; ++j) acc[j] += F[o * d + j];
        }
      if (cnt)
        for (int j = 0; j < d; ++j) mu[e * d + j] = acc[j] / cnt;
    }
    __syncthreads();
    if (!changed) break;
  }
  if (valid) cluster_of[l * E + e] = assign[e];
  if (e == 0 && iters) iters[l] = it > max_iter ? max_iter : it;
}
}  // namespace

static int64_t gram_chunks(int n_fam, const int64_t* P) {
  int64_t kb = 0;
  for (int f = 0; f < n_fam; ++f) kb += (P[f] + kBK - 1) / kBK;
  return (kb + kChunkSlices - 1) / kChunkSlices;
}

// [partial slots: n_chunks][E][E] fp32 | G [L][E][E] fp32 | counter
size_t features_workspace(int L, int E, int n_fam, const int64_t* P) {
  return ((size_t)gram_chunks(n_fam, P) + (size_t)L) * E * E * sizeof(float) + 256;
}
float* features_gram_slot(void* ws, int E, int n_fam, const int64_t* P, int l) {
  return reinterpret_cast<float*>(ws) + ((size_t)gram_chunks(n_fam, P) + (size_t)l) * E * E;
}
int* features_counter(void* ws, int L, int E, int n_fam, const int64_t* P) {
  const uintptr_t p = reinterpret_cast<uintptr_t>(features_gram_slot(ws, E, n_fam, P, L));
  return reinterpret_cast<int*>((p + 15) & ~uintptr_t(15));
}

template <int NPAD, int GRP = 1>
static cudaError_t launch_gram_n(const GramMaps& gm, int E, float* partial, int* counter, int grid, cudaStream_t st) {
  const int smem = GramCfg<NPAD, kGramInflight, GRP>::kBytes;
  cudaError_t e =
      cudaFuncSetAttribute(gram_kernel<NPAD, kGramInflight, GRP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  gram_kernel<NPAD, kGramInflight, GRP><<<grid, 192, smem, st>>>(gm, E, partial, counter);
  return cudaGetLastError();
}

// Gram partials of one layer (families X_f [E][P_f]); *n_slots = number of partial slots written.
cudaError_t launch_gram(int E, int n_fam, const void* const* X, const int64_t* P, float* partial, int* counter,
                        int* n_slots, cudaStream_t st) {
  if (n_fam < 1 || n_fam > kMaxFam) return cudaErrorInvalidValue;
  const int npad = E <= 16 ? 16 : E <= 32 ? 32 : E <= 64 ? 64 : 128;
  GramMaps gm;
  memset(&gm, 0, sizeof(gm));
  gm.n_fam = n_fam;
  int64_t acc = 0;
  for (int f = 0; f < n_fam; ++f) {
    if (!make_tmap_2d(&gm.map[f], X[f], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)E, (uint64_t)P[f],
                      (uint64_t)P[f] * 2, 64, (uint32_t)npad, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
    gm.nblk[f] = P[f] / kBK;
    if (gm.nblk[f] >= slices_of(npad) &&
        !make_tmap_gram_blocks(&gm.map4[f], X[f], (uint64_t)E, (uint64_t)P[f], (uint32_t)npad, slices_of(npad)))
      return cudaErrorInvalidValue;
    if (gm.nblk[f] < slices_of(npad)) gm.nblk[f] = 0;  // too short for a whole stage: per-slice loads only
    acc += (P[f] + kBK - 1) / kBK;
    gm.kb_end[f] = acc;
  }
  const int64_t chunks = gram_chunks(n_fam, P);
  const int grid = (int)std::min<int64_t>(kNumSMs, chunks);
  *n_slots = (int)chunks;
  // paired slices when every stage's slice count is a multiple of the pair size: stages hold
  // slices_of(npad) slices except at a chunk's end (chunks are kChunkSlices, a multiple of 8) and the
  // layer's end
  const int64_t n_kb = gm.kb_end[n_fam - 1];
  switch (npad) {
    case 16: return n_kb % 8 == 0 ? launch_gram_n<16, 8>(gm, E, partial, counter, grid, st)
                                  : launch_gram_n<16>(gm, E, partial, counter, grid, st);
    case 32: return n_kb % 4 == 0 ? launch_gram_n<32, 4>(gm, E, partial, counter, grid, st)
                                  : launch_gram_n<32>(gm, E, partial, counter, grid, st);
    case 64: return n_kb % 2 == 0 ? launch_gram_n<64, 2>(gm, E, partial, counter, grid, st)
                                  : launch_gram_n<64>(gm, E, partial, counter, grid, st);
    default: return launch_gram_n<128>(gm, E, partial, counter, grid, st);
  }
}

cudaError_t launch_gram_reduce(int E, const float* partial, int n_slots, float* G, float* G_user, int* counter,
                               cudaStream_t st) {
  if (E <= 64)
    gram_reduce_kernel<64><<<E, 1024, 0, st>>>(partial, n_slots, E, G, G_user, counter);
  else
    gram_reduce_kernel<128><<<E, 1024, 0, st>>>(partial, n_slots, E, G, G_user, counter);
  return cudaGetLastError();
}

cudaError_t launch_eig(int L, int E, int d, const float* G, float* features, float* eigvals, cudaStream_t st) {
  const int n = E + (E & 1);
  cudaError_t e;
  if (E <= 64) {
    const int smem = n * (n + 1) * (8 + 8);
    e = cudaFuncSetAttribute(eig_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) eig_kernel<double><<<L, kEigThreads, smem, st>>>(G, E, d, features, eigvals);
  } else {
    const int smem = n * (n + 1) * (8 + 4) + 8;
    e = cudaFuncSetAttribute(eig_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) eig_kernel<float><<<L, kEigThreads, smem, st>>>(G, E, d, features, eigvals);
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_kmeans(int L, int E, int d, const float* features, const int64_t* counts, const KMeansArgs& ka,
                          int max_iter, int32_t* cluster_of, int32_t* iters, cudaStream_t st) {
  const int smem = 2 * E * d * (int)sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(kmeans_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kmeans_kernel<<<L, kMaxE, smem, st>>>(E, d, features, counts, ka, max_iter, cluster_of, iters);
  return cudaGetLastError();
}

}  // namespace flux
