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
#include <algorithm>

#include "internal.h"
#include "ptx.cuh"

namespace flux {
namespace {

constexpr int kBM = 128, kBK = 64, kStages = 4, kMaxE = 64;

template <int NPAD>
__global__ void __launch_bounds__(192, 1)
    gram_kernel(const __grid_constant__ CUtensorMap tmap, int64_t n_kb, int E, float* __restrict__ partial) {
  constexpr int kTile = kBM * kBK * 2;  // 16 KB
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kTile);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  constexpr uint32_t kCols = NPAD <= 32 ? 32 : (NPAD <= 64 ? 64 : 128);
  const int warp = warp_id();
  // this CTA's contiguous range of 64-column slices
  const int64_t per = n_kb / gridDim.x, rem = n_kb % gridDim.x;
  const int64_t bx = blockIdx.x;
  const int64_t kb0 = bx * per + (bx < rem ? bx : rem);
  const int nk = (int)(per + (blockIdx.x < rem ? 1 : 0));

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<kCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (elect_one()) {
      tma_prefetch(&tmap);
      for (int i = 0; i < nk; ++i) {
        const int s = i % kStages;
        const uint32_t ph = (i / kStages) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&full[s], kTile);
        tma_load_2d(smem + s * kTile, &tmap, &full[s], (int32_t)((kb0 + i) * kBK), 0);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = umma_idesc_bf16(kBM, NPAD);
    for (int i = 0; i < nk; ++i) {
      const int s = i % kStages;
      const uint32_t ph = (i / kStages) & 1;
      mbar_wait(&full[s], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint64_t desc = umma_desc_sw128(smem_u32(smem + s * kTile));
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) umma_bf16(tmem, desc + 2 * k, desc + 2 * k, idesc, (i | k) != 0);
        umma_commit(&empty[s]);
        if (i == nk - 1) umma_commit(acc_full);
      }
      __syncwarp();
    }
  } else {
    const int q = warp & 3;
    const int row = q * 32 + lane_id();
    float* out = partial + (int64_t)blockIdx.x * kMaxE * kMaxE;
    if (nk == 0) {
      if (row < E)
        for (int c = 0; c < E; ++c) out[row * kMaxE + c] = 0.f;
    } else {
      mbar_wait(acc_full, 0);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < NPAD; c += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + c, v);
        tmem_ld_wait();
        if (row < E)
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (c + i < E) out[row * kMaxE + c + i] = v[i];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<kCols>(tmem);
}

__global__ void gram_reduce_kernel(const float* __restrict__ partial, int n_partial, int E, float* __restrict__ G,
                                   float* __restrict__ G_user) {
  const int i = blockIdx.x, j = threadIdx.x;
  if (j >= E) return;
  double acc = 0.0;  // fixed order over partials: deterministic
  for (int p = 0; p < n_partial; ++p) acc += partial[(int64_t)p * kMaxE * kMaxE + i * kMaxE + j];
  G[i * kMaxE + j] = (float)acc;
  if (G_user) G_user[i * E + j] = (float)acc;
}

// One CTA (256 threads).  A = H G H in fp64 shared memory; parallel cyclic Jacobi.
__global__ void __launch_bounds__(256) eig_kernel(const float* __restrict__ G, int E, int d,
                                                  float* __restrict__ features, float* __restrict__ eigvals) {
  extern __shared__ double eig_smem[];  // A, V: [kMaxE][kMaxE + 1] fp64 each (66.5 KB, dynamic)
  double(*A)[kMaxE + 1] = reinterpret_cast<double(*)[kMaxE + 1]>(eig_smem);
  double(*V)[kMaxE + 1] = reinterpret_cast<double(*)[kMaxE + 1]>(eig_smem + kMaxE * (kMaxE + 1));
  G += (size_t)blockIdx.x * kMaxE * kMaxE;
  features += (size_t)blockIdx.x * E * d;
  if (eigvals) eigvals += (size_t)blockIdx.x * d;
  __shared__ double rc[kMaxE / 2], rs[kMaxE / 2];
  __shared__ int rp[kMaxE / 2], rq[kMaxE / 2];
  __shared__ double red[256];
  __shared__ int order[kMaxE];
  const int tid = threadIdx.x;
  const int n = E + (E & 1);  // even count for the round-robin pairing (dummy index n-1 if E is odd)
  // centring: A = G - r/E 1ᵀ - 1 r/Eᵀ + s/E², r_i = Σ_j G_ij, s = Σ r_i
  __shared__ double rsum[kMaxE];
  __shared__ double tot;
  for (int i = tid; i < E; i += 256) {
    double r = 0.0;
    for (int j = 0; j < E; ++j) r += (double)G[i * kMaxE + j];
    rsum[i] = r;
  }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int i = 0; i < E; ++i) s += rsum[i];
    tot = s;
  }
  __syncthreads();
  for (int idx = tid; idx < n * n; idx += 256) {
    const int i = idx / n, j = idx % n;
    double a = 0.0;
    if (i < E && j < E) a = (double)G[i * kMaxE + j] - rsum[i] / E - rsum[j] / E + tot / ((double)E * E);
    A[i][j] = a;
    V[i][j] = i == j ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int sweep = 0; sweep < 40; ++sweep) {
    // convergence: off-diagonal vs total Frobenius norm
    double off = 0.0, all = 0.0;
    for (int idx = tid; idx < n * n; idx += 256) {
      const int i = idx / n, j = idx % n;
      const double a2 = A[i][j] * A[i][j];
      all += a2;
      if (i != j) off += a2;
    }
    red[tid] = off;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (tid < s) red[tid] += red[tid + s];
      __syncthreads();
    }
    const double off_t = red[0];
    __syncthreads();
    red[tid] = all;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (tid < s) red[tid] += red[tid + s];
      __syncthreads();
    }
    const double all_t = red[0];
    __syncthreads();
    if (off_t <= 1e-24 * all_t || all_t == 0.0) break;  // off-diagonal norm <= 1e-12 of the total
    for (int round = 0; round < n - 1; ++round) {
      // circle method: position 0 fixed, others rotate
      if (tid < n / 2) {
        auto player = [&](int pos) { return pos == 0 ? 0 : 1 + ((pos - 1 + round) % (n - 1)); };
        int p = player(tid), q = player(n - 1 - tid);
        if (p > q) { const int t = p; p = q; q = t; }
        const double apq = A[p][q];
        double c = 1.0, s = 0.0;
        if (fabs(apq) > 1e-300) {
          const double theta = (A[q][q] - A[p][p]) / (2.0 * apq);
          const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          c = 1.0 / sqrt(t * t + 1.0);
          s = t * c;
        }
        rp[tid] = p;
        rq[tid] = q;
        rc[tid] = c;
        rs[tid] = s;
      }
      __syncthreads();
      // A <- Jᵀ A (rows p, q of every pair)
      for (int idx = tid; idx < (n / 2) * n; idx += 256) {
        const int r = idx / n, k = idx % n;
        const int p = rp[r], q = rq[r];
        const double c = rc[r], s = rs[r];
        const double ap = A[p][k], aq = A[q][k];
        A[p][k] = c * ap - s * aq;
        A[q][k] = s * ap + c * aq;
      }
      __syncthreads();
      // A <- A J (columns p, q), V <- V J
      for (int idx = tid; idx < (n / 2) * n; idx += 256) {
        const int r = idx / n, k = idx % n;
        const int p = rp[r], q = rq[r];
        const double c = rc[r], s = rs[r];
        const double ap = A[k][p], aq = A[k][q];
        A[k][p] = c * ap - s * aq;
        A[k][q] = s * ap + c * aq;
        const double vp = V[k][p], vq = V[k][q];
        V[k][p] = c * vp - s * vq;
        V[k][q] = s * vp + c * vq;
      }
      __syncthreads();
    }
  }
  // eigenvalues descending (stable: lower index first on ties)
  if (tid == 0) {
    for (int i = 0; i < E; ++i) order[i] = i;
    for (int i = 0; i < E; ++i)
      for (int j = i + 1; j < E; ++j)
        if (A[order[j]][order[j]] > A[order[i]][order[i]]) {
          const int t = order[i]; order[i] = order[j]; order[j] = t;
        }
  }
  __syncthreads();
  for (int idx = tid; idx < E * d; idx += 256) {
    const int e = idx / d, j = idx % d;
    const int col = order[j];
    const double lam = A[col][col] > 0.0 ? A[col][col] : 0.0;
    features[e * d + j] = (float)(V[e][col] * sqrt(lam));
  }
  if (eigvals)
    for (int j = tid; j < d; j += 256) eigvals[j] = (float)A[order[j]][order[j]];
}

// One CTA per layer; thread e = expert e.  Frequencies enter as the profiled counts (f = count / T
// is monotone in the count, so the initial ranking is the same).
__global__ void __launch_bounds__(kMaxE) kmeans_kernel(int E, int d, const float* __restrict__ features,
                                                       const int64_t* __restrict__ counts,
                                                       const __grid_constant__ KMeansArgs ka, int max_iter,
                                                       int32_t* __restrict__ cluster_of, int32_t* __restrict__ iters) {
  constexpr int kMaxD = 32;
  __shared__ double F[kMaxE][kMaxD];
  __shared__ double mu[kMaxE][kMaxD];
  __shared__ int init_rank[kMaxE];
  __shared__ int assign[kMaxE];
  const int l = blockIdx.x, e = threadIdx.x;
  const int B = ka.n_clusters[l];
  const uint64_t tmask = ka.tuning[l];
  const bool valid = e < E;
  const bool tun = valid && ((tmask >> e) & 1);
  if (valid)
    for (int j = 0; j < d; ++j) F[e][j] = (double)features[((int64_t)l * E + e) * d + j];
  // rank among non-tuning experts by (-freq, id)
  if (valid && !tun) {
    const int64_t fe = counts[l * E + e];
    int r = 0;
    for (int o = 0; o < E; ++o) {
      if ((tmask >> o) & 1) continue;
      const int64_t fo = counts[l * E + o];
      r += (fo > fe) || (fo == fe && o < e);
    }
    init_rank[e] = r;
  } else if (valid) {
    init_rank[e] = -1;
  }
  __syncthreads();
  if (valid && !tun && init_rank[e] < B)
    for (int j = 0; j < d; ++j) mu[init_rank[e]][j] = F[e][j];
  if (valid) assign[e] = -1;
  __syncthreads();
  int it = 0;
  for (it = 1; it <= max_iter; ++it) {
    int mine = -1;
    if (valid && !tun) {
      double nf = 0.0;
      for (int j = 0; j < d; ++j) nf += F[e][j] * F[e][j];
      nf = sqrt(nf);
      double best = INFINITY;
      for (int c = 0; c < B; ++c) {
        double dot = 0.0, nm = 0.0;
        for (int j = 0; j < d; ++j) {
          dot += F[e][j] * mu[c][j];
          nm += mu[c][j] * mu[c][j];
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
          for (int j = 0; j < d; ++j) acc[j] += F[o][j];
        }
      if (cnt)
        for (int j = 0; j < d; ++j) mu[e][j] = acc[j] / cnt;
    }
    __syncthreads();
    if (!changed) break;
  }
  if (valid) cluster_of[l * E + e] = assign[e];
  if (e == 0 && iters) iters[l] = it > max_iter ? max_iter : it;
}
}  // namespace

size_t features_workspace(int L, int n_fam) {
  return ((size_t)n_fam * kNumSMs + (size_t)L) * kMaxE * kMaxE * sizeof(float);
}

// Split-K Gram of one (layer, family) matrix X [E][P] into `partial` slots; returns the slot count.
cudaError_t launch_gram(int E, const void* X, int64_t P, float* partial, int* n_slots, cudaStream_t st) {
  CUtensorMap m;
  if (!make_tmap_2d(&m, X, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)E, (uint64_t)P, (uint64_t)P * 2, 64, kBM,
                    CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  const int64_t n_kb = (P + kBK - 1) / kBK;
  const int grid = (int)std::min<int64_t>(kNumSMs, std::max<int64_t>(n_kb, 1));
  const int smem = kStages * kBM * kBK * 2 + 1024 + 256;
  const int npad = E <= 16 ? 16 : E <= 32 ? 32 : 64;
  cudaError_t e;
  if (npad == 16) {
    e = cudaFuncSetAttribute(gram_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) gram_kernel<16><<<grid, 192, smem, st>>>(m, n_kb, E, partial);
  } else if (npad == 32) {
    e = cudaFuncSetAttribute(gram_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) gram_kernel<32><<<grid, 192, smem, st>>>(m, n_kb, E, partial);
  } else {
    e = cudaFuncSetAttribute(gram_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) gram_kernel<64><<<grid, 192, smem, st>>>(m, n_kb, E, partial);
  }
  if (e != cudaSuccess) return e;
  *n_slots = grid;
  return cudaGetLastError();
}

cudaError_t launch_gram_reduce(int E, const float* partial, int n_slots, float* G, float* G_user, cudaStream_t st) {
  gram_reduce_kernel<<<E, kMaxE, 0, st>>>(partial, n_slots, E, G, G_user);
  return cudaGetLastError();
}

cudaError_t launch_eig(int L, int E, int d, const float* G, float* features, float* eigvals, cudaStream_t st) {
  const int smem = 2 * kMaxE * (kMaxE + 1) * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  eig_kernel<<<L, 256, smem, st>>>(G, E, d, features, eigvals);
  return cudaGetLastError();
}

cudaError_t launch_kmeans(int L, int E, int d, const float* features, const int64_t* counts, const KMeansArgs& ka,
                          int max_iter, int32_t* cluster_of, int32_t* iters, cudaStream_t st) {
  kmeans_kernel<<<L, kMaxE, 0, st>>>(E, d, features, counts, ka, max_iter, cluster_of, iters);
  return cudaGetLastError();
}

}  // namespace flux
