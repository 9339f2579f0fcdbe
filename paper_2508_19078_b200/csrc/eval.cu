// eval.cu — statistics beside the layer forward:
//  * attention_hist_kernel (NEXT-3): the attention-weighted activation counts of eq.(2)'s α = f·ā;
//  * cosine_distance_kernel (NEXT-2): the paper's merge-quality measure, "the average cosine distance between the
// final token embeddings from the MoE model with merged experts and those from the original full
// model":  err = (1/T) Σ_t (1 - a_t·b_t / (|a_t| |b_t|)).
//
// HBM-bound (reads both [T][H] bf16 outputs once).  One warp per token (16-byte vectors, fp64
// accumulation); each CTA sums its tokens' distances in token order, and the last CTA to finish
// (atomic ticket) sums the CTA partials in CTA order: deterministic.
#include "internal.h"
#include "ptx.cuh"

namespace flux {
namespace {

constexpr int kCosBlocks = kNumSMs * 4, kCosThreads = 256;

__global__ void __launch_bounds__(kCosThreads) cosine_distance_kernel(int64_t T, int H, const uint4* __restrict__ a,
                                                                      const uint4* __restrict__ b,
                                                                      double* __restrict__ partial,
                                                                      unsigned* __restrict__ ticket,
                                                                      double* __restrict__ out) {
  __shared__ double warp_sum[kCosThreads / 32];
  __shared__ bool is_last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nvec = H / 8;
  double my = 0.0;  // this warp's tokens, in token order
  for (int64_t t = (int64_t)blockIdx.x * (kCosThreads / 32) + wid; t < T; t += (int64_t)gridDim.x * (kCosThreads / 32)) {
    double dot = 0.0, na = 0.0, nb = 0.0;
    for (int v = lane; v < nvec; v += 32) {
      const uint4 x = __ldcs(&a[t * nvec + v]), y = __ldcs(&b[t * nvec + v]);
      const __nv_bfloat162* hx = reinterpret_cast<const __nv_bfloat162*>(&x);
      const __nv_bfloat162* hy = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 fx = __bfloat1622float2(hx[i]), fy = __bfloat1622float2(hy[i]);
        dot += (double)fx.x * fy.x + (double)fx.y * fy.y;
        na += (double)fx.x * fx.x + (double)fx.y * fx.y;
        nb += (double)fy.x * fy.x + (double)fy.y * fy.y;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dot += __shfl_xor_sync(0xffffffffu, dot, o);
      na += __shfl_xor_sync(0xffffffffu, na, o);
      nb += __shfl_xor_sync(0xffffffffu, nb, o);
    }
    my += (na == 0.0 || nb == 0.0) ? 1.0 : 1.0 - dot / (sqrt(na) * sqrt(nb));
  }
  if (lane == 0) warp_sum[wid] = my;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kCosThreads / 32; ++w) s += warp_sum[w];
    partial[blockIdx.x] = s;
    __threadfence();
    is_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (is_last && threadIdx.x == 0) {
    __threadfence();
    double s = 0.0;
    for (unsigned i = 0; i < gridDim.x; ++i) s += __ldcg(&partial[i]);
    *out = T ? s / (double)T : 0.0;
    *ticket = 0;  // ready for the next call
  }
}

// NEXT-3 (eq.(2) α = f·ā, reading R15): A_e += RNE(a_t · 2^24) over the live picks of
// every token.  Integer sums: exact and order-free (deterministic and identical under any split of
// the tokens, like the histogram).  Per-CTA shared-memory accumulators, one global atomic per expert.
__global__ void __launch_bounds__(256) attention_hist_kernel(int64_t T, int k, int E, const int32_t* __restrict__ ids,
                                                             const float* __restrict__ attn,
                                                             unsigned long long* __restrict__ A) {
  __shared__ unsigned long long acc[1024];
  for (int e = threadIdx.x; e < E; e += blockDim.x) acc[e] = 0ull;
  __syncthreads();
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    const long long a = __double2ll_rn((double)__ldg(&attn[t]) * 16777216.0);  // exact product, RNE
    for (int j = 0; j < k; ++j) {
      const int e = __ldg(&ids[t * k + j]);
      if (e >= 0) atomicAdd(&acc[e], (unsigned long long)a);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    if (acc[e]) atomicAdd(&A[e], acc[e]);
}
// α_e = fl32(count_e / denom) (fp64 quotient, one rounding): the activation frequency f = count / T
// (denom = T) or the attention-weighted α = A / (2^24·T) (R15), on the device, so a
// participant round needs no host round trip between the reduced statistics and the merge.
__global__ void __launch_bounds__(256) frequencies_kernel(int64_t n, const int64_t* __restrict__ counts, double denom,
                                                          float* __restrict__ alpha) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    alpha[i] = __double2float_rn((double)counts[i] / denom);
}
}  // namespace

cudaError_t launch_frequencies(int64_t n, const int64_t* counts, double denom, float* alpha, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, kNumSMs);
  frequencies_kernel<<<grid, 256, 0, st>>>(n, counts, denom, alpha);
  return cudaGetLastError();
}

cudaError_t launch_attention_hist(int64_t T, int k, int E, const int32_t* ids, const float* attn, int64_t* A,
                                  cudaStream_t st) {
  if (T == 0) return cudaSuccess;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((T + 255) / 256, kNumSMs * 2));
  attention_hist_kernel<<<grid, 256, 0, st>>>(T, k, E, ids, attn, reinterpret_cast<unsigned long long*>(A));
  return cudaGetLastError();
}

size_t cosine_workspace() { return (kCosBlocks + 2) * sizeof(double); }

cudaError_t launch_cosine_distance(int64_t T, int H, const void* a, const void* b, double* ws, double* out,
                                   cudaStream_t st) {
  unsigned* ticket = reinterpret_cast<unsigned*>(ws + kCosBlocks);
  cudaError_t e = cudaMemsetAsync(ticket, 0, sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  const int64_t want = (T + kCosThreads / 32 - 1) / (kCosThreads / 32);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, kCosBlocks));
  cosine_distance_kernel<<<grid, kCosThreads, 0, st>>>(T, H, (const uint4*)a, (const uint4*)b, ws, ticket, out);
  return cudaGetLastError();
}

}  // namespace flux
