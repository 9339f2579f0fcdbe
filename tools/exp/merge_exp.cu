// Experiment (not product code): merge kernel variants for the power-capped A/B of DESIGN.md §5.1.
// Built by tools/exp/merge_exp.py into tools/exp/libmerge_exp.so.  All variants compute the same
// outputs as K7 (balanced clusters, member order, fp32 FMA chain, one rounding).
#include <cuda_bf16.h>
#include <stdint.h>
#include <algorithm>

namespace {
constexpr int kMaxE = 128;

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

struct Job { const uint4* ex; const int* cl; const float* al; uint4* out; int C; };
struct Batch { int n_jobs, E; long long nvec; Job jobs[96]; };

// V2: register-based, round-robin chunks of `VPT`·256 vectors, all members' loads of a chunk in flight.
template <int VPT>
__global__ void __launch_bounds__(256) merge_reg(const __grid_constant__ Batch b) {
  __shared__ int s_mem[kMaxE], s_start[kMaxE + 1];
  __shared__ float s_w[kMaxE];
  __shared__ int s_job;
  const long long per = (long long)VPT * 256;
  const long long cpo = (b.nvec + per - 1) / per;
  long long total = 0;
  for (int j = 0; j < b.n_jobs; ++j) total += (long long)b.jobs[j].C * cpo;
  if (threadIdx.x == 0) s_job = -1;
  __syncthreads();
  for (long long ch = blockIdx.x; ch < total; ch += gridDim.x) {
    long long rem = ch;
    int j = 0;
    while (rem >= (long long)b.jobs[j].C * cpo) { rem -= (long long)b.jobs[j].C * cpo; ++j; }
    const Job& J = b.jobs[j];
    if (j != s_job) {
      __syncthreads();
      if (threadIdx.x == 0) {
        int n = 0;
        for (int c = 0; c < J.C; ++c) {
          s_start[c] = n;
          float as = 0.f;
          int m0 = n;
          for (int e = 0; e < b.E; ++e) if (J.cl[e] == c) { s_mem[n++] = e; as += J.al[e]; }
          for (int i = m0; i < n; ++i) s_w[i] = as > 0.f ? __fdiv_rn(J.al[s_mem[i]], as) : __fdiv_rn(1.f, (float)(n - m0));
        }
        s_start[J.C] = n;
        s_job = j;
      }
      __syncthreads();
    }
    const int c = (int)(rem / cpo);
    const long long v0 = (rem - (long long)c * cpo) * per + threadIdx.x;
    float acc[VPT][8];
#pragma unroll
    for (int u = 0; u < VPT; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[u][i] = 0.f;
    const int m0 = s_start[c], m1 = s_start[c + 1];
    for (int m = m0; m < m1; m += 4) {
      uint4 r[4][VPT];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (m + q < m1) {
#pragma unroll
          for (int u = 0; u < VPT; ++u) {
            const long long v = v0 + (long long)u * 256;
            if (v < b.nvec) r[q][u] = __ldcs(J.ex + (long long)s_mem[m + q] * b.nvec + v);
          }
        }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (m + q < m1) {
          const float w = s_w[m + q];
#pragma unroll
          for (int u = 0; u < VPT; ++u) {
            const uint32_t x[4] = {r[q][u].x, r[q][u].y, r[q][u].z, r[q][u].w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              acc[u][2 * i] = fmaf(w, __uint_as_float(x[i] << 16), acc[u][2 * i]);
              acc[u][2 * i + 1] = fmaf(w, __uint_as_float(x[i] & 0xffff0000u), acc[u][2 * i + 1]);
            }
          }
        }
    }
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const long long v = v0 + (long long)u * 256;
      if (v < b.nvec)
        __stcs(J.out + (long long)c * b.nvec + v, make_uint4(pack2(acc[u][0], acc[u][1]), pack2(acc[u][2], acc[u][3]),
                                                             pack2(acc[u][4], acc[u][5]), pack2(acc[u][6], acc[u][7])));
    }
  }
}
}  // namespace

extern "C" int merge_exp(int variant, int blocks_per_sm, int n_jobs, int E, long long numel, void* const* ex,
                         const int* const* cl, const float* const* al, void* const* out, const int* C, void* stream) {
  Batch b{};
  b.n_jobs = n_jobs;
  b.E = E;
  b.nvec = numel / 8;
  for (int j = 0; j < n_jobs; ++j) b.jobs[j] = Job{(const uint4*)ex[j], cl[j], al[j], (uint4*)out[j], C[j]};
  const unsigned grid = 148 * blocks_per_sm;
  cudaStream_t st = (cudaStream_t)stream;
  if (variant == 1) merge_reg<1><<<grid, 256, 0, st>>>(b);
  else if (variant == 2) merge_reg<2><<<grid, 256, 0, st>>>(b);
  else if (variant == 4) merge_reg<4><<<grid, 256, 0, st>>>(b);
  return (int)cudaGetLastError();
}
