// merge.cu — K7: importance-based merge of non-tuning experts, eq.(2)
// (P:827-839):  W_c = Σ_{e∈E_c} α_e / Σ_{e'∈E_c} α_e' · W_e.
// Reading R10: Σα = 0 -> plain mean; cluster_of = -1 marks a tuning expert
// (kept at full size); remap gives the compact slot (tuning
// experts first in ascending id, then clusters 0..C-1: exps_config,
// P:1013-1014).
//
// HBM-bound (read Σ|W_e| once, write Σ|W_c| once).  Every CTA builds the
// member lists and fp32 weights of all clusters in shared memory (members in
// ascending expert id, Σα accumulated in that order: deterministic); threads
// then own 8 consecutive elements of one cluster output, load each member's
// 16-byte vector, accumulate w_e·W_e in fp32 (FMA chain in member order) and
// round once.  A singleton cluster has w = α/α = 1 exactly, so its output is
// the input bit for bit.
#include "internal.h"
#include "ptx.cuh"

namespace flux {
namespace {

constexpr int kMaxE = 1024;

template <bool F32>
__device__ __forceinline__ void load_vec(const void* base, int64_t elem, float (&f)[8]) {
  if constexpr (F32) {
    const float4* p = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base) + elem);
    const float4 a = __ldcs(p), b = __ldcs(p + 1);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  } else {
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(base) + elem));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 p = __bfloat1622float2(h[i]);
      f[2 * i] = p.x;
      f[2 * i + 1] = p.y;
    }
  }
}

template <bool F32>
__device__ __forceinline__ void store_vec(void* base, int64_t elem, const float (&f)[8]) {
  if constexpr (F32) {
    float4* p = reinterpret_cast<float4*>(reinterpret_cast<float*>(base) + elem);
    __stcs(p, make_float4(f[0], f[1], f[2], f[3]));
    __stcs(p + 1, make_float4(f[4], f[5], f[6], f[7]));
  } else {
    uint4 o;
    o.x = pack_bf16x2(f[0], f[1]);
    o.y = pack_bf16x2(f[2], f[3]);
    o.z = pack_bf16x2(f[4], f[5]);
    o.w = pack_bf16x2(f[6], f[7]);
    __stcs(reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(base) + elem), o);
  }
}

// compact = 0: outputs are the C clusters.  compact = 1 (NEXT-2): outputs are the slots of the
// compact model in remap order — every tuning expert as its own slot (ascending id; a singleton
// with weight α/α = 1, so its copy is bit-exact), then the C clusters.
template <bool F32>
__global__ void __launch_bounds__(256) merge_kernel(int E, int64_t numel, const void* __restrict__ experts,
                                                    const int32_t* __restrict__ cluster_of,
                                                    const float* __restrict__ alpha, int C, void* __restrict__ merged,
                                                    int32_t* __restrict__ remap, int compact) {
  __shared__ int s_cl[kMaxE];
  __shared__ float s_w[kMaxE];       // weight of member slot
  __shared__ int s_mem[kMaxE];       // member expert ids grouped by cluster
  __shared__ int s_start[kMaxE + 1]; // cluster -> first member slot
  __shared__ int s_ntun;
  for (int e = threadIdx.x; e < E; e += blockDim.x) s_cl[e] = cluster_of[e];
  __syncthreads();
  if (compact) {  // relabel: tuning expert -> its rank among tuning experts, cluster c -> n_tun + c
    if (threadIdx.x == 0) {
      int n = 0;
      for (int e = 0; e < E; ++e) n += s_cl[e] < 0;
      s_ntun = n;
    }
    __syncthreads();
    const int n_tun = s_ntun;
    __syncthreads();
    if (threadIdx.x == 0) {
      int r = 0;
      for (int e = 0; e < E; ++e) s_cl[e] = s_cl[e] < 0 ? r++ : n_tun + s_cl[e];
    }
    C += n_tun;
    __syncthreads();
  }
  // per cluster: count, Σα (ascending e), then the member slots
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    int cnt = 0;
    for (int e = 0; e < E; ++e) cnt += s_cl[e] == c;
    s_start[c + 1] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    s_start[0] = 0;
    for (int c = 0; c < C; ++c) s_start[c + 1] += s_start[c];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    float asum = 0.f;
    int cnt = 0;
    for (int e = 0; e < E; ++e)
      if (s_cl[e] == c) {
        asum += __ldg(&alpha[e]);
        s_mem[s_start[c] + cnt++] = e;
      }
    for (int i = 0; i < cnt; ++i) {
      const int e = s_mem[s_start[c] + i];
      s_w[s_start[c] + i] = asum > 0.f ? __fdiv_rn(__ldg(&alpha[e]), asum) : __fdiv_rn(1.f, (float)cnt);
    }
  }
  __syncthreads();
  if (remap && blockIdx.x == 0 && threadIdx.x == 0) {
    if (compact) {
      for (int e = 0; e < E; ++e) remap[e] = s_cl[e];
    } else {
      int slot = 0;
      for (int e = 0; e < E; ++e)
        if (s_cl[e] == -1) remap[e] = slot++;
      for (int e = 0; e < E; ++e)
        if (s_cl[e] >= 0) remap[e] = slot + s_cl[e];
    }
  }
  const int64_t nvec = numel / 8;
  const int64_t items = (int64_t)C * nvec;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(it / nvec);
    const int64_t v = it - (int64_t)c * nvec;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int m = s_start[c]; m < s_start[c + 1]; ++m) {
      float f[8];
      load_vec<F32>(experts, (int64_t)s_mem[m] * numel + v * 8, f);
      const float wm = s_w[m];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fmaf(wm, f[i], acc[i]);
    }
    store_vec<F32>(merged, (int64_t)c * numel + v * 8, acc);
  }
}
}  // namespace

cudaError_t launch_merge(bool fp32, int E, int64_t numel, const void* experts, const int32_t* cluster_of,
                         const float* alpha, int C, void* merged, int32_t* remap, cudaStream_t st, int compact) {
  const int64_t items = (int64_t)(compact ? E : C) * (numel / 8);  // upper bound for the compact case
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, (int64_t)kNumSMs * 8));
  if (fp32)
    merge_kernel<true><<<grid, 256, 0, st>>>(E, numel, experts, cluster_of, alpha, C, merged, remap, compact);
  else
    merge_kernel<false><<<grid, 256, 0, st>>>(E, numel, experts, cluster_of, alpha, C, merged, remap, compact);
  return cudaGetLastError();
}

}  // namespace flux
