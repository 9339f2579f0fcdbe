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
// then own 2 × 8 elements of one cluster output, load up to 4 members' 16-byte
// vectors at once, accumulate w_e·W_e in fp32 (FMA chain in member order) and
// round once.  A singleton cluster has w = α/α = 1 exactly, so its output is
// the input bit for bit.
#include "internal.h"
#include "ptx.cuh"

namespace flux {
namespace {

constexpr int kMaxE = 1024;
constexpr int kVecPerThread = 2;

// One 8-element vector kept raw until its FMA (bf16: one uint4 = 4 registers), so a thread can
// hold many loads in flight.
template <bool F32> struct Raw;
template <> struct Raw<false> { uint4 a; };
template <> struct Raw<true> { float4 a, b; };

template <bool F32>
__device__ __forceinline__ void load_raw(const void* base, int64_t elem, Raw<F32>& r) {
  if constexpr (F32) {
    const float4* p = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base) + elem);
    r.a = __ldcs(p);
    r.b = __ldcs(p + 1);
  } else {
    r.a = __ldcs(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(base) + elem));
  }
}

template <bool F32>
__device__ __forceinline__ void to_f32(const Raw<F32>& r, float (&f)[8]) {
  if constexpr (F32) {
    f[0] = r.a.x; f[1] = r.a.y; f[2] = r.a.z; f[3] = r.a.w;
    f[4] = r.b.x; f[5] = r.b.y; f[6] = r.b.z; f[7] = r.b.w;
  } else {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r.a);
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
  __shared__ float s_alpha[kMaxE];
  __shared__ int s_ntun;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    s_cl[e] = cluster_of[e];
    s_alpha[e] = alpha[e];
  }
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
        asum += s_alpha[e];
        s_mem[s_start[c] + cnt++] = e;
      }
    for (int i = 0; i < cnt; ++i) {
      const int e = s_mem[s_start[c] + i];
      s_w[s_start[c] + i] = asum > 0.f ? __fdiv_rn(s_alpha[e], asum) : __fdiv_rn(1.f, (float)cnt);
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
  // Main loop: a CTA owns chunks of kVecPerThread·blockDim.x consecutive 16-byte vectors of one
  // output (chunks dealt round-robin, so at any moment the CTAs stream neighbouring addresses);
  // each thread issues the loads of up to 4 members × kVecPerThread vectors before the first FMA
  // (bytes in flight per SM to cover HBM latency), then accumulates in member order — the same FMA
  // chain as one member at a time, so results are unchanged bit for bit.
  const int64_t nvec = numel / 8;
  const int64_t per_chunk = (int64_t)kVecPerThread * blockDim.x;
  const int64_t chunks_per_c = (nvec + per_chunk - 1) / per_chunk;
  const int64_t chunks = (int64_t)C * chunks_per_c;
  for (int64_t ch = blockIdx.x; ch < chunks; ch += gridDim.x) {
    const int c = (int)(ch / chunks_per_c);
    const int64_t v0 = (ch - (int64_t)c * chunks_per_c) * per_chunk + threadIdx.x;
    float acc[kVecPerThread][8];
#pragma unroll
    for (int u = 0; u < kVecPerThread; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[u][i] = 0.f;
    const int m_end = s_start[c + 1];
    for (int m0 = s_start[c]; m0 < m_end; m0 += 4) {
      Raw<F32> r[4][kVecPerThread];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (m0 + j < m_end) {
          const int64_t base = (int64_t)s_mem[m0 + j] * numel;
#pragma unroll
          for (int u = 0; u < kVecPerThread; ++u) {
            const int64_t v = v0 + (int64_t)u * blockDim.x;
            if (v < nvec) load_raw<F32>(experts, base + v * 8, r[j][u]);
          }
        }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (m0 + j < m_end) {
          const float wm = s_w[m0 + j];
#pragma unroll
          for (int u = 0; u < kVecPerThread; ++u) {
            float f[8];
            to_f32<F32>(r[j][u], f);
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[u][i] = fmaf(wm, f[i], acc[u][i]);
          }
        }
    }
#pragma unroll
    for (int u = 0; u < kVecPerThread; ++u) {
      const int64_t v = v0 + (int64_t)u * blockDim.x;
      if (v < nvec) store_vec<F32>(merged, (int64_t)c * numel + v * 8, acc[u]);
    }
  }
}
}  // namespace

cudaError_t launch_merge(bool fp32, int E, int64_t numel, const void* experts, const int32_t* cluster_of,
                         const float* alpha, int C, void* merged, int32_t* remap, cudaStream_t st, int compact) {
  const int64_t per_chunk = (int64_t)kVecPerThread * 256;
  const int64_t chunks = (int64_t)(compact ? E : C) * ((numel / 8 + per_chunk - 1) / per_chunk);  // upper bound (compact)
  const unsigned grid = (unsigned)std::max<int64_t>(  // one resident wave: 3 (bf16) / 2 (fp32) CTAs per SM
      1, std::min<int64_t>(chunks, (int64_t)kNumSMs * (fp32 ? 2 : 3)));
  if (fp32)
    merge_kernel<true><<<grid, 256, 0, st>>>(E, numel, experts, cluster_of, alpha, C, merged, remap, compact);
  else
    merge_kernel<false><<<grid, 256, 0, st>>>(E, numel, experts, cluster_of, alpha, C, merged, remap, compact);
  return cudaGetLastError();
}

}  // namespace flux
