// merge.cu — K7: importance-based merge of non-tuning experts, eq.(2)
// (P:827-839):  W_c = Σ_{e∈E_c} α_e / Σ_{e'∈E_c} α_e' · W_e.
// Reading R10: Σα = 0 -> plain mean; cluster_of = -1 marks a tuning expert
// (kept at full size); remap gives the compact slot (tuning
// experts first in ascending id, then clusters 0..C-1: exps_config,
// P:1013-1014).
//
// HBM-bound (read Σ|W_e| once, write Σ|W_c| once).  ONE launch covers a batch
// of jobs (a job = one weight family of one layer: the bench merges all L x 3
// families of a model in one persistent launch instead of 3L small ones, whose
// ramp-up / tail cost ~20% of each short launch).  The work is cut into chunks
// of 4,096 consecutive output elements (256 threads x 2 x 16-byte vectors);
// every CTA owns a CONTIGUOUS range of chunks (equal counts: balanced), so it
// rebuilds its member table only when its range crosses into the next output
// (cluster or job) — a few times per CTA.
//
// Per output: the member list (ascending expert id) and fp32 weights
// w_e = α_e / Σα (Σα accumulated in ascending id: deterministic) live in shared
// memory.  Threads load up to 4 members' vectors before the first FMA (bytes in
// flight per SM to cover HBM latency), accumulate w_e·W_e in fp32 (FMA chain in
// member order) and round once.  A singleton cluster has w = α/α = 1 exactly,
// so its output is the input bit for bit.
//
// Out-of-range labels: an expert whose cluster id is < -1 or >= n_clusters
// belongs to no output; an output with no member is written as zeros.
#include <algorithm>

#include "internal.h"
#include "ptx.cuh"

namespace flux {
namespace {

constexpr int kMaxE = 1024;
constexpr int kThreads = 256;
constexpr int kVecPerThread = 2;
constexpr int64_t kChunkVecs = (int64_t)kVecPerThread * kThreads;  // 16-byte vectors per chunk

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

struct SmemTable {
  int lab[kMaxE];    // output index of every expert of the current job (-1: none)
  int mem[kMaxE];    // members of the current output, ascending expert id
  float w[kMaxE];    // their weights
  int n_mem;
  int n_tun;
};

// Labels of the experts of job j.  slot(e) = the compact-model slot: tuning experts
// (cluster_of = -1) take 0..n_tun-1 in ascending id, cluster c takes n_tun + c; an out-of-range id has
// no slot (-1).  Output index: compact = 1 -> slot(e); compact = 0 -> c for cluster_of = c in [0, C),
// none (-1) for tuning experts.  remap (if any) = slot(e) in both modes.  Called by all threads.
__device__ void build_labels(const MergeJob& job, int E, int compact, SmemTable& t) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();  // every thread is done with the previous job's tables
  if (wid == 0) {
    int n_tun = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      n_tun += __popc(__ballot_sync(0xffffffffu, e < E && __ldg(&job.cluster_of[e]) == -1));
    }
    int rank0 = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      const int cl = e < E ? __ldg(&job.cluster_of[e]) : -2;
      const unsigned tun = __ballot_sync(0xffffffffu, cl == -1);
      const bool in_range = cl >= 0 && cl < job.n_clusters;
      const int slot = cl == -1 ? rank0 + __popc(tun & ((1u << lane) - 1u)) : in_range ? n_tun + cl : -1;
      if (e < E) {
        t.lab[e] = compact ? slot : (in_range ? cl : -1);
        if (job.remap) job.remap[e] = slot;
      }
      rank0 += __popc(tun);
    }
    if (lane == 0) t.n_tun = n_tun;
  }
  __syncthreads();
}

// Members (ascending id) and weights of output o of the current job.  Called by all threads.
__device__ void build_members(const MergeJob& job, int E, int o, SmemTable& t) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();  // every thread is done with the previous output's members
  if (wid == 0) {
    int n = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      const bool m = e < E && t.lab[e] == o;
      const unsigned b = __ballot_sync(0xffffffffu, m);
      if (m) t.mem[n + __popc(b & ((1u << lane) - 1u))] = e;
      n += __popc(b);
    }
    __syncwarp();
    if (lane == 0) {
      float asum = 0.f;
      for (int i = 0; i < n; ++i) asum += __ldg(&job.alpha[t.mem[i]]);  // ascending id
      for (int i = 0; i < n; ++i)
        t.w[i] = asum > 0.f ? __fdiv_rn(__ldg(&job.alpha[t.mem[i]]), asum) : __fdiv_rn(1.f, (float)n);
      t.n_mem = n;
    }
  }
  __syncthreads();
}

template <bool F32>
__device__ __forceinline__ void merge_chunk(const MergeJob& job, int64_t numel, int o, int64_t v0,
                                            const SmemTable& t) {
  const int64_t nvec = numel / 8;
  float acc[kVecPerThread][8];
#pragma unroll
  for (int u = 0; u < kVecPerThread; ++u)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[u][i] = 0.f;
  const int m_end = t.n_mem;
  for (int m0 = 0; m0 < m_end; m0 += 4) {
    Raw<F32> r[4][kVecPerThread];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (m0 + j < m_end) {
        const int64_t base = (int64_t)t.mem[m0 + j] * numel;
#pragma unroll
        for (int u = 0; u < kVecPerThread; ++u) {
          const int64_t v = v0 + (int64_t)u * kThreads;
          if (v < nvec) load_raw<F32>(job.experts, base + v * 8, r[j][u]);
        }
      }
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (m0 + j < m_end) {
        const float wm = t.w[m0 + j];
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
    const int64_t v = v0 + (int64_t)u * kThreads;
    if (v < nvec) store_vec<F32>(job.merged, (int64_t)o * numel + v * 8, acc[u]);
  }
}

// chunk_prefix[j] = first chunk of job j (chunks of job j = n_out_j · chunks per output).
// contiguous = 1: CTA b owns chunks [b·n/G, (b+1)·n/G); 0: chunks dealt round-robin (single-job calls
// whose output count is only an upper bound, compact mode).
template <bool F32>
__global__ void __launch_bounds__(kThreads) merge_batch_kernel(MergeBatch b) {
  __shared__ SmemTable t;
  const int64_t nvec = b.numel / 8;
  const int64_t cpo = (nvec + kChunkVecs - 1) / kChunkVecs;  // chunks per output
  const int64_t total = b.chunk_prefix[b.n_jobs];
  int64_t ch0, ch1, step;
  if (b.contiguous) {
    const int64_t per = (total + gridDim.x - 1) / gridDim.x;
    ch0 = (int64_t)blockIdx.x * per;
    ch1 = min(total, ch0 + per);
    step = 1;
  } else {
    ch0 = blockIdx.x;
    ch1 = total;
    step = gridDim.x;
  }
  int j = 0, cur_job = -1, cur_o = -1;
  for (int64_t ch = ch0; ch < ch1; ch += step) {
    while (ch >= b.chunk_prefix[j + 1]) ++j;
    const int64_t local = ch - b.chunk_prefix[j];
    const int o = (int)(local / cpo);
    const int64_t v0 = (local - (int64_t)o * cpo) * kChunkVecs + threadIdx.x;
    if (j != cur_job) {
      build_labels(b.jobs[j], b.E, b.compact, t);
      cur_job = j;
      cur_o = -1;
    }
    if (b.compact && o >= t.n_tun + b.jobs[j].n_clusters) continue;  // beyond the job's slots (upper bound)
    if (o != cur_o) {
      build_members(b.jobs[j], b.E, o, t);
      cur_o = o;
    }
    merge_chunk<F32>(b.jobs[j], b.numel, o, v0, t);
  }
}
}  // namespace

cudaError_t launch_merge_batch(bool fp32, const MergeBatch& b0, cudaStream_t st) {
  MergeBatch b = b0;
  const int64_t cpo = (b.numel / 8 + kChunkVecs - 1) / kChunkVecs;
  b.chunk_prefix[0] = 0;
  for (int j = 0; j < b.n_jobs; ++j) {
    const int64_t n_out = b.compact ? (b.jobs[j].n_slots > 0 ? b.jobs[j].n_slots : b.E) : b.jobs[j].n_clusters;
    b.chunk_prefix[j + 1] = b.chunk_prefix[j] + n_out * cpo;
  }
  const int64_t total = b.chunk_prefix[b.n_jobs];
  if (total == 0) return cudaSuccess;
  // one resident wave: 3 (bf16) / 2 (fp32) CTAs per SM
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(total, (int64_t)kNumSMs * (fp32 ? 2 : 3)));
  if (fp32)
    merge_batch_kernel<true><<<grid, kThreads, 0, st>>>(b);
  else
    merge_batch_kernel<false><<<grid, kThreads, 0, st>>>(b);
  return cudaGetLastError();
}

cudaError_t launch_merge(bool fp32, int E, int64_t numel, const void* experts, const int32_t* cluster_of,
                         const float* alpha, int C, void* merged, int32_t* remap, cudaStream_t st, int compact) {
  MergeBatch b{};
  b.n_jobs = 1;
  b.E = E;
  b.numel = numel;
  b.compact = compact;
  b.contiguous = compact ? 0 : 1;  // compact: the slot count (n_tun + C) is known only on the device
  b.jobs[0] = MergeJob{experts, cluster_of, alpha, merged, remap, C, 0};
  return launch_merge_batch(fp32, b, st);
}

}  // namespace flux
