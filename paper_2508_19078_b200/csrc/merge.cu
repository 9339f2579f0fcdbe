// merge.cu — K7: importance-based merge of non-tuning experts, eq.(2)
// (P:827-839):  W_c = Σ_{e∈E_c} α_e / Σ_{e'∈E_c} α_e' · W_e.
// Reading R10: Σα = 0 -> plain mean; cluster_of = -1 marks a tuning expert
// (kept at full size); remap gives the compact slot (tuning
// experts first in ascending id, then clusters 0..C-1: exps_config,
// P:1013-1014).
//
// HBM-bound (read Σ|W_e| once, write Σ|W_c| once).  ONE persistent launch
// covers a batch of jobs (a job = one weight family of one layer: the bench
// merges all L x 3 families of a model in one launch instead of 3L small ones).
// The work is cut into chunks of 8 KB of consecutive output elements, dealt
// round-robin over one CTA per SM, and streamed with TMA bulk copies through a
// 6-stage shared-memory ring (192 KB of reads in flight per SM; see the kernel).
//
// Per output: the member list (ascending expert id) and fp32 weights
// w_e = α_e / Σα (Σα accumulated in ascending id: deterministic); the FMA chain
// runs in member order in fp32 and rounds once.  A singleton cluster has
// w = α/α = 1 exactly, so its output is the input bit for bit.
//
// Out-of-range labels: an expert whose cluster id is < -1 or >= n_clusters
// belongs to no output; an output with no member is written as zeros.
#include <algorithm>

#include "internal.h"
#include "ptx.cuh"

namespace flux {
namespace {

constexpr int kMaxE = 1024;
// ------------------------------------------------------------------ TMA-bulk pipelined batch kernel
// Warp 0 (producer, one elected lane) walks this CTA's chunks (dealt round-robin over the grid, so at any
// moment the CTAs stream neighbouring addresses), and per chunk issues one 1D bulk copy (cp.async.bulk)
// per member into a ring of kStages stages of 4 member slices each (8 KB per slice); a chunk of a
// cluster with m members takes ceil(m / 4) stages.  The stage header carries the members' weights and
// the output address.  Warps 1..8 (consumers) accumulate w_e·W_e in fp32 registers from shared memory
// (FMA chain in member order, as the per-job kernel), and after the chunk's last stage round once and
// store 16-byte vectors.  The producer keeps the job's member table (all outputs: members in ascending
// id, weights α_e / Σα with Σα in ascending id) in shared memory, rebuilt when the job changes.
constexpr int kSlice = 8192;                  // bytes of one member slice (one chunk of one expert)
constexpr int kSlicesPerStage = 4;
constexpr int kStages = 6;                    // 6 x 32 KB = 192 KB of HBM reads in flight per SM
constexpr int kConsumers = 256;
constexpr int kBThreads = 32 + kConsumers;

struct StageHdr {
  float w[kSlicesPerStage];
  void* out;       // output vector base of this chunk (null when the stage is not the chunk's last)
  int n;           // member slices in this stage
  int nvec;        // 16-byte vectors in this chunk
  int first;       // 1: the chunk's first stage (reset the accumulators)
  int pad;
};

struct BatchSmem {
  uint8_t data[kStages][kSlicesPerStage][kSlice];
  StageHdr hdr[kStages];
  uint64_t full[kStages], empty[kStages];
  int lab[kMaxE];       // output index of every expert of the current job (-1: none)
  int start[kMaxE + 2]; // output -> first member slot
  int mem[kMaxE];       // members grouped by output, ascending id
  float w[kMaxE];
  int fill[kMaxE + 1];
};

// Producer-warp helpers (all 32 lanes).
__device__ int build_job_table(const MergeJob& job, int E, int compact, bool write_remap, BatchSmem& t) {
  const int lane = threadIdx.x & 31;
  int n_tun = 0;
  for (int e0 = 0; e0 < E; e0 += 32) {
    const int e = e0 + lane;
    n_tun += __popc(__ballot_sync(0xffffffffu, e < E && __ldg(&job.cluster_of[e]) == -1));
  }
  const int n_out = compact ? n_tun + job.n_clusters : job.n_clusters;
  for (int o = lane; o <= n_out; o += 32) {
    t.start[o] = 0;
    t.fill[o] = 0;
  }
  __syncwarp();
  int rank0 = 0;
  for (int e0 = 0; e0 < E; e0 += 32) {
    const int e = e0 + lane;
    const int cl = e < E ? __ldg(&job.cluster_of[e]) : -2;
    const unsigned tun = __ballot_sync(0xffffffffu, cl == -1);
    const bool in_range = cl >= 0 && cl < job.n_clusters;
    const int slot = cl == -1 ? rank0 + __popc(tun & ((1u << lane) - 1u)) : in_range ? n_tun + cl : -1;
    if (e < E) {
      const int lab = compact ? slot : (in_range ? cl : -1);
      t.lab[e] = lab;
      if (write_remap && job.remap) job.remap[e] = slot;
      if (lab >= 0) atomicAdd(&t.start[lab + 1], 1);
    }
    rank0 += __popc(tun);
  }
  __syncwarp();
  if (lane == 0)
    for (int o = 0; o < n_out; ++o) t.start[o + 1] += t.start[o];
  __syncwarp();
  for (int e0 = 0; e0 < E; e0 += 32) {  // members in ascending id within every output
    const int e = e0 + lane;
    const int lab = e < E ? t.lab[e] : -1;
    const unsigned same = __match_any_sync(0xffffffffu, lab);
    if (lab >= 0) {
      const int r = __popc(same & ((1u << lane) - 1u));
      t.mem[t.start[lab] + t.fill[lab] + r] = e;
    }
    __syncwarp();
    if (lab >= 0 && __ffs(same) - 1 == lane) t.fill[lab] += __popc(same);
    __syncwarp();
  }
  for (int o = lane; o < n_out; o += 32) {  // Σα in ascending id, then α_e / Σα (or 1/|E_c|)
    const int b = t.start[o], n = t.start[o + 1] - b;
    float asum = 0.f;
    for (int i = 0; i < n; ++i) asum += __ldg(&job.alpha[t.mem[b + i]]);
    for (int i = 0; i < n; ++i)
      t.w[b + i] = asum > 0.f ? __fdiv_rn(__ldg(&job.alpha[t.mem[b + i]]), asum) : __fdiv_rn(1.f, (float)n);
  }
  __syncwarp();
  return n_out;
}

template <bool F32>
__global__ void __launch_bounds__(kBThreads, 1) merge_tma_kernel(const __grid_constant__ MergeBatch b) {
  extern __shared__ uint8_t smem_raw[];
  BatchSmem& t = *reinterpret_cast<BatchSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  constexpr int kEsz = F32 ? 4 : 2;
  constexpr int kChunkElems = kSlice / kEsz;
  const int64_t cpo = (b.numel + kChunkElems - 1) / kChunkElems;  // chunks per output
  const int64_t total = b.chunk_prefix[b.n_jobs];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&t.full[s], 1);
      mbar_init(&t.empty[s], kConsumers / 32);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    const uint64_t pol = policy_evict_first();
    int j = 0, cur_job = -1, n_out = 0, g = 0;
    for (int64_t ch = blockIdx.x; ch < total; ch += gridDim.x) {
      while (ch >= b.chunk_prefix[j + 1]) ++j;
      const int64_t local = ch - b.chunk_prefix[j];
      const int o = (int)(local / cpo);
      const int64_t c_in = local - (int64_t)o * cpo;
      const MergeJob& job = b.jobs[j];
      if (j != cur_job) {
        n_out = build_job_table(job, b.E, b.compact, b.chunk_prefix[j] % gridDim.x == blockIdx.x, t);
        cur_job = j;
      }
      if (o >= n_out) continue;  // compact single-job calls: the slot count was an upper bound
      const int64_t e0 = c_in * kChunkElems;
      const int n_elems = (int)(b.numel - e0 < kChunkElems ? b.numel - e0 : kChunkElems);
      const uint32_t bytes = (uint32_t)n_elems * kEsz;
      const int m0 = t.start[o], m1 = t.start[o + 1];
      int m = m0;
      do {  // one stage per group of up to 4 members (an output with no member still takes one stage)
        const int s = g % kStages;
        mbar_wait(&t.empty[s], ((g / kStages) & 1) ^ 1);
        const int n = min(kSlicesPerStage, m1 - m);
        if ((threadIdx.x & 31) == 0) {
          StageHdr& h = t.hdr[s];
          for (int i = 0; i < kSlicesPerStage; ++i) h.w[i] = i < n ? t.w[m + i] : 0.f;
          h.n = n;
          h.nvec = (int)(bytes / 16);
          h.first = m == m0;
          h.out = m + n >= m1 ? (void*)((uint8_t*)job.merged + ((int64_t)o * b.numel + e0) * kEsz) : nullptr;
          mbar_arrive_expect_tx(&t.full[s], (uint32_t)n * bytes);
          for (int i = 0; i < n; ++i)
            bulk_load_1d(t.data[s][i], (const uint8_t*)job.experts + ((int64_t)t.mem[m + i] * b.numel + e0) * kEsz,
                         bytes, &t.full[s], pol);
        }
        __syncwarp();
        m += n;
        ++g;
      } while (m < m1);
    }
    // end marker: one stage with n = -1
    const int s = g % kStages;
    mbar_wait(&t.empty[s], ((g / kStages) & 1) ^ 1);
    if ((threadIdx.x & 31) == 0) {
      t.hdr[s].n = -1;
      mbar_arrive(&t.full[s]);
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- consumers
    const int tid = threadIdx.x - 32;
    constexpr int kPerVec = 16 / kEsz;  // elements per 16-byte vector
    float acc[2][kPerVec];
    int g = 0;
    for (;; ++g) {
      const int s = g % kStages;
      // the producer signals the end with a stage whose n is -1 (below)
      mbar_wait(&t.full[s], (g / kStages) & 1);
      const StageHdr h = t.hdr[s];
      if (h.n < 0) break;
      if (h.first) {
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int i = 0; i < kPerVec; ++i) acc[u][i] = 0.f;
      }
      for (int mi = 0; mi < h.n; ++mi) {
        const float wm = h.w[mi];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int v = tid + u * kConsumers;
          if (v < h.nvec) {
            const uint4 r = *reinterpret_cast<const uint4*>(t.data[s][mi] + v * 16);
            if constexpr (F32) {
              const float* f = reinterpret_cast<const float*>(&r);
#pragma unroll
              for (int i = 0; i < 4; ++i) acc[u][i] = fmaf(wm, f[i], acc[u][i]);
            } else {
              const __nv_bfloat162* hh = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float2 p = __bfloat1622float2(hh[i]);
                acc[u][2 * i] = fmaf(wm, p.x, acc[u][2 * i]);
                acc[u][2 * i + 1] = fmaf(wm, p.y, acc[u][2 * i + 1]);
              }
            }
          }
        }
      }
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&t.empty[s]);
      if (h.out) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int v = tid + u * kConsumers;
          if (v < h.nvec) {
            uint4 o;
            if constexpr (F32) {
              o = make_uint4(__float_as_uint(acc[u][0]), __float_as_uint(acc[u][1]), __float_as_uint(acc[u][2]),
                             __float_as_uint(acc[u][3]));
            } else {
              o.x = pack_bf16x2(acc[u][0], acc[u][1]);
              o.y = pack_bf16x2(acc[u][2], acc[u][3]);
              o.z = pack_bf16x2(acc[u][4], acc[u][5]);
              o.w = pack_bf16x2(acc[u][6], acc[u][7]);
            }
            __stcs(reinterpret_cast<uint4*>(h.out) + v, o);
          }
        }
      }
    }
  }
}
}  // namespace

cudaError_t launch_merge_batch(bool fp32, const MergeBatch& b0, cudaStream_t st) {
  MergeBatch b = b0;
  const int64_t chunk = kSlice / (fp32 ? 4 : 2);
  const int64_t cpo = (b.numel + chunk - 1) / chunk;
  b.chunk_prefix[0] = 0;
  for (int j = 0; j < b.n_jobs; ++j) {
    const int64_t n_out = b.compact ? (b.jobs[j].n_slots > 0 ? b.jobs[j].n_slots : b.E) : b.jobs[j].n_clusters;
    b.chunk_prefix[j + 1] = b.chunk_prefix[j] + n_out * cpo;
  }
  const int64_t total = b.chunk_prefix[b.n_jobs];
  if (total == 0) return cudaSuccess;
  const int smem = (int)sizeof(BatchSmem) + 128;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(total, (int64_t)kNumSMs));
  cudaError_t e;
  if (fp32) {
    e = cudaFuncSetAttribute(merge_tma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) merge_tma_kernel<true><<<grid, kBThreads, smem, st>>>(b);
  } else {
    e = cudaFuncSetAttribute(merge_tma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e == cudaSuccess) merge_tma_kernel<false><<<grid, kBThreads, smem, st>>>(b);
  }
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_merge(bool fp32, int E, int64_t numel, const void* experts, const int32_t* cluster_of,
                         const float* alpha, int C, void* merged, int32_t* remap, cudaStream_t st, int compact) {
  MergeBatch b{};
  b.n_jobs = 1;
  b.E = E;
  b.numel = numel;
  b.compact = compact;
  b.jobs[0] = MergeJob{experts, cluster_of, alpha, merged, remap, C, 0};
  return launch_merge_batch(fp32, b, st);
}

}  // namespace flux
