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
// Warp 0 (producer, one elected lane) walks this CTA's chunks (dealt round-robin over one CTA per SM, so
// at any moment the CTAs stream neighbouring addresses) and per chunk issues one 1D bulk copy
// (cp.async.bulk, evict_first) per member into a ring of kStages stages of up to 4 member slices (8 KB
// each); a chunk of a cluster with m members takes ceil(m / 4) stages.  The stage header carries the
// members' weights, whether the stage starts the chunk, and (on its last stage) the output address.
// Warps 1..16 (consumers, one 16-byte vector of the chunk per thread) accumulate w_e·W_e in fp32
// (packed FFMA2, bit-identical per lane to fmaf; member order), and after the chunk's last stage round
// once and store.  The producer keeps the job's member table (every output: members in ascending id,
// weights α_e / Σα with Σα in ascending id) in shared memory, rebuilt per job.
constexpr int kSlice = 8192;                  // bytes of one member slice (one chunk of one expert)
constexpr int kPerStage = 4;                  // member slices per stage
constexpr int kStages = 6;                    // 6 x 32 KB = 192 KB of HBM reads in flight per SM
constexpr int kConsumers = kSlice / 16;       // one 16-byte vector per consumer thread
constexpr int kBThreads = 32 + kConsumers;

struct __align__(16) StageHdr {  // read by the consumers as two 16-byte shared loads
  float w[kPerStage];
  void* out;       // output vectors of this chunk when the stage holds its last members, else null
  int n;           // member slices in this stage (0: an output without members -> zeros; -1: end)
  int meta;        // 16-byte vectors in this chunk | (first stage of the chunk: reset the accumulators) << 30
};

struct BatchSmem {
  uint8_t data[kStages][kPerStage][kSlice];
  StageHdr hdr[kStages];
  uint64_t full[kStages], empty[kStages];
  int lab[kMaxE];       // output index of every expert of the current job (-1: none)
  int start[kMaxE + 2]; // output -> first member slot
  int mem[kMaxE];       // members grouped by output, ascending id
  float w[kMaxE];
  int fill[kMaxE + 1];
};

// Producer-warp helper (all 32 lanes): the job's member table; returns its output count.
__device__ int build_job_table(const MergeJob& job, int E, int compact, bool write_remap, BatchSmem& t) {
  const int lane = threadIdx.x & 31;
  int n_tun = 0;
  for (int e0 = 0; e0 < E; e0 += 32) {
    const int e = e0 + lane;
    n_tun += __popc(__ballot_sync(0xffffffffu, e < E && __ldg(&job.cluster_of[e]) == -1));
  }
  // outputs: at most E (the table's bound); n_tun + C > E leaves clusters without members anyway
  const int n_out = min(compact ? n_tun + job.n_clusters : job.n_clusters, E);
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
    int slot = cl == -1 ? rank0 + __popc(tun & ((1u << lane) - 1u)) : in_range ? n_tun + cl : -1;
    if (slot >= n_out && compact) slot = -1;  // beyond the table (only with n_tun + C > E)
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
    if (lab >= 0) t.mem[t.start[lab] + t.fill[lab] + __popc(same & ((1u << lane) - 1u))] = e;
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
  BatchSmem& t = *reinterpret_cast<BatchSmem*>(smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u));
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
    const bool leader = (threadIdx.x & 31) == 0;
    int j = -1, n_out = 0, g = 0;
    int64_t local = 0, c_in = 0;  // chunk index inside job j, inside output o
    int o = 0;
    auto next_stage = [&]() {
      const int s = g % kStages;
      mbar_wait(&t.empty[s], ((g / kStages) & 1) ^ 1);
      ++g;
      return s;
    };
    for (int64_t ch = blockIdx.x; ch < total; ch += gridDim.x) {
      if (j < 0 || ch >= b.chunk_prefix[j + 1]) {  // entering a new job: rebuild the table
        do ++j; while (ch >= b.chunk_prefix[j + 1]);
        local = ch - b.chunk_prefix[j];
        o = (int)(local / cpo);
        c_in = local - (int64_t)o * cpo;
        n_out = build_job_table(b.jobs[j], b.E, b.compact, b.chunk_prefix[j] % gridDim.x == blockIdx.x, t);
      } else {  // the next chunk of this CTA in the same job: advance without a 64-bit division
        c_in += gridDim.x;
        while (c_in >= cpo) {
          c_in -= cpo;
          ++o;
        }
      }
      if (o >= n_out) continue;  // compact single-job calls: the slot count was an upper bound
      const MergeJob& job = b.jobs[j];
      const int64_t e0 = c_in * kChunkElems;
      const int n_elems = (int)(b.numel - e0 < kChunkElems ? b.numel - e0 : kChunkElems);
      const uint32_t bytes = (uint32_t)n_elems * kEsz;
      void* out = (uint8_t*)job.merged + ((int64_t)o * b.numel + e0) * kEsz;
      const int m0 = t.start[o], m1 = t.start[o + 1];
      int m = m0;
      do {  // one stage per group of up to 4 members (an output with no member still takes one stage)
        const int s = next_stage();
        const int n = min(kPerStage, m1 - m);
        if (leader) {
          StageHdr& h = t.hdr[s];
#pragma unroll
          for (int i = 0; i < kPerStage; ++i) h.w[i] = i < n ? t.w[m + i] : 0.f;
          h.out = m + n >= m1 ? out : nullptr;
          h.n = n;
          h.meta = (int)(bytes / 16) | (m == m0 ? 1 << 30 : 0);
          mbar_arrive_expect_tx(&t.full[s], (uint32_t)n * bytes);
          for (int i = 0; i < n; ++i)
            bulk_load_1d(t.data[s][i], (const uint8_t*)job.experts + ((int64_t)t.mem[m + i] * b.numel + e0) * kEsz,
                         bytes, &t.full[s], pol);
        }
        __syncwarp();
        m += n;
      } while (m < m1);
    }
    const int s = next_stage();  // end marker
    if (leader) {
      t.hdr[s].n = -1;
      mbar_arrive(&t.full[s]);
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- consumers
    const int v = threadIdx.x - 32;  // this thread's 16-byte vector of every chunk
    constexpr int kPairs = 16 / kEsz / 2;
    float2 acc[kPairs];
    // one member's FMA into the accumulators (bf16 -> fp32 is exact: the bits shifted into place)
    auto fma_member = [&](const uint4& r, float w) {
      const float2 w2 = make_float2(w, w);
      if constexpr (F32) {
        acc[0] = fma2_rn(w2, make_float2(__uint_as_float(r.x), __uint_as_float(r.y)), acc[0]);
        acc[1] = fma2_rn(w2, make_float2(__uint_as_float(r.z), __uint_as_float(r.w)), acc[1]);
      } else {
        const uint32_t u[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
          acc[i] = fma2_rn(w2, make_float2(__uint_as_float(u[i] << 16), __uint_as_float(u[i] & 0xffff0000u)), acc[i]);
      }
    };
    for (int g = 0;; ++g) {
      const int s = g % kStages;
      mbar_wait(&t.full[s], (g / kStages) & 1);
      const uint32_t ha = smem_u32(&t.hdr[s]);
      const uint4 hw = ld_shared_v4(ha), hm = ld_shared_v4(ha + 16);  // weights; out, n, meta
      const int n = (int)hm.z;
      if (n < 0) break;
      const int nvec = (int)(hm.w & 0x3fffffffu);
      void* out = reinterpret_cast<void*>((uint64_t)hm.x | ((uint64_t)hm.y << 32));
      if (hm.w >> 30) {
#pragma unroll
        for (int i = 0; i < kPairs; ++i) acc[i] = make_float2(0.f, 0.f);
      }
      if (v < nvec) {
        const uint32_t d = smem_u32(t.data[s][0]) + v * 16;
        if (n == kPerStage) {  // full stage (balanced 4-member clusters): every load first, then the FMAs
          const uint4 r0 = ld_shared_v4(d), r1 = ld_shared_v4(d + kSlice), r2 = ld_shared_v4(d + 2 * kSlice),
                      r3 = ld_shared_v4(d + 3 * kSlice);
          fma_member(r0, __uint_as_float(hw.x));
          fma_member(r1, __uint_as_float(hw.y));
          fma_member(r2, __uint_as_float(hw.z));
          fma_member(r3, __uint_as_float(hw.w));
        } else {
          const float ws[4] = {__uint_as_float(hw.x), __uint_as_float(hw.y), __uint_as_float(hw.z),
                               __uint_as_float(hw.w)};
          for (int mi = 0; mi < n; ++mi) fma_member(ld_shared_v4(d + mi * kSlice), ws[mi]);
        }
      }
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&t.empty[s]);
      if (out && v < nvec) {
        uint4 ov;
        if constexpr (F32) {
          ov = make_uint4(__float_as_uint(acc[0].x), __float_as_uint(acc[0].y), __float_as_uint(acc[1].x),
                          __float_as_uint(acc[1].y));
        } else {
          ov.x = pack_bf16x2(acc[0].x, acc[0].y);
          ov.y = pack_bf16x2(acc[1].x, acc[1].y);
          ov.z = pack_bf16x2(acc[2].x, acc[2].y);
          ov.w = pack_bf16x2(acc[3].x, acc[3].y);
        }
        __stcs(reinterpret_cast<uint4*>(out) + v, ov);
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
