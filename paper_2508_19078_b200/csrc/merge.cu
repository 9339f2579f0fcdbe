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
// The work is cut into chunks of 16 KB of consecutive output elements, dealt
// round-robin over one CTA per SM, and streamed with TMA bulk copies through a
// 3-stage shared-memory ring (192 KB of reads in flight per SM; see the kernel).
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
// Warp 0 (producer) walks this CTA's chunks (dealt round-robin over one CTA per SM, so at any moment
// the CTAs stream neighbouring addresses) and turns each chunk into one 16 KB slice per member (an
// output without members: one data-less slice).  Slices fill a ring of kStages stages of 4 slots in
// stream order, across chunk boundaries, so every stage carries 64 KB whatever the cluster sizes (K-Means
// gives 1-9 members per cluster).  Each slot's descriptor: member weight, whether it starts its chunk
// (reset the accumulators), the chunk's vector count, and on a chunk's last slice the output address; a
// stage of four members of one chunk is flagged so the consumers take a straight-line path.  One
// expect-tx per slice, one arrival per stage once its descriptors are final; lane i of the producer warp
// issues slice i of a group.  The producer's instruction stream is what bounds the kernel at the
// power-capped clock (~290 warp instructions per stage with 8 KB slices), hence the 16 KB slices:
// half the producer work per byte.  Warps 1..8 (consumers, four 16-byte vectors of every slice per
// thread) load the stage's slices into registers, release the stage, then accumulate w_e·W_e in fp32
// (packed FFMA2, bit-identical per lane to fmaf; member order), rounding once and storing at a chunk's
// last slice.  The producer keeps the job's member table (every output: members in ascending id, weights
// α_e / Σα with Σα in ascending id) in shared memory, rebuilt per job.
constexpr int kSlice = 16384;                 // bytes of one member slice (one chunk of one expert)
constexpr int kPerStage = 4;                  // slices per stage
constexpr int kStages = 3;                    // 3 x 64 KB = 192 KB of HBM reads in flight per SM
constexpr int kVpt = 4;                       // 16-byte vectors of every slice per consumer thread
constexpr int kConsumers = kSlice / 16 / kVpt;
constexpr int kFast = 1 << 8;                 // stage n field: four data slices of one chunk, in member order
constexpr int kBThreads = 32 + kConsumers;
constexpr int kFirst = 1 << 30;               // slot meta: first slice of its chunk
constexpr int kNoData = 1 << 29;              // slot meta: an output without members (writes zeros)

struct __align__(16) StageHdr {  // read by the consumers as five 16-byte shared loads
  float w[kPerStage];
  int meta[kPerStage];  // vectors in the slot's chunk | kFirst | kNoData
  void* out[kPerStage]; // output vectors of the chunk on its last slice, else null
  int n;                // slots used | kFast (-1: end)
  int pad[3];
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
    const int lane = threadIdx.x & 31;
    const bool leader = lane == 0;
    int j = -1, n_out = 0, g = 0;
    int64_t local = 0, c_in = 0;  // chunk index inside job j, inside output o
    int o = 0;
    auto next_stage = [&]() {
      const int st = g % kStages;
      mbar_wait(&t.empty[st], ((g / kStages) & 1) ^ 1);
      ++g;
      return st;
    };
    int s = -1, slot = 0;  // the stage being filled and its next free slot
    bool fast = false;     // ... and whether it holds four data slices of one chunk
    auto commit = [&]() {  // the stage's descriptors are final: its single arrival
      __syncwarp();
      if (leader) {
        t.hdr[s].n = slot | (fast ? kFast : 0);
        mbar_arrive(&t.full[s]);
      }
      __syncwarp();
      s = -1;
      slot = 0;
      fast = false;
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
      const int nvec = (int)(bytes / 16);
      // the chunk's slices, up to 4 per stage, lane i issuing slice i of the group (warp-parallel: a single
      // lane walking the slices is issue-bound at the power-capped clock)
      const int n_sl = max(m1 - m0, 1);  // an output without members: one data-less slot
      for (int j0 = 0; j0 < n_sl;) {
        if (s < 0) s = next_stage();
        const int take = min(kPerStage - slot, n_sl - j0);
        if (take == kPerStage && m1 > m0) fast = true;  // a whole stage of one chunk's members
        if (lane < take) {
          const int q = j0 + lane, sl = slot + lane;  // slice q of the chunk into slot sl
          const bool data = m1 > m0;
          StageHdr& h = t.hdr[s];
          h.w[sl] = data ? t.w[m0 + q] : 0.f;
          h.meta[sl] = nvec | (q == 0 ? kFirst : 0) | (data ? 0 : kNoData);
          h.out[sl] = q + 1 == n_sl ? out : nullptr;
          if (data) {
            mbar_expect_tx(&t.full[s], bytes);
            bulk_load_1d(t.data[s][sl], (const uint8_t*)job.experts + ((int64_t)t.mem[m0 + q] * b.numel + e0) * kEsz,
                         bytes, &t.full[s], pol);
          }
        }
        j0 += take;
        slot += take;
        if (slot == kPerStage) commit();
      }
    }
    if (s >= 0) commit();
    s = next_stage();  // end marker
    if (leader) {
      t.hdr[s].n = -1;
      mbar_arrive(&t.full[s]);
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- consumers
    const int v0 = threadIdx.x - 32;  // this thread's 16-byte vectors of every slice: v0 + u·kConsumers
    constexpr int kPairs = 16 / kEsz / 2;
    float2 acc[kVpt][kPairs];
    // one member's FMA into the accumulators (bf16 -> fp32 is exact: the bits shifted into place)
    auto fma_member = [&](float2 (&a)[kPairs], const uint4& r, float w) {
      const float2 w2 = make_float2(w, w);
      if constexpr (F32) {
        a[0] = fma2_rn(w2, make_float2(__uint_as_float(r.x), __uint_as_float(r.y)), a[0]);
        a[1] = fma2_rn(w2, make_float2(__uint_as_float(r.z), __uint_as_float(r.w)), a[1]);
      } else {
        const uint32_t u[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
          a[i] = fma2_rn(w2, make_float2(__uint_as_float(u[i] << 16), __uint_as_float(u[i] & 0xffff0000u)), a[i]);
      }
    };
    auto reset = [&](float2 (&a)[kPairs]) {
#pragma unroll
      for (int q = 0; q < kPairs; ++q) a[q] = make_float2(0.f, 0.f);
    };
    auto store = [&](const float2 (&a)[kPairs], uint64_t out, int v) {
      uint4 ov;
      if constexpr (F32) {
        ov = make_uint4(__float_as_uint(a[0].x), __float_as_uint(a[0].y), __float_as_uint(a[1].x), __float_as_uint(a[1].y));
      } else {
        ov.x = pack_bf16x2(a[0].x, a[0].y);
        ov.y = pack_bf16x2(a[1].x, a[1].y);
        ov.z = pack_bf16x2(a[2].x, a[2].y);
        ov.w = pack_bf16x2(a[3].x, a[3].y);
      }
      __stcs(reinterpret_cast<uint4*>(out) + v, ov);
    };
    for (int g = 0;; ++g) {
      const int s = g % kStages;
      mbar_wait(&t.full[s], (g / kStages) & 1);
      const uint32_t ha = smem_u32(&t.hdr[s]);
      const int nf = (int)ld_shared_v4(ha + 64).x;
      if (nf < 0) break;
      const uint32_t d = smem_u32(t.data[s][0]) + v0 * 16;
      const uint4 hw = ld_shared_v4(ha), hm = ld_shared_v4(ha + 16);
      const float ws[kPerStage] = {__uint_as_float(hw.x), __uint_as_float(hw.y), __uint_as_float(hw.z),
                                   __uint_as_float(hw.w)};
      uint4 r[kPerStage][kVpt];
      if (nf & kFast) {  // four members of one chunk: straight-line FMAs, reset / store at most once
        const int nvec = (int)hm.x & (kNoData - 1);
        const uint4 ho23 = ld_shared_v4(ha + 48);
        const uint64_t out = (uint64_t)ho23.z | ((uint64_t)ho23.w << 32);
#pragma unroll
        for (int i = 0; i < kPerStage; ++i)
#pragma unroll
          for (int u = 0; u < kVpt; ++u)
            if (v0 + u * kConsumers < nvec) r[i][u] = ld_shared_v4(d + i * kSlice + u * kConsumers * 16);
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(&t.empty[s]);
#pragma unroll
        for (int u = 0; u < kVpt; ++u) {
          if (hm.x & kFirst) reset(acc[u]);
          if (v0 + u * kConsumers >= nvec) continue;
#pragma unroll
          for (int i = 0; i < kPerStage; ++i) fma_member(acc[u], r[i][u], ws[i]);
          if (out) store(acc[u], out, v0 + u * kConsumers);
        }
        continue;
      }
      const int n = nf & (kFast - 1);
      const uint4 ho01 = ld_shared_v4(ha + 32), ho23 = ld_shared_v4(ha + 48);
      const int meta[kPerStage] = {(int)hm.x, (int)hm.y, (int)hm.z, (int)hm.w};
      const uint64_t outs[kPerStage] = {(uint64_t)ho01.x | ((uint64_t)ho01.y << 32), (uint64_t)ho01.z | ((uint64_t)ho01.w << 32),
                                        (uint64_t)ho23.x | ((uint64_t)ho23.y << 32), (uint64_t)ho23.z | ((uint64_t)ho23.w << 32)};
      // every slice of the stage into registers first, then release the stage
#pragma unroll
      for (int i = 0; i < kPerStage; ++i)
#pragma unroll
        for (int u = 0; u < kVpt; ++u)
          if (i < n && v0 + u * kConsumers < (meta[i] & (kNoData - 1)) && !(meta[i] & kNoData))
            r[i][u] = ld_shared_v4(d + i * kSlice + u * kConsumers * 16);
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&t.empty[s]);
#pragma unroll
      for (int i = 0; i < kPerStage; ++i) {
        if (i >= n) break;
        const int nvec = meta[i] & (kNoData - 1);
#pragma unroll
        for (int u = 0; u < kVpt; ++u) {
          if (meta[i] & kFirst) reset(acc[u]);
          const int v = v0 + u * kConsumers;
          if (v >= nvec) continue;
          if (!(meta[i] & kNoData)) fma_member(acc[u], r[i][u], ws[i]);
          if (outs[i]) store(acc[u], outs[i], v);
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
