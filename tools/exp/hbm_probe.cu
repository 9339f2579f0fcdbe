// hbm_probe.cu — how the HBM access paths scale with the SM clock (experiment, not product code).
//
// Streams a 4 GiB buffer with: LDG copy, LDG read-only, STG write-only, a 4-input-1-output
// weighted sum (the merge's access pattern) with LDG, and a TMA-bulk ring read (the merge's
// producer/consumer structure without the arithmetic).  Each is timed cold (GPU idle) and hot
// (right after bf16 cuBLAS GEMMs, i.e. at the power-capped clock of a profiling step).  One thread
// records %clock64 / %globaltimer at the start and end, so the line gives the SM clock the kernel
// ran at and the bytes per SM clock.
//
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2508_19078_b200/csrc \
//        tools/exp/hbm_probe.cu -o tools/exp/hbm_probe -lcublas -lcuda
#include <cublas_v2.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <unistd.h>

#include <algorithm>
#include <functional>
#include <vector>

#include "ptx.cuh"

using namespace flux;

struct Probe {
  unsigned long long c0, c1, t0, t1;
};

__device__ __forceinline__ void probe_begin(Probe* p) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p->c0 = clock64();
    p->t0 = globaltimer_ns();
  }
}
__device__ __forceinline__ void probe_end(Probe* p) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p->c1 = clock64();
    p->t1 = globaltimer_ns();
  }
}

template <int U>
__global__ void __launch_bounds__(512) copy_ldg(const uint4* __restrict__ in, uint4* __restrict__ out, int64_t n, Probe* p) {
  probe_begin(p);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < n) v[u] = __ldcs(&in[i0 + u * stride]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < n) __stcs(&out[i0 + u * stride], v[u]);
  }
  probe_end(p);
}

template <int U>
__global__ void __launch_bounds__(512) read_ldg(const uint4* __restrict__ in, uint32_t* __restrict__ sink, int64_t n, Probe* p) {
  probe_begin(p);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < n) v[u] = __ldcs(&in[i0 + u * stride]);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < n) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
  probe_end(p);
}

template <int U>
__global__ void __launch_bounds__(512) write_stg(uint4* __restrict__ out, int64_t n, Probe* p) {
  probe_begin(p);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride)
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < n) __stcs(&out[i0 + u * stride], v);
  probe_end(p);
}

// the merge's pattern: out[c][i] = Σ_m w_m in[4c+m][i] (bf16, fp32 accumulate), 4 members per output
template <int U>
__global__ void __launch_bounds__(512) merge4_ldg(const uint4* __restrict__ in, uint4* __restrict__ out, int64_t per,
                                                  int n_out, Probe* p) {
  probe_begin(p);
  const int64_t n = per * n_out;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    uint4 v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i < n) {
        const int64_t c = i / per, o = i - c * per;
#pragma unroll
        for (int m = 0; m < 4; ++m) v[u][m] = __ldcs(&in[(4 * c + m) * per + o]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= n) continue;
      float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const uint32_t w4[4] = {v[u][m].x, v[u][m].y, v[u][m].z, v[u][m].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a[2 * q] = fmaf(0.25f, __uint_as_float(w4[q] << 16), a[2 * q]);
          a[2 * q + 1] = fmaf(0.25f, __uint_as_float(w4[q] & 0xffff0000u), a[2 * q + 1]);
        }
      }
      uint4 r;
      r.x = (__float_as_uint(a[1]) & 0xffff0000u) | (__float_as_uint(a[0]) >> 16);
      r.y = (__float_as_uint(a[3]) & 0xffff0000u) | (__float_as_uint(a[2]) >> 16);
      r.z = (__float_as_uint(a[5]) & 0xffff0000u) | (__float_as_uint(a[4]) >> 16);
      r.w = (__float_as_uint(a[7]) & 0xffff0000u) | (__float_as_uint(a[6]) >> 16);
      __stcs(&out[i], r);
    }
  }
  probe_end(p);
}

// TMA-bulk ring read: one CTA per SM, a producer lane issues SLICE-byte bulk copies into STAGES stages of
// PER slices; 16 consumer warps read one 16-byte vector of each slice (LDS) and release the stage.
template <int SLICE, int PER, int STAGES>
__global__ void __launch_bounds__(544, 1) read_tma(const uint8_t* __restrict__ in, uint32_t* __restrict__ sink,
                                                   int64_t bytes, Probe* p) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint8_t* data = sm;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + STAGES * PER * SLICE);
  uint64_t* empty = full + STAGES;
  probe_begin(p);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 16);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int64_t stage_bytes = (int64_t)SLICE * PER;
  const int64_t n_stage = bytes / stage_bytes;
  const int my = (int)((n_stage - blockIdx.x + gridDim.x - 1) / gridDim.x);
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      const uint64_t pol = policy_evict_first();
      for (int g = 0; g < my; ++g) {
        const int s = g % STAGES;
        mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
        const int64_t st = blockIdx.x + (int64_t)g * gridDim.x;
        mbar_arrive_expect_tx(&full[s], (uint32_t)stage_bytes);
        for (int i = 0; i < PER; ++i)  // PER slices from PER regions (bytes/PER apart), like a merge's members
          bulk_load_1d(data + (s * PER + i) * SLICE, in + (int64_t)i * (bytes / PER) + st * SLICE, SLICE, &full[s], pol);
      }
    }
  } else {
    uint32_t acc = 0;
    const int v = threadIdx.x - 32;
    for (int g = 0; g < my; ++g) {
      const int s = g % STAGES;
      mbar_wait(&full[s], (g / STAGES) & 1);
      for (int i = 0; i < PER; ++i)
        for (int o = v * 16; o < SLICE; o += 512 * 16) acc ^= *reinterpret_cast<const uint32_t*>(data + (s * PER + i) * SLICE + o);
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345678u) sink[0] = acc;
  }
  probe_end(p);
}

// TMA tensor-box ring read: one CTA per SM, a producer lane issues 2D boxes {64 columns (128 B, SW128),
// BOX_ROWS rows} of a bf16 [rows][cols] tensor into STAGES stages; 16 consumer warps touch one word per
// 512 B and release.  Box order: for each row block (row_blocks of BOX_ROWS rows, dealt round-robin to
// the CTAs), every 64-column slice in turn — the router's x stream (rows = tokens) or, with few rows
// far apart, the Gram's expert stream.
template <int BOX_ROWS, int STAGES>
__global__ void __launch_bounds__(544, 1) read_tma2d(const __grid_constant__ CUtensorMap map, int row_blocks,
                                                     int col_slices, uint32_t* __restrict__ sink, Probe* p) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int kBox = BOX_ROWS * 128;
  uint8_t* data = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);  // SW128 boxes: 1 KB aligned
  uint64_t* full = reinterpret_cast<uint64_t*>(data + STAGES * kBox);
  uint64_t* empty = full + STAGES;
  probe_begin(p);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 16);
    }
    fence_barrier_init();
  }
  __syncthreads();
  // work = row_blocks x col_slices boxes in chunks of 64 consecutive column slices of one row block,
  // chunks dealt round-robin to the CTAs (the Gram's order; the router's tiles when col_slices = 32)
  const int per_rb = (col_slices + 63) / 64, n_chunks = row_blocks * per_rb;
  const int my_chunks = (n_chunks - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int csz = col_slices < 64 ? col_slices : 64;
  const int my = my_chunks * csz;
  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {
      const uint64_t pol = policy_evict_first();
      for (int g = 0; g < my; ++g) {
        const int s = g % STAGES;
        mbar_wait(&empty[s], ((g / STAGES) & 1) ^ 1);
        const int ch = (int)blockIdx.x + (g / csz) * (int)gridDim.x;
        const int rb = ch / per_rb, cs = (ch % per_rb) * 64 + g % csz;  // (col_slices % 64 == 0 or < 64)
        mbar_arrive_expect_tx(&full[s], (uint32_t)kBox);
        tma_load_2d_hint(data + s * kBox, &map, &full[s], cs * 64, rb * BOX_ROWS, pol);
      }
    }
  } else {
    uint32_t acc = 0;
    const int v = threadIdx.x - 32;
    for (int g = 0; g < my; ++g) {
      const int s = g % STAGES;
      mbar_wait(&full[s], (g / STAGES) & 1);
      for (int o = v * 16; o < kBox; o += 512 * 16) acc ^= *reinterpret_cast<const uint32_t*>(data + s * kBox + o);
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345678u) sink[0] = acc;
  }
  probe_end(p);
}

static CUtensorMap make_map_2d(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                                            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "cuTensorMapEncodeTiled failed: %d\n", (int)r);
    exit(1);
  }
  return m;
}

__global__ void fill_random(__nv_bfloat16* p, int64_t n, uint32_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    p[i] = __float2bfloat16(((x & 0xffff) / 32768.f - 1.f));  // uniform in [-1, 1): toggling data draws full power
  }
}

// bulk (TMA) stores from shared memory: one lane per CTA streams SLICE-byte copies of a zeroed smem
// buffer to consecutive global addresses, at most DEPTH bulk groups in flight
template <int SLICE, int DEPTH>
__global__ void __launch_bounds__(32) write_tma(uint8_t* __restrict__ out, int64_t bytes, Probe* p) {
  extern __shared__ __align__(128) uint8_t sm[];
  probe_begin(p);
  for (int i = threadIdx.x; i < SLICE / 16; i += 32) reinterpret_cast<uint4*>(sm)[i] = make_uint4(1, 2, 3, 4);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (threadIdx.x == 0) {
    const int64_t n = bytes / SLICE;
    for (int64_t c = blockIdx.x; c < n; c += gridDim.x) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + c * SLICE),
                   "r"(smem_u32(sm)), "r"(SLICE)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DEPTH) : "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  probe_end(p);
}

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

int main() {
  const int64_t bytes = 4ll << 30;
  uint8_t *a, *b;
  uint32_t* sink;
  Probe* pr;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&b, bytes));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMalloc(&pr, sizeof(Probe)));
  CK(cudaMemset(a, 1, bytes));
  CK(cudaMemset(b, 2, bytes));
  // heat: bf16 GEMMs 8192^3
  const int N = 8192;
  __nv_bfloat16 *ga, *gb, *gc;
  CK(cudaMalloc(&ga, (size_t)N * N * 2));
  CK(cudaMalloc(&gb, (size_t)N * N * 2));
  CK(cudaMalloc(&gc, (size_t)N * N * 2));
  fill_random<<<1024, 256>>>(ga, (int64_t)N * N, 1);
  fill_random<<<1024, 256>>>(gb, (int64_t)N * N, 2);
  CK(cudaDeviceSynchronize());
  cublasHandle_t h;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) {
    fprintf(stderr, "cublasCreate failed\n");
    return 1;
  }
  const float one = 1.f, zero = 0.f;
  auto gemm = [&](int n) {
    for (int i = 0; i < n; ++i) {
      const cublasStatus_t st = cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, N, N, N, &one, ga, CUDA_R_16BF, N, gb,
                                             CUDA_R_16BF, N, &zero, gc, CUDA_R_16BF, N, CUBLAS_COMPUTE_32F,
                                             CUBLAS_GEMM_DEFAULT);
      if (st != CUBLAS_STATUS_SUCCESS) {
        fprintf(stderr, "cublasGemmEx failed: %d\n", (int)st);
        exit(1);
      }
    }
  };
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct K {
    const char* name;
    double traffic;
    std::function<void()> run;
  };
  const int64_t nv = bytes / 16;
  std::vector<K> ks;
  auto add = [&](const char* name, double traffic, std::function<void()> f) { ks.push_back({name, traffic, f}); };
  add("copy_ldg U4 2x512/SM", 2.0 * bytes, [&] { copy_ldg<4><<<nsm * 4, 512>>>((uint4*)a, (uint4*)b, nv, pr); });
  add("copy_ldg U2 4x512/SM", 2.0 * bytes, [&] { copy_ldg<2><<<nsm * 4, 512>>>((uint4*)a, (uint4*)b, nv, pr); });
  add("read_ldg U4", 1.0 * bytes, [&] { read_ldg<4><<<nsm * 4, 512>>>((uint4*)a, sink, nv, pr); });
  add("read_ldg U8", 1.0 * bytes, [&] { read_ldg<8><<<nsm * 4, 512>>>((uint4*)a, sink, nv, pr); });
  add("write_stg U4", 1.0 * bytes, [&] { write_stg<4><<<nsm * 4, 512>>>((uint4*)b, nv, pr); });
  add("merge4_ldg U1", 1.25 * bytes, [&] { merge4_ldg<1><<<nsm * 4, 512>>>((uint4*)a, (uint4*)b, nv / 64, 16, pr); });
  add("merge4_ldg U2", 1.25 * bytes, [&] { merge4_ldg<2><<<nsm * 4, 512>>>((uint4*)a, (uint4*)b, nv / 64, 16, pr); });
  {
    constexpr int S = 8192, P = 4, ST = 6;
    const int smem = S * P * ST + 2 * ST * 8;
    cudaFuncSetAttribute(read_tma<S, P, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    add("read_tma 8KBx4x6", 1.0 * bytes, [&, smem] { read_tma<S, P, ST><<<nsm, 544, smem>>>(a, sink, bytes, pr); });
  }
  {
    constexpr int S = 16384, P = 4, ST = 3;
    const int smem = S * P * ST + 2 * ST * 8;
    cudaFuncSetAttribute(read_tma<S, P, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    add("read_tma 16KBx4x3", 1.0 * bytes, [&, smem] { read_tma<S, P, ST><<<nsm, 544, smem>>>(a, sink, bytes, pr); });
  }
  {
    constexpr int S = 4096, P = 4, ST = 12;
    const int smem = S * P * ST + 2 * ST * 8;
    cudaFuncSetAttribute(read_tma<S, P, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    add("read_tma 4KBx4x12", 1.0 * bytes, [&, smem] { read_tma<S, P, ST><<<nsm, 544, smem>>>(a, sink, bytes, pr); });
  }
  {
    constexpr int S = 8192, P = 1, ST = 24;
    const int smem = S * P * ST + 2 * ST * 8;
    cudaFuncSetAttribute(read_tma<S, P, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    add("read_tma 8KBx1x24", 1.0 * bytes, [&, smem] { read_tma<S, P, ST><<<nsm, 544, smem>>>(a, sink, bytes, pr); });
  }
  {
    constexpr int S = 16384;
    cudaFuncSetAttribute(write_tma<S, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, S);
    add("write_tma 16KB d8 1/SM", 1.0 * bytes, [&] { write_tma<S, 8><<<nsm, 32, S>>>(b, bytes, pr); });
    add("write_tma 16KB d8 4/SM", 1.0 * bytes, [&] { write_tma<S, 8><<<nsm * 4, 32, S>>>(b, bytes, pr); });
    add("write_stg U8", 1.0 * bytes, [&] { write_stg<8><<<nsm * 4, 512>>>((uint4*)b, nv, pr); });
    add("write_stg U2 2/SM", 1.0 * bytes, [&] { write_stg<2><<<nsm * 2, 512>>>((uint4*)b, nv, pr); });
  }
  {
    // router-like: [1M tokens][2048] bf16 (4 KB rows), boxes of 256 token rows x 64 columns
    static const CUtensorMap m_router = make_map_2d(a, (uint64_t)(bytes / 4096), 2048, 256);
    constexpr int R = 256, ST = 5;
    const int smem = R * 128 * ST + 2 * ST * 8 + 1024;
    cudaFuncSetAttribute(read_tma2d<R, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    add("tma2d router 256r", 1.0 * bytes, [&, smem] {
      read_tma2d<R, ST><<<nsm, 544, smem>>>(m_router, (int)(bytes / 4096 / R), 32, sink, pr);
    });
    // gram-like: [704 = 11 layers x 64 experts][2,883,584] bf16 (expert rows 5.77 MB apart, the DeepSeek
    // family size), boxes of 64 expert rows x 64 columns, 64-slice chunks
    const uint64_t gcols = 2883584, grows = 704;
    static const CUtensorMap m_gram = make_map_2d(a, grows, gcols, 64);
    constexpr int G = 64, SG = 16;
    const int smemg = G * 128 * SG + 2 * SG * 8 + 1024;
    cudaFuncSetAttribute(read_tma2d<G, SG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemg);
    add("tma2d gram 64r 5.8MB", 2.0 * grows * gcols, [&, smemg] {
      read_tma2d<G, SG><<<nsm, 544, smemg>>>(m_gram, (int)(grows / 64), (int)(gcols / 64), sink, pr);
    });
    // the same with 16-row boxes (16 experts per box: a quarter of the pages touched per box)
    static const CUtensorMap m_gram16 = make_map_2d(a, grows, gcols, 16);
    constexpr int G16 = 16, SG16 = 64;
    const int smemg16 = G16 * 128 * SG16 + 2 * SG16 * 8 + 1024;
    cudaFuncSetAttribute(read_tma2d<G16, SG16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smemg16);
    add("tma2d gram 16r 5.8MB", 2.0 * grows * gcols, [&, smemg16] {
      read_tma2d<G16, SG16><<<nsm, 544, smemg16>>>(m_gram16, (int)(grows / 16), (int)(gcols / 64), sink, pr);
    });
    // contiguous: [32M rows][64] bf16 (128 B rows back to back), boxes of 256 rows = 32 KB contiguous
    static const CUtensorMap m_cont = make_map_2d(a, (uint64_t)(bytes / 128), 64, 256);
    add("tma2d contiguous 256r", 1.0 * bytes, [&, smem] {
      read_tma2d<R, ST><<<nsm, 544, smem>>>(m_cont, (int)(bytes / 128 / R), 1, sink, pr);
    });
  }
  printf("%-22s %5s %9s %9s %8s %10s\n", "kernel", "mode", "ms", "GB/s", "SM MHz", "B/clk/SM");
  const char* only = getenv("PROBE_ONLY");
  for (auto& k : ks) {
    if (only && !strstr(k.name, only)) continue;
    for (int hot = 0; hot < 2; ++hot) {
      std::vector<double> ms_v, mhz_v;
      for (int r = 0; r < 5; ++r) {
        if (hot) gemm(r == 0 ? 2000 : 200);  // ~1.5 s, then ~0.15 s of bf16 GEMMs: the clock settles at the power cap
        else {
          CK(cudaDeviceSynchronize());
          usleep(300000);  // idle
        }
        fprintf(stderr, "%s %s rep %d\n", k.name, hot ? "hot" : "cold", r);
        cudaEventRecord(e0);
        k.run();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        Probe hp;
        CK(cudaMemcpy(&hp, pr, sizeof(hp), cudaMemcpyDeviceToHost));
        ms_v.push_back(ms);
        mhz_v.push_back(1e3 * (double)(hp.c1 - hp.c0) / (double)(hp.t1 - hp.t0));
      }
      std::sort(ms_v.begin(), ms_v.end());
      std::sort(mhz_v.begin(), mhz_v.end());
      const double ms = ms_v[2], mhz = mhz_v[2];
      const double gbs = k.traffic / ms / 1e6;
  printf("%-22s %5s %9.3f %9.0f %8.0f %10.1f\n", k.name, hot ? "hot" : "cold", ms, gbs, mhz,
             gbs * 1e9 / (mhz * 1e6) / nsm);
      fflush(stdout);
    }
  }
  return 0;
}
