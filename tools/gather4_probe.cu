// gather4_probe.cu — standalone probe of TMA tile::gather4 forms on sm_100a (diagnostic tool).
// Builds a bf16 [rows][64] tensor, gathers 4 rows (in reversed order) into shared memory with
// each variant, and checks the bytes (un-swizzling when the map uses the 128-byte swizzle).
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/g4 tools/gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include <vector>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int VARIANT>
__global__ void probe(const __grid_constant__ CUtensorMap map, int r0, int r1, int r2, int r3, uint16_t* out) {
  __shared__ __align__(1024) uint16_t tile[4 * 64];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(512));
    if (VARIANT == 0)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
          "%3, %4, %5, %6}], [%7];" ::"r"(su(tile)),
          "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su(&bar))
          : "memory");
    else if (VARIANT == 1)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
          "%4, %5, %6}], [%7];" ::"r"(su(tile)),
          "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su(&bar))
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes.cta_group::1 [%0], "
          "[%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su(tile)),
          "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su(&bar))
          : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(
          su(&bar))
      : "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = tile[i];
}

typedef CUresult (*Encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main1() {
  const int R = 64, C = 64;
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 256 + c);
  uint16_t *d, *o;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&o, 512);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  Encode enc = (Encode)fn;
  const int rows[4] = {40, 3, 17, 9};
  for (int sw = 0; sw < 2; ++sw) {
    CUtensorMap map;
    cuuint64_t dims[2] = {C, R}, str[1] = {C * 2};
    cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int v = 0; v < 3; ++v) {
      cudaMemset(o, 0, 512);
      if (v == 0) probe<0><<<1, 32>>>(map, rows[0], rows[1], rows[2], rows[3], o);
      if (v == 1) probe<1><<<1, 32>>>(map, rows[0], rows[1], rows[2], rows[3], o);
      if (v == 2) probe<2><<<1, 32>>>(map, rows[0], rows[1], rows[2], rows[3], o);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<uint16_t> g(256);
      cudaMemcpy(g.data(), o, 512, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int j = 0; j < 4; ++j)
        for (int c = 0; c < 64; ++c) {
          int chunk = c / 8, pos = sw ? ((chunk ^ (j & 7)) * 8 + c % 8) : c;
          if (g[j * 64 + pos] != (uint16_t)(rows[j] * 256 + c)) ++bad;
        }
      printf("encode=%d swizzle=%d variant=%d: %s, mismatches=%d\n", (int)cr, sw, v, cudaGetErrorString(e), bad);
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}

// ---- pair forms: CTA 1 gathers into its own smem and completes the transaction on CTA 0's barrier
template <int VARIANT>
__global__ void __cluster_dims__(2, 1, 1) probe_pair(const __grid_constant__ CUtensorMap map, int r0, int r1, int r2,
                                                     int r3, uint16_t* out) {
  __shared__ __align__(1024) uint16_t tile[4 * 64];
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  uint32_t lead;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(lead) : "r"(su(&bar)));
  if (threadIdx.x == 0) {
    if (rank == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(1024));
    if (VARIANT == 3)
      asm volatile(
          "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], "
          "[%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su(tile)),
          "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(lead)
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes.cta_group::2 [%0], "
          "[%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su(tile)),
          "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(lead)
          : "memory");
  }
  if (rank == 0)
    asm volatile(
        "{\n\t.reg .pred P1;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}" ::"r"(
            su(&bar))
        : "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[rank * 256 + i] = tile[i];
}

int main2() {
  const int R = 64, C = 64;
  std::vector<uint16_t> h(R * C);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 256 + c);
  uint16_t *d, *o;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&o, 1024);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* fn;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  Encode enc = (Encode)fn;
  const int rows[4] = {40, 3, 17, 9};
  CUtensorMap map;
  cuuint64_t dims[2] = {C, R}, str[1] = {C * 2};
  cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  for (int v = 4; v >= 3; --v) {
    cudaMemset(o, 0, 1024);
    if (v == 3) probe_pair<3><<<2, 32>>>(map, rows[0], rows[1], rows[2], rows[3], o);
    else probe_pair<4><<<2, 32>>>(map, rows[0], rows[1], rows[2], rows[3], o);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint16_t> g(512);
    cudaMemcpy(g.data(), o, 1024, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int cta = 0; cta < 2; ++cta)
      for (int j = 0; j < 4; ++j)
        for (int c = 0; c < 64; ++c) {
          int pos = ((c / 8) ^ (j & 7)) * 8 + c % 8;
          if (g[cta * 256 + j * 64 + pos] != (uint16_t)(rows[j] * 256 + c)) ++bad;
        }
    printf("pair variant=%d: %s, mismatches=%d\n", v, cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
int main() { int a = main1(); int b = main2(); return a | b; }
