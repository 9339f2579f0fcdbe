// synth/gen_gpu.cu — counter-based synthetic input generator, GPU twin of
// synth/gen_cpu.c (same spec G; see that file's header).  Holds no arithmetic
// of the Flux method.  Built into synth/libsynth_gpu.so; tests check it is
// bit-identical to the CPU twin.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define SYNTH_COL0_ONE 1
#define SYNTH_ROW0_ZERO 2
#define SYNTH_COL0_C0 4

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float synth_value(uint64_t seed, uint64_t stream, uint64_t idx, float c) {
  uint64_t h = splitmix64(seed ^ (stream << 40) ^ idx);
  int n = (int)(h & 0xFFF) + (int)((h >> 16) & 0xFFF) + (int)((h >> 32) & 0xFFF) +
          (int)((h >> 48) & 0xFFF) - 8190;
  return __fmul_rn((float)n, c);
}

__device__ __forceinline__ float element(int64_t r, int64_t col, int64_t cols, uint64_t seed,
                                         uint64_t stream, float c, int flags, float c0) {
  if ((flags & SYNTH_ROW0_ZERO) && r == 0) return 0.0f;
  if ((flags & SYNTH_COL0_ONE) && col == 0) return 1.0f;
  if ((flags & SYNTH_COL0_C0) && col == 0) return synth_value(seed, stream | (1ull << 19), (uint64_t)r, c0);
  return synth_value(seed, stream, (uint64_t)(r * cols + col), c);
}

template <typename T>
__global__ void synth_kernel(T* __restrict__ dst, int64_t rows, int64_t cols, int64_t row0, uint64_t seed,
                             uint64_t stream, float c, int flags, float c0) {
  int64_t n = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / cols, col = i - r * cols;
    float v = element(row0 + r, col, cols, seed, stream, c, flags, c0);
    if constexpr (sizeof(T) == 2)
      dst[i] = __float2bfloat16_rn(v);
    else
      dst[i] = v;
  }
}

extern "C" int synth_gpu_matrix(void* dst, int dtype, int64_t rows, int64_t cols, int64_t row0, uint64_t seed,
                                uint64_t stream, float c, int flags, float c0, void* cuda_stream) {
  if (rows <= 0 || cols <= 0) return 0;
  cudaStream_t s = (cudaStream_t)cuda_stream;
  int64_t n = rows * cols;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  if (dtype == 0)
    synth_kernel<__nv_bfloat16><<<(unsigned)blocks, 256, 0, s>>>((__nv_bfloat16*)dst, rows, cols, row0, seed, stream,
                                                                  c, flags, c0);
  else
    synth_kernel<float><<<(unsigned)blocks, 256, 0, s>>>((float*)dst, rows, cols, row0, seed, stream, c, flags, c0);
  return (int)cudaGetLastError();
}
