/* synth/gen_cpu.c — counter-based synthetic input generator, CPU twin.
 *
 * This module holds NO arithmetic of the Flux method: it only produces the
 * seeded synthetic inputs (tokens, router and expert weights) that both the
 * CUDA path and the CPU oracle consume.  synth/gen_gpu.cu implements the
 * identical generator on the GPU; tests/test_synth.py checks the two agree
 * bit for bit and pins this file against a pure-numpy restatement.
 *
 * Generator spec G:
 *   key  = seed ^ (stream << 40) ^ idx                    (idx < 2^40)
 *   h    = splitmix64(key)   (constants 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9,
 *                             0x94D049BB133111EB; shifts 30/27/31)
 *   n    = Σ_{i=0..3} ((h >> 16 i) & 0xFFF) − 8190        (Irwin–Hall(4), exact int)
 *   v    = fl32((float)n * c),  c = fl32(σ·√3/4096) chosen by the caller
 *   out  = bf16_rne(v)  (or v itself for the fp32 variant)
 * Structure flags (per matrix):
 *   SYNTH_COL0_ONE  : column 0 is exactly 1.0 (the bias feature of x_0)
 *   SYNTH_ROW0_ZERO : row 0 is exactly 0      (row 0 of every W_down)
 *   SYNTH_COL0_C0   : column 0 uses sub-stream (stream | 1<<19), idx = global row,
 *                     scale c0 (the per-expert router skew β_{l,e})
 */
#include <stdint.h>
#include <string.h>

#define SYNTH_COL0_ONE 1
#define SYNTH_ROW0_ZERO 2
#define SYNTH_COL0_C0 4

static inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline float synth_value(uint64_t seed, uint64_t stream, uint64_t idx, float c) {
  uint64_t h = splitmix64(seed ^ (stream << 40) ^ idx);
  int32_t n = (int32_t)(h & 0xFFF) + (int32_t)((h >> 16) & 0xFFF) +
              (int32_t)((h >> 32) & 0xFFF) + (int32_t)((h >> 48) & 0xFFF) - 8190;
  return (float)n * c; /* (float)n exact (|n| < 2^13); one IEEE multiply, RNE */
}

static inline uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  /* finite inputs only (|v| < 2^14 by construction) */
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

static inline float element(int64_t r, int64_t col, int64_t cols, uint64_t seed, uint64_t stream,
                            float c, int flags, float c0) {
  if ((flags & SYNTH_ROW0_ZERO) && r == 0) return 0.0f;
  if ((flags & SYNTH_COL0_ONE) && col == 0) return 1.0f;
  if ((flags & SYNTH_COL0_C0) && col == 0) return synth_value(seed, stream | (1ull << 19), (uint64_t)r, c0);
  return synth_value(seed, stream, (uint64_t)(r * cols + col), c);
}

/* Fill dst[rows][cols] (row-major) with rows row0 .. row0+rows-1 of the
 * generated matrix.  dtype 0 = bf16 bits (uint16), 1 = fp32. */
void synth_cpu_matrix(void* dst, int dtype, int64_t rows, int64_t cols, int64_t row0, uint64_t seed,
                      uint64_t stream, float c, int flags, float c0) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < rows; ++i) {
    int64_t r = row0 + i;
    for (int64_t col = 0; col < cols; ++col) {
      float v = element(r, col, cols, seed, stream, c, flags, c0);
      if (dtype == 0)
        ((uint16_t*)dst)[i * cols + col] = f32_to_bf16_rne(v);
      else
        ((float*)dst)[i * cols + col] = v;
    }
  }
}

/* Gather an arbitrary list of rows (e.g. a sample of token ids). */
void synth_cpu_rows(void* dst, int dtype, const int64_t* row_ids, int64_t n_rows, int64_t cols,
                    uint64_t seed, uint64_t stream, float c, int flags, float c0) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n_rows; ++i) {
    int64_t r = row_ids[i];
    for (int64_t col = 0; col < cols; ++col) {
      float v = element(r, col, cols, seed, stream, c, flags, c0);
      if (dtype == 0)
        ((uint16_t*)dst)[i * cols + col] = f32_to_bf16_rne(v);
      else
        ((float*)dst)[i * cols + col] = v;
    }
  }
}
