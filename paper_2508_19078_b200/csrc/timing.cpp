// timing.cpp — opt-in per-kernel CUDA-event timing and a launch counter, so a
// benchmark can report the live duration of each hot kernel on the stream it
// is launched on (the events are recorded on that stream around the launch).
#include <stdio.h>
#include <stdlib.h>

#include <atomic>
#include <mutex>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only: a no-op unless a profiler (nsys) injects itself

#include "internal.h"

namespace flux {
static const char* kernel_name(int kind) {
  static const char* names[FLUX_NUM_KERNELS] = {"quantize", "dequant", "router", "permute", "scatter",
                                                "gemm_gate_up", "gemm_down", "combine", "merge",
                                                "gemm_down_shared_combine", "gemm_chain", "gram", "gram_reduce", "eig",
                                                "kmeans", "cosine_distance", "attention_hist", "frequencies"};
  return kind >= 0 && kind < FLUX_NUM_KERNELS ? names[kind] : "?";
}
namespace {
std::atomic<int> g_enabled{0};
std::atomic<long long> g_launches{0};
struct Pending {
  int kind;
  cudaEvent_t a, b;
};
std::mutex g_mu;
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_pool;
double g_ms[FLUX_NUM_KERNELS] = {0};
long long g_cnt[FLUX_NUM_KERNELS] = {0};
unsigned long long* g_probe = nullptr;  // device [FLUX_NUM_KERNELS][2]: Σ SM clocks, Σ ns inside probed kernels

cudaEvent_t get_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

KernelTimer::KernelTimer(int kind, cudaStream_t st) : kind_(kind), st_(st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  nvtxRangePushA(kernel_name(kind));  // host-side range around the launch: the step timeline under nsys
  if (!g_enabled.load(std::memory_order_relaxed)) return;
  std::lock_guard<std::mutex> lk(g_mu);
  a_ = get_event();
  b_ = get_event();
  cudaEventRecord(a_, st_);
}

static const char* kernel_name(int kind);
static thread_local char g_last_error[512] = "";
static int debug_sync() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FLUX_DEBUG_SYNC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v;
}

KernelTimer::~KernelTimer() {
  nvtxRangePop();
  if (debug_sync()) {  // diagnostics: surface the failing kernel instead of a later, anonymous error
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(st_);
    if (e != cudaSuccess)
      snprintf(g_last_error, sizeof(g_last_error), "%s: %s", kernel_name(kind_), cudaGetErrorString(e));
  }
  if (!a_) return;
  cudaEventRecord(b_, st_);
  std::lock_guard<std::mutex> lk(g_mu);
  g_pending.push_back({kind_, a_, b_});
}

unsigned long long* clock_probe(int kind) {
  if (!g_enabled.load(std::memory_order_relaxed)) return nullptr;
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_probe) {
    if (cudaMalloc(&g_probe, sizeof(unsigned long long) * 2 * FLUX_NUM_KERNELS) != cudaSuccess) return nullptr;
    cudaMemset(g_probe, 0, sizeof(unsigned long long) * 2 * FLUX_NUM_KERNELS);
  }
  return g_probe + 2 * kind;
}

void set_last_error(const char* what, cudaError_t e) {
  snprintf(g_last_error, sizeof(g_last_error), "%s: %s", what, cudaGetErrorString(e));
}
const char* last_error() { return g_last_error; }

}  // namespace flux

using namespace flux;

extern "C" {

void flux_timing_enable(int on) { g_enabled.store(on ? 1 : 0); }

long long flux_launch_count(void) { return g_launches.load(); }

// Synchronises the recorded events, folds them into per-kind totals, and
// copies totals (ms) and counts out; clears them if reset != 0.
int flux_timing_read(double* ms_out, long long* count_out, int n, int reset) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& p : g_pending) {
    float ms = 0.f;
    if (cudaEventSynchronize(p.b) == cudaSuccess && cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) {
      g_ms[p.kind] += ms;
      g_cnt[p.kind] += 1;
    }
    g_pool.push_back(p.a);
    g_pool.push_back(p.b);
  }
  g_pending.clear();
  for (int i = 0; i < n && i < FLUX_NUM_KERNELS; ++i) {
    if (ms_out) ms_out[i] = g_ms[i];
    if (count_out) count_out[i] = g_cnt[i];
  }
  if (reset)
    for (int i = 0; i < FLUX_NUM_KERNELS; ++i) {
      g_ms[i] = 0;
      g_cnt[i] = 0;
    }
  return FLUX_NUM_KERNELS;
}

// Average SM clock (MHz) inside the probed kernels (the CTA-pair GEMMs) since the last reset: one thread
// of CTA 0 reads %clock64 and %globaltimer at the kernel's start and end.  0 where nothing was probed.
int flux_timing_clocks(double* mhz_out, int n, int reset) {
  std::lock_guard<std::mutex> lk(g_mu);
  unsigned long long h[2 * FLUX_NUM_KERNELS] = {0};
  if (g_probe) {
    cudaDeviceSynchronize();
    cudaMemcpy(h, g_probe, sizeof(h), cudaMemcpyDeviceToHost);
    if (reset) cudaMemset(g_probe, 0, sizeof(h));
  }
  for (int i = 0; i < n && i < FLUX_NUM_KERNELS; ++i)
    mhz_out[i] = h[2 * i + 1] ? 1e3 * (double)h[2 * i] / (double)h[2 * i + 1] : 0.0;
  return FLUX_NUM_KERNELS;
}

const char* flux_kernel_name(int kind) { return flux::kernel_name(kind); }

const char* flux_last_error(void) { return flux::last_error(); }

}  // extern "C"
