// budget.cpp — H1: adaptive expert layer size, eq.(1), host side
// (a pure function of L·E counters).
//   f_l[e] = hist[l][e] / T                     (activation frequency)
//   v_l    = population variance of f_l
//   b_l    = (L - l + 1) / max(v_l, 1e-12)       (l = 1..L: earlier layers keep more, P:684-695;
//                                                  skewed layers merge more)
//   B(l)   = floor( b_l / Σ_k b_k · B_non )      (the printed Σ_{k=1}^L b^l read as Σ_k b^k, R9)
//   C_l    = clamp(B(l), 1, n_non[l])           (R9: a layer never loses all of its experts)
#include <math.h>

#include <vector>

#include "internal.h"

extern "C" flux_status flux_layer_budget(int32_t L, int32_t E, const int64_t* hist, int64_t T, int64_t B_non,
                                         const int32_t* n_non, int32_t* C_out, int64_t* overrun) {
  if (L < 1 || E < 1 || !hist || !C_out || T <= 0 || B_non < 0) return FLUX_E_INVALID;
  std::vector<double> b(L);
  double bsum = 0.0;
  for (int l = 0; l < L; ++l) {
    double mean = 0.0;
    for (int e = 0; e < E; ++e) mean += (double)hist[(int64_t)l * E + e] / (double)T;
    mean /= E;
    double v = 0.0;
    for (int e = 0; e < E; ++e) {
      const double d = (double)hist[(int64_t)l * E + e] / (double)T - mean;
      v += d * d;
    }
    v /= E;
    b[l] = (double)(L - l) / (v < 1e-12 ? 1e-12 : v);
    bsum += b[l];
  }
  int64_t total = 0;
  for (int l = 0; l < L; ++l) {
    int64_t B = (int64_t)floor(b[l] / bsum * (double)B_non);
    const int64_t cap = n_non ? n_non[l] : E;
    if (B < 1) B = 1;
    if (B > cap) B = cap;
    C_out[l] = (int32_t)B;
    total += B;
  }
  if (overrun) *overrun = total - B_non;
  return FLUX_OK;
}
