/* oracle/oracle.c — plain, slow, obviously-correct CPU oracle for the Flux
 * hot path (arXiv 2508.19078).  fp64 throughout, OpenMP only over independent
 * outer loops (tokens / output elements), no blocking, fusion or reordering.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or constant with the CUDA path
 * (paper_2508_19078_b200/), and never reads anything the CUDA path produced.
 *
 * Citations: "P:N" = line N of the paper text.  Where the paper is
 * silent the reading used is the one listed in DESIGN.md §2 ("R#").
 *
 *  O1 orc_quantize       P:556-565, P:575-578 (quantized MoE, bit-level per
 *                        participant); scheme = R1 (symmetric, per-row groups
 *                        of g along K, s = fl32(max|w|/qmax), q = RNE(fl32(w/s))).
 *  O2 orc_router         P:217-220 (a gating network assigns tokens to
 *                        experts), R2 (z = x·W_rᵀ, softmax, top-k, lowest index
 *                        wins ties, w = p or p renormalised over the top-k).
 *  O3 orc_permute        P:579-584 (D_e: the tokens that pass through expert
 *                        e), R3 (stable: ascending token id).
 *  O4-O6 orc_moe_tokens  P:196-220 (MoE layer = experts selected by the gate),
 *                        R4 (SwiGLU experts, bf16 storage points), R5 (shared
 *                        experts), R6 (y = x + shared + Σ_j w_j o_j).
 *  O8 statistics         P:296-298 (activation frequency = activated tokens /
 *                        total tokens) — the histogram is orc_permute's hist.
 *  O9 orc_layer_budget   eq.(1), R9.
 *  O10 orc_merge         eq.(2), R10.
 *
 * Parity pins for every function live in tests/test_oracle_*.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ----------------------------------------------------------------------------
 * bf16 round-to-nearest-even of a real number (the storage points of R4/R6/R10).
 * A bf16 has 8 significant bits: write v = m·2^e with m in [0.5,1), round
 * m·2^8 to the nearest integer (ties to even), scale back.  Values here are
 * far inside bf16's normal range.
 * -------------------------------------------------------------------------- */
double orc_bf16_round(double v) {
  if (v == 0.0 || !isfinite(v)) return v;
  int e;
  double m = frexp(v, &e);            /* v = m * 2^e, 0.5 <= |m| < 1 */
  double r = nearbyint(ldexp(m, 8));  /* default rounding mode: to nearest, ties to even */
  return ldexp(r, e - 8);
}

void orc_bf16_round_array(int64_t n, const double* in, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = orc_bf16_round(in[i]);
}

/* ----------------------------------------------------------------------------
 * O1. Quantize (R1).  w: [R][K] real values; groups of g consecutive k in a row
 * (g == K: per output channel).  qmax = 2^(b-1) - 1, b in {2, 4, 8} (b = 2: NEXT-3).
 *   a = max_{k in group} |w|           (exact, the inputs are fp32 numbers)
 *   s = fl32(a / qmax)                 (one IEEE fp32 division, RNE)
 *   q = 0 if s == 0 else clamp(RNE(fl32(w / s)), -qmax-1, qmax)
 * Outputs: q [R][K] int8 (unpacked), s [R][K/g] fp32.
 * -------------------------------------------------------------------------- */
int orc_quantize(int wbits, int64_t g, int64_t R, int64_t K, const float* w, int8_t* q, float* s) {
  if ((wbits != 2 && wbits != 4 && wbits != 8) || g <= 0 || K % g != 0) return 1;
  const int qmax = (1 << (wbits - 1)) - 1;
  const int64_t G = K / g;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < R; ++r) {
    for (int64_t grp = 0; grp < G; ++grp) {
      const float* wg = w + r * K + grp * g;
      float a = 0.0f;
      for (int64_t i = 0; i < g; ++i) {
        float m = fabsf(wg[i]);
        if (m > a) a = m;
      }
      float sc = a / (float)qmax;
      s[r * G + grp] = sc;
      for (int64_t i = 0; i < g; ++i) {
        int v = 0;
        if (sc != 0.0f) {
          float t = wg[i] / sc;
          v = (int)nearbyintf(t);
          if (v > qmax) v = qmax;
          if (v < -qmax - 1) v = -qmax - 1;
        }
        q[r * K + grp * g + i] = (int8_t)v;
      }
    }
  }
  return 0;
}

/* Canonical INT2 storage (NEXT-3, "2-bit"): four per byte, element k
 * in bits 2·(k mod 4), two's complement. */
void orc_pack_int2(int64_t R, int64_t K, const int8_t* q, uint8_t* packed) {
  for (int64_t r = 0; r < R; ++r)
    for (int64_t k = 0; k < K; k += 4) {
      unsigned b = 0;
      for (int j = 0; j < 4; ++j) b |= (unsigned)(q[r * K + k + j] & 0x3) << (2 * j);
      packed[r * (K / 4) + k / 4] = (uint8_t)b;
    }
}

/* Canonical INT4 storage (boundary, include/flux.h): two per byte, even k in
 * the low nibble, two's complement. */
void orc_pack_int4(int64_t R, int64_t K, const int8_t* q, uint8_t* packed) {
  for (int64_t r = 0; r < R; ++r)
    for (int64_t k = 0; k < K; k += 2)
      packed[r * (K / 2) + k / 2] = (uint8_t)((q[r * K + k] & 0xF) | ((q[r * K + k + 1] & 0xF) << 4));
}

/* ----------------------------------------------------------------------------
 * O2. Router / gating for one token (R2).
 *   z_e = Σ_d x_d W_r[e][d]                         (fp64)
 *   S   = the k largest z, taken one at a time; among equal z the lower e wins;
 *         S is listed in descending z.
 *   p   = softmax(z) = exp(z_e - max z) / Σ_e' exp(z_e' - max z)
 *   w_j = p_{S_j}                  (norm = 0)
 *       = p_{S_j} / Σ_{e in S} p_e (norm = 1)
 *   margin = z_(k) - z_(k+1) (+inf when k == E): the parity contract's near-tie measure.
 * -------------------------------------------------------------------------- */
static void router_one(int H, int E, int k, int norm, const double* x, const double* wr, double* z, int32_t* ids,
                       double* w, double* margin) {
  for (int e = 0; e < E; ++e) {
    double acc = 0.0;
    for (int d = 0; d < H; ++d) acc += x[d] * wr[(int64_t)e * H + d];
    z[e] = acc;
  }
  char taken[1024];
  for (int e = 0; e < E; ++e) taken[e] = 0;
  for (int j = 0; j < k; ++j) {
    int best = -1;
    for (int e = 0; e < E; ++e)
      if (!taken[e] && (best < 0 || z[e] > z[best])) best = e;
    taken[best] = 1;
    ids[j] = best;
  }
  if (k < E) {
    int nxt = -1;
    for (int e = 0; e < E; ++e)
      if (!taken[e] && (nxt < 0 || z[e] > z[nxt])) nxt = e;
    *margin = z[ids[k - 1]] - z[nxt];
  } else {
    *margin = INFINITY;
  }
  double zmax = z[0];
  for (int e = 1; e < E; ++e)
    if (z[e] > zmax) zmax = z[e];
  double denom = 0.0;
  for (int e = 0; e < E; ++e) denom += exp(z[e] - zmax);
  double psel = 0.0;
  for (int j = 0; j < k; ++j) {
    w[j] = exp(z[ids[j]] - zmax) / denom;
    psel += w[j];
  }
  if (norm)
    for (int j = 0; j < k; ++j) w[j] /= psel;
}

int orc_router(int64_t T, int H, int E, int k, int norm, const double* x, const double* wr, double* z, int32_t* ids,
               double* w, double* margin) {
  if (E < 1 || E > 1024 || k < 1 || k > E) return 1;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t)
    router_one(H, E, k, norm, x + t * H, wr, z + t * E, ids + t * k, w + t * k, margin + t);
  return 0;
}

/* ----------------------------------------------------------------------------
 * O3. D_e as CSR (R3) + the histogram of O8.
 *   hist[e]        += #{t : e in S_t}                    (P:296-298 numerator)
 *   offsets        = exclusive prefix sum of this call's counts, offsets[E] = T·k
 *   token_index[offsets[e] + r] = the r-th smallest t with e in S_t
 *   inv_pos[t][j]  = that position for e = S_tj
 * An empty pick (id -1, O11's folded re-routing) is not counted: inv_pos = -1.
 * -------------------------------------------------------------------------- */
void orc_permute(int64_t T, int E, int k, const int32_t* ids, int64_t* hist, int64_t* offsets, int64_t* token_index,
                 int64_t* inv_pos) {
  int64_t* cnt = (int64_t*)calloc((size_t)E, sizeof(int64_t));
  for (int64_t t = 0; t < T; ++t)
    for (int j = 0; j < k; ++j)
      if (ids[t * k + j] >= 0) cnt[ids[t * k + j]]++;
  offsets[0] = 0;
  for (int e = 0; e < E; ++e) {
    offsets[e + 1] = offsets[e] + cnt[e];
    if (hist) hist[e] += cnt[e];
  }
  int64_t* fill = (int64_t*)calloc((size_t)E, sizeof(int64_t));
  for (int64_t t = 0; t < T; ++t)
    for (int j = 0; j < k; ++j) {
      int e = ids[t * k + j];
      if (e < 0) {
        inv_pos[t * k + j] = -1;
        continue;
      }
      int64_t pos = offsets[e] + fill[e]++;
      token_index[pos] = t;
      inv_pos[t * k + j] = pos;
    }
  free(cnt);
  free(fill);
}

/* ----------------------------------------------------------------------------
 * O4. SwiGLU expert with dequantized weights ŵ (R4):
 *   g_f = Σ_h x_h ŵgate[f][h],  u_f = Σ_h x_h ŵup[f][h]
 *   a_f = bf16( SiLU(g_f) · u_f ),      SiLU(v) = v / (1 + e^{-v})
 *   o_h = bf16( Σ_f a_f ŵdown[h][f] )
 * Quantized weights: q int8 [rows][K] unpacked, s fp32 [rows][K/g].
 * Dequantized weight of the quantized model (reading R1b):
 *   per output channel (group_size == 0): ŵ = q·s exactly;
 *   groups along K: ŵ = bf16( q · bf16(s) ) — the W4A16 convention: the quantized
 *   model's weights are materialised in bf16 from the code and the bf16 scale.
 * -------------------------------------------------------------------------- */
typedef struct {
  const int8_t *q_gate, *q_up, *q_down;
  const float *s_gate, *s_up, *s_down;
} orc_expert;

/* ŵ for a whole [rows][K] matrix (g = group length along K, grouped = g came from group_size). */
static void dequantize(const int8_t* q, const float* s, int64_t rows, int64_t K, int64_t g, int grouped,
                       double* out) {
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t k = 0; k < K; ++k) {
      double sc = (double)s[r * (K / g) + k / g];
      double qv = (double)q[r * K + k];
      out[r * K + k] = grouped ? orc_bf16_round(qv * orc_bf16_round(sc)) : qv * sc;
    }
}

typedef struct {
  double *gate, *up, *down; /* [F][H], [F][H], [H][F] */
} deq_expert;

static int deq_alloc(deq_expert* d, int H, int F) {
  d->gate = (double*)malloc(sizeof(double) * (size_t)F * H);
  d->up = (double*)malloc(sizeof(double) * (size_t)F * H);
  d->down = (double*)malloc(sizeof(double) * (size_t)F * H);
  return d->gate && d->up && d->down;
}
static void deq_free(deq_expert* d) {
  free(d->gate);
  free(d->up);
  free(d->down);
}
/* exact != 0: the survey's O4 reading ŵ = q·s for grouped codes as well (no bf16 rounding of the
 * scale or the product) — used only to show that R1b does not decide parity (tests). */
static void deq_fill(deq_expert* d, const orc_expert* ex, int H, int F, int g, int exact) {
  const int grouped = g != 0 && !exact;
  dequantize(ex->q_gate, ex->s_gate, F, H, g ? g : H, grouped, d->gate);
  dequantize(ex->q_up, ex->s_up, F, H, g ? g : H, grouped, d->up);
  dequantize(ex->q_down, ex->s_down, H, F, g ? g : F, grouped, d->down);
}

/* mag (NULL = skip): [H] the largest term of each down-projection dot product,
 * mag_h = max_f |a_f·ŵdown[h][f]| (an act value a_f one bf16 ulp off moves o_h by <= 2^-7·mag_h). */
static void swiglu_expert(int H, int F, const deq_expert* w, const double* x, double* a, double* out,
                          double* mag) {
  for (int f = 0; f < F; ++f) {
    double gs = 0.0, us = 0.0;
    for (int h = 0; h < H; ++h) {
      gs += x[h] * w->gate[(int64_t)f * H + h];
      us += x[h] * w->up[(int64_t)f * H + h];
    }
    double silu = gs / (1.0 + exp(-gs));
    a[f] = orc_bf16_round(silu * us);
  }
  for (int h = 0; h < H; ++h) {
    double acc = 0.0;
    for (int f = 0; f < F; ++f) acc += a[f] * w->down[(int64_t)h * F + f];
    out[h] = orc_bf16_round(acc);
    if (mag) {
      double m = 0.0;
      for (int f = 0; f < F; ++f) m = fmax(m, fabs(a[f] * w->down[(int64_t)h * F + f]));
      mag[h] = m;
    }
  }
}

/* ----------------------------------------------------------------------------
 * O2+O4+O5+O6 for n independent tokens of one layer (tokens never interact
 * on this attention-free path, R7):
 *   (z, S, w, margin) = router(x_t)
 *   o_{t,j}  = expert_{S_tj}(x_t)                       (O4; for e, for t in D_e)
 *   sh_t     = shared SwiGLU(x_t), 0 if F_s == 0        (O5)
 *   y_t      = bf16( r_t + sh_t + Σ_j w_tj · o_{t,j} )  (O6, j in order)
 * r: the residual (R6: "r = residual (optional)"): resid [n][H] when given (e.g. all
 * zeros, so that y is the MoE branch alone), else r_t = x_t.
 * x, y: [n][H] real (bf16-valued) numbers.  experts: array of E routed experts;
 * shared: NULL or one expert of width F_s.  g: group size (0 = per channel).
 * deq_exact: 0 = reading R1b (grouped ŵ = bf16(q·bf16(s))); 1 = ŵ = q·s exactly for every
 * granularity (SURVEY O4's literal reading; a cross-check that R1b is not load-bearing).
 * cond (NULL = skip): [n][H] magnitude of the terms of the O6 sum,
 *   cond_th = |r_th| + |sh_th| + Σ_j w_tj·|o_{t,j,h}|
 * — the condition of the sum: a perturbation of relative size ε in every term moves
 * y_th by at most ε·cond_th (the standard forward error bound of a sum).
 * dmag (NULL = skip): [n][H] Σ_j w_tj·max_f |a_tjf·ŵd_hf| + max_f |a_sh,f·ŵsh_hf| — the largest
 * down-projection term behind each y_th (an act value a_f that lands one bf16 ulp away moves y_th by
 * at most 2^-7 of its term).
 * Work order: each expert's weights are dequantized once, then its tokens run.
 * -------------------------------------------------------------------------- */
int orc_moe_tokens(int64_t n, int H, int E, int k, int F, int Fs, int g, int norm, const double* x, const double* wr,
                   const orc_expert* experts, const orc_expert* shared, const double* resid, double* y, int32_t* ids,
                   double* w, double* z, double* margin, double* cond, double* dmag, int deq_exact) {
  if (orc_router(n, H, E, k, norm, x, wr, z, ids, w, margin)) return 1;
  double* o = (double*)malloc(sizeof(double) * (size_t)n * k * H);   /* o[t][j][h] */
  double* sh = (double*)calloc((size_t)n * H, sizeof(double));       /* sh[t][h]   */
  double* om = dmag ? (double*)calloc((size_t)n * k * H, sizeof(double)) : NULL;  /* down-term magnitudes */
  double* shm = dmag ? (double*)calloc((size_t)n * H, sizeof(double)) : NULL;
  if (!o || !sh || (dmag && (!om || !shm))) { free(o); free(sh); free(om); free(shm); return 2; }
  int ok = 1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int e = 0; e < E; ++e) {
    int used = 0;
    for (int64_t i = 0; i < n * k; ++i) used |= ids[i] == e;
    if (!used) continue;
    deq_expert d;
    double* a = (double*)malloc(sizeof(double) * (size_t)F);
    if (!deq_alloc(&d, H, F) || !a) { ok = 0; deq_free(&d); free(a); continue; }
    deq_fill(&d, &experts[e], H, F, g, deq_exact);
    for (int64_t t = 0; t < n; ++t)
      for (int j = 0; j < k; ++j)
        if (ids[t * k + j] == e) swiglu_expert(H, F, &d, x + t * H, a, o + (t * k + j) * (int64_t)H,
                                                   om ? om + (t * k + j) * (int64_t)H : NULL);
    deq_free(&d);
    free(a);
  }
  if (shared && Fs > 0) {
    deq_expert d;
    if (!deq_alloc(&d, H, Fs)) { ok = 0; }
    else {
      deq_fill(&d, shared, H, Fs, g, deq_exact);
#pragma omp parallel for schedule(dynamic, 1)
      for (int64_t t = 0; t < n; ++t) {
        double* a = (double*)malloc(sizeof(double) * (size_t)Fs);
        swiglu_expert(H, Fs, &d, x + t * H, a, sh + t * H, shm ? shm + t * H : NULL);
        free(a);
      }
    }
    deq_free(&d);
  }
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < n; ++t)
    for (int h = 0; h < H; ++h) {
      const double r = resid ? resid[t * H + h] : x[t * H + h];
      double acc = r;
      acc += sh[t * H + h];
      for (int j = 0; j < k; ++j) acc += w[t * k + j] * o[(t * k + j) * (int64_t)H + h];
      y[t * H + h] = orc_bf16_round(acc);
      if (cond) {
        double m = fabs(r) + fabs(sh[t * H + h]);
        for (int j = 0; j < k; ++j) m += w[t * k + j] * fabs(o[(t * k + j) * (int64_t)H + h]);
        cond[t * H + h] = m;
      }
      if (dmag) {
        double m = shm[t * H + h];
        for (int j = 0; j < k; ++j) m += w[t * k + j] * om[(t * k + j) * (int64_t)H + h];
        dmag[t * H + h] = m;
      }
    }
  free(o);
  free(sh);
  free(om);
  free(shm);
  return ok ? 0 : 2;
}

/* ----------------------------------------------------------------------------
 * O11 (NEXT-2). Gate re-routing after merging (§7: "remaps the
 * original experts assigned by the gate network to new destinations if they have
 * been merged") + the forward of the compact model, reading R14:
 *   (z, S, w, margin) = router(x_t) over the ORIGINAL E_r experts (O2; the gate is
 *                       unchanged, so w is normalised over the original picks)
 *   slot_j  = remap[S_j]  (tuning experts first, then clusters: O10's remap)
 *   a pick whose slot already appeared earlier in S_t (a higher logit) is folded
 *   into that earlier pick: w_i += w_j; pick j becomes empty (id -1, w 0)
 *   o_{t,j} = SwiGLU_{slot_j}(x_t) (O4) with the given full-precision weights
 *   y_t     = bf16( x_t + sh_t + Σ_{j non-empty} w_tj · o_{t,j} )   (O6)
 * Weights: gate/up [S][F][H], down [S][H][F] (real, bf16-valued); sh_* NULL if F_s == 0.
 * ids/w out: the re-routed picks ([n][k], slot or -1).  resid (NULL = x), cond and dmag (NULL = skip)
 * as in orc_moe_tokens (R6: r is an input; the condition terms of the O6 sum).
 * -------------------------------------------------------------------------- */
int orc_compact_tokens(int64_t n, int H, int Er, int k, int S, int F, int Fs, int norm, const double* x,
                       const double* wr, const int32_t* remap, const double* gate, const double* up,
                       const double* down, const double* sh_gate, const double* sh_up, const double* sh_down,
                       const double* resid, double* y, int32_t* ids, double* w, double* z, double* margin,
                       double* cond, double* dmag) {
  if (S < 1) return 1;
  for (int e = 0; e < Er; ++e)
    if (remap[e] < 0 || remap[e] >= S) return 1;
  if (orc_router(n, H, Er, k, norm, x, wr, z, ids, w, margin)) return 1;
  for (int64_t t = 0; t < n; ++t) {  /* gate re-routing with folding of repeated slots */
    int32_t* it = ids + t * k;
    double* wt = w + t * k;
    for (int j = 0; j < k; ++j) it[j] = remap[it[j]];
    for (int j = 1; j < k; ++j)
      for (int i = 0; i < j; ++i)
        if (it[i] >= 0 && it[i] == it[j]) {
          wt[i] += wt[j];
          wt[j] = 0.0;
          it[j] = -1;
          break;
        }
  }
  double* o = (double*)calloc((size_t)n * k * H, sizeof(double)); /* o[t][j][h] */
  double* sh = (double*)calloc((size_t)n * H, sizeof(double));
  double* om = dmag ? (double*)calloc((size_t)n * k * H, sizeof(double)) : NULL;
  double* shm = dmag ? (double*)calloc((size_t)n * H, sizeof(double)) : NULL;
  if (!o || !sh || (dmag && (!om || !shm))) { free(o); free(sh); free(om); free(shm); return 2; }
#pragma omp parallel for schedule(dynamic, 1)
  for (int s = 0; s < S; ++s) {
    deq_expert d = {(double*)gate + (int64_t)s * F * H, (double*)up + (int64_t)s * F * H,
                    (double*)down + (int64_t)s * H * F};
    double* a = (double*)malloc(sizeof(double) * (size_t)F);
    for (int64_t t = 0; t < n; ++t)
      for (int j = 0; j < k; ++j)
        if (ids[t * k + j] == s)
          swiglu_expert(H, F, &d, x + t * H, a, o + (t * k + j) * (int64_t)H, om ? om + (t * k + j) * (int64_t)H : NULL);
    free(a);
  }
  if (Fs > 0 && sh_gate) {
    deq_expert d = {(double*)sh_gate, (double*)sh_up, (double*)sh_down};
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < n; ++t) {
      double* a = (double*)malloc(sizeof(double) * (size_t)Fs);
      swiglu_expert(H, Fs, &d, x + t * H, a, sh + t * H, shm ? shm + t * H : NULL);
      free(a);
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < n; ++t)
    for (int h = 0; h < H; ++h) {
      const double r = resid ? resid[t * H + h] : x[t * H + h];
      double acc = r;
      acc += sh[t * H + h];
      for (int j = 0; j < k; ++j)
        if (ids[t * k + j] >= 0) acc += w[t * k + j] * o[(t * k + j) * (int64_t)H + h];
      y[t * H + h] = orc_bf16_round(acc);
      if (cond) {  /* as in orc_moe_tokens */
        double m = fabs(r) + fabs(sh[t * H + h]);
        for (int j = 0; j < k; ++j)
          if (ids[t * k + j] >= 0) m += w[t * k + j] * fabs(o[(t * k + j) * (int64_t)H + h]);
        cond[t * H + h] = m;
      }
      if (dmag) {
        double m = shm[t * H + h];
        for (int j = 0; j < k; ++j)
          if (ids[t * k + j] >= 0) m += w[t * k + j] * om[(t * k + j) * (int64_t)H + h];
        dmag[t * H + h] = m;
      }
    }
  free(o);
  free(sh);
  free(om);
  free(shm);
  return 0;
}

/* ----------------------------------------------------------------------------
 * O13 (NEXT-3). Attention-weighted importance of eq.(2): α_e = f_e·ā_e,
 * ā_e = "the average attention value of tokens assigned to expert e", f_e = |D_e|/T
 * (P:296-298), so α_e = (1/T) Σ_{t∈D_e} a_t.  Reading R15: a_t is the per-token
 * attention value the model's attention layer supplies (the path has none); the sum is
 * kept like the histogram, as exact integers in fixed point:
 *   A_e += RNE(a_t · 2^24)   for every live pick (t, j) with S_tj = e
 * so α_e = A_e / (2^24 · T) up to the 2^-25 rounding of each a_t, and A is order-free.
 * ids [T][k] (-1 = empty pick), attn [T] fp32 (>= 0), A [E] accumulated.
 * -------------------------------------------------------------------------- */
void orc_attention_hist(int64_t T, int k, const int32_t* ids, const float* attn, int64_t* A) {
  for (int64_t t = 0; t < T; ++t) {
    const int64_t a = (int64_t)nearbyint((double)attn[t] * 16777216.0);
    for (int j = 0; j < k; ++j)
      if (ids[t * k + j] >= 0) A[ids[t * k + j]] += a;
  }
}

/* ----------------------------------------------------------------------------
 * O9. Adaptive expert layer size, eq.(1), reading R9:
 *   f_l[e] = hist[l][e] / T
 *   v_l    = (1/E) Σ_e (f_l[e] - mean_l)^2       (population variance)
 *   b_l    = (L - l + 1) / max(v_l, 1e-12),  l = 1..L
 *   B(l)   = floor( b_l / Σ_k b_k · B_non )
 *   C_l    = clamp(B(l), 1, n_non[l])    (R9: never discard a layer's experts)
 * Returns Σ_l C_l - B_non (> 0 = overrun forced by the clamp).
 * -------------------------------------------------------------------------- */
int64_t orc_layer_budget(int L, int E, const int64_t* hist, int64_t T, int64_t B_non, const int32_t* n_non,
                         int32_t* C_out, double* b_out, double* v_out) {
  double* b = (double*)malloc(sizeof(double) * (size_t)L);
  double bsum = 0.0;
  for (int l = 0; l < L; ++l) {
    double mean = 0.0;
    for (int e = 0; e < E; ++e) mean += (double)hist[(int64_t)l * E + e] / (double)T;
    mean /= E;
    double v = 0.0;
    for (int e = 0; e < E; ++e) {
      double d = (double)hist[(int64_t)l * E + e] / (double)T - mean;
      v += d * d;
    }
    v /= E;
    if (v_out) v_out[l] = v;
    if (v < 1e-12) v = 1e-12;
    b[l] = (double)(L - (l + 1) + 1) / v;
    bsum += b[l];
  }
  int64_t total = 0;
  for (int l = 0; l < L; ++l) {
    int64_t B = (int64_t)floor(b[l] / bsum * (double)B_non);
    if (B < 1) B = 1;
    /* R9: at most the layer's non-tuning experts; n_non NULL = every expert is non-tuning (E) */
    if (B > (n_non ? n_non[l] : E)) B = n_non ? n_non[l] : E;
    C_out[l] = (int32_t)B;
    if (b_out) b_out[l] = b[l];
    total += B;
  }
  free(b);
  return total - B_non;
}

/* ----------------------------------------------------------------------------
 * O10. Importance-based merge, eq.(2), reading R10:
 *   for each cluster c:  E_c = {e : cluster_of[e] == c}
 *     w_e = α_e / Σ_{e' in E_c} α_e'   (if Σ α = 0: w_e = 1/|E_c|)
 *     W_c = Σ_{e in E_c} w_e · W_e      (element-wise, fp64; caller rounds once)
 *   cluster_of[e] == -1: tuning expert, kept, not merged.
 *   remap[e] = slot of e in the compact layer: tuning experts first in
 *   ascending id, then clusters 0..C-1 (the per-layer expert count of
 *   exps_config).
 * experts: [E][numel] real; merged: [C][numel] real.  A cluster with no member
 * is an error (returns 1).
 * -------------------------------------------------------------------------- */
int orc_merge(int E, int64_t numel, const double* experts, const int32_t* cluster_of, const double* alpha, int C,
              double* merged, int32_t* remap) {
  double* wsum = (double*)calloc((size_t)C, sizeof(double));
  int* count = (int*)calloc((size_t)C, sizeof(int));
  for (int e = 0; e < E; ++e) {
    int c = cluster_of[e];
    if (c < -1 || c >= C) { free(wsum); free(count); return 1; }
    if (c >= 0) { wsum[c] += alpha[e]; count[c]++; }
  }
  for (int c = 0; c < C; ++c)
    if (count[c] == 0) { free(wsum); free(count); return 1; }
  double* we = (double*)malloc(sizeof(double) * (size_t)E);
  for (int e = 0; e < E; ++e) {
    int c = cluster_of[e];
    we[e] = 0.0;
    if (c >= 0) we[e] = wsum[c] > 0.0 ? alpha[e] / wsum[c] : 1.0 / count[c];
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < numel; ++i) {
    for (int c = 0; c < C; ++c) merged[(int64_t)c * numel + i] = 0.0;
    for (int e = 0; e < E; ++e) {
      int c = cluster_of[e];
      if (c >= 0) merged[(int64_t)c * numel + i] += we[e] * experts[(int64_t)e * numel + i];
    }
  }
  if (remap) {
    int slot = 0;
    for (int e = 0; e < E; ++e)
      if (cluster_of[e] == -1) remap[e] = slot++;
    for (int e = 0; e < E; ++e)
      if (cluster_of[e] >= 0) remap[e] = slot + cluster_of[e];
  }
  free(we);
  free(wsum);
  free(count);
  return 0;
}
