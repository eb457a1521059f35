/*
 * oracle.c -- CPU restatement of the reference INT8 training hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see i8t_oracle.h).  Written from the reference's
 * behaviour, not copied: convolutions are direct loops (exact integer sums, so
 * the order differs harmlessly from the reference's im2col+GEMM), floating
 * reductions keep the reference's sequential double order so that they agree
 * bit-for-bit with the compiled reference (tests/test_oracle_vs_ref.py).
 *
 * Build: oracle/Makefile (gcc -std=gnu11 -O3 -march=x86-64-v3 -fopenmp), the
 * same FP-contraction regime as the reference's gnu++20 build.
 */
#include "i8t_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define LCG_A 1664525u
#define LCG_C 1013904223u

/* ------------------------------------------------------------------------ */
/* LCG: X <- a*X + c mod 2^32, u = X * 2^-32 (quantize.hpp:32-50).           */

uint32_t or_lcg_next(uint32_t* state) {
  *state = LCG_A * *state + LCG_C;
  return *state;
}

/* k-step jump by binary doubling of the affine map. */
uint32_t or_lcg_jump(uint32_t state, uint64_t k) {
  uint32_t mul = 1u, add = 0u;          /* accumulated map x -> mul*x + add */
  uint32_t am = LCG_A, cm = LCG_C;      /* map for 2^bit steps */
  while (k) {
    if (k & 1u) { mul = am * mul; add = am * add + cm; }
    cm = am * cm + cm;
    am = am * am;
    k >>= 1u;
  }
  return mul * state + add;
}

/* ------------------------------------------------------------------------ */
/* Quantizer (quantize.cpp:11-87).                                           */

/* QuantParams::from_clip (quantize.cpp:11-14): s = c / 127.0f. */
int or_quant_params(float clip, float* scale_out) {
  if (!(clip > 0.0f) || !isfinite(clip)) return OR_EINVAL;
  *scale_out = clip / 127.0f;
  return OR_OK;
}

static inline double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* quantize_value (quantize.cpp:16-31): clamp and divide in double; nearest is
 * lround (ties away from zero); stochastic is floor + (u < frac) with exactly
 * one draw per element; result clamped to +-127. */
int or_quantize_value(float x, float clip, float scale, int mode, uint32_t* stream, int8_t* out) {
  if (!isfinite(x)) return OR_EDOMAIN;
  const double v = clampd((double)x, -(double)clip, (double)clip);
  const double scaled = clampd(v / (double)scale, -127.0, 127.0);
  long q;
  if (mode == OR_NEAREST) {
    q = lround(scaled);
  } else {
    const double fl = floor(scaled);
    const double frac = scaled - fl;
    const double u = (double)or_lcg_next(stream) * 0x1.0p-32;
    q = (long)fl + (u < frac ? 1 : 0);
  }
  if (q > 127) q = 127;
  if (q < -127) q = -127;
  *out = (int8_t)q;
  return OR_OK;
}

/* quantize (quantize.cpp:33-43): row-major walk, stream iff stochastic. */
int or_quantize(const float* x, int64_t n, float clip, int mode, uint32_t* stream, int8_t* q) {
  if ((mode == OR_STOCHASTIC) != (stream != NULL)) return OR_EINVAL;
  float s;
  int st = or_quant_params(clip, &s);
  if (st) return st;
  for (int64_t i = 0; i < n; ++i) {
    st = or_quantize_value(x[i], clip, s, mode, stream, &q[i]);
    if (st) return st;
  }
  return OR_OK;
}

/* quantize_partitioned (quantize.cpp:45-79): chunk k = [n*k/P, n*(k+1)/P)
 * draws from a fresh stream seeded base_seed + k. */
int or_quantize_partitioned(const float* x, int64_t n, float clip, uint32_t base_seed,
                            int partitions, int8_t* q) {
  if (partitions < 1) return OR_EINVAL;
  float s;
  int st = or_quant_params(clip, &s);
  if (st) return st;
  for (int k = 0; k < partitions; ++k) {
    const int64_t lo = n * k / partitions, hi = n * (k + 1) / partitions;
    uint32_t stream = base_seed + (uint32_t)k;
    for (int64_t i = lo; i < hi; ++i) {
      st = or_quantize_value(x[i], clip, s, OR_STOCHASTIC, &stream, &q[i]);
      if (st) return st;
    }
  }
  return OR_OK;
}

/* dequantize (quantize.cpp:81-87): float(q) * scale, one float multiply. */
void or_dequantize(const int8_t* q, int64_t n, float scale, float* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = (float)q[i] * scale;
}

/* ------------------------------------------------------------------------ */
/* Reductions (tensor.cpp:72-101), sequential double order.                  */

double or_sq_l2_norm(const float* x, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += (double)x[i] * (double)x[i];
  return acc;
}

double or_dot(const float* a, const float* b, int64_t n) {
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc += (double)a[i] * (double)b[i];
  return acc;
}

/* max_abs: float compare `a > m`, so NaN never wins (tensor.cpp:87-94). */
float or_max_abs(const float* x, int64_t n) {
  float m = 0.0f;
  for (int64_t i = 0; i < n; ++i) {
    const float a = fabsf(x[i]);
    if (a > m) m = a;
  }
  return m;
}

int or_has_nonfinite(const float* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) return 1;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* INT8 GEMM (gemm.cpp:18-40): exact integer sum, so any order is the same.  */

void or_gemm_i8(const int8_t* a, const int8_t* b, int64_t m, int64_t k, int64_t n, int32_t* c) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    int32_t* crow = c + i * n;
    for (int64_t j = 0; j < n; ++j) crow[j] = 0;
    for (int64_t kk = 0; kk < k; ++kk) {
      const int32_t av = a[i * k + kk];
      if (av == 0) continue;
      const int8_t* brow = b + kk * n;
      for (int64_t j = 0; j < n; ++j) crow[j] += av * (int32_t)brow[j];
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Convolution geometry (conv.hpp:14-28, conv.cpp:11-18) + EXT.              */

int64_t or_out_h(const or_geom* g) { return (g->h + 2 * g->pad_h - g->kh) / g->stride_h + 1; }
int64_t or_out_w(const or_geom* g) { return (g->w + 2 * g->pad_w - g->kw) / g->stride_w + 1; }

int or_geom_validate(const or_geom* g) {
  if (g->n < 1 || g->c < 1 || g->h < 1 || g->w < 1 || g->k < 1 || g->kh < 1 || g->kw < 1 ||
      g->stride_h < 1 || g->stride_w < 1 || g->pad_h < 0 || g->pad_w < 0)
    return OR_EINVAL;
  if (g->depthwise && g->k != g->c) return OR_EINVAL;
  if (g->h + 2 * g->pad_h < g->kh || g->w + 2 * g->pad_w < g->kw) return OR_EINVAL;
  if (!g->floor_mode &&
      ((g->h + 2 * g->pad_h - g->kh) % g->stride_h != 0 || (g->w + 2 * g->pad_w - g->kw) % g->stride_w != 0))
    return OR_EINVAL;
  return OR_OK;
}

/* im2col layout (conv.cpp:23-47): row (c*kh+i)*kw+j, column (n*OH+oh)*OW+ow. */
int or_im2col_i8(const int8_t* x, const or_geom* g, int8_t* out) {
  int st = or_geom_validate(g);
  if (st) return st;
  const int64_t oh = or_out_h(g), ow = or_out_w(g), cols = g->n * oh * ow;
  int64_t r = 0;
  for (int64_t c = 0; c < g->c; ++c)
    for (int64_t i = 0; i < g->kh; ++i)
      for (int64_t j = 0; j < g->kw; ++j, ++r)
        for (int64_t n = 0; n < g->n; ++n)
          for (int64_t p = 0; p < oh; ++p)
            for (int64_t q = 0; q < ow; ++q) {
              const int64_t ih = p * g->stride_h + i - g->pad_h, iw = q * g->stride_w + j - g->pad_w;
              int8_t v = 0;
              if (ih >= 0 && ih < g->h && iw >= 0 && iw < g->w) v = x[((n * g->c + c) * g->h + ih) * g->w + iw];
              out[r * cols + (n * oh + p) * ow + q] = v;
            }
  return OR_OK;
}

/* Range of output columns q for which iw = q*sw + j - pw lies in [0, W). */
static void valid_range(int64_t j, int64_t stride, int64_t pad, int64_t in, int64_t out, int64_t* lo,
                        int64_t* hi) {
  int64_t a = 0;
  while (a < out && a * stride + j - pad < 0) ++a;
  int64_t b = out;
  while (b > a && (b - 1) * stride + j - pad >= in) --b;
  *lo = a;
  *hi = b;
}

/* conv2d_q (conv.cpp:108-145): z[n,k,p,q] = float(double(s_a)*double(s_w)*acc). */
int or_conv_fwd(const int8_t* qa, const int8_t* qw, const or_geom* g, float s_a, float s_w,
                int32_t* acc_out, float* z_out) {
  int st = or_geom_validate(g);
  if (st) return st;
  const int64_t oh = or_out_h(g), ow = or_out_w(g);
  const int64_t kout = g->depthwise ? g->c : g->k;
  const double rescale = (double)s_a * (double)s_w;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t n = 0; n < g->n; ++n)
    for (int64_t ko = 0; ko < kout; ++ko) {
      int64_t* acc = (int64_t*)calloc((size_t)(oh * ow), sizeof(int64_t));
      const int64_t c_lo = g->depthwise ? ko : 0, c_hi = g->depthwise ? ko + 1 : g->c;
      for (int64_t c = c_lo; c < c_hi; ++c) {
        const int8_t* xc = qa + (n * g->c + c) * g->h * g->w;
        for (int64_t i = 0; i < g->kh; ++i)
          for (int64_t j = 0; j < g->kw; ++j) {
            const int64_t widx = g->depthwise ? (ko * g->kh + i) * g->kw + j
                                              : ((ko * g->c + c) * g->kh + i) * g->kw + j;
            const int64_t wv = qw[widx];
            if (wv == 0) continue;
            int64_t q_lo, q_hi;
            valid_range(j, g->stride_w, g->pad_w, g->w, ow, &q_lo, &q_hi);
            for (int64_t p = 0; p < oh; ++p) {
              const int64_t ih = p * g->stride_h + i - g->pad_h;
              if (ih < 0 || ih >= g->h) continue;
              const int8_t* xr = xc + ih * g->w;
              int64_t* ar = acc + p * ow;
              for (int64_t q = q_lo; q < q_hi; ++q) ar[q] += wv * xr[q * g->stride_w + j - g->pad_w];
            }
          }
      }
      const int64_t base = (n * kout + ko) * oh * ow;
      for (int64_t e = 0; e < oh * ow; ++e) {
        const int32_t a32 = (int32_t)acc[e];
        if (acc_out) acc_out[base + e] = a32;
        if (z_out) z_out[base + e] = (float)(rescale * (double)a32);
      }
      free(acc);
    }
  return OR_OK;
}

/* conv2d_backward_q dgrad (conv.cpp:197-203 and depthwise :159-184): the
 * scatter of W^T.G through col2im, accumulated in int64, then
 * float(double(s_gz)*double(s_w)*acc). */
int or_conv_dgrad(const int8_t* qg, const int8_t* qw, const or_geom* g, float s_g, float s_w,
                  int64_t* acc_out, float* ga_out) {
  int st = or_geom_validate(g);
  if (st) return st;
  const int64_t oh = or_out_h(g), ow = or_out_w(g);
  const int64_t kout = g->depthwise ? g->c : g->k;
  const double rescale = (double)s_g * (double)s_w;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t n = 0; n < g->n; ++n)
    for (int64_t c = 0; c < g->c; ++c) {
      int64_t* acc = (int64_t*)calloc((size_t)(g->h * g->w), sizeof(int64_t));
      const int64_t k_lo = g->depthwise ? c : 0, k_hi = g->depthwise ? c + 1 : kout;
      for (int64_t ko = k_lo; ko < k_hi; ++ko) {
        const int8_t* gk = qg + (n * kout + ko) * oh * ow;
        for (int64_t i = 0; i < g->kh; ++i)
          for (int64_t j = 0; j < g->kw; ++j) {
            const int64_t widx = g->depthwise ? (c * g->kh + i) * g->kw + j
                                              : ((ko * g->c + c) * g->kh + i) * g->kw + j;
            const int64_t wv = qw[widx];
            if (wv == 0) continue;
            int64_t q_lo, q_hi;
            valid_range(j, g->stride_w, g->pad_w, g->w, ow, &q_lo, &q_hi);
            for (int64_t p = 0; p < oh; ++p) {
              const int64_t ih = p * g->stride_h + i - g->pad_h;
              if (ih < 0 || ih >= g->h) continue;
              int64_t* ar = acc + ih * g->w;
              const int8_t* gr = gk + p * ow;
              for (int64_t q = q_lo; q < q_hi; ++q) ar[q * g->stride_w + j - g->pad_w] += wv * gr[q];
            }
          }
      }
      const int64_t base = (n * g->c + c) * g->h * g->w;
      for (int64_t e = 0; e < g->h * g->w; ++e) {
        if (acc_out) acc_out[base + e] = acc[e];
        if (ga_out) ga_out[base + e] = (float)(rescale * (double)acc[e]);
      }
      free(acc);
    }
  return OR_OK;
}

/* conv2d_backward_q wgrad (conv.cpp:186-195 and depthwise :170-172):
 * gW[k,c,i,j] = sum_{n,p,q} G[n,k,p,q] * A[n,c,ih,iw].  EXT: int64, no depth
 * bound; the float output keeps the reference's float(double(s)*acc) form. */
int or_conv_wgrad(const int8_t* qg, const int8_t* qa, const or_geom* g, float s_g, float s_a,
                  int64_t* acc_out, float* gw_out) {
  int st = or_geom_validate(g);
  if (st) return st;
  const int64_t oh = or_out_h(g), ow = or_out_w(g);
  const int64_t kout = g->depthwise ? g->c : g->k;
  const int64_t cin = g->depthwise ? 1 : g->c;
  const double rescale = (double)s_g * (double)s_a;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t ko = 0; ko < kout; ++ko)
    for (int64_t cw = 0; cw < cin; ++cw) {
      const int64_t c = g->depthwise ? ko : cw;
      for (int64_t i = 0; i < g->kh; ++i)
        for (int64_t j = 0; j < g->kw; ++j) {
          int64_t q_lo, q_hi;
          valid_range(j, g->stride_w, g->pad_w, g->w, ow, &q_lo, &q_hi);
          int64_t acc = 0;
          for (int64_t n = 0; n < g->n; ++n) {
            const int8_t* gk = qg + (n * kout + ko) * oh * ow;
            const int8_t* xc = qa + (n * g->c + c) * g->h * g->w;
            for (int64_t p = 0; p < oh; ++p) {
              const int64_t ih = p * g->stride_h + i - g->pad_h;
              if (ih < 0 || ih >= g->h) continue;
              const int8_t* gr = gk + p * ow;
              const int8_t* xr = xc + ih * g->w;
              int32_t part = 0;
              for (int64_t q = q_lo; q < q_hi; ++q) part += (int32_t)gr[q] * (int32_t)xr[q * g->stride_w + j - g->pad_w];
              acc += part;
            }
          }
          const int64_t widx = ((ko * cin + cw) * g->kh + i) * g->kw + j;
          if (acc_out) acc_out[widx] = acc;
          if (gw_out) gw_out[widx] = (float)(rescale * (double)acc);
        }
    }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* DSGC (clip.cpp:8-93).                                                     */

/* cosine_distance (clip.cpp:8-22): three sequential double sums. */
double or_cosine_distance(const float* g, const float* h, int64_t n) {
  double num = 0.0, sq_g = 0.0, sq_h = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double a = g[i], b = h[i];
    num += a * b;
    sq_g += a * a;
    sq_h += b * b;
  }
  if (sq_g == 0.0 && sq_h == 0.0) return 0.0;
  if (sq_g == 0.0 || sq_h == 0.0) return 1.0;
  return 1.0 - num / (sqrt(sq_g) * sqrt(sq_h));
}

/* measure_dc (clip.cpp:24-28): nearest quantize -> dequantize -> cosine. */
int or_measure_dc(const float* g, int64_t n, float clip, double* dc_out) {
  float s;
  int st = or_quant_params(clip, &s);
  if (st) return st;
  double num = 0.0, sq_g = 0.0, sq_h = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    int8_t q;
    st = or_quantize_value(g[i], clip, s, OR_NEAREST, NULL, &q);
    if (st) return st;
    const double a = g[i], b = (float)q * s;
    num += a * b;
    sq_g += a * a;
    sq_h += b * b;
  }
  if (sq_g == 0.0 && sq_h == 0.0) *dc_out = 0.0;
  else if (sq_g == 0.0 || sq_h == 0.0) *dc_out = 1.0;
  else *dc_out = 1.0 - num / (sqrt(sq_g) * sqrt(sq_h));
  return OR_OK;
}

typedef struct { float clip; double dc; } best_t;

static int consider(best_t* best, const float* g, int64_t n, float c) {
  if (!(c > 0.0f)) return OR_OK;
  double dc;
  int st = or_measure_dc(g, n, c, &dc);
  if (st) return st;
  if (dc < best->dc || (dc == best->dc && c > best->clip)) { best->clip = c; best->dc = dc; }
  return OR_OK;
}

static void track(best_t* best, double x, double f) {
  if (f < best->dc || (f == best->dc && (float)x > best->clip)) { best->clip = (float)x; best->dc = f; }
}

/* search_clip (clip.cpp:30-78): grid c_i = m*(float(i)/float(R)), i=1..R,
 * then `rounds` golden-section steps over [best-m/R, best+m/R]; ties go to
 * the larger clip; all-zero g returns {prev_clip, 0}. */
int or_search_clip(const float* g, int64_t n, int grid, int rounds, float prev_clip,
                   float* clip_out, double* dc_out) {
  if (grid < 8) return OR_EINVAL;
  const float m = or_max_abs(g, n);
  if (m == 0.0f) { *clip_out = prev_clip; *dc_out = 0.0; return OR_OK; }
  if (or_has_nonfinite(g, n)) return OR_EDOMAIN;
  best_t best = {0.0f, 2.0 + 1.0};
  int st;
  for (int i = 1; i <= grid; ++i) {
    st = consider(&best, g, n, m * ((float)i / (float)grid));
    if (st) return st;
  }
  if (rounds > 0) {
    const double step = (double)m / grid;
    double lo = (double)best.clip - step;
    if (lo < 0.0) lo = 0.0;
    double hi = (double)best.clip + step;
    if (hi > (double)m) hi = (double)m;
    const double kInvPhi = 0.6180339887498949;
    double x1 = hi - (hi - lo) * kInvPhi;
    double x2 = lo + (hi - lo) * kInvPhi;
    double f1, f2;
    if ((st = or_measure_dc(g, n, (float)x1, &f1))) return st;
    if ((st = or_measure_dc(g, n, (float)x2, &f2))) return st;
    track(&best, x1, f1);
    track(&best, x2, f2);
    for (int r = 0; r < rounds; ++r) {
      if (f1 < f2) {
        hi = x2; x2 = x1; f2 = f1;
        x1 = hi - (hi - lo) * kInvPhi;
        if ((st = or_measure_dc(g, n, (float)x1, &f1))) return st;
        track(&best, x1, f1);
      } else {
        lo = x1; x1 = x2; f1 = f2;
        x2 = lo + (hi - lo) * kInvPhi;
        if ((st = or_measure_dc(g, n, (float)x2, &f2))) return st;
        track(&best, x2, f2);
      }
    }
  }
  *clip_out = best.clip;
  *dc_out = best.dc;
  return OR_OK;
}

/* maybe_update (clip.cpp:80-93): Periodic Update. */
int or_maybe_update(or_clip_state* st, const float* g, int64_t n, int64_t iter, int grid, int rounds) {
  if (iter < st->iter_of_last_update) return OR_EINVAL;
  const int uninit = !(st->clip > 0.0f);
  const int due = uninit || st->iter_of_last_update < 0 || (iter - st->iter_of_last_update) >= st->period;
  int rc;
  if (due) {
    float c;
    double dc;
    if ((rc = or_search_clip(g, n, grid, rounds, st->clip, &c, &dc))) return rc;
    if (c > 0.0f) st->clip = c;
    st->last_dc = dc;
    st->iter_of_last_update = iter;
  } else {
    if (or_max_abs(g, n) == 0.0f) {
      st->last_dc = 0.0;
    } else {
      if ((rc = or_measure_dc(g, n, st->clip, &st->last_dc))) return rc;
    }
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* DCLR (lr_scale.cpp:8-20).                                                 */

int or_scale_factor(double dc, double alpha, double beta, int form, double* out) {
  if (!(alpha > 0.0)) return OR_EINVAL;
  if (!(beta > 0.0 && beta <= 1.0)) return OR_EINVAL;
  if (!(dc >= 0.0 && dc <= 2.0)) return OR_EINVAL;
  double raw;
  switch (form) {
    case OR_EXP: raw = exp(-alpha * dc); break;
    case OR_LINEAR: raw = 1.0 - dc; break;
    case OR_QUADRATIC: raw = 1.0 - dc * dc; break;
    default: raw = 1.0; break;
  }
  *out = raw > beta ? raw : beta;
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* quantize_gradient (layers.cpp:19-59).                                     */

int or_quantize_gradient(or_clip_state* st, const float* g, int64_t n, int64_t iter,
                         int grid, int rounds, int search_enabled, int lr_scaling_enabled,
                         double alpha, double beta, int form, uint32_t* stream,
                         int8_t* q_out, float* scale_out, double* stats_out) {
  int rc;
  if (search_enabled) {
    if ((rc = or_maybe_update(st, g, n, iter, grid, rounds))) return rc;
  } else {
    const float m = or_max_abs(g, n);
    if (m > 0.0f) {
      st->clip = m;
      if ((rc = or_measure_dc(g, n, m, &st->last_dc))) return rc;
    } else {
      st->last_dc = 0.0;
    }
    st->iter_of_last_update = iter;
  }
  const double dc = st->last_dc;
  double phi = 1.0;
  if (lr_scaling_enabled) {
    const double dcc = dc < 0.0 ? 0.0 : (dc > 2.0 ? 2.0 : dc);
    if ((rc = or_scale_factor(dcc, alpha, beta, form, &phi))) return rc;
  }
  stats_out[0] = dc;
  stats_out[1] = phi;
  if (or_max_abs(g, n) == 0.0f || !(st->clip > 0.0f)) {
    memset(q_out, 0, (size_t)n);
    or_quant_params(1.0f, scale_out);
    stats_out[2] = 0.0;
    stats_out[3] = 0.0;
    return OR_OK;
  }
  if ((rc = or_quantize(g, n, st->clip, OR_STOCHASTIC, stream, q_out))) return rc;
  float s;
  or_quant_params(st->clip, &s);
  *scale_out = s;
  double eps_sq = 0.0, gh = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const float ghat = (float)q_out[i] * s;
    const double e = (double)g[i] - (double)ghat;
    eps_sq += e * e;
  }
  for (int64_t i = 0; i < n; ++i) {
    const float ghat = (float)q_out[i] * s;
    gh += (double)ghat * (double)ghat;
  }
  stats_out[2] = sqrt(eps_sq);
  stats_out[3] = gh;
  return OR_OK;
}

/* SGD step of Trainer::train_step, momentum 0 (train.cpp:112-114):
 * w -= float(lr * g) with lr = base_lr_t * phi computed in double. */
void or_sgd_update(float* w, const float* g, int64_t n, double lr) {
  for (int64_t i = 0; i < n; ++i) w[i] -= (float)(lr * (double)g[i]);
}

/* ------------------------------------------------------------------------ */
/* Synthetic inputs: SplitMix64 + Box-Muller (rng.hpp:13-50).                */

typedef struct { uint64_t s; int have; double spare; } rng_t;

static uint64_t rng_u64(rng_t* r) {
  uint64_t z = (r->s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
static double rng_uniform(rng_t* r) { return (double)(rng_u64(r) >> 11) * 0x1.0p-53; }
static double rng_gauss(rng_t* r) {
  if (r->have) { r->have = 0; return r->spare; }
  double u1 = rng_uniform(r), u2 = rng_uniform(r);
  while (u1 <= 0.0) u1 = rng_uniform(r);
  const double rad = sqrt(-2.0 * log(u1)), th = 2.0 * 3.141592653589793 * u2;
  r->spare = rad * sin(th);
  r->have = 1;
  return rad * cos(th);
}

void or_fill_gaussian(float* x, int64_t n, uint64_t seed, double stddev, int relu) {
  rng_t r = {seed, 0, 0.0};
  for (int64_t i = 0; i < n; ++i) {
    float v = (float)(rng_gauss(&r) * stddev);
    x[i] = (relu && v < 0.0f) ? 0.0f : v;
  }
}

/* Laplace bulk with occasional x40 outliers (mirrors test_clip.cpp:12-22). */
void or_fill_gradient_like(float* x, int64_t n, uint64_t seed, double scale, double outlier_rate) {
  rng_t r = {seed, 0, 0.0};
  for (int64_t i = 0; i < n; ++i) {
    const double u = rng_uniform(&r) - 0.5;
    double v = -copysign(log(1.0 - 2.0 * fabs(u)), u) * scale;
    if (rng_uniform(&r) < outlier_rate) v *= 40.0;
    x[i] = (float)v;
  }
}

/* ------------------------------------------------------------------------ */
/* FP32 layers around the INT8 convolutions (layers.cpp:230-529), NCHW.      */
/* Sequential double sums in the reference's loop order; expressions are     */
/* written in the reference's form so GCC's FP contraction treats them alike */
/* (pinned against the compiled reference Trainer, tests/test_oracle_model). */

/* BatchNorm2d::forward, training (layers.cpp:262-291).  xhat (float, the
 * reference's cached_xhat_) and invstd (double per channel) are outputs for
 * the backward; running stats are updated in place. */
void or_bn_forward_train(const float* x, int64_t n, int64_t c, int64_t hw, const float* gamma, const float* beta,
                         float* running_mean, float* running_var, double momentum, double eps, float* y,
                         float* xhat, double* invstd_out) {
  const int64_t m = n * hw;
  for (int64_t ch = 0; ch < c; ++ch) {
    double sum = 0.0, sq = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const float* px = x + (i * c + ch) * hw;
      for (int64_t p = 0; p < hw; ++p) {
        sum += px[p];
        sq += (double)px[p] * (double)px[p];
      }
    }
    const double mean = sum / m;
    const double v0 = sq / m - mean * mean;
    const double var = v0 > 0.0 ? v0 : 0.0;
    const double invstd = 1.0 / sqrt(var + eps);
    invstd_out[ch] = invstd;
    running_mean[ch] = (float)((1.0 - momentum) * running_mean[ch] + momentum * mean);
    running_var[ch] = (float)((1.0 - momentum) * running_var[ch] + momentum * var);
    const double g = gamma[ch], b = beta[ch];
    for (int64_t i = 0; i < n; ++i) {
      const float* px = x + (i * c + ch) * hw;
      float* ph = xhat + (i * c + ch) * hw;
      float* py = y + (i * c + ch) * hw;
      for (int64_t p = 0; p < hw; ++p) {
        const double xv = ((double)px[p] - mean) * invstd;
        ph[p] = (float)xv;
        py[p] = (float)(g * xv + b);
      }
    }
  }
}

/* BatchNorm2d::forward, inference (layers.cpp:247-259). */
void or_bn_forward_eval(const float* x, int64_t n, int64_t c, int64_t hw, const float* gamma, const float* beta,
                        const float* running_mean, const float* running_var, double eps, float* y) {
  for (int64_t ch = 0; ch < c; ++ch) {
    const double invstd = 1.0 / sqrt((double)running_var[ch] + eps);
    const double mean = running_mean[ch];
    const double g = gamma[ch], b = beta[ch];
    for (int64_t i = 0; i < n; ++i) {
      const float* px = x + (i * c + ch) * hw;
      float* py = y + (i * c + ch) * hw;
      for (int64_t p = 0; p < hw; ++p) py[p] = (float)(g * (((double)px[p] - mean) * invstd) + b);
    }
  }
}

/* BatchNorm2d::backward (layers.cpp:295-323). */
void or_bn_backward(const float* g_out, const float* xhat, const double* invstd, int64_t n, int64_t c, int64_t hw,
                    const float* gamma, float* g_in, float* grad_gamma, float* grad_beta) {
  const int64_t m = n * hw;
  for (int64_t ch = 0; ch < c; ++ch) {
    double s1 = 0.0, s2 = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const float* pg = g_out + (i * c + ch) * hw;
      const float* ph = xhat + (i * c + ch) * hw;
      for (int64_t p = 0; p < hw; ++p) {
        s1 += pg[p];
        s2 += (double)pg[p] * (double)ph[p];
      }
    }
    grad_beta[ch] = (float)s1;
    grad_gamma[ch] = (float)s2;
    const double coeff = (double)gamma[ch] * invstd[ch];
    for (int64_t i = 0; i < n; ++i) {
      const float* pg = g_out + (i * c + ch) * hw;
      const float* ph = xhat + (i * c + ch) * hw;
      float* pi = g_in + (i * c + ch) * hw;
      for (int64_t p = 0; p < hw; ++p)
        pi[p] = (float)(coeff * ((double)pg[p] - s1 / m - (double)ph[p] * s2 / m));
    }
  }
}

/* Pool2d::forward (layers.cpp:349-391) with EXT zero-cost padding for max
 * pooling (padded taps never win; the reference Pool2d has no padding,
 * SURVEY.md A.3-5).  kind 0 = max (strict '>' keeps the first maximum; argmax
 * is the flat index h*W+w inside the (n,c) plane), 1 = average (double sum
 * over the window in (ki,kj) order / (k*k)).  floor-mode output size. */
int or_pool_forward(const float* x, int64_t n, int64_t c, int64_t h, int64_t w, int kind, int64_t k, int64_t s,
                    int64_t pad, float* y, int64_t* argmax) {
  if (k < 1 || s < 1 || pad < 0 || h + 2 * pad < k || w + 2 * pad < k || (kind == 1 && pad)) return OR_EINVAL;
  const int64_t oh = (h + 2 * pad - k) / s + 1, ow = (w + 2 * pad - k) / s + 1;
  for (int64_t i = 0; i < n * c; ++i) {
    const float* px = x + i * h * w;
    float* py = y + i * oh * ow;
    for (int64_t a = 0; a < oh; ++a)
      for (int64_t b = 0; b < ow; ++b) {
        if (kind == 0) {
          float best = -INFINITY;
          int64_t best_idx = 0;
          for (int64_t ki = 0; ki < k; ++ki)
            for (int64_t kj = 0; kj < k; ++kj) {
              const int64_t ih = a * s + ki - pad, iw = b * s + kj - pad;
              if (ih < 0 || ih >= h || iw < 0 || iw >= w) continue;
              const int64_t idx = ih * w + iw;
              if (px[idx] > best) {
                best = px[idx];
                best_idx = idx;
              }
            }
          py[a * ow + b] = best;
          if (argmax) argmax[i * oh * ow + a * ow + b] = best_idx;
        } else {
          double acc = 0.0;
          for (int64_t ki = 0; ki < k; ++ki)
            for (int64_t kj = 0; kj < k; ++kj) acc += px[(a * s + ki) * w + (b * s + kj)];
          py[a * ow + b] = (float)(acc / (double)(k * k));
        }
      }
  }
  return OR_OK;
}

/* Pool2d::backward (layers.cpp:393-415): float scatter-add in loop order. */
int or_pool_backward(const float* g_out, const int64_t* argmax, int64_t n, int64_t c, int64_t h, int64_t w, int kind,
                     int64_t k, int64_t s, int64_t pad, float* g_in) {
  if (k < 1 || s < 1 || pad < 0 || h + 2 * pad < k || w + 2 * pad < k || (kind == 1 && pad)) return OR_EINVAL;
  const int64_t oh = (h + 2 * pad - k) / s + 1, ow = (w + 2 * pad - k) / s + 1;
  memset(g_in, 0, sizeof(float) * (size_t)(n * c * h * w));
  for (int64_t i = 0; i < n * c; ++i) {
    const float* pg = g_out + i * oh * ow;
    float* pi = g_in + i * h * w;
    for (int64_t a = 0; a < oh; ++a)
      for (int64_t b = 0; b < ow; ++b) {
        if (kind == 0) {
          pi[argmax[i * oh * ow + a * ow + b]] += pg[a * ow + b];
        } else {
          const float share = pg[a * ow + b] / (float)(k * k);
          for (int64_t ki = 0; ki < k; ++ki)
            for (int64_t kj = 0; kj < k; ++kj) pi[(a * s + ki) * w + (b * s + kj)] += share;
        }
      }
  }
  return OR_OK;
}

/* SoftmaxCrossEntropy::loss_and_grad (layers.cpp:507-529): per row max, a
 * sequential double sum of exp, log_z, g = float((p - y)/n).  Returns the
 * mean loss; OR_EINVAL via *status for a label out of range. */
double or_softmax_ce(const float* logits, int64_t n, int64_t classes, const int32_t* labels, float* g_logits,
                     int* status) {
  double total = 0.0;
  *status = OR_OK;
  for (int64_t i = 0; i < n; ++i) {
    if (labels[i] < 0 || labels[i] >= classes) {
      *status = OR_EINVAL;
      return 0.0;
    }
    const float* row = logits + i * classes;
    double mx = row[0];
    for (int64_t c = 1; c < classes; ++c) mx = mx > (double)row[c] ? mx : (double)row[c];
    double sum = 0.0;
    for (int64_t c = 0; c < classes; ++c) sum += exp((double)row[c] - mx);
    const double log_z = mx + log(sum);
    total += log_z - (double)row[labels[i]];
    for (int64_t c = 0; c < classes; ++c) {
      const double p = exp((double)row[c] - log_z);
      const double yv = (c == labels[i]) ? 1.0 : 0.0;
      g_logits[i * classes + c] = (float)((p - yv) / (double)n);
    }
  }
  return total / (double)n;
}

/* Trainer::train_step momentum update (train.cpp:106-111):
 * buf = float(m*buf + g); w -= float(lr*buf). */
void or_sgd_momentum_update(float* w, const float* g, float* buf, int64_t n, double lr, double momentum) {
  for (int64_t i = 0; i < n; ++i) {
    buf[i] = (float)(momentum * buf[i] + g[i]);
    w[i] -= (float)(lr * buf[i]);
  }
}

/* conv2d_f32 forward (conv.cpp:206-236 through gemm_f32, gemm.cpp:66-82):
 * per output a double accumulator over r = (c, i, j) ascending (products of
 * two floats are exact in double, so contraction cannot change the sum);
 * padding taps contribute +-0.  Used for the FP32 calibration forwards
 * (train.cpp:29-32).  EXT geometry. */
int or_conv_fwd_f32(const float* x, const float* w, const or_geom* g, float* z) {
  int st = or_geom_validate(g);
  if (st) return st;
  const int64_t oh = or_out_h(g), ow = or_out_w(g);
  const int64_t kout = g->depthwise ? g->c : g->k;
#pragma omp parallel for collapse(2) schedule(static)
  for (int64_t n = 0; n < g->n; ++n)
    for (int64_t ko = 0; ko < kout; ++ko)
      for (int64_t p = 0; p < oh; ++p)
        for (int64_t q = 0; q < ow; ++q) {
          double acc = 0.0;
          const int64_t c_lo = g->depthwise ? ko : 0, c_hi = g->depthwise ? ko + 1 : g->c;
          for (int64_t c = c_lo; c < c_hi; ++c)
            for (int64_t i = 0; i < g->kh; ++i)
              for (int64_t j = 0; j < g->kw; ++j) {
                const int64_t ih = p * g->stride_h + i - g->pad_h, iw = q * g->stride_w + j - g->pad_w;
                if (ih < 0 || ih >= g->h || iw < 0 || iw >= g->w) continue;
                const int64_t widx = g->depthwise ? (ko * g->kh + i) * g->kw + j
                                                  : ((ko * g->c + c) * g->kh + i) * g->kw + j;
                const double a = w[widx];
                if (a == 0.0) continue;
                acc += a * (double)x[((n * g->c + c) * g->h + ih) * g->w + iw];
              }
          z[((n * kout + ko) * oh + p) * ow + q] = (float)acc;
        }
  return OR_OK;
}
