// quant.cu -- HBM-bound kernels of the INT8 training path on sm_100a:
//   K1/K2 nearest quantisers (activations, weights) with fused max_abs,
//   K3 fused stochastic gradient quantiser (DSGC d_c sums at the current clip,
//      eps / g_hat statistics, LCG jump-ahead in the reference's NCHW draw order),
//   K4 multi-candidate d_c reductions driving the DSGC clip search,
//   DCLR phi and the SGD+DCLR update.
// All floating reductions are double, reduced per block then across blocks in
// a fixed order (deterministic for a given n).  Vectorised float4 loads,
// warp-shuffle block reductions.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>

#include "internal.cuh"

namespace i8t_dev {

// ============================================================== scalar core
__device__ __forceinline__ float scale_of(float clip) { return __fdiv_rn(clip, 127.0f); }

// quantize_value, kNearest (quantize.cpp:16-31) computed exactly in FP32:
// lround(RN64(v/s)) == round-half-away(v/s) because RN64 cannot cross a
// half-integer for float v, s; the tie test a >= s*(k+1/2) is
// decided by the sign of one FMA.
__device__ __forceinline__ int quant_nearest(float x, float clip, float s, float inv_s) {
  const float v = fminf(fmaxf(x, -clip), clip);
  const float a = fabsf(v);
  float k = floorf(__fmaf_rn(a, inv_s, 0.5f));
  if (__fmaf_rn(-s, k + 0.5f, a) >= 0.0f) k += 1.0f;
  else if (__fmaf_rn(-s, k - 0.5f, a) < 0.0f) k -= 1.0f;
  k = fminf(k, 127.0f);
  const int qi = static_cast<int>(k);
  return v < 0.0f ? -qi : qi;
}

// quantize_value, kStochastic: floor(t) + (u < frac(t)) with t = RN64(v/s)
// clamped to +-127 and u = X * 2^-32.  FP32 decides when the margins exceed
// 2^-13 (|t32 - t| < 2e-5); otherwise the exact FP64 formula runs.
__device__ __forceinline__ int quant_stoch(float x, float clip, float s, float inv_s, uint32_t X) {
  if (x == 0.0f) return 0;
  const float v = fminf(fmaxf(x, -clip), clip);
  const float t = v * inv_s;
  const float fl = floorf(t);
  const float frac = t - fl;
  const float u = static_cast<float>(X >> 8) * 0x1.0p-24f;
  constexpr float D = 0x1.0p-13f;
  int q;
  if (frac > D && frac < 1.0f - D && fabsf(frac - u) > D) {
    q = static_cast<int>(fl) + (u < frac ? 1 : 0);
  } else {
    double td = static_cast<double>(v) / static_cast<double>(s);
    td = fmin(fmax(td, -127.0), 127.0);
    const double fd = floor(td);
    const double fr = td - fd;
    const double ud = static_cast<double>(X) * 0x1.0p-32;
    q = static_cast<int>(fd) + (ud < fr ? 1 : 0);
  }
  return max(-127, min(127, q));
}

__device__ __forceinline__ uint32_t apply(Affine m, uint32_t x) { return m.a * x + m.c; }

// ============================================================== block reduce
template <int NV>
__device__ __forceinline__ void block_reduce_store(double (&v)[NV], double* out, bool is_max0) {
  __shared__ double sh[NV][RED_THREADS / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double x = v[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, x, o);
      x = (is_max0 && j == 0) ? fmax(x, y) : x + y;
    }
    if (lane == 0) sh[j][wid] = x;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    const int j = threadIdx.x;
    double x = sh[j][0];
    for (int w = 1; w < RED_THREADS / 32; ++w) x = (is_max0 && j == 0) ? fmax(x, sh[j][w]) : x + sh[j][w];
    out[static_cast<size_t>(blockIdx.x) * NV + j] = x;
  }
}

// Sum partials[b][j] over blocks in index order; j == 0 is a max when is_max0.
__device__ __forceinline__ double reduce_col(const double* p, int nblk, int stride, int j, bool is_max) {
  double x = p[j];
  for (int b = 1; b < nblk; ++b) x = is_max ? fmax(x, p[static_cast<size_t>(b) * stride + j]) : x + p[static_cast<size_t>(b) * stride + j];
  return x;
}

__device__ __forceinline__ double cosine_from(double num, double sq_g, double sq_h) {
  if (sq_g == 0.0 && sq_h == 0.0) return 0.0;
  if (sq_g == 0.0 || sq_h == 0.0) return 1.0;
  return 1.0 - num / (sqrt(sq_g) * sqrt(sq_h));
}

// phi(d_c) (lr_scale.cpp:8-20); argument checks are done on the host.
__device__ __forceinline__ double phi_of(double dc, double alpha, double beta, int form) {
  double raw;
  if (form == 0) raw = exp(-alpha * dc);
  else if (form == 1) raw = 1.0 - dc;
  else if (form == 2) raw = 1.0 - dc * dc;
  else raw = 1.0;
  return fmax(raw, beta);
}

// ============================================================== K1: nearest quantisers
// Flat / row-padded activations: x [rows][cols] -> q [rows][ld_q], amax fused.
__global__ void __launch_bounds__(256) k_quant_nearest_rows(const float* __restrict__ x, int64_t rows, int64_t cols,
                                                            const float* __restrict__ clip_p, int8_t* __restrict__ q,
                                                            int64_t ld_q, float* amax, int* err) {
  const float clip = *clip_p, s = scale_of(clip), inv_s = 1.0f / s;
  float m = 0.0f;
  bool bad = false;
  if (ld_q == cols && (cols * rows) % 4 == 0) {
    const int64_t n4 = rows * cols / 4;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    char4* q4 = reinterpret_cast<char4*>(q);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
      const float4 v = __ldg(x4 + i);
      bad |= !isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w);
      m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
      char4 o;
      o.x = (signed char)quant_nearest(v.x, clip, s, inv_s);
      o.y = (signed char)quant_nearest(v.y, clip, s, inv_s);
      o.z = (signed char)quant_nearest(v.z, clip, s, inv_s);
      o.w = (signed char)quant_nearest(v.w, clip, s, inv_s);
      q4[i] = o;
    }
  } else {
    const int64_t tot = rows * ld_q;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t r = i / ld_q, c = i - r * ld_q;
      int8_t o = 0;
      if (c < cols) {
        const float v = x[r * cols + c];
        bad |= !isfinite(v);
        m = fmaxf(m, fabsf(v));
        o = (int8_t)quant_nearest(v, clip, s, inv_s);
      }
      q[i] = o;
    }
  }
  if (bad) atomicOr(err, ERR_NONFINITE);
  if (amax) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    // non-negative floats order like their bit patterns
    if ((threadIdx.x & 31) == 0 && m > 0.0f) atomicMax(reinterpret_cast<int*>(amax), __float_as_int(m));
  }
}

// NCHW float -> NHWC int8 (channel stride c_pad), via a 32x32 smem transpose.
__global__ void __launch_bounds__(256) k_quant_nearest_nchw(const float* __restrict__ x, int64_t C, int64_t HW,
                                                            const float* __restrict__ clip_p, int8_t* __restrict__ q,
                                                            int64_t c_pad, float* amax, int* err) {
  __shared__ float tile[32][33];
  const float clip = *clip_p, s = scale_of(clip), inv_s = 1.0f / s;
  const int64_t n = blockIdx.z;
  const int64_t c0 = blockIdx.y * 32, p0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32
  float m = 0.0f;
  bool bad = false;
  for (int r = ty; r < 32; r += 8) {
    const int64_t c = c0 + r, p = p0 + tx;
    float v = 0.0f;
    if (c < C && p < HW) {
      v = x[(n * C + c) * HW + p];
      bad |= !isfinite(v);
      m = fmaxf(m, fabsf(v));
    }
    tile[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t p = p0 + r, c = c0 + tx;
    if (p < HW && c < c_pad) q[(n * HW + p) * c_pad + c] = (c < C) ? (int8_t)quant_nearest(tile[tx][r], clip, s, inv_s) : 0;
  }
  if (bad) atomicOr(err, ERR_NONFINITE);
  if (amax) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0f) atomicMax(reinterpret_cast<int*>(amax), __float_as_int(m));
  }
}

// K2: weights KCRS (or KRSC) float -> KRSC int8 [K][ld_krsc] and CRSK int8 [C][ld_crsk].
__global__ void __launch_bounds__(256) k_quant_weight(const float* __restrict__ w, int src_krsc, int64_t K, int64_t C,
                                                      int64_t RS, const float* __restrict__ clip_p, int8_t* q_krsc,
                                                      int64_t c_pad, int64_t ld_krsc, int8_t* q_crsk, int64_t k_pad,
                                                      int64_t ld_crsk, float* amax, int* err) {
  const float clip = *clip_p, s = scale_of(clip), inv_s = 1.0f / s;
  const int64_t tot = K * C * RS;
  float m = 0.0f;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t k, c, rs;
    if (src_krsc) {
      c = i % C;
      rs = (i / C) % RS;
      k = i / (C * RS);
    } else {
      rs = i % RS;
      c = (i / RS) % C;
      k = i / (RS * C);
    }
    const float v = w[i];
    bad |= !isfinite(v);
    m = fmaxf(m, fabsf(v));
    const int8_t qv = (int8_t)quant_nearest(v, clip, s, inv_s);
    if (q_krsc) q_krsc[k * ld_krsc + rs * c_pad + c] = qv;
    if (q_crsk) q_crsk[c * ld_crsk + rs * k_pad + k] = qv;
  }
  if (bad) atomicOr(err, ERR_NONFINITE);
  if (amax) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0f) atomicMax(reinterpret_cast<int*>(amax), __float_as_int(m));
  }
}

__global__ void k_dequantize(const int8_t* __restrict__ q, int64_t n, const float* __restrict__ clip_p,
                             float* __restrict__ out) {
  const float s = scale_of(*clip_p);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __fmul_rn(static_cast<float>(q[i]), s);
}

// ============================================================== LCG tables
// tab[i] = jump map for (offset + i*stride) steps.
__global__ void k_lcg_table(Affine* tab, int64_t count, int64_t stride, int64_t offset) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    tab[i] = lcg_jump_map(static_cast<uint64_t>(offset + i * stride));
}

// ============================================================== K3: fused gradient quantiser
// g is NHWC [N*HW][C] (C % 4 == 0) or flat (FLAT: C == 1 logically).  Element
// (n, c, hw) consumes LCG draw index (n*C + c)*HW + hw + 1 relative to the
// state at entry (reference NCHW order, quantize.cpp:38-41).
// Per-block partials (8 doubles): max|g|, nonfinite, sum g^2, sum g*gn, sum gn^2,
// sum (g-gs)^2, sum gs^2, 0     (gn: nearest at clip; gs: stochastic).
constexpr int QG_NV = 8;

template <bool FLAT, bool DC_SUMS>
__global__ void __launch_bounds__(RED_THREADS) k_quant_grad(const float* __restrict__ g, int64_t numel, int64_t C,
                                                            int64_t HW, const Affine* __restrict__ tab_a,
                                                            const Affine* __restrict__ tab_b,
                                                            const Affine* __restrict__ tab_n, Affine step,
                                                            const DsgcState* st, const float* clip_override,
                                                            const uint32_t* __restrict__ lcg_state,
                                                            int8_t* __restrict__ q, double* partials) {
  float clip = clip_override ? *clip_override : st->v.clip;
  if (!(clip > 0.0f)) clip = 1.0f;  // only reachable with an all-zero g (q == 0 either way)
  const float s = scale_of(clip), inv_s = 1.0f / s;
  const uint32_t X0 = *lcg_state;
  double acc[QG_NV] = {0, 0, 0, 0, 0, 0, 0, 0};
  float m = 0.0f;
  const int64_t n4 = numel / 4;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  char4* q4 = reinterpret_cast<char4*>(q);
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n4; f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = f * 4;
    uint32_t X;
    if (FLAT) {
      X = apply(tab_b[e >> 16], apply(tab_a[e & 0xFFFF], X0));  // tab_a[j] = jump(j+1), tab_b[h] = jump(h<<16)
    } else {
      const int64_t pix = e / C, c = e - pix * C;
      const int64_t nimg = pix / HW, hw = pix - nimg * HW;
      X = apply(tab_n[nimg], apply(tab_b[c], apply(tab_a[hw], X0)));  // tab_a[hw]=jump(hw+1), tab_b[c]=jump(c*HW)
    }
    const float4 v4 = __ldg(g4 + f);
    const float vv[4] = {v4.x, v4.y, v4.z, v4.w};
    signed char qq[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (j) X = apply(step, X);
      const float v = vv[j];
      const float a = fabsf(v);
      if (!isfinite(v)) acc[1] += 1.0;
      m = fmaxf(m, a);
      const int qs = quant_stoch(v, clip, s, inv_s, X);
      qq[j] = (signed char)qs;
      const float gs = __fmul_rn(static_cast<float>(qs), s);
      const double vd = v;
      const double e2 = vd - static_cast<double>(gs);
      acc[5] = fma(e2, e2, acc[5]);
      acc[6] = fma((double)gs, (double)gs, acc[6]);
      if (DC_SUMS) {
        const float gn = __fmul_rn(static_cast<float>(quant_nearest(v, clip, s, inv_s)), s);
        acc[2] = fma(vd, vd, acc[2]);
        acc[3] = fma(vd, (double)gn, acc[3]);
        acc[4] = fma((double)gn, (double)gn, acc[4]);
      }
    }
    q4[f] = make_char4(qq[0], qq[1], qq[2], qq[3]);
  }
  acc[0] = m;
  block_reduce_store<QG_NV>(acc, partials, true);
}

// Finalize of K3 (quantize_gradient tail, layers.cpp:32-58).  mode bits:
// 1 = d_c from the DC sums (non-search iteration), 2 = lr scaling enabled.
__global__ void k_quant_grad_finalize(DsgcState* st, const double* partials, int nblk, int mode, double alpha,
                                      double beta, int form, uint32_t* lcg_state, int64_t numel, int* err) {
  __shared__ double tot[QG_NV];
  if (threadIdx.x < QG_NV) tot[threadIdx.x] = reduce_col(partials, nblk, QG_NV, threadIdx.x, threadIdx.x == 0);
  __syncthreads();
  if (threadIdx.x != 0) return;
  const float m = static_cast<float>(tot[0]);
  const bool nonfinite = tot[1] > 0.0;
  if (nonfinite && m != 0.0f) atomicOr(err, ERR_NONFINITE);
  if (mode & 1) st->v.last_dc = (m == 0.0f) ? 0.0 : cosine_from(tot[3], tot[2], tot[4]);
  const double dc = st->v.last_dc;
  st->v.lr_scale = (mode & 2) ? phi_of(fmin(fmax(dc, 0.0), 2.0), alpha, beta, form) : 1.0;
  st->v.max_abs = m;
  if (m == 0.0f || !(st->v.clip > 0.0f)) {
    st->v.scale = scale_of(1.0f);
    st->v.eps_norm = 0.0;
    st->v.ghat_sqnorm = 0.0;
    st->v.flags = (nonfinite ? 1u : 0u) | 2u;
  } else {
    st->v.scale = scale_of(st->v.clip);
    st->v.eps_norm = sqrt(tot[5]);
    st->v.ghat_sqnorm = tot[6];
    st->v.flags = nonfinite ? 1u : 0u;
    *lcg_state = apply(lcg_jump_map(static_cast<uint64_t>(numel)), *lcg_state);
  }
}

// ============================================================== K4: d_c statistics for NC candidates
// partial layout: [0] max|g|, [1] nonfinite, [2] sum g^2, [3+2j] sum g*gh_j, [4+2j] sum gh_j^2
template <int NC>
__global__ void __launch_bounds__(RED_THREADS) k_dc_stats(const float* __restrict__ g, int64_t n,
                                                          const float* __restrict__ cands, const int32_t* active,
                                                          double* partials) {
  constexpr int NV = 3 + 2 * NC;
  if (active && *active == 0) return;
  float cl[NC > 0 ? NC : 1], sc[NC > 0 ? NC : 1], is[NC > 0 ? NC : 1];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    cl[j] = cands[j];
    sc[j] = scale_of(cl[j]);
    is[j] = 1.0f / sc[j];
  }
  double acc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) acc[j] = 0.0;
  float m = 0.0f;
  const int64_t n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto body = [&](float v) {
    if (!isfinite(v)) acc[1] += 1.0;
    m = fmaxf(m, fabsf(v));
    const double vd = v;
    acc[2] = fma(vd, vd, acc[2]);
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const float gh = __fmul_rn(static_cast<float>(quant_nearest(v, cl[j], sc[j], is[j])), sc[j]);
      acc[3 + 2 * j] = fma(vd, (double)gh, acc[3 + 2 * j]);
      acc[4 + 2 * j] = fma((double)gh, (double)gh, acc[4 + 2 * j]);
    }
  };
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < n4; f += stride) {
    const float4 v = __ldg(g4 + f);
    body(v.x);
    body(v.y);
    body(v.z);
    body(v.w);
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) body(g[i]);
  acc[0] = m;
  block_reduce_store<NV>(acc, partials, true);
}

// ---- DSGC search state machine (clip.cpp:30-78), single thread per step.
__device__ __forceinline__ void ds_consider(DsgcState* st, float c, double dc) {
  if (!(c > 0.0f)) return;
  if (dc < st->best_dc || (dc == st->best_dc && c > st->best_clip)) {
    st->best_clip = c;
    st->best_dc = dc;
  }
}
__device__ __forceinline__ void ds_track(DsgcState* st, double x, double f) {
  if (f < st->best_dc || (f == st->best_dc && static_cast<float>(x) > st->best_clip)) {
    st->best_clip = static_cast<float>(x);
    st->best_dc = f;
  }
}
__device__ __forceinline__ void ds_grid_chunk(DsgcState* st, int R) {
  const int left = R - st->grid_done;
  const int nc = left < 32 ? left : 32;
  for (int j = 0; j < nc; ++j) {
    const int i = st->grid_done + j + 1;
    st->cand[j] = __fmul_rn(st->m, __fdiv_rn(static_cast<float>(i), static_cast<float>(R)));
  }
  st->ncand = nc;
}
constexpr double kInvPhi = 0.6180339887498949;

// Stage 0: after the k_dc_stats<0> pass: m, non-finite, sum g^2.
__global__ void k_search_begin(DsgcState* st, const double* partials, int nblk, int R, float prev_clip, int prev_from_state,
                               int* err) {
  if (prev_from_state) prev_clip = st->v.clip;
  __shared__ double tot[3];
  if (threadIdx.x < 3) tot[threadIdx.x] = reduce_col(partials, nblk, 3, threadIdx.x, threadIdx.x == 0);
  __syncthreads();
  if (threadIdx.x) return;
  st->m = static_cast<float>(tot[0]);
  st->v.max_abs = st->m;
  st->sq_g = tot[2];
  st->prev_clip = prev_clip;
  st->best_clip = 0.0f;
  st->best_dc = 3.0;
  st->grid_done = 0;
  st->phase = 0;
  if (st->m == 0.0f) {
    st->active = 0;  // all-zero g: {prev_clip, 0}
    st->best_clip = prev_clip;
    st->best_dc = 0.0;
    return;
  }
  if (tot[1] > 0.0) {
    atomicOr(err, ERR_NONFINITE);
    st->active = 0;
    st->best_clip = prev_clip;
    st->best_dc = 0.0;
    return;
  }
  st->active = 1;
  ds_grid_chunk(st, R);
}

// After a k_dc_stats<NC> pass over st->cand.
__global__ void k_search_step(DsgcState* st, const double* partials, int nblk, int nc, int R, int rounds) {
  constexpr int MAXV = 3 + 2 * 32;
  __shared__ double tot[MAXV];
  const int nv = 3 + 2 * nc;
  if (st->active == 0) return;
  for (int j = threadIdx.x; j < nv; j += blockDim.x) tot[j] = reduce_col(partials, nblk, nv, j, j == 0);
  __syncthreads();
  if (threadIdx.x) return;
  double dcs[32];
  for (int j = 0; j < nc; ++j) dcs[j] = cosine_from(tot[3 + 2 * j], st->sq_g, tot[4 + 2 * j]);
  if (st->phase == 0) {  // grid
    for (int j = 0; j < nc; ++j) ds_consider(st, st->cand[j], dcs[j]);
    st->grid_done += nc;
    if (st->grid_done < R) {
      ds_grid_chunk(st, R);
      return;
    }
    if (rounds <= 0) {
      st->active = 0;
      return;
    }
    const double step = static_cast<double>(st->m) / R;
    double lo = static_cast<double>(st->best_clip) - step;
    double hi = static_cast<double>(st->best_clip) + step;
    lo = lo < 0.0 ? 0.0 : lo;
    hi = hi > static_cast<double>(st->m) ? static_cast<double>(st->m) : hi;
    st->lo = lo;
    st->hi = hi;
    // x1 = hi - (hi-lo)*kInvPhi, x2 = lo + (hi-lo)*kInvPhi as GCC contracts them
    st->x1 = __fma_rn(-(hi - lo), kInvPhi, hi);
    st->x2 = __fma_rn(hi - lo, kInvPhi, lo);
    st->cand[0] = static_cast<float>(st->x1);
    st->cand[1] = static_cast<float>(st->x2);
    st->ncand = 2;
    st->phase = 1;
    return;
  }
  if (st->phase == 1) {  // golden init: f1, f2
    st->f1 = dcs[0];
    st->f2 = dcs[1];
    ds_track(st, st->x1, st->f1);
    ds_track(st, st->x2, st->f2);
  } else {  // round (phase-2) just measured
    const int r = st->phase - 2;
    (void)r;
    if (st->pad_ == 0) {  // new x1 measured
      st->f1 = dcs[0];
      ds_track(st, st->x1, st->f1);
    } else {
      st->f2 = dcs[0];
      ds_track(st, st->x2, st->f2);
    }
  }
  const int next_round = st->phase - 1;  // rounds completed so far
  if (next_round >= rounds) {
    st->active = 0;
    return;
  }
  if (st->f1 < st->f2) {
    st->hi = st->x2;
    st->x2 = st->x1;
    st->f2 = st->f1;
    st->x1 = __fma_rn(-(st->hi - st->lo), kInvPhi, st->hi);
    st->cand[0] = static_cast<float>(st->x1);
    st->pad_ = 0;
  } else {
    st->lo = st->x1;
    st->x1 = st->x2;
    st->f1 = st->f2;
    st->x2 = __fma_rn(st->hi - st->lo, kInvPhi, st->lo);
    st->cand[0] = static_cast<float>(st->x2);
    st->pad_ = 1;
  }
  st->ncand = 1;
  st->phase += 1;
}

// End of maybe_update's search branch (clip.cpp:84-88) or raw search_clip.
__global__ void k_search_end(DsgcState* st, int64_t iter, int update_state, float* clip_out, double* dc_out) {
  if (threadIdx.x) return;
  const float c = st->best_clip;
  const double dc = st->best_dc;
  if (clip_out) *clip_out = c;
  if (dc_out) *dc_out = dc;
  if (update_state) {
    if (c > 0.0f) st->v.clip = c;
    st->v.last_dc = dc;
    st->v.iter_of_last_update = iter;
  }
}

// Search-disabled branch of quantize_gradient (layers.cpp:27-36): clip = max_abs.
__global__ void k_clip_from_max(DsgcState* st, const double* partials, int nblk, int64_t iter) {
  __shared__ double m;
  if (threadIdx.x == 0) m = reduce_col(partials, nblk, 3, 0, true);
  __syncthreads();
  if (threadIdx.x) return;
  const float mf = static_cast<float>(m);
  if (mf > 0.0f) st->v.clip = mf;
  st->v.iter_of_last_update = iter;
}

// Plain reductions -> device scalars.
__global__ void k_fin_scalar(const double* partials, int nblk, int nv, int which, float* out_f, double* out_d,
                             int32_t* out_i) {
  if (threadIdx.x) return;
  const double v = reduce_col(partials, nblk, nv, which, which == 0);
  if (out_f) *out_f = static_cast<float>(v);
  if (out_d) *out_d = v;
  if (out_i) *out_i = v > 0.0 ? 1 : 0;
}

__global__ void k_fin_measure_dc(const double* partials, int nblk, double* out, int* err) {
  __shared__ double tot[5];
  if (threadIdx.x < 5) tot[threadIdx.x] = reduce_col(partials, nblk, 5, threadIdx.x, threadIdx.x == 0);
  __syncthreads();
  if (threadIdx.x) return;
  if (tot[1] > 0.0) atomicOr(err, ERR_NONFINITE);
  *out = cosine_from(tot[3], tot[2], tot[4]);
}

// dot / cosine: partials [0] sum a*b [1] sum a^2 [2] sum b^2
__global__ void __launch_bounds__(RED_THREADS) k_dot3(const float* __restrict__ a, const float* __restrict__ b,
                                                      int64_t n, double* partials) {
  double acc[3] = {0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = a[i], y = b[i];
    acc[0] = fma(x, y, acc[0]);
    acc[1] = fma(x, x, acc[1]);
    acc[2] = fma(y, y, acc[2]);
  }
  block_reduce_store<3>(acc, partials, false);
}

__global__ void k_fin_cosine(const double* partials, int nblk, double* dot_out, double* cos_out) {
  if (threadIdx.x) return;
  const double num = reduce_col(partials, nblk, 3, 0, false);
  const double sa = reduce_col(partials, nblk, 3, 1, false);
  const double sb = reduce_col(partials, nblk, 3, 2, false);
  if (dot_out) *dot_out = num;
  if (cos_out) *cos_out = cosine_from(num, sa, sb);
}

// Plain stochastic quantize of a flat tensor (no statistics), and partitioned.
__global__ void k_quant_partitioned(const float* __restrict__ x, int64_t n, const float* __restrict__ clip_p,
                                    uint32_t base_seed, int parts, int8_t* __restrict__ q, int* err) {
  const float clip = *clip_p, s = scale_of(clip), inv_s = 1.0f / s;
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    // chunk k = largest k with n*k/P <= i
    int64_t k = (i * parts) / n;
    while (k + 1 < parts && (n * (k + 1)) / parts <= i) ++k;
    while (k > 0 && (n * k) / parts > i) --k;
    const int64_t lo = (n * k) / parts;
    const uint32_t X = apply(lcg_jump_map(static_cast<uint64_t>(i - lo + 1)), base_seed + static_cast<uint32_t>(k));
    const float v = x[i];
    bad |= !isfinite(v);
    q[i] = (int8_t)quant_stoch(v, clip, s, inv_s, X);
  }
  if (bad) atomicOr(err, ERR_NONFINITE);
}

// ============================================================== optimiser
// w -= float(lr * g), lr = base_lr * phi (train.cpp:97-117, momentum 0).
__global__ void __launch_bounds__(256) k_sgd_dclr(float* __restrict__ w, const float* __restrict__ grad, int64_t n,
                                                  double base_lr, const DsgcState* st) {
  const double lr = st ? base_lr * st->v.lr_scale : base_lr;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    w[i] -= static_cast<float>(lr * static_cast<double>(grad[i]));
}

// ============================================================== layout helpers
__global__ void k_nhwc_to_nchw_f32(const float* __restrict__ src, int64_t C, int64_t HW, int64_t ld,
                                   float* __restrict__ dst) {
  __shared__ float tile[32][33];
  const int64_t n = blockIdx.z, c0 = blockIdx.y * 32, p0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int64_t p = p0 + r, c = c0 + tx;
    tile[r][tx] = (p < HW && c < C) ? src[(n * HW + p) * ld + c] : 0.0f;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t c = c0 + r, p = p0 + tx;
    if (c < C && p < HW) dst[(n * C + c) * HW + p] = tile[tx][r];
  }
}

__global__ void k_nchw_to_nhwc_i8(const int8_t* __restrict__ src, int64_t C, int64_t HW, int8_t* __restrict__ dst,
                                  int64_t c_pad) {
  const int64_t n = blockIdx.z;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < HW * c_pad; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / c_pad, c = i - p * c_pad;
    dst[n * HW * c_pad + i] = (c < C) ? src[(n * C + c) * HW + p] : (int8_t)0;
  }
}

__global__ void k_kcrs_relayout_i8(const int8_t* __restrict__ src, int64_t K, int64_t C, int64_t RS, int8_t* dst,
                                   int64_t pad, int64_t ld, int to_crsk) {
  const int64_t tot = K * C * RS;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rs = i % RS, c = (i / RS) % C, k = i / (RS * C);
    if (to_crsk) dst[c * ld + rs * pad + k] = src[i];
    else dst[k * ld + rs * pad + c] = src[i];
  }
}

// Non-search branch of maybe_update: last_dc = max_abs == 0 ? 0 : measure_dc(g, clip).
__global__ void k_fin_maybe_dc(DsgcState* st, const double* partials, int nblk, int* err) {
  __shared__ double tot[5];
  if (threadIdx.x < 5) tot[threadIdx.x] = reduce_col(partials, nblk, 5, threadIdx.x, threadIdx.x == 0);
  __syncthreads();
  if (threadIdx.x) return;
  const float m = static_cast<float>(tot[0]);
  st->v.max_abs = m;
  if (m == 0.0f) {
    st->v.last_dc = 0.0;
    return;
  }
  if (tot[1] > 0.0) atomicOr(err, ERR_NONFINITE);
  st->v.last_dc = cosine_from(tot[3], tot[2], tot[4]);
}

// Plain stochastic quantize tail: non-finite check, advance the stream by n.
__global__ void k_fin_stoch(const double* partials, int nblk, uint32_t* lcg_state, int64_t n, int* err) {
  if (threadIdx.x) return;
  if (reduce_col(partials, nblk, QG_NV, 1, false) > 0.0) atomicOr(err, ERR_NONFINITE);
  *lcg_state = apply(lcg_jump_map(static_cast<uint64_t>(n)), *lcg_state);
}

// ============================================================== host launchers
int red_blocks(int64_t n) {
  int64_t b = (n + RED_THREADS * 8 - 1) / (RED_THREADS * 8);
  if (b < 1) b = 1;
  if (b > 592) b = 592;
  return static_cast<int>(b);
}

static int grid_for(int64_t n, int threads = 256, int64_t cap = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return static_cast<int>(b);
}

}  // namespace i8t_dev

using namespace i8t_dev;

// ---- entry points implemented here are declared in i8t_cuda.h; Ctx plumbing in capi.cu
#define CTX(c) reinterpret_cast<Ctx*>(c)
#define LAUNCHED(n) count_launch(n)

extern "C" {

int i8t_quantize_nearest_rows(i8t_ctx* ctx, const float* x, int64_t rows, int64_t cols, const float* clip, int8_t* q,
                              int64_t ld_q, float* amax, int accumulate_amax) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !clip || !q || rows < 0 || cols < 0 || ld_q < cols) return set_error(I8T_EINVAL, "quantize: bad arguments");
  if (rows * cols == 0) return I8T_OK;
  if (amax && !accumulate_amax) cudaMemsetAsync(amax, 0, sizeof(float), c->stream);
  k_quant_nearest_rows<<<grid_for(rows * ld_q / 4 + 1), 256, 0, c->stream>>>(x, rows, cols, clip, q, ld_q, amax, c->d_err);
  LAUNCHED(1);
  return cuda_check("k_quant_nearest_rows");
}

int i8t_quantize_nearest(i8t_ctx* ctx, const float* x, int64_t n, const float* clip, int8_t* q, float* amax,
                         int accumulate_amax) {
  return i8t_quantize_nearest_rows(ctx, x, 1, n, clip, q, n, amax, accumulate_amax);
}

int i8t_quantize_nearest_nchw_to_nhwc(i8t_ctx* ctx, const float* x, int64_t n, int64_t c, int64_t hw, const float* clip,
                                      int8_t* q, int64_t c_pad, float* amax, int accumulate_amax) {
  Ctx* cx = CTX(ctx);
  if (!cx || !x || !clip || !q || c_pad < c || n < 0) return set_error(I8T_EINVAL, "quantize_nchw: bad arguments");
  if (n * c * hw == 0) return I8T_OK;
  if (amax && !accumulate_amax) cudaMemsetAsync(amax, 0, sizeof(float), cx->stream);
  dim3 grid((unsigned)((hw + 31) / 32), (unsigned)((c_pad + 31) / 32), (unsigned)n);
  k_quant_nearest_nchw<<<grid, 256, 0, cx->stream>>>(x, c, hw, clip, q, c_pad, amax, cx->d_err);
  LAUNCHED(1);
  return cuda_check("k_quant_nearest_nchw");
}

int i8t_quantize_weight(i8t_ctx* ctx, const float* w, int src_krsc, int64_t k, int64_t c, int64_t kh, int64_t kw,
                        const float* clip, int8_t* q_krsc, int64_t c_pad, int64_t ld_krsc, int8_t* q_crsk, int64_t k_pad,
                        int64_t ld_crsk, float* amax) {
  Ctx* cx = CTX(ctx);
  if (!cx || !w || !clip || (q_krsc && (c_pad < c || ld_krsc < kh * kw * c_pad)) ||
      (q_crsk && (k_pad < k || ld_crsk < kh * kw * k_pad)))
    return set_error(I8T_EINVAL, "quantize_weight: bad arguments");
  if (q_krsc && (c_pad != c || ld_krsc != kh * kw * c_pad)) cudaMemsetAsync(q_krsc, 0, k * ld_krsc, cx->stream);
  if (q_crsk && (k_pad != k || ld_crsk != kh * kw * k_pad)) cudaMemsetAsync(q_crsk, 0, c * ld_crsk, cx->stream);
  if (amax) cudaMemsetAsync(amax, 0, sizeof(float), cx->stream);
  k_quant_weight<<<grid_for(k * c * kh * kw), 256, 0, cx->stream>>>(w, src_krsc, k, c, kh * kw, clip, q_krsc, c_pad,
                                                                     ld_krsc, q_crsk, k_pad, ld_crsk, amax, cx->d_err);
  LAUNCHED(1);
  return cuda_check("k_quant_weight");
}

int i8t_dequantize(i8t_ctx* ctx, const int8_t* q, int64_t n, const float* clip, float* out) {
  Ctx* c = CTX(ctx);
  if (!c || !q || !clip || !out) return set_error(I8T_EINVAL, "dequantize: bad arguments");
  if (!n) return I8T_OK;
  k_dequantize<<<grid_for(n), 256, 0, c->stream>>>(q, n, clip, out);
  LAUNCHED(1);
  return cuda_check("k_dequantize");
}

int i8t_nhwc_to_nchw_f32(i8t_ctx* ctx, const float* src, int64_t n, int64_t c, int64_t hw, int64_t ld, float* dst) {
  Ctx* cx = CTX(ctx);
  if (!cx || !src || !dst || ld < c) return set_error(I8T_EINVAL, "nhwc_to_nchw: bad arguments");
  if (n * c * hw == 0) return I8T_OK;
  dim3 grid((unsigned)((hw + 31) / 32), (unsigned)((c + 31) / 32), (unsigned)n);
  k_nhwc_to_nchw_f32<<<grid, 256, 0, cx->stream>>>(src, c, hw, ld, dst);
  LAUNCHED(1);
  return cuda_check("k_nhwc_to_nchw_f32");
}

int i8t_nchw_to_nhwc_i8(i8t_ctx* ctx, const int8_t* src, int64_t n, int64_t c, int64_t hw, int8_t* dst, int64_t c_pad) {
  Ctx* cx = CTX(ctx);
  if (!cx || !src || !dst || c_pad < c) return set_error(I8T_EINVAL, "nchw_to_nhwc: bad arguments");
  if (!n) return I8T_OK;
  dim3 grid((unsigned)grid_for(hw * c_pad, 256, 1024), 1, (unsigned)n);
  k_nchw_to_nhwc_i8<<<grid, 256, 0, cx->stream>>>(src, c, hw, dst, c_pad);
  LAUNCHED(1);
  return cuda_check("k_nchw_to_nhwc_i8");
}

int i8t_kcrs_to_krsc_i8(i8t_ctx* ctx, const int8_t* src, int64_t k, int64_t c, int64_t kh, int64_t kw, int8_t* dst,
                        int64_t c_pad, int64_t ld) {
  Ctx* cx = CTX(ctx);
  if (!cx || !src || !dst || c_pad < c || ld < kh * kw * c_pad) return set_error(I8T_EINVAL, "kcrs_to_krsc: bad arguments");
  cudaMemsetAsync(dst, 0, k * ld, cx->stream);
  k_kcrs_relayout_i8<<<grid_for(k * c * kh * kw), 256, 0, cx->stream>>>(src, k, c, kh * kw, dst, c_pad, ld, 0);
  LAUNCHED(1);
  return cuda_check("k_kcrs_relayout_i8");
}

int i8t_kcrs_to_crsk_i8(i8t_ctx* ctx, const int8_t* src, int64_t k, int64_t c, int64_t kh, int64_t kw, int8_t* dst,
                        int64_t k_pad, int64_t ld) {
  Ctx* cx = CTX(ctx);
  if (!cx || !src || !dst || k_pad < k || ld < kh * kw * k_pad) return set_error(I8T_EINVAL, "kcrs_to_crsk: bad arguments");
  cudaMemsetAsync(dst, 0, c * ld, cx->stream);
  k_kcrs_relayout_i8<<<grid_for(k * c * kh * kw), 256, 0, cx->stream>>>(src, k, c, kh * kw, dst, k_pad, ld, 1);
  LAUNCHED(1);
  return cuda_check("k_kcrs_relayout_i8");
}

// ---- reductions
static int launch_stats0(Ctx* c, const float* x, int64_t n, int& nblk) {
  nblk = red_blocks(n);
  double* p = ensure_partials(c, (size_t)nblk * 3);
  if (!p) return set_error(I8T_ECUDA, "partials alloc failed");
  k_dc_stats<0><<<nblk, RED_THREADS, 0, c->stream>>>(x, n, nullptr, nullptr, p);
  LAUNCHED(1);
  return cuda_check("k_dc_stats<0>");
}

int i8t_max_abs(i8t_ctx* ctx, const float* x, int64_t n, float* out) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !out) return set_error(I8T_EINVAL, "max_abs: bad arguments");
  int nblk, rc = launch_stats0(c, x, n, nblk);
  if (rc) return rc;
  k_fin_scalar<<<1, 32, 0, c->stream>>>(c->d_partials, nblk, 3, 0, out, nullptr, nullptr);
  LAUNCHED(1);
  return cuda_check("k_fin_scalar");
}

int i8t_sq_l2_norm(i8t_ctx* ctx, const float* x, int64_t n, double* out) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !out) return set_error(I8T_EINVAL, "sq_l2_norm: bad arguments");
  int nblk, rc = launch_stats0(c, x, n, nblk);
  if (rc) return rc;
  k_fin_scalar<<<1, 32, 0, c->stream>>>(c->d_partials, nblk, 3, 2, nullptr, out, nullptr);
  LAUNCHED(1);
  return cuda_check("k_fin_scalar");
}

int i8t_has_nonfinite(i8t_ctx* ctx, const float* x, int64_t n, int32_t* out) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !out) return set_error(I8T_EINVAL, "has_nonfinite: bad arguments");
  int nblk, rc = launch_stats0(c, x, n, nblk);
  if (rc) return rc;
  k_fin_scalar<<<1, 32, 0, c->stream>>>(c->d_partials, nblk, 3, 1, nullptr, nullptr, out);
  LAUNCHED(1);
  return cuda_check("k_fin_scalar");
}

int i8t_dot(i8t_ctx* ctx, const float* a, const float* b, int64_t n, double* out) {
  Ctx* c = CTX(ctx);
  if (!c || !a || !b || !out) return set_error(I8T_EINVAL, "dot: bad arguments");
  const int nblk = red_blocks(n);
  double* p = ensure_partials(c, (size_t)nblk * 3);
  if (!p) return set_error(I8T_ECUDA, "partials alloc failed");
  k_dot3<<<nblk, RED_THREADS, 0, c->stream>>>(a, b, n, p);
  k_fin_cosine<<<1, 32, 0, c->stream>>>(p, nblk, out, nullptr);
  LAUNCHED(2);
  return cuda_check("k_dot3");
}

int i8t_cosine_distance(i8t_ctx* ctx, const float* g, const float* h, int64_t n, double* out) {
  Ctx* c = CTX(ctx);
  if (!c || !g || !h || !out) return set_error(I8T_EINVAL, "cosine_distance: bad arguments");
  const int nblk = red_blocks(n);
  double* p = ensure_partials(c, (size_t)nblk * 3);
  if (!p) return set_error(I8T_ECUDA, "partials alloc failed");
  k_dot3<<<nblk, RED_THREADS, 0, c->stream>>>(g, h, n, p);
  k_fin_cosine<<<1, 32, 0, c->stream>>>(p, nblk, nullptr, out);
  LAUNCHED(2);
  return cuda_check("k_dot3");
}

int i8t_measure_dc(i8t_ctx* ctx, const float* g, int64_t n, float clip, double* out) {
  Ctx* c = CTX(ctx);
  if (!c || !g || !out) return set_error(I8T_EINVAL, "measure_dc: bad arguments");
  if (!(clip > 0.0f) || !std::isfinite(clip)) return set_error(I8T_EINVAL, "QuantParams: clip must be positive and finite");
  float* dclip = reinterpret_cast<float*>(ensure_scratch(c, 256));
  if (!dclip) return set_error(I8T_ECUDA, "scratch alloc failed");
  cudaMemcpyAsync(dclip, &clip, sizeof(float), cudaMemcpyHostToDevice, c->stream);
  const int nblk = red_blocks(n);
  double* p = ensure_partials(c, (size_t)nblk * 5);
  if (!p) return set_error(I8T_ECUDA, "partials alloc failed");
  k_dc_stats<1><<<nblk, RED_THREADS, 0, c->stream>>>(g, n, dclip, nullptr, p);
  k_fin_measure_dc<<<1, 32, 0, c->stream>>>(p, nblk, out, c->d_err);
  LAUNCHED(2);
  // the host clip is copied from a stack variable: make the copy complete before returning
  cudaStreamSynchronize(c->stream);
  return cuda_check("k_dc_stats<1>");
}

// search over g into the DsgcState st (device).  Returns launches via LAUNCHED.
static int run_search(Ctx* c, DsgcState* st, const float* g, int64_t n, int R, int rounds, float prev_clip,
                      int prev_from_state) {
  int nblk, rc = launch_stats0(c, g, n, nblk);
  if (rc) return rc;
  k_search_begin<<<1, 32, 0, c->stream>>>(st, c->d_partials, nblk, R, prev_clip, prev_from_state, c->d_err);
  LAUNCHED(1);
  double* p = ensure_partials(c, (size_t)nblk * (3 + 2 * 32));
  if (!p) return set_error(I8T_ECUDA, "partials alloc failed");
  for (int done = 0; done < R; done += 32) {
    const int nc = (R - done) < 32 ? (R - done) : 32;
    if (nc == 32) k_dc_stats<32><<<nblk, RED_THREADS, 0, c->stream>>>(g, n, st->cand, &st->active, p);
    else if (nc >= 16) {
      // pad to 32 evaluations would change nothing but cost; use exact count templates
      switch (nc) {
#define CASE(K) case K: k_dc_stats<K><<<nblk, RED_THREADS, 0, c->stream>>>(g, n, st->cand, &st->active, p); break;
        CASE(16) CASE(17) CASE(18) CASE(19) CASE(20) CASE(21) CASE(22) CASE(23) CASE(24) CASE(25) CASE(26) CASE(27)
        CASE(28) CASE(29) CASE(30) CASE(31)
#undef CASE
      }
    } else {
      switch (nc) {
#define CASE(K) case K: k_dc_stats<K><<<nblk, RED_THREADS, 0, c->stream>>>(g, n, st->cand, &st->active, p); break;
        CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13)
        CASE(14) CASE(15)
#undef CASE
      }
    }
    k_search_step<<<1, 128, 0, c->stream>>>(st, p, nblk, nc, R, rounds);
    LAUNCHED(2);
  }
  if (rounds > 0) {
    k_dc_stats<2><<<nblk, RED_THREADS, 0, c->stream>>>(g, n, st->cand, &st->active, p);
    k_search_step<<<1, 128, 0, c->stream>>>(st, p, nblk, 2, R, rounds);
    LAUNCHED(2);
    for (int r = 0; r < rounds; ++r) {
      k_dc_stats<1><<<nblk, RED_THREADS, 0, c->stream>>>(g, n, st->cand, &st->active, p);
      k_search_step<<<1, 128, 0, c->stream>>>(st, p, nblk, 1, R, rounds);
      LAUNCHED(2);
    }
  }
  return cuda_check("search_clip");
}

int i8t_search_clip(i8t_ctx* ctx, const float* g, int64_t n, int grid, int rounds, float prev_clip, float* clip_out,
                    double* dc_out) {
  Ctx* c = CTX(ctx);
  if (!c || !g) return set_error(I8T_EINVAL, "search_clip: bad arguments");
  if (grid < 8) return set_error(I8T_EINVAL, "search_clip: grid resolution must be >= 8");
  DsgcState* st = reinterpret_cast<DsgcState*>(ensure_scratch(c, sizeof(DsgcState)));
  if (!st) return set_error(I8T_ECUDA, "scratch alloc failed");
  int rc = run_search(c, st, g, n, grid, rounds, prev_clip, 0);
  if (rc) return rc;
  k_search_end<<<1, 32, 0, c->stream>>>(st, 0, 0, clip_out, dc_out);
  LAUNCHED(1);
  return cuda_check("k_search_end");
}

int64_t i8t_dsgc_state_size(void) { return static_cast<int64_t>(sizeof(DsgcState)); }

int i8t_dsgc_init(i8t_ctx* ctx, void* state, int64_t period) {
  Ctx* c = CTX(ctx);
  if (!c || !state) return set_error(I8T_EINVAL, "dsgc_init: bad arguments");
  DsgcState h{};
  h.v.iter_of_last_update = -1;
  h.v.period = period;
  h.v.lr_scale = 1.0;
  cudaMemcpyAsync(state, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream);
  cudaStreamSynchronize(c->stream);
  return cuda_check("dsgc_init");
}

int i8t_dsgc_read(i8t_ctx* ctx, const void* state, i8t_dsgc_view* out) {
  Ctx* c = CTX(ctx);
  if (!c || !state || !out) return set_error(I8T_EINVAL, "dsgc_read: bad arguments");
  cudaMemcpyAsync(out, state, sizeof(i8t_dsgc_view), cudaMemcpyDeviceToHost, c->stream);
  cudaStreamSynchronize(c->stream);
  return cuda_check("dsgc_read");
}

int i8t_dsgc_write(i8t_ctx* ctx, void* state, const i8t_dsgc_view* in) {
  Ctx* c = CTX(ctx);
  if (!c || !state || !in) return set_error(I8T_EINVAL, "dsgc_write: bad arguments");
  cudaMemcpyAsync(state, in, sizeof(i8t_dsgc_view), cudaMemcpyHostToDevice, c->stream);
  cudaStreamSynchronize(c->stream);
  return cuda_check("dsgc_write");
}


int i8t_maybe_update(i8t_ctx* ctx, void* state, const float* g, int64_t n, int64_t iter, int grid, int rounds, int due) {
  Ctx* c = CTX(ctx);
  DsgcState* st = reinterpret_cast<DsgcState*>(state);
  if (!c || !st || !g) return set_error(I8T_EINVAL, "maybe_update: bad arguments");
  if (grid < 8) return set_error(I8T_EINVAL, "search_clip: grid resolution must be >= 8");
  if (due) {
    int rc = run_search(c, st, g, n, grid, rounds, 0.0f, 1);
    if (rc) return rc;
    k_search_end<<<1, 32, 0, c->stream>>>(st, iter, 1, nullptr, nullptr);
    LAUNCHED(1);
    return cuda_check("maybe_update");
  }
  const int nblk = red_blocks(n);
  double* p = ensure_partials(c, (size_t)nblk * 5);
  if (!p) return set_error(I8T_ECUDA, "partials alloc failed");
  k_dc_stats<1><<<nblk, RED_THREADS, 0, c->stream>>>(g, n, &st->v.clip, nullptr, p);
  k_fin_maybe_dc<<<1, 32, 0, c->stream>>>(st, p, nblk, c->d_err);
  LAUNCHED(2);
  return cuda_check("maybe_update");
}

// LCG draw-order tables for the gradient quantiser, cached per (n, c, hw).
// NHWC: tab[0:hw] = jump(hw+1), tab[hw:hw+c] = jump(c*HW), tab[hw+c:] = jump(n*C*HW)
// FLAT: tab[0:65536] = jump(j+1), tab[65536:] = jump(h << 16)
static Affine* lcg_tables(Ctx* c, bool flat, int64_t n_img, int64_t C, int64_t HW, int64_t numel) {
  const int64_t key_n = flat ? -2 : n_img, key_c = flat ? (numel + 65535) / 65536 : C, key_hw = flat ? 65536 : HW;
  const int64_t need = flat ? 65536 + key_c : HW + C + n_img;
  if (c->d_tab && c->tab_n == key_n && c->tab_c == key_c && c->tab_hw == key_hw) return c->d_tab;
  if ((size_t)need > c->tab_cap) {
    if (c->d_tab) cudaFree(c->d_tab);
    c->d_tab = nullptr;
    if (cudaMalloc(&c->d_tab, need * sizeof(Affine)) != cudaSuccess) return nullptr;
    c->tab_cap = need;
  }
  if (flat) {
    k_lcg_table<<<grid_for(65536), 256, 0, c->stream>>>(c->d_tab, 65536, 1, 1);
    k_lcg_table<<<grid_for(key_c), 256, 0, c->stream>>>(c->d_tab + 65536, key_c, 65536, 0);
  } else {
    k_lcg_table<<<grid_for(HW), 256, 0, c->stream>>>(c->d_tab, HW, 1, 1);
    k_lcg_table<<<grid_for(C), 256, 0, c->stream>>>(c->d_tab + HW, C, HW, 0);
    k_lcg_table<<<grid_for(n_img), 256, 0, c->stream>>>(c->d_tab + HW + C, n_img, C * HW, 0);
  }
  LAUNCHED(flat ? 2 : 3);
  c->tab_n = key_n;
  c->tab_c = key_c;
  c->tab_hw = key_hw;
  return c->d_tab;
}

// One pass of K3.  clip_override: device clip used instead of st->v.clip (plain quantize).
static int launch_quant_grad(Ctx* c, DsgcState* st, const float* clip_override, const float* g, int64_t n_img, int64_t C,
                             int64_t HW, bool dc_sums, uint32_t* lcg, int8_t* q, int& nblk) {
  const int64_t numel = n_img * C * HW;
  const bool flat = (C == 1);
  if (numel % 4 != 0 || (!flat && C % 4 != 0))
    return set_error(I8T_EUNSUPPORTED, "quantize_gradient: needs C % 4 == 0 (or flat) and numel % 4 == 0");
  Affine* tab = lcg_tables(c, flat, n_img, C, HW, numel);
  if (!tab) return set_error(I8T_ECUDA, "lcg table alloc failed");
  nblk = red_blocks(numel);
  double* p = ensure_partials(c, (size_t)nblk * QG_NV);
  if (!p) return set_error(I8T_ECUDA, "partials alloc failed");
  const Affine step = flat ? lcg_jump_map(1) : lcg_jump_map(static_cast<uint64_t>(HW));
  const Affine* ta = tab;
  const Affine* tb = flat ? tab + 65536 : tab + HW;
  const Affine* tn = flat ? nullptr : tab + HW + C;
  const int64_t Ck = flat ? 1 : C;
  if (flat) {
    if (dc_sums) k_quant_grad<true, true><<<nblk, RED_THREADS, 0, c->stream>>>(g, numel, Ck, HW, ta, tb, tn, step, st, clip_override, lcg, q, p);
    else k_quant_grad<true, false><<<nblk, RED_THREADS, 0, c->stream>>>(g, numel, Ck, HW, ta, tb, tn, step, st, clip_override, lcg, q, p);
  } else {
    if (dc_sums) k_quant_grad<false, true><<<nblk, RED_THREADS, 0, c->stream>>>(g, numel, Ck, HW, ta, tb, tn, step, st, clip_override, lcg, q, p);
    else k_quant_grad<false, false><<<nblk, RED_THREADS, 0, c->stream>>>(g, numel, Ck, HW, ta, tb, tn, step, st, clip_override, lcg, q, p);
  }
  LAUNCHED(1);
  return cuda_check("k_quant_grad");
}

int i8t_quantize_gradient(i8t_ctx* ctx, void* state, const float* g, int64_t n_img, int64_t C, int64_t HW, int64_t iter,
                          int grid, int rounds, int search_enabled, int due, int lr_scaling_enabled, double alpha,
                          double beta, int form, uint32_t* lcg_state, int8_t* q, int64_t ld_q) {
  Ctx* c = CTX(ctx);
  DsgcState* st = reinterpret_cast<DsgcState*>(state);
  if (!c || !st || !g || !lcg_state || !q || n_img < 1 || C < 1 || HW < 1) return set_error(I8T_EINVAL, "quantize_gradient: bad arguments");
  if (ld_q != C) return set_error(I8T_EUNSUPPORTED, "quantize_gradient: ld_q must equal C");
  if (lr_scaling_enabled) {
    if (!(alpha > 0.0)) return set_error(I8T_EINVAL, "scale_factor: alpha must be > 0");
    if (!(beta > 0.0 && beta <= 1.0)) return set_error(I8T_EINVAL, "scale_factor: beta must be in (0,1]");
  }
  const int64_t numel = n_img * C * HW;
  int rc, nblk;
  bool dc_sums;
  if (search_enabled) {
    if (grid < 8) return set_error(I8T_EINVAL, "search_clip: grid resolution must be >= 8");
    if (due) {
      if ((rc = run_search(c, st, g, numel, grid, rounds, 0.0f, 1))) return rc;
      k_search_end<<<1, 32, 0, c->stream>>>(st, iter, 1, nullptr, nullptr);
      LAUNCHED(1);
      dc_sums = false;
    } else {
      dc_sums = true;
    }
  } else {
    int nb0;
    if ((rc = launch_stats0(c, g, numel, nb0))) return rc;
    k_clip_from_max<<<1, 32, 0, c->stream>>>(st, c->d_partials, nb0, iter);
    LAUNCHED(1);
    dc_sums = true;
  }
  if ((rc = launch_quant_grad(c, st, nullptr, g, n_img, C, HW, dc_sums, lcg_state, q, nblk))) return rc;
  const int mode = (dc_sums ? 1 : 0) | (lr_scaling_enabled ? 2 : 0);
  k_quant_grad_finalize<<<1, 32, 0, c->stream>>>(st, c->d_partials, nblk, mode, alpha, beta, form, lcg_state, numel, c->d_err);
  LAUNCHED(1);
  return cuda_check("quantize_gradient");
}

int i8t_quantize_stochastic(i8t_ctx* ctx, const float* x, int64_t n, const float* clip, uint32_t* lcg_state, int8_t* q) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !clip || !lcg_state || !q) return set_error(I8T_EINVAL, "quantize: stream required iff mode is stochastic");
  if (n == 0) return I8T_OK;
  DsgcState* st = reinterpret_cast<DsgcState*>(ensure_scratch(c, sizeof(DsgcState)));
  if (!st) return set_error(I8T_ECUDA, "scratch alloc failed");
  int rc, nblk;
  if (n % 4 != 0) return set_error(I8T_EUNSUPPORTED, "quantize_stochastic: numel % 4 != 0 (pad on the host)");
  if ((rc = launch_quant_grad(c, st, clip, x, 1, 1, n, false, lcg_state, q, nblk))) return rc;
  k_fin_stoch<<<1, 32, 0, c->stream>>>(c->d_partials, nblk, lcg_state, n, c->d_err);
  LAUNCHED(1);
  return cuda_check("quantize_stochastic");
}

int i8t_quantize_partitioned(i8t_ctx* ctx, const float* x, int64_t n, const float* clip, uint32_t base_seed, int parts,
                             int8_t* q) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !clip || !q) return set_error(I8T_EINVAL, "quantize_partitioned: bad arguments");
  if (parts < 1) return set_error(I8T_EINVAL, "quantize_partitioned: partitions must be >= 1");
  if (n == 0) return I8T_OK;
  k_quant_partitioned<<<grid_for(n), 256, 0, c->stream>>>(x, n, clip, base_seed, parts, q, c->d_err);
  LAUNCHED(1);
  return cuda_check("k_quant_partitioned");
}

int i8t_sgd_dclr(i8t_ctx* ctx, float* w, const float* grad, int64_t n, double base_lr, const void* state) {
  Ctx* c = CTX(ctx);
  if (!c || !w || !grad) return set_error(I8T_EINVAL, "sgd: bad arguments");
  if (!n) return I8T_OK;
  k_sgd_dclr<<<grid_for(n), 256, 0, c->stream>>>(w, grad, n, base_lr, reinterpret_cast<const DsgcState*>(state));
  LAUNCHED(1);
  return cuda_check("k_sgd_dclr");
}

int i8t_scale_factor(double dc, double alpha, double beta, int form, double* out) {
  if (!(alpha > 0.0)) return set_error(I8T_EINVAL, "scale_factor: alpha must be > 0");
  if (!(beta > 0.0 && beta <= 1.0)) return set_error(I8T_EINVAL, "scale_factor: beta must be in (0,1]");
  if (!(dc >= 0.0 && dc <= 2.0)) return set_error(I8T_EINVAL, "scale_factor: dc must be in [0,2]");
  double raw;
  switch (form) {
    case 0: raw = std::exp(-alpha * dc); break;
    case 1: raw = 1.0 - dc; break;
    case 2: raw = 1.0 - dc * dc; break;
    default: raw = 1.0; break;
  }
  *out = raw > beta ? raw : beta;
  return I8T_OK;
}

int i8t_lcg_jump_host(uint32_t state, uint64_t k, uint32_t* out) {
  if (!out) return set_error(I8T_EINVAL, "lcg_jump: null output");
  const Affine m = lcg_jump_map(k);
  *out = m.a * state + m.c;
  return I8T_OK;
}

}  // extern "C"
