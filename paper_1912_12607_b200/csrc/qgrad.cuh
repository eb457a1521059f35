// qgrad.cuh -- K3, the fused gradient quantiser (quantize_gradient,
// layers.cpp:19-59), templated over its input source so the same stochastic
// quantisation + DSGC statistics run on a materialised gradient (PlainSrc) or
// on a value computed on the fly (the fused BatchNorm backward, bnfuse.cu).
#pragma once
#include <cuda_runtime.h>

#include "internal.cuh"
#include "qcore.cuh"

namespace i8t_dev {

// Input source: fetch() issues the raw loads of one float4 of consecutive
// elements (so the kernel can keep several in flight), value() turns them into
// the gradient values; init() receives the first channel of the thread's fixed
// channel quad (NHWC) before any load.
struct PlainSrc {
  const float4* g;
  using Raw = float4;
  __device__ __forceinline__ void init(uint32_t) {}
  __device__ __forceinline__ Raw fetch(uint32_t e4) const { return __ldg(g + e4); }
  __device__ __forceinline__ float4 value(const Raw& r) const { return r; }
  __device__ __forceinline__ float4 value_fast(const Raw& r, bool&) const { return r; }
};

// totals layout of K3 (QG_NV doubles): max|g|, nonfinite, sum g^2, sum g*gn,
// sum gn^2, sum (g-gs)^2, sum gs^2, 0.
constexpr int QG_NV = 8;

struct QgFin {
  int mode;  // bit0: d_c from the sums (non-search), bit1: lr scaling, bit2: plain quantize (no DSGC state)
  double alpha, beta;
  int form;
  uint32_t advance;  // LCG draws consumed by the whole (global) tensor
};

// Tail of quantize_gradient (layers.cpp:32-58) from global totals.
static __device__ void fin_quant_grad(DsgcState* st, const double* tot, const QgFin& f, uint32_t* lcg_state, int* err) {
  const float m = static_cast<float>(tot[0]);
  const bool nonfinite = tot[1] > 0.0;
  if (f.mode & 4) {  // plain stochastic quantize (quantize.cpp:33-43): any non-finite throws
    if (nonfinite) atomicOr(err, ERR_NONFINITE);
    *lcg_state = apply(lcg_jump_map(f.advance), *lcg_state);
    return;
  }
  if (nonfinite && m != 0.0f) atomicOr(err, ERR_NONFINITE);
  if (f.mode & 1) st->v.last_dc = (m == 0.0f) ? 0.0 : cosine_from(tot[3], tot[2], tot[4]);
  const double dc = st->v.last_dc;
  st->v.lr_scale = (f.mode & 2) ? phi_of(fmin(fmax(dc, 0.0), 2.0), f.alpha, f.beta, f.form) : 1.0;
  st->v.max_abs = m;
  if (m == 0.0f || !(st->v.clip > 0.0f)) {  // zero-gradient skip: no draws (layers.cpp:40-47)
    st->v.clip_q = 1.0f;
    st->v.scale = scale_of(1.0f);
    st->v.eps_norm = 0.0;
    st->v.ghat_sqnorm = 0.0;
    st->v.flags = (nonfinite ? 1u : 0u) | 2u;
  } else {
    st->v.clip_q = st->v.clip;
    st->v.scale = scale_of(st->v.clip);
    st->v.eps_norm = sqrt(tot[5]);
    st->v.ghat_sqnorm = tot[6];
    st->v.flags = nonfinite ? 1u : 0u;
    *lcg_state = apply(lcg_jump_map(f.advance), *lcg_state);
  }
}

// K3.  NHWC g [N*HW][C] (C % 4 == 0) or FLAT (row-major order = draw order).
// gridDim.x*blockDim.x*4 is a multiple of C so each thread keeps its channel quad.
// Two float4 fetches stay in flight ahead of the one being quantised; the
// dequantised values come from a per-block table (no conversions on the XU pipe
// except double(g)).
template <class Src, bool FLAT, bool DC_SUMS, bool FUSED>
__global__ void __launch_bounds__(RED_THREADS, 2) k_quant_grad(Src src, uint32_t numel, uint32_t C,
                                                            uint32_t HW, uint32_t draw_offset, Affine step_iter,
                                                            Affine step_elem, Affine step_wrap, uint32_t dpix,
                                                            const float* clip_override, DsgcState* st,
                                                            uint32_t* lcg_state, int8_t* __restrict__ q,
                                                            double* partials, double* totals, unsigned* ticket, QgFin fin,
                                                            int* err) {
  __shared__ double tab[256];
  float clip = clip_override ? *clip_override : st->v.clip;
  if (!(clip > 0.0f)) clip = 1.0f;  // only with an all-zero g (q == 0 either way)
  const float s = scale_of(clip), inv_s = 1.0f / s;
  build_dequant_table(tab, s);
  __syncthreads();
  const double* tab0 = tab + 127;  // tab0[q], q in [-127, 127]
  const uint32_t X0 = *lcg_state;
  const uint32_t T4 = gridDim.x * blockDim.x * 4u;
  uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) * 4u;
  double a2 = 0.0, a3 = 0.0, a4 = 0.0, a5 = 0.0, a6 = 0.0;
  bool bad = false;
  float m = 0.0f;
  if (e < numel) {
    uint32_t X, hw = 0;
    if (FLAT) {
      X = apply(lcg_jump_map(static_cast<uint64_t>(e) + draw_offset + 1u), X0);
      src.init(0u);
    } else {
      const uint32_t pix = e / C, c = e - pix * C;
      const uint32_t n = pix / HW;
      hw = pix - n * HW;
      X = apply(lcg_jump_map(static_cast<uint64_t>((n * C + c) * HW + hw) + draw_offset + 1u), X0);
      src.init(c);
    }
    typename Src::Raw r0 = src.fetch(e / 4), r1 = r0;
    uint32_t e1 = e + T4;
    if (e1 < numel) r1 = src.fetch(e1 / 4);
    while (true) {
      const uint32_t e2 = e1 + T4;  // < 2^31 + 2*T4: no wrap
      typename Src::Raw r2 = r1;
      if (e2 < numel) r2 = src.fetch(e2 / 4);
      // fast path for the float4 (branch-free); any element within 2^-13 of a
      // rounding boundary (or with a float-subnormal BN x_hat) redoes the
      // float4 with the exact functions
      bool slow = false;
      const float4 v4 = src.value_fast(r0, slow);
      float vv[4] = {v4.x, v4.y, v4.z, v4.w};
      uint32_t Xs[4];
      Xs[0] = X;
#pragma unroll
      for (int j = 1; j < 4; ++j) Xs[j] = apply(step_elem, Xs[j - 1]);
      int qs[4], qn[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float t = __fmul_rn(fminf(fmaxf(vv[j], -clip), clip), inv_s);
        qs[j] = qs_fast(t, Xs[j], slow);
        if (DC_SUMS) qn[j] = qn_fast(t, slow);
      }
      if (slow) {
        const float4 w4 = src.value(r0);
        vv[0] = w4.x; vv[1] = w4.y; vv[2] = w4.z; vv[3] = w4.w;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          qs[j] = quant_stoch(vv[j], clip, s, inv_s, Xs[j]);
          if (DC_SUMS) qn[j] = quant_nearest(vv[j], clip, s, inv_s);
        }
      }
      signed char qq[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float v = vv[j];
        bad |= !isfinite(v);
        m = fmaxf(m, fabsf(v));
        qq[j] = static_cast<signed char>(qs[j]);
        const double vd = v, gsd = tab0[qs[j]];
        const double d = vd - gsd;
        a5 = fma(d, d, a5);
        a6 = fma(gsd, gsd, a6);
        if (DC_SUMS) {
          const double gn = tab0[qn[j]];
          a2 = fma(vd, vd, a2);
          a3 = fma(vd, gn, a3);
          a4 = fma(gn, gn, a4);
        }
      }
      reinterpret_cast<char4*>(q)[e / 4] = make_char4(qq[0], qq[1], qq[2], qq[3]);
      if (e1 >= numel) break;
      e = e1;
      e1 = e2;
      r0 = r1;
      r1 = r2;
      X = apply(step_iter, X);
      if (!FLAT) {
        hw += dpix;
        while (hw >= HW) {
          hw -= HW;
          X = apply(step_wrap, X);
        }
      }
    }
  }
  double acc[QG_NV] = {m, bad ? 1.0 : 0.0, a2, a3, a4, a5, a6, 0.0};
  if (grid_reduce<QG_NV>(acc, 1u, partials, totals, ticket) && FUSED && threadIdx.x == 0)
    fin_quant_grad(st, totals, fin, lcg_state, err);
}

static __global__ void k_fin_quant_grad(DsgcState* st, const double* totals, QgFin fin, uint32_t* lcg_state, int* err) {
  if (threadIdx.x == 0) fin_quant_grad(st, totals, fin, lcg_state, err);
}

inline int nblocks(int64_t n, int64_t multiple = 1, int64_t cap = 592) {
  int64_t b = (n + RED_THREADS * 8 - 1) / (RED_THREADS * 8);
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  b = (b + multiple - 1) / multiple * multiple;
  return static_cast<int>(b);
}

inline int gcd_i(int64_t a, int64_t b) { return b == 0 ? static_cast<int>(a) : gcd_i(b, a % b); }

// Global totals for data parallelism: totals[0] MAX, totals[1..nv) SUM.
// One collective per phase: op 2 = MAX on element 0, SUM on the rest.
inline int allreduce_totals(Ctx* c, int nv) {
  if (!c->allreduce) return I8T_OK;
  return ctx_allreduce(c, c->d_totals, nv, 2);
}

// K3 launcher over any input source.
template <class Src>
int launch_quant_grad_src(Ctx* c, DsgcState* st, const float* clip_override, Src src, int64_t n_img,
                                 int64_t C, int64_t HW, bool dc_sums, uint32_t* lcg, int8_t* q, QgFin fin) {
  const int64_t numel = n_img * C * HW;
  const bool flat = (C == 1);
  if (numel % 4 != 0 || (!flat && C % 4 != 0))
    return set_error(I8T_EUNSUPPORTED, "quantize_gradient: needs C % 4 == 0 (or flat) and numel % 4 == 0");
  if (numel >= (int64_t(1) << 31)) return set_error(I8T_EUNSUPPORTED, "quantize_gradient: tensor >= 2^31 elements");
  // grid: threads*4 must be a multiple of C (each thread keeps its channel quad)
  const int64_t mult = flat ? 1 : C / gcd_i(C, RED_THREADS * 4);
  int nb = nblocks(numel, mult, 2 * 148);  // one resident wave (__launch_bounds__(256, 2))
  double* p = ensure_partials(c, static_cast<size_t>(nb) * QG_NV);
  if (!p) return set_error(I8T_ECUDA, "partials alloc failed");
  const uint32_t T4 = static_cast<uint32_t>(nb) * RED_THREADS * 4u;
  const uint32_t draw_offset = static_cast<uint32_t>(static_cast<uint64_t>(c->rank) * static_cast<uint64_t>(numel));
  Affine step_iter, step_elem, step_wrap{1u, 0u};
  uint32_t dpix = 0;
  if (flat) {
    step_iter = lcg_jump_map(T4);
    step_elem = lcg_jump_map(1);
  } else {
    dpix = T4 / static_cast<uint32_t>(C);
    step_iter = lcg_jump_map(dpix);
    step_elem = lcg_jump_map(static_cast<uint64_t>(HW));
    step_wrap = lcg_jump_map(static_cast<uint64_t>(C - 1) * static_cast<uint64_t>(HW));
  }
  fin.advance = static_cast<uint32_t>(static_cast<uint64_t>(c->world) * static_cast<uint64_t>(numel));
  const bool fused = (c->allreduce == nullptr);
  const uint32_t un = static_cast<uint32_t>(numel), uc = static_cast<uint32_t>(flat ? 1 : C),
                 uhw = static_cast<uint32_t>(flat ? numel : HW);
#define LAUNCH(F, D, U)                                                                                               \
  k_quant_grad<Src, F, D, U><<<nb, RED_THREADS, 0, c->stream>>>(src, un, uc, uhw, draw_offset, step_iter,          \
                                                                step_elem,                                      \
                                                           step_wrap, dpix, clip_override, st, lcg, q, p,           \
                                                           c->d_totals, c->d_ticket, fin, c->d_err)
  if (flat) {
    if (dc_sums) { if (fused) LAUNCH(true, true, true); else LAUNCH(true, true, false); }
    else { if (fused) LAUNCH(true, false, true); else LAUNCH(true, false, false); }
  } else {
    if (dc_sums) { if (fused) LAUNCH(false, true, true); else LAUNCH(false, true, false); }
    else { if (fused) LAUNCH(false, false, true); else LAUNCH(false, false, false); }
  }
#undef LAUNCH
  count_launch(1);
  int rc = cuda_check("k_quant_grad");
  if (rc || fused) return rc;
  if ((rc = allreduce_totals(c, QG_NV))) return rc;
  k_fin_quant_grad<<<1, 32, 0, c->stream>>>(st, c->d_totals, fin, lcg, c->d_err);
  count_launch(1);
  return cuda_check("k_fin_quant_grad");
}

}  // namespace i8t_dev
