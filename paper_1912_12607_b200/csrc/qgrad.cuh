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
// resident blocks per SM of K3 (register budget 65536 / (256 * QG_BLOCKS))
#ifndef I8T_QG_BLOCKS
#define I8T_QG_BLOCKS 2
#endif
constexpr int QG_BLOCKS = I8T_QG_BLOCKS;

struct QgFin {
  int mode;  // bit0: d_c from the sums (non-search), bit1: lr scaling, bit2: plain quantize (no DSGC state)
  double alpha, beta;
  int form;
  uint32_t advance;  // LCG draws consumed by the whole (global) tensor
};

// Tail of quantize_gradient (layers.cpp:32-58) from global totals.
static __device__ void fin_quant_grad(DsgcState* st, const double* tot, const QgFin& f, uint32_t* lcg_state, int* err) {
  const float m = static_cast<float>(tot[0]);
  const bool nonfinite = tot[1] > 0.0 || !isfinite(tot[5]);
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
__global__ void __launch_bounds__(RED_THREADS, QG_BLOCKS) k_quant_grad(Src src, uint32_t numel, uint32_t C,
                                                            uint32_t HW, uint32_t draw_offset, Affine step_iter,
                                                            Affine step_elem, Affine step_wrap, uint32_t dpix,
                                                            const float* clip_override, DsgcState* st,
                                                            uint32_t* lcg_state, int8_t* __restrict__ q,
                                                            double* partials, double* totals, unsigned* ticket, QgFin fin,
                                                            int* err) {
  pdl_entry();
  __shared__ double tab[256];
  const uint32_t T4 = gridDim.x * blockDim.x * 4u;
  uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) * 4u;
  const bool live = e < numel;
  // the first two data fetches and the per-channel coefficients go out before
  // the chain of dependent scalar loads (clip -> table, LCG state -> jump)
  uint32_t hw = 0, draw0 = 0;
  typename Src::Raw ra{}, rb{}, rc{};
  if (live) {
    if (FLAT) {
      draw0 = e;
      src.init(0u);
    } else {
      const uint32_t pix = e / C, c = e - pix * C;
      const uint32_t n = pix / HW;
      hw = pix - n * HW;
      draw0 = (n * C + c) * HW + hw;
      src.init(c);
    }
    ra = src.fetch(e / 4);
    rb = ra;
    rc = ra;
    if (e + T4 < numel) rb = src.fetch((e + T4) / 4);
  }
  float clip = clip_override ? *clip_override : st->v.clip;
  if (!(clip > 0.0f)) clip = 1.0f;  // only with an all-zero g (q == 0 either way)
  const float s = scale_of(clip), inv_s = 1.0f / s, hs = __fdiv_rn(0.5f, clip);
  const bool tiny = !(s >= 0x1p-126f);  // subnormal scale: every element through the exact functions
  build_dequant_table(tab, s);
  __syncthreads();
  // tab[q + 127] at the bit patterns qs_bits / qn_bits return (32-bit wrap)
  const uint32_t tab_s = static_cast<uint32_t>(__cvta_generic_to_shared(tab)) + 8u * (127u - RMAGIC_BITS);
  const uint32_t tab_n = tab_s - 8u;
  const uint32_t X0 = *lcg_state;
  double a2 = 0.0, a3 = 0.0, a4 = 0.0, a5 = 0.0, a6 = 0.0;
  float m = 0.0f;
  if (live) {
    uint32_t X = apply(lcg_jump_map(static_cast<uint64_t>(draw0) + draw_offset + 1u), X0);
    // one float4: fast path; any element within QK of a rounding boundary (or
    // with a float-subnormal BN x_hat) sends the float4 to the exact functions
    auto process = [&](const typename Src::Raw& r) {
      bool slow = tiny;
      const float4 v4 = src.value_fast(r, slow);
      float vv[4] = {v4.x, v4.y, v4.z, v4.w};
      uint32_t Xs[4];
      Xs[0] = X;
#pragma unroll
      for (int j = 1; j < 4; ++j) Xs[j] = apply(step_elem, Xs[j - 1]);
      uint32_t ks[4], kn[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float t1 = q_t1(vv[j], hs);
        ks[j] = qs_bits(t1, Xs[j], slow);
        if (DC_SUMS) kn[j] = qn_bits(t1, slow);
      }
      if (slow) {  // rare: the float4 again through the exact functions
        const float4 w4 = src.value(r);
        vv[0] = w4.x; vv[1] = w4.y; vv[2] = w4.z; vv[3] = w4.w;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          ks[j] = static_cast<uint32_t>(RMAGIC_BITS + quant_stoch(vv[j], clip, s, inv_s, Xs[j]));
          if (DC_SUMS) kn[j] = static_cast<uint32_t>(RMAGIC_BITS + 1 + quant_nearest(vv[j], clip, s, inv_s));
        }
      }
      m = fmaxf(m, fmaxf(fmaxf(fabsf(vv[0]), fabsf(vv[1])), fmaxf(fabsf(vv[2]), fabsf(vv[3]))));
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double vd = vv[j], gsd = lds_f64(tab_s + 8u * ks[j]);
        const double d = vd - gsd;
        a5 = fma(d, d, a5);
        a6 = fma(gsd, gsd, a6);
        if (DC_SUMS) {
          const double gn = lds_f64(tab_n + 8u * kn[j]);
          a2 = fma(vd, vd, a2);
          a3 = fma(vd, gn, a3);
          a4 = fma(gn, gn, a4);
        }
      }
      reinterpret_cast<uint32_t*>(q)[e / 4] = __byte_perm(__byte_perm(ks[0], ks[1], 0x0040),
                                                          __byte_perm(ks[2], ks[3], 0x0040), 0x5410);
    };
    auto advance = [&]() {
      e += T4;
      X = apply(step_iter, X);  // NHWC: includes the dpix / HW whole image wraps
      if (!FLAT) {
        hw += dpix;  // dpix % HW
        if (hw >= HW) {
          hw -= HW;
          X = apply(step_wrap, X);
        }
      }
    };
    // three-slot ring, two float4 fetches in flight ahead of the one being
    // quantised (the first two issued above); unrolled so the slots never move
    // between registers
    while (true) {  // e + 2*T4 < 2^31 + 2*T4: no wrap
      if (e + 2 * T4 < numel) rc = src.fetch((e + 2 * T4) / 4);
      process(ra);
      if (e + T4 >= numel) break;
      advance();
      if (e + 2 * T4 < numel) ra = src.fetch((e + 2 * T4) / 4);
      process(rb);
      if (e + T4 >= numel) break;
      advance();
      if (e + 2 * T4 < numel) rb = src.fetch((e + 2 * T4) / 4);
      process(rc);
      if (e + T4 >= numel) break;
      advance();
    }
  }
  // non-finite inputs show up as a non-finite sum of squared errors
  // (|v - g_s|^2 summed in double cannot overflow for finite float v)
  double acc[QG_NV] = {m, 0.0, a2, a3, a4, a5, a6, 0.0};
  pdl_trigger();  // only the grid reduction remains: let a dependent conv grid start its prologue
  if (grid_reduce<QG_NV>(acc, 1u, partials, totals, ticket) && FUSED && threadIdx.x == 0)
    fin_quant_grad(st, totals, fin, lcg_state, err);
}

static __global__ void k_fin_quant_grad(DsgcState* st, const double* totals, QgFin fin, uint32_t* lcg_state, int* err) {
  pdl_entry();
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
  if (!ctx_dp(c)) return I8T_OK;
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
  int nb = nblocks(numel, mult, QG_BLOCKS * 148);  // one resident wave (__launch_bounds__(256, QG_BLOCKS))
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
    // a thread steps dpix pixels: q = dpix / HW whole images (each adds
    // (C-1)*HW draws beyond the pixels) folded into step_iter, and at most one
    // more image wrap from the remainder (small-HW layers would otherwise loop)
    const uint32_t dp = T4 / static_cast<uint32_t>(C);
    const uint64_t q = dp / static_cast<uint64_t>(HW);
    dpix = static_cast<uint32_t>(dp - q * static_cast<uint64_t>(HW));
    step_iter = lcg_jump_map(static_cast<uint64_t>(dp) + q * static_cast<uint64_t>(C - 1) * static_cast<uint64_t>(HW));
    step_elem = lcg_jump_map(static_cast<uint64_t>(HW));
    step_wrap = lcg_jump_map(static_cast<uint64_t>(C - 1) * static_cast<uint64_t>(HW));
  }
  fin.advance = static_cast<uint32_t>(static_cast<uint64_t>(c->world) * static_cast<uint64_t>(numel));
  const bool fused = !ctx_dp(c);
  const uint32_t un = static_cast<uint32_t>(numel), uc = static_cast<uint32_t>(flat ? 1 : C),
                 uhw = static_cast<uint32_t>(flat ? numel : HW);
#define LAUNCH(F, D, U)                                                                                  \
  launch_k(k_quant_grad<Src, F, D, U>, nb, RED_THREADS, 0, c->stream, src, un, uc, uhw, draw_offset, step_iter,     \
           step_elem, step_wrap, dpix, clip_override, st, lcg, q, p, c->d_totals, c->d_ticket, fin, c->d_err)
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
  launch_k(k_fin_quant_grad, 1, 32, 0, c->stream, st, c->d_totals, fin, lcg, c->d_err);
  count_launch(1);
  return cuda_check("k_fin_quant_grad");
}

}  // namespace i8t_dev
