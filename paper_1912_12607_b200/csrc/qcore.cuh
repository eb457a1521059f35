// qcore.cuh -- device-side numerics shared by the quantiser and DSGC kernels:
// the exact FP32 restatements of quantize_value (quantize.cpp:16-31), the
// reference's cosine / phi formulas, deterministic block reductions and the
// "last block finishes" grid reduction.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.cuh"

namespace i8t_dev {

// Streaming 16-byte load the compiler keeps in program order (asm volatile):
// loops that issue several of these before using them get the memory-level
// parallelism they ask for instead of loads sunk next to their uses.
__device__ __forceinline__ float4 ldg_stream(const float* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ float scale_of(float clip) { return __fdiv_rn(clip, 127.0f); }

// x + RMAGIC rounds x (|x| < 2^22) to an integer held in the low mantissa bits:
// rint on the FMA pipe, and the integer is __float_as_int(x + RMAGIC) - RMAGIC_BITS.
// (FRND / F2I / I2F run on the quarter-rate XU pipe, which bounded K3 / K4.)
constexpr float RMAGIC = 12582912.0f;  // 1.5 * 2^23
constexpr int RMAGIC_BITS = 0x4B400000;

// quantize_value, kNearest: lround(RN64(v/s)) == round-half-away(v/s) since
// RN64 cannot cross a half-integer for float v, s; the tie
// test a >= s*(k+1/2) is decided exactly by the sign of one FMA.
__device__ __forceinline__ int quant_nearest(float x, float clip, float s, float inv_s) {
  const float v = fminf(fmaxf(x, -clip), clip);
  float a = fabsf(v);
  if (!(s >= 0x1p-126f)) {  // subnormal scale (clip < 127 * FLT_MIN): a and s scaled by 2^64, exactly
    a *= 0x1p64f;
    s *= 0x1p64f;
    inv_s = __frcp_rn(s);
  }
  const float kb = __fadd_rn(__fmul_rn(a, inv_s), RMAGIC);
  const float k = __fsub_rn(kb, RMAGIC);
  int ki = __float_as_int(kb) - RMAGIC_BITS;
  if (__fmaf_rn(-s, k + 0.5f, a) >= 0.0f) ++ki;
  else if (__fmaf_rn(-s, k - 0.5f, a) < 0.0f) --ki;
  ki = min(ki, 127);
  return v < 0.0f ? -ki : ki;
}

// Branch-free fast paths for the hot loops: they take t = float(clamp(v)) * inv_s
// (within 2^-15 of RN64(v/s)) and raise `slow` when the FP32 decision is
// within 2^-13 of a rounding boundary; the caller then redoes the element
// with the exact functions below.
constexpr float QD = 0x1.0p-13f;

// kNearest: round-half-away(t).  t + RMAGIC keeps t's sign in the integer read
// from the mantissa (|t| <= 127.0001 also needs no clamp: it rounds to <= 127);
// ties (|t - rint(t)| = 1/2, where rint goes to even) and near-ties are slow.
__device__ __forceinline__ int qn_fast(float t, bool& slow) {
  const float kb = __fadd_rn(t, RMAGIC);
  const float dn = __fsub_rn(t, __fsub_rn(kb, RMAGIC));  // in [-1/2, 1/2]
  slow |= fabsf(dn) > 0.5f - QD;
  return __float_as_int(kb) - RMAGIC_BITS;
}

// kStochastic: floor(t) + (u < frac(t)) == ceil(t - u) for t = RN64(v/s)
// clamped to +-127, u = X * 2^-32 (u == frac gives floor(t) both ways).  u is
// formed from the top 23 bits without a conversion; ceil(y) lies in
// [-127, 127] whenever the decision is not flagged slow.
__device__ __forceinline__ int qs_fast(float t, uint32_t X, bool& slow) {
  const float u = __fsub_rn(__uint_as_float(0x3F800000u | (X >> 9)), 1.0f);
  const float y = __fsub_rn(t, u);
  const float rb = __fadd_rn(y, RMAGIC);
  const float d = __fsub_rn(y, __fsub_rn(rb, RMAGIC));
  slow |= !(fabsf(d) > QD);
  return (__float_as_int(rb) - RMAGIC_BITS) + (d > 0.0f ? 1 : 0);
}

// Leaner fast path of K3: the decision is within 2^-15 of the exact one
// (3 * 2^-17 from s, 0.5/clip and w, 2^-18 each from t1 and y, 2^-23 from
// the truncated u), so a margin QK = 2^-14 suffices.  Clamp and scale in
// two FMA-pipe ops: w = sat(v * (0.5/clip) + 0.5) (NaN -> 0, like the clamp
// of the exact path), t1 = 254 w - 126 = t + 1 within 2^-15 of RN64(v/s) + 1
// for |v| <= clip and exactly 127 + 1 (-127 + 1) beyond it.  The quantised
// values come back as the float bit patterns of RMAGIC + q (qs) and
// RMAGIC + q + 1 (qn): their low byte is the int8 and they index the dequant
// table directly; callers that take the exact path build the same patterns.
constexpr float QK = 0x1.0p-14f;
__device__ __forceinline__ float q_t1(float v, float hs) {
  return __fmaf_rn(__saturatef(__fmaf_rn(v, hs, 0.5f)), 254.0f, -126.0f);
}
// kStochastic: ceil(t - u) = round(t - u + 1/2) away from the boundaries;
// 1 + u is the float with X's top 23 bits as significand (one funnel shift).
__device__ __forceinline__ uint32_t qs_bits(float t1, uint32_t X, bool& slow) {
  const float uh = __fsub_rn(__uint_as_float(__funnelshift_r(X, 0x7Fu, 9)), 0.5f);  // 1/2 + u, exact
  const float yh = __fsub_rn(t1, uh);                                                // t - u + 1/2
  const float kb = __fadd_rn(yh, RMAGIC);
  slow |= fabsf(__fsub_rn(yh, __fsub_rn(kb, RMAGIC))) > 0.5f - QK;
  return __float_as_uint(kb);
}
// kNearest: round-half-away(t); ties and near-ties are slow.
__device__ __forceinline__ uint32_t qn_bits(float t1, bool& slow) {
  const float kb = __fadd_rn(t1, RMAGIC);
  slow |= fabsf(__fsub_rn(t1, __fsub_rn(kb, RMAGIC))) > 0.5f - QK;
  return __float_as_uint(kb);
}
// quantize_value kNearest through the fast path, the exact function only near
// a rounding tie (hs = 0.5 / clip).
__device__ __forceinline__ int quant_nearest_fast(float v, float clip, float hs, float s, float inv_s) {
  bool slow = !(s >= 0x1p-126f);  // the fast paths assume a normal scale
  const uint32_t kb = qn_bits(q_t1(v, hs), slow);
  if (slow) return quant_nearest(v, clip, s, inv_s);
  return static_cast<int>(kb) - (RMAGIC_BITS + 1);
}
// 8-byte shared load at a 32-bit shared-window address.
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

// quantize_value, kStochastic, exact: the FP32 fast path where it decides,
// else the reference's FP64 formula (quantize.cpp:16-31).
__device__ __forceinline__ int quant_stoch(float x, float clip, float s, float inv_s, uint32_t X) {
  const float v = fminf(fmaxf(x, -clip), clip);
  bool slow = !(s >= 0x1p-126f);
  const int qf = qs_fast(__fmul_rn(v, inv_s), X, slow);
  if (!slow) return qf;
  double td = static_cast<double>(v) / static_cast<double>(s);
  td = fmin(fmax(td, -127.0), 127.0);
  const double fd = floor(td);
  const double fr = td - fd;
  const double ud = static_cast<double>(X) * 0x1.0p-32;
  const int q = static_cast<int>(fd) + (ud < fr ? 1 : 0);
  return max(-127, min(127, q));
}

// x rounded to a 24-bit significand (nearest-even) in the integer pipe: the
// value of double(float(x)) without the two XU conversions for float-normal
// |x| in [2^-126, 2^128); zero, inf and NaN map to themselves.
__device__ __forceinline__ double rn24(double x) {
  long long b = __double_as_longlong(x);
  b += 0x0FFFFFFFLL + ((b >> 29) & 1);
  b &= ~0x1FFFFFFFLL;
  return __longlong_as_double(b);
}

// Dequantised values double(float(q) * s) for q in [-127, 127] (quantize.cpp:81-87),
// built once per block in shared memory: tab[q + 127].
__device__ __forceinline__ void build_dequant_table(double* tab, float s) {
  for (int i = threadIdx.x; i < 255; i += blockDim.x) tab[i] = __fmul_rn(static_cast<float>(i - 127), s);
}

__device__ __forceinline__ uint32_t apply(Affine m, uint32_t x) { return m.a * x + m.c; }

__device__ __forceinline__ double cosine_from(double num, double sq_g, double sq_h) {
  if (sq_g == 0.0 && sq_h == 0.0) return 0.0;
  if (sq_g == 0.0 || sq_h == 0.0) return 1.0;
  return 1.0 - num / (sqrt(sq_g) * sqrt(sq_h));
}

// phi(d_c) (lr_scale.cpp:8-20); argument checks happen on the host.
__device__ __forceinline__ double phi_of(double dc, double alpha, double beta, int form) {
  double raw;
  if (form == 0) raw = exp(-alpha * dc);
  else if (form == 1) raw = 1.0 - dc;
  else if (form == 2) raw = 1.0 - dc * dc;
  else raw = 1.0;
  return fmax(raw, beta);
}

// Block reduce NV doubles (bit j of maxmask: max instead of sum) in a fixed
// order; result valid in thread 0's out[] (and broadcast through smem).
template <int NV>
__device__ __forceinline__ void block_reduce(double (&v)[NV], uint32_t maxmask, double* out_smem) {
  __shared__ double sh[NV][RED_THREADS / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    double x = v[j];
    const bool mx = (maxmask >> j) & 1u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double y = __shfl_xor_sync(0xffffffffu, x, o);
      x = mx ? fmax(x, y) : x + y;
    }
    if (lane == 0) sh[j][wid] = x;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < NV; j += blockDim.x) {
    const bool mx = (maxmask >> j) & 1u;
    double x = sh[j][0];
    for (int w = 1; w < RED_THREADS / 32; ++w) x = mx ? fmax(x, sh[j][w]) : x + sh[j][w];
    out_smem[j] = x;
  }
  __syncthreads();
}

// Grid reduction: every block stores its partial; the last block to arrive
// sums the partials in block order (deterministic) into totals[] and resets
// the ticket.  Returns true in the last block (all threads).
template <int NV>
__device__ __forceinline__ bool grid_reduce(double (&v)[NV], uint32_t maxmask, double* partials, double* totals,
                                            unsigned* ticket) {
  __shared__ double blk[NV];
  __shared__ bool last;
  block_reduce<NV>(v, maxmask, blk);
  if (threadIdx.x < NV) partials[static_cast<size_t>(blockIdx.x) * NV + threadIdx.x] = blk[threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return false;
  __threadfence();
  // Final reduction over the blocks: thread t folds blocks t, t+256, ... (fixed
  // order, independent loads in flight), then the fixed-order block tree.
  double w[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) w[j] = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      const double y = __ldcg(partials + static_cast<size_t>(b) * NV + j);
      w[j] = ((maxmask >> j) & 1u) ? fmax(w[j], y) : w[j] + y;
    }
  }
  __shared__ double fin[NV];
  block_reduce<NV>(w, maxmask, fin);
  for (int j = threadIdx.x; j < NV; j += blockDim.x) totals[j] = fin[j];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) *ticket = 0u;
  return true;
}

}  // namespace i8t_dev
