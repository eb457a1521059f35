// bncore.cuh -- per-element BatchNorm2d arithmetic of the reference
// (layers.cpp:262-290) shared by the fused BN kernels and the pooling kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace i8t_dev {

__device__ __forceinline__ float bn_y(double gm, double xv, double bt) { return static_cast<float>(fma(gm, xv, bt)); }
// float(gamma*x_hat + beta) > 0 without the conversion: RN32(d) > 0 <=> d > 2^-150
// (2^-150 itself rounds to +0 under ties-to-even).
__device__ __forceinline__ bool bn_pos(double gm, double xv, double bt) { return fma(gm, xv, bt) > 0x1.0p-150; }

// ReLU mask of BN as a float interval: for x_hat = (double(z) - mean) * invstd
// and f(z) = fma(gamma, x_hat, beta), f(z) > 2^-150 (i.e. float(f) > 0) is
// monotone in z (every step rounds monotonically; invstd > 0), so the set of
// floats z where it holds is an interval [lo, hi] found by bisection over the
// ordered float bit patterns (NaN bounds = empty; NaN z never passes).
__device__ __forceinline__ uint32_t fkey(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}
__device__ inline float2 bn_mask_bounds(double mean, double invstd, double gm, double bt) {
  auto pred = [&](uint32_t key) { return bn_pos(gm, (static_cast<double>(fkey_inv(key)) - mean) * invstd, bt); };
  const float inf = __uint_as_float(0x7F800000u), nan = __uint_as_float(0x7FC00000u);
  const uint32_t klo = fkey(-inf), khi = fkey(inf);
  if (gm == 0.0) {  // f = beta for finite z, NaN for infinite z
    return bt > 0x1.0p-150 ? make_float2(-3.402823466e38f, 3.402823466e38f) : make_float2(nan, nan);
  }
  if (gm > 0.0) {  // pred(+inf) holds: smallest key with pred
    uint32_t a = klo, b = khi;
    while (a < b) {
      const uint32_t m = a + (b - a) / 2;
      if (pred(m)) b = m; else a = m + 1;
    }
    return make_float2(fkey_inv(a), inf);
  }
  uint32_t a = klo, b = khi;  // gm < 0: pred(-inf) holds: largest key with pred
  while (a < b) {
    const uint32_t m = a + (b - a + 1) / 2;
    if (pred(m)) a = m; else b = m - 1;
  }
  return make_float2(-inf, fkey_inv(a));
}

// Per-thread channel-quad coefficients of a BN layer.
struct BnQuad {
  double mean[4], invstd[4], gm[4], bt[4];
  __device__ __forceinline__ void load(const double* bn, const float* gamma, const float* beta, uint32_t c,
                                       uint32_t c0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mean[j] = bn[c0 + j];
      invstd[j] = bn[c + c0 + j];
      gm[j] = gamma[c0 + j];
      bt[j] = beta[c0 + j];
    }
  }
  __device__ __forceinline__ float y(int j, float z) const {
    return bn_y(gm[j], (static_cast<double>(z) - mean[j]) * invstd[j], bt[j]);
  }
};

}  // namespace i8t_dev
