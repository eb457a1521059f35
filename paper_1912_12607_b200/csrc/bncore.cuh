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
