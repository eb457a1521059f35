// bnfuse.cu -- BatchNorm2d (layers.cpp:230-323) + ReLU fused around the INT8
// convolutions so the FP32 activation / gradient between two convs is read
// the minimum number of times:
//   forward   z --(column stats)--> mean, invstd
//             z --(BN-apply + ReLU + nearest quantise + amax)--> int8 input of the next conv
//             z --(BN-apply [+ residual] + ReLU)--> fp32 block output (only where it is reused)
//   backward  g, z --(column sums, ReLU mask recomputed from z)--> dgamma, dbeta, coefficients
//             g, z --(BN-backward apply -> K3 stochastic quantiser + DSGC sums)--> int8 gradient
// Numerics follow the reference BN: double statistics, biased variance,
// x_hat = float((z-mean)*invstd), y = float(gamma*x_hat_d + beta),
// g_in = float(gamma*invstd * (g - s1/m - x_hat*(s2/m))).
// Tensors are NHWC [m][c] fp32 with c % 4 == 0.  bn: device doubles [5c] =
// mean, invstd, s1/m, s2/m, gamma*invstd.
#include <cuda_runtime.h>

#include <cstdlib>

#include <cmath>

#include "internal.cuh"
#include "qcore.cuh"
#include "qgrad.cuh"
#include "bncore.cuh"

#ifndef I8T_BNQ_BLOCKS
#define I8T_BNQ_BLOCKS 3
#endif
namespace i8t_dev {

// resident blocks per SM of k_bn_act_quant: its grid is one such wave
constexpr int BNQ_BLOCKS = I8T_BNQ_BLOCKS;

constexpr int BN_GROUP = 128;  // channels per column-reduction block group

// mask mode 3: the 4 mask bits of elements e..e+3 (e % 4 == 0) of a packed
// ReLU mask (word e/32, bit e%32), as written by i8t_bn_act_q
__device__ __forceinline__ uint32_t mask_nibble(const float* mask, uint64_t e) {
  return (__ldg(reinterpret_cast<const uint32_t*>(mask) + (e >> 5)) >> (e & 31u)) & 0xFu;
}

struct ColArgs {
  const float* z;
  const float* g;       // MODE 1
  const float* mask_y;  // MODE 1, mask 2
  const float* gamma;
  const float* beta;
  double* bn;
  uint32_t m, c;
  int mask_mode;        // 0 none, 1 relu(bn(z)) > 0, 2 mask_y > 0, 3 packed mask bits (mask_y = uint32 words)
  double momentum, eps;
  float* running_mean;  // MODE 0
  float* running_var;
  float* grad_gamma;    // MODE 1
  float* grad_beta;
  // MODE 2 (MODE 1 after an identity-shortcut join): g_out = ja + g * jbit is
  // materialised into gout (k_add_masked_bits, bit for bit) and reduced as g
  const float* ja;
  const uint32_t* jbits;
  float* gout;
  // MODE 3 (MODE 2 + a second BN on the same masked g: the projection block's
  // shortcut BN beside the main branch's last BN): z2 / bn2 / gamma2, sums
  // sum g_m * x_hat2 into grad_gamma2; grad_beta2 = grad_beta
  const float* z2;
  double* bn2;
  const float* gamma2;
  float* grad_gamma2;
  float* grad_beta2;
};

// Column sums over the m rows for one 128-channel group per blockIdx.y.
// MODE 0: sum z, sum z^2.  MODE 1: sum g_m, sum g_m * x_hat (g_m = masked g).
// MODE 2: MODE 1 on g = ja + g * jbit, which is also written to gout (the
// residual join of the next block's backward and this BN's reduction in one
// pass: g is read once instead of written, then read).
template <int MODE, int MASK = 0>
__global__ void __launch_bounds__(256, 2) k_bn_colsum(const ColArgs a, double* partials, unsigned* tickets,
                                                   unsigned* set_tickets) {
  pdl_entry();
  const uint32_t c0 = blockIdx.y * BN_GROUP;
  const uint32_t gw = min(static_cast<uint32_t>(BN_GROUP), a.c - c0);  // group width (multiple of 4)
  const uint32_t lpr = gw / 4;                                         // lanes per row
  const uint32_t rpw = 32 / lpr;                                       // rows per warp per step
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool active = lane < rpw * lpr;
  const uint32_t quad = lane % lpr, sub = lane / lpr;
  const uint32_t ch = c0 + quad * 4;
  constexpr int NS = MODE == 3 ? 3 : 2;  // column sums per channel
  double acc0[4] = {0, 0, 0, 0}, acc1[4] = {0, 0, 0, 0}, acc2[4] = {0, 0, 0, 0};
  double mean[4] = {0, 0, 0, 0}, invstd[4] = {0, 0, 0, 0}, mean2[4] = {0, 0, 0, 0}, invstd2[4] = {0, 0, 0, 0};
  float lo[4] = {0, 0, 0, 0}, hi[4] = {0, 0, 0, 0};
  if (MODE >= 1 && MASK == 1) {
    // ReLU-mask bounds of this block's channel group, bisected in the prologue
    // (redundantly per block: cheaper than a launch); block x == 0 stores them
    // in bn[5c..6c) for the gradient quantiser.
    __shared__ float2 sbound[BN_GROUP];
    if (threadIdx.x < gw) {
      const uint32_t cc = c0 + threadIdx.x;
      const float2 b = bn_mask_bounds(a.bn[cc], a.bn[a.c + cc], a.gamma[cc], a.beta[cc]);
      sbound[threadIdx.x] = b;
      if (blockIdx.x == 0) reinterpret_cast<float2*>(a.bn + 5 * a.c)[cc] = b;
    }
    __syncthreads();
    if (active) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        lo[j] = sbound[quad * 4 + j].x;
        hi[j] = sbound[quad * 4 + j].y;
      }
    }
  }
  if (MODE >= 1 && active) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mean[j] = a.bn[ch + j];
      invstd[j] = a.bn[a.c + ch + j];
      if (MODE == 3) {
        mean2[j] = a.bn2[ch + j];
        invstd2[j] = a.bn2[a.c + ch + j];
      }
    }
  }
  if (active) {
    // U rows per thread per trip: all loads of a trip are issued before any math
    constexpr int U = MODE == 0 ? 10 : MODE == 1 ? 4 : 2;
    constexpr int U2 = MODE == 3 ? U : 1;  // second z (MODE 3)
    const uint32_t row_step = gridDim.x * 8 * rpw;
    uint32_t r = (blockIdx.x * 8 + warp) * rpw + sub;
    // software pipeline: the U rows of the next trip are loaded before the
    // current trip's math, so U (x tensors) 16-byte loads are always in flight
    float4 zv[U], gv[U], yv[U], zn[U], gn[U], yn[U];
    uint32_t bv[U], bn_[U];  // MASK 3: raw mask words (the nibble is extracted at use: keeps the loads in flight)
    uint32_t jv[U], jn[U];   // MODE 2: join mask words (yv / yn carry the join addend)
    float4 z2v[U2], z2n[U2];
    auto fetch = [&](uint32_t rr, float4* zd, float4* gd, float4* yd, uint32_t* bd, uint32_t* jd, float4* z2d) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t ru = rr + u * row_step;
        const size_t off = static_cast<size_t>(ru < a.m ? ru : r) * a.c + ch;
        zd[u] = ldg_stream(a.z + off);
        if (MODE >= 1) gd[u] = ldg_stream(a.g + off);
        if (MODE == 1 && MASK == 2) yd[u] = ldg_stream(a.mask_y + off);
        if (MODE >= 2) yd[u] = ldg_stream(a.ja + off);
        if (MODE >= 2) jd[u] = __ldg(a.jbits + (off >> 5));
        if (MODE == 3) z2d[u] = ldg_stream(a.z2 + off);
        if (MODE >= 1 && MASK == 3) bd[u] = __ldg(reinterpret_cast<const uint32_t*>(a.mask_y) + (off >> 5));
      }
    };
    if (r < a.m) fetch(r, zv, gv, yv, bv, jv, z2v);
    for (; r < a.m; r += U * row_step) {
      const uint32_t rn = r + U * row_step;
      if (rn < a.m) fetch(rn, zn, gn, yn, bn_, jn, z2n);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool valid = r + u * row_step < a.m;  // rows past the end re-read row r: not accumulated
        const float zz[4] = {zv[u].x, zv[u].y, zv[u].z, zv[u].w};
        if (MODE == 0) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const double zd = valid ? static_cast<double>(zz[j]) : 0.0;
            acc0[j] += zd;
            acc1[j] = fma(zd, zd, acc1[j]);
          }
        } else {
          float gg[4] = {gv[u].x, gv[u].y, gv[u].z, gv[u].w};
          const float yy[4] = {yv[u].x, yv[u].y, yv[u].z, yv[u].w};
          if (MODE >= 2) {  // the join, exactly as k_add_masked_bits
            const uint32_t row = r + u * row_step;
            const uint32_t jb = jv[u] >> ((row * a.c + ch) & 31u);
#pragma unroll
            for (int j = 0; j < 4; ++j) gg[j] = __fadd_rn(yy[j], ((jb >> j) & 1u) ? gg[j] : 0.0f);
            if (valid)
              *reinterpret_cast<float4*>(a.gout + static_cast<size_t>(row) * a.c + ch) = make_float4(gg[0], gg[1], gg[2], gg[3]);
          }
          double xh[4], gm[4], xh2[4];
          // MASK 3: this row's nibble (ch % 4 == 0, so the 4 bits share a word)
          const uint32_t w = (MASK == 3 && valid) ? bv[u] >> (((r + u * row_step) * a.c + ch) & 31u) : 0u;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const double xv = (static_cast<double>(zz[j]) - mean[j]) * invstd[j];
            bool mk = valid;
            if (MASK == 1) mk = mk && zz[j] >= lo[j] && zz[j] <= hi[j];
            else if (MODE == 1 && MASK == 2) mk = mk && yy[j] > 0.0f;
            else if (MASK == 3) mk = (w >> j) & 1u;
            float gmf;  // masked g as a float select, converted once
            asm("{.reg .pred p; setp.ne.u32 p, %1, 0; selp.f32 %0, %2, 0f00000000, p;}"
                : "=f"(gmf) : "r"(mk ? 1u : 0u), "f"(gg[j]));
            gm[j] = static_cast<double>(gmf);
            xh[j] = rn24(xv);  // x_hat as in BnBwdSrc::elem
            if (MODE == 3) {
              const float z2 = j == 0 ? z2v[u].x : j == 1 ? z2v[u].y : j == 2 ? z2v[u].z : z2v[u].w;
              xh2[j] = rn24((static_cast<double>(z2) - mean2[j]) * invstd2[j]);
            }
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc0[j] += gm[j];
            acc1[j] = fma(gm[j], xh[j], acc1[j]);
            if (MODE == 3) acc2[j] = fma(gm[j], xh2[j], acc2[j]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        zv[u] = zn[u];
        if (MODE >= 1) gv[u] = gn[u];
        if ((MODE == 1 && MASK == 2) || MODE >= 2) yv[u] = yn[u];
        if (MODE >= 2) jv[u] = jn[u];
        if (MODE == 3) z2v[u] = z2n[u];
        if (MODE >= 1 && MASK == 3) bv[u] = bn_[u];
      }
    }
  }
  // block reduction in a fixed order: warps, then sub-rows
  __shared__ double red[8][32][4 * NS];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    red[warp][lane][j] = acc0[j];
    red[warp][lane][4 + j] = acc1[j];
    if (NS == 3) red[warp][lane][8 + j] = acc2[j];
  }
  __syncthreads();
  if (threadIdx.x < gw) {
    const uint32_t q = threadIdx.x / 4, j = threadIdx.x % 4;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int w = 0; w < 8; ++w)
      for (uint32_t sr = 0; sr < rpw; ++sr) {
        s0 += red[w][sr * lpr + q][j];
        s1 += red[w][sr * lpr + q][4 + j];
        if (NS == 3) s2 += red[w][sr * lpr + q][8 + j];
      }
    double* p = partials + (static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) * (NS * BN_GROUP);
    p[threadIdx.x] = s0;
    p[BN_GROUP + threadIdx.x] = s1;
    if (NS == 3) p[2 * BN_GROUP + threadIdx.x] = s2;
  }
  // two-level fixed-order reduction of the per-block partials: the last block
  // of each set of COL_SET blocks folds its set (in block order), the last set
  // finisher folds the set sums (in set order) -- a single finisher reading
  // every partial was the fixed cost of the small layers' launches
  constexpr uint32_t COL_SET = 16;
  const uint32_t gx = gridDim.x, set = blockIdx.x / COL_SET, nsets = (gx + COL_SET - 1) / COL_SET;
  const uint32_t set_lo = set * COL_SET, set_n = min(COL_SET, gx - set_lo);
  double* const level2 = partials + static_cast<size_t>(gridDim.y) * gx * (NS * BN_GROUP);
  __threadfence();
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) last = atomicAdd(&set_tickets[blockIdx.y * 32 + set], 1u) == set_n - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (uint32_t t = threadIdx.x; t < NS * gw; t += blockDim.x) {  // thread t: column t % gw, sum t / gw
    const uint32_t col = t % gw, which = t / gw;
    const double* base = partials + (static_cast<size_t>(blockIdx.y) * gx + set_lo) * (NS * BN_GROUP) +
                         which * BN_GROUP + col;
    double v[COL_SET];
#pragma unroll
    for (uint32_t k = 0; k < COL_SET; ++k) v[k] = k < set_n ? __ldcg(base + static_cast<size_t>(k) * (NS * BN_GROUP)) : 0.0;
    double sum = 0.0;
#pragma unroll
    for (uint32_t k = 0; k < COL_SET; ++k) sum += v[k];
    level2[(static_cast<size_t>(blockIdx.y) * nsets + set) * (NS * BN_GROUP) + which * BN_GROUP + col] = sum;
  }
  if (threadIdx.x == 0) set_tickets[blockIdx.y * 32 + set] = 0u;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&tickets[blockIdx.y], 1u) == nsets - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double fold[NS][BN_GROUP];
  for (uint32_t tt = threadIdx.x; tt < NS * gw; tt += blockDim.x) {
    const uint32_t col = tt % gw, which = tt / gw;
    const double* base = level2 + static_cast<size_t>(blockIdx.y) * nsets * (NS * BN_GROUP) + which * BN_GROUP + col;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};  // 4 chains, combined in a fixed order
    uint32_t k = 0;
    for (; k + 3 < nsets; k += 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] += __ldcg(base + static_cast<size_t>(k + j) * (NS * BN_GROUP));
    }
    for (int j = 0; k < nsets; ++k, ++j) acc[j] += __ldcg(base + static_cast<size_t>(k) * (NS * BN_GROUP));
    fold[which][col] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
  }
  __syncthreads();
  if (threadIdx.x < gw) {
    double s0 = fold[0][threadIdx.x];
    double s1 = fold[1][threadIdx.x];
    const uint32_t cc = c0 + threadIdx.x;
    const double m = static_cast<double>(a.m);
    if (MODE == 0) {  // layers.cpp:260-268
      const double mean_c = s0 / m;
      const double var = fmax(s1 / m - mean_c * mean_c, 0.0);
      const double inv = 1.0 / sqrt(var + a.eps);
      a.bn[cc] = mean_c;
      a.bn[a.c + cc] = inv;
      if (a.running_mean) {
        a.running_mean[cc] = static_cast<float>((1.0 - a.momentum) * a.running_mean[cc] + a.momentum * mean_c);
        a.running_var[cc] = static_cast<float>((1.0 - a.momentum) * a.running_var[cc] + a.momentum * var);
      }
    } else {  // layers.cpp:285-300
      a.grad_beta[cc] = static_cast<float>(s0);
      a.grad_gamma[cc] = static_cast<float>(s1);
      const double k = static_cast<double>(a.gamma[cc]) * a.bn[a.c + cc];
      a.bn[2 * a.c + cc] = k * (s0 / m);
      a.bn[3 * a.c + cc] = k * (s1 / m);
      a.bn[4 * a.c + cc] = k;
      if (MODE == 3) {  // the second BN on the same masked g
        const double s2 = fold[NS - 1][threadIdx.x];
        a.grad_beta2[cc] = static_cast<float>(s0);
        a.grad_gamma2[cc] = static_cast<float>(s2);
        const double k2 = static_cast<double>(a.gamma2[cc]) * a.bn2[a.c + cc];
        a.bn2[2 * a.c + cc] = k2 * (s0 / m);
        a.bn2[3 * a.c + cc] = k2 * (s2 / m);
        a.bn2[4 * a.c + cc] = k2;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) tickets[blockIdx.y] = 0u;
}

// Forward: q = quantize_nearest(act(bn(z))), running max|act| (layers.cpp:101, 108-109).
__global__ void __launch_bounds__(256, BNQ_BLOCKS) k_bn_act_quant(const float* __restrict__ z, uint32_t n, uint32_t c,
                                                      const double* bn, const float* gamma, const float* beta, int relu,
                                                      const float* clip_p, int8_t* __restrict__ q, float* amax,
                                                      int* err) {
  pdl_entry();
  const float clip = *clip_p, s = scale_of(clip), inv_s = 1.0f / s, hs = __fdiv_rn(0.5f, clip);
  const uint32_t T4 = gridDim.x * blockDim.x * 4u;
  uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) * 4u;
  float m = 0.0f;
  bool bad = false;
  if (e < n) {
    BnQuad k;
    k.load(bn, gamma, beta, c, e % c);
    // software pipeline: the next trip's two float4 are in flight while this
    // trip's two are converted (four 16-byte loads outstanding per thread)
    float4 n0 = __ldg(reinterpret_cast<const float4*>(z + e)), n1 = n0;
    if (e + T4 < n) n1 = __ldg(reinterpret_cast<const float4*>(z + e + T4));
    for (; e < n; e += 2 * T4) {
      const bool two = e + T4 < n;
      const float4 v0 = n0, v1 = n1;
      if (e + 2 * T4 < n) n0 = __ldg(reinterpret_cast<const float4*>(z + e + 2 * T4));
      if (e + 3 * T4 < n) n1 = __ldg(reinterpret_cast<const float4*>(z + e + 3 * T4));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h && !two) break;
        const float4 v = h ? v1 : v0;
        const float zz[4] = {v.x, v.y, v.z, v.w};
        signed char qq[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float y = k.y(j, zz[j]);
          if (relu) y = y > 0.0f ? y : 0.0f;
          bad |= !isfinite(y);
          m = fmaxf(m, fabsf(y));
          qq[j] = static_cast<signed char>(quant_nearest_fast(y, clip, hs, s, inv_s));
        }
        reinterpret_cast<char4*>(q)[(e + h * T4) / 4] = make_char4(qq[0], qq[1], qq[2], qq[3]);
      }
    }
  }
  pdl_trigger();
  if (bad) atomicOr(err, ERR_NONFINITE);
  if (amax) {
    __shared__ float sm[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < 8; ++w) m = fmaxf(m, sm[w]);
      if (m > 0.0f) atomicMax(reinterpret_cast<int*>(amax), __float_as_int(m));
    }
  }
}

// Forward: y = act(bn(z) [+ residual]); residual is fp32 `res` or a second BN
// applied lazily to res_z (ResidualBlock, layers.cpp:451-456: float add, then ReLU).
// Optional extra outputs of the block-output pass (QOUT: any of them set):
//   q     = quantize_nearest(y, clip) with running max|y| -- the next conv's
//           input quantiser (layers.cpp:101, 108-109) on the value just computed;
//   mbits = the ReLU mask y > 0 packed one bit per element (word e/32, bit e%32),
//           all the backward needs of y (mask mode 3).
// The loop is warp-uniform (a warp covers 128 consecutive elements per trip) so
// the 4-bit nibbles of 8 lanes can be OR-ed into a word with shuffles.
template <bool QOUT, int RES>  // RES: 0 none, 1 dense fp32 residual, 2 residual = bn'(res_z) (lazy)
__global__ void __launch_bounds__(256, RES == 2 ? 2 : 3) k_bn_act(const float* __restrict__ z, uint32_t n, uint32_t c, const double* bn,
                                                const float* gamma, const float* beta, int relu,
                                                const float* __restrict__ res, const float* __restrict__ res_z,
                                                const double* res_bn, const float* res_gamma, const float* res_beta,
                                                float* __restrict__ y, const float* clip_p, int8_t* __restrict__ q,
                                                uint32_t* __restrict__ mbits, float* amax, int* err) {
  pdl_entry();
  const uint32_t T4 = gridDim.x * blockDim.x * 4u;  // multiple of 128 and of c
  const uint32_t lane = threadIdx.x & 31;
  uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) * 4u;
  float clip = 1.0f, s = 1.0f, inv_s = 1.0f, hs = 0.5f, m = 0.0f;
  bool bad = false;
  if (QOUT && q) {
    clip = *clip_p;
    s = scale_of(clip);
    inv_s = 1.0f / s;
    hs = __fdiv_rn(0.5f, clip);
  }
  BnQuad k, kr;
  k.load(bn, gamma, beta, c, e % c);
  if (RES == 2) kr.load(res_bn, res_gamma, res_beta, c, e % c);
  // warp-uniform trips of two float4 per thread, software-pipelined: the next
  // trip's loads are issued before this trip's math
  float4 nv[2], nr[2];
  auto fetch = [&](uint32_t eb) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t eh = eb + h * T4;
      const uint32_t ee = eh < n ? eh : 0u;
      nv[h] = __ldg(reinterpret_cast<const float4*>(z + ee));
      nr[h] = RES ? __ldg(reinterpret_cast<const float4*>((RES == 1 ? res : res_z) + ee))
                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  if (e - lane * 4u < n) fetch(e);
  for (; e - lane * 4u < n; e += 2 * T4) {
    float4 v[2] = {nv[0], nv[1]}, r[2] = {nr[0], nr[1]};
    if (e + 2 * T4 - lane * 4u < n) fetch(e + 2 * T4);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t eh = e + h * T4;
      const bool ok = eh < n;
      const float zz[4] = {v[h].x, v[h].y, v[h].z, v[h].w};
      float rr[4] = {r[h].x, r[h].y, r[h].z, r[h].w};
      if (RES == 2) {
#pragma unroll
        for (int j = 0; j < 4; ++j) rr[j] = kr.y(j, rr[j]);
      }
      float o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float t = k.y(j, zz[j]);
        if (RES) t = __fadd_rn(t, rr[j]);
        o[j] = (relu && !(t > 0.0f)) ? 0.0f : t;
      }
      if (ok) reinterpret_cast<float4*>(y)[eh / 4] = make_float4(o[0], o[1], o[2], o[3]);
      if (QOUT && q && ok) {
        signed char qq[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          bad |= !isfinite(o[j]);
          m = fmaxf(m, fabsf(o[j]));
          qq[j] = static_cast<signed char>(quant_nearest_fast(o[j], clip, hs, s, inv_s));
        }
        reinterpret_cast<char4*>(q)[eh / 4] = make_char4(qq[0], qq[1], qq[2], qq[3]);
      }
      if (QOUT && mbits) {  // eh - 4*lane is warp-uniform: all 32 lanes take part in the shuffles
        uint32_t w = ok ? ((o[0] > 0.0f ? 1u : 0u) | (o[1] > 0.0f ? 2u : 0u) | (o[2] > 0.0f ? 4u : 0u) |
                           (o[3] > 0.0f ? 8u : 0u)) << (4 * (lane & 7))
                        : 0u;
        w |= __shfl_xor_sync(0xffffffffu, w, 1);
        w |= __shfl_xor_sync(0xffffffffu, w, 2);
        w |= __shfl_xor_sync(0xffffffffu, w, 4);
        if ((lane & 7) == 0 && ok) mbits[eh / 32] = w;
      }
    }
  }
  pdl_trigger();
  if (QOUT && q) {
    if (bad) atomicOr(err, ERR_NONFINITE);
    if (amax) {
      __shared__ float sm[8];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) m = fmaxf(m, sm[w]);
        if (m > 0.0f) atomicMax(reinterpret_cast<int*>(amax), __float_as_int(m));
      }
    }
  }
}

// Backward value source: g_in = float(k*g_m - (k*s1/m + x_hat*(k*s2/m))) with
// k = gamma*invstd (layers.cpp:309-318 regrouped into two FMAs: the double
// rounding differs from the reference's by ~2^-53 of the largest term, below
// the final float cast), g_m = g masked by the ReLU that followed the BN
// (MASK 1: relu(bn(z)) > 0 recomputed from z; MASK 2: a stored output y > 0;
// MASK 3: packed mask bits; MASK 0: none).
template <int MASK>
struct BnBwdSrc {
  const float* g;
  const float* z;
  const float* mask_y;
  const double* bn;
  const float* gamma;
  const float* beta;
  uint32_t c;
  double mean[4], invstd[4], ka[4], kb[4], k[4];
  float lo[4], hi[4];  // MASK 1: relu(bn(z)) > 0 <=> lo <= z <= hi
  struct Raw {
    float4 g, z, y;
    uint32_t bits, shift;  // MASK 3: the mask word and this float4's bit offset in it
  };
  __device__ __forceinline__ void init(uint32_t c0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mean[j] = bn[c0 + j];
      invstd[j] = bn[c + c0 + j];
      ka[j] = bn[2 * c + c0 + j];
      kb[j] = bn[3 * c + c0 + j];
      k[j] = bn[4 * c + c0 + j];
      if (MASK == 1) {
        const float2 lh = reinterpret_cast<const float2*>(bn + 5 * c)[c0 + j];
        lo[j] = lh.x;
        hi[j] = lh.y;
      }
    }
  }
  __device__ __forceinline__ Raw fetch(uint32_t e4) const {
    Raw r;
    r.g = __ldg(reinterpret_cast<const float4*>(g) + e4);
    r.z = __ldg(reinterpret_cast<const float4*>(z) + e4);
    if (MASK == 2) r.y = __ldg(reinterpret_cast<const float4*>(mask_y) + e4);
    if (MASK == 3) r.bits = __ldg(reinterpret_cast<const uint32_t*>(mask_y) + (e4 >> 3));
    if (MASK == 3) r.shift = (e4 & 7u) * 4u;
    return r;
  }
  // element j; w = the float4's mask bits (MASK 3).  x_hat (here and in the
  // MODE 1 column sums) is rounded to a
  // 24-bit significand in the integer pipe (rn24), i.e. the reference's
  // float(x) without the float-subnormal range: the two differ only for
  // |x_hat| < 2^-126, where the effect on g_in is below 2^-149 * |k s2/m|.
  __device__ __forceinline__ float elem(const Raw& r, int j, uint32_t w) const {
    const float zz = j == 0 ? r.z.x : j == 1 ? r.z.y : j == 2 ? r.z.z : r.z.w;
    const float gg = j == 0 ? r.g.x : j == 1 ? r.g.y : j == 2 ? r.g.z : r.g.w;
    const double xv = (static_cast<double>(zz) - mean[j]) * invstd[j];
    bool mk = true;
    if (MASK == 1) mk = zz >= lo[j] && zz <= hi[j];
    if (MASK == 2) mk = (j == 0 ? r.y.x : j == 1 ? r.y.y : j == 2 ? r.y.z : r.y.w) > 0.0f;
    if (MASK == 3) mk = (w >> j) & 1u;
    float gm;  // the masked g as a float select (the conversion then runs once)
    asm("{.reg .pred p; setp.ne.u32 p, %1, 0; selp.f32 %0, %2, 0f00000000, p;}" : "=f"(gm) : "r"(mk ? 1u : 0u), "f"(gg));
    const double xh = rn24(xv);
    return static_cast<float>(fma(k[j], static_cast<double>(gm), -fma(xh, kb[j], ka[j])));
  }
  __device__ __forceinline__ float4 value(const Raw& r) const {
    const uint32_t w = (MASK == 3) ? (r.bits >> r.shift) : 0u;
    return make_float4(elem(r, 0, w), elem(r, 1, w), elem(r, 2, w), elem(r, 3, w));
  }
  __device__ __forceinline__ float4 value_fast(const Raw& r, bool&) const { return value(r); }
  __device__ __forceinline__ float4 load(uint32_t e4) const { return value(fetch(e4)); }
};

template <int MASK>
__global__ void __launch_bounds__(256) k_bn_bwd_apply(BnBwdSrc<MASK> src, uint32_t n, float* __restrict__ out) {
  pdl_entry();
  const uint32_t T4 = gridDim.x * blockDim.x * 4u;
  uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) * 4u;
  if (e >= n) return;
  src.init(e % src.c);
  for (; e < n; e += T4) reinterpret_cast<float4*>(out)[e / 4] = src.load(e / 4);
}

// The same with the statistics of the first DSGC search pass (clip.cpp:32-34)
// of the value it writes: stats[0] = max|g|, [1] = non-finite count, [2] =
// sum g^2 (fixed-order grid reduction) -- the search then skips that pass.
template <int MASK>
__global__ void __launch_bounds__(256) k_bn_bwd_apply_stats(BnBwdSrc<MASK> src, uint32_t n, float* __restrict__ out,
                                                            double* partials, double* stats, unsigned* ticket) {
  pdl_entry();
  const uint32_t T4 = gridDim.x * blockDim.x * 4u;
  uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) * 4u;
  float m = 0.0f;
  bool bad = false;
  double sq = 0.0;
  if (e < n) {
    src.init(e % src.c);
    for (; e < n; e += T4) {
      const float4 v = src.load(e / 4);
      reinterpret_cast<float4*>(out)[e / 4] = v;
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bad |= !isfinite(vv[j]);
        m = fmaxf(m, fabsf(vv[j]));
        const double d = vv[j];
        sq = fma(d, d, sq);
      }
    }
  }
  double acc[3] = {m, bad ? 1.0 : 0.0, sq};
  grid_reduce<3>(acc, 1u, partials, stats, ticket);
}

// out = a + g * (y > 0): identity-shortcut gradient joined with the main branch.
__global__ void __launch_bounds__(256) k_add_masked(const float* __restrict__ a, const float* __restrict__ g,
                                                    const float* __restrict__ y, uint32_t n4, float* __restrict__ out) {
  pdl_entry();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
    const float4 av = __ldg(reinterpret_cast<const float4*>(a) + i), gv = __ldg(reinterpret_cast<const float4*>(g) + i),
                 yv = __ldg(reinterpret_cast<const float4*>(y) + i);
    float4 o;
    o.x = __fadd_rn(av.x, yv.x > 0.0f ? gv.x : 0.0f);
    o.y = __fadd_rn(av.y, yv.y > 0.0f ? gv.y : 0.0f);
    o.z = __fadd_rn(av.z, yv.z > 0.0f ? gv.z : 0.0f);
    o.w = __fadd_rn(av.w, yv.w > 0.0f ? gv.w : 0.0f);
    reinterpret_cast<float4*>(out)[i] = o;
  }
}

// out = a + g * mask (packed mask bits): the identity-shortcut join of mask mode 3.
__global__ void __launch_bounds__(256) k_add_masked_bits(const float* __restrict__ a, const float* __restrict__ g,
                                                         const float* __restrict__ bits, uint32_t n4,
                                                         float* __restrict__ out) {
  pdl_entry();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
    const float4 av = __ldg(reinterpret_cast<const float4*>(a) + i), gv = __ldg(reinterpret_cast<const float4*>(g) + i);
    const uint32_t b = mask_nibble(bits, 4ull * i);
    float4 o;
    o.x = __fadd_rn(av.x, (b & 1u) ? gv.x : 0.0f);
    o.y = __fadd_rn(av.y, (b & 2u) ? gv.y : 0.0f);
    o.z = __fadd_rn(av.z, (b & 4u) ? gv.z : 0.0f);
    o.w = __fadd_rn(av.w, (b & 8u) ? gv.w : 0.0f);
    reinterpret_cast<float4*>(out)[i] = o;
  }
}

// ---------------------------------------------------------------- host
static int ew_blocks(int64_t n, int64_t c, int64_t cap = 148 * 8) {
  // grid such that blocks*256*4 % c == 0 (fixed channel quad per thread)
  const int64_t mult = c / gcd_i(c, 1024);
  int64_t b = (n / 4 + 255) / 256;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  b = (b + mult - 1) / mult * mult;
  return static_cast<int>(b);
}

template <bool QOUT>
static void launch_bn_act(Ctx* cx, const float* z, int64_t m, int64_t c, const double* bn, const float* gamma,
                          const float* beta, int relu, const float* res, const float* res_z, const double* res_bn,
                          const float* res_gamma, const float* res_beta, float* y, const float* clip, int8_t* q,
                          uint32_t* mbits, float* amax) {
  const uint32_t n = static_cast<uint32_t>(m * c), uc = static_cast<uint32_t>(c);
  // one resident wave (k_bn_act's __launch_bounds__: 2 blocks per SM with a lazy residual BN, else 3)
  const int nb = ew_blocks(m * c, c, 148 * (res_z ? 2 : 3));
  if (res_z)
    launch_k(k_bn_act<QOUT, 2>, nb, 256, 0, cx->stream, z, n, uc, bn, gamma, beta, relu, nullptr, res_z, res_bn, res_gamma,
                                                  res_beta, y, clip, q, mbits, amax, cx->d_err);
  else if (res)
    launch_k(k_bn_act<QOUT, 1>, nb, 256, 0, cx->stream, z, n, uc, bn, gamma, beta, relu, res, nullptr, nullptr, nullptr,
                                                  nullptr, y, clip, q, mbits, amax, cx->d_err);
  else
    launch_k(k_bn_act<QOUT, 0>, nb, 256, 0, cx->stream, z, n, uc, bn, gamma, beta, relu, nullptr, nullptr, nullptr, nullptr,
                                                  nullptr, y, clip, q, mbits, amax, cx->d_err);
}

// per-(group, set) tickets of the two-level column-sum reduction: 64 groups x 32 sets
// (self-resetting; one array per context: the column sums of one stream run in order)
static unsigned* set_tickets(Ctx* c) {
  if (!c->d_set_tickets) {
    if (cudaMalloc(&c->d_set_tickets, 64 * 32 * sizeof(unsigned)) != cudaSuccess) return nullptr;
    cudaMemset(c->d_set_tickets, 0, 64 * 32 * sizeof(unsigned));
  }
  return c->d_set_tickets;
}

unsigned* group_tickets(Ctx* c) {
  if (!c->d_tickets) {
    if (cudaMalloc(&c->d_tickets, 64 * sizeof(unsigned)) != cudaSuccess) return nullptr;
    cudaMemset(c->d_tickets, 0, 64 * sizeof(unsigned));
  }
  return c->d_tickets;
}

static int colsum(Ctx* c, const ColArgs& a, int mode) {
  const int groups = static_cast<int>((a.c + BN_GROUP - 1) / BN_GROUP);
  if (groups > 64) return set_error(I8T_EUNSUPPORTED, "bn: more than 8192 channels");
  // >= 128 rows per block; the grid is one resident wave (2 blocks of ~100
  // registers per SM), two for >= 2048 channels, where a group's rows are few
  // and the trips per warp many (tools/bn_bench.py on B200)
  int bx = static_cast<int>((a.m + 127) / 128);
  const int waves = groups >= 16 ? 4 : 2;
  const int cap = (148 * waves + groups - 1) / groups;
  if (bx > cap) bx = cap;
  if (bx < 1) bx = 1;
  if (bx > 32 * 16) bx = 32 * 16;  // <= 32 sets of 16 blocks per group
  const int nsets = (bx + 15) / 16;
  double* p = ensure_partials(c, static_cast<size_t>(bx + nsets) * groups * 3 * BN_GROUP);
  unsigned* t = group_tickets(c);
  unsigned* st = set_tickets(c);
  if (!p || !t || !st) return set_error(I8T_ECUDA, "bn: scratch alloc failed");
  dim3 grid(static_cast<unsigned>(bx), static_cast<unsigned>(groups));
  if (mode == 0) launch_k(k_bn_colsum<0>, grid, 256, 0, c->stream, a, p, t, st);
  else if (mode == 2) launch_k(k_bn_colsum<2, 3>, grid, 256, 0, c->stream, a, p, t, st);
  else if (mode == 3) launch_k(k_bn_colsum<3, 3>, grid, 256, 0, c->stream, a, p, t, st);
  else if (a.mask_mode == 1) launch_k(k_bn_colsum<1, 1>, grid, 256, 0, c->stream, a, p, t, st);
  else if (a.mask_mode == 2) launch_k(k_bn_colsum<1, 2>, grid, 256, 0, c->stream, a, p, t, st);
  else if (a.mask_mode == 3) launch_k(k_bn_colsum<1, 3>, grid, 256, 0, c->stream, a, p, t, st);
  else launch_k(k_bn_colsum<1, 0>, grid, 256, 0, c->stream, a, p, t, st);
  count_launch(1);
  return cuda_check("k_bn_colsum");
}

static int bn_check(int64_t m, int64_t c, const void* z) {
  if (m < 1 || c < 4 || c % 4 != 0 || !z) return set_error(I8T_EUNSUPPORTED, "bn: needs c % 4 == 0");
  if (m * c >= (int64_t(1) << 31)) return set_error(I8T_EUNSUPPORTED, "bn: tensor >= 2^31 elements");
  if (reinterpret_cast<uintptr_t>(z) & 15u) return set_error(I8T_EUNSUPPORTED, "bn: 16-byte alignment");
  return I8T_OK;
}

}  // namespace i8t_dev

using namespace i8t_dev;
#define CTX(c) reinterpret_cast<Ctx*>(c)

extern "C" {

int i8t_bn_fwd_stats(i8t_ctx* ctx, const float* z, int64_t m, int64_t c, double momentum, double eps, double* bn,
                     float* running_mean, float* running_var) {
  Ctx* cx = CTX(ctx);
  int rc = bn_check(m, c, z);
  if (rc) return rc;
  if (!cx || !bn) return set_error(I8T_EINVAL, "bn_fwd_stats: bad arguments");
  ColArgs a{};
  a.z = z; a.bn = bn; a.m = static_cast<uint32_t>(m); a.c = static_cast<uint32_t>(c);
  a.momentum = momentum; a.eps = eps; a.running_mean = running_mean; a.running_var = running_var;
  return colsum(cx, a, 0);
}

int i8t_bn_act_quant(i8t_ctx* ctx, const float* z, int64_t m, int64_t c, const double* bn, const float* gamma,
                     const float* beta, int relu, const float* clip, int8_t* q, float* amax) {
  Ctx* cx = CTX(ctx);
  int rc = bn_check(m, c, z);
  if (rc) return rc;
  if (!cx || !bn || !gamma || !beta || !clip || !q) return set_error(I8T_EINVAL, "bn_act_quant: bad arguments");
  launch_k(k_bn_act_quant, ew_blocks(m * c, c, 148 * BNQ_BLOCKS), 256, 0, cx->stream, z, static_cast<uint32_t>(m * c), static_cast<uint32_t>(c),
                                                               bn, gamma, beta, relu, clip, q, amax, cx->d_err);
  count_launch(1);
  return cuda_check("k_bn_act_quant");
}

int i8t_bn_act(i8t_ctx* ctx, const float* z, int64_t m, int64_t c, const double* bn, const float* gamma,
               const float* beta, int relu, const float* res, const float* res_z, const double* res_bn,
               const float* res_gamma, const float* res_beta, float* y) {
  Ctx* cx = CTX(ctx);
  int rc = bn_check(m, c, z);
  if (rc) return rc;
  if (!cx || !bn || !gamma || !beta || !y || (res_z && (!res_bn || !res_gamma || !res_beta)))
    return set_error(I8T_EINVAL, "bn_act: bad arguments");
  launch_bn_act<false>(cx, z, m, c, bn, gamma, beta, relu, res, res_z, res_bn, res_gamma, res_beta, y, nullptr,
                       nullptr, nullptr, nullptr);
  count_launch(1);
  return cuda_check("k_bn_act");
}

int i8t_bn_act_q(i8t_ctx* ctx, const float* z, int64_t m, int64_t c, const double* bn, const float* gamma,
                 const float* beta, int relu, const float* res, const float* res_z, const double* res_bn,
                 const float* res_gamma, const float* res_beta, float* y, const float* clip, int8_t* q, float* amax,
                 uint32_t* mask_bits) {
  Ctx* cx = CTX(ctx);
  int rc = bn_check(m, c, z);
  if (rc) return rc;
  if (!cx || !bn || !gamma || !beta || !y || (q && !clip) || (res_z && (!res_bn || !res_gamma || !res_beta)))
    return set_error(I8T_EINVAL, "bn_act_q: bad arguments");
  launch_bn_act<true>(cx, z, m, c, bn, gamma, beta, relu, res, res_z, res_bn, res_gamma, res_beta, y, clip, q,
                      mask_bits, amax);
  count_launch(1);
  return cuda_check("k_bn_act_q");
}

int i8t_bn_bwd_reduce(i8t_ctx* ctx, const float* g, const float* z, int64_t m, int64_t c, double* bn,
                      const float* gamma, const float* beta, int mask_mode, const float* mask_y, float* grad_gamma,
                      float* grad_beta) {
  Ctx* cx = CTX(ctx);
  int rc = bn_check(m, c, z);
  if (rc) return rc;
  if (!cx || !g || !bn || !gamma || !beta || !grad_gamma || !grad_beta || mask_mode < 0 || mask_mode > 3 ||
      (mask_mode >= 2 && !mask_y))
    return set_error(I8T_EINVAL, "bn_bwd_reduce: bad arguments");
  ColArgs a{};
  a.z = z; a.g = g; a.mask_y = mask_y; a.gamma = gamma; a.beta = beta; a.bn = bn;
  a.m = static_cast<uint32_t>(m); a.c = static_cast<uint32_t>(c); a.mask_mode = mask_mode;
  a.grad_gamma = grad_gamma; a.grad_beta = grad_beta;
  // mask_mode 1: the column-sum kernel bisects the ReLU-mask bounds in its
  // prologue and stores them in bn[5c..6c)
  return colsum(cx, a, 1);
}

int i8t_bn_bwd_reduce_join(i8t_ctx* ctx, const float* a_add, const float* g, const uint32_t* join_bits,
                           const float* z, int64_t m, int64_t c, double* bn, const float* gamma, const float* beta,
                           const uint32_t* mask_bits, float* grad_gamma, float* grad_beta, float* g_out) {
  Ctx* cx = CTX(ctx);
  int rc = bn_check(m, c, z);
  if (rc) return rc;
  if (!cx || !a_add || !g || !join_bits || !bn || !gamma || !beta || !mask_bits || !grad_gamma || !grad_beta || !g_out)
    return set_error(I8T_EINVAL, "bn_bwd_reduce_join: bad arguments");
  if ((reinterpret_cast<uintptr_t>(a_add) | reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(g_out)) & 15u)
    return set_error(I8T_EUNSUPPORTED, "bn_bwd_reduce_join: 16-byte alignment");
  ColArgs a{};
  a.z = z; a.g = g; a.mask_y = reinterpret_cast<const float*>(mask_bits); a.gamma = gamma; a.beta = beta; a.bn = bn;
  a.m = static_cast<uint32_t>(m); a.c = static_cast<uint32_t>(c); a.mask_mode = 3;
  a.grad_gamma = grad_gamma; a.grad_beta = grad_beta;
  a.ja = a_add; a.jbits = join_bits; a.gout = g_out;
  return colsum(cx, a, 2);
}

int i8t_bn_bwd_reduce_join2(i8t_ctx* ctx, const float* a_add, const float* g, const uint32_t* join_bits,
                            const float* z, int64_t m, int64_t c, double* bn, const float* gamma, const float* beta,
                            const uint32_t* mask_bits, float* grad_gamma, float* grad_beta, const float* z2,
                            double* bn2, const float* gamma2, float* grad_gamma2, float* grad_beta2, float* g_out) {
  Ctx* cx = CTX(ctx);
  int rc = bn_check(m, c, z);
  if (rc || (rc = bn_check(m, c, z2))) return rc;
  if (!cx || !a_add || !g || !join_bits || !bn || !gamma || !beta || !mask_bits || !grad_gamma || !grad_beta ||
      !g_out || !bn2 || !gamma2 || !grad_gamma2 || !grad_beta2)
    return set_error(I8T_EINVAL, "bn_bwd_reduce_join2: bad arguments");
  if ((reinterpret_cast<uintptr_t>(a_add) | reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(g_out)) & 15u)
    return set_error(I8T_EUNSUPPORTED, "bn_bwd_reduce_join2: 16-byte alignment");
  ColArgs a{};
  a.z = z; a.g = g; a.mask_y = reinterpret_cast<const float*>(mask_bits); a.gamma = gamma; a.beta = beta; a.bn = bn;
  a.m = static_cast<uint32_t>(m); a.c = static_cast<uint32_t>(c); a.mask_mode = 3;
  a.grad_gamma = grad_gamma; a.grad_beta = grad_beta;
  a.ja = a_add; a.jbits = join_bits; a.gout = g_out;
  a.z2 = z2; a.bn2 = bn2; a.gamma2 = gamma2; a.grad_gamma2 = grad_gamma2; a.grad_beta2 = grad_beta2;
  return colsum(cx, a, 3);
}

int i8t_bn_bwd_apply(i8t_ctx* ctx, const float* g, const float* z, int64_t m, int64_t c, const double* bn,
                     const float* gamma, const float* beta, int mask_mode, const float* mask_y, float* gz) {
  Ctx* cx = CTX(ctx);
  int rc = bn_check(m, c, z);
  if (rc) return rc;
  if (!cx || !g || !bn || !gz || mask_mode < 0 || mask_mode > 3 || (mask_mode >= 2 && !mask_y))
    return set_error(I8T_EINVAL, "bn_bwd_apply: bad arguments");
  const uint32_t un = static_cast<uint32_t>(m * c), uc = static_cast<uint32_t>(c);
  const int nb = ew_blocks(m * c, c);
  if (mask_mode == 1) launch_k(k_bn_bwd_apply<1>, nb, 256, 0, cx->stream, BnBwdSrc<1>{g, z, mask_y, bn, gamma, beta, uc}, un, gz);
  else if (mask_mode == 2) launch_k(k_bn_bwd_apply<2>, nb, 256, 0, cx->stream, BnBwdSrc<2>{g, z, mask_y, bn, gamma, beta, uc}, un, gz);
  else if (mask_mode == 3) launch_k(k_bn_bwd_apply<3>, nb, 256, 0, cx->stream, BnBwdSrc<3>{g, z, mask_y, bn, gamma, beta, uc}, un, gz);
  else launch_k(k_bn_bwd_apply<0>, nb, 256, 0, cx->stream, BnBwdSrc<0>{g, z, mask_y, bn, gamma, beta, uc}, un, gz);
  count_launch(1);
  return cuda_check("k_bn_bwd_apply");
}

int i8t_bn_bwd_apply_stats(i8t_ctx* ctx, const float* g, const float* z, int64_t m, int64_t c, const double* bn,
                           const float* gamma, const float* beta, int mask_mode, const float* mask_y, float* gz,
                           double* stats) {
  Ctx* cx = CTX(ctx);
  int rc = bn_check(m, c, z);
  if (rc) return rc;
  if (!cx || !g || !bn || !gz || !stats || mask_mode < 0 || mask_mode > 3 || (mask_mode >= 2 && !mask_y))
    return set_error(I8T_EINVAL, "bn_bwd_apply_stats: bad arguments");
  const uint32_t un = static_cast<uint32_t>(m * c), uc = static_cast<uint32_t>(c);
  const int nb = ew_blocks(m * c, c);
  double* p = ensure_partials(cx, static_cast<size_t>(nb) * 3);
  if (!p) return set_error(I8T_ECUDA, "partials alloc failed");
#define BNS(M) launch_k(k_bn_bwd_apply_stats<M>, nb, 256, 0, cx->stream, BnBwdSrc<M>{g, z, mask_y, bn, gamma, beta, uc}, \
                        un, gz, p, stats, cx->d_ticket)
  if (mask_mode == 1) BNS(1);
  else if (mask_mode == 2) BNS(2);
  else if (mask_mode == 3) BNS(3);
  else BNS(0);
#undef BNS
  count_launch(1);
  return cuda_check("k_bn_bwd_apply_stats");
}

int i8t_quantize_gradient_bn(i8t_ctx* ctx, void* state, const float* g, const float* z, int64_t n_img, int64_t c,
                             int64_t hw, const double* bn, const float* gamma, const float* beta, int mask_mode,
                             const float* mask_y, int lr_scaling_enabled, double alpha, double beta_, int form,
                             uint32_t* lcg_state, int8_t* q) {
  Ctx* cx = CTX(ctx);
  DsgcState* st = reinterpret_cast<DsgcState*>(state);
  int rc = bn_check(n_img * hw, c, z);
  if (rc) return rc;
  if (!cx || !st || !g || !bn || !gamma || !beta || !lcg_state || !q || mask_mode < 0 || mask_mode > 3 ||
      (mask_mode >= 2 && !mask_y))
    return set_error(I8T_EINVAL, "quantize_gradient_bn: bad arguments");
  if (lr_scaling_enabled && (!(alpha > 0.0) || !(beta_ > 0.0 && beta_ <= 1.0)))
    return set_error(I8T_EINVAL, "scale_factor: alpha must be > 0, beta in (0,1]");
  QgFin fin{1 | (lr_scaling_enabled ? 2 : 0), alpha, beta_, form, 0u};
  const uint32_t uc = static_cast<uint32_t>(c);
  if (mask_mode == 1)
    return launch_quant_grad_src(cx, st, nullptr, BnBwdSrc<1>{g, z, mask_y, bn, gamma, beta, uc}, n_img, c, hw, true, lcg_state, q, fin);
  if (mask_mode == 2)
    return launch_quant_grad_src(cx, st, nullptr, BnBwdSrc<2>{g, z, mask_y, bn, gamma, beta, uc}, n_img, c, hw, true, lcg_state, q, fin);
  if (mask_mode == 3)
    return launch_quant_grad_src(cx, st, nullptr, BnBwdSrc<3>{g, z, mask_y, bn, gamma, beta, uc}, n_img, c, hw, true, lcg_state, q, fin);
  return launch_quant_grad_src(cx, st, nullptr, BnBwdSrc<0>{g, z, mask_y, bn, gamma, beta, uc}, n_img, c, hw, true, lcg_state, q, fin);
}

int i8t_add_masked_bits(i8t_ctx* ctx, const float* a, const float* g, const uint32_t* bits, int64_t n, float* out) {
  Ctx* cx = CTX(ctx);
  if (!cx || !a || !g || !bits || !out || n % 4 != 0) return set_error(I8T_EINVAL, "add_masked_bits: bad arguments");
  if (!n) return I8T_OK;
  int b = static_cast<int>((n / 4 + 255) / 256);
  if (b > 148 * 8) b = 148 * 8;
  launch_k(k_add_masked_bits, b, 256, 0, cx->stream, a, g, reinterpret_cast<const float*>(bits), static_cast<uint32_t>(n / 4),
                                                out);
  count_launch(1);
  return cuda_check("k_add_masked_bits");
}

int i8t_add_masked(i8t_ctx* ctx, const float* a, const float* g, const float* y, int64_t n, float* out) {
  Ctx* cx = CTX(ctx);
  if (!cx || !a || !g || !y || !out || n % 4 != 0) return set_error(I8T_EINVAL, "add_masked: bad arguments");
  if (!n) return I8T_OK;
  int b = static_cast<int>((n / 4 + 255) / 256);
  if (b > 148 * 8) b = 148 * 8;
  launch_k(k_add_masked, b, 256, 0, cx->stream, a, g, y, static_cast<uint32_t>(n / 4), out);
  count_launch(1);
  return cuda_check("k_add_masked");
}

}  // extern "C"
