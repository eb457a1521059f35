// conv_dw.cu -- depthwise INT8 convolutions (conv.cpp:115-131 forward,
// :159-184 backward).  One filter per channel: 9 MACs per output element, so
// these are HBM-bound and stay on CUDA cores (integer IMAD), NHWC so a warp's
// lanes walk consecutive channels (coalesced).  Exact int32/int64 sums, FP64
// rescale epilogue identical to the dense path.
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.cuh"

namespace i8t_dev {

struct DwArgs {
  int N, H, W, C, Cp, R, S, sh, sw, ph, pw, P, Q;
};

__device__ __forceinline__ double dw_rescale(const float* x, const float* y) {
  return static_cast<double>(__fdiv_rn(*x, 127.0f)) * static_cast<double>(__fdiv_rn(*y, 127.0f));
}

// z[n,p,q,c] = sum_{r,s} a[n, p*sh-ph+r, q*sw-pw+s, c] * w[c][r*S+s]
__global__ void __launch_bounds__(256) k_dw_fwd(const DwArgs d, const int8_t* __restrict__ a, const int8_t* __restrict__ w,
                                                const float* clip_a, const float* clip_w, float* z, int32_t* acc) {
  pdl_entry();
  const double rs = dw_rescale(clip_a, clip_w);
  const int64_t tot = static_cast<int64_t>(d.N) * d.P * d.Q * d.C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(i % d.C);
    const int64_t pix = i / d.C;
    const int q = static_cast<int>(pix % d.Q), p = static_cast<int>((pix / d.Q) % d.P), n = static_cast<int>(pix / (static_cast<int64_t>(d.P) * d.Q));
    int32_t s = 0;
    for (int r = 0; r < d.R; ++r) {
      const int ih = p * d.sh - d.ph + r;
      if (ih < 0 || ih >= d.H) continue;
      for (int t = 0; t < d.S; ++t) {
        const int iw = q * d.sw - d.pw + t;
        if (iw < 0 || iw >= d.W) continue;
        s += static_cast<int32_t>(__ldg(a + ((static_cast<int64_t>(n) * d.H + ih) * d.W + iw) * d.Cp + c)) *
             static_cast<int32_t>(__ldg(w + c * d.R * d.S + r * d.S + t));
      }
    }
    if (z) z[i] = static_cast<float>(rs * static_cast<double>(s));
    if (acc) acc[i] = s;
  }
}

// ga[n,h,w,c] = sum_{r,s: (h+ph-r) % sh == 0 ...} g[n,p,q,c] * w[c][r*S+s]
__global__ void __launch_bounds__(256) k_dw_dgrad(const DwArgs d, const int8_t* __restrict__ g, const int8_t* __restrict__ w,
                                                  const float* clip_g, const float* clip_w, float* ga, int32_t* acc) {
  pdl_entry();
  const double rs = dw_rescale(clip_g, clip_w);
  const int64_t tot = static_cast<int64_t>(d.N) * d.H * d.W * d.C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = static_cast<int>(i % d.C);
    const int64_t pix = i / d.C;
    const int x = static_cast<int>(pix % d.W), y = static_cast<int>((pix / d.W) % d.H), n = static_cast<int>(pix / (static_cast<int64_t>(d.H) * d.W));
    int32_t s = 0;
    for (int r = 0; r < d.R; ++r) {
      const int pn = y + d.ph - r;
      if (pn < 0 || pn % d.sh) continue;
      const int p = pn / d.sh;
      if (p >= d.P) continue;
      for (int t = 0; t < d.S; ++t) {
        const int qn = x + d.pw - t;
        if (qn < 0 || qn % d.sw) continue;
        const int q = qn / d.sw;
        if (q >= d.Q) continue;
        s += static_cast<int32_t>(__ldg(g + ((static_cast<int64_t>(n) * d.P + p) * d.Q + q) * d.Cp + c)) *
             static_cast<int32_t>(__ldg(w + c * d.R * d.S + r * d.S + t));
      }
    }
    if (ga) ga[i] = static_cast<float>(rs * static_cast<double>(s));
    if (acc) acc[i] = s;
  }
}

// gw[c][r*S+s] = sum_{n,p,q} g[n,p,q,c] * a[n, p*sh-ph+r, q*sw-pw+s, c]
// Block = 64 channels x 4 pixel-lanes; each thread walks a strided slice of
// the npq range holding up to 49 per-tap int64 sums, then one atomic per tap.
constexpr int DW_MAXTAP = 49;
__global__ void __launch_bounds__(256) k_dw_wgrad(const DwArgs d, const int8_t* __restrict__ g, const int8_t* __restrict__ a,
                                                  unsigned long long* acc, int64_t npq_per_block) {
  pdl_entry();
  const int c = blockIdx.x * 64 + (threadIdx.x & 63);
  const int lane4 = threadIdx.x >> 6;
  if (c >= d.C) return;
  const int RS = d.R * d.S;
  long long sum[DW_MAXTAP];
  for (int t = 0; t < RS; ++t) sum[t] = 0;
  const int64_t npq = static_cast<int64_t>(d.N) * d.P * d.Q;
  const int64_t lo = blockIdx.y * npq_per_block;
  int64_t hi = lo + npq_per_block;
  if (hi > npq) hi = npq;
  for (int64_t e = lo + lane4; e < hi; e += 4) {
    const int32_t gv = __ldg(g + e * d.Cp + c);
    if (gv == 0) continue;
    const int q = static_cast<int>(e % d.Q), p = static_cast<int>((e / d.Q) % d.P), n = static_cast<int>(e / (static_cast<int64_t>(d.P) * d.Q));
    for (int r = 0; r < d.R; ++r) {
      const int ih = p * d.sh - d.ph + r;
      if (ih < 0 || ih >= d.H) continue;
      for (int t = 0; t < d.S; ++t) {
        const int iw = q * d.sw - d.pw + t;
        if (iw < 0 || iw >= d.W) continue;
        sum[r * d.S + t] += gv * static_cast<int32_t>(__ldg(a + ((static_cast<int64_t>(n) * d.H + ih) * d.W + iw) * d.Cp + c));
      }
    }
  }
  for (int t = 0; t < RS; ++t)
    if (sum[t]) atomicAdd(acc + static_cast<int64_t>(c) * RS + t, static_cast<unsigned long long>(sum[t]));
}

__global__ void k_dw_wgrad_finalize(const long long* __restrict__ acc, int64_t n, const float* clip_g, const float* clip_a,
                                    float* gw) {
  pdl_entry();
  const double rs = dw_rescale(clip_g, clip_a);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    gw[i] = static_cast<float>(rs * static_cast<double>(acc[i]));
}

// ------------------------------------------------------------------ channel-quad kernels
// C % 4 == 0, c_pad == C (every MobileNetV2 depthwise layer): a thread owns 4
// consecutive channels (one 32-bit load per tap, a warp reads 128 contiguous
// bytes), the 4 x R*S int8 weights of its quad packed in R*S registers, 32-bit
// index math, R, S and the stride as template constants.  Same integer sums
// (exact) and the same FP64 rescale as the generic kernels above.
__device__ __forceinline__ int sbyte(uint32_t v, int k) { return static_cast<int>(static_cast<int8_t>(v >> (8 * k))); }

template <int R, int S>
__device__ __forceinline__ void dw_load_wq(const int8_t* __restrict__ w, int c0, uint32_t (&wq)[R * S]) {
#pragma unroll
  for (int t = 0; t < R * S; ++t)
    wq[t] = static_cast<uint32_t>(static_cast<uint8_t>(w[(c0 + 0) * R * S + t])) |
            static_cast<uint32_t>(static_cast<uint8_t>(w[(c0 + 1) * R * S + t])) << 8 |
            static_cast<uint32_t>(static_cast<uint8_t>(w[(c0 + 2) * R * S + t])) << 16 |
            static_cast<uint32_t>(static_cast<uint8_t>(w[(c0 + 3) * R * S + t])) << 24;
}

// 3x3 taps with DP4A: the four channels' weights of taps 0-3 and 4-7 transposed
// into per-channel words (byte t = tap), tap 8 kept per channel.
struct DwW9 {
  uint32_t t03[4], t47[4];
  int t8[4];
};
__device__ __forceinline__ void transpose4x4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&c)[4]);
__device__ __forceinline__ DwW9 dw_w9(const uint32_t (&wq)[9]) {
  DwW9 r;
  transpose4x4(wq[0], wq[1], wq[2], wq[3], r.t03);
  transpose4x4(wq[4], wq[5], wq[6], wq[7], r.t47);
#pragma unroll
  for (int k = 0; k < 4; ++k) r.t8[k] = sbyte(wq[8], k);
  return r;
}
// s[k] += sum over the 9 taps of a[t] byte k * w[t] byte k (a[t]: the 4 channels of tap t)
__device__ __forceinline__ void dw_dot9(int (&s)[4], const uint32_t (&av)[9], const DwW9& w) {
  uint32_t c03[4], c47[4];
  transpose4x4(av[0], av[1], av[2], av[3], c03);
  transpose4x4(av[4], av[5], av[6], av[7], c47);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    s[k] = __dp4a(static_cast<int>(c03[k]), static_cast<int>(w.t03[k]), s[k]);
    s[k] = __dp4a(static_cast<int>(c47[k]), static_cast<int>(w.t47[k]), s[k]);
    s[k] += sbyte(av[8], k) * w.t8[k];
  }
}

__device__ __forceinline__ void dw_mac4(int (&s)[4], uint32_t a, uint32_t w) {
#pragma unroll
  for (int k = 0; k < 4; ++k) s[k] += sbyte(a, k) * sbyte(w, k);
}

__device__ __forceinline__ void dw_store4(const int (&s)[4], double rs, float* out, int32_t* acc, uint32_t i4) {
  if (out)
    reinterpret_cast<float4*>(out)[i4] =
        make_float4(static_cast<float>(rs * s[0]), static_cast<float>(rs * s[1]), static_cast<float>(rs * s[2]),
                    static_cast<float>(rs * s[3]));
  if (acc) reinterpret_cast<int4*>(acc)[i4] = make_int4(s[0], s[1], s[2], s[3]);
}

// grid-stride over (pixel, quad); T = threads in the grid is a multiple of C/4,
// so the quad is fixed per thread and the pixel advances by T / (C/4)
template <int R, int S, int SH>
__global__ void __launch_bounds__(256) k_dw_fwd4(const DwArgs d, const uint32_t* __restrict__ a,
                                                 const int8_t* __restrict__ w, const float* clip_a,
                                                 const float* clip_w, float* z, int32_t* acc) {
  pdl_entry();
  const double rs = dw_rescale(clip_a, clip_w);
  const uint32_t nq = d.C / 4, T = gridDim.x * blockDim.x;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t qd = tid % nq;
  uint32_t wq[R * S];
  dw_load_wq<R, S>(w, 4 * qd, wq);
  DwW9 w9;
  if constexpr (R == 3 && S == 3) w9 = dw_w9(wq);
  const uint32_t tot = static_cast<uint32_t>(d.N) * d.P * d.Q * nq;
  for (uint32_t i = tid; i < tot; i += T) {
    const uint32_t pix = i / nq;
    const uint32_t q = pix % d.Q, np = pix / d.Q, p = np % d.P, n = np / d.P;
    const int y0 = static_cast<int>(p) * SH - d.ph, x0 = static_cast<int>(q) * SH - d.pw;
    const uint32_t* img = a + static_cast<uint32_t>(n) * d.H * d.W * nq + qd;
    int s[4] = {0, 0, 0, 0};
    if constexpr (R == 3 && S == 3) {  // every tap loaded (0 outside), four taps per DP4A
      uint32_t av[9];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const int ih = y0 + r;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int iw = x0 + t;
          const bool ok = ih >= 0 && ih < d.H && iw >= 0 && iw < d.W;
          av[r * 3 + t] = ok ? __ldg(img + (static_cast<uint32_t>(ih) * d.W + iw) * nq) : 0u;
        }
      }
      dw_dot9(s, av, w9);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int ih = y0 + r;
        if (ih < 0 || ih >= d.H) continue;
#pragma unroll
        for (int t = 0; t < S; ++t) {
          const int iw = x0 + t;
          if (iw < 0 || iw >= d.W) continue;
          dw_mac4(s, __ldg(img + (static_cast<uint32_t>(ih) * d.W + iw) * nq), wq[r * S + t]);
        }
      }
    }
    dw_store4(s, rs, z, acc, i);
  }
}

// ga[n,h,w,c] = sum over the taps with (h+ph-r) % SH == 0, (w+pw-s) % SH == 0
template <int R, int S, int SH>
__global__ void __launch_bounds__(256) k_dw_dgrad4(const DwArgs d, const uint32_t* __restrict__ g,
                                                   const int8_t* __restrict__ w, const float* clip_g,
                                                   const float* clip_w, float* ga, int32_t* acc) {
  pdl_entry();
  const double rs = dw_rescale(clip_g, clip_w);
  const uint32_t nq = d.C / 4, T = gridDim.x * blockDim.x;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t qd = tid % nq;
  uint32_t wq[R * S];
  dw_load_wq<R, S>(w, 4 * qd, wq);
  DwW9 w9;
  if constexpr (R == 3 && S == 3) w9 = dw_w9(wq);
  const uint32_t tot = static_cast<uint32_t>(d.N) * d.H * d.W * nq;
  for (uint32_t i = tid; i < tot; i += T) {
    const uint32_t pix = i / nq;
    const uint32_t x = pix % d.W, ny = pix / d.W, y = ny % d.H, n = ny / d.H;
    const uint32_t* img = g + static_cast<uint32_t>(n) * d.P * d.Q * nq + qd;
    int s[4] = {0, 0, 0, 0};
    if constexpr (R == 3 && S == 3) {  // every tap loaded (0 where it does not reach), DP4A over 4 taps
      uint32_t av[9];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const int pn = static_cast<int>(y) + d.ph - r;
        const int p = pn / SH;
        const bool rok = pn >= 0 && (SH == 1 || pn % SH == 0) && p < d.P;
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const int qn = static_cast<int>(x) + d.pw - t;
          const int qq = qn / SH;
          const bool ok = rok && qn >= 0 && (SH == 1 || qn % SH == 0) && qq < d.Q;
          av[r * 3 + t] = ok ? __ldg(img + (static_cast<uint32_t>(p) * d.Q + qq) * nq) : 0u;
        }
      }
      dw_dot9(s, av, w9);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int pn = static_cast<int>(y) + d.ph - r;
        if (pn < 0 || (SH > 1 && pn % SH)) continue;
        const int p = pn / SH;
        if (p >= d.P) continue;
#pragma unroll
        for (int t = 0; t < S; ++t) {
          const int qn = static_cast<int>(x) + d.pw - t;
          if (qn < 0 || (SH > 1 && qn % SH)) continue;
          const int qq = qn / SH;
          if (qq >= d.Q) continue;
          dw_mac4(s, __ldg(img + (static_cast<uint32_t>(p) * d.Q + qq) * nq), wq[r * S + t]);
        }
      }
    }
    dw_store4(s, rs, ga, acc, i);
  }
}

// gw[c][r*S+s] = sum_{n,p,q} g[n,p,q,c] * a[n, p*SH-ph+r, q*SH-pw+s, c]:
// a lane takes groups of 4 consecutive output pixels of one row for its channel
// quad, transposes the 4 pixels x 4 channels byte blocks with PRMT and
// accumulates each channel's 4-pixel dot product with one DP4A per tap.
// block = 64 quads x 4 lanes over a run of pixel groups (int32 partials stay
// exact), the lanes folded in smem, one int32 partial row per block, summed in
// int64 over the blocks by k_dw_wgrad_reduce.

__device__ __forceinline__ void transpose4x4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t (&c)[4]) {
  const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w2, w3, 0x5140);
  const uint32_t t2 = __byte_perm(w0, w1, 0x7362), t3 = __byte_perm(w2, w3, 0x7362);
  c[0] = __byte_perm(t0, t1, 0x5410);
  c[1] = __byte_perm(t0, t1, 0x7632);
  c[2] = __byte_perm(t2, t3, 0x5410);
  c[3] = __byte_perm(t2, t3, 0x7632);
}

template <int R, int S, int SH, int QB>
__global__ void __launch_bounds__(256) k_dw_wgrad4(const DwArgs d, const uint32_t* __restrict__ g,
                                                   const uint32_t* __restrict__ a, int32_t* __restrict__ part,
                                                   uint32_t groups_per_block) {
  pdl_entry();
  constexpr int LANES = 256 / QB;  // QB channel quads per block, LANES pixel-group lanes per quad
  const uint32_t nq = d.C / 4;
  const uint32_t qd = blockIdx.x * QB + (threadIdx.x % QB);
  const bool live = qd < nq;  // no early return: the block folds its lanes with a barrier
  const uint32_t lane4 = threadIdx.x / QB;
  const uint32_t qgs = (d.Q + 3) / 4;  // pixel groups per output row
  const uint32_t ngroups = static_cast<uint32_t>(d.N) * d.P * qgs;
  const uint32_t lo = blockIdx.y * groups_per_block;
  const uint32_t hi = min(lo + groups_per_block, ngroups);
  int sum[R * S][4];
#pragma unroll
  for (int t = 0; t < R * S; ++t) sum[t][0] = sum[t][1] = sum[t][2] = sum[t][3] = 0;
  for (uint32_t gi = lo + lane4; live && gi < hi; gi += LANES) {
    const uint32_t qg = gi % qgs, np = gi / qgs, p = np % d.P, n = np / d.P;
    const uint32_t q0 = qg * 4;
    const uint32_t* grow = g + ((static_cast<uint32_t>(n) * d.P + p) * d.Q) * nq + qd;
    uint32_t gw[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) gw[i] = (q0 + i < static_cast<uint32_t>(d.Q)) ? __ldg(grow + (q0 + i) * nq) : 0u;
    if ((gw[0] | gw[1] | gw[2] | gw[3]) == 0u) continue;  // common: sparse quantised gradients
    uint32_t gc[4];
    transpose4x4(gw[0], gw[1], gw[2], gw[3], gc);
    const uint32_t* img = a + static_cast<uint32_t>(n) * d.H * d.W * nq + qd;
    const int y0 = static_cast<int>(p) * SH - d.ph, x0 = static_cast<int>(q0) * SH - d.pw;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int ih = y0 + r;
      if (ih < 0 || ih >= d.H) continue;
      const uint32_t* arow = img + static_cast<uint32_t>(ih) * d.W * nq;
      if constexpr (SH == 1 && S == 3) {
        // sliding window: the 3 taps of 4 consecutive pixels span 6 input
        // columns -- load each once, transpose two 4-column blocks, shift per tap
        uint32_t aw[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          const int iw = x0 + j;
          aw[j] = (iw >= 0 && iw < d.W) ? __ldg(arow + iw * nq) : 0u;
        }
        uint32_t c0[4], c1[4];
        transpose4x4(aw[0], aw[1], aw[2], aw[3], c0);
        transpose4x4(aw[4], aw[5], 0u, 0u, c1);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          sum[r * 3 + 0][k] = __dp4a(static_cast<int>(gc[k]), static_cast<int>(c0[k]), sum[r * 3 + 0][k]);
          sum[r * 3 + 1][k] = __dp4a(static_cast<int>(gc[k]), static_cast<int>(__byte_perm(c0[k], c1[k], 0x4321)),
                                     sum[r * 3 + 1][k]);
          sum[r * 3 + 2][k] = __dp4a(static_cast<int>(gc[k]), static_cast<int>(__byte_perm(c0[k], c1[k], 0x5432)),
                                     sum[r * 3 + 2][k]);
        }
        continue;
      }
#pragma unroll
      for (int t = 0; t < S; ++t) {
        uint32_t aw[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int iw = x0 + i * SH + t;
          aw[i] = (iw >= 0 && iw < d.W && q0 + i < static_cast<uint32_t>(d.Q)) ? __ldg(arow + iw * nq) : 0u;
        }
        uint32_t ac[4];
        transpose4x4(aw[0], aw[1], aw[2], aw[3], ac);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          sum[r * S + t][k] = __dp4a(static_cast<int>(gc[k]), static_cast<int>(ac[k]), sum[r * S + t][k]);
      }
    }
  }
  __shared__ int red[LANES - 1][QB][R * S * 4 + 1];  // lanes 1.. (+1 pad: bank spread)
  if (lane4) {
#pragma unroll
    for (int t = 0; t < R * S; ++t)
#pragma unroll
      for (int k = 0; k < 4; ++k) red[lane4 - 1][threadIdx.x % QB][t * 4 + k] = sum[t][k];
  }
  __syncthreads();
  if (lane4) return;
  // this block's exact partial per (channel, tap): int32 (groups_per_block x 4 pixels x 127^2 < 2^31),
  // one row per block -- summed in int64 by k_dw_wgrad_reduce (no contended atomics)
  int32_t* prow = part + static_cast<size_t>(blockIdx.y) * d.C * (R * S);
#pragma unroll
  for (int t = 0; t < R * S; ++t)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int v = sum[t][k];
#pragma unroll
      for (int l = 0; l < LANES - 1; ++l) v += red[l][threadIdx.x][t * 4 + k];
      if (live) prow[(4 * qd + k) * (R * S) + t] = v;
    }
}

// acc[i] = sum over the blocks' partial rows (int64, exact), and gw[i] =
// float(s_g * s_a * acc[i]); P threads per output fold strided row subsets.
constexpr int DWR_P = 32;
__global__ void __launch_bounds__(256) k_dw_wgrad_reduce(const int32_t* __restrict__ part, int rows, int n,
                                                         long long* __restrict__ acc, const float* clip_g,
                                                         const float* clip_a, float* __restrict__ gw) {
  pdl_entry();
  constexpr int W = 256 / DWR_P;
  __shared__ long long red[DWR_P][W];
  const int lo = threadIdx.x % W, ph = threadIdx.x / W;
  const int i = blockIdx.x * W + lo;
  long long sum = 0;
  if (i < n)
    for (int r = ph; r < rows; r += DWR_P) sum += __ldg(part + static_cast<size_t>(r) * n + i);
  red[ph][lo] = sum;
  __syncthreads();
  if (ph == 0 && i < n) {
#pragma unroll
    for (int p = 1; p < DWR_P; ++p) sum += red[p][lo];
    if (acc) acc[i] = sum;
    if (gw) gw[i] = static_cast<float>(dw_rescale(clip_g, clip_a) * static_cast<double>(sum));
  }
}

static bool dw_quad_ok(const DwArgs& d, const void* p0, const void* p1) {
  return d.C % 4 == 0 && d.Cp == d.C && d.R == 3 && d.S == 3 && d.sh == d.sw && (d.sh == 1 || d.sh == 2) &&
         (reinterpret_cast<uintptr_t>(p0) & 3u) == 0 && (reinterpret_cast<uintptr_t>(p1) & 3u) == 0 &&
         static_cast<int64_t>(d.N) * d.H * d.W * d.C < (int64_t(1) << 32) &&
         static_cast<int64_t>(d.N) * d.P * d.Q * d.C < (int64_t(1) << 32);
}

static int quad_grid(int64_t tot_quads, int nq) {
  int64_t b = (tot_quads + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  if (b < 1) b = 1;
  // threads (b*256) a multiple of nq: the quad stays fixed per thread
  int64_t g = 1, x = 256, y = nq;
  while (y) { const int64_t t = x % y; x = y; y = t; }
  g = nq / x;
  return static_cast<int>((b + g - 1) / g * g);
}

static int dw_args(const i8t_conv_geom* g, int64_t c_pad, DwArgs& d) {
  if (!g || !g->depthwise || g->k != g->c) return set_error(I8T_EINVAL, "conv_dw: geometry must be depthwise with k == c");
  if (g->n < 1 || g->c < 1 || g->h < 1 || g->w < 1 || g->kh < 1 || g->kw < 1 || g->stride_h < 1 || g->stride_w < 1 ||
      g->pad_h < 0 || g->pad_w < 0 || g->h + 2 * g->pad_h < g->kh || g->w + 2 * g->pad_w < g->kw)
    return set_error(I8T_EINVAL, "ConvGeometry: extents must be positive, pad nonnegative");
  if (!g->floor_mode && ((g->h + 2 * g->pad_h - g->kh) % g->stride_h != 0 || (g->w + 2 * g->pad_w - g->kw) % g->stride_w != 0))
    return set_error(I8T_EINVAL, "ConvGeometry: output size is not a positive integer");
  if (g->kh * g->kw > DW_MAXTAP) return set_error(I8T_EUNSUPPORTED, "conv_dw: kernel larger than 7x7");
  if (c_pad < g->c) return set_error(I8T_EINVAL, "conv_dw: c_pad < c");
  d.N = (int)g->n; d.H = (int)g->h; d.W = (int)g->w; d.C = (int)g->c; d.Cp = (int)c_pad;
  d.R = (int)g->kh; d.S = (int)g->kw; d.sh = (int)g->stride_h; d.sw = (int)g->stride_w; d.ph = (int)g->pad_h; d.pw = (int)g->pad_w;
  d.P = (int)((g->h + 2 * g->pad_h - g->kh) / g->stride_h + 1);
  d.Q = (int)((g->w + 2 * g->pad_w - g->kw) / g->stride_w + 1);
  return I8T_OK;
}

static int blocks_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)(b < 1 ? 1 : (b > 148 * 32 ? 148 * 32 : b));
}

}  // namespace i8t_dev

using namespace i8t_dev;

extern "C" {

int i8t_conv_dw_fwd(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* a, int64_t c_pad, const int8_t* w,
                    const float* clip_a, const float* clip_w, float* z, int32_t* acc) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  DwArgs d;
  int rc = dw_args(g, c_pad, d);
  if (rc) return rc;
  if (!c || !a || !w || !clip_a || !clip_w) return set_error(I8T_EINVAL, "conv_dw_fwd: null argument");
  if (dw_quad_ok(d, a, z ? static_cast<const void*>(z) : static_cast<const void*>(acc))) {
    const int nq = d.C / 4, grid = quad_grid(static_cast<int64_t>(d.N) * d.P * d.Q * nq, nq);
    const uint32_t* a4 = reinterpret_cast<const uint32_t*>(a);
    if (d.sh == 1) launch_k(k_dw_fwd4<3, 3, 1>, grid, 256, 0, c->stream, d, a4, w, clip_a, clip_w, z, acc);
    else launch_k(k_dw_fwd4<3, 3, 2>, grid, 256, 0, c->stream, d, a4, w, clip_a, clip_w, z, acc);
    count_launch(1);
    return cuda_check("k_dw_fwd4");
  }
  launch_k(k_dw_fwd, blocks_for((int64_t)d.N * d.P * d.Q * d.C), 256, 0, c->stream, d, a, w, clip_a, clip_w, z, acc);
  count_launch(1);
  return cuda_check("k_dw_fwd");
}

int i8t_conv_dw_dgrad(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, int64_t c_pad, const int8_t* w,
                      const float* clip_g, const float* clip_w, float* ga, int32_t* acc) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  DwArgs d;
  int rc = dw_args(g, c_pad, d);
  if (rc) return rc;
  if (!c || !gz || !w || !clip_g || !clip_w) return set_error(I8T_EINVAL, "conv_dw_dgrad: null argument");
  if (dw_quad_ok(d, gz, ga ? static_cast<const void*>(ga) : static_cast<const void*>(acc))) {
    const int nq = d.C / 4, grid = quad_grid(static_cast<int64_t>(d.N) * d.H * d.W * nq, nq);
    const uint32_t* g4 = reinterpret_cast<const uint32_t*>(gz);
    if (d.sh == 1) launch_k(k_dw_dgrad4<3, 3, 1>, grid, 256, 0, c->stream, d, g4, w, clip_g, clip_w, ga, acc);
    else launch_k(k_dw_dgrad4<3, 3, 2>, grid, 256, 0, c->stream, d, g4, w, clip_g, clip_w, ga, acc);
    count_launch(1);
    return cuda_check("k_dw_dgrad4");
  }
  launch_k(k_dw_dgrad, blocks_for((int64_t)d.N * d.H * d.W * d.C), 256, 0, c->stream, d, gz, w, clip_g, clip_w, ga, acc);
  count_launch(1);
  return cuda_check("k_dw_dgrad");
}

int i8t_conv_dw_wgrad(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, const int8_t* a, int64_t c_pad,
                      const float* clip_g, const float* clip_a, int64_t* acc, float* gw) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  DwArgs d;
  int rc = dw_args(g, c_pad, d);
  if (rc) return rc;
  if (!c || !gz || !a || !clip_g || !clip_a || !acc) return set_error(I8T_EINVAL, "conv_dw_wgrad: null argument");
  const int64_t RS = (int64_t)d.R * d.S, npq = (int64_t)d.N * d.P * d.Q;
  if (dw_quad_ok(d, gz, a)) {
    const int nq = d.C / 4;
    const int64_t ngroups = static_cast<int64_t>(d.N) * d.P * ((d.Q + 3) / 4);
    // ~4 blocks per SM over the pixel groups; each block's partial stays an exact int32
    // quads per block: the width that leaves the fewest threads without a channel
    int qb = 64;
    for (int cand : {64, 32, 16})
      if (static_cast<int64_t>(nq) * 1000 / ((nq + cand - 1) / cand * cand) >
          static_cast<int64_t>(nq) * 1000 / ((nq + qb - 1) / qb * qb))
        qb = cand;
    const int64_t cblk = (nq + qb - 1) / qb;
    int64_t ysplit = std::max<int64_t>(1, (4 * 148 + cblk - 1) / cblk);
    int64_t per = (ngroups + ysplit - 1) / ysplit;
    per = std::min<int64_t>(std::max<int64_t>(per, 64), 8192);
    ysplit = (ngroups + per - 1) / per;
    const dim3 grid(static_cast<unsigned>(cblk), static_cast<unsigned>(ysplit));
    const uint32_t *g4 = reinterpret_cast<const uint32_t*>(gz), *a4 = reinterpret_cast<const uint32_t*>(a);
    int32_t* part = reinterpret_cast<int32_t*>(ensure_scratch(c, sizeof(int32_t) * static_cast<size_t>(ysplit * d.C * RS)));
    if (!part) return set_error(I8T_ECUDA, "conv_dw_wgrad: scratch alloc failed");
#define DW_WG(SH_, QB_) launch_k(k_dw_wgrad4<3, 3, SH_, QB_>, grid, 256, 0, c->stream, d, g4, a4, part, static_cast<uint32_t>(per))
    if (d.sh == 1) {
      if (qb == 64) DW_WG(1, 64); else if (qb == 32) DW_WG(1, 32); else DW_WG(1, 16);
    } else {
      if (qb == 64) DW_WG(2, 64); else if (qb == 32) DW_WG(2, 32); else DW_WG(2, 16);
    }
#undef DW_WG
    count_launch(1);
    if ((rc = cuda_check("k_dw_wgrad4"))) return rc;
    const int n = static_cast<int>(d.C * RS);
    launch_k(k_dw_wgrad_reduce, (n + 256 / DWR_P - 1) / (256 / DWR_P), 256, 0, c->stream, part, static_cast<int>(ysplit), n,
             reinterpret_cast<long long*>(acc), clip_g, clip_a, gw);
    count_launch(1);
    return cuda_check("k_dw_wgrad_reduce");
  }
  cudaMemsetAsync(acc, 0, sizeof(int64_t) * d.C * RS, c->stream);
  const int cblk = (d.C + 63) / 64;
  int64_t ysplit = (4 * 148 + cblk - 1) / cblk;
  int64_t per = (npq + ysplit - 1) / ysplit;
  if (per < 256) per = 256;
  ysplit = (npq + per - 1) / per;
  launch_k(k_dw_wgrad, dim3((unsigned)cblk, (unsigned)ysplit), 256, 0, c->stream, d, gz, a, reinterpret_cast<unsigned long long*>(acc), per);
  count_launch(1);
  if (gw) {
    launch_k(k_dw_wgrad_finalize, blocks_for(d.C * RS), 256, 0, c->stream, reinterpret_cast<const long long*>(acc), d.C * RS, clip_g, clip_a, gw);
    count_launch(1);
  }
  return cuda_check("k_dw_wgrad");
}

int i8t_conv_dw_wgrad_finalize(i8t_ctx* ctx, const i8t_conv_geom* g, const int64_t* acc, const float* clip_g,
                               const float* clip_a, float* gw) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !g || !acc || !clip_g || !clip_a || !gw) return set_error(I8T_EINVAL, "conv_dw_wgrad_finalize: null argument");
  const int64_t n = g->c * g->kh * g->kw;
  launch_k(k_dw_wgrad_finalize, blocks_for(n), 256, 0, c->stream, reinterpret_cast<const long long*>(acc), n, clip_g, clip_a, gw);
  count_launch(1);
  return cuda_check("k_dw_wgrad_finalize");
}

}  // extern "C"
