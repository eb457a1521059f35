// pool.cu -- max pooling with padding on NHWC fp32 (the EXT of SURVEY.md A.3-5:
// the reference Pool2d, layers.cpp:346-380, has no padding), fused with the
// BatchNorm + ReLU that precede it in the ResNet stem:
//   forward   y[n,p,q,c] = max over the k x k window of act(bn(z)) (or of x),
//             idx = the window slot (dy*k + dx) of the first maximum, one byte;
//   backward  gx[n,h,w,c] = sum of gy over the windows whose argmax is (h, w),
//             gathered per input pixel in increasing (p, q) order.
// Padded positions never win (they are skipped, i.e. -inf).  NaN wins like
// torch's max_pool2d.  One thread per (pixel, channel quad); float4 I/O.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "bncore.cuh"
#include "internal.cuh"

namespace i8t_dev {

struct PoolGeom {
  int N, H, W, C, P, Q, k, s, pad;
};

template <bool BN>
__global__ void __launch_bounds__(256) k_maxpool_fwd(const float* __restrict__ x, PoolGeom g, const double* bn,
                                                     const float* gamma, const float* beta, int relu,
                                                     float* __restrict__ y, uint8_t* __restrict__ idx) {
  pdl_entry();
  const uint32_t c4n = g.C / 4;
  const uint32_t tot = static_cast<uint32_t>(g.N) * g.P * g.Q * c4n;  // < 2^31 (host check)
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
    const uint32_t c4 = i % c4n, pix = i / c4n;
    const int q = static_cast<int>(pix % g.Q);
    const uint32_t np = pix / g.Q;
    const int p = static_cast<int>(np % g.P), n = static_cast<int>(np / g.P);
    BnQuad k;
    if (BN) k.load(bn, gamma, beta, g.C, c4 * 4);
    float best[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    int arg[4] = {0, 0, 0, 0};
    bool any[4] = {false, false, false, false};
    const int h0 = p * g.s - g.pad, w0 = q * g.s - g.pad;
    for (int dy = 0; dy < g.k; ++dy) {
      const int h = h0 + dy;
      if (h < 0 || h >= g.H) continue;
      for (int dx = 0; dx < g.k; ++dx) {
        const int w = w0 + dx;
        if (w < 0 || w >= g.W) continue;
        const float4 v4 = __ldg(reinterpret_cast<const float4*>(x) + ((static_cast<uint32_t>(n) * g.H + h) * g.W + w) * c4n + c4);
        float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (BN) {
            v[j] = k.y(j, v[j]);
            if (relu) v[j] = v[j] > 0.0f ? v[j] : 0.0f;
          }
          if (!any[j] || v[j] > best[j] || isnan(v[j])) {  // torch's max_pool2d update rule
            best[j] = v[j];
            arg[j] = dy * g.k + dx;
            any[j] = true;
          }
        }
      }
    }
    reinterpret_cast<float4*>(y)[i] = make_float4(best[0], best[1], best[2], best[3]);
    reinterpret_cast<uchar4*>(idx)[i] = make_uchar4(arg[0], arg[1], arg[2], arg[3]);
  }
}

// 3x3 / stride 2 / pad 1 with H == 2P, W == 2Q (the ResNet stem): a thread
// walks a column of RUN windows (n, p0.., q, quad) downwards, so the window's
// top row (2p-1) is the previous window's bottom row, already loaded and
// normalised: 6 loads and 24 BN evaluations per window instead of 9 and 36.
// The 9 slots are scanned in the same (dy, dx) order with the same update rule
// as k_maxpool_fwd; only the top row (p = 0) and the left column (q = 0) pad.
template <bool BN>
__global__ void __launch_bounds__(256, 3) k_maxpool_fwd_s2k3(const float* __restrict__ x, PoolGeom g, const double* bn,
                                                          const float* gamma, const float* beta, int relu, int run,
                                                          float* __restrict__ y, uint8_t* __restrict__ idx) {
  pdl_entry();
  const uint32_t c4n = g.C / 4;
  const uint32_t nrun = (g.P + run - 1) / run;
  const uint32_t tot = static_cast<uint32_t>(g.N) * nrun * g.Q * c4n;  // < 2^31 (host check)
  const float4* x4 = reinterpret_cast<const float4*>(x);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
    const uint32_t c4 = i % c4n, t = i / c4n;
    const int q = static_cast<int>(t % g.Q);
    const uint32_t t2 = t / g.Q;
    const int pr = static_cast<int>(t2 % nrun), n = static_cast<int>(t2 / nrun);
    BnQuad k;
    if (BN) k.load(bn, gamma, beta, g.C, c4 * 4);
    const bool lok = q > 0;  // the left column 2q-1 exists
    const int wl = lok ? 2 * q - 1 : 2 * q;  // clamped (the value is then ignored)
    const uint32_t rowp = static_cast<uint32_t>(g.W) * c4n;
    const float4* xn = x4 + static_cast<uint32_t>(n) * g.H * rowp + c4;
    auto act = [&](const float4 v4, float (&v)[4]) {
      v[0] = v4.x; v[1] = v4.y; v[2] = v4.z; v[3] = v4.w;
      if (BN) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v[j] = k.y(j, v[j]);
          if (relu) v[j] = v[j] > 0.0f ? v[j] : 0.0f;
        }
      }
    };
    int p = pr * run;
    const int pe = p + run < g.P ? p + run : g.P;
    float top[3][4];
    bool top_ok = p > 0;
    if (top_ok) {
      const float4* r = xn + static_cast<uint32_t>(2 * p - 1) * rowp;
      const float4 a = __ldg(r + static_cast<uint32_t>(wl) * c4n), b = __ldg(r + static_cast<uint32_t>(2 * q) * c4n),
                   c = __ldg(r + static_cast<uint32_t>(2 * q + 1) * c4n);
      act(a, top[0]);
      act(b, top[1]);
      act(c, top[2]);
    }
    for (; p < pe; ++p) {
      const float4* r1 = xn + static_cast<uint32_t>(2 * p) * rowp;
      const float4* r2 = r1 + rowp;
      float4 l[6];
      l[0] = __ldg(r1 + static_cast<uint32_t>(wl) * c4n);
      l[1] = __ldg(r1 + static_cast<uint32_t>(2 * q) * c4n);
      l[2] = __ldg(r1 + static_cast<uint32_t>(2 * q + 1) * c4n);
      l[3] = __ldg(r2 + static_cast<uint32_t>(wl) * c4n);
      l[4] = __ldg(r2 + static_cast<uint32_t>(2 * q) * c4n);
      l[5] = __ldg(r2 + static_cast<uint32_t>(2 * q + 1) * c4n);
      float mid[3][4], bot[3][4];
      act(l[0], mid[0]); act(l[1], mid[1]); act(l[2], mid[2]);
      act(l[3], bot[0]); act(l[4], bot[1]); act(l[5], bot[2]);
      float best[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      int arg[4] = {0, 0, 0, 0};
      bool any[4] = {false, false, false, false};
      auto take = [&](const float (&v)[4], int slot) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (!any[j] || v[j] > best[j] || isnan(v[j])) {  // torch's max_pool2d update rule
            best[j] = v[j];
            arg[j] = slot;
            any[j] = true;
          }
      };
      if (top_ok) {
        if (lok) take(top[0], 0);
        take(top[1], 1);
        take(top[2], 2);
      }
      if (lok) take(mid[0], 3);
      take(mid[1], 4);
      take(mid[2], 5);
      if (lok) take(bot[0], 6);
      take(bot[1], 7);
      take(bot[2], 8);
      const uint32_t o = ((static_cast<uint32_t>(n) * g.P + p) * g.Q + q) * c4n + c4;
      reinterpret_cast<float4*>(y)[o] = make_float4(best[0], best[1], best[2], best[3]);
      reinterpret_cast<uchar4*>(idx)[o] = make_uchar4(arg[0], arg[1], arg[2], arg[3]);
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int j = 0; j < 4; ++j) top[c][j] = bot[c][j];
      top_ok = true;
    }
  }
}

__global__ void __launch_bounds__(256) k_maxpool_bwd(const float* __restrict__ gy, const uint8_t* __restrict__ idx,
                                                     PoolGeom g, float* __restrict__ gx) {
  pdl_entry();
  const uint32_t c4n = g.C / 4;
  const uint32_t tot = static_cast<uint32_t>(g.N) * g.H * g.W * c4n;  // < 2^31 (host check)
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
    const uint32_t c4 = i % c4n, pix = i / c4n;
    const int w = static_cast<int>(pix % g.W);
    const uint32_t nh = pix / g.W;
    const int h = static_cast<int>(nh % g.H), n = static_cast<int>(nh / g.H);
    // windows p with p*s - pad <= h <= p*s - pad + k - 1
    const int hp = h + g.pad, wp = w + g.pad;
    const int p_lo = hp - g.k + 1 <= 0 ? 0 : (hp - g.k + g.s) / g.s, p_hi = min(hp / g.s, g.P - 1);
    const int q_lo = wp - g.k + 1 <= 0 ? 0 : (wp - g.k + g.s) / g.s, q_hi = min(wp / g.s, g.Q - 1);
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int p = p_lo; p <= p_hi; ++p) {
      const int dy = hp - p * g.s;
      for (int q = q_lo; q <= q_hi; ++q) {
        const int slot = dy * g.k + (wp - q * g.s);
        const uint32_t o = ((static_cast<uint32_t>(n) * g.P + p) * g.Q + q) * c4n + c4;
        const uchar4 a = reinterpret_cast<const uchar4*>(idx)[o];
        const float4 v = __ldg(reinterpret_cast<const float4*>(gy) + o);
        if (a.x == slot) acc[0] = __fadd_rn(acc[0], v.x);
        if (a.y == slot) acc[1] = __fadd_rn(acc[1], v.y);
        if (a.z == slot) acc[2] = __fadd_rn(acc[2], v.z);
        if (a.w == slot) acc[3] = __fadd_rn(acc[3], v.w);
      }
    }
    reinterpret_cast<float4*>(gx)[i] = make_float4(acc[0], acc[1], acc[2], acc[3]);
  }
}

// 3x3 / stride 2 / pad 1 with even H, W (the ResNet stem): a thread owns the
// 2x2 input block (2p', 2q') .. (2p'+1, 2q'+1) and reads only the four windows
// (p'..p'+1, q'..q'+1) that can reach it -- the same terms, in the same
// (p, q) order, as k_maxpool_bwd.
__global__ void __launch_bounds__(256) k_maxpool_bwd_s2k3(const float* __restrict__ gy, const uint8_t* __restrict__ idx,
                                                          PoolGeom g, float* __restrict__ gx) {
  pdl_entry();
  const uint32_t c4n = g.C / 4;
  const uint32_t tot = static_cast<uint32_t>(g.N) * g.P * g.Q * c4n;  // one 2x2 block per (n, p', q', quad)
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
    const uint32_t c4 = i % c4n, blk = i / c4n;
    const uint32_t q = blk % g.Q, np = blk / g.Q;
    const uint32_t p = np % g.P, n = np / g.P;
    const bool pn = p + 1 < static_cast<uint32_t>(g.P), qn = q + 1 < static_cast<uint32_t>(g.Q);
    auto win = [&](uint32_t pp, uint32_t qq, uchar4& a, float4& v) {
      const uint32_t o = ((n * g.P + pp) * g.Q + qq) * c4n + c4;
      a = reinterpret_cast<const uchar4*>(idx)[o];
      v = __ldg(reinterpret_cast<const float4*>(gy) + o);
    };
    uchar4 a00, a01 = make_uchar4(9, 9, 9, 9), a10 = a01, a11 = a01;
    float4 g00, g01 = make_float4(0, 0, 0, 0), g10 = g01, g11 = g01;
    win(p, q, a00, g00);
    if (qn) win(p, q + 1, a01, g01);
    if (pn) win(p + 1, q, a10, g10);
    if (pn && qn) win(p + 1, q + 1, a11, g11);
    const uint8_t s00[4] = {a00.x, a00.y, a00.z, a00.w}, s01[4] = {a01.x, a01.y, a01.z, a01.w},
                  s10[4] = {a10.x, a10.y, a10.z, a10.w}, s11[4] = {a11.x, a11.y, a11.z, a11.w};
    const float v00[4] = {g00.x, g00.y, g00.z, g00.w}, v01[4] = {g01.x, g01.y, g01.z, g01.w},
                v10[4] = {g10.x, g10.y, g10.z, g10.w}, v11[4] = {g11.x, g11.y, g11.z, g11.w};
    float o[4][4];  // [pixel of the 2x2 block][channel]
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      o[0][j] = s00[j] == 4 ? __fadd_rn(0.0f, v00[j]) : 0.0f;
      float t = s00[j] == 5 ? __fadd_rn(0.0f, v00[j]) : 0.0f;
      o[1][j] = s01[j] == 3 ? __fadd_rn(t, v01[j]) : t;
      t = s00[j] == 7 ? __fadd_rn(0.0f, v00[j]) : 0.0f;
      o[2][j] = s10[j] == 1 ? __fadd_rn(t, v10[j]) : t;
      t = s00[j] == 8 ? __fadd_rn(0.0f, v00[j]) : 0.0f;
      t = s01[j] == 6 ? __fadd_rn(t, v01[j]) : t;
      t = s10[j] == 2 ? __fadd_rn(t, v10[j]) : t;
      o[3][j] = s11[j] == 0 ? __fadd_rn(t, v11[j]) : t;
    }
    const uint32_t h = 2 * p, w = 2 * q;
    float4* base = reinterpret_cast<float4*>(gx);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t hh = h + (k >> 1), ww = w + (k & 1);
      base[((n * g.H + hh) * g.W + ww) * c4n + c4] = make_float4(o[k][0], o[k][1], o[k][2], o[k][3]);
    }
  }
}

static int pool_geom(int64_t n, int64_t h, int64_t w, int64_t c, int64_t k, int64_t s, int64_t pad, PoolGeom* g) {
  if (n < 1 || h < 1 || w < 1 || c < 4 || c % 4 != 0 || k < 1 || k > 15 || s < 1 || pad < 0 || 2 * pad > k)
    return set_error(I8T_EINVAL, "maxpool: bad geometry (needs c % 4 == 0, k <= 15, pad <= k/2)");
  if (h + 2 * pad < k || w + 2 * pad < k) return set_error(I8T_EINVAL, "maxpool: window larger than the input");
  if (n * h * w * c >= (int64_t(1) << 33)) return set_error(I8T_EUNSUPPORTED, "maxpool: tensor >= 2^33 elements");
  g->N = (int)n; g->H = (int)h; g->W = (int)w; g->C = (int)c; g->k = (int)k; g->s = (int)s; g->pad = (int)pad;
  g->P = (int)((h + 2 * pad - k) / s + 1);
  g->Q = (int)((w + 2 * pad - k) / s + 1);
  return I8T_OK;
}

static int grid_of(int64_t tot) {
  int64_t b = (tot + 255) / 256;
  return static_cast<int>(b > 148 * 16 ? 148 * 16 : (b < 1 ? 1 : b));
}

}  // namespace i8t_dev

using namespace i8t_dev;

// Global average pool over NHWC [n][hw][c] (Pool2d kAvg with the window the
// whole map, layers.cpp:383-388): one thread per (n, c) sums its hw values in
// double in the reference's order, then float(acc / hw).
__global__ void __launch_bounds__(256) k_gap_fwd(const float* __restrict__ x, int n, int hw, int c,
                                                 float* __restrict__ y) {
  pdl_entry();
  const int64_t tot = static_cast<int64_t>(n) * c;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < tot;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = i / c, ch = i - b * c;
    const float* p = x + b * hw * c + ch;
    double acc = 0.0;
#pragma unroll 8
    for (int k = 0; k < hw; ++k) acc += __ldg(p + static_cast<int64_t>(k) * c);
    y[i] = static_cast<float>(acc / hw);
  }
}

// Its backward (layers.cpp:392-414): every position of (n, c) gets
// g[n][c] / float(hw).
__global__ void __launch_bounds__(256) k_gap_bwd(const float* __restrict__ g, int n, int hw, int c,
                                                 float* __restrict__ gx) {
  pdl_entry();
  const float inv = static_cast<float>(hw);
  const int64_t c4 = c / 4, tot = static_cast<int64_t>(n) * c4;
  // thread per (n, channel quad): the four shares once, then the hw positions
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < tot;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = i / c4, q = i - b * c4;
    const float4 v = __ldg(reinterpret_cast<const float4*>(g) + i);
    const float4 o = make_float4(__fdiv_rn(v.x, inv), __fdiv_rn(v.y, inv), __fdiv_rn(v.z, inv), __fdiv_rn(v.w, inv));
    float4* dst = reinterpret_cast<float4*>(gx) + b * hw * c4 + q;
    for (int k = 0; k < hw; ++k) dst[static_cast<int64_t>(k) * c4] = o;
  }
}

extern "C" {

int i8t_maxpool_fwd(i8t_ctx* ctx, const float* x, int64_t n, int64_t h, int64_t w, int64_t c, int64_t k, int64_t s,
                    int64_t pad, const double* bn, const float* gamma, const float* beta, int relu, float* y,
                    uint8_t* idx) {
  Ctx* cx = reinterpret_cast<Ctx*>(ctx);
  PoolGeom g;
  int rc = pool_geom(n, h, w, c, k, s, pad, &g);
  if (rc) return rc;
  if (!cx || !x || !y || !idx || (bn && (!gamma || !beta))) return set_error(I8T_EINVAL, "maxpool_fwd: bad arguments");
  static const bool no_run = getenv("I8T_NO_POOL_RUN") != nullptr;  // A/B: the per-window kernel
  if (!no_run && g.k == 3 && g.s == 2 && g.pad == 1 && g.H == 2 * g.P && g.W == 2 * g.Q) {
    const int run = 7;
    const int64_t tr = static_cast<int64_t>(g.N) * ((g.P + run - 1) / run) * g.Q * (g.C / 4);
    if (bn)
      launch_k(k_maxpool_fwd_s2k3<true>, grid_of(tr), 256, 0, cx->stream, x, g, bn, gamma, beta, relu, run, y, idx);
    else
      launch_k(k_maxpool_fwd_s2k3<false>, grid_of(tr), 256, 0, cx->stream, x, g, nullptr, nullptr, nullptr, 0, run, y,
               idx);
    count_launch(1);
    return cuda_check("k_maxpool_fwd_s2k3");
  }
  const int64_t tot = static_cast<int64_t>(g.N) * g.P * g.Q * (g.C / 4);
  if (bn) launch_k(k_maxpool_fwd<true>, grid_of(tot), 256, 0, cx->stream, x, g, bn, gamma, beta, relu, y, idx);
  else launch_k(k_maxpool_fwd<false>, grid_of(tot), 256, 0, cx->stream, x, g, nullptr, nullptr, nullptr, 0, y, idx);
  count_launch(1);
  return cuda_check("k_maxpool_fwd");
}

int i8t_maxpool_bwd(i8t_ctx* ctx, const float* gy, const uint8_t* idx, int64_t n, int64_t h, int64_t w, int64_t c,
                    int64_t k, int64_t s, int64_t pad, float* gx) {
  Ctx* cx = reinterpret_cast<Ctx*>(ctx);
  PoolGeom g;
  int rc = pool_geom(n, h, w, c, k, s, pad, &g);
  if (rc) return rc;
  if (!cx || !gy || !idx || !gx) return set_error(I8T_EINVAL, "maxpool_bwd: bad arguments");
  if (g.k == 3 && g.s == 2 && g.pad == 1 && g.H == 2 * g.P && g.W == 2 * g.Q) {
    const int64_t blocks = static_cast<int64_t>(g.N) * g.P * g.Q * (g.C / 4);
    launch_k(k_maxpool_bwd_s2k3, grid_of(blocks), 256, 0, cx->stream, gy, idx, g, gx);
    count_launch(1);
    return cuda_check("k_maxpool_bwd_s2k3");
  }
  const int64_t tot = static_cast<int64_t>(g.N) * g.H * g.W * (g.C / 4);
  launch_k(k_maxpool_bwd, grid_of(tot), 256, 0, cx->stream, gy, idx, g, gx);
  count_launch(1);
  return cuda_check("k_maxpool_bwd");
}

int i8t_global_avgpool_fwd(i8t_ctx* ctx, const float* x, int64_t n, int64_t hw, int64_t c, float* y) {
  Ctx* cx = reinterpret_cast<Ctx*>(ctx);
  if (!cx || !x || !y || n < 1 || hw < 1 || c < 1) return set_error(I8T_EINVAL, "global_avgpool_fwd: bad arguments");
  if (n * hw * c >= (int64_t(1) << 31)) return set_error(I8T_EUNSUPPORTED, "global_avgpool: tensor >= 2^31 elements");
  launch_k(k_gap_fwd, grid_of(n * c), 256, 0, cx->stream, x, static_cast<int>(n), static_cast<int>(hw),
           static_cast<int>(c), y);
  count_launch(1);
  return cuda_check("k_gap_fwd");
}

int i8t_global_avgpool_bwd(i8t_ctx* ctx, const float* g, int64_t n, int64_t hw, int64_t c, float* gx) {
  Ctx* cx = reinterpret_cast<Ctx*>(ctx);
  if (!cx || !g || !gx || n < 1 || hw < 1 || c < 4 || c % 4 ||
      ((reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(gx)) & 15u))
    return set_error(I8T_EINVAL, "global_avgpool_bwd: bad arguments (c % 4, 16-byte alignment)");
  if (n * hw * c >= (int64_t(1) << 31)) return set_error(I8T_EUNSUPPORTED, "global_avgpool: tensor >= 2^31 elements");
  launch_k(k_gap_bwd, grid_of(n * (c / 4)), 256, 0, cx->stream, g, static_cast<int>(n), static_cast<int>(hw),
           static_cast<int>(c), gx);
  count_launch(1);
  return cuda_check("k_gap_bwd");
}

}  // extern "C"
