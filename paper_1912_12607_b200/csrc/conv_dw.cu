// conv_dw.cu -- depthwise INT8 convolutions (conv.cpp:115-131 forward,
// :159-184 backward).  One filter per channel: 9 MACs per output element, so
// these are HBM-bound and stay on CUDA cores (integer IMAD), NHWC so a warp's
// lanes walk consecutive channels (coalesced).  Exact int32/int64 sums, FP64
// rescale epilogue identical to the dense path.
#include <cuda_runtime.h>

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
  const double rs = dw_rescale(clip_g, clip_a);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    gw[i] = static_cast<float>(rs * static_cast<double>(acc[i]));
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
  k_dw_fwd<<<blocks_for((int64_t)d.N * d.P * d.Q * d.C), 256, 0, c->stream>>>(d, a, w, clip_a, clip_w, z, acc);
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
  k_dw_dgrad<<<blocks_for((int64_t)d.N * d.H * d.W * d.C), 256, 0, c->stream>>>(d, gz, w, clip_g, clip_w, ga, acc);
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
  cudaMemsetAsync(acc, 0, sizeof(int64_t) * d.C * RS, c->stream);
  const int cblk = (d.C + 63) / 64;
  int64_t ysplit = (4 * 148 + cblk - 1) / cblk;
  int64_t per = (npq + ysplit - 1) / ysplit;
  if (per < 256) per = 256;
  ysplit = (npq + per - 1) / per;
  k_dw_wgrad<<<dim3((unsigned)cblk, (unsigned)ysplit), 256, 0, c->stream>>>(d, gz, a, reinterpret_cast<unsigned long long*>(acc), per);
  count_launch(1);
  if (gw) {
    k_dw_wgrad_finalize<<<blocks_for(d.C * RS), 256, 0, c->stream>>>(reinterpret_cast<const long long*>(acc), d.C * RS, clip_g, clip_a, gw);
    count_launch(1);
  }
  return cuda_check("k_dw_wgrad");
}

int i8t_conv_dw_wgrad_finalize(i8t_ctx* ctx, const i8t_conv_geom* g, const int64_t* acc, const float* clip_g,
                               const float* clip_a, float* gw) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !g || !acc || !clip_g || !clip_a || !gw) return set_error(I8T_EINVAL, "conv_dw_wgrad_finalize: null argument");
  const int64_t n = g->c * g->kh * g->kw;
  k_dw_wgrad_finalize<<<blocks_for(n), 256, 0, c->stream>>>(reinterpret_cast<const long long*>(acc), n, clip_g, clip_a, gw);
  count_launch(1);
  return cuda_check("k_dw_wgrad_finalize");
}

}  // extern "C"
