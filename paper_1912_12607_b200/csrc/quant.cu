// quant.cu -- forward-side HBM-bound kernels on sm_100a:
//   K1 nearest activation quantiser (float -> int8, fused running max|x|),
//      flat / row-padded NHWC / NCHW->NHWC variants;
//   K2 weight quantiser writing both conv layouts (KRSC for forward, CRSK for
//      backward-data) in one pass;
//   dequantize, quantize_partitioned, layout helpers and the SGD+DCLR update.
// float4 loads / char4 stores, 32-bit index math, one atomicMax per block.
#include <cuda_runtime.h>

#include <cmath>

#include "internal.cuh"
#include "qcore.cuh"

namespace i8t_dev {

// one atomicMax per block (non-negative floats order like their bit patterns)
__device__ __forceinline__ void block_amax(float m, float* amax) {
  __shared__ float sm[RED_THREADS / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) m = fmaxf(m, sm[w]);
    if (m > 0.0f) atomicMax(reinterpret_cast<int*>(amax), __float_as_int(m));
  }
}

// K1 flat: x [n] -> q [n] (n % 4 == 0 path vectorised).
__global__ void __launch_bounds__(RED_THREADS) k_quant_nearest_flat(const float* __restrict__ x, uint32_t n,
                                                                    const float* __restrict__ clip_p,
                                                                    int8_t* __restrict__ q, float* amax, int* err) {
  pdl_entry();
  const float clip = *clip_p, s = scale_of(clip), inv_s = 1.0f / s, hs = __fdiv_rn(0.5f, clip);
  float m = 0.0f;
  bool bad = false;
  const uint32_t n4 = n / 4, stride = gridDim.x * blockDim.x;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  char4* q4 = reinterpret_cast<char4*>(q);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = __ldg(x4 + i);
    bad |= !isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    q4[i] = make_char4(static_cast<signed char>(quant_nearest_fast(v.x, clip, hs, s, inv_s)),
                       static_cast<signed char>(quant_nearest_fast(v.y, clip, hs, s, inv_s)),
                       static_cast<signed char>(quant_nearest_fast(v.z, clip, hs, s, inv_s)),
                       static_cast<signed char>(quant_nearest_fast(v.w, clip, hs, s, inv_s)));
  }
  for (uint32_t i = n4 * 4 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = x[i];
    bad |= !isfinite(v);
    m = fmaxf(m, fabsf(v));
    q[i] = static_cast<int8_t>(quant_nearest_fast(v, clip, hs, s, inv_s));
  }
  if (bad) atomicOr(err, ERR_NONFINITE);
  if (amax) block_amax(m, amax);
}

// K1 of a second consumer of the same activations (the projection shortcut
// conv beside the block's first conv): when its clip equals the first
// consumer's bit for bit, the int8 tensor is the same -- copy it (2 B per
// element instead of 5) and take over the first consumer's running max;
// otherwise quantise as k_quant_nearest_flat.
__global__ void __launch_bounds__(RED_THREADS) k_quant_nearest_share(const float* __restrict__ x, uint32_t n,
                                                                     const float* __restrict__ clip_p,
                                                                     const float* __restrict__ ref_clip,
                                                                     const int8_t* __restrict__ ref_q,
                                                                     const float* ref_amax, int8_t* __restrict__ q,
                                                                     float* amax, int* err) {
  pdl_entry();
  const float clip = *clip_p;
  if (__float_as_uint(clip) == __float_as_uint(*ref_clip)) {
    const uint32_t n16 = n / 16, stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride)
      reinterpret_cast<uint4*>(q)[i] = __ldg(reinterpret_cast<const uint4*>(ref_q) + i);
    for (uint32_t i = n16 * 16 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) q[i] = ref_q[i];
    if (amax && ref_amax && blockIdx.x == 0 && threadIdx.x == 0) {
      const float r = *ref_amax;
      if (r > 0.0f) atomicMax(reinterpret_cast<int*>(amax), __float_as_int(r));
    }
    return;
  }
  const float s = scale_of(clip), inv_s = 1.0f / s, hs = __fdiv_rn(0.5f, clip);
  float m = 0.0f;
  bool bad = false;
  const uint32_t n4 = n / 4, stride = gridDim.x * blockDim.x;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  char4* q4 = reinterpret_cast<char4*>(q);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 v = __ldg(x4 + i);
    bad |= !isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
    q4[i] = make_char4(static_cast<signed char>(quant_nearest_fast(v.x, clip, hs, s, inv_s)),
                       static_cast<signed char>(quant_nearest_fast(v.y, clip, hs, s, inv_s)),
                       static_cast<signed char>(quant_nearest_fast(v.z, clip, hs, s, inv_s)),
                       static_cast<signed char>(quant_nearest_fast(v.w, clip, hs, s, inv_s)));
  }
  for (uint32_t i = n4 * 4 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = x[i];
    bad |= !isfinite(v);
    m = fmaxf(m, fabsf(v));
    q[i] = static_cast<int8_t>(quant_nearest_fast(v, clip, hs, s, inv_s));
  }
  if (bad) atomicOr(err, ERR_NONFINITE);
  if (amax) block_amax(m, amax);
}

// K1 rows: x [rows][cols] -> q [rows][ld_q], zero pad (e.g. the C=3 stem -> 4).
__global__ void __launch_bounds__(RED_THREADS) k_quant_nearest_rows(const float* __restrict__ x, uint32_t rows,
                                                                    uint32_t cols, const float* __restrict__ clip_p,
                                                                    int8_t* __restrict__ q, uint32_t ld_q, float* amax,
                                                                    int* err) {
  pdl_entry();
  const float clip = *clip_p, s = scale_of(clip), inv_s = 1.0f / s, hs = __fdiv_rn(0.5f, clip);
  float m = 0.0f;
  bool bad = false;
  const uint32_t tot = rows * ld_q;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
    const uint32_t r = i / ld_q, c = i - r * ld_q;
    int8_t o = 0;
    if (c < cols) {
      const float v = x[static_cast<size_t>(r) * cols + c];
      bad |= !isfinite(v);
      m = fmaxf(m, fabsf(v));
      o = static_cast<int8_t>(quant_nearest_fast(v, clip, hs, s, inv_s));
    }
    q[i] = o;
  }
  if (bad) atomicOr(err, ERR_NONFINITE);
  if (amax) block_amax(m, amax);
}

// K1 rows for 3-channel pixels padded to 4 (the stem's RGB input): four pixels
// per thread, three float4 loads in, one 16-byte store out.
__global__ void __launch_bounds__(RED_THREADS) k_quant_nearest_rgb(const float4* __restrict__ x, uint32_t rows4,
                                                                   const float* __restrict__ clip_p,
                                                                   uint4* __restrict__ q, float* amax, int* err) {
  pdl_entry();
  const float clip = *clip_p, s = scale_of(clip), inv_s = 1.0f / s, hs = __fdiv_rn(0.5f, clip);
  float m = 0.0f;
  bool bad = false;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < rows4; i += gridDim.x * blockDim.x) {
    const float4 a = __ldg(x + 3 * i), b = __ldg(x + 3 * i + 1), c = __ldg(x + 3 * i + 2);
    const float v[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
    uint32_t w[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      uint32_t word = 0;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const float f = v[3 * p + ch];
        bad |= !isfinite(f);
        m = fmaxf(m, fabsf(f));
        word |= static_cast<uint32_t>(static_cast<uint8_t>(quant_nearest_fast(f, clip, hs, s, inv_s))) << (8 * ch);
      }
      w[p] = word;  // channel 3 = 0 (padding)
    }
    q[i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  if (bad) atomicOr(err, ERR_NONFINITE);
  if (amax) block_amax(m, amax);
}

// K2 over every quantised layer of a model in one launch (blockIdx.y = layer):
// the per-layer launches cost more than their ~150 MB of traffic.  Padding
// bytes of the outputs are never written (zeroed once at allocation).
// All layers' weights in one launch (blockIdx.y = layer).  Each block
// quantises a [32 k x TC c x RS] tile into shared memory from contiguous
// source rows, then writes both device layouts from it in 32-byte runs:
// KRSC (c fastest) and CRSK (k fastest) -- a per-element transpose would
// scatter single bytes across the two outputs.
constexpr int WQ_TK = 32, WQ_TILE = 32 * 32 * 9;
__global__ void __launch_bounds__(256) k_quant_weight_multi(const i8t_wq_desc* __restrict__ descs, int n_layers,
                                                             int* err) {
  pdl_entry();
  __shared__ int8_t tq[WQ_TILE];
  bool bad = false;
  // one flat list of tiles over all layers (a per-layer grid would run the
  // layers one after another, each at the latency of a single tile)
  int layer = 0, first = 0;  // tiles of layers [0, layer) come before `first`
  for (int t = blockIdx.x;; t += gridDim.x) {
    int K = 0, C = 0, RS = 0, TK = 0, TC = 0, ktiles = 0, ctiles = 0;
    for (; layer < n_layers; ++layer) {
      const i8t_wq_desc& dl = descs[layer];
      K = dl.k; C = dl.c; RS = dl.rs;
      TK = min(WQ_TK, max(1, WQ_TILE / RS));
      TC = min(256, max(1, WQ_TILE / (TK * RS)));  // TK*TC*RS <= tile (1x1 layers: 32 x 256)
      ktiles = (K + TK - 1) / TK;
      ctiles = (C + TC - 1) / TC;
      if (t < first + ktiles * ctiles) break;
      first += ktiles * ctiles;
    }
    if (layer >= n_layers) break;
    const i8t_wq_desc d = descs[layer];
    const float clip = *d.clip, s = scale_of(clip), inv_s = 1.0f / s, hs = __fdiv_rn(0.5f, clip);
    const int tl = t - first;
    const int k0 = (tl / ctiles) * TK, c0 = (tl % ctiles) * TC;
    const int nk = min(TK, K - k0), nc = min(TC, C - c0), row = nc * RS;  // row: (c, rs) of one k
    __syncthreads();  // the previous tile's writes have read tq
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (!d.src_krsc) {
      // KCRS rows: (c, rs) contiguous; each warp streams four k rows at once so
      // four independent loads per lane are in flight
      const float* w0 = d.w + static_cast<size_t>(k0) * C * RS + static_cast<size_t>(c0) * RS;
      for (int kb = warp; kb < nk; kb += 32)
        for (int cr = lane; cr < row; cr += 32) {
          float v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int kk = kb + 8 * u;
            v[u] = kk < nk ? __ldg(w0 + static_cast<size_t>(kk) * C * RS + cr) : 0.0f;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int kk = kb + 8 * u;
            if (kk < nk) {
              bad |= !isfinite(v[u]);
              tq[kk * TC * RS + cr] = static_cast<int8_t>(quant_nearest_fast(v[u], clip, hs, s, inv_s));
            }
          }
        }
    } else {
      for (int kk = warp; kk < nk; kk += 8) {  // KRSC rows
        const float* wrow = d.w + static_cast<size_t>(k0 + kk) * RS * C + c0;
        int8_t* trow = tq + kk * TC * RS;
        for (int rs = 0; rs < RS; ++rs)
          for (int cc = lane; cc < nc; cc += 32) {
            const float v = __ldg(wrow + static_cast<size_t>(rs) * C + cc);
            bad |= !isfinite(v);
            trow[cc * RS + rs] = static_cast<int8_t>(quant_nearest_fast(v, clip, hs, s, inv_s));
          }
      }
    }
    __syncthreads();
    // write-out, four bytes per lane (one 32-bit store): the lanes of a warp
    // cover several rows when a row has fewer than 32 quads
    auto put4 = [](int8_t* dst, int n4, const int8_t* src, int stride) {  // n4 = valid bytes (1..4)
      const uint32_t b0 = static_cast<uint8_t>(src[0]);
      const uint32_t b1 = n4 > 1 ? static_cast<uint8_t>(src[stride]) : 0u;
      const uint32_t b2 = n4 > 2 ? static_cast<uint8_t>(src[2 * stride]) : 0u;
      const uint32_t b3 = n4 > 3 ? static_cast<uint8_t>(src[3 * stride]) : 0u;
      if (n4 == 4 && (reinterpret_cast<uintptr_t>(dst) & 3u) == 0) {
        *reinterpret_cast<uint32_t*>(dst) = b0 | (b1 << 8) | (b2 << 16) | (b3 << 24);
      } else {
        dst[0] = static_cast<int8_t>(b0);
        if (n4 > 1) dst[1] = static_cast<int8_t>(b1);
        if (n4 > 2) dst[2] = static_cast<int8_t>(b2);
        if (n4 > 3) dst[3] = static_cast<int8_t>(b3);
      }
    };
    if (d.q_krsc) {  // [k][rs][c]: c along the lanes
      const int q4 = (nc + 3) / 4, lpr = q4 < 32 ? q4 : 32, rpw = 32 / lpr;
      const int sub = lane / lpr, l = lane - sub * lpr;
      if (sub < rpw)
        for (int pr = warp * rpw + sub; pr < nk * RS; pr += 8 * rpw) {
          const int kk = pr / RS, rs = pr - kk * RS;
          int8_t* dst = d.q_krsc + static_cast<size_t>(k0 + kk) * d.ld_krsc + rs * d.c_pad + c0;
          for (int c4 = l; c4 < q4; c4 += lpr)
            put4(dst + 4 * c4, min(4, nc - 4 * c4), tq + kk * TC * RS + 4 * c4 * RS + rs, RS);
        }
    }
    if (d.q_crsk) {  // [c][rs][k]: k along the lanes
      const int q4 = (nk + 3) / 4, lpr = q4 < 32 ? q4 : 32, rpw = 32 / lpr;
      const int sub = lane / lpr, l = lane - sub * lpr;
      if (sub < rpw)
        for (int pr = warp * rpw + sub; pr < nc * RS; pr += 8 * rpw) {
          const int cc = pr / RS, rs = pr - cc * RS;
          int8_t* dst = d.q_crsk + static_cast<size_t>(c0 + cc) * d.ld_crsk + rs * d.k_pad + k0;
          for (int k4 = l; k4 < q4; k4 += lpr)
            put4(dst + 4 * k4, min(4, nk - 4 * k4), tq + 4 * k4 * TC * RS + cc * RS + rs, TC * RS);
        }
    }
  }
  if (bad) atomicOr(err, ERR_NONFINITE);
}

// NCHW float -> NHWC int8 (channel stride c_pad) through a 32x32 smem transpose.
__global__ void __launch_bounds__(256) k_quant_nearest_nchw(const float* __restrict__ x, uint32_t C, uint32_t HW,
                                                            const float* __restrict__ clip_p, int8_t* __restrict__ q,
                                                            uint32_t c_pad, float* amax, int* err) {
  pdl_entry();
  __shared__ float tile[32][33];
  const float clip = *clip_p, s = scale_of(clip), inv_s = 1.0f / s, hs = __fdiv_rn(0.5f, clip);
  const size_t n = blockIdx.z;
  const uint32_t c0 = blockIdx.y * 32, p0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  float m = 0.0f;
  bool bad = false;
  for (int r = ty; r < 32; r += 8) {
    const uint32_t c = c0 + r, p = p0 + tx;
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
    const uint32_t p = p0 + r, c = c0 + tx;
    if (p < HW && c < c_pad)
      q[(n * HW + p) * c_pad + c] = (c < C) ? static_cast<int8_t>(quant_nearest_fast(tile[tx][r], clip, hs, s, inv_s)) : 0;
  }
  if (bad) atomicOr(err, ERR_NONFINITE);
  if (amax) block_amax(m, amax);
}

// K2: weights KCRS (or KRSC) float -> KRSC int8 [K][ld_krsc] and CRSK int8 [C][ld_crsk].
__global__ void __launch_bounds__(256) k_quant_weight(const float* __restrict__ w, int src_krsc, uint32_t K, uint32_t C,
                                                      uint32_t RS, const float* __restrict__ clip_p, int8_t* q_krsc,
                                                      uint32_t c_pad, uint32_t ld_krsc, int8_t* q_crsk, uint32_t k_pad,
                                                      uint32_t ld_crsk, float* amax, int* err) {
  pdl_entry();
  const float clip = *clip_p, s = scale_of(clip), inv_s = 1.0f / s, hs = __fdiv_rn(0.5f, clip);
  const uint32_t tot = K * C * RS;
  float m = 0.0f;
  bool bad = false;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
    uint32_t k, c, rs;
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
    const int8_t qv = static_cast<int8_t>(quant_nearest_fast(v, clip, hs, s, inv_s));
    if (q_krsc) q_krsc[static_cast<size_t>(k) * ld_krsc + rs * c_pad + c] = qv;
    if (q_crsk) q_crsk[static_cast<size_t>(c) * ld_crsk + rs * k_pad + k] = qv;
  }
  if (bad) atomicOr(err, ERR_NONFINITE);
  if (amax) block_amax(m, amax);
}

__global__ void k_dequantize(const int8_t* __restrict__ q, uint32_t n, const float* __restrict__ clip_p,
                             float* __restrict__ out) {
  pdl_entry();
  const float s = scale_of(*clip_p);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = __fmul_rn(static_cast<float>(q[i]), s);
}

// quantize_partitioned (quantize.cpp:45-79): chunk k = [n*k/P, n*(k+1)/P) draws from LcgStream(base+k).
__global__ void k_quant_partitioned(const float* __restrict__ x, int64_t n, const float* __restrict__ clip_p,
                                    uint32_t base_seed, int parts, int8_t* __restrict__ q, int* err) {
  pdl_entry();
  const float clip = *clip_p, s = scale_of(clip), inv_s = 1.0f / s, hs = __fdiv_rn(0.5f, clip);
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = (i * parts) / n;
    while (k + 1 < parts && (n * (k + 1)) / parts <= i) ++k;
    while (k > 0 && (n * k) / parts > i) --k;
    const int64_t lo = (n * k) / parts;
    const uint32_t X = apply(lcg_jump_map(static_cast<uint64_t>(i - lo + 1)), base_seed + static_cast<uint32_t>(k));
    const float v = x[i];
    bad |= !isfinite(v);
    q[i] = static_cast<int8_t>(quant_stoch(v, clip, s, inv_s, X));
  }
  if (bad) atomicOr(err, ERR_NONFINITE);
}

// SGD step (train.cpp:97-117, momentum 0): w -= float(lr * g), lr = base_lr * phi.
__global__ void __launch_bounds__(256) k_sgd_dclr(float* __restrict__ w, const float* __restrict__ grad, uint32_t n,
                                                  double base_lr, const DsgcState* st, const int32_t* skip) {
  pdl_entry();
  if (skip && *skip) return;
  const double lr = st ? base_lr * st->v.lr_scale : base_lr;
  const uint32_t n4 = n / 4, stride = gridDim.x * blockDim.x;
  float4* w4 = reinterpret_cast<float4*>(w);
  const float4* g4 = reinterpret_cast<const float4*>(grad);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 a = w4[i];
    const float4 g = __ldg(g4 + i);
    a.x -= static_cast<float>(lr * static_cast<double>(g.x));
    a.y -= static_cast<float>(lr * static_cast<double>(g.y));
    a.z -= static_cast<float>(lr * static_cast<double>(g.z));
    a.w -= static_cast<float>(lr * static_cast<double>(g.w));
    w4[i] = a;
  }
  for (uint32_t i = n4 * 4 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    w[i] -= static_cast<float>(lr * static_cast<double>(grad[i]));
}

// Segmented SGD+DCLR over flat arenas: one launch for every parameter.
// lr = base_lr (or *lr_dev) * phi_layer; momentum (train.cpp:106-111):
//   buf = float(m*buf + g)  (the reference's GNU build contracts m*buf + g to one FMA)
//   w  -= float(lr*buf)
__device__ __forceinline__ float sgd_elem(float w, float g, float* buf, double lr, double m) {
  if (buf) {
    const float b = static_cast<float>(fma(m, static_cast<double>(*buf), static_cast<double>(g)));
    *buf = b;
    g = b;
  }
  return w - static_cast<float>(lr * static_cast<double>(g));
}

__global__ void __launch_bounds__(256) k_sgd_dclr_multi(float* __restrict__ w, const float* __restrict__ grad,
                                                        int nseg, const int64_t* __restrict__ seg_off,
                                                        const void* const* __restrict__ seg_state, double base_lr,
                                                        const double* __restrict__ lr_dev, const int32_t* skip,
                                                        float* __restrict__ mom, double momentum) {
  pdl_entry();
  if (skip && *skip) return;
  if (lr_dev) base_lr = *lr_dev;
  const int64_t n4 = seg_off[nseg] / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 4;
    int lo = 0, hi = nseg - 1;  // segment with seg_off[s] <= e < seg_off[s+1]
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (seg_off[mid] <= e) lo = mid;
      else hi = mid - 1;
    }
    const DsgcState* st = reinterpret_cast<const DsgcState*>(seg_state[lo]);
    const double lr = st ? base_lr * st->v.lr_scale : base_lr;
    float4 a = reinterpret_cast<float4*>(w)[i];
    const float4 g = __ldg(reinterpret_cast<const float4*>(grad) + i);
    if (mom) {
      float4 b = reinterpret_cast<float4*>(mom)[i];
      a.x = sgd_elem(a.x, g.x, &b.x, lr, momentum);
      a.y = sgd_elem(a.y, g.y, &b.y, lr, momentum);
      a.z = sgd_elem(a.z, g.z, &b.z, lr, momentum);
      a.w = sgd_elem(a.w, g.w, &b.w, lr, momentum);
      reinterpret_cast<float4*>(mom)[i] = b;
    } else {
      a.x = sgd_elem(a.x, g.x, nullptr, lr, 0.0);
      a.y = sgd_elem(a.y, g.y, nullptr, lr, 0.0);
      a.z = sgd_elem(a.z, g.z, nullptr, lr, 0.0);
      a.w = sgd_elem(a.w, g.w, nullptr, lr, 0.0);
    }
    reinterpret_cast<float4*>(w)[i] = a;
  }
}

__global__ void __launch_bounds__(256) k_nonfinite_flag(const float* __restrict__ x, int64_t n, int32_t* flag) {
  pdl_entry();
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n / 4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
    bad |= !isfinite(v.x) || !isfinite(v.y) || !isfinite(v.z) || !isfinite(v.w);
  }
  for (int64_t i = (n / 4) * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

// ---- layout helpers
__global__ void k_nhwc_to_nchw_f32(const float* __restrict__ src, uint32_t C, uint32_t HW, uint32_t ld,
                                   float* __restrict__ dst) {
  pdl_entry();
  __shared__ float tile[32][33];
  const size_t n = blockIdx.z;
  const uint32_t c0 = blockIdx.y * 32, p0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const uint32_t p = p0 + r, c = c0 + tx;
    tile[r][tx] = (p < HW && c < C) ? src[(n * HW + p) * ld + c] : 0.0f;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const uint32_t c = c0 + r, p = p0 + tx;
    if (c < C && p < HW) dst[(n * C + c) * HW + p] = tile[tx][r];
  }
}

__global__ void k_nchw_to_nhwc_i8(const int8_t* __restrict__ src, uint32_t C, uint32_t HW, int8_t* __restrict__ dst,
                                  uint32_t c_pad) {
  pdl_entry();
  const size_t n = blockIdx.z;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < HW * c_pad; i += gridDim.x * blockDim.x) {
    const uint32_t p = i / c_pad, c = i - p * c_pad;
    dst[n * HW * c_pad + i] = (c < C) ? src[(n * C + c) * HW + p] : static_cast<int8_t>(0);
  }
}

__global__ void k_kcrs_relayout_i8(const int8_t* __restrict__ src, uint32_t K, uint32_t C, uint32_t RS, int8_t* dst,
                                   uint32_t pad, uint32_t ld, int to_crsk) {
  pdl_entry();
  const uint32_t tot = K * C * RS;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
    const uint32_t rs = i % RS, c = (i / RS) % C, k = i / (RS * C);
    if (to_crsk) dst[static_cast<size_t>(c) * ld + rs * pad + k] = src[i];
    else dst[static_cast<size_t>(k) * ld + rs * pad + c] = src[i];
  }
}

static int grid_for(int64_t n, int threads = 256, int64_t cap = 148 * 8) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return static_cast<int>(b);
}

static bool too_big(int64_t n) { return n >= (int64_t(1) << 31); }

}  // namespace i8t_dev

using namespace i8t_dev;
#define CTX(c) reinterpret_cast<Ctx*>(c)

extern "C" {

int i8t_quantize_nearest_shared(i8t_ctx* ctx, const float* x, int64_t n, const float* clip, const float* ref_clip,
                                const int8_t* ref_q, const float* ref_amax, int8_t* q, float* amax) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !clip || !ref_clip || !ref_q || !q || n < 0) return set_error(I8T_EINVAL, "quantize: bad arguments");
  if (n == 0) return I8T_OK;
  if (too_big(n)) return set_error(I8T_EUNSUPPORTED, "quantize: tensor >= 2^31 elements");
  if (((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(ref_q)) & 15u))
    return set_error(I8T_EUNSUPPORTED, "quantize_nearest_shared: 16-byte alignment");
  launch_k(k_quant_nearest_share, grid_for(n / 4 + 1), RED_THREADS, 0, c->stream, x, static_cast<uint32_t>(n), clip,
           ref_clip, ref_q, ref_amax, q, amax, c->d_err);
  count_launch(1);
  return cuda_check("k_quant_nearest_share");
}

int i8t_quantize_nearest_rows(i8t_ctx* ctx, const float* x, int64_t rows, int64_t cols, const float* clip, int8_t* q,
                              int64_t ld_q, float* amax, int accumulate_amax) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !clip || !q || rows < 0 || cols < 0 || ld_q < cols) return set_error(I8T_EINVAL, "quantize: bad arguments");
  if (rows * cols == 0) return I8T_OK;
  if (too_big(rows * ld_q)) return set_error(I8T_EUNSUPPORTED, "quantize: tensor >= 2^31 elements");
  if (amax && !accumulate_amax) cudaMemsetAsync(amax, 0, sizeof(float), c->stream);
  if (ld_q == cols) {
    const int64_t n = rows * cols;
    launch_k(k_quant_nearest_flat, grid_for(n / 4 + 1), RED_THREADS, 0, c->stream, x, static_cast<uint32_t>(n), clip, q, amax,
                                                                              c->d_err);
  } else if (cols == 3 && ld_q == 4 && rows % 4 == 0 &&
             ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(q)) & 15u) == 0) {
    launch_k(k_quant_nearest_rgb, grid_for(rows / 4), RED_THREADS, 0, c->stream, reinterpret_cast<const float4*>(x),
             static_cast<uint32_t>(rows / 4), clip, reinterpret_cast<uint4*>(q), amax, c->d_err);
  } else {
    launch_k(k_quant_nearest_rows, grid_for(rows * ld_q), RED_THREADS, 0, c->stream, 
        x, static_cast<uint32_t>(rows), static_cast<uint32_t>(cols), clip, q, static_cast<uint32_t>(ld_q), amax, c->d_err);
  }
  count_launch(1);
  return cuda_check("k_quant_nearest");
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
  dim3 grid(static_cast<unsigned>((hw + 31) / 32), static_cast<unsigned>((c_pad + 31) / 32), static_cast<unsigned>(n));
  launch_k(k_quant_nearest_nchw, grid, 256, 0, cx->stream, x, static_cast<uint32_t>(c), static_cast<uint32_t>(hw), clip, q,
                                                      static_cast<uint32_t>(c_pad), amax, cx->d_err);
  count_launch(1);
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
  launch_k(k_quant_weight, grid_for(k * c * kh * kw), 256, 0, cx->stream, 
      w, src_krsc, static_cast<uint32_t>(k), static_cast<uint32_t>(c), static_cast<uint32_t>(kh * kw), clip, q_krsc,
      static_cast<uint32_t>(c_pad), static_cast<uint32_t>(ld_krsc), q_crsk, static_cast<uint32_t>(k_pad),
      static_cast<uint32_t>(ld_crsk), amax, cx->d_err);
  count_launch(1);
  return cuda_check("k_quant_weight");
}

int i8t_quantize_weights_multi(i8t_ctx* ctx, const i8t_wq_desc* dev_descs, int n_layers) {
  Ctx* cx = CTX(ctx);
  if (!cx || !dev_descs || n_layers < 1 || n_layers > 65535) return set_error(I8T_EINVAL, "quantize_weights_multi: bad arguments");
  launch_k(k_quant_weight_multi, 148 * 4, 256, 0, cx->stream, dev_descs, n_layers, cx->d_err);
  count_launch(1);
  return cuda_check("k_quant_weight_multi");
}

int i8t_dequantize(i8t_ctx* ctx, const int8_t* q, int64_t n, const float* clip, float* out) {
  Ctx* c = CTX(ctx);
  if (!c || !q || !clip || !out) return set_error(I8T_EINVAL, "dequantize: bad arguments");
  if (!n) return I8T_OK;
  launch_k(k_dequantize, grid_for(n), 256, 0, c->stream, q, static_cast<uint32_t>(n), clip, out);
  count_launch(1);
  return cuda_check("k_dequantize");
}

int i8t_quantize_partitioned(i8t_ctx* ctx, const float* x, int64_t n, const float* clip, uint32_t base_seed, int parts,
                             int8_t* q) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !clip || !q) return set_error(I8T_EINVAL, "quantize_partitioned: bad arguments");
  if (parts < 1) return set_error(I8T_EINVAL, "quantize_partitioned: partitions must be >= 1");
  if (n == 0) return I8T_OK;
  launch_k(k_quant_partitioned, grid_for(n), 256, 0, c->stream, x, n, clip, base_seed, parts, q, c->d_err);
  count_launch(1);
  return cuda_check("k_quant_partitioned");
}

int i8t_sgd_dclr(i8t_ctx* ctx, float* w, const float* grad, int64_t n, double base_lr, const void* state,
                 const int32_t* skip) {
  Ctx* c = CTX(ctx);
  if (!c || !w || !grad) return set_error(I8T_EINVAL, "sgd: bad arguments");
  if (!n) return I8T_OK;
  if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(grad)) & 15u)
    return set_error(I8T_EUNSUPPORTED, "sgd: pointers must be 16-byte aligned");
  launch_k(k_sgd_dclr, grid_for(n / 4 + 1), 256, 0, c->stream, w, grad, static_cast<uint32_t>(n), base_lr,
                                                          reinterpret_cast<const DsgcState*>(state), skip);
  count_launch(1);
  return cuda_check("k_sgd_dclr");
}

int i8t_sgd_dclr_multi(i8t_ctx* ctx, float* w, const float* grad, int nseg, const int64_t* seg_off,
                       const void* const* seg_state, double base_lr, const double* lr_dev, const int32_t* skip,
                       float* mom, double momentum) {
  Ctx* c = CTX(ctx);
  if (!c || !w || !grad || nseg < 1 || !seg_off || !seg_state) return set_error(I8T_EINVAL, "sgd_multi: bad arguments");
  if ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(grad)) & 15u)
    return set_error(I8T_EUNSUPPORTED, "sgd_multi: arenas must be 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(mom) & 15u) return set_error(I8T_EUNSUPPORTED, "sgd_multi: momentum arena must be 16-byte aligned");
  launch_k(k_sgd_dclr_multi, 148 * 8, 256, 0, c->stream, w, grad, nseg, seg_off, seg_state, base_lr, lr_dev, skip,
           mom, momentum);
  count_launch(1);
  return cuda_check("k_sgd_dclr_multi");
}

int i8t_nonfinite_flag(i8t_ctx* ctx, const float* x, int64_t n, int32_t* flag) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !flag) return set_error(I8T_EINVAL, "nonfinite_flag: bad arguments");
  if (reinterpret_cast<uintptr_t>(x) & 15u) return set_error(I8T_EUNSUPPORTED, "nonfinite_flag: 16-byte alignment");
  cudaMemsetAsync(flag, 0, sizeof(int32_t), c->stream);
  launch_k(k_nonfinite_flag, 148 * 4, 256, 0, c->stream, x, n, flag);
  count_launch(1);
  return cuda_check("k_nonfinite_flag");
}

int i8t_nhwc_to_nchw_f32(i8t_ctx* ctx, const float* src, int64_t n, int64_t c, int64_t hw, int64_t ld, float* dst) {
  Ctx* cx = CTX(ctx);
  if (!cx || !src || !dst || ld < c) return set_error(I8T_EINVAL, "nhwc_to_nchw: bad arguments");
  if (n * c * hw == 0) return I8T_OK;
  dim3 grid(static_cast<unsigned>((hw + 31) / 32), static_cast<unsigned>((c + 31) / 32), static_cast<unsigned>(n));
  launch_k(k_nhwc_to_nchw_f32, grid, 256, 0, cx->stream, src, static_cast<uint32_t>(c), static_cast<uint32_t>(hw),
                                                    static_cast<uint32_t>(ld), dst);
  count_launch(1);
  return cuda_check("k_nhwc_to_nchw_f32");
}

// im2col_i8 / im2col_channel_i8 (conv.cpp:23-47, 98-106): channels [c_lo,
// c_hi) of an NCHW int8 tensor -> col[((c-c_lo)*kh + i)*kw + j][(n*oh + p)*ow + q],
// zero where the tap falls into the padding.  One thread per output byte,
// consecutive threads along q: the col row writes are coalesced.
static __global__ void k_im2col_i8(const int8_t* __restrict__ x, i8t_conv_geom g, int64_t oh, int64_t ow, int64_t c_lo,
                                   int64_t rows, int8_t* __restrict__ col) {
  pdl_entry();
  const int64_t cols = g.n * oh * ow, total = rows * cols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = e / cols, m = e - r * cols;
    const int64_t j = r % g.kw, i = (r / g.kw) % g.kh, c = c_lo + r / (g.kw * g.kh);
    const int64_t q = m % ow, p = (m / ow) % oh, n = m / (ow * oh);
    const int64_t y = p * g.stride_h + i - g.pad_h, xx = q * g.stride_w + j - g.pad_w;
    col[e] = (y >= 0 && y < g.h && xx >= 0 && xx < g.w) ? x[((n * g.c + c) * g.h + y) * g.w + xx] : int8_t(0);
  }
}

int i8t_im2col_s8(i8t_ctx* ctx, const int8_t* x, const i8t_conv_geom* g, int64_t c_lo, int64_t c_hi, int8_t* col) {
  Ctx* cx = CTX(ctx);
  if (!cx || !x || !g || !col || c_lo < 0 || c_hi > g->c || c_lo >= c_hi) return set_error(I8T_EINVAL, "im2col: bad arguments");
  const int64_t oh = (g->h + 2 * g->pad_h - g->kh) / g->stride_h + 1, ow = (g->w + 2 * g->pad_w - g->kw) / g->stride_w + 1;
  if (oh < 1 || ow < 1) return set_error(I8T_EINVAL, "im2col: empty output");
  const int64_t rows = (c_hi - c_lo) * g->kh * g->kw;
  launch_k(k_im2col_i8, grid_for(rows * g->n * oh * ow), 256, 0, cx->stream, x, *g, oh, ow, c_lo, rows, col);
  count_launch(1);
  return cuda_check("k_im2col_i8");
}

int i8t_nchw_to_nhwc_i8(i8t_ctx* ctx, const int8_t* src, int64_t n, int64_t c, int64_t hw, int8_t* dst, int64_t c_pad) {
  Ctx* cx = CTX(ctx);
  if (!cx || !src || !dst || c_pad < c) return set_error(I8T_EINVAL, "nchw_to_nhwc: bad arguments");
  if (!n) return I8T_OK;
  dim3 grid(static_cast<unsigned>(grid_for(hw * c_pad, 256, 1024)), 1, static_cast<unsigned>(n));
  launch_k(k_nchw_to_nhwc_i8, grid, 256, 0, cx->stream, src, static_cast<uint32_t>(c), static_cast<uint32_t>(hw), dst,
                                                   static_cast<uint32_t>(c_pad));
  count_launch(1);
  return cuda_check("k_nchw_to_nhwc_i8");
}

int i8t_kcrs_to_krsc_i8(i8t_ctx* ctx, const int8_t* src, int64_t k, int64_t c, int64_t kh, int64_t kw, int8_t* dst,
                        int64_t c_pad, int64_t ld) {
  Ctx* cx = CTX(ctx);
  if (!cx || !src || !dst || c_pad < c || ld < kh * kw * c_pad) return set_error(I8T_EINVAL, "kcrs_to_krsc: bad arguments");
  cudaMemsetAsync(dst, 0, k * ld, cx->stream);
  launch_k(k_kcrs_relayout_i8, grid_for(k * c * kh * kw), 256, 0, cx->stream, 
      src, static_cast<uint32_t>(k), static_cast<uint32_t>(c), static_cast<uint32_t>(kh * kw), dst,
      static_cast<uint32_t>(c_pad), static_cast<uint32_t>(ld), 0);
  count_launch(1);
  return cuda_check("k_kcrs_relayout_i8");
}

int i8t_kcrs_to_crsk_i8(i8t_ctx* ctx, const int8_t* src, int64_t k, int64_t c, int64_t kh, int64_t kw, int8_t* dst,
                        int64_t k_pad, int64_t ld) {
  Ctx* cx = CTX(ctx);
  if (!cx || !src || !dst || k_pad < k || ld < kh * kw * k_pad) return set_error(I8T_EINVAL, "kcrs_to_crsk: bad arguments");
  cudaMemsetAsync(dst, 0, c * ld, cx->stream);
  launch_k(k_kcrs_relayout_i8, grid_for(k * c * kh * kw), 256, 0, cx->stream, 
      src, static_cast<uint32_t>(k), static_cast<uint32_t>(c), static_cast<uint32_t>(kh * kw), dst,
      static_cast<uint32_t>(k_pad), static_cast<uint32_t>(ld), 1);
  count_launch(1);
  return cuda_check("k_kcrs_relayout_i8");
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
