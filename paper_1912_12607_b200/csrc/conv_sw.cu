// conv_sw.cu -- stride-1 R x S (<= 3 x 3) convolutions, forward and
// backward-data, as "shifted-window" implicit GEMMs on tcgen05 kind::i8.
//
// The im2col gather of conv_tc.cu re-reads every input pixel R*S times from
// L2.  Here a CTA tile is 16 x 8 output pixels (M = 128); its input halo of
// (16+R-1) x (8+S-1) pixels x 64 channels is loaded ONCE by one TMA 4-D box
// (zero fill = the padding) as 64-byte pixel rows with the 64B swizzle,
//     halo[pixel = y*HW + x][64 B],
// and the A operand of tap (r, s) is the same smem with the descriptor start
// moved by (r*HW + s) pixels (+32 B for the second K=32 MMA): an 8-pixel
// output row is 8 consecutive halo rows, the next output row is HW pixels
// further (SBO = HW*64).  The swizzle is a function of the absolute smem
// address (descriptor base offset 0), which is what makes the row-shifted view
// legal -- checked bit-exact against the oracle in tests/test_gpu_conv.py.
// The weights of the CTA's n-tile (BN rows x R*S*C bytes, no-swizzle K-major
// 16-byte core-matrix columns) are loaded once per CTA and stay resident, so
// the main loop streams only halos.
//
//   FWD   z[n,p,q,k]  = sum_{r,s,c} a[n, p+r-ph, q+s-pw, c] * W_krsc[k][(r,s,c)]
//   DGRAD gA[n,h,w,c] = sum_{r,s,k} gz[n, h+ph-r, w+pw-s, k] * W_crsk[c][(r,s,k)]
// (DGRAD = the same kernel on gz with the taps mirrored: halo origin
//  (h0+ph-R+1, w0+pw-S+1), tap (r,s) at halo offset (R-1-r, S-1-s).)
//
// Warp roles (persistent CTA, one per SM): warp 0 lane 0 = TMA producer,
// warp 1 lane 0 = MMA issuer (double-buffered TMEM accumulator), warps 2..9 =
// epilogue: FP64 rescale float(double(s_x)*double(s_y)*acc) (conv.cpp:139-143,
// 201-203), 32x32 fp32 sub-tiles through swizzled smem, 4-D TMA stores that
// clip the tile overhang at the image border.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "internal.cuh"
#include "ptx.cuh"

namespace i8t_dev {

namespace sw {

constexpr int TH = 16, TW = 8;  // output tile (rows x cols) = 128 GEMM rows
constexpr int CC = 64;          // reduction channels per halo (4 x 16-byte K chunks)
constexpr int NH = 4;           // halo ring depth
constexpr int MMA_WARP = 1, EPI_WARP0 = 2, NEPI = 256;
constexpr int NTHREADS = 64 + NEPI;  // 320
constexpr int HALO_MAX_PX = (TH + 2) * (TW + 2);  // R, S <= 3
constexpr int HALO_BYTES = ((HALO_MAX_PX * CC + 1023) / 1024) * 1024;
constexpr int EPI_BYTES = 8 * 32 * 128;
constexpr int SMEM_FIXED = NH * HALO_BYTES + EPI_BYTES + 1024 /*align*/ + 256 /*barriers*/;
constexpr int SMEM_MAX = 232448;
constexpr int B_MAX = SMEM_MAX - SMEM_FIXED;

struct Args {
  int N, IH, IW, OH, OW;  // input (halo source) and output spatial dims
  int R, S, HH, HW;       // filter, halo height / width (pixels)
  int oy, ox;             // halo origin relative to the tile origin
  int mirror;             // DGRAD: tap (r, s) at halo offset (R-1-r, S-1-s)
  int ncc;                // reduction chunks of 64 channels
  int tiles_h, tiles_w, n_tiles, Ng;
  int Cred;
  const float* clip_x;
  const float* clip_y;
  int32_t* acc32;       // optional raw accumulators [N*OH*OW][Ng]
};

__device__ __forceinline__ double i32_to_f64(uint32_t x) {
  return __hiloint2double(0x43300000, static_cast<int>(x ^ 0x80000000u)) - 4503601774854144.0;
}

template <int BN, int R, int S, bool MIRROR>
__global__ void __launch_bounds__(NTHREADS, 1) k_conv_sw(const Args a, const __grid_constant__ CUtensorMap tm_in,
                                                         const __grid_constant__ CUtensorMap tm_w,
                                                         const __grid_constant__ CUtensorMap tm_out) {
  pdl_entry();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sHalo = smem;
  uint8_t* sEpi = smem + NH * HALO_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + EPI_BYTES);
  uint64_t* hfull = bars;           // [NH]
  uint64_t* hempty = bars + NH;     // [NH]
  uint64_t* tfull = bars + 2 * NH;  // [2]
  uint64_t* tempty = tfull + 2;     // [2]
  uint64_t* bfull = tempty + 2;     // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);
  uint8_t* sB = sEpi + EPI_BYTES + 256;  // resident weights [R*S][ncc][4][BN][16 B]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int taps = R * S, HWc = TW + S - 1, HHc = TH + R - 1;
  const int spatial = a.N * a.tiles_h * a.tiles_w;
  const int total = spatial * a.n_tiles;
  const int n_tile = blockIdx.x % a.n_tiles;  // fixed per CTA (gridDim.x % n_tiles == 0)
  const int n0 = n_tile * BN;

  if (warp == MMA_WARP) {
    if (lane == 0) {
      for (int i = 0; i < NH; ++i) {
        mbar_init(&hfull[i], 1);
        mbar_init(&hempty[i], 1);
      }
      for (int i = 0; i < 2; ++i) {
        mbar_init(&tfull[i], 1);
        mbar_init(&tempty[i], NEPI);
      }
      mbar_init(bfull, 1);
      fence_mbar_init();
    }
    __syncwarp();
    tmem_alloc(tmem_slot, 2 * BN);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ================================================= TMA producer (one thread): the CTA's
    // weights once, then one halo box per (tile, 64-channel chunk)
    if (lane == 0) {
      tma_prefetch(&tm_w);
      tma_prefetch(&tm_in);
      mbar_arrive_expect_tx(bfull, static_cast<uint32_t>(taps * a.ncc * 4) * BN * 16);
      for (int t = 0; t < taps; ++t)
        for (int cc = 0; cc < a.ncc; ++cc)
          for (int j = 0; j < 4; ++j)
            tma_load_2d(smem_u32(sB + ((t * a.ncc + cc) * 4 + j) * BN * 16), &tm_w, bfull,
                        t * a.Cred + cc * CC + j * 16, n0);
      int hc = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int sp = t / a.n_tiles;
        const int tw = sp % a.tiles_w, th = (sp / a.tiles_w) % a.tiles_h, n = sp / (a.tiles_w * a.tiles_h);
        const int y0 = th * TH + a.oy, x0 = tw * TW + a.ox;
        for (int cc = 0; cc < a.ncc; ++cc, ++hc) {
          const int slot = hc % NH;
          if (hc >= NH) mbar_wait(&hempty[slot], ((hc / NH) - 1) & 1);
          mbar_arrive_expect_tx(&hfull[slot], static_cast<uint32_t>(HHc * HWc) * CC);
          tma_load_4d(smem_u32(sHalo + slot * HALO_BYTES), &tm_in, &hfull[slot], cc * CC, x0, y0, n);
        }
      }
    }
  } else if (warp == MMA_WARP) {
    // ================================================= MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_i8(128, BN, false, false);
      mbar_wait(bfull, 0);
      tc_fence_after();
      // descriptor templates; the per-tap / per-K-chunk offsets are compile-time
      // constants added to the start-address field (>> 4) inside the loop
      const uint64_t a_tmpl = make_sdesc_sw64(0u, HWc * 64, 0u);
      const uint64_t b_tmpl = make_sdesc_interleave(smem_u32(sB), BN * 16, 128);
      int hc = 0, it = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int cc = 0; cc < a.ncc; ++cc, ++hc) {
          const int slot = hc % NH;
          mbar_wait(&hfull[slot], (hc / NH) & 1);
          tc_fence_after();
          const uint64_t a_base = a_tmpl + (smem_u32(sHalo + slot * HALO_BYTES) >> 4);
          const uint64_t b_base = b_tmpl + static_cast<uint64_t>(cc * 4 * BN);  // (cc*4 kchunks * BN*16 B) >> 4
#pragma unroll
          for (int tap = 0; tap < taps; ++tap) {
                    const int r = tap / S, s = tap - r * S;
            const int dy = MIRROR ? R - 1 - r : r, dx = MIRROR ? S - 1 - s : s;
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              const uint32_t aoff = static_cast<uint32_t>((dy * HWc + dx) * 64 + kk * 32);
              const uint64_t ad = a_base + (aoff >> 4);
              const uint64_t bd = b_base + static_cast<uint64_t>(((tap * a.ncc) * 4 + 2 * kk) * BN);  // >> 4 of bytes
              mma_i8(d_tmem, ad, bd, idesc, (cc | tap | kk) != 0 ? 1u : 0u);
            }
          }
          mma_commit(&hempty[slot]);  // halo slot free once these MMAs have read it
        }
        mma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // ================================================= epilogue (warps 2..9)
    const int ew = warp - EPI_WARP0;
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int half = ew >> 2;
    const int row = quad * 32 + lane;  // tile row: output (4*quad + lane/8, lane%8)
    const double rescale =
        static_cast<double>(__fdiv_rn(*a.clip_x, 127.0f)) * static_cast<double>(__fdiv_rn(*a.clip_y, 127.0f));
    const uint32_t stage_s = smem_u32(sEpi + ew * (32 * 128));
    constexpr int HALF = BN / 2;
    constexpr int NCH = HALF / 32;
    int it = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++it) {
      const int sp = t / a.n_tiles;
      const int tw = sp % a.tiles_w, th = (sp / a.tiles_w) % a.tiles_h, n = sp / (a.tiles_w * a.tiles_h);
      const int p0 = th * TH, q0 = tw * TW;
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(acc * BN);
#pragma unroll 1
      for (int ci = 0; ci < NCH; ++ci) {
        const int col = half * HALF + ci * 32;
        uint32_t v[32];
        tmem_ld32(t_row + static_cast<uint32_t>(col), v);
        tmem_ld_wait();
        if (ci == NCH - 1) {
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
        }
        // rescale into registers first, then wait for the previous chunk's
        // store to release the (single) staging tile: the FP64 rescale
        // overlaps the TMA store's read instead of following it
        uint32_t f[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) f[i] = __float_as_uint(static_cast<float>(rescale * i32_to_f64(v[i])));
        if (lane == 0) bulk_wait_read<0>();
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j)
          sts128(stage_s + sw128_offset(static_cast<uint32_t>(lane), static_cast<uint32_t>(j * 16)),
                 make_uint4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]));
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_4d(&tm_out, stage_s, n0 + col, q0, p0 + 4 * quad, n);
          bulk_commit();
        }
        if (a.acc32) {
          const int p = p0 + 4 * quad + (lane >> 3), q = q0 + (lane & 7);
          if (p < a.OH && q < a.OW) {
            int32_t* dst = a.acc32 + ((static_cast<int64_t>(n) * a.OH + p) * a.OW + q) * a.Ng + n0 + col;
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (n0 + col + i < a.Ng) dst[i] = static_cast<int32_t>(v[i]);
          }
        }
        (void)row;
      }
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 2 * BN);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

static int encode(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* base, const cuuint64_t* dims,
                  const cuuint64_t* strides, const cuuint32_t* box, CUtensorMapSwizzle swz, const char* what) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return set_error(I8T_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  CUresult r = fn(m, dt, rank, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(I8T_ECUDA, std::string("conv_sw: tensor map (") + what + ") failed");
  return I8T_OK;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, int R, int S, bool MIRROR>
static int launch(cudaStream_t st, const Args& a, const CUtensorMap& ti, const CUtensorMap& tw, const CUtensorMap& to) {
  const int smem = SMEM_FIXED + R * S * a.ncc * CC * BN;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_conv_sw<BN, R, S, MIRROR>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
    configured = true;
  }
  const int total = a.N * a.tiles_h * a.tiles_w * a.n_tiles;
  int grid = std::min(total, num_sms());
  grid = grid / a.n_tiles * a.n_tiles;
  launch_k(k_conv_sw<BN, R, S, MIRROR>, grid, NTHREADS, smem, st, a, ti, tw, to);
  count_launch(1);
  return cuda_check("k_conv_sw");
}

template <int R, int S, bool MIRROR>
static int launch_bn(cudaStream_t st, const Args& a, int bn, const CUtensorMap& ti, const CUtensorMap& tw,
                     const CUtensorMap& to) {
  if (bn == 64) return launch<64, R, S, MIRROR>(st, a, ti, tw, to);
  if (bn == 128) return launch<128, R, S, MIRROR>(st, a, ti, tw, to);
  return launch<256, R, S, MIRROR>(st, a, ti, tw, to);
}

template <bool MIRROR>
static int launch_rs(cudaStream_t st, const Args& a, int bn, const CUtensorMap& ti, const CUtensorMap& tw,
                     const CUtensorMap& to) {
  if (a.R == 3 && a.S == 3) return launch_bn<3, 3, MIRROR>(st, a, bn, ti, tw, to);
  if (a.R == 1 && a.S == 3) return launch_bn<1, 3, MIRROR>(st, a, bn, ti, tw, to);
  if (a.R == 3 && a.S == 1) return launch_bn<3, 1, MIRROR>(st, a, bn, ti, tw, to);
  return set_error(I8T_EUNSUPPORTED, "conv_sw: filter shape");
}

}  // namespace sw

// Shifted-window launcher (called by i8t_conv_fwd / i8t_conv_dgrad when
// conv_sw_eligible holds).  in: NHWC int8 [N][IH][IW][Cred]; wts: rows of the
// n dimension (KRSC for FWD, CRSK for DGRAD), row stride ldw; out: NHWC fp32
// [N][OH][OW][Ng].
int conv_sw_run(Ctx* c, bool dgrad, const i8t_conv_geom* g, const int8_t* in, int64_t Cred, int IH, int IW,
                const int8_t* wts, int64_t ldw, int Ng, int OH, int OW, const float* clip_x, const float* clip_y,
                float* out, int32_t* acc) {
  using namespace sw;
  Args a{};
  a.N = (int)g->n; a.IH = IH; a.IW = IW; a.OH = OH; a.OW = OW;
  a.R = (int)g->kh; a.S = (int)g->kw;
  a.HH = TH + a.R - 1; a.HW = TW + a.S - 1;
  a.mirror = dgrad ? 1 : 0;
  a.oy = dgrad ? (int)g->pad_h - a.R + 1 : -(int)g->pad_h;
  a.ox = dgrad ? (int)g->pad_w - a.S + 1 : -(int)g->pad_w;
  a.ncc = (int)(Cred / CC);
  a.Cred = (int)Cred;
  a.tiles_h = (OH + TH - 1) / TH; a.tiles_w = (OW + TW - 1) / TW;
  a.Ng = Ng;
  a.clip_x = clip_x; a.clip_y = clip_y; a.acc32 = acc;
  const int bn = Ng <= 64 ? 64 : (Ng <= 128 ? 128 : 256);
  a.n_tiles = (Ng + bn - 1) / bn;
  CUtensorMap ti{}, tw, to;
  {  // input halo source: int8 (C, W, H, N), box {64 B, HW, HH, 1}, SWIZZLE_64B
    cuuint64_t dims[4] = {(cuuint64_t)Cred, (cuuint64_t)IW, (cuuint64_t)IH, (cuuint64_t)g->n};
    cuuint64_t str[3] = {(cuuint64_t)Cred, (cuuint64_t)(Cred * IW), (cuuint64_t)(Cred * IW * IH)};
    cuuint32_t box[4] = {64u, (cuuint32_t)a.HW, (cuuint32_t)a.HH, 1u};
    int rc = encode(&ti, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, in, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B, "input");
    if (rc) return rc;
  }
  {  // weights: int8 [rows][ldw], box {16 B, bn rows}
    cuuint64_t dims[2] = {(cuuint64_t)ldw, (cuuint64_t)Ng};
    cuuint64_t str[1] = {(cuuint64_t)ldw};
    cuuint32_t box[2] = {16u, (cuuint32_t)bn};
    int rc = encode(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, wts, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE, "weights");
    if (rc) return rc;
  }
  {  // output: fp32 (Ng, OW, OH, N), box {32, 8, 4, 1}, SWIZZLE_128B staging
    cuuint64_t dims[4] = {(cuuint64_t)Ng, (cuuint64_t)OW, (cuuint64_t)OH, (cuuint64_t)g->n};
    cuuint64_t str[3] = {(cuuint64_t)Ng * 4, (cuuint64_t)Ng * 4 * OW, (cuuint64_t)Ng * 4 * OW * OH};
    cuuint32_t box[4] = {32u, 8u, 4u, 1u};
    int rc = encode(&to, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, out, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B, "output");
    if (rc) return rc;
  }
  return dgrad ? launch_rs<true>(c->stream, a, bn, ti, tw, to) : launch_rs<false>(c->stream, a, bn, ti, tw, to);
}

// Stride 1, R, S <= 3, 64-channel reduction chunks, resident weights fit in smem,
// feature map large enough that the 16 x 8 tiles waste little.
bool conv_sw_eligible(const i8t_conv_geom* g, int64_t Cred, int Ng, int OH, int OW, const void* in, const void* out,
                      int64_t ldw) {
  static const bool off = getenv("I8T_NO_CONV_SW") != nullptr;
  static const int max_c = [] {  // tuning experiments: widest reduction channel count routed here
    const char* e = getenv("I8T_CONV_SW_MAXC");
    return e ? atoi(e) : 1 << 30;
  }();
  if (off || g->depthwise || g->stride_h != 1 || g->stride_w != 1 || Cred > max_c) return false;
  if (!((g->kh == 3 && g->kw == 3) || (g->kh == 1 && g->kw == 3) || (g->kh == 3 && g->kw == 1))) return false;
  if (Cred % sw::CC != 0 || Ng % 4 != 0 || ldw % 16 != 0) return false;
  if ((reinterpret_cast<uintptr_t>(in) & 15u) || (reinterpret_cast<uintptr_t>(out) & 15u) || !out) return false;
  const int bn = Ng <= 64 ? 64 : (Ng <= 128 ? 128 : 256);
  if (g->kh * g->kw * Cred * bn > sw::B_MAX) return false;
  const double eff = static_cast<double>(OH) * OW /
                     (static_cast<double>((OH + sw::TH - 1) / sw::TH * sw::TH) * ((OW + sw::TW - 1) / sw::TW * sw::TW));
  return eff >= 0.75;
}

}  // namespace i8t_dev
