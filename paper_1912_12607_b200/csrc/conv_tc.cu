// conv_tc.cu -- INT8 convolutions as implicit GEMMs on 5th-gen tensor cores
// (tcgen05.mma.cta_group::1.kind::i8, int32 accumulators in TMEM).
//
//   FWD   D[npq][k]   = sum_{r,s,c} A_im2col[npq][(r,s,c)] * W_krsc[k][(r,s,c)]
//   DGRAD D[nhw][c]   = sum_{r,s,k} G_col2im[nhw][(r,s,k)] * W_crsk[c][(r,s,k)]
//   WGRAD D[(r,s,c)][k] = sum_{npq} A_im2col[npq][(r,s,c)] * G[npq][k]   (split over npq)
//
// One CTA computes a 128 x BN tile.  Eight producer warps gather the operand
// rows (implicit im2col / col2im, zero padding via cp.async zero-fill) straight
// into SWIZZLE_128B shared-memory tiles; a ring of STAGES buffers is handed to
// a single MMA-issuing thread through mbarriers; the MMA thread's
// tcgen05.commit frees a stage; after the last k-tile the same eight warps
// drain TMEM (tcgen05.ld) and apply the reference's FP64 rescale epilogue
// float(double(s_x)*double(s_y)*acc) (conv.cpp:139-143, :190-191, :201-203),
// or, for WGRAD, add the exact int32 split partial into an int64 accumulator.
// FWD/DGRAD operands are K-major; WGRAD operands are MN-major (the reduction
// runs over pixel rows), which tcgen05 supports for int8.
#include <cuda_runtime.h>

#include <cstdio>

#include "internal.cuh"
#include "ptx.cuh"

namespace i8t_dev {

enum ConvMode { MODE_FWD = 0, MODE_DGRAD = 1, MODE_WGRAD = 2 };

struct ConvArgs {
  const int8_t* act;  // NHWC [N][H][W][Cp]
  const int8_t* gz;   // NHWC [N][P][Q][Kp]
  const int8_t* wt;   // FWD: KRSC rows [K][ldw]; DGRAD: CRSK rows [C][ldw]
  int64_t ldw;
  int N, H, W, Cp, Kp, R, S, sh, sw, ph, pw, P, Q;
  int64_t M;      // GEMM rows
  int Ng;         // GEMM cols (valid)
  int64_t Kd;     // reduction length (valid)
  int k_tiles;    // k tiles per CTA
  const float* clip_x;
  const float* clip_y;
  float* out;
  int64_t ldo;
  int32_t* acc32;
  unsigned long long* acc64;
};

constexpr int BM = 128;
constexpr int BKB = 128;  // bytes of reduction per stage (4 MMAs of K=32)
constexpr int NPROD = 256;
constexpr int NTHREADS = NPROD + 32;

template <int MODE, int BN>
struct Cfg {
  static constexpr int STAGES = 4;
  static constexpr int A_BYTES = BM * BKB;  // 16 KB
  // B: K-major [BN rows][128 B] or MN-major [128 rows][128 B] x ceil(BN/128)
  static constexpr int B_SUB = (BN + 127) / 128;
  static constexpr int B_BYTES = (MODE == MODE_WGRAD) ? 128 * 128 * B_SUB : BN * BKB;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t TMEM_COLS = BN < 32 ? 32 : BN;
};

__device__ __forceinline__ int ifloordiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

template <int MODE, int BN, int VA, int VB>
__global__ void __launch_bounds__(NTHREADS, 1) k_conv_tc(const ConvArgs args) {
  using C = Cfg<MODE, BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tmem_full = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t m0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int n0 = blockIdx.y * BN;
  const int kt0 = blockIdx.z * args.k_tiles;  // first k tile of this split
  int nk = args.k_tiles;
  {
    const int64_t total_kt = (args.Kd + BKB - 1) / BKB;
    if (kt0 + nk > total_kt) nk = static_cast<int>(total_kt - kt0);
  }

  if (warp == 8) {
    if (lane == 0) {
      for (int s = 0; s < C::STAGES; ++s) {
        mbar_init(&full[s], NPROD);
        mbar_init(&empty[s], 1);
      }
      mbar_init(tmem_full, 1);
      fence_mbar_init();
    }
    __syncwarp();
    tmem_alloc(tmem_slot, C::TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 8) {
    // ------------------------------------------------ MMA issuer (one thread)
    if (lane == 0 && nk > 0) {
      constexpr bool AMN = (MODE == MODE_WGRAD), BMN = (MODE == MODE_WGRAD);
      constexpr uint32_t idesc = make_idesc_i8(BM, BN, AMN, BMN);
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % C::STAGES;
        mbar_wait(&full[s], (kt / C::STAGES) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BKB / 32; ++kk) {
          uint64_t ad, bd;
          if constexpr (MODE == MODE_WGRAD) {
            // MN-major: 32 reduction rows per MMA = 4096 B; SBO = 8-row atom stride, LBO = 128-col sub-tile stride
            ad = make_sdesc_sw128(a0 + s * C::A_BYTES + kk * 4096, 16384, 1024);
            bd = make_sdesc_sw128(b0 + s * C::B_BYTES + kk * 4096, 16384, 1024);
          } else {
            // K-major: 32 bytes of reduction per MMA inside the 128 B swizzled row; SBO = 8 rows x 128 B
            ad = make_sdesc_sw128(a0 + s * C::A_BYTES + kk * 32, 16, 1024);
            bd = make_sdesc_sw128(b0 + s * C::B_BYTES + kk * 32, 16, 1024);
          }
          mma_i8(tmem_base, ad, bd, idesc, (kt | kk) != 0 ? 1u : 0u);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(tmem_full);
    }
  } else {
    // ------------------------------------------------ producers (warps 0-7)
    constexpr int PPR_A = BKB / VA;                 // pieces per 128 B row
    constexpr int ROWS_PER_PASS_A = NPROD / PPR_A;  // rows covered per pass
    constexpr int PASSES_A = BM / ROWS_PER_PASS_A;
    const int ja = tid % PPR_A, ra0 = tid / PPR_A;

    // per-row precompute for FWD / DGRAD (rows are output/input pixels, fixed per CTA)
    int rowA_n[PASSES_A], rowA_y[PASSES_A], rowA_x[PASSES_A];
    bool rowA_ok[PASSES_A];
    if constexpr (MODE != MODE_WGRAD) {
#pragma unroll
      for (int i = 0; i < PASSES_A; ++i) {
        const int64_t m = m0 + ra0 + i * ROWS_PER_PASS_A;
        rowA_ok[i] = m < args.M;
        const int64_t mm = rowA_ok[i] ? m : 0;
        if constexpr (MODE == MODE_FWD) {
          const int64_t pq = static_cast<int64_t>(args.P) * args.Q;
          const int n = static_cast<int>(mm / pq);
          const int rem = static_cast<int>(mm - static_cast<int64_t>(n) * pq);
          const int p = rem / args.Q, q = rem - (rem / args.Q) * args.Q;
          rowA_n[i] = n;
          rowA_y[i] = p * args.sh - args.ph;
          rowA_x[i] = q * args.sw - args.pw;
        } else {
          const int64_t hw = static_cast<int64_t>(args.H) * args.W;
          const int n = static_cast<int>(mm / hw);
          const int rem = static_cast<int>(mm - static_cast<int64_t>(n) * hw);
          const int h = rem / args.W, w = rem - (rem / args.W) * args.W;
          rowA_n[i] = n;
          rowA_y[i] = h + args.ph;
          rowA_x[i] = w + args.pw;
        }
      }
    }

    constexpr int LAG = C::STAGES - 1;
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % C::STAGES;
      if (kt >= C::STAGES) mbar_wait(&empty[s], ((kt / C::STAGES) - 1) & 1);
      const uint32_t a_st = smem_u32(sA + s * C::A_BYTES);
      const uint32_t b_st = smem_u32(sB + s * C::B_BYTES);
      const int64_t kbase = static_cast<int64_t>(kt0 + kt) * BKB;

      if constexpr (MODE == MODE_FWD || MODE == MODE_DGRAD) {
        // ---- A: implicit im2col (FWD) / col2im gather (DGRAD) rows, K-major
        const int64_t kk = kbase + ja * VA;
        const bool kok = kk < args.Kd;
        const int CH = (MODE == MODE_FWD) ? args.Cp : args.Kp;
        const int tap = kok ? static_cast<int>(kk / CH) : 0;
        const int ch = kok ? static_cast<int>(kk - static_cast<int64_t>(tap) * CH) : 0;
        const int r = tap / args.S, sx = tap - (tap / args.S) * args.S;
#pragma unroll
        for (int i = 0; i < PASSES_A; ++i) {
          const int row = ra0 + i * ROWS_PER_PASS_A;
          bool ok = kok && rowA_ok[i];
          const int8_t* src = args.act;
          if constexpr (MODE == MODE_FWD) {
            const int ih = rowA_y[i] + r, iw = rowA_x[i] + sx;
            ok = ok && ih >= 0 && ih < args.H && iw >= 0 && iw < args.W;
            if (ok) src = args.act + ((static_cast<int64_t>(rowA_n[i]) * args.H + ih) * args.W + iw) * args.Cp + ch;
          } else {
            const int pn = rowA_y[i] - r, qn = rowA_x[i] - sx;
            int p = 0, q = 0;
            if (args.sh == 1) p = pn; else { p = ifloordiv(pn, args.sh); ok = ok && (pn - p * args.sh) == 0; }
            if (args.sw == 1) q = qn; else { q = ifloordiv(qn, args.sw); ok = ok && (qn - q * args.sw) == 0; }
            ok = ok && p >= 0 && p < args.P && q >= 0 && q < args.Q;
            src = args.gz;
            if (ok) src = args.gz + ((static_cast<int64_t>(rowA_n[i]) * args.P + p) * args.Q + q) * args.Kp + ch;
          }
          cp_async_vec<VA>(a_st + sw128_offset(row, ja * VA), src, ok);
        }
        // ---- B: weight rows, K-major (16 B pieces; rows zero-padded to ldw)
        constexpr int PPR_B = BKB / 16;
        constexpr int RPP_B = NPROD / PPR_B;  // 32 rows per pass
        constexpr int PASSES_B = (BN + RPP_B - 1) / RPP_B;
        const int jb = tid % PPR_B, rb0 = tid / PPR_B;
        const int64_t kb = kbase + jb * 16;
#pragma unroll
        for (int i = 0; i < PASSES_B; ++i) {
          const int row = rb0 + i * RPP_B;
          if (row < BN) {
            const int gr = n0 + row;
            const bool ok = gr < args.Ng && kb < args.ldw;
            const int8_t* src = ok ? args.wt + static_cast<int64_t>(gr) * args.ldw + kb : args.wt;
            cp_async16(b_st + sw128_offset(row, jb * 16), src, ok ? 16u : 0u);
          }
        }
      } else {
        // ---- WGRAD: smem rows = npq (reduction), columns = M bytes (A) / N bytes (B), MN-major
        const int64_t pq = static_cast<int64_t>(args.P) * args.Q;
        // A: act im2col^T.  column piece ja -> m = m0 + ja*VA -> (tap, c) fixed per CTA
        const int64_t mA = m0 + ja * VA;
        const bool mok = mA < args.M;
        const int tapA = mok ? static_cast<int>(mA / args.Cp) : 0;
        const int cA = mok ? static_cast<int>(mA - static_cast<int64_t>(tapA) * args.Cp) : 0;
        const int rA = tapA / args.S, sA_ = tapA - (tapA / args.S) * args.S;
#pragma unroll 4
        for (int i = 0; i < PASSES_A; ++i) {
          const int row = ra0 + i * ROWS_PER_PASS_A;
          const int64_t kd = kbase + row;
          bool ok = mok && kd < args.Kd;
          const int8_t* src = args.act;
          if (ok) {
            const int n = static_cast<int>(kd / pq);
            const int rem = static_cast<int>(kd - static_cast<int64_t>(n) * pq);
            const int p = rem / args.Q, q = rem - (rem / args.Q) * args.Q;
            const int ih = p * args.sh - args.ph + rA, iw = q * args.sw - args.pw + sA_;
            ok = ih >= 0 && ih < args.H && iw >= 0 && iw < args.W;
            if (ok) src = args.act + ((static_cast<int64_t>(n) * args.H + ih) * args.W + iw) * args.Cp + cA;
          }
          cp_async_vec<VA>(a_st + sw128_offset(row, ja * VA), src, ok);
        }
        // B: G rows (npq) x BN channel bytes, in 128-column sub-tiles
        constexpr int PPR_B = BKB / VB;
        constexpr int RPP_B = NPROD / PPR_B;
        constexpr int PASSES_B = BM / RPP_B;
        const int jb = tid % PPR_B, rb0 = tid / PPR_B;
#pragma unroll
        for (int sub = 0; sub < C::B_SUB; ++sub) {
          const int col = sub * 128 + jb * VB;
          if (col < BN) {
            const int kch = n0 + col;
            const bool cok = kch < args.Kp;
#pragma unroll 4
            for (int i = 0; i < PASSES_B; ++i) {
              const int row = rb0 + i * RPP_B;
              const int64_t kd = kbase + row;
              const bool ok = cok && kd < args.Kd;
              const int8_t* src = ok ? args.gz + kd * args.Kp + kch : args.gz;
              cp_async_vec<VB>(b_st + sub * 16384 + sw128_offset(row, jb * VB), src, ok);
            }
          }
        }
      }
      cp_async_commit();
      if (kt >= LAG) {
        cp_async_wait<LAG>();
        fence_proxy_async_smem();
        mbar_arrive(&full[(kt - LAG) % C::STAGES]);
      }
    }
    cp_async_wait<0>();
    fence_proxy_async_smem();
    for (int kt = (nk > LAG ? nk - LAG : 0); kt < nk; ++kt) mbar_arrive(&full[kt % C::STAGES]);

    // ------------------------------------------------ epilogue (same 8 warps)
    if (nk > 0) {
      mbar_wait(tmem_full, 0);
      tc_fence_after();
    }
    const int quad = warp & 3, half = warp >> 2;
    const int row = quad * 32 + lane;
    const int64_t m = m0 + row;
    const double rescale =
        static_cast<double>(__fdiv_rn(*args.clip_x, 127.0f)) * static_cast<double>(__fdiv_rn(*args.clip_y, 127.0f));
    constexpr int HALF = BN / 2;
#pragma unroll 1
    for (int cc = 0; cc < HALF; cc += 16) {
      const int col = half * HALF + cc;
      uint32_t v[16];
      if (nk > 0) {
        tmem_ld16(tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(col), v);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = 0;
      }
      if (m >= args.M) continue;
      if constexpr (MODE == MODE_WGRAD) {
        unsigned long long* dst = args.acc64 + m * args.Ng;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int gc = n0 + col + i;
          const int32_t a = static_cast<int32_t>(v[i]);
          if (gc < args.Ng && a != 0) atomicAdd(dst + gc, static_cast<unsigned long long>(static_cast<long long>(a)));
        }
      } else {
        const int gc0 = n0 + col;
        if (args.out) {
          float* dst = args.out + m * args.ldo + gc0;
          if (gc0 + 16 <= args.Ng && (args.ldo % 4) == 0 && (gc0 % 4) == 0) {
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
              float4 f;
              f.x = static_cast<float>(rescale * static_cast<double>(static_cast<int32_t>(v[i + 0])));
              f.y = static_cast<float>(rescale * static_cast<double>(static_cast<int32_t>(v[i + 1])));
              f.z = static_cast<float>(rescale * static_cast<double>(static_cast<int32_t>(v[i + 2])));
              f.w = static_cast<float>(rescale * static_cast<double>(static_cast<int32_t>(v[i + 3])));
              *reinterpret_cast<float4*>(dst + i) = f;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              if (gc0 + i < args.Ng) dst[i] = static_cast<float>(rescale * static_cast<double>(static_cast<int32_t>(v[i])));
          }
        }
        if (args.acc32) {
          int32_t* dst = args.acc32 + m * args.Ng + gc0;
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (gc0 + i < args.Ng) dst[i] = static_cast<int32_t>(v[i]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// WGRAD finalize: int64 acc [(r,s,c_pad)][K] -> float KCRS or KRSC, reference rescale.
__global__ void k_wgrad_finalize(const long long* __restrict__ acc, int K, int C, int Cp, int RS,
                                 const float* clip_g, const float* clip_a, float* __restrict__ gw, int out_kcrs) {
  const double rescale =
      static_cast<double>(__fdiv_rn(*clip_g, 127.0f)) * static_cast<double>(__fdiv_rn(*clip_a, 127.0f));
  const int64_t tot = static_cast<int64_t>(K) * C * RS;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    int k, c, rs;
    if (out_kcrs) {
      rs = static_cast<int>(i % RS);
      c = static_cast<int>((i / RS) % C);
      k = static_cast<int>(i / (static_cast<int64_t>(RS) * C));
    } else {
      c = static_cast<int>(i % C);
      rs = static_cast<int>((i / C) % RS);
      k = static_cast<int>(i / (static_cast<int64_t>(C) * RS));
    }
    const long long a = acc[(static_cast<int64_t>(rs) * Cp + c) * K + k];
    gw[i] = static_cast<float>(rescale * static_cast<double>(a));
  }
}

__global__ void k_transpose_i8(const int8_t* __restrict__ src, int64_t rows, int64_t cols, int8_t* __restrict__ dst,
                               int64_t ld_dst) {
  const int64_t tot = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    dst[c * ld_dst + r] = src[i];
  }
}

__global__ void k_pad_rows_i8(const int8_t* __restrict__ src, int64_t rows, int64_t cols, int8_t* __restrict__ dst,
                              int64_t ld_dst) {
  const int64_t tot = rows * ld_dst;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ld_dst, c = i - r * ld_dst;
    dst[i] = c < cols ? src[r * cols + c] : (int8_t)0;
  }
}

// ---------------------------------------------------------------- host side
static int vec_of(int64_t ch) { return (ch % 16 == 0) ? 16 : (ch % 8 == 0) ? 8 : 4; }

template <int MODE, int BN, int VA, int VB>
static int launch_one(cudaStream_t st, const ConvArgs& a, dim3 grid) {
  using C = Cfg<MODE, BN>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_conv_tc<MODE, BN, VA, VB>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    configured = true;
  }
  k_conv_tc<MODE, BN, VA, VB><<<grid, NTHREADS, C::SMEM, st>>>(a);
  count_launch(1);
  return cuda_check("k_conv_tc");
}

template <int MODE, int BN>
static int dispatch_vec(cudaStream_t st, const ConvArgs& a, dim3 grid, int va, int vb) {
  if constexpr (MODE == MODE_WGRAD) {
    if (vb == 16) {
      if (va == 16) return launch_one<MODE, BN, 16, 16>(st, a, grid);
      if (va == 8) return launch_one<MODE, BN, 8, 16>(st, a, grid);
      return launch_one<MODE, BN, 4, 16>(st, a, grid);
    }
    if (vb == 8) {
      if (va == 16) return launch_one<MODE, BN, 16, 8>(st, a, grid);
      if (va == 8) return launch_one<MODE, BN, 8, 8>(st, a, grid);
      return launch_one<MODE, BN, 4, 8>(st, a, grid);
    }
    if (va == 16) return launch_one<MODE, BN, 16, 4>(st, a, grid);
    if (va == 8) return launch_one<MODE, BN, 8, 4>(st, a, grid);
    return launch_one<MODE, BN, 4, 4>(st, a, grid);
  } else {
    if (va == 16) return launch_one<MODE, BN, 16, 16>(st, a, grid);
    if (va == 8) return launch_one<MODE, BN, 8, 16>(st, a, grid);
    return launch_one<MODE, BN, 4, 16>(st, a, grid);
  }
}

template <int MODE>
static int dispatch(cudaStream_t st, const ConvArgs& a, int bn, dim3 grid, int va, int vb) {
  if (bn == 64) return dispatch_vec<MODE, 64>(st, a, grid, va, vb);
  if (bn == 128) return dispatch_vec<MODE, 128>(st, a, grid, va, vb);
  return dispatch_vec<MODE, 256>(st, a, grid, va, vb);
}

static int pick_bn(int64_t ng) { return ng <= 64 ? 64 : (ng <= 128 ? 128 : 256); }

static int geom_common(const i8t_conv_geom* g, int64_t& P, int64_t& Q) {
  if (!g) return set_error(I8T_EINVAL, "conv: null geometry");
  if (g->n < 1 || g->c < 1 || g->h < 1 || g->w < 1 || g->k < 1 || g->kh < 1 || g->kw < 1 || g->stride_h < 1 ||
      g->stride_w < 1 || g->pad_h < 0 || g->pad_w < 0)
    return set_error(I8T_EINVAL, "ConvGeometry: extents must be positive, pad nonnegative");
  if (g->depthwise && g->k != g->c) return set_error(I8T_EINVAL, "ConvGeometry: depthwise requires k == c");
  if (g->h + 2 * g->pad_h < g->kh || g->w + 2 * g->pad_w < g->kw)
    return set_error(I8T_EINVAL, "ConvGeometry: output size is not a positive integer");
  if (!g->floor_mode && ((g->h + 2 * g->pad_h - g->kh) % g->stride_h != 0 || (g->w + 2 * g->pad_w - g->kw) % g->stride_w != 0))
    return set_error(I8T_EINVAL, "ConvGeometry: output size is not a positive integer");
  P = (g->h + 2 * g->pad_h - g->kh) / g->stride_h + 1;
  Q = (g->w + 2 * g->pad_w - g->kw) / g->stride_w + 1;
  if (g->n * g->h * g->w > (int64_t)1 << 31 || g->n * P * Q > (int64_t)1 << 31)
    return set_error(I8T_EUNSUPPORTED, "conv: tensor too large");
  return I8T_OK;
}

}  // namespace i8t_dev

using namespace i8t_dev;

extern "C" {

int i8t_conv_fwd(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* a, int64_t c_pad, const int8_t* w, int64_t ld_w,
                 const float* clip_a, const float* clip_w, float* z, int32_t* acc) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  int64_t P, Q;
  int rc = geom_common(g, P, Q);
  if (rc) return rc;
  if (!c || !a || !w || !clip_a || !clip_w) return set_error(I8T_EINVAL, "conv_fwd: null argument");
  if (g->depthwise) return set_error(I8T_EINVAL, "conv_fwd: use i8t_conv_dw_fwd for depthwise");
  if (c_pad < g->c || c_pad % 4 != 0) return set_error(I8T_EUNSUPPORTED, "conv_fwd: c_pad must be >= c and a multiple of 4");
  const int64_t Kd = g->kh * g->kw * c_pad;
  if (ld_w < Kd || ld_w % 16 != 0) return set_error(I8T_EUNSUPPORTED, "conv_fwd: ld_w must be >= kh*kw*c_pad and a multiple of 16");
  if (g->kh * g->kw * g->c > 130000) return set_error(I8T_EINVAL, "conv: reduction depth exceeds i32 overflow bound");
  ConvArgs x{};
  x.act = a; x.gz = nullptr; x.wt = w; x.ldw = ld_w;
  x.N = (int)g->n; x.H = (int)g->h; x.W = (int)g->w; x.Cp = (int)c_pad; x.Kp = (int)g->k;
  x.R = (int)g->kh; x.S = (int)g->kw; x.sh = (int)g->stride_h; x.sw = (int)g->stride_w; x.ph = (int)g->pad_h; x.pw = (int)g->pad_w;
  x.P = (int)P; x.Q = (int)Q;
  x.M = g->n * P * Q; x.Ng = (int)g->k; x.Kd = Kd;
  x.k_tiles = (int)((Kd + BKB - 1) / BKB);
  x.clip_x = clip_a; x.clip_y = clip_w; x.out = z; x.ldo = g->k; x.acc32 = acc;
  const int bn = pick_bn(g->k);
  dim3 grid((unsigned)((x.M + BM - 1) / BM), (unsigned)((g->k + bn - 1) / bn), 1);
  return dispatch<MODE_FWD>(c->stream, x, bn, grid, vec_of(c_pad), 16);
}

int i8t_conv_dgrad(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, int64_t k_pad, const int8_t* wt, int64_t ld_wt,
                   const float* clip_g, const float* clip_w, float* ga, int32_t* acc) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  int64_t P, Q;
  int rc = geom_common(g, P, Q);
  if (rc) return rc;
  if (!c || !gz || !wt || !clip_g || !clip_w) return set_error(I8T_EINVAL, "conv_dgrad: null argument");
  if (g->depthwise) return set_error(I8T_EINVAL, "conv_dgrad: use i8t_conv_dw_dgrad for depthwise");
  if (k_pad < g->k || k_pad % 4 != 0) return set_error(I8T_EUNSUPPORTED, "conv_dgrad: k_pad must be >= k and a multiple of 4");
  const int64_t Kd = g->kh * g->kw * k_pad;
  if (ld_wt < Kd || ld_wt % 16 != 0) return set_error(I8T_EUNSUPPORTED, "conv_dgrad: ld_wt must be >= kh*kw*k_pad, multiple of 16");
  if (g->k > 130000) return set_error(I8T_EINVAL, "conv: reduction depth exceeds i32 overflow bound");
  if (g->k * g->kh * g->kw > 133000) return set_error(I8T_EUNSUPPORTED, "conv_dgrad: int32 accumulator bound");
  ConvArgs x{};
  x.act = nullptr; x.gz = gz; x.wt = wt; x.ldw = ld_wt;
  x.N = (int)g->n; x.H = (int)g->h; x.W = (int)g->w; x.Cp = (int)g->c; x.Kp = (int)k_pad;
  x.R = (int)g->kh; x.S = (int)g->kw; x.sh = (int)g->stride_h; x.sw = (int)g->stride_w; x.ph = (int)g->pad_h; x.pw = (int)g->pad_w;
  x.P = (int)P; x.Q = (int)Q;
  x.M = g->n * g->h * g->w; x.Ng = (int)g->c; x.Kd = Kd;
  x.k_tiles = (int)((Kd + BKB - 1) / BKB);
  x.clip_x = clip_g; x.clip_y = clip_w; x.out = ga; x.ldo = g->c; x.acc32 = acc;
  const int bn = pick_bn(g->c);
  dim3 grid((unsigned)((x.M + BM - 1) / BM), (unsigned)((g->c + bn - 1) / bn), 1);
  return dispatch<MODE_DGRAD>(c->stream, x, bn, grid, vec_of(k_pad), 16);
}

int i8t_conv_wgrad(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, int64_t k_pad, const int8_t* a, int64_t c_pad,
                   const float* clip_g, const float* clip_a, int64_t* acc, float* gw, int out_kcrs) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  int64_t P, Q;
  int rc = geom_common(g, P, Q);
  if (rc) return rc;
  if (!c || !gz || !a || !clip_g || !clip_a || !acc) return set_error(I8T_EINVAL, "conv_wgrad: null argument");
  if (g->depthwise) return set_error(I8T_EINVAL, "conv_wgrad: use i8t_conv_dw_wgrad for depthwise");
  if (c_pad < g->c || c_pad % 4 != 0 || k_pad < g->k || k_pad % 4 != 0)
    return set_error(I8T_EUNSUPPORTED, "conv_wgrad: channel strides must be multiples of 4");
  ConvArgs x{};
  x.act = a; x.gz = gz; x.wt = nullptr; x.ldw = 0;
  x.N = (int)g->n; x.H = (int)g->h; x.W = (int)g->w; x.Cp = (int)c_pad; x.Kp = (int)k_pad;
  x.R = (int)g->kh; x.S = (int)g->kw; x.sh = (int)g->stride_h; x.sw = (int)g->stride_w; x.ph = (int)g->pad_h; x.pw = (int)g->pad_w;
  x.P = (int)P; x.Q = (int)Q;
  x.M = g->kh * g->kw * c_pad; x.Ng = (int)g->k; x.Kd = g->n * P * Q;
  const int bn = pick_bn(g->k);
  const int64_t m_tiles = (x.M + BM - 1) / BM, n_tiles = (g->k + bn - 1) / bn;
  const int64_t total_kt = (x.Kd + BKB - 1) / BKB;
  // split the npq reduction: <= 1015 k-tiles (129,920 rows) per split keeps each int32 partial exact,
  // and enough splits to give ~2 CTAs per SM.
  int64_t splits = (2 * 148 + m_tiles * n_tiles - 1) / (m_tiles * n_tiles);
  if (splits < 1) splits = 1;
  int64_t per = (total_kt + splits - 1) / splits;
  if (per > 1015) per = 1015;
  if (per < 4 && total_kt >= 4) per = 4;
  splits = (total_kt + per - 1) / per;
  x.k_tiles = (int)per;
  x.acc64 = reinterpret_cast<unsigned long long*>(acc);
  x.clip_x = clip_g; x.clip_y = clip_a;
  cudaMemsetAsync(acc, 0, sizeof(int64_t) * x.M * g->k, c->stream);
  dim3 grid((unsigned)m_tiles, (unsigned)n_tiles, (unsigned)splits);
  rc = dispatch<MODE_WGRAD>(c->stream, x, bn, grid, vec_of(c_pad), vec_of(k_pad));
  if (rc) return rc;
  if (gw) {
    const int64_t tot = g->k * g->c * g->kh * g->kw;
    int blocks = (int)((tot + 255) / 256);
    if (blocks > 4096) blocks = 4096;
    k_wgrad_finalize<<<blocks, 256, 0, c->stream>>>(reinterpret_cast<const long long*>(acc), (int)g->k, (int)g->c,
                                                     (int)c_pad, (int)(g->kh * g->kw), clip_g, clip_a, gw, out_kcrs);
    count_launch(1);
    return cuda_check("k_wgrad_finalize");
  }
  return I8T_OK;
}

int i8t_conv_wgrad_finalize(i8t_ctx* ctx, const i8t_conv_geom* g, const int64_t* acc, int64_t c_pad,
                            const float* clip_g, const float* clip_a, float* gw, int out_kcrs) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  int64_t P, Q;
  int rc = geom_common(g, P, Q);
  if (rc) return rc;
  if (!c || !acc || !gw || !clip_g || !clip_a || c_pad < g->c) return set_error(I8T_EINVAL, "wgrad_finalize: bad arguments");
  const int64_t tot = g->k * g->c * g->kh * g->kw;
  int blocks = (int)((tot + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  k_wgrad_finalize<<<blocks, 256, 0, c->stream>>>(reinterpret_cast<const long long*>(acc), (int)g->k, (int)g->c,
                                                   (int)c_pad, (int)(g->kh * g->kw), clip_g, clip_a, gw, out_kcrs);
  count_launch(1);
  return cuda_check("k_wgrad_finalize");
}

// gemm_i8 as a 1x1 convolution: A [m][k] = NHWC activations (N=m, H=W=1, C=k),
// B^T [n][k] = KRSC weights.  Temporaries come from the context scratch.
int i8t_gemm_s8(i8t_ctx* ctx, const int8_t* a, const int8_t* b, int64_t m, int64_t k, int64_t n, int32_t* cout) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !a || !b || !cout || m < 1 || k < 1 || n < 1) return set_error(I8T_EINVAL, "gemm_i8: bad arguments");
  if (k > 130000) return set_error(I8T_EINVAL, "gemm_i8: depth exceeds i32 overflow bound");
  const int64_t kp = (k + 3) / 4 * 4, ldw = (kp + 15) / 16 * 16;
  const size_t need_a = (kp == k) ? 0 : (size_t)(m * kp), need_b = (size_t)(n * ldw);
  uint8_t* scratch = reinterpret_cast<uint8_t*>(ensure_scratch(c, need_a + need_b + 4096 + 256));
  if (!scratch) return set_error(I8T_ECUDA, "gemm_i8: scratch alloc failed");
  float* ones = reinterpret_cast<float*>(scratch);  // clip 127 -> scale 1 for both operands
  int8_t* bt = reinterpret_cast<int8_t*>(scratch + 256);
  int8_t* ap = need_a ? bt + need_b : nullptr;
  const float h127[2] = {127.0f, 127.0f};
  cudaMemcpyAsync(ones, h127, sizeof(h127), cudaMemcpyHostToDevice, c->stream);
  cudaMemsetAsync(bt, 0, need_b, c->stream);
  k_transpose_i8<<<(unsigned)std::min<int64_t>((k * n + 255) / 256, 4096), 256, 0, c->stream>>>(b, k, n, bt, ldw);
  count_launch(1);
  if (ap) {
    k_pad_rows_i8<<<(unsigned)std::min<int64_t>((m * kp + 255) / 256, 4096), 256, 0, c->stream>>>(a, m, k, ap, kp);
    count_launch(1);
  }
  i8t_conv_geom g{m, kp, 1, 1, n, 1, 1, 1, 1, 0, 0, 0, 1};
  int rc = i8t_conv_fwd(ctx, &g, ap ? ap : a, kp, bt, ldw, ones, ones + 1, nullptr, cout);
  cudaStreamSynchronize(c->stream);  // h127 lives on this stack frame
  return rc;
}

}  // extern "C"
