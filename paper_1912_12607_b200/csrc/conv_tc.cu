// conv_tc.cu -- INT8 convolutions as implicit GEMMs on 5th-gen tensor cores
// (tcgen05.mma.cta_group::1.kind::i8, int32 accumulators in TMEM).
//
//   FWD   D[npq][k]     = sum_{r,s,c} A_im2col[npq][(r,s,c)] * W_krsc[k][(r,s,c)]
//   DGRAD D[nhw][c]     = sum_{r,s,k} G_col2im[nhw][(r,s,k)] * W_crsk[c][(r,s,k)]
//   WGRAD D[(r,s,c)][k] = sum_{npq} A_im2col[npq][(r,s,c)] * G[npq][k]   (npq split)
//
// Persistent, warp-specialised CTA (one per SM) walking a static tile queue:
//   warps 0-7   gather the implicit-im2col / col2im operand rows straight into
//               SWIZZLE_128B smem tiles with cp.async (zero padding = zero-fill);
//               thread 0 also issues the weight tile as one TMA
//               (cp.async.bulk.tensor, SWIZZLE_128B) for FWD / DGRAD;
//   warp 8      one elected thread issues tcgen05.mma (4 x K=32 per stage),
//               tcgen05.commit frees the smem stage / publishes the accumulator;
//   warps 9-12  drain TMEM (tcgen05.ld) and apply the reference's FP64 rescale
//               float(double(s_x)*double(s_y)*acc) (conv.cpp:139-143, 190-191,
//               201-203), or for WGRAD add the exact int32 split partial into
//               the int64 accumulator.
// The accumulator is double-buffered in TMEM (2 x BN columns) so the epilogue
// of tile i overlaps the main loop of tile i+1.  FWD/DGRAD operands are
// K-major; WGRAD operands are MN-major (the reduction runs over pixel rows).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <mutex>
#include <type_traits>

#include "internal.cuh"
#include "ptx.cuh"

namespace i8t_dev {

enum ConvMode { MODE_FWD = 0, MODE_DGRAD = 1, MODE_WGRAD = 2 };

// Division of a non-negative int32 by a kernel-invariant divisor d >= 1 as a
// multiply-high: q = (umulhi(x, m) + x) >> s with s = ceil(log2 d),
// m = floor(2^32 (2^s - d) / d) + 1 (exact for 0 <= x < 2^31).  The conv
// producers decode (n, p, q) / (tap, channel) per row and per k-block; a
// runtime integer division is ~20 dependent instructions (a 64-bit one a call).
struct FDiv {
  uint32_t m, s;
};
inline FDiv fdiv_of(int d) {
  uint32_t sh = 0;
  while ((1ull << sh) < static_cast<uint64_t>(d)) ++sh;
  const uint64_t m = ((1ull << 32) * ((1ull << sh) - static_cast<uint64_t>(d))) / static_cast<uint64_t>(d) + 1;
  return FDiv{d > 1 ? static_cast<uint32_t>(m) : 0u, sh};
}
__device__ __forceinline__ int fdiv(int64_t x, FDiv f) {
  const uint32_t u = static_cast<uint32_t>(x);
  return static_cast<int>((__umulhi(u, f.m) + u) >> f.s);
}

struct ConvArgs {
  const int8_t* act;  // NHWC [N][H][W][Cp]
  const int8_t* gz;   // NHWC [N][P][Q][Kp]
  const int8_t* wt;   // FWD: KRSC rows [K][ldw]; DGRAD: CRSK rows [C][ldw]
  int64_t ldw;
  int N, H, W, Cp, Kp, R, S, sh, sw, ph, pw, P, Q;
  int64_t M;      // GEMM rows
  int Ng;         // GEMM cols (valid)
  int64_t Kd;     // reduction length (valid)
  int k_tiles;    // k tiles per split
  int m_tiles, n_tiles, splits;
  const float* clip_x;
  const float* clip_y;
  float* out;
  int64_t ldo;
  int32_t* acc32;
  int use_tma_out;  // epilogue writes through the output tensor map (else direct stores)
  int m_pad;        // WGRAD: rows per split in the int32 partial workspace
  // DGRAD stride phase (sh or sw > 1): rows are the input pixels
  // (n, hh*sh + fh, ww*sw + fw) of one phase, the reduction runs over that
  // phase's taps r = r0 + ir*sh, s = s0 + is*sw only (p = hh + dh - ir,
  // q = ww + dw - is), every k-tile inside one tap (Kp % 128 == 0).
  int phase;
  int Hq, Wq, fh, fw, r0, s0, ns, dh, dw;
  int nr;  // phase taps along r (with ns along s)
  // phase rows padded to 2^prow_lg (> 0: on): GEMM row m = gr * 2^prow_lg + ww
  // with gr = n * Hq + hh, rows ww >= Wq computed and dropped, so every
  // 32-row quadrant is whole phase-grid rows -- one 3-D TMA box of the output
  // ([C][Wq][N*Hq], strides sw*C and sh*W*C floats; needs H == sh*Hq) -- and
  // the A tile stays one im2col box (its pixel box widened to 2^prow_lg)
  int prow_lg;
  // 1x1 / stride 1 / pad 0: the A operand rows are plain matrix rows, loaded
  // by TMA (tmap_a; WGRAD also takes its B = g_z rows from tmap_b) by one
  // thread -- no cp.async gather
  int tma_a;
  int tma_b;  // WGRAD with a gathered A: B = g_z rows still come by TMA (tmap_b)
  int wg_cb;  // WGRAD tma_a == 3: channel block of the im2col boxes (64 or 32 bytes), 128 / wg_cb boxes per m-tile
  // DGRAD residual join fused into the epilogue: out = dgrad + add_g, or
  // dgrad + add_g * (add_y > 0) when add_y is set (a single float add, so the
  // result equals the separate join bit for bit)
  const float* add_g;
  const float* add_y;
  const uint32_t* add_bits;  // instead of add_y: packed mask (bit e of word e/32 for flat NHWC index e)
  // fast divisions by the invariant extents (set_divs, before every launch)
  FDiv dCp, dKp, dS, dQ, dW, dWq, dns, dpq, dhw, dhwq, dHq;
};

inline void set_divs(ConvArgs& a) {
  a.dCp = fdiv_of(a.Cp > 0 ? a.Cp : 1);
  a.dKp = fdiv_of(a.Kp > 0 ? a.Kp : 1);
  a.dS = fdiv_of(a.S > 0 ? a.S : 1);
  a.dQ = fdiv_of(a.Q > 0 ? a.Q : 1);
  a.dW = fdiv_of(a.W > 0 ? a.W : 1);
  a.dWq = fdiv_of(a.Wq > 0 ? a.Wq : 1);
  a.dns = fdiv_of(a.ns > 0 ? a.ns : 1);
  a.dpq = fdiv_of(a.P * a.Q > 0 ? a.P * a.Q : 1);
  a.dhw = fdiv_of(a.H * a.W > 0 ? a.H * a.W : 1);
  a.dhwq = fdiv_of(a.Hq * a.Wq > 0 ? a.Hq * a.Wq : 1);
  a.dHq = fdiv_of(a.Hq > 0 ? a.Hq : 1);
}

// residual addend of output row `orow`, columns c0..c0+3
__device__ __forceinline__ float4 join_addend(const ConvArgs& a, int64_t orow, int c0) {
  const int64_t o = orow * a.ldo + c0;
  float4 g = __ldg(reinterpret_cast<const float4*>(a.add_g + o));
  if (a.add_y) {
    const float4 y = __ldg(reinterpret_cast<const float4*>(a.add_y + o));
    g.x = y.x > 0.0f ? g.x : 0.0f;
    g.y = y.y > 0.0f ? g.y : 0.0f;
    g.z = y.z > 0.0f ? g.z : 0.0f;
    g.w = y.w > 0.0f ? g.w : 0.0f;
  } else if (a.add_bits) {
    const uint32_t w = __ldg(a.add_bits + (o >> 5)) >> (o & 31);  // o % 4 == 0: one word
    g.x = (w & 1u) ? g.x : 0.0f;
    g.y = (w & 2u) ? g.y : 0.0f;
    g.z = (w & 4u) ? g.z : 0.0f;
    g.w = (w & 8u) ? g.w : 0.0f;
  }
  return g;
}


// exact int32 -> double on the FP64 pipe (no XU conversion): 2^52 + (x + 2^31) - (2^52 + 2^31)
__device__ __forceinline__ double i32_to_f64(uint32_t x) {
  return __hiloint2double(0x43300000, static_cast<int>(x ^ 0x80000000u)) - 4503601774854144.0;
}
// reference rescale float(double(s_x) * double(s_y) * acc) (conv.cpp:139-143)
__device__ __forceinline__ float dequant_acc(double rescale, uint32_t v) {
  return static_cast<float>(rescale * i32_to_f64(v));
}

// output row of GEMM row m (identity except in DGRAD phase mode)
__device__ __forceinline__ int64_t out_row_of(const ConvArgs& a, int64_t m) {
  if (!a.phase) return m;
  if (a.prow_lg) {
    const int gr = static_cast<int>(m >> a.prow_lg), ww = static_cast<int>(m & ((1 << a.prow_lg) - 1));
    const int n = fdiv(gr, a.dHq), hh = gr - n * a.Hq;
    return (static_cast<int64_t>(n) * a.H + hh * a.sh + a.fh) * a.W + ww * a.sw + a.fw;
  }
  const int hwq = a.Hq * a.Wq;
  const int n = fdiv(m, a.dhwq), rem = static_cast<int>(m - static_cast<int64_t>(n) * hwq);
  const int hh = fdiv(rem, a.dWq), ww = rem - hh * a.Wq;
  return (static_cast<int64_t>(n) * a.H + hh * a.sh + a.fh) * a.W + ww * a.sw + a.fw;
}
// GEMM row m maps to an output row (not a padding row of the phase mode)
__device__ __forceinline__ bool row_ok(const ConvArgs& a, int64_t m) {
  return m < a.M && (!a.prow_lg || static_cast<int>(m & ((1 << a.prow_lg) - 1)) < a.Wq);
}


constexpr int BM = 128;
constexpr int BKB = 128;  // bytes of reduction per stage (4 MMAs of K=32)
constexpr int NPROD = 256;
constexpr int MMA_WARP = 8;
constexpr int EPI_WARP0 = 9;
constexpr int NEPI = 256;                    // 8 epilogue warps: 2 per TMEM lane quadrant
constexpr int NTHREADS = NPROD + 32 + NEPI;  // 544

// EDB = 1: two staging buffers per epilogue warp (a chunk's TMA store can still
// be reading one while the next chunk is written to the other) at the price of
// pipeline stages -- for the short-reduction convs whose fp32 epilogue is the
// bottleneck (a tile of 1-4 k-blocks).
template <int MODE, int BN, int CG = 1, int EDB = 0>
struct Cfg {
  static constexpr int A_BYTES = BM * BKB;  // 16 KB
  static constexpr int B_SUB = (BN + 127) / 128;
  // CG == 2 (CTA pair): each CTA holds half of the B tile's N rows
  static constexpr int B_BYTES = (MODE == MODE_WGRAD) ? 128 * 128 * B_SUB : (BN / CG) * BKB;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_BYTES = (EDB ? 2 : 1) * 8 * 32 * 128;  // per epilogue warp: [32 rows x 128 B] staging tile(s)
  static constexpr int BUDGET = 232448 - EPI_BYTES - 1024 - 256;
  static constexpr int STAGES = BUDGET / STAGE_BYTES > 8 ? 8 : BUDGET / STAGE_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t TMEM_COLS = 2 * BN;  // double-buffered accumulator
  static constexpr bool TMA_B = (MODE != MODE_WGRAD);
};

__device__ __forceinline__ int ifloordiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

struct TileCoord {
  int m_tile, n_tile, split;
};
__device__ __forceinline__ TileCoord tile_of(const ConvArgs& a, int t) {
  const int per_split = a.m_tiles * a.n_tiles;
  TileCoord c;
  c.split = t / per_split;
  const int r = t - c.split * per_split;
  c.m_tile = r / a.n_tiles;  // n fastest: CTAs sharing an A tile run together (L2 reuse)
  c.n_tile = r - c.m_tile * a.n_tiles;
  return c;
}
__device__ __forceinline__ int tile_nk(const ConvArgs& a, int split) {
  const int total_kt = static_cast<int>((a.Kd + BKB - 1) / BKB);
  const int k0 = split * a.k_tiles;
  const int n = total_kt - k0;
  return n < a.k_tiles ? n : a.k_tiles;
}

// CG == 2: a CTA pair (cluster of 2) runs 256-row tiles with
// tcgen05.mma.cta_group::2 -- each CTA loads its 128 A rows and half of the B
// rows (TMA, completion counted on the leader's barrier), the leader issues
// the M = 256 MMAs and multicasts their commits; TMA-operand path only.
// DGX = false: a DGRAD without stride phases or residual join (the common
// case) compiled without those paths -- the same epilogue as FWD (the extra
// code and its per-chunk argument loads cost the plain dgrads ~10 %).
template <int MODE, int BN, int VA, int VB, int CG = 1, int EDB = 0, bool DGX = true>
__global__ void __launch_bounds__(NTHREADS, 1) k_conv_tc(const ConvArgs args, const __grid_constant__ CUtensorMap tmap_a,
                                                          const __grid_constant__ CUtensorMap tmap_b,
                                                          const __grid_constant__ CUtensorMap tmap_out) {
  using C = Cfg<MODE, BN, CG, EDB>;
  constexpr bool PAIR = CG == 2;
  constexpr bool DX = MODE == MODE_DGRAD && DGX;  // stride phases / residual join compiled in
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sEpi = smem + C::STAGES * C::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + C::EPI_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;  // [2]
  uint64_t* tempty = tfull + 2;         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int total_tiles = args.m_tiles * args.n_tiles * args.splits;
  const uint32_t crank = PAIR ? cluster_ctarank() : 0u;
  const int cta0 = PAIR ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);  // tile-queue slot
  const int ncta = PAIR ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  const int row_base = PAIR ? static_cast<int>(crank) * 128 : 0;  // this CTA's rows inside a tile
  constexpr int TM = PAIR ? 2 * BM : BM;                          // tile rows

  if (warp == MMA_WARP) {
    if (lane == 0) {
      for (int s = 0; s < C::STAGES; ++s) {
        mbar_init(&full[s], args.tma_a ? 1 : NPROD);
        mbar_init(&empty[s], 1);
      }
      for (int a = 0; a < 2; ++a) {
        mbar_init(&tfull[a], 1);
        mbar_init(&tempty[a], PAIR ? 2 * (NEPI / 32) : NEPI);  // PAIR: one arrival per epilogue warp of both CTAs
      }
      fence_mbar_init();
      if (C::TMA_B || args.tma_a || args.tma_b) tma_prefetch(&tmap_b);
      if (args.tma_a) tma_prefetch(&tmap_a);
      if (args.use_tma_out) tma_prefetch(&tmap_out);
    }
    __syncwarp();
    if constexpr (PAIR) {
      tmem_alloc_pair(tmem_slot, C::TMEM_COLS);
      tmem_relinquish_pair();
    } else {
      tmem_alloc(tmem_slot, C::TMEM_COLS);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // the peer's barriers are initialised before any remote signal
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // the prologue above (barriers, descriptor prefetch, TMEM) touches no global
  // data: it overlaps the predecessor grid's tail under programmatic launch
  pdl_entry();

  if (warp < MMA_WARP && args.tma_a) {
    // ================================================= TMA producer (thread 0)
    if (tid == 0) {
      int kc = 0;
      for (int t = cta0; t < total_tiles; t += ncta) {
        const TileCoord tc = tile_of(args, t);
        const int m0 = tc.m_tile * TM + row_base, n0 = tc.n_tile * BN;
        const int kt0 = tc.split * args.k_tiles;
        const int nk = tile_nk(args, tc.split);
        for (int kt = 0; kt < nk; ++kt, ++kc) {
          const int s = kc % C::STAGES;
          if (kc >= C::STAGES) mbar_wait(&empty[s], ((kc / C::STAGES) - 1) & 1);
          const uint32_t a_st = smem_u32(sA + s * C::A_BYTES);
          const uint32_t b_st = smem_u32(sB + s * C::B_BYTES);
          const int kb = (kt0 + kt) * BKB;
          if constexpr (PAIR) {
            // both CTAs' A and B halves complete on the leader's barrier
            if (crank == 0) mbar_arrive_expect_tx(&full[s], 2 * (C::A_BYTES + C::B_BYTES));
            const uint32_t lbar = mapa_shared(smem_u32(&full[s]), 0);
            if (MODE == MODE_FWD && args.tma_a == 2) {  // this CTA's 128 output pixels, im2col
              const int pq = args.P * args.Q;
              const int n = fdiv(m0, args.dpq), rem = m0 - n * pq, p = fdiv(rem, args.dQ), q = rem - p * args.Q;
              const int tap = fdiv(kb, args.dCp), cb = kb - tap * args.Cp;
              const int r = fdiv(tap, args.dS), sx = tap - r * args.S;
              tma_load_im2col_4d_pair(a_st, &tmap_a, lbar, cb, q * args.sw - args.pw, p * args.sh - args.ph, n,
                                      static_cast<uint16_t>(sx), static_cast<uint16_t>(r));
            } else if (MODE == MODE_DGRAD && args.tma_a == 2) {
              const int hw = args.H * args.W;
              const int n = fdiv(m0, args.dhw), rem = m0 - n * hw, h = fdiv(rem, args.dW), w = rem - h * args.W;
              const int tap = fdiv(kb, args.dKp), kc = kb - tap * args.Kp;
              const int r = fdiv(tap, args.dS), sx = tap - r * args.S;
              tma_load_im2col_4d_pair(a_st, &tmap_a, lbar, kc, w - (args.S - 1 - args.pw), h - (args.R - 1 - args.ph),
                                      n, static_cast<uint16_t>(args.S - 1 - sx), static_cast<uint16_t>(args.R - 1 - r));
            } else {
              tma_load_2d_pair(a_st, &tmap_a, lbar, kb, m0);
            }
            tma_load_2d_pair(b_st, &tmap_b, lbar, kb, n0 + static_cast<int>(crank) * (BN / 2));
            continue;
          }
          if (MODE == MODE_FWD && args.tma_a == 3) {
            // 32-channel taps (the stem's folded taps): the k-block's four 32-byte K
            // chunks are four im2col boxes [128 output pixels][32 channels]
            // (SWIZZLE_32B), one per MMA; a chunk past Kd is not loaded -- its
            // weights are the zero fill of the weight box, so whatever int8 the
            // stage's A slot still holds contributes 0
            const int nbox = static_cast<int>(args.Kd - kb) / 32 < 4 ? static_cast<int>(args.Kd - kb) / 32 : 4;
            mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(nbox) * 4096u + C::B_BYTES);
            const int pq = args.P * args.Q;
            const int n = fdiv(m0, args.dpq), rem = m0 - n * pq, p = fdiv(rem, args.dQ), q = rem - p * args.Q;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              if (h >= nbox) break;
              const int kh = kb + 32 * h;
              const int tap = fdiv(kh, args.dCp), cb = kh - tap * args.Cp;
              const int r = fdiv(tap, args.dS), sx = tap - r * args.S;
              tma_load_im2col_4d(a_st + h * 4096, &tmap_a, &full[s], cb, q * args.sw - args.pw, p * args.sh - args.ph,
                                 n, static_cast<uint16_t>(sx), static_cast<uint16_t>(r));
            }
            tma_load_2d(b_st, &tmap_b, &full[s], kb, n0);
            continue;
          }
          mbar_arrive_expect_tx(&full[s], C::A_BYTES + C::B_BYTES);  // the stage's single arrival
          if (MODE == MODE_FWD && args.tma_a == 2) {
            // implicit im2col by TMA: 128 consecutive output pixels of tap (r, s),
            // 128 channels from cb; zero padding = out-of-box fill
            const int pq = args.P * args.Q;
            const int n = fdiv(m0, args.dpq), rem = m0 - n * pq, p = fdiv(rem, args.dQ), q = rem - p * args.Q;
            const int tap = fdiv(kb, args.dCp), cb = kb - tap * args.Cp;
            const int r = fdiv(tap, args.dS), sx = tap - r * args.S;
            tma_load_im2col_4d(a_st, &tmap_a, &full[s], cb, q * args.sw - args.pw, p * args.sh - args.ph, n,
                               static_cast<uint16_t>(sx), static_cast<uint16_t>(r));
            tma_load_2d(b_st, &tmap_b, &full[s], kb, n0);
            continue;
          }
          if constexpr (MODE == MODE_WGRAD) {
            if (args.tma_a == 3) {
              // 64- / 32-channel taps: the m-tile's 128 rows are 128 / cb im2col boxes
              // [128 npq rows][cb channels] (SWIZZLE_64B / 32B) of their own (tap, c0);
              // a box past M repeats the last valid rows (its output rows are dropped)
              const int pq = args.P * args.Q;
              const int n = fdiv(kb, args.dpq), rem = kb - n * pq, p = fdiv(rem, args.dQ), q = rem - p * args.Q;
              auto boxes = [&](auto cb_c) {
                constexpr int CB = decltype(cb_c)::value;
#pragma unroll
                for (int h = 0; h < 128 / CB; ++h) {
                  int mh = static_cast<int>(m0) + CB * h;
                  if (mh >= args.M) mh = static_cast<int>(args.M) - CB;
                  const int tap = fdiv(mh, args.dCp), c0 = mh - tap * args.Cp;
                  const int r = fdiv(tap, args.dS), sx = tap - r * args.S;
                  tma_load_im2col_4d(a_st + h * 128 * CB, &tmap_a, &full[s], c0, q * args.sw - args.pw,
                                     p * args.sh - args.ph, n, static_cast<uint16_t>(sx), static_cast<uint16_t>(r));
                }
              };
              if (args.wg_cb == 64) boxes(std::integral_constant<int, 64>{});
              else boxes(std::integral_constant<int, 32>{});
            } else if (args.tma_a == 2) {  // im2col rows npq = kb.. of tap (r, s), channels c0 of the m-tile
              const int pq = args.P * args.Q;
              const int n = fdiv(kb, args.dpq), rem = kb - n * pq, p = fdiv(rem, args.dQ), q = rem - p * args.Q;
              const int tap = fdiv(m0, args.dCp), c0 = m0 - tap * args.Cp;
              const int r = fdiv(tap, args.dS), sx = tap - r * args.S;
              tma_load_im2col_4d(a_st, &tmap_a, &full[s], c0, q * args.sw - args.pw, p * args.sh - args.ph, n,
                                 static_cast<uint16_t>(sx), static_cast<uint16_t>(r));
            } else {
              tma_load_2d(a_st, &tmap_a, &full[s], m0, kb);  // [128 npq rows][128 channels], MN-major
            }
#pragma unroll
            for (int sub = 0; sub < C::B_SUB; ++sub) tma_load_2d(b_st + sub * 16384, &tmap_b, &full[s], n0 + sub * 128, kb);
          } else {
            if (DX && args.tma_a == 2 && args.phase) {
              // one stride phase: rows (n, hh, ww) of the phase grid, compact tap
              // (ir, is) reads g_z at (hh + dh - ir, ww + dw - is) = base (hh + dh -
              // (nr-1), ww + dw - (ns-1)) + mirrored offset (nr-1-ir, ns-1-is)
              const int it = fdiv(kb, args.dKp), kc = kb - it * args.Kp;
              const int ir = fdiv(it, args.dns), is = it - ir * args.ns;
              const uint16_t ow = static_cast<uint16_t>(args.ns - 1 - is), oh = static_cast<uint16_t>(args.nr - 1 - ir);
              if (args.prow_lg) {
                // the pixel box is 2^prow_lg wide (its columns past Wq read padding
                // rows: zero fill or neighbours, dropped by the store), so the
                // traversal order is the padded row order: one box as usual
                const int gr0 = m0 >> args.prow_lg;
                const int n = fdiv(gr0, args.dHq), hh = gr0 - n * args.Hq;
                tma_load_im2col_4d(a_st, &tmap_a, &full[s], kc, args.dw - (args.ns - 1), hh + args.dh - (args.nr - 1), n,
                                   ow, oh);
              } else {
                const int hwq = args.Hq * args.Wq;
                const int n = fdiv(m0, args.dhwq), rem = m0 - n * hwq, hh = fdiv(rem, args.dWq), ww = rem - hh * args.Wq;
                tma_load_im2col_4d(a_st, &tmap_a, &full[s], kc, ww + args.dw - (args.ns - 1),
                                   hh + args.dh - (args.nr - 1), n, ow, oh);
              }
              const int bx = ((args.r0 + ir * args.sh) * args.S + args.s0 + is * args.sw) * args.Kp + kc;
              tma_load_2d(b_st, &tmap_b, &full[s], bx, n0);
              continue;
            }
            if (MODE == MODE_DGRAD && args.tma_a == 2) {
              // stride-1 backward-data as the im2col of g_z over the input grid:
              // tap (r, s) reads g_z at (h + ph - r, w + pw - s) = base (h - (R-1-ph),
              // w - (S-1-pw)) + mirrored offset (R-1-r, S-1-s)
              const int hw = args.H * args.W;
              const int n = fdiv(m0, args.dhw), rem = m0 - n * hw, h = fdiv(rem, args.dW), w = rem - h * args.W;
              const int tap = fdiv(kb, args.dKp), kc = kb - tap * args.Kp;
              const int r = fdiv(tap, args.dS), sx = tap - r * args.S;
              tma_load_im2col_4d(a_st, &tmap_a, &full[s], kc, w - (args.S - 1 - args.pw), h - (args.R - 1 - args.ph), n,
                                 static_cast<uint16_t>(args.S - 1 - sx), static_cast<uint16_t>(args.R - 1 - r));
            } else {
              tma_load_2d(a_st, &tmap_a, &full[s], kb, m0);  // [128 pixel rows][128 B of channels], K-major
            }
            tma_load_2d(b_st, &tmap_b, &full[s], kb, n0);
          }
        }
      }
    }
  } else if (warp < MMA_WARP) {
    // ================================================= producers (warps 0-7)
    constexpr int PPR_A = BKB / VA;                 // pieces per 128 B row
    constexpr int ROWS_PER_PASS_A = NPROD / PPR_A;  // rows covered per pass
    constexpr int PASSES_A = BM / ROWS_PER_PASS_A;
    const int ja = tid % PPR_A, ra0 = tid / PPR_A;
    const int adv_p = BKB / args.Q, adv_q = BKB - adv_p * args.Q;  // WGRAD: 128 pixels = adv_p rows + adv_q
    int kc = 0;  // global stage counter across tiles
    if constexpr (PAIR) __trap();  // CTA pairs take the TMA-operand path only
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
      const TileCoord tc = tile_of(args, t);
      const int64_t m0 = static_cast<int64_t>(tc.m_tile) * BM;
      const int n0 = tc.n_tile * BN;
      const int kt0 = tc.split * args.k_tiles;
      const int nk = tile_nk(args, tc.split);
      int rowA_n[PASSES_A], rowA_y[PASSES_A], rowA_x[PASSES_A];
      bool rowA_ok[PASSES_A];
      int runR = 0, runS = 0, runC = 0;  // WGRAD run path: (r, s, c) of this thread's column run
      bool runOk = false;
      if constexpr (MODE != MODE_WGRAD) {
#pragma unroll
        for (int i = 0; i < PASSES_A; ++i) {
          const int64_t m = m0 + ra0 + i * ROWS_PER_PASS_A;
          rowA_ok[i] = m < args.M;
          const int mm = rowA_ok[i] ? static_cast<int>(m) : 0;
          if constexpr (MODE == MODE_FWD) {
            const int pq = args.P * args.Q;
            const int n = fdiv(mm, args.dpq), rem = mm - n * pq;
            const int p = fdiv(rem, args.dQ), q = rem - p * args.Q;
            rowA_n[i] = n;
            rowA_y[i] = p * args.sh - args.ph;
            rowA_x[i] = q * args.sw - args.pw;
          } else if (DX && args.phase) {
            const int hwq = args.Hq * args.Wq;
            const int n = fdiv(mm, args.dhwq), rem = mm - n * hwq;
            const int hh = fdiv(rem, args.dWq), ww = rem - hh * args.Wq;
            rowA_n[i] = n;
            rowA_y[i] = hh + args.dh;
            rowA_x[i] = ww + args.dw;
          } else {
            const int hw = args.H * args.W;
            const int n = fdiv(mm, args.dhw), rem = mm - n * hw;
            const int h = fdiv(rem, args.dW), w = rem - h * args.W;
            rowA_n[i] = n;
            rowA_y[i] = h + args.ph;
            rowA_x[i] = w + args.pw;
          }
        }
      }
      for (int kt = 0; kt < nk; ++kt, ++kc) {
        const int s = kc % C::STAGES;
        if (kc >= C::STAGES) mbar_wait(&empty[s], ((kc / C::STAGES) - 1) & 1);
        const uint32_t a_st = smem_u32(sA + s * C::A_BYTES);
        const uint32_t b_st = smem_u32(sB + s * C::B_BYTES);
        const int64_t kbase = static_cast<int64_t>(kt0 + kt) * BKB;
        if constexpr (MODE == MODE_FWD || MODE == MODE_DGRAD) {
          if (tid == 0) {  // weight tile [BN rows][128 B] by TMA (OOB rows / columns zero-filled)
            mbar_expect_tx(&full[s], C::B_BYTES);
            int bx = static_cast<int>(kbase);
            if (DX && args.phase) {  // compact tap index -> CRSK column of (r, s)
              const int it = fdiv(kbase, args.dKp);
              const int ir = fdiv(it, args.dns), is = it - ir * args.ns;
              bx = ((args.r0 + ir * args.sh) * args.S + args.s0 + is * args.sw) * args.Kp +
                   static_cast<int>(kbase - static_cast<int64_t>(it) * args.Kp);
            }
            tma_load_2d(b_st, &tmap_b, &full[s], bx, n0);
          }
          const int64_t kk = kbase + ja * VA;
          const bool kok = kk < args.Kd;
          const int CH = (MODE == MODE_FWD) ? args.Cp : args.Kp;
          const int tap = kok ? fdiv(kk, (MODE == MODE_FWD) ? args.dCp : args.dKp) : 0;
          const int ch = kok ? static_cast<int>(kk - static_cast<int64_t>(tap) * CH) : 0;
          const int tS = (DX && args.phase) ? args.ns : args.S;
          const int r = fdiv(tap, (DX && args.phase) ? args.dns : args.dS), sx = tap - r * tS;
#pragma unroll
          for (int i = 0; i < PASSES_A; ++i) {
            const int row = ra0 + i * ROWS_PER_PASS_A;
            bool ok = kok && rowA_ok[i];
            const int8_t* src = args.act;
            if constexpr (MODE == MODE_FWD) {
              const int ih = rowA_y[i] + r, iw = rowA_x[i] + sx;
              ok = ok && ih >= 0 && ih < args.H && iw >= 0 && iw < args.W;
              if (ok) src = args.act + ((static_cast<int64_t>(rowA_n[i]) * args.H + ih) * args.W + iw) * args.Cp + ch;
            } else if (DX && args.phase) {
              const int p = rowA_y[i] - r, q = rowA_x[i] - sx;  // r, sx = compact (ir, is)
              ok = ok && p >= 0 && p < args.P && q >= 0 && q < args.Q;
              src = args.gz;
              if (ok) src = args.gz + ((static_cast<int64_t>(rowA_n[i]) * args.P + p) * args.Q + q) * args.Kp + ch;
            } else {
              const int pn = rowA_y[i] - r, qn = rowA_x[i] - sx;
              int p, q;
              if (args.sh == 1) p = pn; else { p = ifloordiv(pn, args.sh); ok = ok && (pn - p * args.sh) == 0; }
              if (args.sw == 1) q = qn; else { q = ifloordiv(qn, args.sw); ok = ok && (qn - q * args.sw) == 0; }
              ok = ok && p >= 0 && p < args.P && q >= 0 && q < args.Q;
              src = args.gz;
              if (ok) src = args.gz + ((static_cast<int64_t>(rowA_n[i]) * args.P + p) * args.Q + q) * args.Kp + ch;
            }
            cp_async_vec<VA>(a_st + sw128_offset(row, ja * VA), src, ok);
          }
        } else {
          // ---- WGRAD: smem rows = npq (reduction), columns = M bytes (A) / N bytes (B), MN-major
          // Channel strides that are multiples of 32 / 64 bytes: a thread copies a
          // whole run of 32 / 64 contiguous bytes of one (pixel, tap) -- one
          // address per run instead of per 16-byte piece, tap decoded once per tile
          // (the 64-channel 3x3 layers and the stem's 32-byte folded taps).
          if constexpr (VA == 16) {
            if (args.Cp % 32 == 0) {
              auto runs = [&](auto run_c) {
                constexpr int RUN = decltype(run_c)::value;
                constexpr int TPR = BKB / RUN, RPP = NPROD / TPR, PASSES = BM / RPP;
                static_assert(PASSES <= PASSES_A, "row state");
                const int jr = tid % TPR, r0 = tid / TPR;
                if (kt == 0) {
                  const int64_t mR = m0 + jr * RUN;
                  runOk = mR < args.M;
                  const int tapR = runOk ? fdiv(mR, args.dCp) : 0;
                  runC = runOk ? static_cast<int>(mR - static_cast<int64_t>(tapR) * args.Cp) : 0;
                  runR = fdiv(tapR, args.dS);
                  runS = tapR - runR * args.S;
#pragma unroll
                  for (int i = 0; i < PASSES; ++i) {
                    const int kdi = static_cast<int>(kbase) + r0 + i * RPP;
                    const int pq = args.P * args.Q;
                    const int n = fdiv(kdi, args.dpq), rem = kdi - n * pq;
                    rowA_n[i] = n;
                    rowA_y[i] = fdiv(rem, args.dQ);
                    rowA_x[i] = rem - rowA_y[i] * args.Q;
                  }
                }
#pragma unroll
                for (int i = 0; i < PASSES; ++i) {
                  const int row = r0 + i * RPP;
                  const int64_t kd = kbase + row;
                  bool ok = runOk && kd < args.Kd;
                  const int ih = rowA_y[i] * args.sh - args.ph + runR, iw = rowA_x[i] * args.sw - args.pw + runS;
                  ok = ok && ih >= 0 && ih < args.H && iw >= 0 && iw < args.W;
                  const int8_t* src =
                      ok ? args.act + ((static_cast<int64_t>(rowA_n[i]) * args.H + ih) * args.W + iw) * args.Cp + runC
                         : args.act;
#pragma unroll
                  for (int u = 0; u < RUN / 16; ++u)
                    cp_async_vec<16>(a_st + sw128_offset(row, jr * RUN + u * 16), ok ? src + u * 16 : src, ok);
                  int q = rowA_x[i] + adv_q, p = rowA_y[i] + adv_p, n = rowA_n[i];
                  if (q >= args.Q) { q -= args.Q; ++p; }
                  while (p >= args.P) { p -= args.P; ++n; }
                  rowA_x[i] = q; rowA_y[i] = p; rowA_n[i] = n;
                }
              };
              if (args.Cp % 64 == 0) runs(std::integral_constant<int, 64>{});
              else runs(std::integral_constant<int, 32>{});
            }
          }
          const bool run_path = VA == 16 && args.Cp % 32 == 0;
          if (!run_path) {
          const int64_t mA = m0 + ja * VA;
          const bool mok = mA < args.M;
          const int tapA = mok ? fdiv(mA, args.dCp) : 0;
          const int cA = mok ? static_cast<int>(mA - static_cast<int64_t>(tapA) * args.Cp) : 0;
          const int rA = fdiv(tapA, args.dS), sA_ = tapA - rA * args.S;
          if (kt == 0) {  // decode this thread's rows once per tile, then advance 128 pixels per k-tile
#pragma unroll
            for (int i = 0; i < PASSES_A; ++i) {
              const int kdi = static_cast<int>(kbase) + ra0 + i * ROWS_PER_PASS_A;
              const int pq = args.P * args.Q;
              const int n = fdiv(kdi, args.dpq), rem = kdi - n * pq;
              rowA_n[i] = n;
              rowA_y[i] = fdiv(rem, args.dQ);
              rowA_x[i] = rem - rowA_y[i] * args.Q;
            }
          }
#pragma unroll
          for (int i = 0; i < PASSES_A; ++i) {
            const int row = ra0 + i * ROWS_PER_PASS_A;
            const int64_t kd = kbase + row;
            bool ok = mok && kd < args.Kd;
            const int8_t* src = args.act;
            const int ih = rowA_y[i] * args.sh - args.ph + rA, iw = rowA_x[i] * args.sw - args.pw + sA_;
            ok = ok && ih >= 0 && ih < args.H && iw >= 0 && iw < args.W;
            if (ok) src = args.act + ((static_cast<int64_t>(rowA_n[i]) * args.H + ih) * args.W + iw) * args.Cp + cA;
            cp_async_vec<VA>(a_st + sw128_offset(row, ja * VA), src, ok);
            // advance (n, p, q) by BKB pixels for the next k-tile
            int q = rowA_x[i] + adv_q, p = rowA_y[i] + adv_p, n = rowA_n[i];
            if (q >= args.Q) { q -= args.Q; ++p; }
            while (p >= args.P) { p -= args.P; ++n; }
            rowA_x[i] = q; rowA_y[i] = p; rowA_n[i] = n;
          }
          }  // !run_path
          if (args.tma_b) {  // g_z rows by TMA (thread 0; same barrier protocol as the FWD weights)
            if (tid == 0) {
              mbar_expect_tx(&full[s], C::B_BYTES);
#pragma unroll
              for (int sub = 0; sub < C::B_SUB; ++sub)
                tma_load_2d(b_st + sub * 16384, &tmap_b, &full[s], n0 + sub * 128, static_cast<int>(kbase));
            }
          } else {
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
        }
        // the stage's full barrier completes when every producer's copies have
        // landed (no producer-side wait: the loads of several stages overlap)
        cp_async_mbar_arrive(&full[s]);
      }
    }
    cp_async_wait<0>();
  } else if (warp == MMA_WARP) {
    // ================================================= MMA issuer (one thread)
    if (lane == 0 && crank == 0) {
      constexpr bool MN = (MODE == MODE_WGRAD);
      constexpr uint32_t idesc = make_idesc_i8(TM, BN, MN, MN);
      const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
      // A descriptor of stage 0, kk 0 and its per-kk start-address step (the
      // start field holds addr >> 4 in the low 14 bits: plain adds stay in it)
      uint64_t a_desc0;
      uint32_t a_kstep;
      if constexpr (MN) {
        const int cb = args.tma_a == 3 ? args.wg_cb : 128;
        a_desc0 = cb == 128 ? make_sdesc_sw128(a0, 16384, 1024)
                  : cb == 64 ? make_sdesc_sw64_mn(a0, 8192, 512) : make_sdesc_sw32_mn(a0, 4096, 256);
        a_kstep = (32u * static_cast<uint32_t>(cb)) >> 4;
      } else if (MODE == MODE_FWD && args.tma_a == 3) {
        a_desc0 = make_sdesc_sw32_k(a0, 256);  // MMA kk reads box kk: [128 rows][32 B]
        a_kstep = 4096u >> 4;
      } else {
        a_desc0 = make_sdesc_sw128(a0, 16, 1024);
        a_kstep = 32u >> 4;
      }
      int kc = 0, it = 0;
      for (int t = cta0; t < total_tiles; t += ncta, ++it) {
        const TileCoord tc = tile_of(args, t);
        const int nk = tile_nk(args, tc.split);
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);  // epilogue drained this accumulator
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kt = 0; kt < nk; ++kt, ++kc) {
          const int s = kc % C::STAGES;
          mbar_wait(&full[s], (kc / C::STAGES) & 1);
          // cp.async (generic proxy) writes -> tcgen05.mma operand reads; TMA-only
          // stages were written by the async proxy and need no proxy fence
          if (!args.tma_a) fence_proxy_async_smem();
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < BKB / 32; ++kk) {
            uint64_t ad, bd;
            // A: the stage-0 / kk-0 descriptor advanced in its start-address field
            ad = a_desc0 + static_cast<uint64_t>((static_cast<uint32_t>(s) * C::A_BYTES >> 4) + kk * a_kstep);
            if constexpr (MN) {
              // MN-major: 32 reduction rows per MMA = 4096 B; SBO = 8-row atom stride, LBO = 128-col sub-tile
              bd = make_sdesc_sw128(b0 + s * C::B_BYTES + kk * 4096, 16384, 1024);
            } else {
              // K-major: 32 B of reduction per MMA inside the 128 B swizzled row; SBO = 8 rows x 128 B
              bd = make_sdesc_sw128(b0 + s * C::B_BYTES + kk * 32, 16, 1024);
            }
            if constexpr (PAIR) mma_i8_pair(d_tmem, ad, bd, idesc, (kt | kk) != 0 ? 1u : 0u);
            else mma_i8(d_tmem, ad, bd, idesc, (kt | kk) != 0 ? 1u : 0u);
          }
          if constexpr (PAIR) mma_commit_pair(&empty[s], 3);
          else mma_commit(&empty[s]);
        }
        if constexpr (PAIR) mma_commit_pair(&tfull[acc], 3);
        else mma_commit(&tfull[acc]);
      }
    }
    __syncwarp();
  } else {
    // ================================================= epilogue (warps 9-12)
    const int quad = warp & 3;  // TMEM lane quadrant accessible to this warp
    const int half = (warp - EPI_WARP0) >> 2;  // which half of the BN columns
    const int row = quad * 32 + lane;
    const double rescale =
        static_cast<double>(__fdiv_rn(*args.clip_x, 127.0f)) * static_cast<double>(__fdiv_rn(*args.clip_y, 127.0f));
    const uint32_t stage_s = smem_u32(sEpi + (warp - EPI_WARP0) * ((EDB ? 2 : 1) * 32 * 128));
    int it = 0, nst = 0;
    constexpr int HALF = BN / 2 < 32 ? 32 : BN / 2;
    constexpr int NCH = HALF / 32;  // 32-column chunks per epilogue warp per tile
    const int c_begin0 = half * HALF;
    // PAIR: the epilogue warps of both CTAs hand the accumulator back to the leader
    const uint32_t tempty_leader = PAIR ? mapa_shared(smem_u32(&tempty[0]), 0) : 0u;
    auto release_acc = [&](int acc) {
      tc_fence_before();
      if constexpr (PAIR) {
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_leader + 8u * static_cast<uint32_t>(acc));
      } else {
        mbar_arrive(&tempty[acc]);
      }
    };
    for (int t = cta0; t < total_tiles; t += ncta, ++it) {
      const TileCoord tc = tile_of(args, t);
      const int64_t m = static_cast<int64_t>(tc.m_tile) * TM + row_base + row;
      const int n0 = tc.n_tile * BN;
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(acc * BN);
      const int c_begin = c_begin0, c_end = (half + 1) * HALF < BN ? (half + 1) * HALF : BN;
      if (c_begin >= c_end) {  // BN == 32 would leave the second half idle
        release_acc(acc);
        continue;
      }
      auto chunk = [&](const int ci) {
        const int col = c_begin + ci * 32;
        uint32_t v[32];
        tmem_ld32(t_row + static_cast<uint32_t>(col), v);
        tmem_ld_wait();
        if (col + 32 >= c_end) release_acc(acc);  // last read of this accumulator: hand it back to the MMA warp
        const int gc0 = n0 + col;
        if (args.use_tma_out) {
          // 32x32 sub-tile -> swizzled smem staging -> one TMA bulk store
          const uint32_t buf_s = stage_s + (EDB ? static_cast<uint32_t>(nst & 1) * (32 * 128) : 0u);
          if (lane == 0) {  // the store that last used this buffer has finished reading it
            if constexpr (EDB) bulk_wait_read<1>();
            else bulk_wait_read<0>();
          }
          __syncwarp();
          // the residual join decided once per chunk (a per-float4 test of the
          // kernel arguments cost the dgrad epilogue ~15 % more instructions)
          auto stage = [&](auto join_c) {
            constexpr bool JOIN = decltype(join_c)::value;
            const int64_t orow = JOIN ? out_row_of(args, m) : 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              uint4 w;
              if constexpr (MODE == MODE_WGRAD) {
                w = make_uint4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
              } else {
                float4 f = make_float4(dequant_acc(rescale, v[4 * j + 0]), dequant_acc(rescale, v[4 * j + 1]),
                                       dequant_acc(rescale, v[4 * j + 2]), dequant_acc(rescale, v[4 * j + 3]));
                if (JOIN && gc0 + 4 * j < args.Ng) {
                  const float4 ad = join_addend(args, orow, gc0 + 4 * j);
                  f.x = __fadd_rn(f.x, ad.x); f.y = __fadd_rn(f.y, ad.y); f.z = __fadd_rn(f.z, ad.z); f.w = __fadd_rn(f.w, ad.w);
                }
                w = make_uint4(__float_as_uint(f.x), __float_as_uint(f.y), __float_as_uint(f.z), __float_as_uint(f.w));
              }
              sts128(buf_s + sw128_offset(static_cast<uint32_t>(lane), static_cast<uint32_t>(j * 16)), w);
            }
          };
          if (DX && args.add_g && row_ok(args, m)) stage(std::true_type{});
          else stage(std::false_type{});
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int r0 = (MODE == MODE_WGRAD ? tc.split * args.m_pad : 0) + tc.m_tile * TM + row_base + quad * 32;
            if (DX && args.prow_lg) tma_store_3d(&tmap_out, buf_s, gc0, 0, r0 >> args.prow_lg);
            else tma_store_2d(&tmap_out, buf_s, gc0, r0);
            bulk_commit();
          }
          ++nst;
        } else if (DX ? row_ok(args, m) : m < args.M) {
          if constexpr (MODE != MODE_WGRAD) {
            if (args.out) {
              float* dst = args.out + (DX ? out_row_of(args, m) : m) * args.ldo + gc0;
              if (gc0 + 32 <= args.Ng && (args.ldo % 4) == 0) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                  float4 w;
                  w.x = dequant_acc(rescale, v[4 * j + 0]);
                  w.y = dequant_acc(rescale, v[4 * j + 1]);
                  w.z = dequant_acc(rescale, v[4 * j + 2]);
                  w.w = dequant_acc(rescale, v[4 * j + 3]);
                  if (DX && args.add_g) {
                    const float4 ad = join_addend(args, out_row_of(args, m), gc0 + 4 * j);
                    w.x = __fadd_rn(w.x, ad.x); w.y = __fadd_rn(w.y, ad.y); w.z = __fadd_rn(w.z, ad.z); w.w = __fadd_rn(w.w, ad.w);
                  }
                  reinterpret_cast<float4*>(dst)[j] = w;
                }
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (gc0 + i < args.Ng) {
                    float o = dequant_acc(rescale, v[i]);
                    if (DX && args.add_g) {
                      const int64_t ai = out_row_of(args, m) * args.ldo + gc0 + i;
                      const bool mk = args.add_y ? args.add_y[ai] > 0.0f
                                                 : !args.add_bits || ((args.add_bits[ai >> 5] >> (ai & 31)) & 1u);
                      o = __fadd_rn(o, mk ? args.add_g[ai] : 0.0f);
                    }
                    dst[i] = o;
                  }
              }
            }
          }
        }
        if (args.acc32 && (DX ? row_ok(args, m) : m < args.M) && MODE != MODE_WGRAD) {
          int32_t* dst = args.acc32 + (DX ? out_row_of(args, m) : m) * args.Ng + gc0;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (gc0 + i < args.Ng) dst[i] = static_cast<int32_t>(v[i]);
        }
      };
#pragma unroll 1
      for (int ci = 0; ci < NCH; ++ci) chunk(ci);
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // no remote arrival or multicast targets an exited CTA
  if (warp == MMA_WARP) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair(tmem_base, C::TMEM_COLS);
    else tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

// WGRAD finalize: int64 acc [(r,s,c_pad)][K] -> float KCRS or KRSC, reference rescale.
__global__ void k_wgrad_finalize(const long long* __restrict__ acc, int K, int C, int Cp, int RS,
                                 const float* clip_g, const float* clip_a, float* __restrict__ gw, int out_kcrs) {
  pdl_entry();
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

// WGRAD split reduction: acc[m][k] = sum_s part[s][m][k] (int64, exact, fixed order),
// optionally rescaled into float weights (KCRS or KRSC); acc may be NULL.
__global__ void k_wgrad_reduce(const int32_t* __restrict__ part, int splits, int m_pad, int Kp, int M, int K, int C,
                               int Cp, int RS, long long* __restrict__ acc, const float* clip_g, const float* clip_a,
                               float* __restrict__ gw, int out_kcrs) {
  pdl_entry();
  const double rescale =
      static_cast<double>(__fdiv_rn(*clip_g, 127.0f)) * static_cast<double>(__fdiv_rn(*clip_a, 127.0f));
  const int64_t tot = static_cast<int64_t>(M) * K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = static_cast<int>(i / K), k = static_cast<int>(i - static_cast<int64_t>(m) * K);
    long long sum = 0;
    for (int sp = 0; sp < splits; ++sp) sum += __ldg(part + (static_cast<int64_t>(sp) * m_pad + m) * Kp + k);
    if (acc) acc[i] = sum;
    if (gw) {
      const int rs = m / Cp, c = m - rs * Cp;
      if (c < C) {
        const int64_t o = out_kcrs ? (static_cast<int64_t>(k) * C + c) * RS + rs : (static_cast<int64_t>(k) * RS + rs) * C + c;
        gw[o] = static_cast<float>(rescale * static_cast<double>(sum));
      }
    }
  }
}

// Few outputs, many splits (the deep layers' wgrads: M*K of a few thousand,
// ~100 splits): P split phases per output, 256/P consecutive outputs per block
// (coalesced per warp), the phases summed through shared memory.  Integer sums,
// so the result is the same whatever the order.
template <int P>
__global__ void __launch_bounds__(256) k_wgrad_reduce_split(const int32_t* __restrict__ part, int splits, int m_pad,
                                                            int Kp, int M, int K, int C, int Cp, int RS,
                                                            long long* __restrict__ acc, const float* clip_g,
                                                            const float* clip_a, float* __restrict__ gw, int out_kcrs) {
  pdl_entry();
  constexpr int W = 256 / P;
  __shared__ long long red[P][W];
  const double rescale =
      static_cast<double>(__fdiv_rn(*clip_g, 127.0f)) * static_cast<double>(__fdiv_rn(*clip_a, 127.0f));
  const int64_t tot = static_cast<int64_t>(M) * K;
  const int lo = threadIdx.x % W, ph = threadIdx.x / W;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * W; base < tot; base += static_cast<int64_t>(gridDim.x) * W) {
    const int64_t i = base + lo;
    const int m = static_cast<int>(i / K), k = static_cast<int>(i - static_cast<int64_t>(m) * K);
    long long sum = 0;
    if (i < tot)
      for (int sp = ph; sp < splits; sp += P) sum += __ldg(part + (static_cast<int64_t>(sp) * m_pad + m) * Kp + k);
    red[ph][lo] = sum;
    __syncthreads();
    if (ph == 0 && i < tot) {
#pragma unroll
      for (int p = 1; p < P; ++p) sum += red[p][lo];
      if (acc) acc[i] = sum;
      if (gw) {
        const int rs = m / Cp, c = m - rs * Cp;
        if (c < C) {
          const int64_t o =
              out_kcrs ? (static_cast<int64_t>(k) * C + c) * RS + rs : (static_cast<int64_t>(k) * RS + rs) * C + c;
          gw[o] = static_cast<float>(rescale * static_cast<double>(sum));
        }
      }
    }
    __syncthreads();
  }
}

// Narrow-channel convolutions (c_pad == 4, e.g. the RGB stem): fold the kw
// horizontal taps into the channel dimension,
//   X'[n][h][q][s*4 + c] = X[n][h][q*sw + s - pw][c]  (zero outside; bytes 4*kw..31 zero),
// so the conv becomes (C' = 32, W' = Q, S' = 1, stride (sh, 1), pad (ph, 0)) with
// 32-byte operand pieces instead of 4-byte ones.  Its reduction order (r, s, c)
// is the original KRSC order, so the weight rows only gain 4 zero bytes per r.
__global__ void k_fold_taps(const int8_t* __restrict__ x, int64_t NH, int W, int Q, int kw, int sw, int pw,
                            int8_t* __restrict__ xf) {
  pdl_entry();
  const int64_t tot = NH * Q;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t nh = i / Q;
    const int q = static_cast<int>(i - nh * Q);
    const int32_t* row = reinterpret_cast<const int32_t*>(x) + nh * W;
    int32_t w[8];
#pragma unroll
    for (int sx = 0; sx < 8; ++sx) {
      const int wx = q * sw + sx - pw;
      w[sx] = (sx < kw && wx >= 0 && wx < W) ? __ldg(row + wx) : 0;
    }
    int4* o = reinterpret_cast<int4*>(xf + i * 32);
    o[0] = make_int4(w[0], w[1], w[2], w[3]);
    o[1] = make_int4(w[4], w[5], w[6], w[7]);
  }
}

// KRSC [K][ldw] (c_pad 4) -> [K][R*32]: each r's kw*4 bytes, zero padded to 32.
__global__ void k_fold_weights(const int8_t* __restrict__ w, int64_t ldw, int K, int R, int kw, int8_t* __restrict__ wf) {
  pdl_entry();
  const int tot = K * R * 32;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
    const int k = i / (R * 32), rem = i - k * R * 32, r = rem / 32, j = rem - r * 32;
    wf[i] = j < 4 * kw ? w[k * ldw + r * kw * 4 + j] : static_cast<int8_t>(0);
  }
}

// folded wgrad accumulator [R*32][K] -> original [(r*kw + s)*4 + c][K]
__global__ void k_unfold_wacc(const long long* __restrict__ accf, int R, int kw, int K, long long* __restrict__ acc) {
  pdl_entry();
  const int tot = R * kw * 4 * K;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += gridDim.x * blockDim.x) {
    const int m = i / K, k = i - m * K;
    const int r = m / (kw * 4), j = m - r * kw * 4;
    acc[i] = accf[(r * 32 + j) * K + k];
  }
}

// 1x1 / stride 1 / pad 0 convolution whose operand rows are TMA-addressable.
static bool plain_1x1(const i8t_conv_geom* g, const void* p0, int64_t ld0, const void* p1 = nullptr, int64_t ld1 = 16) {
  static const bool off = getenv("I8T_NO_TMA_A") != nullptr;
  return !off && g->kh == 1 && g->kw == 1 && g->stride_h == 1 && g->stride_w == 1 && g->pad_h == 0 && g->pad_w == 0 &&
         !g->depthwise && ld0 % 16 == 0 && ld1 % 16 == 0 && (reinterpret_cast<uintptr_t>(p0) & 15u) == 0 &&
         (reinterpret_cast<uintptr_t>(p1) & 15u) == 0;
}

static bool foldable(const i8t_conv_geom* g, int64_t c_pad) {
  static const bool off = getenv("I8T_NO_FOLD") != nullptr;
  return !off && c_pad == 4 && !g->depthwise && g->kw > 1 && g->kw <= 8;
}

static i8t_conv_geom folded_geom(const i8t_conv_geom* g, int64_t Q) {
  i8t_conv_geom f = *g;
  f.c = 32; f.w = Q; f.kw = 1; f.stride_w = 1; f.pad_w = 0;
  return f;
}

static int8_t* fold_input(Ctx* c, const i8t_conv_geom* g, int64_t Q, const int8_t* a, size_t extra, int8_t** extra_out) {
  const size_t xbytes = static_cast<size_t>(g->n * g->h * Q) * 32;
  int8_t* buf = reinterpret_cast<int8_t*>(ensure_fold(c, xbytes + extra + 256));
  if (!buf) return nullptr;
  const int64_t tot = g->n * g->h * Q;
  const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * 16);
  launch_k(k_fold_taps, blocks, 256, 0, c->stream, a, g->n * g->h, (int)g->w, (int)Q, (int)g->kw, (int)g->stride_w,
                                             (int)g->pad_w, buf);
  count_launch(1);
  *extra_out = buf + ((xbytes + 255) / 256) * 256;
  return buf;
}

// DGRAD phase with no taps (e.g. 1x1 stride 2, odd pixels): rows are zero.
__global__ void k_zero_phase(ConvArgs a) {
  pdl_entry();
  const int64_t rows = static_cast<int64_t>(a.N) * a.Hq * a.Wq;
  const int c4 = a.Ng / 4;  // Ng % 4 == 0 on this path
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t m = blockIdx.x * 8ll + warp; m < rows; m += gridDim.x * 8ll) {
    const int64_t o = out_row_of(a, m);
    float4* dst = reinterpret_cast<float4*>(a.out + o * a.ldo);
    int4* acc = a.acc32 ? reinterpret_cast<int4*>(a.acc32 + o * a.Ng) : nullptr;
    for (int c = lane; c < c4; c += 32) {
      if (a.out) {
        float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        if (a.add_g) {  // the join adds the addend to this (+0) dgrad value
          const float4 ad = join_addend(a, o, 4 * c);
          z = make_float4(__fadd_rn(0.f, ad.x), __fadd_rn(0.f, ad.y), __fadd_rn(0.f, ad.z), __fadd_rn(0.f, ad.w));
        }
        dst[c] = z;
      }
      if (acc) acc[c] = make_int4(0, 0, 0, 0);
    }
  }
}

__global__ void k_transpose_i8(const int8_t* __restrict__ src, int64_t rows, int64_t cols, int8_t* __restrict__ dst,
                               int64_t ld_dst) {
  pdl_entry();
  const int64_t tot = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    dst[c * ld_dst + r] = src[i];
  }
}

__global__ void k_pad_rows_i8(const int8_t* __restrict__ src, int64_t rows, int64_t cols, int8_t* __restrict__ dst,
                              int64_t ld_dst) {
  pdl_entry();
  const int64_t tot = rows * ld_dst;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ld_dst, c = i - r * ld_dst;
    dst[i] = c < cols ? src[r * cols + c] : (int8_t)0;
  }
}

// ---------------------------------------------------------------- host side
static int vec_of(int64_t ch) { return (ch % 16 == 0) ? 16 : (ch % 8 == 0) ? 8 : 4; }

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

typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);
static EncodeIm2colFn encode_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(p);
  });
  return fn;
}

// NHWC int8 tensor [N][H][W][C] -> im2col TMA map: 128-pixel columns of 128
// channels (SWIZZLE_128B: the K-major A tile of FWD / DGRAD and the MN-major
// A tile of WGRAD alike), traversing the pixel box [lower, dim - 1 + upper]
// with strides (sw, sh); out-of-tensor taps are zero-filled.
static int make_im2col_map(CUtensorMap* map, const int8_t* t, int64_t N, int64_t H, int64_t W, int64_t C, int lower_w,
                           int lower_h, int upper_w, int upper_h, int sw, int sh, uint32_t cbox = 128u,
                           CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B, uint32_t pix = BM) {
  EncodeIm2colFn fn = encode_im2col_fn();
  if (!fn) return set_error(I8T_ECUDA, "cuTensorMapEncodeIm2col unavailable");
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(N)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(W * C), static_cast<cuuint64_t>(H * W * C)};
  const int lower[2] = {lower_w, lower_h};
  const int upper[2] = {upper_w, upper_h};
  cuuint32_t estr[4] = {1u, static_cast<cuuint32_t>(sw), static_cast<cuuint32_t>(sh), 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(t), dims, strides, lower, upper, cbox,
                  static_cast<cuuint32_t>(pix), estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(I8T_ECUDA, "cuTensorMapEncodeIm2col failed (" + std::to_string(int(r)) + ")");
  return I8T_OK;
}
// the forward / backward-weight activation map: box = the output positions
static int make_im2col_map(CUtensorMap* map, const int8_t* a, const i8t_conv_geom* g, int64_t c_pad,
                           uint32_t cbox = 128u, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  return make_im2col_map(map, a, g->n, g->h, g->w, c_pad, static_cast<int>(-g->pad_w), static_cast<int>(-g->pad_h),
                         static_cast<int>(g->pad_w - (g->kw - 1)), static_cast<int>(g->pad_h - (g->kh - 1)),
                         static_cast<int>(g->stride_w), static_cast<int>(g->stride_h), cbox, swz);
}

// Forward convs whose A operand TMA im2col can load: 128-channel blocks, the
// output grid exactly the pixel box (floor mode with an exact fit), offsets in
// range.  I8T_NO_IM2COL=1 keeps the cp.async gather (A/B experiments).
static bool im2col_ok(const i8t_conv_geom* g, int64_t c_pad, const void* a, int64_t P, int64_t Q, int64_t cblk = 128) {
  static const bool off = getenv("I8T_NO_IM2COL") != nullptr;
  if (off || g->depthwise || c_pad % cblk != 0 || (reinterpret_cast<uintptr_t>(a) & 15u)) return false;
  if (g->kh * g->kw == 1 && g->stride_h == 1 && g->stride_w == 1 && g->pad_h == 0 && g->pad_w == 0) return false;
  if (g->stride_h > 8 || g->stride_w > 8 || g->kh > 8 || g->kw > 8 || g->pad_h >= g->kh || g->pad_w >= g->kw) return false;
  // the box [-pad, W - 1 + pad - (k - 1)] traversed with stride s has exactly
  // floor((W + 2 pad - k) / s) + 1 = Q positions per row (P per column)
  return (g->w + 2 * g->pad_w - g->kw) / g->stride_w + 1 == Q && (g->h + 2 * g->pad_h - g->kh) / g->stride_h + 1 == P;
}

// I8T_NO_WG64=1 keeps the cp.async gather for 64 / 32-channel-block wgrads (A/B experiments).
static bool wg64_off() {
  static const bool off = getenv("I8T_NO_WG64") != nullptr;
  return off;
}

// 2-D int8 weight matrix [rows][ld] -> TMA map with box {128 B, box_rows}, SWIZZLE_128B.
static int make_weight_map(CUtensorMap* map, const int8_t* w, int64_t rows, int64_t ld, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return set_error(I8T_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(ld), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld)};
  cuuint32_t box[2] = {128u, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(w), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(I8T_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return I8T_OK;
}

// 2-D [rows][ld] fp32/int32 output -> TMA store map, box {32 elements, 32 rows}, SWIZZLE_128B.
static int make_out_map(CUtensorMap* map, void* base, int64_t cols, int64_t rows, int64_t ld, bool is_int) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return set_error(I8T_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * 4)};
  cuuint32_t box[2] = {32u, 32u};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(map, is_int ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(I8T_ECUDA, "cuTensorMapEncodeTiled(out) failed (" + std::to_string(int(r)) + ")");
  return I8T_OK;
}

// One stride phase (fh, fw) of an NHWC fp32 output [N][H][W][C] as a 3-D map
// [C][Wq][N*Hq] (rows n*Hq + hh merge because H == sh*Hq), box {32 channels,
// 2^lg pixels, 32 >> lg rows}, SWIZZLE_128B: a 32-row quadrant of the padded
// phase rows (prow_lg) in one store, the padding columns ww >= Wq clipped.
static int make_phase_out_map(CUtensorMap* map, float* out, const ConvArgs& x, int lg) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return set_error(I8T_ECUDA, "cuTensorMapEncodeTiled unavailable");
  float* base = out + (static_cast<int64_t>(x.fh) * x.W + x.fw) * x.ldo;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(x.Ng), static_cast<cuuint64_t>(x.Wq),
                        static_cast<cuuint64_t>(x.N) * static_cast<cuuint64_t>(x.Hq)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(x.sw * x.ldo * 4),
                           static_cast<cuuint64_t>(x.sh) * static_cast<cuuint64_t>(x.W) * x.ldo * 4};
  cuuint32_t box[3] = {32u, 1u << lg, 32u >> lg};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(I8T_ECUDA, "cuTensorMapEncodeTiled(phase out) failed (" + std::to_string(int(r)) + ")");
  return I8T_OK;
}

static bool tma_out_ok(const void* p, int64_t ld) {
  static const bool off = getenv("I8T_NO_TMA_OUT") != nullptr;  // tuning experiments: direct epilogue stores
  return !off && p && (ld % 4) == 0 && (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
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

// CTA-pair launch (TMA-operand path, 256-row tiles): a.m_tiles counts 256-row tiles.
template <int MODE, int BN>
static int launch_pair(cudaStream_t st, const ConvArgs& a0, const CUtensorMap& amap, const CUtensorMap& map,
                       const CUtensorMap& omap) {
  ConvArgs a = a0;
  set_divs(a);
  using C = Cfg<MODE, BN, 2>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_conv_tc<MODE, BN, 16, 16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    configured = true;
  }
  const int tiles = a.m_tiles * a.n_tiles * a.splits;
  const int pairs = tiles < num_sms() / 2 ? tiles : num_sms() / 2;
  launch_k_cluster(k_conv_tc<MODE, BN, 16, 16, 2>, 2 * pairs, NTHREADS, C::SMEM, st, 2u, a, amap, map, omap);
  count_launch(1);
  return cuda_check("k_conv_tc<pair>");
}

// Opt-in (I8T_CONV_PAIR=1): correct (tests/test_gpu_conv_pair.py); on the 1x1
// shapes it covers it runs within +-5 % of the single-CTA kernel (those are
// bound by the fp32 output and the epilogue, not the operand loads) -- kept as
// the base for pairing the gathered 3x3 path.
static bool pair_enabled() {
  static const bool on = [] {
    const char* e = getenv("I8T_CONV_PAIR");
    return e && e[0] == '1';
  }();
  return on;
}

// k-blocks per tile up to which FWD / DGRAD take the double-buffered epilogue
// staging (I8T_EDB_KT; 0 turns it off)
static int edb_max_ktiles() {
  static const int v = [] {
    const char* e = getenv("I8T_EDB_KT");
    return e ? atoi(e) : 4;
  }();
  return v;
}

template <int MODE, int BN, int VA, int VB, int EDB = 0, bool DGX = true>
static int launch_one(cudaStream_t st, const ConvArgs& a0, const CUtensorMap& amap, const CUtensorMap& map,
                      const CUtensorMap& omap) {
  ConvArgs a = a0;
  set_divs(a);
  using C = Cfg<MODE, BN, 1, EDB>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k_conv_tc<MODE, BN, VA, VB, 1, EDB, DGX>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    configured = true;
  }
  const int tiles = a.m_tiles * a.n_tiles * a.splits;
  static const int cap = [] {
    const char* e = getenv("I8T_CONV_GRID");  // tuning experiments: fewer persistent CTAs
    return e ? atoi(e) : 0;
  }();
  const int sms = cap > 0 && cap < num_sms() ? cap : num_sms();
  const int grid = tiles < sms ? tiles : sms;
  launch_k(k_conv_tc<MODE, BN, VA, VB, 1, EDB, DGX>, grid, NTHREADS, C::SMEM, st, a, amap, map, omap);
  count_launch(1);
  return cuda_check("k_conv_tc");
}

template <int MODE, int BN>
static int dispatch_vec(cudaStream_t st, const ConvArgs& a, const CUtensorMap& am, const CUtensorMap& m,
                        const CUtensorMap& o, int va, int vb) {
  if (a.tma_a) {  // no gather: vector widths unused
    if constexpr (MODE != MODE_WGRAD) {
      const bool plain = MODE == MODE_DGRAD && !a.phase && !a.add_g;  // DGX = false
      // (with BN = 256 only on small grids: the fourth pipeline stage it costs
      // matters more than the staging once every SM runs tens of tiles)
      if (a.use_tma_out && a.k_tiles <= edb_max_ktiles() && (BN <= 128 || a.M < 131072))
        return plain ? launch_one<MODE, BN, 16, 16, 1, false>(st, a, am, m, o)
                     : launch_one<MODE, BN, 16, 16, 1>(st, a, am, m, o);
      if (plain) return launch_one<MODE, BN, 16, 16, 0, false>(st, a, am, m, o);
    }
    return launch_one<MODE, BN, 16, 16>(st, a, am, m, o);
  }
  if constexpr (MODE == MODE_WGRAD) {
    if (vb == 16) {
      if (va == 16) return launch_one<MODE, BN, 16, 16>(st, a, am, m, o);
      if (va == 8) return launch_one<MODE, BN, 8, 16>(st, a, am, m, o);
      return launch_one<MODE, BN, 4, 16>(st, a, am, m, o);
    }
    if (vb == 8) {
      if (va == 16) return launch_one<MODE, BN, 16, 8>(st, a, am, m, o);
      if (va == 8) return launch_one<MODE, BN, 8, 8>(st, a, am, m, o);
      return launch_one<MODE, BN, 4, 8>(st, a, am, m, o);
    }
    if (va == 16) return launch_one<MODE, BN, 16, 4>(st, a, am, m, o);
    if (va == 8) return launch_one<MODE, BN, 8, 4>(st, a, am, m, o);
    return launch_one<MODE, BN, 4, 4>(st, a, am, m, o);
  } else {
    if (va == 16) return launch_one<MODE, BN, 16, 16>(st, a, am, m, o);
    if (va == 8) return launch_one<MODE, BN, 8, 16>(st, a, am, m, o);
    return launch_one<MODE, BN, 4, 16>(st, a, am, m, o);
  }
}

template <int MODE>
static int dispatch(cudaStream_t st, const ConvArgs& a, int bn, const CUtensorMap& am, const CUtensorMap& m,
                    const CUtensorMap& o, int va, int vb) {
  if (bn == 64) return dispatch_vec<MODE, 64>(st, a, am, m, o, va, vb);
  if (bn == 128) return dispatch_vec<MODE, 128>(st, a, am, m, o, va, vb);
  return dispatch_vec<MODE, 256>(st, a, am, m, o, va, vb);
}

static int pick_bn(int64_t ng) { return ng <= 64 ? 64 : (ng <= 128 ? 128 : 256); }

// Tile width for FWD / DGRAD.
static int pick_bn_balanced(int64_t ng, int64_t m_tiles, int sms) {
  static const int force = [] {
    const char* e = getenv("I8T_FORCE_BN");  // tuning experiments: 64 / 128 / 256
    return e ? atoi(e) : 0;
  }();
  if (force == 64 || force == 128 || force == 256) return force;
  // A CTA's k-stage costs about the same whatever the tile width (the operand
  // loads, not the MMA, set its pace: B200 measurements), so a narrower tile
  // only pays when the wide one would leave most SMs idle.
  int bn = pick_bn(ng);
  while (bn > 64 && m_tiles * ((ng + bn - 1) / bn) * 2 < sms) bn /= 2;
  return bn;
}

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
  if (g->n * g->h * g->w >= (int64_t)1 << 31 || g->n * P * Q >= (int64_t)1 << 31 ||
      g->n * g->h * g->w * g->c >= (int64_t)1 << 40)
    return set_error(I8T_EUNSUPPORTED, "conv: tensor too large");
  return I8T_OK;
}

static void fill_geom(ConvArgs& x, const i8t_conv_geom* g, int64_t P, int64_t Q) {
  x.N = (int)g->n; x.H = (int)g->h; x.W = (int)g->w;
  x.R = (int)g->kh; x.S = (int)g->kw; x.sh = (int)g->stride_h; x.sw = (int)g->stride_w; x.ph = (int)g->pad_h; x.pw = (int)g->pad_w;
  x.P = (int)P; x.Q = (int)Q;
}

// Strided DGRAD as sh*sw stride-1 sub-problems: phase (fh, fw) holds the input
// pixels h = hh*sh + fh, w = ww*sw + fw; only the taps with
// (fh + ph - r) % sh == 0 and (fw + pw - s) % sw == 0 reach them, so no MMA
// runs on the zero-stuffed positions of the reference's col2im (conv.cpp:60-84).
static int dgrad_phases(Ctx* c, const i8t_conv_geom* g, int64_t P, int64_t Q, const int8_t* gz, int64_t k_pad,
                        const int8_t* wt, int64_t ld_wt, const float* clip_g, const float* clip_w, float* ga,
                        int32_t* acc, const float* add_g, const float* add_y, const uint32_t* add_bits) {
  const int sh = (int)g->stride_h, sw = (int)g->stride_w;
  for (int fh = 0; fh < sh; ++fh) {
    for (int fw = 0; fw < sw; ++fw) {
      ConvArgs x{};
      fill_geom(x, g, P, Q);
      x.act = nullptr; x.gz = gz; x.wt = wt; x.ldw = ld_wt; x.Cp = (int)g->c; x.Kp = (int)k_pad;
      x.phase = 1; x.fh = fh; x.fw = fw;
      x.Hq = (int)((g->h - fh + sh - 1) / sh);
      x.Wq = (int)((g->w - fw + sw - 1) / sw);
      if (x.Hq <= 0 || x.Wq <= 0) continue;
      x.r0 = (int)((fh + g->pad_h) % sh);
      x.s0 = (int)((fw + g->pad_w) % sw);
      const int nr = x.r0 < g->kh ? (int)((g->kh - 1 - x.r0) / sh + 1) : 0;
      x.ns = x.s0 < g->kw ? (int)((g->kw - 1 - x.s0) / sw + 1) : 0;
      x.dh = (int)((fh + g->pad_h - x.r0) / sh);
      x.dw = (int)((fw + g->pad_w - x.s0) / sw);
      x.M = g->n * x.Hq * x.Wq; x.Ng = (int)g->c;
      x.clip_x = clip_g; x.clip_y = clip_w; x.out = ga; x.ldo = g->c; x.acc32 = acc;
      x.add_g = add_g; x.add_y = add_y; x.add_bits = add_bits;
      x.use_tma_out = 0;
      if (nr == 0 || x.ns == 0) {
        // in-place join (out is the addend, no mask): the phase already holds
        // 0 + addend (up to the sign of a zero addend)
        if (x.add_g && static_cast<const void*>(x.add_g) == static_cast<const void*>(x.out) && !x.add_y &&
            !x.add_bits && !x.acc32)
          continue;
        const int blocks = (int)std::min<int64_t>((x.M + 7) / 8, 148 * 16);
        set_divs(x);
        launch_k(k_zero_phase, blocks, 256, 0, c->stream, x);
        count_launch(1);
        int rc = cuda_check("k_zero_phase");
        if (rc) return rc;
        continue;
      }
      x.Kd = (int64_t)nr * x.ns * k_pad;
      x.nr = nr;
      x.k_tiles = (int)((x.Kd + BKB - 1) / BKB);
      static const bool no_im2col = getenv("I8T_NO_IM2COL") != nullptr;
      static const bool no_prow = getenv("I8T_NO_PHASE_TMA") != nullptr;
      const bool im2col = !no_im2col && (reinterpret_cast<uintptr_t>(gz) & 15u) == 0;
      // padded phase rows + TMA stores (im2col operand only) when a phase-grid
      // row fits a quadrant (5 <= Wq <= 32) and the (n, hh) rows merge (H == sh*Hq)
      int lg = 3;
      while ((1 << lg) < x.Wq) ++lg;
      if (im2col && !no_prow && x.Wq >= 5 && lg <= 5 && g->h == static_cast<int64_t>(sh) * x.Hq &&
          tma_out_ok(ga, g->c) && (static_cast<int64_t>(x.N) * x.Hq << lg) < (int64_t(1) << 31)) {
        x.prow_lg = lg;
        x.M = static_cast<int64_t>(x.N) * x.Hq << lg;
        x.use_tma_out = 1;
      }
      x.m_tiles = (int)((x.M + BM - 1) / BM);
      const int bn = pick_bn_balanced(g->c, x.m_tiles, num_sms());
      x.n_tiles = (int)((g->c + bn - 1) / bn); x.splits = 1;
      CUtensorMap amap{}, map, omap{};
      int rc = make_weight_map(&map, wt, g->c, ld_wt, bn);
      if (rc) return rc;
      if (x.prow_lg && (rc = make_phase_out_map(&omap, ga, x, x.prow_lg))) return rc;
      if (im2col) {
        // the phase grid Hq x Wq as the pixel box over g_z [N][P][Q][k_pad]
        const int lw = x.dw - (x.ns - 1), lh = x.dh - (nr - 1);
        x.tma_a = 2;
        const int bw = x.prow_lg ? (1 << x.prow_lg) : x.Wq;  // pixel-box width (padded rows)
        if ((rc = make_im2col_map(&amap, gz, g->n, P, Q, k_pad, lw, lh, bw - (int)Q + lw, x.Hq - (int)P + lh, 1, 1)))
          return rc;
      }
      if ((rc = dispatch<MODE_DGRAD>(c->stream, x, bn, amap, map, omap, vec_of(k_pad), 16))) return rc;
    }
  }
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
  if (foldable(g, c_pad)) {
    int8_t* wf = nullptr;
    const int8_t* xf = fold_input(c, g, Q, a, static_cast<size_t>(g->k) * g->kh * 32, &wf);
    if (!xf) return set_error(I8T_ECUDA, "conv_fwd: fold buffer alloc failed");
    const int tot = (int)(g->k * g->kh * 32);
    launch_k(k_fold_weights, (tot + 255) / 256, 256, 0, c->stream, w, ld_w, (int)g->k, (int)g->kh, (int)g->kw, wf);
    count_launch(1);
    if ((rc = cuda_check("k_fold"))) return rc;
    const i8t_conv_geom f = folded_geom(g, Q);
    return i8t_conv_fwd(ctx, &f, xf, 32, wf, g->kh * 32, clip_a, clip_w, z, acc);
  }
  if (conv_sw_eligible(g, c_pad, (int)g->k, (int)P, (int)Q, a, z, ld_w))
    return conv_sw_run(c, false, g, a, c_pad, (int)g->h, (int)g->w, w, ld_w, (int)g->k, (int)P, (int)Q, clip_a, clip_w,
                       z, acc);
  ConvArgs x{};
  fill_geom(x, g, P, Q);
  x.act = a; x.gz = nullptr; x.wt = w; x.ldw = ld_w; x.Cp = (int)c_pad; x.Kp = (int)g->k;
  x.M = g->n * P * Q; x.Ng = (int)g->k; x.Kd = Kd;
  x.k_tiles = (int)((Kd + BKB - 1) / BKB);
  x.clip_x = clip_a; x.clip_y = clip_w; x.out = z; x.ldo = g->k; x.acc32 = acc;
  x.m_tiles = (int)((x.M + BM - 1) / BM);
  const int bn = pick_bn_balanced(g->k, x.m_tiles, num_sms());
  x.n_tiles = (int)((g->k + bn - 1) / bn); x.splits = 1;
  CUtensorMap amap{}, map, omap{};
  const bool pair = pair_enabled() && bn == 256 && (plain_1x1(g, a, c_pad) || im2col_ok(g, c_pad, a, P, Q));
  if ((rc = make_weight_map(&map, w, g->k, ld_w, pair ? bn / 2 : bn))) return rc;
  if (plain_1x1(g, a, c_pad)) {
    x.tma_a = 1;
    if ((rc = make_weight_map(&amap, a, x.M, c_pad, BM))) return rc;
  } else if (im2col_ok(g, c_pad, a, P, Q)) {
    x.tma_a = 2;
    if ((rc = make_im2col_map(&amap, a, g, c_pad))) return rc;
  } else if (!pair && !wg64_off() && c_pad == 32 && im2col_ok(g, c_pad, a, P, Q, 32)) {
    x.tma_a = 3;  // 32-channel taps: four SWIZZLE_32B im2col boxes per k-block (K-major SW32 descriptor)
    if ((rc = make_im2col_map(&amap, a, g, c_pad, 32u, CU_TENSOR_MAP_SWIZZLE_32B))) return rc;
  }
  x.use_tma_out = tma_out_ok(z, g->k) ? 1 : 0;
  if (x.use_tma_out && (rc = make_out_map(&omap, z, g->k, x.M, g->k, false))) return rc;
  if (pair) {
    x.m_tiles = (int)((x.M + 2 * BM - 1) / (2 * BM));
    return launch_pair<MODE_FWD, 256>(c->stream, x, amap, map, omap);
  }
  return dispatch<MODE_FWD>(c->stream, x, bn, amap, map, omap, vec_of(c_pad), 16);
}


static int dgrad_impl(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, int64_t k_pad, const int8_t* wt,
                      int64_t ld_wt, const float* clip_g, const float* clip_w, float* ga, int32_t* acc,
                      const float* add_g, const float* add_y, const uint32_t* add_bits = nullptr);

int i8t_conv_dgrad(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, int64_t k_pad, const int8_t* wt, int64_t ld_wt,
                   const float* clip_g, const float* clip_w, float* ga, int32_t* acc) {
  return dgrad_impl(ctx, g, gz, k_pad, wt, ld_wt, clip_g, clip_w, ga, acc, nullptr, nullptr);
}

int i8t_conv_dgrad_join(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, int64_t k_pad, const int8_t* wt,
                        int64_t ld_wt, const float* clip_g, const float* clip_w, float* ga, const float* add_g,
                        const float* add_y) {
  if (!ga || !add_g) return set_error(I8T_EINVAL, "conv_dgrad_join: null output or addend");
  if ((reinterpret_cast<uintptr_t>(add_g) & 15u) || (reinterpret_cast<uintptr_t>(add_y) & 15u) || (g && g->c % 4))
    return set_error(I8T_EUNSUPPORTED, "conv_dgrad_join: addends must be 16-byte aligned with c % 4 == 0");
  return dgrad_impl(ctx, g, gz, k_pad, wt, ld_wt, clip_g, clip_w, ga, nullptr, add_g, add_y);
}

int i8t_conv_dgrad_join_bits(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, int64_t k_pad, const int8_t* wt,
                             int64_t ld_wt, const float* clip_g, const float* clip_w, float* ga, const float* add_g,
                             const uint32_t* add_bits) {
  if (!ga || !add_g) return set_error(I8T_EINVAL, "conv_dgrad_join_bits: null output or addend");
  if ((reinterpret_cast<uintptr_t>(add_g) & 15u) || (g && g->c % 4))
    return set_error(I8T_EUNSUPPORTED, "conv_dgrad_join_bits: addend must be 16-byte aligned with c % 4 == 0");
  return dgrad_impl(ctx, g, gz, k_pad, wt, ld_wt, clip_g, clip_w, ga, nullptr, add_g, nullptr, add_bits);
}

}  // extern "C"

static int dgrad_impl(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, int64_t k_pad, const int8_t* wt,
                      int64_t ld_wt, const float* clip_g, const float* clip_w, float* ga, int32_t* acc,
                      const float* add_g, const float* add_y, const uint32_t* add_bits) {
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
  if ((g->stride_h > 1 || g->stride_w > 1) && k_pad % 128 == 0 && g->c % 4 == 0 && (ld_wt % 16) == 0) {
    static const bool off = getenv("I8T_NO_DGRAD_PHASE") != nullptr;
    if (!off) return dgrad_phases(c, g, P, Q, gz, k_pad, wt, ld_wt, clip_g, clip_w, ga, acc, add_g, add_y, add_bits);
  }
  if (!add_g && conv_sw_eligible(g, k_pad, (int)g->c, (int)g->h, (int)g->w, gz, ga, ld_wt))
    return conv_sw_run(c, true, g, gz, k_pad, (int)P, (int)Q, wt, ld_wt, (int)g->c, (int)g->h, (int)g->w, clip_g,
                       clip_w, ga, acc);
  ConvArgs x{};
  fill_geom(x, g, P, Q);
  x.act = nullptr; x.gz = gz; x.wt = wt; x.ldw = ld_wt; x.Cp = (int)g->c; x.Kp = (int)k_pad;
  x.M = g->n * g->h * g->w; x.Ng = (int)g->c; x.Kd = Kd;
  x.k_tiles = (int)((Kd + BKB - 1) / BKB);
  x.clip_x = clip_g; x.clip_y = clip_w; x.out = ga; x.ldo = g->c; x.acc32 = acc;
  x.add_g = add_g; x.add_y = add_y; x.add_bits = add_bits;
  x.m_tiles = (int)((x.M + BM - 1) / BM);
  const int bn = pick_bn_balanced(g->c, x.m_tiles, num_sms());
  x.n_tiles = (int)((g->c + bn - 1) / bn); x.splits = 1;
  CUtensorMap amap{}, map, omap{};
  const bool dg_im2col = g->stride_h == 1 && g->stride_w == 1 && im2col_ok(g, k_pad, gz, P, Q) &&
                         P + g->kh - 1 - 2 * g->pad_h == g->h && Q + g->kw - 1 - 2 * g->pad_w == g->w;
  const bool pair = pair_enabled() && bn == 256 && (plain_1x1(g, gz, k_pad) || dg_im2col) && !add_g;
  if ((rc = make_weight_map(&map, wt, g->c, ld_wt, pair ? bn / 2 : bn))) return rc;
  if (plain_1x1(g, gz, k_pad)) {
    x.tma_a = 1;
    if ((rc = make_weight_map(&amap, gz, x.M, k_pad, BM))) return rc;
  } else if (dg_im2col) {
    // g_z [N][P][Q][k_pad] traversed over the input positions: box [-(S-1-pw), Q-1-pw]
    x.tma_a = 2;
    if ((rc = make_im2col_map(&amap, gz, g->n, P, Q, k_pad, static_cast<int>(-(g->kw - 1 - g->pad_w)),
                              static_cast<int>(-(g->kh - 1 - g->pad_h)), static_cast<int>(-g->pad_w),
                              static_cast<int>(-g->pad_h), 1, 1)))
      return rc;
  }
  x.use_tma_out = tma_out_ok(ga, g->c) ? 1 : 0;
  if (x.use_tma_out && (rc = make_out_map(&omap, ga, g->c, x.M, g->c, false))) return rc;
  if (pair) {
    x.m_tiles = (int)((x.M + 2 * BM - 1) / (2 * BM));
    return launch_pair<MODE_DGRAD, 256>(c->stream, x, amap, map, omap);
  }
  return dispatch<MODE_DGRAD>(c->stream, x, bn, amap, map, omap, vec_of(k_pad), 16);
}

extern "C" {

int i8t_conv_wgrad(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, int64_t k_pad, const int8_t* a, int64_t c_pad,
                   const float* clip_g, const float* clip_a, int64_t* acc, float* gw, int out_kcrs) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  int64_t P, Q;
  int rc = geom_common(g, P, Q);
  if (rc) return rc;
  if (!c || !gz || !a || !clip_g || !clip_a || (!acc && !gw)) return set_error(I8T_EINVAL, "conv_wgrad: null argument");
  if (g->depthwise) return set_error(I8T_EINVAL, "conv_wgrad: use i8t_conv_dw_wgrad for depthwise");
  if (c_pad < g->c || c_pad % 4 != 0 || k_pad < g->k || k_pad % 4 != 0)
    return set_error(I8T_EUNSUPPORTED, "conv_wgrad: channel strides must be multiples of 4");
  if (foldable(g, c_pad)) {
    int8_t* ex = nullptr;
    const int8_t* xf = fold_input(c, g, Q, a, sizeof(long long) * static_cast<size_t>(g->kh * 32 * g->k), &ex);
    if (!xf) return set_error(I8T_ECUDA, "conv_wgrad: fold buffer alloc failed");
    int64_t* accf = reinterpret_cast<int64_t*>(ex);
    const i8t_conv_geom f = folded_geom(g, Q);
    if ((rc = i8t_conv_wgrad(ctx, &f, gz, k_pad, xf, 32, clip_g, clip_a, accf, nullptr, out_kcrs))) return rc;
    const int tot = (int)(g->kh * g->kw * 4 * g->k);
    if (!acc) acc = reinterpret_cast<int64_t*>(ensure_scratch(c, sizeof(long long) * static_cast<size_t>(tot)));
    if (!acc) return set_error(I8T_ECUDA, "conv_wgrad: scratch alloc failed");
    launch_k(k_unfold_wacc, (tot + 255) / 256, 256, 0, c->stream, reinterpret_cast<const long long*>(accf), (int)g->kh,
                                                            (int)g->kw, (int)g->k, reinterpret_cast<long long*>(acc));
    count_launch(1);
    if ((rc = cuda_check("k_unfold_wacc"))) return rc;
    return gw ? i8t_conv_wgrad_finalize(ctx, g, acc, c_pad, clip_g, clip_a, gw, out_kcrs) : I8T_OK;
  }
  ConvArgs x{};
  fill_geom(x, g, P, Q);
  x.act = a; x.gz = gz; x.wt = nullptr; x.ldw = 0; x.Cp = (int)c_pad; x.Kp = (int)k_pad;
  x.M = g->kh * g->kw * c_pad; x.Ng = (int)g->k; x.Kd = g->n * P * Q;
  const int bn = pick_bn(g->k);
  const int64_t m_tiles = (x.M + BM - 1) / BM, n_tiles = (g->k + bn - 1) / bn;
  const int64_t total_kt = (x.Kd + BKB - 1) / BKB;
  // split the npq reduction (<= 1015 k-tiles = 129,920 rows per split keeps each
  // int32 partial exact): pick the split count minimising
  //   waves * (k-tiles per split + C0),  waves = ceil(tiles / SMs),
  // C0 ~ the per-tile prologue + partial write-out in k-tile units.
  const int64_t mn = m_tiles * n_tiles, sms = num_sms();
  static const int c0 = [] {
    const char* e = getenv("I8T_WGRAD_C0");
    return e ? atoi(e) : 6;
  }();
  int64_t per = total_kt, best = -1;
  for (int64_t sp = (total_kt + 1014) / 1015; sp <= total_kt; ++sp) {
    const int64_t pk = (total_kt + sp - 1) / sp;
    if (pk < 8 && sp > 1) break;
    const int64_t nsp = (total_kt + pk - 1) / pk;  // splits actually used
    const int64_t waves = (mn * nsp + sms - 1) / sms;
    const int64_t cost = waves * (pk + c0);
    if (best < 0 || cost < best) {
      best = cost;
      per = pk;
    }
    if (mn * nsp > 16 * sms) break;
  }
  int64_t splits = (total_kt + per - 1) / per;
  x.k_tiles = (int)per;
  x.m_tiles = (int)m_tiles; x.n_tiles = (int)n_tiles; x.splits = (int)splits;
  x.m_pad = (int)(m_tiles * BM);
  x.clip_x = clip_g; x.clip_y = clip_a;
  // per-split int32 partial tiles [splits][m_pad][k_pad], TMA-stored, reduced below in a fixed order
  const size_t part_bytes = sizeof(int32_t) * static_cast<size_t>(splits) * x.m_pad * k_pad;
  int32_t* part = reinterpret_cast<int32_t*>(ensure_wgrad(c, part_bytes));
  if (!part) return set_error(I8T_ECUDA, "wgrad workspace alloc failed");
  CUtensorMap amap{}, map{}, omap{};  // no weight operand in WGRAD: tmap_b carries g_z in TMA mode
  if (plain_1x1(g, a, c_pad, gz, k_pad)) {
    x.tma_a = 1;
    if ((rc = make_weight_map(&amap, a, x.Kd, c_pad, BKB))) return rc;   // [npq][c_pad], box {128 ch, 128 rows}
  } else if (im2col_ok(g, c_pad, a, P, Q) && k_pad % 16 == 0 && (reinterpret_cast<uintptr_t>(gz) & 15u) == 0) {
    x.tma_a = 2;  // A = im2col of the activations (128 npq rows x 128 channels of one tap), B = g_z rows
    if ((rc = make_im2col_map(&amap, a, g, c_pad))) return rc;
  } else if (!wg64_off() && im2col_ok(g, c_pad, a, P, Q, 32) && k_pad % 16 == 0 &&
             (reinterpret_cast<uintptr_t>(gz) & 15u) == 0 && x.M >= (c_pad % 64 == 0 ? 64 : 32)) {
    // 64 / 32-channel blocks: 2 / 4 im2col boxes per m-tile (SWIZZLE_64B / 32B,
    // MN-major SW64 / SW32 descriptor) -- the 64-channel layers, the stem's folded taps
    x.tma_a = 3;
    x.wg_cb = c_pad % 64 == 0 ? 64 : 32;
    if ((rc = make_im2col_map(&amap, a, g, c_pad, static_cast<uint32_t>(x.wg_cb),
                              x.wg_cb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B)))
      return rc;
  }
  static const bool no_tma_b = getenv("I8T_NO_TMA_A") != nullptr;
  if (x.tma_a || (!no_tma_b && k_pad % 16 == 0 && (reinterpret_cast<uintptr_t>(gz) & 15u) == 0)) {
    x.tma_b = !x.tma_a;
    if ((rc = make_weight_map(&map, gz, x.Kd, k_pad, BKB))) return rc;   // [npq][k_pad], box {128 k, 128 rows}
  }
  x.use_tma_out = 1;
  if ((rc = make_out_map(&omap, part, k_pad, splits * x.m_pad, k_pad, true))) return rc;
  rc = dispatch<MODE_WGRAD>(c->stream, x, bn, amap, map, omap, vec_of(c_pad), vec_of(k_pad));
  if (rc) return rc;
  const int64_t tot = x.M * g->k;
  if (tot < 148 * 256 * 2 && splits >= 8) {  // too few outputs to fill the GPU one per thread
    int blocks = (int)((tot + 31) / 32);
    if (blocks > 148 * 16) blocks = 148 * 16;
    launch_k(k_wgrad_reduce_split<8>, blocks, 256, 0, c->stream, part, (int)splits, x.m_pad, (int)k_pad, (int)x.M,
             (int)g->k, (int)g->c, (int)c_pad, (int)(g->kh * g->kw), reinterpret_cast<long long*>(acc), clip_g, clip_a,
             gw, out_kcrs);
    count_launch(1);
    return cuda_check("k_wgrad_reduce_split");
  }
  int blocks = (int)((tot + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  launch_k(k_wgrad_reduce, blocks, 256, 0, c->stream, part, (int)splits, x.m_pad, (int)k_pad, (int)x.M, (int)g->k, (int)g->c,
                                                 (int)c_pad, (int)(g->kh * g->kw), reinterpret_cast<long long*>(acc),
                                                 clip_g, clip_a, gw, out_kcrs);
  count_launch(1);
  return cuda_check("k_wgrad_reduce");
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
  launch_k(k_wgrad_finalize, blocks, 256, 0, c->stream, reinterpret_cast<const long long*>(acc), (int)g->k, (int)g->c,
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
  launch_k(k_transpose_i8, (unsigned)std::min<int64_t>((k * n + 255) / 256, 4096), 256, 0, c->stream, b, k, n, bt, ldw);
  count_launch(1);
  if (ap) {
    launch_k(k_pad_rows_i8, (unsigned)std::min<int64_t>((m * kp + 255) / 256, 4096), 256, 0, c->stream, a, m, k, ap, kp);
    count_launch(1);
  }
  i8t_conv_geom g{m, kp, 1, 1, n, 1, 1, 1, 1, 0, 0, 0, 1};
  int rc = i8t_conv_fwd(ctx, &g, ap ? ap : a, kp, bt, ldw, ones, ones + 1, nullptr, cout);
  cudaStreamSynchronize(c->stream);  // h127 lives on this stack frame
  return rc;
}

// gemm_i8_fused_lhs (gemm.cpp:49-64): quantise the fp32 lhs on the device --
// nearest, or stochastic with the draws in row-major order from the device
// LCG state (advanced by m*k) -- straight into the GEMM's A operand (an int8
// copy of m*k bytes that stays in L2 for the GEMM that follows), then the
// tcgen05 GEMM.  Bit-identical to quantize() + gemm_i8() incl. the stream.
int i8t_gemm_s8_fused_lhs(i8t_ctx* ctx, const float* a, int64_t m, int64_t k, const float* clip, int stochastic,
                          uint32_t* lcg_state, const int8_t* b, int64_t n, int32_t* cout) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !a || !b || !cout || !clip || m < 1 || k < 1 || n < 1 || (stochastic && !lcg_state))
    return set_error(I8T_EINVAL, "gemm_i8_fused_lhs: bad arguments");
  if (k > 130000) return set_error(I8T_EINVAL, "gemm_i8: depth exceeds i32 overflow bound");
  int8_t* qa = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&qa), (size_t)(m * k), c->stream) != cudaSuccess)
    return set_error(I8T_ECUDA, "gemm_i8_fused_lhs: alloc failed");
  int rc = stochastic ? i8t_quantize_stochastic(ctx, a, m * k, clip, lcg_state, qa)
                      : i8t_quantize_nearest(ctx, a, m * k, clip, qa, nullptr, 0);
  if (rc == I8T_OK) rc = i8t_gemm_s8(ctx, qa, b, m, k, n, cout);
  cudaFreeAsync(qa, c->stream);
  return rc;
}

}  // extern "C"
