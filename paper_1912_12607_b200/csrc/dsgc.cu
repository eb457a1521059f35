// dsgc.cu -- gradient side of the INT8 path on sm_100a:
//   K3  fused gradient quantiser (quantize_gradient, layers.cpp:19-59): one
//       pass over g computes max|g|, the non-finite flag, the nearest-rounding
//       d_c sums at the current clip (Periodic-Update measurement, clip.cpp:90),
//       the stochastic int8 payload and the eps / g_hat statistics;
//   K4  d_c sums for up to 32 candidate clips per pass, driving the DSGC
//       search state machine (search_clip, clip.cpp:30-78);
//   the plain reductions of tensor.cpp:72-101 and cosine_distance.
// HBM-bound: float4 loads, char4 stores, warp-shuffle + fixed-order block
// reductions, one grid-wide "last block finishes" reduction per pass (no extra
// launch), optional allreduce hook between passes for data parallelism.
//
// LCG draw order: the reference draws once per element in row-major NCHW
// order from one caller-owned stream (quantize.cpp:38-41).  Element
// (n, c, hw) of a channels-last tensor uses draw index (n*C + c)*HW + hw.  A
// thread owns a fixed channel quad and steps by a constant number of pixels,
// so its LCG state advances by a constant affine map (plus a fixed map per
// image wrap) -- one IMAD per element, no tables.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "internal.cuh"
#include "qcore.cuh"
#include "qgrad.cuh"

namespace i8t_dev {

// K4.  totals: [0] max|g|, [1] nonfinite, [2] sum g^2, [3+2j] sum g*gh_j, [4+2j] sum gh_j^2.
// NC == 0: the first three only.
__global__ void __launch_bounds__(RED_THREADS) k_dc_stats0(const float* __restrict__ g, uint32_t n, double* partials,
                                                           double* totals, unsigned* ticket) {
  pdl_entry();
  double acc[3] = {0.0, 0.0, 0.0};
  float m = 0.0f;
  bool bad = false;
  auto body = [&](float v) {
    bad |= !isfinite(v);
    m = fmaxf(m, fabsf(v));
    const double vd = v;
    acc[2] = fma(vd, vd, acc[2]);
  };
  const uint32_t stride = gridDim.x * blockDim.x, n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  constexpr int U = 4;  // float4 loads in flight per thread (HBM-bound passes)
  uint32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if constexpr (U > 1)
  for (; f + (U - 1) * stride < n4; f += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(g4 + f + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      body(v[u].x);
      body(v[u].y);
      body(v[u].z);
      body(v[u].w);
    }
  }
  for (; f < n4; f += stride) {
    const float4 v = __ldg(g4 + f);
    body(v.x);
    body(v.y);
    body(v.z);
    body(v.w);
  }
  for (uint32_t i = n4 * 4 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) body(g[i]);
  acc[0] = m;
  acc[1] = bad ? 1.0 : 0.0;
  grid_reduce<3>(acc, 1u, partials, totals, ticket);
}

// Candidates in groups of NG per blockIdx.y (every group streams g once): the
// per-element work is NG nearest quantisations (FMA-pipe fast path, the exact
// function for an element near a tie of any of its candidates), NG table
// lookups and 2*NG FMAs, in registers small enough for three blocks per SM.
// Group y reduces over blockIdx.x into its own partials / ticket, and its last
// block scatters the candidate sums (and, for y == 0, [0..2]) into totals.
__device__ __noinline__ void search_step_dev(DsgcState* st, const double* tot, int nc, int R, int rounds);

// STATS = false (the search passes after k_search_begin): max|g|, the
// non-finite flag and sum g^2 are already known; only the candidate sums run.
template <int NG, bool STATS>
__global__ void __launch_bounds__(RED_THREADS, 3) k_dc_stats(const float* __restrict__ g, uint32_t n,
                                                          const float* __restrict__ cands, int nc,
                                                          const int32_t* active, double* partials, double* gtot,
                                                          double* totals, unsigned* tickets, DsgcState* step_st,
                                                          int R, int rounds) {
  pdl_entry();
  constexpr int NV = 3 + 2 * NG;
  if (active && *active == 0) return;  // uniform across the grid: nobody takes a ticket
  // NG <= 2 (memory-bound passes): dequantisation tables as separate high / low
  // 32-bit words -- a lane's two 4-byte loads conflict only for entries 32
  // apart, an 8-byte load from a double table for entries 16 apart (9.4 -> 6.8 ms
  // for the single-candidate passes of a ResNet-50 search step).  NG = 8 is
  // issue-bound: one 8-byte load per candidate beats two 4-byte loads there.
  constexpr bool SPLIT = NG <= 2;
  __shared__ uint32_t dq_w[NG * 512];  // SPLIT: [hi words | lo words] per candidate; else doubles
  const int j0 = blockIdx.y * NG;
  float hs[NG];
  bool tiny = false;  // a subnormal candidate scale: the exact function for every element
  uint32_t tab_n[NG];  // table entry of q at the qn_bits pattern RMAGIC + q + 1 (32-bit wrap)
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(dq_w));
#pragma unroll
  for (int j = 0; j < NG; ++j) {
    const float cl = cands[min(j0 + j, nc - 1)];  // past nc: a duplicate, never scattered
    hs[j] = __fdiv_rn(0.5f, cl);
    tiny |= !(scale_of(cl) >= 0x1p-126f);
    const float sc = scale_of(cl);
    for (int i = threadIdx.x; i < 255; i += blockDim.x) {
      const double d = __fmul_rn(static_cast<float>(i - 127), sc);
      if (SPLIT) {
        dq_w[j * 512 + i] = static_cast<uint32_t>(__double2hiint(d));
        dq_w[j * 512 + 256 + i] = static_cast<uint32_t>(__double2loint(d));
      } else {
        reinterpret_cast<double*>(dq_w)[j * 256 + i] = d;
      }
    }
    tab_n[j] = SPLIT ? base + 4u * (j * 512u + 126u - RMAGIC_BITS) : base + 8u * (j * 256u + 126u - RMAGIC_BITS);
  }
  __syncthreads();
  double acc[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) acc[j] = 0.0;
  float m = 0.0f;
  bool bad = false;
  auto body = [&](float v) {
    if (STATS) {
      bad |= !isfinite(v);
      m = fmaxf(m, fabsf(v));
    }
    const double vd = v;
    if (STATS) acc[2] = fma(vd, vd, acc[2]);
    uint32_t kb[NG];
    bool slow = tiny;
#pragma unroll
    for (int j = 0; j < NG; ++j) kb[j] = qn_bits(q_t1(v, hs[j]), slow);
    if (slow) {
#pragma unroll
      for (int j = 0; j < NG; ++j) {
        const float cl = cands[min(j0 + j, nc - 1)], sc = scale_of(cl);
        kb[j] = static_cast<uint32_t>(RMAGIC_BITS + 1 + quant_nearest(v, cl, sc, 1.0f / sc));
      }
    }
#pragma unroll
    for (int j = 0; j < NG; ++j) {
      double gh;
      if (SPLIT) {
        const uint32_t a = tab_n[j] + 4u * kb[j];
        gh = __hiloint2double(static_cast<int>(lds_u32(a)), static_cast<int>(lds_u32(a + 1024u)));
      } else {
        gh = lds_f64(tab_n[j] + 8u * kb[j]);
      }
      acc[3 + 2 * j] = fma(vd, gh, acc[3 + 2 * j]);
      acc[4 + 2 * j] = fma(gh, gh, acc[4 + 2 * j]);
    }
  };
  const uint32_t stride = gridDim.x * blockDim.x, n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  constexpr int U = NG <= 4 ? 4 : 1;  // float4 loads in flight per thread (HBM-bound passes)
  uint32_t f = blockIdx.x * blockDim.x + threadIdx.x;
  if constexpr (U > 1)
  for (; f + (U - 1) * stride < n4; f += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(g4 + f + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      body(v[u].x);
      body(v[u].y);
      body(v[u].z);
      body(v[u].w);
    }
  }
  for (; f < n4; f += stride) {
    const float4 v = __ldg(g4 + f);
    body(v.x);
    body(v.y);
    body(v.z);
    body(v.w);
  }
  for (uint32_t i = n4 * 4 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) body(g[i]);
  acc[0] = m;
  acc[1] = bad ? 1.0 : 0.0;
  double* gt = gtot + blockIdx.y * NV;
  if (!grid_reduce<NV>(acc, 1u, partials + static_cast<size_t>(blockIdx.y) * gridDim.x * NV, gt,
                       tickets + blockIdx.y))
    return;
  const int ncg = min(NG, nc - j0);
  for (int t = threadIdx.x; t < 2 * ncg; t += blockDim.x) totals[3 + 2 * j0 + t] = __ldcg(gt + 3 + t);
  if (STATS && blockIdx.y == 0 && threadIdx.x < 3) totals[threadIdx.x] = __ldcg(gt + threadIdx.x);
  if (step_st) {  // one group, no allreduce: the last block runs the search step itself
    __syncthreads();
    if (threadIdx.x == 0) search_step_dev(step_st, totals, nc, R, rounds);
  }
}

// ---- DSGC search state machine (clip.cpp:30-78), one thread, on totals.
__device__ __forceinline__ void ds_consider(DsgcState* st, float c, double dc) {
  if (!(c > 0.0f)) return;
  if (dc < st->best_dc || (dc == st->best_dc && c > st->best_clip)) {
    st->best_clip = c;
    st->best_dc = dc;
  }
}
__device__ __forceinline__ void ds_track(DsgcState* st, double x, double f) {
  if (f < st->best_dc || (f == st->best_dc && static_cast<float>(x) > st->best_clip)) {
    st->best_clip = static_cast<float>(x);
    st->best_dc = f;
  }
}
__device__ __forceinline__ void ds_grid_chunk(DsgcState* st, int R) {
  const int left = R - st->grid_done;
  const int nc = left < 32 ? left : 32;
  for (int j = 0; j < nc; ++j) {
    const int i = st->grid_done + j + 1;
    st->cand[j] = __fmul_rn(st->m, __fdiv_rn(static_cast<float>(i), static_cast<float>(R)));
  }
  st->ncand = nc;
}
constexpr double kInvPhi = 0.6180339887498949;

// After the k_dc_stats<0> pass: m, non-finite, sum g^2 (clip.cpp:32-34).
__global__ void k_search_begin(DsgcState* st, const double* tot, int R, float prev_clip, int prev_from_state, int* err) {
  pdl_entry();
  if (threadIdx.x) return;
  if (prev_from_state) prev_clip = st->v.clip;
  st->m = static_cast<float>(tot[0]);
  st->v.max_abs = st->m;
  st->sq_g = tot[2];
  st->prev_clip = prev_clip;
  st->best_clip = 0.0f;
  st->best_dc = 3.0;
  st->grid_done = 0;
  st->phase = 0;
  if (st->m == 0.0f || tot[1] > 0.0) {
    if (st->m != 0.0f) atomicOr(err, ERR_NONFINITE);
    st->active = 0;  // all-zero g: {prev_clip, 0}
    st->best_clip = prev_clip;
    st->best_dc = 0.0;
    return;
  }
  st->active = 1;
  ds_grid_chunk(st, R);
}

// After a k_dc_stats<nc> pass over st->cand.
__device__ __noinline__ void search_step_dev(DsgcState* st, const double* tot, int nc, int R, int rounds) {
  if (st->active == 0) return;
  double dcs[32];
  for (int j = 0; j < nc; ++j) dcs[j] = cosine_from(tot[3 + 2 * j], st->sq_g, tot[4 + 2 * j]);
  if (st->phase == 0) {  // grid
    for (int j = 0; j < nc; ++j) ds_consider(st, st->cand[j], dcs[j]);
    st->grid_done += nc;
    if (st->grid_done < R) {
      ds_grid_chunk(st, R);
      return;
    }
    if (rounds <= 0) {
      st->active = 0;
      return;
    }
    const double step = static_cast<double>(st->m) / R;
    double lo = static_cast<double>(st->best_clip) - step;
    double hi = static_cast<double>(st->best_clip) + step;
    lo = lo < 0.0 ? 0.0 : lo;
    hi = hi > static_cast<double>(st->m) ? static_cast<double>(st->m) : hi;
    st->lo = lo;
    st->hi = hi;
    // x1 = hi - (hi-lo)*kInvPhi, x2 = lo + (hi-lo)*kInvPhi, FMA-contracted like the reference build
    st->x1 = __fma_rn(-(hi - lo), kInvPhi, hi);
    st->x2 = __fma_rn(hi - lo, kInvPhi, lo);
    // the first golden-section round's two possible probes ride along with
    // x1 and x2 in the same pass: f1 < f2 probes A, else B
    const double A = __fma_rn(-(st->x2 - lo), kInvPhi, st->x2);
    const double B = __fma_rn(hi - st->x1, kInvPhi, st->x1);
    st->cand[0] = static_cast<float>(st->x1);
    st->cand[1] = static_cast<float>(st->x2);
    st->cand[2] = static_cast<float>(A);
    st->cand[3] = static_cast<float>(B);
    st->ncand = 4;
    st->phase = 1;
    return;
  }
  if (st->phase == 1) {  // x1, x2 and round 1 (clip.cpp:57-75)
    st->f1 = dcs[0];
    st->f2 = dcs[1];
    ds_track(st, st->x1, st->f1);
    ds_track(st, st->x2, st->f2);
    if (st->f1 < st->f2) {
      st->hi = st->x2;
      st->x2 = st->x1;
      st->f2 = st->f1;
      st->x1 = __fma_rn(-(st->hi - st->lo), kInvPhi, st->hi);
      st->f1 = dcs[2];
      ds_track(st, st->x1, st->f1);
    } else {
      st->lo = st->x1;
      st->x1 = st->x2;
      st->f1 = st->f2;
      st->x2 = __fma_rn(st->hi - st->lo, kInvPhi, st->lo);
      st->f2 = dcs[3];
      ds_track(st, st->x2, st->f2);
    }
    st->phase = 2;
  } else if (st->pad_ == 0) {
    st->f1 = dcs[0];
    ds_track(st, st->x1, st->f1);
  } else {
    st->f2 = dcs[0];
    ds_track(st, st->x2, st->f2);
  }
  if (st->phase - 1 >= rounds) {
    st->active = 0;
    return;
  }
  if (st->f1 < st->f2) {
    st->hi = st->x2;
    st->x2 = st->x1;
    st->f2 = st->f1;
    st->x1 = __fma_rn(-(st->hi - st->lo), kInvPhi, st->hi);
    st->cand[0] = static_cast<float>(st->x1);
    st->pad_ = 0;
  } else {
    st->lo = st->x1;
    st->x1 = st->x2;
    st->f1 = st->f2;
    st->x2 = __fma_rn(st->hi - st->lo, kInvPhi, st->lo);
    st->cand[0] = static_cast<float>(st->x2);
    st->pad_ = 1;
  }
  st->ncand = 1;
  st->phase += 1;
}

// The state machine as its own one-thread launch: after an allreduce of the
// totals (data parallel) or after the per-candidate grid pass; skipped when
// *only_if == 0 (the histogram finaliser already ran it).
__global__ void k_search_step(DsgcState* st, const double* tot, int nc, int R, int rounds, const int32_t* only_if) {
  pdl_entry();
  if (threadIdx.x || (only_if && *only_if == 0)) return;
  search_step_dev(st, tot, nc, R, rounds);
}

// End of maybe_update's search branch (clip.cpp:84-88) or a raw search_clip.
__global__ void k_search_end(DsgcState* st, int64_t iter, int update_state, float* clip_out, double* dc_out) {
  pdl_entry();
  if (threadIdx.x) return;
  const float c = st->best_clip;
  const double dc = st->best_dc;
  if (clip_out) *clip_out = c;
  if (dc_out) *dc_out = dc;
  if (update_state) {
    if (c > 0.0f) st->v.clip = c;
    st->v.last_dc = dc;
    st->v.iter_of_last_update = iter;
  }
}

// Search-disabled branch of quantize_gradient (layers.cpp:27-36): clip = max_abs.
__global__ void k_clip_from_max(DsgcState* st, const double* tot, int64_t iter) {
  pdl_entry();
  if (threadIdx.x) return;
  const float mf = static_cast<float>(tot[0]);
  if (mf > 0.0f) st->v.clip = mf;
  st->v.iter_of_last_update = iter;
}

// Non-search branch of maybe_update: last_dc = max_abs == 0 ? 0 : measure_dc.
__global__ void k_fin_maybe_dc(DsgcState* st, const double* tot, int* err) {
  pdl_entry();
  if (threadIdx.x) return;
  const float m = static_cast<float>(tot[0]);
  st->v.max_abs = m;
  if (m == 0.0f) {
    st->v.last_dc = 0.0;
    return;
  }
  if (tot[1] > 0.0) atomicOr(err, ERR_NONFINITE);
  st->v.last_dc = cosine_from(tot[3], tot[2], tot[4]);
}

__global__ void k_fin_scalar(const double* tot, int which, float* out_f, double* out_d, int32_t* out_i) {
  pdl_entry();
  if (threadIdx.x) return;
  const double v = tot[which];
  if (out_f) *out_f = static_cast<float>(v);
  if (out_d) *out_d = v;
  if (out_i) *out_i = v > 0.0 ? 1 : 0;
}

__global__ void k_fin_measure_dc(const double* tot, double* out, int* err) {
  pdl_entry();
  if (threadIdx.x) return;
  if (tot[1] > 0.0) atomicOr(err, ERR_NONFINITE);
  *out = cosine_from(tot[3], tot[2], tot[4]);
}

// dot / cosine totals: [0] sum a*b [1] sum a^2 [2] sum b^2
__global__ void __launch_bounds__(RED_THREADS) k_dot3(const float* __restrict__ a, const float* __restrict__ b,
                                                      uint32_t n, double* partials, double* totals, unsigned* ticket) {
  pdl_entry();
  double acc[3] = {0, 0, 0};
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double x = a[i], y = b[i];
    acc[0] = fma(x, y, acc[0]);
    acc[1] = fma(x, x, acc[1]);
    acc[2] = fma(y, y, acc[2]);
  }
  grid_reduce<3>(acc, 0u, partials, totals, ticket);
}

__global__ void k_fin_cosine(const double* tot, double* dot_out, double* cos_out) {
  pdl_entry();
  if (threadIdx.x) return;
  if (dot_out) *dot_out = tot[0];
  if (cos_out) *cos_out = cosine_from(tot[0], tot[1], tot[2]);
}

// max|x| over the finite samples (the histogram range) into totals[0].
__global__ void __launch_bounds__(RED_THREADS) k_finite_absmax(const float* __restrict__ x, uint32_t n,
                                                               double* partials, double* totals, unsigned* ticket) {
  pdl_entry();
  float m = 0.0f;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float a = fabsf(__ldg(x + i));
    if (a < __uint_as_float(0x7F800000u)) m = fmaxf(m, a);  // NaN and inf fail the compare
  }
  double acc[1] = {m};
  grid_reduce<1>(acc, 1u, partials, totals, ticket);
}

// Histogram of x over `bins` uniform bins of [-m, m], m = max|x| over the
// finite samples (k_finite_absmax); [-1, 1] when m == 0 (stats.hpp:11-20,
// declared there without an implementation).  Bin of v: floor((v - lo) /
// (hi - lo) * bins) in double, clamped to [0, bins - 1]; non-finite samples
// are not counted.  Per-block smem counts, one 64-bit atomic per bin per block.
__global__ void __launch_bounds__(256) k_histogram(const float* __restrict__ x, uint32_t n, const double* totals,
                                                   int bins, unsigned long long* counts, double* lo_hi) {
  pdl_entry();
  extern __shared__ unsigned int hcount[];
  for (int b = threadIdx.x; b < bins; b += blockDim.x) hcount[b] = 0u;
  const double m = static_cast<double>(static_cast<float>(totals[0]));
  const double lo = m > 0.0 ? -m : -1.0, hi = m > 0.0 ? m : 1.0;
  const double scale = static_cast<double>(bins) / (hi - lo);
  __syncthreads();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const float v = __ldg(x + i);
    if (!isfinite(v)) continue;
    int b = static_cast<int>(floor((static_cast<double>(v) - lo) * scale));
    b = b < 0 ? 0 : (b >= bins ? bins - 1 : b);
    atomicAdd(&hcount[b], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < bins; b += blockDim.x)
    if (hcount[b]) atomicAdd(counts + b, static_cast<unsigned long long>(hcount[b]));
  if (blockIdx.x == 0 && threadIdx.x == 0 && lo_hi) {
    lo_hi[0] = lo;
    lo_hi[1] = hi;
  }
}

// ---- K4H: the grid pass of search_clip (clip.cpp:45-46) as one histogram pass.
//
// For the R <= 32 grid candidates c_i = m * (i/R), quantize_value kNearest
// (quantize.cpp:16-31) is a step function of |g|: q_i(x) >= q + 1 exactly
// when x >= b_{i,q}, the smallest float with that property (monotone: the
// exact round-half-away of x/s_i).  The R*127 boundaries, sorted, cut |g| into
// fine bins; every element of fine bin F (F boundaries <= x) has the same q_i
// for every candidate, so
//   sum g*g_hat_i = sum_F tab_i(q_i(F)) * (sum of |g| over F),
//   sum g_hat_i^2 = sum_F tab_i(q_i(F))^2 * count(F)
// (g_hat keeps g's sign).  One pass over g bins the elements (count and an
// exact fixed-point sum of |g| per bin: integer adds, order-independent);
// a one-block finaliser walks the bins per candidate.  The sums are the
// reference's double sums up to their rounding (the reference's own
// accumulation error), like the per-candidate passes they replace.
//
// Bin lookup: cell(x) = min(floor(x*K + 1/2), tmax) with K = 254 R / m puts
// every boundary (~ (2q+1) i / K) mid-cell; lut[t] = first boundary with
// cell >= t.  cell() is monotone, so only the boundaries of x's own cell are
// compared with x (usually 0-2).
constexpr int HR_MAX = 32;
constexpr int HNB_PAD = 4096;                    // >= HR_MAX * 127, power of two (bitonic sort)
constexpr int HCELLS = 2 * 127 * HR_MAX + 4;     // cells 0..tmax = 2*127*R + 1, plus lut[tmax + 1]
constexpr int HIST_THREADS = 512;

struct HistBuf {
  int fail;  // a boundary search gave up (never observed): per-candidate passes; cleared by k_hist_final
  float K;
  int nb;    // R * 127 boundaries
  int e0;    // biased exponent of the smallest boundary: |g| >= B[0] is a multiple of 2^(e0 - 150)
  int tmax;
  float s[HR_MAX];
  float B[HNB_PAD];
  alignas(16) uint32_t Bu[HNB_PAD];  // b_{i,q} bits at (i-1)*127 + q, unsorted
  uint16_t pos[HNB_PAD];  // sorted position of b_{i,q} at (i-1)*127 + q
  uint8_t tag[HNB_PAD];   // candidate (i-1) of the boundary at each sorted position
  uint16_t lut[HCELLS];
  unsigned long long cnt[HNB_PAD + 1];
  unsigned long long sum[3][HNB_PAD + 1];  // fixed-point |g| sums of the digits at bits 0, 14, 28
};

__device__ __forceinline__ int hist_cell(float x, float K, int tmax) {
  return min(__float2int_rz(__fmaf_rn(x, K, 0.5f)), tmax);
}

// Setup, part 1 (R blocks of 128 threads, thread q of block i-1): the exact
// boundary b_{i,q}, the smallest float with quantize_value(x, c_i) >= q + 1,
// found by stepping from (q + 1/2) s_i (within an ulp or two); the blocks also
// clear the global bins.
__device__ __forceinline__ bool hist_ok(const DsgcState* st, int R) {
  // below 2^-100 the candidate scales approach the float-subnormal range: per-candidate passes
  const float m = st->m;
  return st->active != 0 && R >= 1 && R <= HR_MAX && m >= 0x1p-100f && m <= 3.4e38f;
}
__device__ __forceinline__ float hist_cand(float m, int i, int R) {  // ds_grid_chunk, i = 1..R
  return __fmul_rn(m, __fdiv_rn(static_cast<float>(i), static_cast<float>(R)));
}
__global__ void __launch_bounds__(128) k_hist_bounds(const DsgcState* st, int R, HistBuf* hb) {
  pdl_entry();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= HNB_PAD; i += gridDim.x * blockDim.x) {
    hb->cnt[i] = 0ull;
    hb->sum[0][i] = 0ull;
    hb->sum[1][i] = 0ull;
    hb->sum[2][i] = 0ull;
  }
  if (!hist_ok(st, R)) return;
  const int i = blockIdx.x, q = threadIdx.x;
  const float cl = hist_cand(st->m, i + 1, R);
  const float sc = scale_of(cl), isc = 1.0f / sc;
  if (q == 0) hb->s[i] = sc;
  if (q >= 127) return;
  const int target = q + 1;
  uint32_t b;
  if (quant_nearest(cl, cl, sc, isc) < target) {
    b = 0x7F800000u;  // never reached (x <= m): +inf
  } else {
    b = __float_as_uint(__fmul_rn(static_cast<float>(q) + 0.5f, sc));
    int steps = 0;
    if (quant_nearest(__uint_as_float(b), cl, sc, isc) >= target) {
      while (b > 0u && quant_nearest(__uint_as_float(b - 1u), cl, sc, isc) >= target && ++steps < 4096) --b;
    } else {
      while (quant_nearest(__uint_as_float(b), cl, sc, isc) < target && ++steps < 4096) ++b;
    }
    if (steps >= 4096) atomicOr(&hb->fail, 1);
  }
  hb->Bu[i * 127 + q] = b;
}

// Setup, part 2 (R blocks of 128): boundary (i, q)'s position in the sorted
// order (key: bits, then candidate, then q -- each candidate's list is already
// sorted) by binary searches in the other candidates' lists, and its share of
// the lookup table, lut[t] = first position p with cell(B[p]) >= t: the cells
// (cell(predecessor), cell(own)], and for the last boundary the cells after it.
__global__ void __launch_bounds__(128) k_hist_rank(DsgcState* st, int R, HistBuf* hb) {
  pdl_entry();
  __shared__ uint32_t sbu[HNB_PAD];
  const bool ok = hist_ok(st, R);
  if (!ok) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->hist = 0;
      st->grid_active = st->active;
    }
    return;
  }
  const int nb = R * 127;
  {
    const uint4* src = reinterpret_cast<const uint4*>(hb->Bu);
    uint4* dst = reinterpret_cast<uint4*>(sbu);
#pragma unroll 8
    for (int k = threadIdx.x; k < (nb + 3) / 4; k += blockDim.x) dst[k] = src[k];
  }
  __syncthreads();
  const float m = st->m;
  const float K = __fdiv_rn(static_cast<float>(2 * 127 * R), m);
  const int tmax = 2 * 127 * R + 1;
  const int i = blockIdx.x, q = threadIdx.x;
  if (q < 127) {
    const uint32_t b = sbu[i * 127 + q];
    int rank = q;
    uint64_t pred = q > 0 ? (static_cast<uint64_t>(sbu[i * 127 + q - 1]) << 32) | static_cast<uint32_t>(i * 127 + q - 1) : 0ull;
    bool has_pred = q > 0;
    for (int j = 0; j < R; ++j) {
      if (j == i) continue;
      const uint32_t* L = sbu + j * 127;
      int lo = 0, hi = 127;  // count of list-j keys below (b, i): bits first, then candidate order
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (L[mid] < b || (L[mid] == b && j < i)) lo = mid + 1;
        else hi = mid;
      }
      rank += lo;
      if (lo > 0) {
        const uint64_t kp = (static_cast<uint64_t>(L[lo - 1]) << 32) | static_cast<uint32_t>(j * 127 + lo - 1);
        if (!has_pred || kp > pred) pred = kp;
        has_pred = true;
      }
    }
    const float bf = __uint_as_float(b);
    hb->B[rank] = bf;
    hb->tag[rank] = static_cast<uint8_t>(i);
    hb->pos[i * 127 + q] = static_cast<uint16_t>(rank);
    const int c_own = hist_cell(bf, K, tmax);
    const int t0 = has_pred ? hist_cell(__uint_as_float(static_cast<uint32_t>(pred >> 32)), K, tmax) + 1 : 0;
    for (int t = t0; t <= c_own; ++t) hb->lut[t] = static_cast<uint16_t>(rank);
    if (rank == nb - 1)
      for (int t = c_own + 1; t <= tmax + 1; ++t) hb->lut[t] = static_cast<uint16_t>(nb);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    uint32_t b0 = sbu[0];
    for (int j = 1; j < R; ++j) b0 = min(b0, sbu[j * 127]);
    const int e0 = static_cast<int>(b0 >> 23);
    const bool good = hb->fail == 0 && e0 >= 1 && e0 < 255;
    hb->K = K;
    hb->nb = nb;
    hb->e0 = e0;
    hb->tmax = tmax;
    st->hist = good ? 1 : 0;
    st->grid_active = good ? 0 : st->active;
  }
}

// The pass over g: per-block bins in shared memory -- a count and the sums of
// the 14-, 14- and 10-bit digits of |g| in units of 2^(e0 - 150) (< 2^38), all with
// native 32-bit shared atomics (a 64-bit shared add is a CAS loop, which
// serialises on the few bins where gradients pile up).  A block flushes its
// bins to the global 64-bit totals every HIST_ROUND elements, before any
// 32-bit digit sum can wrap.
constexpr int HIST_ITERS = 64;  // iterations of 2 float4 per thread per round: 2^18 elements per block
__global__ void __launch_bounds__(HIST_THREADS, 2) k_hist_pass(const float* __restrict__ g, uint32_t n,
                                                             const DsgcState* st, HistBuf* hb) {
  pdl_entry();
  if (!st->hist) return;
  extern __shared__ __align__(16) unsigned char hsm[];
  const int nb = hb->nb, tmax = hb->tmax, e0 = hb->e0;
  const float K = hb->K;
  uint4* sbin = reinterpret_cast<uint4*>(hsm);                 // [nb + 1] {count, digit 0, 1, 2}
  float* sB = reinterpret_cast<float*>(sbin + (nb + 1));      // [nb]
  uint16_t* slut = reinterpret_cast<uint16_t*>(sB + nb);      // [tmax + 2]
  for (int i = threadIdx.x; i <= nb; i += blockDim.x) sbin[i] = make_uint4(0u, 0u, 0u, 0u);
  for (int i = threadIdx.x; i < nb; i += blockDim.x) sB[i] = hb->B[i];
  for (int i = threadIdx.x; i <= tmax + 1; i += blockDim.x) slut[i] = hb->lut[i];
  __syncthreads();
  unsigned* sw = reinterpret_cast<unsigned*>(sbin);
  auto body = [&](float v) {
    const float x = fabsf(v);
    const int t = hist_cell(x, K, tmax);
    int p = slut[t];
    const int pe = slut[t + 1];
    // a cell's boundaries sit within rounding of one value: x is past all of
    // them or before all of them but for a few ulps around it
    if (p < pe) {
      if (sB[pe - 1] <= x) {
        p = pe;
      } else if (sB[p] <= x) {
        ++p;
        while (sB[p] <= x) ++p;  // stops before pe - 1
      }
    }
    if (p) {
      const uint32_t b = __float_as_uint(x);
      const unsigned long long fx = static_cast<unsigned long long>((b & 0x7FFFFFu) | 0x800000u)
                                    << ((b >> 23) - static_cast<uint32_t>(e0));
      unsigned* w = sw + 4 * p;
      atomicAdd(w, 1u);
      atomicAdd(w + 1, static_cast<unsigned>(fx) & 0x3FFFu);
      atomicAdd(w + 2, static_cast<unsigned>(fx >> 14) & 0x3FFFu);
      const unsigned d2 = static_cast<unsigned>(fx >> 28);  // 0 for all but the top 4 binades above B[0]
      if (d2) atomicAdd(w + 3, d2);
    }
  };
  auto flush = [&]() {
    __syncthreads();
    for (int p = threadIdx.x + 1; p <= nb; p += blockDim.x) {
      const uint4 c = sbin[p];
      if (!c.x) continue;
      atomicAdd(hb->cnt + p, static_cast<unsigned long long>(c.x));
      atomicAdd(hb->sum[0] + p, static_cast<unsigned long long>(c.y));
      atomicAdd(hb->sum[1] + p, static_cast<unsigned long long>(c.z));
      atomicAdd(hb->sum[2] + p, static_cast<unsigned long long>(c.w));
      sbin[p] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
  };
  const uint32_t stride = gridDim.x * blockDim.x, n4 = n / 4;
  const float4* g4 = reinterpret_cast<const float4*>(g);
  // rounds of HIST_ITERS block-wide iterations; the loop bounds are block-uniform
  // (every thread reaches the flush barriers)
  const uint32_t base0 = blockIdx.x * blockDim.x;
  uint32_t fb = base0;  // block's first float4 of the iteration
  while (fb < n4) {
    for (int it = 0; it < HIST_ITERS && fb < n4; ++it, fb += 2 * stride) {
      const uint32_t f = fb + threadIdx.x;
      if (f + stride < n4) {
        const float4 a = __ldg(g4 + f), c = __ldg(g4 + f + stride);
        body(a.x); body(a.y); body(a.z); body(a.w);
        body(c.x); body(c.y); body(c.z); body(c.w);
      } else if (f < n4) {
        const float4 a = __ldg(g4 + f);
        body(a.x); body(a.y); body(a.z); body(a.w);
      }
    }
    flush();
  }
  for (uint32_t i = n4 * 4 + base0 + threadIdx.x; i < n; i += stride) body(g[i]);
  flush();
}

// Finaliser (one block of 32 warps): the bins are staged in shared memory as
// doubles (count, sum of |g|), then warp w walks a slice of them with lane j
// tracking candidate j's q; fixed-order combination into totals[3 + 2j], [4 + 2j].
__global__ void __launch_bounds__(1024) k_hist_final(DsgcState* st, HistBuf* hb, int R, double* totals, int rounds,
                                                     int fuse_step) {
  pdl_entry();
  if (threadIdx.x == 0 && hb->fail) hb->fail = 0;
  if (!st->hist) return;
  extern __shared__ __align__(16) unsigned char fsm[];
  __shared__ double part[32][HR_MAX][2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nb = hb->nb;
  double2* sbin = reinterpret_cast<double2*>(fsm);                 // [nb + 1] {count, sum}
  uint8_t* stag = reinterpret_cast<uint8_t*>(sbin + (nb + 1));     // [nb]
  for (int F = threadIdx.x; F <= nb; F += blockDim.x) {
    const double S = static_cast<double>(hb->sum[2][F]) * 268435456.0 + static_cast<double>(hb->sum[1][F]) * 16384.0 +
                     static_cast<double>(hb->sum[0][F]);
    sbin[F] = make_double2(static_cast<double>(hb->cnt[F]), S);
  }
  for (int F = threadIdx.x; F < nb; F += blockDim.x) stag[F] = hb->tag[F];
  __syncthreads();
  const int per = (nb + 32) / 32;  // bins 1..nb
  const int F0 = 1 + w * per, F1 = min(nb + 1, F0 + per);
  double num = 0.0, sqh = 0.0;
  if (lane < R && F0 < F1) {
    const float s = hb->s[lane];
    // q at F0 = boundaries of candidate `lane` at sorted positions < F0
    int lo = 0, hi = 127;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (hb->pos[lane * 127 + mid] < F0) lo = mid + 1;
      else hi = mid;
    }
    int q = lo;
    for (int F = F0; F < F1; ++F) {
      const double2 b = sbin[F];
      if (b.x != 0.0) {
        const double td = __fmul_rn(static_cast<float>(q), s);
        num = fma(td, b.y, num);
        sqh = fma(b.x, td * td, sqh);
      }
      if (F < nb && stag[F] == lane) ++q;
    }
  }
  part[w][lane][0] = num;
  part[w][lane][1] = sqh;
  __syncthreads();
  if (threadIdx.x < R) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < 32; ++k) {
      a += part[k][threadIdx.x][0];
      b += part[k][threadIdx.x][1];
    }
    totals[3 + 2 * threadIdx.x] = ldexp(a, hb->e0 - 150);
    totals[4 + 2 * threadIdx.x] = b;
  }
  if (fuse_step) {
    __syncthreads();
    if (threadIdx.x == 0) search_step_dev(st, totals, R, R, rounds);
  }
}

// ---------------------------------------------------------------- host side

static int stats_pass0(Ctx* c, const float* x, int64_t n) {
  const int nb = nblocks(n);
  double* p = ensure_partials(c, static_cast<size_t>(nb) * 3);
  if (!p) return set_error(I8T_ECUDA, "partials alloc failed");
  launch_k(k_dc_stats0, nb, RED_THREADS, 0, c->stream, x, static_cast<uint32_t>(n), p, c->d_totals, c->d_ticket);
  count_launch(1);
  return cuda_check("k_dc_stats0");
}

// K4 over nc <= 32 candidates: groups of 8 (or one group of 1 / 2 for the
// golden-section rounds).
// step_st: run the search state machine in the pass's last block (one
// candidate group only; *fused reports whether it did).
static int dc_pass_n(Ctx* c, const float* g, int64_t n, const float* cands, const int32_t* active, int nc,
                     bool stats, DsgcState* step_st = nullptr, int R = 0, int rounds = 0, bool* fused = nullptr) {
  if (nc < 1 || nc > 32) return set_error(I8T_EINVAL, "dc pass: bad candidate count");
  const int ng = nc <= 1 ? 1 : nc <= 2 ? 2 : nc <= 4 ? 4 : 8;
  const int groups = (nc + ng - 1) / ng;
  const int nb = nblocks(n, 1, 3 * 148);
  const int nv = 3 + 2 * ng;
  double* p = ensure_partials(c, static_cast<size_t>(nb) * groups * nv + static_cast<size_t>(groups) * nv);
  unsigned* t = group_tickets(c);
  if (!p || !t) return set_error(I8T_ECUDA, "partials alloc failed");
  double* gt = p + static_cast<size_t>(nb) * groups * nv;
  const dim3 grid(nb, groups);
  const uint32_t un = static_cast<uint32_t>(n);
  DsgcState* sst = groups == 1 ? step_st : nullptr;
  if (fused) *fused = sst != nullptr;
#define DCS(NG, ST) launch_k(k_dc_stats<NG, ST>, grid, RED_THREADS, 0, c->stream, g, un, cands, nc, active, p, gt, c->d_totals, t + 32, sst, R, rounds)
  if (stats) {
    if (ng == 1) DCS(1, true);
    else if (ng == 2) DCS(2, true);
    else DCS(8, true);
  } else {
    if (ng == 1) DCS(1, false);
    else if (ng == 2) DCS(2, false);
    else if (ng == 4) DCS(4, false);
    else DCS(8, false);
  }
#undef DCS
  count_launch(1);
  return cuda_check("k_dc_stats");
}

static bool hist_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("I8T_DSGC_HIST");
    return !(e && e[0] == '0');
  }();
  return on;
}

static size_t hist_smem(int R) {
  const size_t nb = static_cast<size_t>(R) * 127, tmax = 2 * 127 * static_cast<size_t>(R) + 1;
  return (nb + 1) * 16 + nb * 4 + (tmax + 2) * 2;
}

static size_t hist_final_smem(int R) {
  const size_t nb = static_cast<size_t>(R) * 127;
  return (nb + 1) * 16 + nb;
}

static HistBuf* ensure_hist(Ctx* c) {
  if (c->d_hist) return reinterpret_cast<HistBuf*>(c->d_hist);
  static const bool attr = [] {
    return cudaFuncSetAttribute(k_hist_pass, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(hist_smem(HR_MAX))) == cudaSuccess &&
           cudaFuncSetAttribute(k_hist_final, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(hist_final_smem(HR_MAX))) == cudaSuccess;
  }();
  if (!attr) return nullptr;
  cudaStreamSynchronize(c->stream);
  if (cudaMalloc(&c->d_hist, sizeof(HistBuf)) != cudaSuccess) {
    c->d_hist = nullptr;
    return nullptr;
  }
  cudaMemset(c->d_hist, 0, sizeof(HistBuf));
  return reinterpret_cast<HistBuf*>(c->d_hist);
}

static int run_search(Ctx* c, DsgcState* st, const float* g, int64_t n, int R, int rounds, float prev_clip,
                      int prev_from_state, const double* stats = nullptr) {
  // stats: max|g|, non-finite, sum g^2 of g already reduced by its producer
  // (i8t_bn_bwd_apply_stats): the first pass over g is skipped
  int rc = stats ? (cudaMemcpyAsync(c->d_totals, stats, 3 * sizeof(double), cudaMemcpyDeviceToDevice, c->stream),
                    cuda_check("stats copy"))
                 : stats_pass0(c, g, n);
  if (rc || (rc = allreduce_totals(c, 3))) return rc;
  launch_k(k_search_begin, 1, 32, 0, c->stream, st, c->d_totals, R, prev_clip, prev_from_state, c->d_err);
  count_launch(1);
  // The device decides whether the search short-circuits (st->active); under
  // data parallelism every rank takes the same branch (global totals), and a
  // skipped pass contributes a zero totals buffer to the hook.
  auto pass = [&](int nc) -> int {
    if (ctx_dp(c)) cudaMemsetAsync(c->d_totals, 0, sizeof(double) * (3 + 2 * nc), c->stream);
    bool fused = false;
    int r = dc_pass_n(c, g, n, st->cand, &st->active, nc, false, ctx_dp(c) ? nullptr : st, R, rounds, &fused);
    if (r || fused) return r;
    if ((r = allreduce_totals(c, 3 + 2 * nc))) return r;
    launch_k(k_search_step, 1, 32, 0, c->stream, st, c->d_totals, nc, R, rounds, static_cast<const int32_t*>(nullptr));
    count_launch(1);
    return cuda_check("k_search_step");
  };
  if (R <= HR_MAX && hist_enabled()) {
    // the grid as one histogram pass; the per-candidate pass stays queued for
    // the inputs the histogram declines (st->grid_active), e.g. tiny max|g|
    HistBuf* hb = ensure_hist(c);
    if (!hb) return set_error(I8T_ECUDA, "histogram buffer alloc failed");
    if (ctx_dp(c)) cudaMemsetAsync(c->d_totals, 0, sizeof(double) * (3 + 2 * R), c->stream);
    launch_k(k_hist_bounds, R, 128, 0, c->stream, static_cast<const DsgcState*>(st), R, hb);
    launch_k(k_hist_rank, R, 128, 0, c->stream, st, R, hb);
    const size_t smem = hist_smem(R);
    const int64_t want = (n + HIST_THREADS * 16 - 1) / (HIST_THREADS * 16);
    const int nbk = static_cast<int>(want < 1 ? 1 : want > 2 * 148 ? 2 * 148 : want);
    launch_k(k_hist_pass, nbk, HIST_THREADS, smem, c->stream, g, static_cast<uint32_t>(n),
             static_cast<const DsgcState*>(st), hb);
    const bool fuse = !ctx_dp(c);
    launch_k(k_hist_final, 1, 1024, hist_final_smem(R), c->stream, st, hb, R, c->d_totals, rounds, fuse ? 1 : 0);
    count_launch(4);
    if ((rc = cuda_check("k_hist"))) return rc;
    if ((rc = dc_pass_n(c, g, n, st->cand, &st->grid_active, R, false))) return rc;
    if ((rc = allreduce_totals(c, 3 + 2 * R))) return rc;
    // the state machine already ran in k_hist_final unless the fallback pass did the work
    launch_k(k_search_step, 1, 32, 0, c->stream, st, c->d_totals, R, R, rounds,
             fuse ? static_cast<const int32_t*>(&st->grid_active) : static_cast<const int32_t*>(nullptr));
    count_launch(1);
    if ((rc = cuda_check("k_search_step"))) return rc;
  } else {
    for (int done = 0; done < R; done += 32)
      if ((rc = pass((R - done) < 32 ? (R - done) : 32))) return rc;
  }
  if (rounds > 0) {
    if ((rc = pass(4))) return rc;  // x1, x2 and both possible probes of round 1
    for (int r = 1; r < rounds; ++r)
      if ((rc = pass(1))) return rc;
  }
  return I8T_OK;
}

static int launch_quant_grad(Ctx* c, DsgcState* st, const float* clip_override, const float* g, int64_t n_img,
                             int64_t C, int64_t HW, bool dc_sums, uint32_t* lcg, int8_t* q, QgFin fin) {
  return launch_quant_grad_src(c, st, clip_override, PlainSrc{reinterpret_cast<const float4*>(g)}, n_img, C, HW,
                               dc_sums, lcg, q, fin);
}

}  // namespace i8t_dev

using namespace i8t_dev;
#define CTX(c) reinterpret_cast<Ctx*>(c)

// state <- state advanced by k draws (k mod 2^32; 2^32 - d steps back by d)
static __global__ void k_lcg_jump(uint32_t* state, uint64_t k) {
  pdl_entry();
  *state = apply(lcg_jump_map(k), *state);
}

extern "C" {

int i8t_max_abs(i8t_ctx* ctx, const float* x, int64_t n, float* out) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !out) return set_error(I8T_EINVAL, "max_abs: bad arguments");
  int rc = stats_pass0(c, x, n);
  if (rc) return rc;
  launch_k(k_fin_scalar, 1, 32, 0, c->stream, c->d_totals, 0, out, nullptr, nullptr);
  count_launch(1);
  return cuda_check("k_fin_scalar");
}

int i8t_histogram(i8t_ctx* ctx, const float* x, int64_t n, int bins, int64_t* counts, double* lo_hi) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !counts || bins < 1 || bins > 8192 || n < 0) return set_error(I8T_EINVAL, "histogram: bad arguments");
  if (n >= (int64_t(1) << 31)) return set_error(I8T_EUNSUPPORTED, "histogram: tensor >= 2^31 elements");
  cudaMemsetAsync(counts, 0, sizeof(int64_t) * static_cast<size_t>(bins), c->stream);
  int nb = nblocks(n);
  double* p = ensure_partials(c, static_cast<size_t>(nb));
  if (!p) return set_error(I8T_ECUDA, "partials alloc failed");
  launch_k(k_finite_absmax, nb, RED_THREADS, 0, c->stream, x, static_cast<uint32_t>(n), p, c->d_totals, c->d_ticket);
  count_launch(1);
  int rc = cuda_check("k_finite_absmax");
  if (rc) return rc;
  nb = nblocks(n, 1, 4 * 148);
  launch_k(k_histogram, nb, 256, sizeof(unsigned int) * static_cast<size_t>(bins), c->stream, x,
           static_cast<uint32_t>(n), static_cast<const double*>(c->d_totals), bins,
           reinterpret_cast<unsigned long long*>(counts), lo_hi);
  count_launch(1);
  return cuda_check("k_histogram");
}

int i8t_sq_l2_norm(i8t_ctx* ctx, const float* x, int64_t n, double* out) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !out) return set_error(I8T_EINVAL, "sq_l2_norm: bad arguments");
  int rc = stats_pass0(c, x, n);
  if (rc) return rc;
  launch_k(k_fin_scalar, 1, 32, 0, c->stream, c->d_totals, 2, nullptr, out, nullptr);
  count_launch(1);
  return cuda_check("k_fin_scalar");
}

int i8t_has_nonfinite(i8t_ctx* ctx, const float* x, int64_t n, int32_t* out) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !out) return set_error(I8T_EINVAL, "has_nonfinite: bad arguments");
  int rc = stats_pass0(c, x, n);
  if (rc) return rc;
  launch_k(k_fin_scalar, 1, 32, 0, c->stream, c->d_totals, 1, nullptr, nullptr, out);
  count_launch(1);
  return cuda_check("k_fin_scalar");
}

static int dot_like(Ctx* c, const float* a, const float* b, int64_t n, double* dot_out, double* cos_out) {
  const int nb = nblocks(n);
  double* p = ensure_partials(c, static_cast<size_t>(nb) * 3);
  if (!p) return set_error(I8T_ECUDA, "partials alloc failed");
  launch_k(k_dot3, nb, RED_THREADS, 0, c->stream, a, b, static_cast<uint32_t>(n), p, c->d_totals, c->d_ticket);
  launch_k(k_fin_cosine, 1, 32, 0, c->stream, c->d_totals, dot_out, cos_out);
  count_launch(2);
  return cuda_check("k_dot3");
}

int i8t_dot(i8t_ctx* ctx, const float* a, const float* b, int64_t n, double* out) {
  Ctx* c = CTX(ctx);
  if (!c || !a || !b || !out) return set_error(I8T_EINVAL, "dot: bad arguments");
  return dot_like(c, a, b, n, out, nullptr);
}

int i8t_cosine_distance(i8t_ctx* ctx, const float* g, const float* h, int64_t n, double* out) {
  Ctx* c = CTX(ctx);
  if (!c || !g || !h || !out) return set_error(I8T_EINVAL, "cosine_distance: bad arguments");
  return dot_like(c, g, h, n, nullptr, out);
}

int i8t_measure_dc(i8t_ctx* ctx, const float* g, int64_t n, float clip, double* out) {
  Ctx* c = CTX(ctx);
  if (!c || !g || !out) return set_error(I8T_EINVAL, "measure_dc: bad arguments");
  if (!(clip > 0.0f) || !std::isfinite(clip)) return set_error(I8T_EINVAL, "QuantParams: clip must be positive and finite");
  float* dclip = reinterpret_cast<float*>(ensure_scratch(c, 256));
  if (!dclip) return set_error(I8T_ECUDA, "scratch alloc failed");
  cudaMemcpyAsync(dclip, &clip, sizeof(float), cudaMemcpyHostToDevice, c->stream);
  int rc = dc_pass_n(c, g, n, dclip, nullptr, 1, true);
  if (rc) return rc;
  launch_k(k_fin_measure_dc, 1, 32, 0, c->stream, c->d_totals, out, c->d_err);
  count_launch(1);
  cudaStreamSynchronize(c->stream);  // `clip` lives on the caller's stack
  return cuda_check("measure_dc");
}

int i8t_search_clip(i8t_ctx* ctx, const float* g, int64_t n, int grid, int rounds, float prev_clip, float* clip_out,
                    double* dc_out) {
  Ctx* c = CTX(ctx);
  if (!c || !g) return set_error(I8T_EINVAL, "search_clip: bad arguments");
  if (grid < 8) return set_error(I8T_EINVAL, "search_clip: grid resolution must be >= 8");
  DsgcState* st = reinterpret_cast<DsgcState*>(ensure_scratch(c, sizeof(DsgcState)));
  if (!st) return set_error(I8T_ECUDA, "scratch alloc failed");
  int rc = run_search(c, st, g, n, grid, rounds, prev_clip, 0);
  if (rc) return rc;
  launch_k(k_search_end, 1, 32, 0, c->stream, st, 0, 0, clip_out, dc_out);
  count_launch(1);
  return cuda_check("k_search_end");
}

int64_t i8t_dsgc_state_size(void) { return static_cast<int64_t>(sizeof(DsgcState)); }

int i8t_dsgc_init(i8t_ctx* ctx, void* state, int64_t period) {
  Ctx* c = CTX(ctx);
  if (!c || !state) return set_error(I8T_EINVAL, "dsgc_init: bad arguments");
  DsgcState h{};
  h.v.iter_of_last_update = -1;
  h.v.period = period;
  h.v.lr_scale = 1.0;
  cudaMemcpyAsync(state, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream);
  cudaStreamSynchronize(c->stream);
  return cuda_check("dsgc_init");
}

int i8t_dsgc_read(i8t_ctx* ctx, const void* state, i8t_dsgc_view* out) {
  Ctx* c = CTX(ctx);
  if (!c || !state || !out) return set_error(I8T_EINVAL, "dsgc_read: bad arguments");
  cudaMemcpyAsync(out, state, sizeof(i8t_dsgc_view), cudaMemcpyDeviceToHost, c->stream);
  cudaStreamSynchronize(c->stream);
  return cuda_check("dsgc_read");
}

int i8t_dsgc_write(i8t_ctx* ctx, void* state, const i8t_dsgc_view* in) {
  Ctx* c = CTX(ctx);
  if (!c || !state || !in) return set_error(I8T_EINVAL, "dsgc_write: bad arguments");
  cudaMemcpyAsync(state, in, sizeof(i8t_dsgc_view), cudaMemcpyHostToDevice, c->stream);
  cudaStreamSynchronize(c->stream);
  return cuda_check("dsgc_write");
}

int i8t_maybe_update(i8t_ctx* ctx, void* state, const float* g, int64_t n, int64_t iter, int grid, int rounds, int due) {
  Ctx* c = CTX(ctx);
  DsgcState* st = reinterpret_cast<DsgcState*>(state);
  if (!c || !st || !g) return set_error(I8T_EINVAL, "maybe_update: bad arguments");
  if (grid < 8) return set_error(I8T_EINVAL, "search_clip: grid resolution must be >= 8");
  int rc;
  if (due) {
    if ((rc = run_search(c, st, g, n, grid, rounds, 0.0f, 1))) return rc;
    launch_k(k_search_end, 1, 32, 0, c->stream, st, iter, 1, nullptr, nullptr);
    count_launch(1);
    return cuda_check("maybe_update");
  }
  if ((rc = dc_pass_n(c, g, n, &st->v.clip, nullptr, 1, true)) || (rc = allreduce_totals(c, 5))) return rc;
  launch_k(k_fin_maybe_dc, 1, 32, 0, c->stream, st, c->d_totals, c->d_err);
  count_launch(1);
  return cuda_check("maybe_update");
}

static int quantize_gradient_impl(i8t_ctx* ctx, void* state, const float* g, int64_t n_img, int64_t C, int64_t HW,
                                  int64_t iter, int grid, int rounds, int search_enabled, int due,
                                  int lr_scaling_enabled, double alpha, double beta, int form, uint32_t* lcg_state,
                                  int8_t* q, int64_t ld_q, const double* stats);

int i8t_quantize_gradient(i8t_ctx* ctx, void* state, const float* g, int64_t n_img, int64_t C, int64_t HW, int64_t iter,
                          int grid, int rounds, int search_enabled, int due, int lr_scaling_enabled, double alpha,
                          double beta, int form, uint32_t* lcg_state, int8_t* q, int64_t ld_q) {
  return quantize_gradient_impl(ctx, state, g, n_img, C, HW, iter, grid, rounds, search_enabled, due,
                                lr_scaling_enabled, alpha, beta, form, lcg_state, q, ld_q, nullptr);
}

int i8t_quantize_gradient_stats(i8t_ctx* ctx, void* state, const float* g, int64_t n_img, int64_t C, int64_t HW,
                                int64_t iter, int grid, int rounds, int search_enabled, int due, int lr_scaling_enabled,
                                double alpha, double beta, int form, uint32_t* lcg_state, int8_t* q, int64_t ld_q,
                                const double* stats) {
  if (!stats) return set_error(I8T_EINVAL, "quantize_gradient_stats: null stats");
  return quantize_gradient_impl(ctx, state, g, n_img, C, HW, iter, grid, rounds, search_enabled, due,
                                lr_scaling_enabled, alpha, beta, form, lcg_state, q, ld_q, stats);
}

static int quantize_gradient_impl(i8t_ctx* ctx, void* state, const float* g, int64_t n_img, int64_t C, int64_t HW,
                                  int64_t iter, int grid, int rounds, int search_enabled, int due,
                                  int lr_scaling_enabled, double alpha, double beta, int form, uint32_t* lcg_state,
                                  int8_t* q, int64_t ld_q, const double* stats) {
  Ctx* c = CTX(ctx);
  DsgcState* st = reinterpret_cast<DsgcState*>(state);
  if (!c || !st || !g || !lcg_state || !q || n_img < 1 || C < 1 || HW < 1)
    return set_error(I8T_EINVAL, "quantize_gradient: bad arguments");
  if (ld_q != C) return set_error(I8T_EUNSUPPORTED, "quantize_gradient: ld_q must equal C");
  if (lr_scaling_enabled) {
    if (!(alpha > 0.0)) return set_error(I8T_EINVAL, "scale_factor: alpha must be > 0");
    if (!(beta > 0.0 && beta <= 1.0)) return set_error(I8T_EINVAL, "scale_factor: beta must be in (0,1]");
  }
  const int64_t numel = n_img * C * HW;
  int rc;
  bool dc_sums;
  if (search_enabled) {
    if (grid < 8) return set_error(I8T_EINVAL, "search_clip: grid resolution must be >= 8");
    if (due) {
      if ((rc = run_search(c, st, g, numel, grid, rounds, 0.0f, 1, stats))) return rc;
      launch_k(k_search_end, 1, 32, 0, c->stream, st, iter, 1, nullptr, nullptr);
      count_launch(1);
      dc_sums = false;
    } else {
      dc_sums = true;
    }
  } else {
    if ((rc = stats_pass0(c, g, numel)) || (rc = allreduce_totals(c, 3))) return rc;
    launch_k(k_clip_from_max, 1, 32, 0, c->stream, st, c->d_totals, iter);
    count_launch(1);
    dc_sums = true;
  }
  QgFin fin{(dc_sums ? 1 : 0) | (lr_scaling_enabled ? 2 : 0), alpha, beta, form, 0u};
  return launch_quant_grad(c, st, nullptr, g, n_img, C, HW, dc_sums, lcg_state, q, fin);
}

int i8t_quantize_stochastic(i8t_ctx* ctx, const float* x, int64_t n, const float* clip, uint32_t* lcg_state, int8_t* q) {
  Ctx* c = CTX(ctx);
  if (!c || !x || !clip || !lcg_state || !q) return set_error(I8T_EINVAL, "quantize: stream required iff mode is stochastic");
  if (n == 0) return I8T_OK;
  DsgcState* st = reinterpret_cast<DsgcState*>(ensure_scratch(c, sizeof(DsgcState)));
  if (!st) return set_error(I8T_ECUDA, "scratch alloc failed");
  QgFin fin{4, 0.0, 0.0, 0, 0u};
  if (n % 4 == 0) return launch_quant_grad(c, st, clip, x, 1, 1, n, false, lcg_state, q, fin);
  // ragged length: quantise a zero-padded copy (the kernel reads float4s), keep
  // the first n bytes, then step the stream back over the pad's draws (the LCG
  // has period 2^32, so a jump of 2^32 - d is d steps back): one draw per element
  const int64_t np = (n + 3) / 4 * 4;
  float* xp = nullptr;
  int8_t* qp = nullptr;
  if (cudaMallocAsync(reinterpret_cast<void**>(&xp), sizeof(float) * np, c->stream) != cudaSuccess ||
      cudaMallocAsync(reinterpret_cast<void**>(&qp), np, c->stream) != cudaSuccess)
    return set_error(I8T_ECUDA, "quantize_stochastic: alloc failed");
  cudaMemcpyAsync(xp, x, sizeof(float) * n, cudaMemcpyDeviceToDevice, c->stream);
  cudaMemsetAsync(xp + n, 0, sizeof(float) * (np - n), c->stream);
  int rc = launch_quant_grad(c, st, clip, xp, 1, 1, np, false, lcg_state, qp, fin);
  if (rc == I8T_OK) {
    cudaMemcpyAsync(q, qp, n, cudaMemcpyDeviceToDevice, c->stream);
    launch_k(k_lcg_jump, 1, 1, 0, c->stream, lcg_state, (uint64_t)((uint64_t(1) << 32) - uint64_t(np - n)));
    count_launch(1);
    rc = cuda_check("k_lcg_jump");
  }
  cudaFreeAsync(xp, c->stream);
  cudaFreeAsync(qp, c->stream);
  return rc;
}

}  // extern "C"
