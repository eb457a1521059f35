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
template <int NG>
__global__ void __launch_bounds__(RED_THREADS, 3) k_dc_stats(const float* __restrict__ g, uint32_t n,
                                                          const float* __restrict__ cands, int nc,
                                                          const int32_t* active, double* partials, double* gtot,
                                                          double* totals, unsigned* tickets) {
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
    bad |= !isfinite(v);
    m = fmaxf(m, fabsf(v));
    const double vd = v;
    acc[2] = fma(vd, vd, acc[2]);
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
  constexpr int U = NG <= 2 ? 4 : 1;  // float4 loads in flight per thread (HBM-bound passes)
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
  if (blockIdx.y == 0 && threadIdx.x < 3) totals[threadIdx.x] = __ldcg(gt + threadIdx.x);
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
__global__ void k_search_step(DsgcState* st, const double* tot, int nc, int R, int rounds) {
  pdl_entry();
  if (threadIdx.x || st->active == 0) return;
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
    st->cand[0] = static_cast<float>(st->x1);
    st->cand[1] = static_cast<float>(st->x2);
    st->ncand = 2;
    st->phase = 1;
    return;
  }
  if (st->phase == 1) {
    st->f1 = dcs[0];
    st->f2 = dcs[1];
    ds_track(st, st->x1, st->f1);
    ds_track(st, st->x2, st->f2);
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
static int dc_pass_n(Ctx* c, const float* g, int64_t n, const float* cands, const int32_t* active, int nc) {
  if (nc < 1 || nc > 32) return set_error(I8T_EINVAL, "dc pass: bad candidate count");
  const int ng = nc <= 1 ? 1 : nc <= 2 ? 2 : 8;
  const int groups = (nc + ng - 1) / ng;
  const int nb = nblocks(n, 1, 3 * 148);
  const int nv = 3 + 2 * ng;
  double* p = ensure_partials(c, static_cast<size_t>(nb) * groups * nv + static_cast<size_t>(groups) * nv);
  unsigned* t = group_tickets(c);
  if (!p || !t) return set_error(I8T_ECUDA, "partials alloc failed");
  double* gt = p + static_cast<size_t>(nb) * groups * nv;
  const dim3 grid(nb, groups);
  const uint32_t un = static_cast<uint32_t>(n);
  if (ng == 1) launch_k(k_dc_stats<1>, grid, RED_THREADS, 0, c->stream, g, un, cands, nc, active, p, gt, c->d_totals, t + 32);
  else if (ng == 2) launch_k(k_dc_stats<2>, grid, RED_THREADS, 0, c->stream, g, un, cands, nc, active, p, gt, c->d_totals, t + 32);
  else launch_k(k_dc_stats<8>, grid, RED_THREADS, 0, c->stream, g, un, cands, nc, active, p, gt, c->d_totals, t + 32);
  count_launch(1);
  return cuda_check("k_dc_stats");
}

static int run_search(Ctx* c, DsgcState* st, const float* g, int64_t n, int R, int rounds, float prev_clip,
                      int prev_from_state) {
  int rc = stats_pass0(c, g, n);
  if (rc || (rc = allreduce_totals(c, 3))) return rc;
  launch_k(k_search_begin, 1, 32, 0, c->stream, st, c->d_totals, R, prev_clip, prev_from_state, c->d_err);
  count_launch(1);
  // The device decides whether the search short-circuits (st->active); under
  // data parallelism every rank takes the same branch (global totals), and a
  // skipped pass contributes a zero totals buffer to the hook.
  auto pass = [&](int nc) -> int {
    if (ctx_dp(c)) cudaMemsetAsync(c->d_totals, 0, sizeof(double) * (3 + 2 * nc), c->stream);
    int r = dc_pass_n(c, g, n, st->cand, &st->active, nc);
    if (r || (r = allreduce_totals(c, 3 + 2 * nc))) return r;
    launch_k(k_search_step, 1, 32, 0, c->stream, st, c->d_totals, nc, R, rounds);
    count_launch(1);
    return cuda_check("k_search_step");
  };
  for (int done = 0; done < R; done += 32)
    if ((rc = pass((R - done) < 32 ? (R - done) : 32))) return rc;
  if (rounds > 0) {
    if ((rc = pass(2))) return rc;
    for (int r = 0; r < rounds; ++r)
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
  int rc = dc_pass_n(c, g, n, dclip, nullptr, 1);
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
  if ((rc = dc_pass_n(c, g, n, &st->v.clip, nullptr, 1)) || (rc = allreduce_totals(c, 5))) return rc;
  launch_k(k_fin_maybe_dc, 1, 32, 0, c->stream, st, c->d_totals, c->d_err);
  count_launch(1);
  return cuda_check("maybe_update");
}

int i8t_quantize_gradient(i8t_ctx* ctx, void* state, const float* g, int64_t n_img, int64_t C, int64_t HW, int64_t iter,
                          int grid, int rounds, int search_enabled, int due, int lr_scaling_enabled, double alpha,
                          double beta, int form, uint32_t* lcg_state, int8_t* q, int64_t ld_q) {
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
      if ((rc = run_search(c, st, g, numel, grid, rounds, 0.0f, 1))) return rc;
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
