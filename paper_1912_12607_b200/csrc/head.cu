// head.cu -- the loss at the top of the network on sm_100a:
// SoftmaxCrossEntropy::loss_and_grad (layers.cpp:507-529) in one launch.
// One block per row: the row max, sum of exp(x - max) and the label logit in
// double (fixed-order block reductions), log_z = max + log(sum), the row loss
// log_z - x[label] and g = float((exp(x - log_z) - y) / N); the row losses are
// summed over the grid in block order by the last block (deterministic), which
// also raises the divergence flag of train.cpp:73-77 (non-finite loss or
// logits).  N is the global batch under data parallelism.
#include <cuda_runtime.h>

#include <cmath>

#include "internal.cuh"
#include "qcore.cuh"

namespace i8t_dev {

__global__ void __launch_bounds__(RED_THREADS) k_softmax_ce(const float* __restrict__ logits,
                                                           const int64_t* __restrict__ labels, int classes,
                                                           double n_total, float* __restrict__ g,
                                                           double* partials, double* totals, unsigned* ticket,
                                                           double* loss_out, int32_t* bad_out) {
  pdl_entry();
  __shared__ double red[2];
  const int row = blockIdx.x;
  const float* x = logits + static_cast<int64_t>(row) * classes;
  const int64_t lab = labels[row];
  double v[2] = {-INFINITY, 0.0};  // max, non-finite count
  for (int c = threadIdx.x; c < classes; c += blockDim.x) {
    const float f = __ldg(x + c);
    v[0] = fmax(v[0], static_cast<double>(f));
    v[1] += isfinite(f) ? 0.0 : 1.0;
  }
  block_reduce<2>(v, 1u, red);
  const double mx = red[0], nonfinite = red[1];
  double s[1] = {0.0};
  for (int c = threadIdx.x; c < classes; c += blockDim.x) s[0] += exp(static_cast<double>(__ldg(x + c)) - mx);
  block_reduce<1>(s, 0u, red);
  const double log_z = mx + log(red[0]);
  for (int c = threadIdx.x; c < classes; c += blockDim.x) {
    const double p = exp(static_cast<double>(__ldg(x + c)) - log_z);
    g[static_cast<int64_t>(row) * classes + c] = static_cast<float>((p - (c == lab ? 1.0 : 0.0)) / n_total);
  }
  double acc[2] = {0.0, 0.0};
  if (threadIdx.x == 0) {
    acc[0] = (lab >= 0 && lab < classes) ? log_z - static_cast<double>(__ldg(x + lab)) : NAN;
    acc[1] = nonfinite;
  }
  if (grid_reduce<2>(acc, 0u, partials, totals, ticket) && threadIdx.x == 0) {
    const double loss = totals[0] / n_total;
    *loss_out = loss;
    *bad_out = (!isfinite(loss) || totals[1] > 0.0) ? 1 : 0;
  }
}

}  // namespace i8t_dev

using namespace i8t_dev;

extern "C" {

int i8t_softmax_ce(i8t_ctx* ctx, const float* logits, const int64_t* labels, int64_t n, int64_t classes,
                   int64_t n_total, float* g_logits, double* loss, int32_t* bad) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !logits || !labels || !g_logits || !loss || !bad || n < 1 || classes < 1 || n_total < 1)
    return set_error(I8T_EINVAL, "softmax_ce: bad arguments");
  if (n > (1 << 30) || classes > (1 << 30)) return set_error(I8T_EUNSUPPORTED, "softmax_ce: too large");
  double* p = ensure_partials(c, static_cast<size_t>(n) * 2);
  if (!p) return set_error(I8T_ECUDA, "partials alloc failed");
  const double nt = static_cast<double>(n_total);
  launch_k(k_softmax_ce, static_cast<int>(n), RED_THREADS, 0, c->stream, logits, labels, static_cast<int>(classes),
           nt, g_logits, p, c->d_totals, c->d_ticket, loss, bad);
  count_launch(1);
  return cuda_check("k_softmax_ce");
}

}  // extern "C"
