/*
 * i8t_oracle.h -- CPU restatement of the reference INT8 training hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA product
 * path.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it.  Nothing in paper_1912_12607_b200/ links or calls it.
 *
 * Every function restates the reference algorithm (arXiv 1912.12607 reference,
 * /root/reference/proj/core) and cites the file:line it follows.  The
 * restatement is pinned two ways:
 *   1. against the reference itself, compiled unmodified from its sources into
 *      oracle/_ref/ by oracle/Makefile (tests/test_oracle_vs_ref.py, here only);
 *   2. against golden vectors dumped from that build into tests/golden/
 *      (tests/test_oracle_golden.py, runs anywhere).
 *
 * Extensions beyond what the reference can express, all marked
 * "EXT" below: separate stride/pad per dimension, floor-mode output size, and
 * int64 weight-gradient accumulation without the 130000 depth bound.
 */
#ifndef I8T_ORACLE_H
#define I8T_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_OK = 0, OR_EINVAL = 1, OR_EDOMAIN = 2 };
enum { OR_NEAREST = 0, OR_STOCHASTIC = 1 };
enum { OR_EXP = 0, OR_LINEAR = 1, OR_QUADRATIC = 2 };

typedef struct or_geom {
  int64_t n, c, h, w;   /* input (N,C,H,W) */
  int64_t k, kh, kw;    /* filters (K,C,kh,kw) or (C,1,kh,kw) when depthwise */
  int64_t stride_h, stride_w, pad_h, pad_w;
  int32_t depthwise;
  int32_t floor_mode;   /* EXT: 0 = reference exact-division rule (conv.cpp:11-18) */
} or_geom;

typedef struct or_clip_state {
  float clip;                  /* 0 = uninitialised (clip.hpp:12-18) */
  double last_dc;
  int64_t iter_of_last_update; /* -1 initially */
  int64_t period;
} or_clip_state;

/* ---- LCG (quantize.hpp:32-50) ---- */
uint32_t or_lcg_next(uint32_t* state);
uint32_t or_lcg_jump(uint32_t state, uint64_t k);

/* ---- quantizer (quantize.cpp:11-87) ---- */
int or_quant_params(float clip, float* scale_out);
int or_quantize_value(float x, float clip, float scale, int mode, uint32_t* stream, int8_t* out);
int or_quantize(const float* x, int64_t n, float clip, int mode, uint32_t* stream, int8_t* q);
int or_quantize_partitioned(const float* x, int64_t n, float clip, uint32_t base_seed,
                            int partitions, int8_t* q);
void or_dequantize(const int8_t* q, int64_t n, float scale, float* out);

/* ---- reductions (tensor.cpp:72-101) ---- */
double or_sq_l2_norm(const float* x, int64_t n);
double or_dot(const float* a, const float* b, int64_t n);
float or_max_abs(const float* x, int64_t n);
int or_has_nonfinite(const float* x, int64_t n);

/* ---- GEMM (gemm.cpp:18-47) ---- */
void or_gemm_i8(const int8_t* a, const int8_t* b, int64_t m, int64_t k, int64_t n, int32_t* c);

/* ---- convolution (conv.cpp:11-205) ---- */
int or_geom_validate(const or_geom* g);
int64_t or_out_h(const or_geom* g);
int64_t or_out_w(const or_geom* g);
int or_im2col_i8(const int8_t* x, const or_geom* g, int8_t* out);
/* forward: int32 accumulator (N,K,P,Q) and rescaled float output */
int or_conv_fwd(const int8_t* qa, const int8_t* qw, const or_geom* g, float s_a, float s_w,
                int32_t* acc_out, float* z_out);
/* dgrad: int64 accumulator (N,C,H,W) and float output (conv.cpp:197-203) */
int or_conv_dgrad(const int8_t* qg, const int8_t* qw, const or_geom* g, float s_g, float s_w,
                  int64_t* acc_out, float* ga_out);
/* wgrad: int64 accumulator in weight shape and float output (conv.cpp:186-195) */
int or_conv_wgrad(const int8_t* qg, const int8_t* qa, const or_geom* g, float s_g, float s_a,
                  int64_t* acc_out, float* gw_out);

/* ---- DSGC (clip.cpp:8-93) ---- */
double or_cosine_distance(const float* g, const float* h, int64_t n);
int or_measure_dc(const float* g, int64_t n, float clip, double* dc_out);
int or_search_clip(const float* g, int64_t n, int grid, int rounds, float prev_clip,
                   float* clip_out, double* dc_out);
int or_maybe_update(or_clip_state* st, const float* g, int64_t n, int64_t iter, int grid,
                    int rounds);

/* ---- DCLR (lr_scale.cpp:8-20) ---- */
int or_scale_factor(double dc, double alpha, double beta, int form, double* out);

/* ---- layer glue: quantize_gradient (layers.cpp:19-59) ----
 * stats_out = {dc, lr_scale, eps_norm, ghat_sqnorm}; scale_out = scale of q. */
int or_quantize_gradient(or_clip_state* st, const float* g, int64_t n, int64_t iter,
                         int grid, int rounds, int search_enabled, int lr_scaling_enabled,
                         double alpha, double beta, int form, uint32_t* stream,
                         int8_t* q_out, float* scale_out, double* stats_out);

/* ---- SGD with DCLR factor (train.cpp:97-117, momentum 0) ---- */
void or_sgd_update(float* w, const float* g, int64_t n, double lr);

/* ---- FP32 layers (layers.cpp:230-529), NCHW ---- */
void or_bn_forward_train(const float* x, int64_t n, int64_t c, int64_t hw, const float* gamma, const float* beta,
                         float* running_mean, float* running_var, double momentum, double eps, float* y,
                         float* xhat, double* invstd_out);
void or_bn_forward_eval(const float* x, int64_t n, int64_t c, int64_t hw, const float* gamma, const float* beta,
                        const float* running_mean, const float* running_var, double eps, float* y);
void or_bn_backward(const float* g_out, const float* xhat, const double* invstd, int64_t n, int64_t c, int64_t hw,
                    const float* gamma, float* g_in, float* grad_gamma, float* grad_beta);
int or_pool_forward(const float* x, int64_t n, int64_t c, int64_t h, int64_t w, int kind, int64_t k, int64_t s,
                    int64_t pad, float* y, int64_t* argmax);
int or_pool_backward(const float* g_out, const int64_t* argmax, int64_t n, int64_t c, int64_t h, int64_t w, int kind,
                     int64_t k, int64_t s, int64_t pad, float* g_in);
double or_softmax_ce(const float* logits, int64_t n, int64_t classes, const int32_t* labels, float* g_logits,
                     int* status);
int or_conv_fwd_f32(const float* x, const float* w, const or_geom* g, float* z);
void or_sgd_momentum_update(float* w, const float* g, float* buf, int64_t n, double lr, double momentum);

/* ---- synthetic inputs (rng.hpp:13-50 SplitMix64 + Box-Muller) ---- */
void or_fill_gaussian(float* x, int64_t n, uint64_t seed, double stddev, int relu);
void or_fill_gradient_like(float* x, int64_t n, uint64_t seed, double scale, double outlier_rate);

#ifdef __cplusplus
}
#endif
#endif
