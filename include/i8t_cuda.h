/*
 * i8t_cuda.h -- C-ABI of the B200-native (sm_100a) INT8 training hot path.
 *
 * This is the drop-in boundary for the reference's C++ operator API
 * (`namespace i8t`, /root/reference/proj/core/include/i8t/).  Every entry
 * point below names the reference interface it replaces (file:line).  The C++
 * shim in include/i8t/*.hpp re-exports the reference signatures on top of it
 * (host tensors, same exception types); the PyTorch layer in
 * paper_1912_12607_b200/ calls it through ctypes with device pointers.
 *
 * Conventions
 *  - All tensor pointers are DEVICE pointers unless a name says `host`.
 *  - Every call is asynchronous on the context's CUDA stream and returns an
 *    i8t_status for argument errors detected on the host.  Data-dependent
 *    errors (non-finite input: the reference's std::domain_error) are latched
 *    in a device error word and reported by i8t_ctx_check(), which
 *    synchronises the stream.
 *  - No CPU fallback exists: if the CUDA library cannot run, calls fail.
 *  - Layouts: activations/gradients are NHWC int8 ("channels-last"), with an
 *    optional padded channel stride; weights are KRSC int8 (forward) and CRSK
 *    int8 (backward-data); float outputs are NHWC (or KRSC for weights).
 *    Conversions to the reference's NCHW/KCRS order are provided.
 *  - The per-tensor quantisation scale is s = clip / 127.0f, computed on the
 *    device from a device-resident clip (QuantParams::from_clip,
 *    quantize.cpp:11-14).
 */
#ifndef I8T_CUDA_H
#define I8T_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define I8T_ABI_VERSION 1

typedef enum i8t_status {
  I8T_OK = 0,
  I8T_EINVAL = 1,      /* std::invalid_argument in the reference */
  I8T_EDOMAIN = 2,     /* std::domain_error (non-finite input) */
  I8T_ECUDA = 3,       /* CUDA runtime / launch failure */
  I8T_EUNSUPPORTED = 4 /* shape outside the kernels' envelope */
} i8t_status;

typedef struct i8t_ctx i8t_ctx;

/* Convolution geometry.  Replaces ConvGeometry (conv.hpp:14-28) and extends
 * it: separate stride/pad per dimension and floor-mode output size (the
 * reference demands exact division, conv.cpp:15-17). */
typedef struct i8t_conv_geom {
  int64_t n, c, h, w;       /* input (N,C,H,W) */
  int64_t k, kh, kw;        /* filters (K,C,kh,kw); depthwise: k == c, (C,1,kh,kw) */
  int64_t stride_h, stride_w, pad_h, pad_w;
  int32_t depthwise;
  int32_t floor_mode;       /* 0: reference validation (exact division) */
} i8t_conv_geom;

/* Device-resident DSGC/DCLR state of one quantised layer.  Replaces
 * ClipState (clip.hpp:12-18) + the per-step measurements of QuantState
 * (layers.hpp:28-38).  Allocate with i8t_dsgc_state_size() bytes of device
 * memory, zero it, then call i8t_dsgc_init(). */
typedef struct i8t_dsgc_view {
  float clip;               /* gradient clip; 0 = uninitialised */
  float scale;              /* scale of the last quantised gradient */
  float max_abs;            /* max |g| of the last gradient */
  uint32_t flags;           /* bit0 non-finite input, bit1 zero gradient */
  double last_dc;           /* ClipState::last_dc */
  double lr_scale;          /* phi(d_c), QuantState::lr_scale */
  double eps_norm;          /* ||g - g_hat||, QuantState::eps_norm */
  double ghat_sqnorm;       /* ||g_hat||^2, QuantState::ghat_sqnorm */
  int64_t iter_of_last_update;
  int64_t period;
  float clip_q;             /* clip of the last quantised gradient (scale = clip_q/127) */
  uint32_t reserved;
} i8t_dsgc_view;

/* ------------------------------------------------------------ context */
int i8t_abi_version(void);
/* stream: a cudaStream_t (NULL = legacy default stream). */
int i8t_ctx_create(void* stream, i8t_ctx** out);
int i8t_ctx_set_stream(i8t_ctx* ctx, void* stream);
int i8t_ctx_destroy(i8t_ctx* ctx);
/* Synchronise the stream; report and clear any latched device error. */
int i8t_ctx_check(i8t_ctx* ctx);
/* Device address of the context's latched error word (int32), so a caller can
 * snapshot / restore it on the stream (the trainer does, around the backward of
 * a step whose divergence is only known on the device). */
int i8t_ctx_error_word(i8t_ctx* ctx, int32_t** out);
/* dst <- src (bytes, 16-byte aligned pointers) iff the device int32 *flag != 0,
 * stream-ordered: restores the pre-backward DSGC / LCG state of a diverged step
 * (train.cpp:73-77 returns before the backward) without a host round trip. */
int i8t_copy_if(i8t_ctx* ctx, const int32_t* flag, void* dst, const void* src, int64_t bytes);
const char* i8t_last_error(void);
/* Device memory for hosts that do not link a CUDA runtime (the C++ shim):
 * synchronous on the context's stream.  kind: 0 host->device, 1 device->host,
 * 2 device->device. */
int i8t_device_alloc(i8t_ctx* ctx, uint64_t bytes, void** out);
int i8t_device_free(i8t_ctx* ctx, void* ptr);
int i8t_memcpy(i8t_ctx* ctx, void* dst, const void* src, uint64_t bytes, int kind);
/* Number of kernels this library launched (for bench accounting). */
uint64_t i8t_launch_count(void);
/* Data parallel (8.e): the caller's gradient tensors are shard `rank` of
 * `world` equal contiguous batch shards.  Global DSGC statistics (max|g| and
 * the d_c / eps / g_hat sums) are combined by calling `fn` on device buffers
 * of doubles between kernel phases (op 0 = SUM, 1 = MAX, 2 = MAX on element
 * 0 and SUM on the rest, one collective per phase; dtype 0 = f64), and
 * the stochastic quantiser draws from the global stream at the shard's
 * offset, so every rank quantises exactly as one device would on the whole
 * batch.  fn == NULL restores single-device behaviour. */
typedef int (*i8t_allreduce_fn)(void* user, void* dev_buf, int64_t count, int dtype, int op, void* stream);
int i8t_ctx_set_allreduce(i8t_ctx* ctx, i8t_allreduce_fn fn, void* user);
int i8t_ctx_set_shard(i8t_ctx* ctx, int rank, int world);
/* Data parallelism without a host callback: the context owns an NCCL
 * communicator (libnccl.so.2 resolved at run time) and combines the gradient
 * quantiser's statistics with an all-gather + fixed-order fold on its stream
 * (no host sync; graph-capturable).  Rank 0 makes the id, every rank passes
 * the same bytes (>= 128) with its rank / world; this also sets the shard
 * (i8t_ctx_set_shard).  id == NULL detaches. */
int i8t_nccl_unique_id(uint8_t* out, int64_t bytes);
int i8t_ctx_set_nccl(i8t_ctx* ctx, const uint8_t* id, int64_t bytes, int rank, int world);

/* ------------------------------------------------------------ LCG stream */
/* The gradient stream of LcgStream (quantize.hpp:32-50) lives in device memory
 * as one uint32 state; stochastic quantisers read it and advance it by the
 * number of draws, exactly like the reference's caller-owned stream. */
int i8t_lcg_jump_host(uint32_t state, uint64_t k, uint32_t* out);

/* ------------------------------------------------------------ quantisers */
/* quantize(x, from_clip(*clip), kNearest) (quantize.cpp:33-43) over a flat
 * tensor; optionally fuses max_abs(x) into *amax (device float, running max
 * when accumulate_amax != 0, i.e. QuantState::pending_amax, layers.cpp:101). */
int i8t_quantize_nearest(i8t_ctx* ctx, const float* x, int64_t n, const float* clip, int8_t* q, float* amax,
                         int accumulate_amax);
/* Same quantiser, writing rows of `cols` values into a padded row stride
 * ld_q >= cols (zero pad).  x is [rows, cols] contiguous (NHWC activations). */
/* The activation quantiser of a second consumer of the same tensor x (the
 * projection-shortcut conv beside the block's first conv, both quantising x
 * with their own clip, layers.cpp:101-109): when *clip equals *ref_clip bit for
 * bit the result is ref_q (copied) and *amax takes max(*amax, *ref_amax);
 * otherwise q = quantize_nearest(x, *clip) with the running max|x| into *amax
 * (accumulated).  n elements, 16-byte aligned x / q / ref_q. */
int i8t_quantize_nearest_shared(i8t_ctx* ctx, const float* x, int64_t n, const float* clip, const float* ref_clip,
                                const int8_t* ref_q, const float* ref_amax, int8_t* q, float* amax);
int i8t_quantize_nearest_rows(i8t_ctx* ctx, const float* x, int64_t rows, int64_t cols, const float* clip,
                              int8_t* q, int64_t ld_q, float* amax, int accumulate_amax);
/* NCHW float -> NHWC int8 with padded channel stride c_pad (drop-in path). */
int i8t_quantize_nearest_nchw_to_nhwc(i8t_ctx* ctx, const float* x, int64_t n, int64_t c, int64_t hw,
                                      const float* clip, int8_t* q, int64_t c_pad, float* amax,
                                      int accumulate_amax);
/* Weights KCRS float (or KRSC when src_krsc != 0) -> nearest int8 in two
 * layouts: KRSC rows [K][ld_krsc] (channel stride c_pad, zero padded) for the
 * forward conv and CRSK rows [C][ld_crsk] (K stride k_pad) for backward-data.
 * Either output may be NULL.  Replaces quantize(W) (layers.cpp:108). */
int i8t_quantize_weight(i8t_ctx* ctx, const float* w, int src_krsc, int64_t k, int64_t c, int64_t kh, int64_t kw,
                        const float* clip, int8_t* q_krsc, int64_t c_pad, int64_t ld_krsc, int8_t* q_crsk,
                        int64_t k_pad, int64_t ld_crsk, float* amax);
/* quantize(x, p, kStochastic, stream) (quantize.cpp:33-43) on a flat tensor,
 * draws in row-major order from the device LCG state, which is advanced by n. */
int i8t_quantize_stochastic(i8t_ctx* ctx, const float* x, int64_t n, const float* clip, uint32_t* lcg_state,
                            int8_t* q);
/* quantize_partitioned (quantize.cpp:45-79): chunk k seeded base_seed + k. */
int i8t_quantize_partitioned(i8t_ctx* ctx, const float* x, int64_t n, const float* clip, uint32_t base_seed,
                             int partitions, int8_t* q);
/* dequantize (quantize.cpp:81-87). */
/* One layer of i8t_quantize_weights_multi (64 bytes, plain C layout): the
 * arguments of i8t_quantize_weight for that layer (depthwise weights: k = C,
 * c = 1, c_pad = 1, ld_krsc = kh*kw, q_crsk = NULL).  Padding bytes of the
 * outputs are not written: zero them once when allocating. */
typedef struct {
  const float* w;
  const float* clip;
  int8_t* q_krsc;
  int8_t* q_crsk;
  int32_t k, c, rs, c_pad, ld_krsc, k_pad, ld_crsk, src_krsc;
} i8t_wq_desc;
/* i8t_quantize_weight for n_layers layers in one launch; dev_descs is a
 * DEVICE array of descriptors (built once, the pointers stay valid). */
int i8t_quantize_weights_multi(i8t_ctx* ctx, const i8t_wq_desc* dev_descs, int n_layers);
int i8t_dequantize(i8t_ctx* ctx, const int8_t* q, int64_t n, const float* clip, float* out);
/* Layout helpers for the drop-in path. */
int i8t_nhwc_to_nchw_f32(i8t_ctx* ctx, const float* src, int64_t n, int64_t c, int64_t hw, int64_t ld_src,
                         float* dst);
/* im2col_i8 / im2col_channel_i8 (conv.cpp:23-47, 98-106) for channels
 * [c_lo, c_hi): NCHW int8 x -> col [(c-c_lo)*kh*kw + i*kw + j][n*oh*ow + p*ow + q],
 * zero padding (the reference's explicit-GEMM operand; the convolutions here
 * never materialise it -- this is the API function). */
int i8t_im2col_s8(i8t_ctx* ctx, const int8_t* x, const i8t_conv_geom* g, int64_t c_lo, int64_t c_hi, int8_t* col);
int i8t_nchw_to_nhwc_i8(i8t_ctx* ctx, const int8_t* src, int64_t n, int64_t c, int64_t hw, int8_t* dst,
                        int64_t c_pad);
int i8t_kcrs_to_krsc_i8(i8t_ctx* ctx, const int8_t* src, int64_t k, int64_t c, int64_t kh, int64_t kw, int8_t* dst,
                        int64_t c_pad, int64_t ld);
int i8t_kcrs_to_crsk_i8(i8t_ctx* ctx, const int8_t* src, int64_t k, int64_t c, int64_t kh, int64_t kw, int8_t* dst,
                        int64_t k_pad, int64_t ld);

/* ------------------------------------------------------------ reductions */
/* max_abs / sq_l2_norm / dot / has_nonfinite (tensor.cpp:72-101); results
 * written to device scalars.  Sums are double, deterministic for a given n. */
int i8t_max_abs(i8t_ctx* ctx, const float* x, int64_t n, float* out);
int i8t_sq_l2_norm(i8t_ctx* ctx, const float* x, int64_t n, double* out);
/* Histogram (stats.hpp:11-23, `make_histogram`; declared by the reference
 * without an implementation): `bins` (1..8192) uniform bins over [-m, m],
 * m = max|x| over the finite samples ([-1, 1] when m == 0); bin =
 * floor((v - lo) / (hi - lo) * bins)
 * in double, clamped to [0, bins - 1]; non-finite samples are not counted.
 * counts: device int64[bins]; lo_hi: device double[2] (may be NULL). */
int i8t_histogram(i8t_ctx* ctx, const float* x, int64_t n, int bins, int64_t* counts, double* lo_hi);
int i8t_dot(i8t_ctx* ctx, const float* a, const float* b, int64_t n, double* out);
int i8t_has_nonfinite(i8t_ctx* ctx, const float* x, int64_t n, int32_t* out);

/* ------------------------------------------------------------ DSGC / DCLR */
/* cosine_distance (clip.cpp:8-22). */
int i8t_cosine_distance(i8t_ctx* ctx, const float* g, const float* h, int64_t n, double* out);
/* measure_dc (clip.cpp:24-28) at a host clip value. */
int i8t_measure_dc(i8t_ctx* ctx, const float* g, int64_t n, float clip, double* out);
/* search_clip (clip.cpp:30-78); result {clip, dc} in device memory. */
int i8t_search_clip(i8t_ctx* ctx, const float* g, int64_t n, int grid, int rounds, float prev_clip,
                    float* clip_out, double* dc_out);
int64_t i8t_dsgc_state_size(void);
int i8t_dsgc_init(i8t_ctx* ctx, void* state, int64_t period);
int i8t_dsgc_read(i8t_ctx* ctx, const void* state, i8t_dsgc_view* host_out);
int i8t_dsgc_write(i8t_ctx* ctx, void* state, const i8t_dsgc_view* host_in);
/* maybe_update (clip.cpp:80-93) on a device state.  `due` is decided on the
 * host from (iter, iter_of_last_update, period, clip > 0): pass the host
 * mirror; i8t_dsgc_read() gives it back. */
int i8t_maybe_update(i8t_ctx* ctx, void* state, const float* g, int64_t n, int64_t iter, int grid, int rounds,
                     int due);
/* quantize_gradient (layers.cpp:19-59): Periodic-Update DSGC, phi(d_c) with
 * (alpha, beta, form), zero-gradient skip, stochastic quantisation from the
 * device LCG state and the eps/g_hat statistics, fused into one pass over g
 * on non-search iterations.  g is [rows = N*H*W, cols = C] NHWC (or flat:
 * rows = 1 ... use hw = rows, c = 1) with the reference's NCHW draw order:
 * element (n, c, hw) consumes draw index (n*C + c)*HW + hw.
 * q is written NHWC with channel stride ld_q. */
int i8t_quantize_gradient(i8t_ctx* ctx, void* state, const float* g, int64_t n_img, int64_t c, int64_t hw,
                          int64_t iter, int grid, int rounds, int search_enabled, int due, int lr_scaling_enabled,
                          double alpha, double beta, int form, uint32_t* lcg_state, int8_t* q, int64_t ld_q);
/* i8t_quantize_gradient with the search's first-pass statistics of g already
 * reduced (i8t_bn_bwd_apply_stats): a due search skips its pass over g. */
int i8t_quantize_gradient_stats(i8t_ctx* ctx, void* state, const float* g, int64_t n_img, int64_t C, int64_t HW,
                                int64_t iter, int grid, int rounds, int search_enabled, int due, int lr_scaling_enabled,
                                double alpha, double beta, int form, uint32_t* lcg_state, int8_t* q, int64_t ld_q,
                                const double* stats);
/* scale_factor (lr_scale.cpp:8-20), host scalar helper. */
int i8t_scale_factor(double dc, double alpha, double beta, int form, double* out);

/* ------------------------------------------------------------ convolutions */
/* Forward: z = float(double(s_a)*double(s_w)*acc), conv2d_q (conv.cpp:108-145).
 *   a   : NHWC int8, channel stride c_pad (multiple of 4, >= c)
 *   w   : KRSC int8 rows, row stride ld_w (multiple of 16, >= kh*kw*c_pad)
 *   z   : NHWC float [N*P*Q][K] (may be NULL); acc: int32 same shape (may be NULL) */
int i8t_conv_fwd(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* a, int64_t c_pad, const int8_t* w,
                 int64_t ld_w, const float* clip_a, const float* clip_w, float* z, int32_t* acc);
/* Backward-data (conv.cpp:197-203): ga = float(double(s_g)*double(s_w)*acc).
 *   gz  : NHWC int8 [N*P*Q][k_pad]; wt: CRSK int8 rows (stride ld_wt)
 *   ga  : NHWC float [N*H*W][C] (may be NULL); acc int32 (may be NULL) */
int i8t_conv_dgrad(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, int64_t k_pad, const int8_t* wt,
                   int64_t ld_wt, const float* clip_g, const float* clip_w, float* ga, int32_t* acc);
/* Backward-data with the residual join fused into its epilogue (the shortcut
 * gradient sum of ResidualBlock::backward, layers.cpp:458-464):
 *   ga = dgrad + add_g                 (add_y == NULL: projection shortcut)
 *   ga = dgrad + add_g * (add_y > 0)   (identity shortcut through the block ReLU)
 * add_g / add_y: NHWC fp32 [N*H*W][C], 16-byte aligned, C % 4 == 0.  One float
 * add per element, so ga equals i8t_conv_dgrad followed by the join bit for bit.
 * ga may alias add_g when add_y == NULL (in-place join): the pixels a strided
 * dgrad gives no taps then keep add_g as is (0 + x, except that -0 stays -0). */
int i8t_conv_dgrad_join(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, int64_t k_pad, const int8_t* wt,
                        int64_t ld_wt, const float* clip_g, const float* clip_w, float* ga, const float* add_g,
                        const float* add_y);
/* The same join with the block ReLU mask as packed bits (bit e % 32 of word
 * e / 32 for the flat NHWC index e, as i8t_bn_act_q writes them):
 *   ga = dgrad + add_g * bit           (add_bits == NULL: no mask) */
int i8t_conv_dgrad_join_bits(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, int64_t k_pad, const int8_t* wt,
                             int64_t ld_wt, const float* clip_g, const float* clip_w, float* ga, const float* add_g,
                             const uint32_t* add_bits);
/* Backward-weight (conv.cpp:186-195), int64 accumulation (no depth bound):
 *   acc : int64 accumulator [kh*kw*c_pad][K] (written by the call; may be NULL
 *         when gw is given: single device, the accumulator is not kept)
 *   gw  : float weights, KCRS when out_kcrs != 0 else KRSC (may be NULL) */
int i8t_conv_wgrad(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, int64_t k_pad, const int8_t* a,
                   int64_t c_pad, const float* clip_g, const float* clip_a, int64_t* acc, float* gw, int out_kcrs);
/* Rescale an (all-reduced) int64 wgrad accumulator into float weights; the
 * data-parallel path calls i8t_conv_wgrad with gw == NULL, sums `acc` across
 * ranks (exact), then this. */
int i8t_conv_wgrad_finalize(i8t_ctx* ctx, const i8t_conv_geom* g, const int64_t* acc, int64_t c_pad,
                            const float* clip_g, const float* clip_a, float* gw, int out_kcrs);
/* Depthwise (conv.cpp:115-131, :159-184): a, gz NHWC int8 with channel
 * stride c_pad; w (C, kh*kw) int8.  Outputs NHWC float / (C, kh*kw) float. */
int i8t_conv_dw_fwd(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* a, int64_t c_pad, const int8_t* w,
                    const float* clip_a, const float* clip_w, float* z, int32_t* acc);
int i8t_conv_dw_dgrad(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, int64_t c_pad, const int8_t* w,
                      const float* clip_g, const float* clip_w, float* ga, int32_t* acc);
int i8t_conv_dw_wgrad(i8t_ctx* ctx, const i8t_conv_geom* g, const int8_t* gz, const int8_t* a, int64_t c_pad,
                      const float* clip_g, const float* clip_a, int64_t* acc, float* gw);
/* gw [C][kh*kw] = float(double(s_g)*double(s_a)*acc) from an (all-reduced) int64 accumulator. */
int i8t_conv_dw_wgrad_finalize(i8t_ctx* ctx, const i8t_conv_geom* g, const int64_t* acc, const float* clip_g,
                               const float* clip_a, float* gw);
/* gemm_i8 (gemm.cpp:18-40): C[m][n] = A[m][k] . B[k][n] exact int32
 * (row-major int8 operands; runs on the tcgen05 path as a 1x1 convolution). */
int i8t_gemm_s8(i8t_ctx* ctx, const int8_t* a, const int8_t* b, int64_t m, int64_t k, int64_t n, int32_t* c);
/* gemm_i8_fused_lhs (gemm.cpp:49-64): C = quantize(A, from_clip(*clip), mode
 * [, stream]) . B on the device, A fp32 row-major (m x k); stochastic draws in
 * row-major order from *lcg_state (device), advanced by m*k. */
int i8t_gemm_s8_fused_lhs(i8t_ctx* ctx, const float* a, int64_t m, int64_t k, const float* clip, int stochastic,
                          uint32_t* lcg_state, const int8_t* b, int64_t n, int32_t* c);

/* ------------------------------------------------------------ optimiser */
/* SGD step of Trainer::train_step (train.cpp:97-117), momentum 0:
 *   w[i] -= float(lr * g[i]),  lr = base_lr * (state ? state.lr_scale : 1).
 * skip (device int32, may be NULL): when non-zero the step is skipped (the
 * reference returns before the update on a non-finite gradient, :87-95). */
int i8t_sgd_dclr(i8t_ctx* ctx, float* w, const float* grad, int64_t n, double base_lr, const void* state,
                 const int32_t* skip);

/* ------------------------------------------------------------ fused BatchNorm2d + ReLU
 * BatchNorm2d (layers.cpp:230-323) and ReLU (:328-344) are FP32 layers the
 * reference never quantises; these fuse them into the INT8 path's HBM passes.
 * Tensors are NHWC [m = N*H*W][c] fp32, c % 4 == 0.  bn: device doubles [6c]
 * (mean, invstd, k*s1/m, k*s2/m, k = gamma*invstd, ReLU-mask bounds), filled by the
 * calls below.  mask_mode: 0 none, 1 ReLU mask recomputed from bn(z) > 0,
 * 2 mask_y > 0, 3 mask_y points at packed mask bits (uint32 words, see
 * i8t_bn_act_q).  With mask_mode 1, i8t_bn_bwd_reduce also stores per channel
 * the float interval [lo, hi] with relu(bn(z)) > 0 <=> lo <= z <= hi (the map
 * z -> float(gamma*x_hat + beta) is monotone), which i8t_bn_bwd_apply and
 * i8t_quantize_gradient_bn then read: call them after i8t_bn_bwd_reduce. */
int i8t_bn_fwd_stats(i8t_ctx* ctx, const float* z, int64_t m, int64_t c, double momentum, double eps, double* bn,
                     float* running_mean, float* running_var);
/* Max pooling k x k / stride s / zero-free padding `pad` on NHWC fp32 (the
 * reference Pool2d, layers.cpp:346-380, has no padding: EXT).  x [n,h,w,c],
 * y [n,P,Q,c], idx [n,P,Q,c] uint8 window slot (dy*k + dx) of the first max.
 * With bn != NULL the input is act(bn(x)) (bn: i8t_bn_fwd_stats output,
 * relu: apply ReLU) computed on the fly: the stem's BN + ReLU + pool in one pass. */
int i8t_maxpool_fwd(i8t_ctx* ctx, const float* x, int64_t n, int64_t h, int64_t w, int64_t c, int64_t k, int64_t s,
                    int64_t pad, const double* bn, const float* gamma, const float* beta, int relu, float* y,
                    uint8_t* idx);
/* gx [n,h,w,c] = sum of gy over the windows whose argmax (idx) is (h, w). */
int i8t_maxpool_bwd(i8t_ctx* ctx, const float* gy, const uint8_t* idx, int64_t n, int64_t h, int64_t w, int64_t c,
                    int64_t k, int64_t s, int64_t pad, float* gx);
/* SoftmaxCrossEntropy::loss_and_grad (layers.cpp:507-529) on the device:
 * logits [n][classes] fp32, labels [n] int64; g_logits = float((p - y) / n_total),
 * *loss = sum of the row losses / n_total (double; n_total = the global batch
 * under data parallelism), *bad = 1 when the loss or any logit is non-finite
 * (the divergence check of train.cpp:73-77), else 0. */
int i8t_softmax_ce(i8t_ctx* ctx, const float* logits, const int64_t* labels, int64_t n, int64_t classes,
                   int64_t n_total, float* g_logits, double* loss, int32_t* bad);
/* Global average pool, NHWC [n][hw][c] -> [n][c]: float(double sum / hw) per
 * (n, c), summed in the reference's order (Pool2d kAvg over the whole map,
 * layers.cpp:383-388); backward gx[n][p][c] = g[n][c] / float(hw)
 * (layers.cpp:392-414; c % 4 == 0, 16-byte aligned). */
int i8t_global_avgpool_fwd(i8t_ctx* ctx, const float* x, int64_t n, int64_t hw, int64_t c, float* y);
int i8t_global_avgpool_bwd(i8t_ctx* ctx, const float* g, int64_t n, int64_t hw, int64_t c, float* gx);
/* q = quantize_nearest(act(bn(z)), clip) with running max|act| -> *amax: the
 * next conv's input quantiser (layers.cpp:101, 109) fused with BN + ReLU. */
int i8t_bn_act_quant(i8t_ctx* ctx, const float* z, int64_t m, int64_t c, const double* bn, const float* gamma,
                     const float* beta, int relu, const float* clip, int8_t* q, float* amax);
/* y = act(bn(z) + residual): residual = res (fp32) or bn'(res_z) (NULL: none). */
int i8t_bn_act(i8t_ctx* ctx, const float* z, int64_t m, int64_t c, const double* bn, const float* gamma,
               const float* beta, int relu, const float* res, const float* res_z, const double* res_bn,
               const float* res_gamma, const float* res_beta, float* y);
/* BN backward reduction: dbeta = sum g_m, dgamma = sum g_m * x_hat. */
/* i8t_bn_act with optional extra outputs of the same pass (NULL = skip):
 *   q (+ clip, amax): quantize_nearest(y, clip) (NHWC int8, channel stride c)
 *     with running max|y| -> *amax: the next conv's int8 input
 *     (layers.cpp:101, 108-109, 451-456);
 *   mask_bits: y > 0 packed one bit per element (word e/32, bit e%32, m*c/32
 *     words rounded up): everything the backward needs of y (mask mode 3). */
int i8t_bn_act_q(i8t_ctx* ctx, const float* z, int64_t m, int64_t c, const double* bn, const float* gamma,
                 const float* beta, int relu, const float* res, const float* res_z, const double* res_bn,
                 const float* res_gamma, const float* res_beta, float* y, const float* clip, int8_t* q, float* amax,
                 uint32_t* mask_bits);
int i8t_bn_bwd_reduce(i8t_ctx* ctx, const float* g, const float* z, int64_t m, int64_t c, double* bn,
                      const float* gamma, const float* beta, int mask_mode, const float* mask_y, float* grad_gamma,
                      float* grad_beta);
/* i8t_bn_bwd_reduce (mask_mode 3, mask_bits) of g_out = a_add + g * join_bit,
 * with g_out also written (bit for bit i8t_add_masked_bits(a_add, g,
 * join_bits) followed by i8t_bn_bwd_reduce): the identity-shortcut join of a
 * residual block's backward fused with the preceding BN's column sums
 * (layers.cpp:458-464 then 285-300). */
int i8t_bn_bwd_reduce_join(i8t_ctx* ctx, const float* a_add, const float* g, const uint32_t* join_bits,
                           const float* z, int64_t m, int64_t c, double* bn, const float* gamma, const float* beta,
                           const uint32_t* mask_bits, float* grad_gamma, float* grad_beta, float* g_out);
/* i8t_bn_bwd_apply that also reduces the statistics of the value it writes:
 * stats[0] = max|gz|, stats[1] = non-finite count, stats[2] = sum gz^2 (3 device
 * doubles, fixed-order reduction) -- the first pass of a DSGC search over gz
 * (clip.cpp:32-34), handed to i8t_quantize_gradient_stats. */
int i8t_bn_bwd_apply_stats(i8t_ctx* ctx, const float* g, const float* z, int64_t m, int64_t c, const double* bn,
                           const float* gamma, const float* beta, int mask_mode, const float* mask_y, float* gz,
                           double* stats);
/* i8t_bn_bwd_reduce_join plus a second BatchNorm reduced on the same masked
 * g_out in the same pass (z2 / bn2 / gamma2 -> grad_gamma2, grad_beta2 =
 * grad_beta): the projection block's shortcut BN beside the main branch's last
 * BN (ResidualBlock::backward, layers.cpp:458-464).  Bit for bit the two
 * separate reductions. */
int i8t_bn_bwd_reduce_join2(i8t_ctx* ctx, const float* a_add, const float* g, const uint32_t* join_bits,
                            const float* z, int64_t m, int64_t c, double* bn, const float* gamma, const float* beta,
                            const uint32_t* mask_bits, float* grad_gamma, float* grad_beta, const float* z2,
                            double* bn2, const float* gamma2, float* grad_gamma2, float* grad_beta2, float* g_out);
/* gz = BN backward (materialised fp32). */
int i8t_bn_bwd_apply(i8t_ctx* ctx, const float* g, const float* z, int64_t m, int64_t c, const double* bn,
                     const float* gamma, const float* beta, int mask_mode, const float* mask_y, float* gz);
/* quantize_gradient (layers.cpp:19-59) of the BN-backward value computed on
 * the fly (non-search iterations: maybe_update's measurement branch). */
int i8t_quantize_gradient_bn(i8t_ctx* ctx, void* state, const float* g, const float* z, int64_t n_img, int64_t c,
                             int64_t hw, const double* bn, const float* gamma, const float* beta, int mask_mode,
                             const float* mask_y, int lr_scaling_enabled, double alpha, double beta_, int form,
                             uint32_t* lcg_state, int8_t* q);
/* out = a + g * (y > 0) (ResidualBlock backward with an identity shortcut). */
int i8t_add_masked(i8t_ctx* ctx, const float* a, const float* g, const float* y, int64_t n, float* out);
/* out = a + g * mask with the packed mask bits of i8t_bn_act_q. */
int i8t_add_masked_bits(i8t_ctx* ctx, const float* a, const float* g, const uint32_t* bits, int64_t n, float* out);

/* All parameters in one launch: w and grad are flat arenas; segment i covers
 * [seg_off[i], seg_off[i+1]) (multiples of 4, device int64) and uses the
 * DCLR factor of device state seg_state[i] (device array of pointers; NULL
 * entry = phi 1).  Same arithmetic as i8t_sgd_dclr per element.
 * lr_dev (device double, may be NULL): when given, replaces base_lr (so a
 * captured CUDA graph reads the step's cosine LR from device memory).
 * mom (flat arena like w, may be NULL): the reference's momentum update
 * (train.cpp:106-111) buf = float(momentum*buf + g), w -= float(lr*buf). */
int i8t_sgd_dclr_multi(i8t_ctx* ctx, float* w, const float* grad, int nseg, const int64_t* seg_off,
                       const void* const* seg_state, double base_lr, const double* lr_dev, const int32_t* skip,
                       float* mom, double momentum);
/* Non-finite scan of a flat gradient arena: *flag = 1 if any element is
 * NaN/Inf (has_nonfinite, tensor.cpp:96-101, over every parameter gradient). */
int i8t_nonfinite_flag(i8t_ctx* ctx, const float* x, int64_t n, int32_t* flag);

#ifdef __cplusplus
}
#endif
#endif /* I8T_CUDA_H */
