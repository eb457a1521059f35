// ref_capi.cpp -- extern "C" probe over the UNMODIFIED reference i8t_core.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference's own sources, where they lie under /root/reference/proj/core,
// into oracle/_ref/libi8t_ref.so (git-ignored; it travels to the GPU box as a
// prebuilt file).  It is used to (1) pin the C restatement in oracle/oracle.c,
// (2) dump golden vectors into tests/golden/, (3) time the reference CPU path
// for bench.py's cpu_baseline / --impl reference arm.  No reference source is
// copied into this repo; this file only calls the reference's public API.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <vector>

#include <memory>
#include <string>

#include "i8t/checkpoint.hpp"
#include "i8t/clip.hpp"
#include "i8t/conv.hpp"
#include "i8t/dataset.hpp"
#include "i8t/models.hpp"
#include "i8t/train.hpp"
#include "i8t/gemm.hpp"
#include "i8t/layers.hpp"
#include "i8t/lr_scale.hpp"
#include "i8t/quantize.hpp"
#include "i8t/rng.hpp"
#include "i8t/tensor.hpp"

using namespace i8t;

namespace {

// 0 ok, 1 invalid_argument, 2 domain_error, 3 other
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::domain_error&) {
    return 2;
  } catch (...) {
    return 3;
  }
}

Tensor vec_tensor(const float* x, int64_t n) { return Tensor(Shape{n}, std::vector<float>(x, x + n)); }

Tensor shaped(const float* x, Shape s) {
  const int64_t n = s.numel();
  return Tensor(std::move(s), std::vector<float>(x, x + n));
}

QuantizedTensor wrap(const int8_t* q, Shape s, float clip) {
  QuantizedTensor t;
  t.q.assign(q, q + s.numel());
  t.shape = std::move(s);
  t.params = QuantParams::from_clip(clip);
  return t;
}

ConvGeometry geom(const int64_t* g) {
  // g = {n, c, h, w, k, kh, kw, stride, pad, depthwise}
  ConvGeometry cg;
  cg.n = g[0]; cg.c = g[1]; cg.h = g[2]; cg.w = g[3];
  cg.k = g[4]; cg.kh = g[5]; cg.kw = g[6];
  cg.stride = g[7]; cg.pad = g[8]; cg.depthwise = g[9] != 0;
  return cg;
}

}  // namespace

extern "C" {

uint32_t ref_lcg_next(uint32_t* state) {
  LcgStream s(*state);
  uint32_t v = s.next_state();
  *state = s.state();
  return v;
}

double ref_lcg_uniform(uint32_t* state) {
  LcgStream s(*state);
  double u = s.next_uniform();
  *state = s.state();
  return u;
}

int ref_quant_params(float clip, float* scale) {
  return guard([&] { *scale = QuantParams::from_clip(clip).scale; });
}

int ref_quantize(const float* x, int64_t n, float clip, int mode, uint32_t* stream, int8_t* q) {
  return guard([&] {
    Tensor t = vec_tensor(x, n);
    QuantParams p = QuantParams::from_clip(clip);
    if (mode == 0) {
      auto r = quantize(t, p, RoundingMode::kNearest, nullptr);
      std::memcpy(q, r.q.data(), static_cast<size_t>(n));
    } else {
      LcgStream s(*stream);
      auto r = quantize(t, p, RoundingMode::kStochastic, &s);
      std::memcpy(q, r.q.data(), static_cast<size_t>(n));
      *stream = s.state();
    }
  });
}

int ref_quantize_partitioned(const float* x, int64_t n, float clip, uint32_t seed, int parts, int threads,
                             int8_t* q) {
  return guard([&] {
    auto r = quantize_partitioned(vec_tensor(x, n), QuantParams::from_clip(clip), seed, parts, threads);
    std::memcpy(q, r.q.data(), static_cast<size_t>(n));
  });
}

int ref_dequantize(const int8_t* q, int64_t n, float clip, float* out) {
  return guard([&] {
    Tensor t = dequantize(wrap(q, Shape{n}, clip));
    std::memcpy(out, t.data(), sizeof(float) * static_cast<size_t>(n));
  });
}

float ref_max_abs(const float* x, int64_t n) { return max_abs(vec_tensor(x, n)); }
double ref_sq_l2_norm(const float* x, int64_t n) { return sq_l2_norm(vec_tensor(x, n)); }
double ref_dot(const float* a, const float* b, int64_t n) { return dot(vec_tensor(a, n), vec_tensor(b, n)); }
int ref_has_nonfinite(const float* x, int64_t n) { return has_nonfinite(vec_tensor(x, n)) ? 1 : 0; }

int ref_gemm_i8(const int8_t* a, const int8_t* b, int64_t m, int64_t k, int64_t n, int threads, int32_t* c) {
  return guard([&] {
    Int8Matrix A(m, k), B(k, n);
    std::memcpy(A.data.data(), a, static_cast<size_t>(m * k));
    std::memcpy(B.data.data(), b, static_cast<size_t>(k * n));
    Int32Matrix C = gemm_i8(A, B, threads);
    std::memcpy(c, C.data.data(), sizeof(int32_t) * static_cast<size_t>(m * n));
  });
}

int ref_im2col_i8(const int8_t* x, const int64_t* g, int8_t* out) {
  return guard([&] {
    ConvGeometry cg = geom(g);
    cg.validate();
    im2col_i8(x, cg, out);
  });
}

int ref_conv2d_q(const int8_t* qa, float clip_a, const int8_t* qw, float clip_w, const int64_t* g, int threads,
                 float* z) {
  return guard([&] {
    ConvGeometry cg = geom(g);
    Tensor out = conv2d_q(wrap(qa, cg.input_shape(), clip_a), wrap(qw, cg.weight_shape(), clip_w), cg, threads);
    std::memcpy(z, out.data(), sizeof(float) * static_cast<size_t>(out.numel()));
  });
}

int ref_conv2d_backward_q(const int8_t* qg, float clip_g, const int8_t* qa, float clip_a, const int8_t* qw,
                          float clip_w, const int64_t* g, int threads, float* gw, float* ga) {
  return guard([&] {
    ConvGeometry cg = geom(g);
    auto [tw, ta] = conv2d_backward_q(wrap(qg, cg.output_shape(), clip_g), wrap(qa, cg.input_shape(), clip_a),
                                      wrap(qw, cg.weight_shape(), clip_w), cg, threads);
    std::memcpy(gw, tw.data(), sizeof(float) * static_cast<size_t>(tw.numel()));
    std::memcpy(ga, ta.data(), sizeof(float) * static_cast<size_t>(ta.numel()));
  });
}

double ref_cosine_distance(const float* g, const float* h, int64_t n) {
  return cosine_distance(vec_tensor(g, n), vec_tensor(h, n));
}

int ref_measure_dc(const float* g, int64_t n, float clip, double* dc) {
  return guard([&] { *dc = measure_dc(vec_tensor(g, n), clip); });
}

int ref_search_clip(const float* g, int64_t n, int grid, int rounds, float prev, float* clip, double* dc) {
  return guard([&] {
    ClipSearchConfig cfg{.grid_resolution = grid, .refine_rounds = rounds};
    auto r = search_clip(vec_tensor(g, n), cfg, prev);
    *clip = r.clip;
    *dc = r.dc;
  });
}

// state = {clip(float), last_dc(double), iter_of_last_update(int64), period(int64)} as a struct
struct RefClipState {
  float clip;
  double last_dc;
  int64_t iter_of_last_update;
  int64_t period;
};

int ref_maybe_update(RefClipState* st, const float* g, int64_t n, int64_t iter, int grid, int rounds) {
  return guard([&] {
    ClipState cs;
    cs.clip = st->clip;
    cs.last_dc = st->last_dc;
    cs.iter_of_last_update = st->iter_of_last_update;
    cs.period = st->period;
    maybe_update(cs, vec_tensor(g, n), iter, ClipSearchConfig{.grid_resolution = grid, .refine_rounds = rounds});
    st->clip = cs.clip;
    st->last_dc = cs.last_dc;
    st->iter_of_last_update = cs.iter_of_last_update;
  });
}

int ref_scale_factor(double dc, double alpha, double beta, int form, double* out) {
  return guard([&] {
    LrScaleConfig cfg{.alpha = alpha, .beta = beta, .form = static_cast<ScaleForm>(form)};
    *out = scale_factor(dc, cfg);
  });
}

// One INT8 Conv2d layer step through the reference layer API
// (layers.cpp:98-126 forward/backward, quantize_gradient :19-59).
// io_stats out: {clip_w, clip_a, grad_clip, dc, lr_scale, eps_norm, ghat_sqnorm}
int ref_conv_layer_step(const int64_t* g, const float* weight, const float* x, const float* g_out, int64_t iter,
                        int64_t period, int grid, int rounds, uint32_t* stream, RefClipState* cs, float* z,
                        float* gw, float* ga, double* stats) {
  return guard([&] {
    ConvGeometry cg = geom(g);
    if (cg.kh != cg.kw) throw std::invalid_argument("square kernels only");
    InitRng rng(1);
    Conv2d conv(cg.c, cg.depthwise ? cg.c : cg.k, cg.kh, cg.stride, cg.pad, cg.depthwise, rng);
    conv.set_quantized(true);
    Tensor& w = conv.weight();
    std::memcpy(w.data(), weight, sizeof(float) * static_cast<size_t>(w.numel()));
    QuantState* qs = conv.quant_state();
    qs->clip_state.clip = cs->clip;
    qs->clip_state.last_dc = cs->last_dc;
    qs->clip_state.iter_of_last_update = cs->iter_of_last_update;
    ForwardCtx f{.mode = Mode::kInt8, .training = true, .track_amax = true, .threads = 0};
    Tensor out = conv.forward(shaped(x, cg.input_shape()), f);
    std::memcpy(z, out.data(), sizeof(float) * static_cast<size_t>(out.numel()));
    LcgStream s(*stream);
    BackwardCtx b;
    b.mode = Mode::kInt8;
    b.iter = iter;
    b.grad_stream = &s;
    b.clip_cfg = ClipSearchConfig{.grid_resolution = grid, .refine_rounds = rounds};
    b.clip_period = period;
    b.threads = 0;
    Tensor gin = conv.backward(shaped(g_out, cg.output_shape()), b);
    std::memcpy(ga, gin.data(), sizeof(float) * static_cast<size_t>(gin.numel()));
    for (ParamRef p : conv.params())
      if (p.name == "weight") std::memcpy(gw, p.grad->data(), sizeof(float) * static_cast<size_t>(p.grad->numel()));
    *stream = s.state();
    cs->clip = qs->clip_state.clip;
    cs->last_dc = qs->clip_state.last_dc;
    cs->iter_of_last_update = qs->clip_state.iter_of_last_update;
    stats[0] = qs->clip_w;
    stats[1] = qs->clip_a;
    stats[2] = qs->clip_state.clip;
    stats[3] = qs->dc;
    stats[4] = qs->lr_scale;
    stats[5] = qs->eps_norm;
    stats[6] = qs->ghat_sqnorm;
  });
}

// InitRng-driven synthetic fills, for cross-checking the oracle generators.
void ref_fill_gaussian(float* x, int64_t n, uint64_t seed, double stddev) {
  InitRng r(seed);
  for (int64_t i = 0; i < n; ++i) x[i] = static_cast<float>(r.next_gaussian() * stddev);
}


// ---------------------------------------------------------------------------
// Model / Trainer / checkpoint probe over the reference's own classes
// (models.cpp, train.cpp, checkpoint.cpp).  Models: the reference's
// build_model names, plus two nets composed here from the reference's public
// Layer classes with only the geometry the reference accepts (stride 1):
//   "res_s1"  stem conv3x3(3->8) bn relu, ResidualBlock(8,8,1),
//             ResidualBlock(8,16,1) (projection shortcut), gap, fc(16)
//   "mbv2_s1" stem conv3x3(3->8) bn relu, InvertedResidual(8,12,1,2),
//             InvertedResidual(12,12,1,2), head conv1x1(12->16) bn relu, gap, fc(16)
// gap = Pool2d(avg, side, side) over the (side x side) input plane.

int ref_model_new(const char* name, uint64_t seed, int side, int classes, void** out) {
  return guard([&] {
    std::string nm(name);
    auto m = std::make_unique<Model>();
    if (nm == "res_s1" || nm == "mbv2_s1") {
      InitRng rng(seed);
      m->name = nm;
      m->input_shape = Shape{3, side, side};
      m->num_classes = classes;
      m->net = std::make_unique<Sequential>();
      m->net->add("stem", std::make_unique<Conv2d>(3, 8, 3, 1, 1, false, rng));
      m->net->add("stem_bn", std::make_unique<BatchNorm2d>(8));
      m->net->add("stem_relu", std::make_unique<ReLU>());
      int64_t last = 16;
      if (nm == "res_s1") {
        m->net->add("block1", std::make_unique<ResidualBlock>(8, 8, 1, rng));
        m->net->add("block2", std::make_unique<ResidualBlock>(8, 16, 1, rng));
      } else {
        m->net->add("block1", std::make_unique<InvertedResidual>(8, 12, 1, 2, rng));
        m->net->add("block2", std::make_unique<InvertedResidual>(12, 12, 1, 2, rng));
        m->net->add("head", std::make_unique<Conv2d>(12, 16, 1, 1, 0, false, rng));
        m->net->add("head_bn", std::make_unique<BatchNorm2d>(16));
        m->net->add("head_relu", std::make_unique<ReLU>());
      }
      m->net->add("gap", std::make_unique<Pool2d>(PoolKind::kAvg, side, side));
      m->net->add("fc", std::make_unique<Dense>(last, classes, rng));
    } else {
      *m = build_model(nm, seed, 3 * 32 * 32, classes);
    }
    *out = m.release();
  });
}

void ref_model_free(void* m) { delete static_cast<Model*>(m); }

namespace {
std::vector<std::pair<std::string, Tensor*>> model_tensors(Model* m) {
  std::vector<std::pair<std::string, Tensor*>> out;
  for (auto& [path, layer] : m->leaves()) {
    for (ParamRef p : layer->params()) out.emplace_back(path + "." + p.name, p.value);
    for (ParamRef p : layer->buffers()) out.emplace_back(path + "." + p.name, p.value);
  }
  return out;
}
}  // namespace

int ref_model_ntensors(void* m) { return static_cast<int>(model_tensors(static_cast<Model*>(m)).size()); }

// name (NUL-terminated, truncated to cap), rank and dims[<=4] of tensor i
int ref_model_tensor_info(void* m, int i, char* name, int cap, int* rank, int64_t* dims) {
  return guard([&] {
    auto t = model_tensors(static_cast<Model*>(m)).at(static_cast<size_t>(i));
    std::snprintf(name, static_cast<size_t>(cap), "%s", t.first.c_str());
    *rank = t.second->shape().rank();
    for (int d = 0; d < *rank; ++d) dims[d] = t.second->shape()[d];
  });
}

int ref_model_tensor_get(void* m, int i, float* out) {
  return guard([&] {
    Tensor* t = model_tensors(static_cast<Model*>(m)).at(static_cast<size_t>(i)).second;
    std::memcpy(out, t->data(), sizeof(float) * static_cast<size_t>(t->numel()));
  });
}

int ref_model_tensor_set(void* m, int i, const float* in) {
  return guard([&] {
    Tensor* t = model_tensors(static_cast<Model*>(m)).at(static_cast<size_t>(i)).second;
    std::memcpy(t->data(), in, sizeof(float) * static_cast<size_t>(t->numel()));
  });
}

int ref_model_int8_replace(void* m) { return int8_replace(*static_cast<Model*>(m)->net); }

// cfg = {base_lr, momentum, alpha, beta}; icfg = {mode(0 fp32/1 int8), constant schedule, lr_scaling_enabled,
//        clip_enabled, clip_period, seed, grid, rounds, form}
int ref_trainer_new(void* m, const double* cfg, const int64_t* icfg, void** out) {
  return guard([&] {
    TrainConfig tc;
    tc.base_lr = cfg[0];
    tc.momentum = cfg[1];
    tc.lr_scale.alpha = cfg[2];
    tc.lr_scale.beta = cfg[3];
    tc.mode = icfg[0] ? Mode::kInt8 : Mode::kFp32;
    tc.schedule = icfg[1] ? LrSchedule::kConstant : LrSchedule::kCosine;
    tc.lr_scaling_enabled = icfg[2] != 0;
    tc.clip_enabled = icfg[3] != 0;
    tc.clip_period = icfg[4];
    tc.seed = static_cast<uint64_t>(icfg[5]);
    tc.clip_search.grid_resolution = static_cast<int>(icfg[6]);
    tc.clip_search.refine_rounds = static_cast<int>(icfg[7]);
    tc.lr_scale.form = static_cast<ScaleForm>(icfg[8]);
    tc.threads = 0;
    *out = new Trainer(*static_cast<Model*>(m), tc);
  });
}

void ref_trainer_free(void* t) { delete static_cast<Trainer*>(t); }

int ref_trainer_calibrate(void* t, void* m, const float* images, int64_t n) {
  return guard([&] {
    Model* mm = static_cast<Model*>(m);
    Shape s{n, mm->input_shape[0], mm->input_shape[1], mm->input_shape[2]};
    static_cast<Trainer*>(t)->calibrate(shaped(images, s));
  });
}

int ref_trainer_finish_calibration(void* t) { return guard([&] { static_cast<Trainer*>(t)->finish_calibration(); }); }
int ref_trainer_refresh(void* t) { return guard([&] { static_cast<Trainer*>(t)->refresh_wa_clips(); }); }

// one Trainer::train_step; out = {loss, diverged, base_lr_t}; layer_stats[5*L] = {dc, clip, lr_scale, eps, ghat2}
int ref_train_step(void* t, void* m, const float* images, int64_t n, const int32_t* labels, int64_t iter,
                   int64_t total, double* out, double* layer_stats) {
  return guard([&] {
    Model* mm = static_cast<Model*>(m);
    Shape s{n, mm->input_shape[0], mm->input_shape[1], mm->input_shape[2]};
    std::vector<int32_t> lab(labels, labels + n);
    StepReport r = static_cast<Trainer*>(t)->train_step(shaped(images, s), lab, iter, total);
    out[0] = r.loss;
    out[1] = r.diverged ? 1.0 : 0.0;
    out[2] = r.base_lr_t;
    for (size_t i = 0; i < r.layers.size(); ++i) {
      layer_stats[5 * i + 0] = r.layers[i].dc;
      layer_stats[5 * i + 1] = r.layers[i].clip;
      layer_stats[5 * i + 2] = r.layers[i].lr_scale;
      layer_stats[5 * i + 3] = r.layers[i].eps_norm;
      layer_stats[5 * i + 4] = r.layers[i].ghat_sqnorm;
    }
  });
}

// QuantState of quantised layer i: f = {clip_w, clip_a, pending_amax}, clip state
int ref_trainer_quant_state(void* t, int i, float* f, RefClipState* cs) {
  return guard([&] {
    Layer* l = static_cast<Trainer*>(t)->quant_layers().at(static_cast<size_t>(i)).second;
    QuantState* qs = l->quant_state();
    f[0] = qs->clip_w;
    f[1] = qs->clip_a;
    f[2] = qs->pending_amax;
    cs->clip = qs->clip_state.clip;
    cs->last_dc = qs->clip_state.last_dc;
    cs->iter_of_last_update = qs->clip_state.iter_of_last_update;
    cs->period = qs->clip_state.period;
  });
}

int ref_save_checkpoint(void* m, const char* path) {
  return guard([&] { save_checkpoint(*static_cast<Model*>(m), path); });
}
int ref_load_checkpoint(void* m, const char* path) {
  return guard([&] { load_checkpoint(*static_cast<Model*>(m), path); });
}

}  // extern "C"

// dataset.cpp does not compile, and the probe never loads a
// dataset; train.cpp's run_training/evaluate reference these two members, so
// the probe defines them (its own code) to fail loudly if ever reached.
namespace i8t {
Tensor Dataset::gather(const std::vector<int64_t>&) const {
  throw std::logic_error("ref_capi: datasets are outside the probe");
}
std::vector<int32_t> Dataset::gather_labels(const std::vector<int64_t>&) const {
  throw std::logic_error("ref_capi: datasets are outside the probe");
}
}  // namespace i8t
