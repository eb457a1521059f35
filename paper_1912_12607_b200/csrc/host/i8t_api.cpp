// i8t_api.cpp -- the reference's C++ operator API (include/i8t/i8t.hpp) on top
// of the C-ABI (include/i8t_cuda.h).  Host value types in, host value types
// out; every arithmetic op runs on the B200 through libi8t_cuda.so.  Argument
// validation mirrors the reference so errors surface as the same exception
// types (std::invalid_argument / std::domain_error), thrown before any device
// work where the reference throws before computing.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <stdexcept>

#include "i8t/i8t.hpp"
#include "i8t_cuda.h"

namespace i8t {
namespace {

// ---------------------------------------------------------------- plumbing
i8t_ctx* ctx() {
  static i8t_ctx* c = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    if (i8t_ctx_create(nullptr, &c) != I8T_OK) c = nullptr;
  });
  if (!c) throw std::runtime_error(std::string("i8t: no usable B200 device: ") + i8t_last_error());
  return c;
}

void throw_status(int rc) {
  const std::string msg = i8t_last_error();
  if (rc == I8T_EINVAL) throw std::invalid_argument(msg);
  if (rc == I8T_EDOMAIN) throw std::domain_error(msg);
  throw std::runtime_error("i8t: " + msg);
}
void ok(int rc) {
  if (rc != I8T_OK) throw_status(rc);
}
// synchronise + surface latched device errors (non-finite input -> domain_error)
void sync() { ok(i8t_ctx_check(ctx())); }

struct Dev {
  void* p = nullptr;
  size_t n = 0;
  explicit Dev(size_t bytes) : n(bytes) {
    if (bytes) ok(i8t_device_alloc(ctx(), bytes, &p));
  }
  Dev(const void* host, size_t bytes) : Dev(bytes) {
    if (bytes) ok(i8t_memcpy(ctx(), p, host, bytes, 0));
  }
  ~Dev() {
    if (p) i8t_device_free(ctx(), p);
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
  void to_host(void* host, size_t bytes) const {
    if (bytes) ok(i8t_memcpy(ctx(), host, p, bytes, 1));
  }
};

Dev dev_scalar(float v) { return Dev(&v, sizeof(v)); }

template <class T>
T read_scalar(const Dev& d) {
  T v{};
  d.to_host(&v, sizeof(T));
  return v;
}

i8t_conv_geom cgeom(const ConvGeometry& g) {
  return i8t_conv_geom{g.n, g.c, g.h, g.w, g.depthwise ? g.c : g.k, g.kh, g.kw, g.stride, g.stride, g.pad, g.pad,
                       g.depthwise ? 1 : 0, 0};
}

int64_t pad4(int64_t c) { return (c + 3) / 4 * 4; }
int64_t pad16(int64_t c) { return (c + 15) / 16 * 16; }

}  // namespace

// ================================================================ tensor.hpp
Shape::Shape(std::initializer_list<int64_t> dims) : Shape(std::vector<int64_t>(dims)) {}
Shape::Shape(std::vector<int64_t> dims) : d_(std::move(dims)) {
  for (int64_t v : d_)
    if (v < 1) throw std::invalid_argument("Shape: every extent must be >= 1");
}
int64_t Shape::numel() const {
  int64_t n = 1;
  for (int64_t v : d_) n *= v;
  return n;
}
int64_t Shape::flatten(std::span<const int64_t> idx) const {
  if (idx.size() != d_.size()) throw std::invalid_argument("Shape::flatten: rank mismatch");
  int64_t f = 0;
  for (size_t i = 0; i < d_.size(); ++i) {
    if (idx[i] < 0 || idx[i] >= d_[i]) throw std::out_of_range("Shape::flatten: index out of range");
    f = f * d_[i] + idx[i];
  }
  return f;
}
std::vector<int64_t> Shape::unflatten(int64_t flat) const {
  if (flat < 0 || flat >= numel()) throw std::out_of_range("Shape::unflatten: out of range");
  std::vector<int64_t> idx(d_.size());
  for (size_t i = d_.size(); i-- > 0;) {
    idx[i] = flat % d_[i];
    flat /= d_[i];
  }
  return idx;
}
std::string Shape::str() const {
  std::ostringstream os;
  os << '(';
  for (size_t i = 0; i < d_.size(); ++i) os << (i ? "," : "") << d_[i];
  os << ')';
  return os.str();
}

Tensor::Tensor(Shape shape) : shape_(std::move(shape)), v_(static_cast<size_t>(shape_.numel()), 0.0f) {}
Tensor::Tensor(Shape shape, std::vector<float> data) : shape_(std::move(shape)), v_(std::move(data)) {
  if (static_cast<int64_t>(v_.size()) != shape_.numel())
    throw std::invalid_argument("Tensor: data length does not match shape element count");
}
Tensor Tensor::full(Shape shape, float value) {
  Tensor t(std::move(shape));
  std::fill(t.v_.begin(), t.v_.end(), value);
  return t;
}
float Tensor::at4(int64_t n, int64_t c, int64_t h, int64_t w) const {
  return v_[static_cast<size_t>(((n * shape_[1] + c) * shape_[2] + h) * shape_[3] + w)];
}
float& Tensor::at4(int64_t n, int64_t c, int64_t h, int64_t w) {
  return v_[static_cast<size_t>(((n * shape_[1] + c) * shape_[2] + h) * shape_[3] + w)];
}

double sq_l2_norm(const Tensor& t) {
  if (t.numel() == 0) return 0.0;
  Dev x(t.data(), sizeof(float) * t.numel()), out(sizeof(double));
  ok(i8t_sq_l2_norm(ctx(), x.as<float>(), t.numel(), out.as<double>()));
  sync();
  return read_scalar<double>(out);
}
double l2_norm(const Tensor& t) { return std::sqrt(sq_l2_norm(t)); }
double dot(const Tensor& a, const Tensor& b) {
  if (a.numel() != b.numel()) throw std::invalid_argument("dot: size mismatch");
  if (a.numel() == 0) return 0.0;
  Dev x(a.data(), sizeof(float) * a.numel()), y(b.data(), sizeof(float) * b.numel()), out(sizeof(double));
  ok(i8t_dot(ctx(), x.as<float>(), y.as<float>(), a.numel(), out.as<double>()));
  sync();
  return read_scalar<double>(out);
}
float max_abs(const Tensor& t) {
  if (t.numel() == 0) return 0.0f;
  Dev x(t.data(), sizeof(float) * t.numel()), out(sizeof(float));
  ok(i8t_max_abs(ctx(), x.as<float>(), t.numel(), out.as<float>()));
  sync();
  return read_scalar<float>(out);
}
bool has_nonfinite(const Tensor& t) {
  if (t.numel() == 0) return false;
  Dev x(t.data(), sizeof(float) * t.numel()), out(sizeof(int32_t));
  ok(i8t_has_nonfinite(ctx(), x.as<float>(), t.numel(), out.as<int32_t>()));
  sync();
  return read_scalar<int32_t>(out) != 0;
}

// ================================================================ quantize.hpp
QuantParams QuantParams::from_clip(float c) {
  if (!(c > 0.0f) || !std::isfinite(c)) throw std::invalid_argument("QuantParams: clip must be positive and finite");
  return QuantParams{c, c / 127.0f};
}

QuantizedTensor quantize(const Tensor& x, const QuantParams& p, RoundingMode mode, LcgStream* stream) {
  if ((mode == RoundingMode::kStochastic) != (stream != nullptr))
    throw std::invalid_argument("quantize: stream required iff mode is stochastic");
  QuantizedTensor out;
  out.shape = x.shape();
  out.params = p;
  const int64_t n = x.numel();
  out.q.assign(static_cast<size_t>(n), 0);
  if (n == 0) return out;
  Dev clip = dev_scalar(p.clip);
  if (mode == RoundingMode::kNearest) {
    Dev xd(x.data(), sizeof(float) * n), qd(static_cast<size_t>(n));
    ok(i8t_quantize_nearest(ctx(), xd.as<float>(), n, clip.as<float>(), qd.as<int8_t>(), nullptr, 0));
    sync();
    qd.to_host(out.q.data(), static_cast<size_t>(n));
    return out;
  }
  // stochastic: draws in row-major order from the caller's stream (padded to 4)
  const int64_t np = (n + 3) / 4 * 4;
  std::vector<float> xp(x.values().begin(), x.values().end());
  xp.resize(static_cast<size_t>(np), 0.0f);
  Dev xd(xp.data(), sizeof(float) * np), qd(static_cast<size_t>(np));
  const uint32_t s0 = stream->state();
  Dev st(&s0, sizeof(s0));
  ok(i8t_quantize_stochastic(ctx(), xd.as<float>(), np, clip.as<float>(), st.as<uint32_t>(), qd.as<int8_t>()));
  sync();
  std::vector<int8_t> qp(static_cast<size_t>(np));
  qd.to_host(qp.data(), qp.size());
  std::copy_n(qp.begin(), n, out.q.begin());
  uint32_t s1 = 0;
  ok(i8t_lcg_jump_host(s0, static_cast<uint64_t>(n), &s1));  // exactly one draw per real element
  stream->seek(s1);
  return out;
}

int8_t quantize_value(float x, const QuantParams& p, RoundingMode mode, LcgStream* stream) {
  Tensor t(Shape{1}, {x});
  return quantize(t, p, mode, stream).q[0];
}

QuantizedTensor quantize_partitioned(const Tensor& x, const QuantParams& p, uint32_t base_seed, int partitions,
                                     int /*threads: device-parallel, result independent of it*/) {
  if (partitions < 1) throw std::invalid_argument("quantize_partitioned: partitions must be >= 1");
  QuantizedTensor out;
  out.shape = x.shape();
  out.params = p;
  const int64_t n = x.numel();
  out.q.assign(static_cast<size_t>(n), 0);
  if (n == 0) return out;
  Dev xd(x.data(), sizeof(float) * n), qd(static_cast<size_t>(n));
  Dev clip = dev_scalar(p.clip);
  ok(i8t_quantize_partitioned(ctx(), xd.as<float>(), n, clip.as<float>(), base_seed, partitions, qd.as<int8_t>()));
  sync();
  qd.to_host(out.q.data(), static_cast<size_t>(n));
  return out;
}

Tensor dequantize(const QuantizedTensor& qt) {
  Tensor out(qt.shape);
  const int64_t n = qt.numel();
  if (n == 0) return out;
  Dev qd(qt.q.data(), static_cast<size_t>(n)), od(sizeof(float) * n);
  Dev clip = dev_scalar(qt.params.clip);
  ok(i8t_dequantize(ctx(), qd.as<int8_t>(), n, clip.as<float>(), od.as<float>()));
  sync();
  od.to_host(out.data(), sizeof(float) * n);
  return out;
}

// ================================================================ gemm.hpp
Int32Matrix gemm_i8(const Int8Matrix& a, const Int8Matrix& b, int /*threads*/) {
  if (a.cols != b.rows) throw std::invalid_argument("gemm_i8: inner dimensions do not match");
  if (a.cols > kMaxGemmDepth) throw std::invalid_argument("gemm_i8: depth exceeds i32 overflow bound");
  Int32Matrix c(a.rows, b.cols);
  if (a.rows == 0 || b.cols == 0 || a.cols == 0) return c;
  Dev ad(a.data.data(), a.data.size()), bd(b.data.data(), b.data.size()), cd(sizeof(int32_t) * c.data.size());
  ok(i8t_gemm_s8(ctx(), ad.as<int8_t>(), bd.as<int8_t>(), a.rows, a.cols, b.cols, cd.as<int32_t>()));
  sync();
  cd.to_host(c.data.data(), sizeof(int32_t) * c.data.size());
  return c;
}

Int8Matrix transpose(const Int8Matrix& m) {
  Int8Matrix t(m.cols, m.rows);
  for (int64_t i = 0; i < m.rows; ++i)
    for (int64_t j = 0; j < m.cols; ++j) t.at(j, i) = m.at(i, j);
  return t;
}

// gemm_i8_fused_lhs (gemm.cpp:49-64): the lhs is quantised on the device
// straight into the GEMM's A operand (i8t_gemm_s8_fused_lhs); stochastic draws
// run in row-major order from the caller's stream, which is advanced by m*k --
// bit-identical to quantize() followed by gemm_i8().
Int32Matrix gemm_i8_fused_lhs(const Tensor& a_rowmajor, const QuantParams& pa, RoundingMode mode, LcgStream* stream,
                              const Int8Matrix& b) {
  if (a_rowmajor.shape().rank() != 2) throw std::invalid_argument("gemm_i8_fused_lhs: lhs must be 2-D");
  if ((mode == RoundingMode::kStochastic) != (stream != nullptr))
    throw std::invalid_argument("quantize: stream required iff mode is stochastic");
  const int64_t m = a_rowmajor.shape()[0], k = a_rowmajor.shape()[1];
  if (k != b.rows) throw std::invalid_argument("gemm_i8: inner dimensions do not match");
  if (k > kMaxGemmDepth) throw std::invalid_argument("gemm_i8: depth exceeds i32 overflow bound");
  Int32Matrix c(m, b.cols);
  if (m == 0 || b.cols == 0 || k == 0) return c;
  Dev ad(a_rowmajor.data(), sizeof(float) * m * k), bd(b.data.data(), b.data.size()),
      cd(sizeof(int32_t) * c.data.size());
  Dev clip = dev_scalar(pa.clip);
  const uint32_t s0 = stream ? stream->state() : 0u;
  Dev st(&s0, sizeof(s0));
  ok(i8t_gemm_s8_fused_lhs(ctx(), ad.as<float>(), m, k, clip.as<float>(), stream ? 1 : 0,
                           stream ? st.as<uint32_t>() : nullptr, bd.as<int8_t>(), b.cols, cd.as<int32_t>()));
  sync();
  cd.to_host(c.data.data(), sizeof(int32_t) * c.data.size());
  if (stream) stream->seek(read_scalar<uint32_t>(st));
  return c;
}

// ================================================================ conv.hpp
void ConvGeometry::validate() const {
  if (n < 1 || c < 1 || h < 1 || w < 1 || k < 1 || kh < 1 || kw < 1 || stride < 1 || pad < 0)
    throw std::invalid_argument("ConvGeometry: extents must be positive, pad nonnegative");
  if (depthwise && k != c) throw std::invalid_argument("ConvGeometry: depthwise requires k == c");
  if ((h + 2 * pad - kh) % stride != 0 || (w + 2 * pad - kw) % stride != 0 || h + 2 * pad < kh || w + 2 * pad < kw)
    throw std::invalid_argument("ConvGeometry: output size is not a positive integer");
}

namespace {
void check_conv_operands(const QuantizedTensor& a, const QuantizedTensor& w, const ConvGeometry& g) {
  g.validate();
  if (!(a.shape == g.input_shape())) throw std::invalid_argument("conv2d_q: activation shape mismatch");
  if (!(w.shape == g.weight_shape())) throw std::invalid_argument("conv2d_q: weight shape mismatch");
}
void check_depth(int64_t d) {
  if (d > kMaxGemmDepth) throw std::invalid_argument("conv: reduction depth exceeds i32 overflow bound");
}

// NCHW int8 (host) -> NHWC int8 (device, channel stride c_pad)
std::unique_ptr<Dev> to_nhwc(const std::vector<int8_t>& q, int64_t n, int64_t c, int64_t hw, int64_t c_pad) {
  Dev src(q.data(), q.size());
  auto dst = std::make_unique<Dev>(static_cast<size_t>(n * hw * c_pad));
  ok(i8t_nchw_to_nhwc_i8(ctx(), src.as<int8_t>(), n, c, hw, dst->as<int8_t>(), c_pad));
  sync();
  return dst;
}
}  // namespace

// im2col (conv.cpp:23-47, 98-106) on the device: host buffers in and out, as
// the reference's raw-pointer signature requires.
static void im2col_device(const int8_t* x, const ConvGeometry& g, int64_t c_lo, int64_t c_hi, int8_t* out) {
  g.validate();
  if (c_lo < 0 || c_hi > g.c) throw std::invalid_argument("im2col_channel_i8: channel out of range");
  const int64_t in_bytes = g.n * g.c * g.h * g.w, rows = (c_hi - c_lo) * g.kh * g.kw;
  const int64_t out_bytes = rows * g.n * g.out_h() * g.out_w();
  Dev xd(x, static_cast<size_t>(in_bytes)), od(static_cast<size_t>(out_bytes));
  const i8t_conv_geom cg = cgeom(g);
  ok(i8t_im2col_s8(ctx(), xd.as<int8_t>(), &cg, c_lo, c_hi, od.as<int8_t>()));
  sync();
  od.to_host(out, static_cast<size_t>(out_bytes));
}
void im2col_i8(const int8_t* x, const ConvGeometry& g, int8_t* out) { im2col_device(x, g, 0, g.c, out); }
void im2col_channel_i8(const int8_t* x, const ConvGeometry& g, int64_t channel, int8_t* out) {
  im2col_device(x, g, channel, channel + 1, out);
}

Tensor conv2d_q(const QuantizedTensor& a, const QuantizedTensor& w, const ConvGeometry& g, int /*threads*/) {
  check_conv_operands(a, w, g);
  check_depth(g.depthwise ? g.kh * g.kw : g.c * g.kh * g.kw);
  const int64_t oh = g.out_h(), ow = g.out_w(), kout = g.depthwise ? g.c : g.k, m = g.out_positions();
  const i8t_conv_geom cg = cgeom(g);
  Dev ca = dev_scalar(a.params.clip), cw = dev_scalar(w.params.clip);
  Dev z(sizeof(float) * m * kout), zc(sizeof(float) * m * kout);
  if (g.depthwise) {
    auto an = to_nhwc(a.q, g.n, g.c, g.h * g.w, g.c);
    Dev wd(w.q.data(), w.q.size());
    ok(i8t_conv_dw_fwd(ctx(), &cg, an->as<int8_t>(), g.c, wd.as<int8_t>(), ca.as<float>(), cw.as<float>(), z.as<float>(),
                       nullptr));
  } else {
    const int64_t cp = pad4(g.c), ld = pad16(g.kh * g.kw * cp);
    auto an = to_nhwc(a.q, g.n, g.c, g.h * g.w, cp);
    Dev wsrc(w.q.data(), w.q.size()), wk(static_cast<size_t>(g.k * ld));
    ok(i8t_kcrs_to_krsc_i8(ctx(), wsrc.as<int8_t>(), g.k, g.c, g.kh, g.kw, wk.as<int8_t>(), cp, ld));
    ok(i8t_conv_fwd(ctx(), &cg, an->as<int8_t>(), cp, wk.as<int8_t>(), ld, ca.as<float>(), cw.as<float>(), z.as<float>(),
                    nullptr));
  }
  ok(i8t_nhwc_to_nchw_f32(ctx(), z.as<float>(), g.n, kout, oh * ow, kout, zc.as<float>()));
  sync();
  Tensor out(g.output_shape());
  zc.to_host(out.data(), sizeof(float) * out.numel());
  return out;
}

std::pair<Tensor, Tensor> conv2d_backward_q(const QuantizedTensor& g_z, const QuantizedTensor& a,
                                            const QuantizedTensor& w, const ConvGeometry& g, int /*threads*/) {
  check_conv_operands(a, w, g);
  if (!(g_z.shape == g.output_shape())) throw std::invalid_argument("conv2d_backward_q: g_z shape mismatch");
  const int64_t m = g.out_positions(), hw = g.h * g.w, ohw = g.out_h() * g.out_w();
  check_depth(m);
  if (!g.depthwise) check_depth(g.k);
  const i8t_conv_geom cg = cgeom(g);
  Dev cgz = dev_scalar(g_z.params.clip), ca = dev_scalar(a.params.clip), cw = dev_scalar(w.params.clip);
  Tensor grad_w(g.weight_shape()), grad_a(g.input_shape());
  Dev ga(sizeof(float) * g.n * hw * g.c), gac(sizeof(float) * g.n * hw * g.c), gw(sizeof(float) * grad_w.numel());
  if (g.depthwise) {
    auto gn = to_nhwc(g_z.q, g.n, g.c, ohw, g.c);
    auto an = to_nhwc(a.q, g.n, g.c, hw, g.c);
    Dev wd(w.q.data(), w.q.size()), acc(sizeof(int64_t) * g.c * g.kh * g.kw);
    ok(i8t_conv_dw_dgrad(ctx(), &cg, gn->as<int8_t>(), g.c, wd.as<int8_t>(), cgz.as<float>(), cw.as<float>(),
                         ga.as<float>(), nullptr));
    ok(i8t_conv_dw_wgrad(ctx(), &cg, gn->as<int8_t>(), an->as<int8_t>(), g.c, cgz.as<float>(), ca.as<float>(),
                         acc.as<int64_t>(), gw.as<float>()));
  } else {
    const int64_t cp = pad4(g.c), kp = pad4(g.k), ldt = pad16(g.kh * g.kw * kp);
    auto gn = to_nhwc(g_z.q, g.n, g.k, ohw, kp);
    auto an = to_nhwc(a.q, g.n, g.c, hw, cp);
    Dev wsrc(w.q.data(), w.q.size()), wt(static_cast<size_t>(g.c * ldt));
    Dev acc(sizeof(int64_t) * g.kh * g.kw * cp * g.k);
    ok(i8t_kcrs_to_crsk_i8(ctx(), wsrc.as<int8_t>(), g.k, g.c, g.kh, g.kw, wt.as<int8_t>(), kp, ldt));
    ok(i8t_conv_dgrad(ctx(), &cg, gn->as<int8_t>(), kp, wt.as<int8_t>(), ldt, cgz.as<float>(), cw.as<float>(),
                      ga.as<float>(), nullptr));
    ok(i8t_conv_wgrad(ctx(), &cg, gn->as<int8_t>(), kp, an->as<int8_t>(), cp, cgz.as<float>(), ca.as<float>(),
                      acc.as<int64_t>(), gw.as<float>(), 1));
  }
  ok(i8t_nhwc_to_nchw_f32(ctx(), ga.as<float>(), g.n, g.c, hw, g.c, gac.as<float>()));
  sync();
  gac.to_host(grad_a.data(), sizeof(float) * grad_a.numel());
  gw.to_host(grad_w.data(), sizeof(float) * grad_w.numel());
  return {std::move(grad_w), std::move(grad_a)};
}

// ================================================================ clip.hpp
double cosine_distance(const Tensor& g, const Tensor& g_hat) {
  if (!(g.shape() == g_hat.shape())) throw std::invalid_argument("cosine_distance: shape mismatch");
  if (g.numel() == 0) return 0.0;
  Dev a(g.data(), sizeof(float) * g.numel()), b(g_hat.data(), sizeof(float) * g.numel()), out(sizeof(double));
  ok(i8t_cosine_distance(ctx(), a.as<float>(), b.as<float>(), g.numel(), out.as<double>()));
  sync();
  return read_scalar<double>(out);
}

double measure_dc(const Tensor& g, float clip) {
  QuantParams::from_clip(clip);  // same validation / exception as the reference
  Dev a(g.data(), sizeof(float) * g.numel()), out(sizeof(double));
  ok(i8t_measure_dc(ctx(), a.as<float>(), g.numel(), clip, out.as<double>()));
  sync();
  return read_scalar<double>(out);
}

ClipSearchResult search_clip(const Tensor& g, const ClipSearchConfig& cfg, float prev_clip) {
  if (cfg.grid_resolution < 8) throw std::invalid_argument("search_clip: grid resolution must be >= 8");
  Dev a(g.data(), sizeof(float) * g.numel()), c(sizeof(float)), d(sizeof(double));
  ok(i8t_search_clip(ctx(), a.as<float>(), g.numel(), cfg.grid_resolution, cfg.refine_rounds, prev_clip, c.as<float>(),
                     d.as<double>()));
  sync();  // a non-finite g with max_abs != 0 throws std::domain_error here (clip.cpp:34)
  return ClipSearchResult{read_scalar<float>(c), read_scalar<double>(d)};
}

void maybe_update(ClipState& state, const Tensor& g, int64_t iter, const ClipSearchConfig& cfg) {
  if (iter < state.iter_of_last_update) throw std::invalid_argument("maybe_update: iter went backwards");
  if (cfg.grid_resolution < 8) throw std::invalid_argument("search_clip: grid resolution must be >= 8");
  const bool uninitialized = !(state.clip > 0.0f);
  const bool due = uninitialized || state.iter_of_last_update < 0 || (iter - state.iter_of_last_update) >= state.period;
  Dev st(static_cast<size_t>(i8t_dsgc_state_size()));
  ok(i8t_dsgc_init(ctx(), st.p, state.period));
  i8t_dsgc_view v{};
  ok(i8t_dsgc_read(ctx(), st.p, &v));
  v.clip = state.clip;
  v.last_dc = state.last_dc;
  v.iter_of_last_update = state.iter_of_last_update;
  v.period = state.period;
  ok(i8t_dsgc_write(ctx(), st.p, &v));
  Dev a(g.data(), sizeof(float) * g.numel());
  ok(i8t_maybe_update(ctx(), st.p, a.as<float>(), g.numel(), iter, cfg.grid_resolution, cfg.refine_rounds, due ? 1 : 0));
  sync();
  ok(i8t_dsgc_read(ctx(), st.p, &v));
  state.clip = v.clip;
  state.last_dc = v.last_dc;
  state.iter_of_last_update = v.iter_of_last_update;
}

// ================================================================ lr_scale.hpp
double scale_factor(double dc, const LrScaleConfig& cfg) {
  double out = 0.0;
  ok(i8t_scale_factor(dc, cfg.alpha, cfg.beta, static_cast<int>(cfg.form), &out));
  return out;
}

std::map<std::string, double> effective_lr(double base_lr, const std::map<std::string, double>& dc_per_layer,
                                           const LrScaleConfig& cfg) {
  if (!(base_lr > 0.0)) throw std::invalid_argument("effective_lr: base_lr must be > 0");
  std::map<std::string, double> out;
  for (const auto& [layer, dc] : dc_per_layer) out[layer] = base_lr * scale_factor(dc, cfg);
  return out;
}

}  // namespace i8t
