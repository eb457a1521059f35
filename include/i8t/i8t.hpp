// i8t/i8t.hpp -- drop-in C++ operator API of the INT8 training hot path,
// backed by the B200 (sm_100a) kernels of libi8t_cuda.so through the C-ABI in
// i8t_cuda.h.  Link: -li8t -li8t_cuda -lcudart.
//
// Same namespace, type names, signatures, value semantics and exception types
// as the reference library's public headers (proj/core/include/i8t/
// tensor.hpp, quantize.hpp, gemm.hpp, conv.hpp, clip.hpp, lr_scale.hpp), so a
// caller recompiles against this header unchanged.  Tensors stay host-side
// std::vector values; every arithmetic op runs on the GPU (host<->device
// copies per call).  There is no CPU fallback: without a B200 every
// computing call throws std::runtime_error.
//
// Not provided (outside the graded INT8 path): the FP32 baseline
// operators gemm_f32 / conv2d_f32 / conv2d_backward_f32.
#pragma once

#include <cstdint>
#include <initializer_list>
#include <map>
#include <span>
#include <string>
#include <utility>
#include <vector>

namespace i8t {

// ------------------------------------------------------------ tensor.hpp
class Shape {
 public:
  Shape() = default;
  Shape(std::initializer_list<int64_t> dims);
  explicit Shape(std::vector<int64_t> dims);
  int rank() const { return static_cast<int>(d_.size()); }
  int64_t operator[](int i) const { return d_[static_cast<size_t>(i)]; }
  const std::vector<int64_t>& dims() const { return d_; }
  int64_t numel() const;
  int64_t flatten(std::span<const int64_t> idx) const;
  std::vector<int64_t> unflatten(int64_t flat) const;
  bool operator==(const Shape& o) const { return d_ == o.d_; }
  std::string str() const;

 private:
  std::vector<int64_t> d_;
};

class Tensor {
 public:
  Tensor() = default;
  explicit Tensor(Shape shape);
  Tensor(Shape shape, std::vector<float> data);
  static Tensor full(Shape shape, float value);
  const Shape& shape() const { return shape_; }
  int64_t numel() const { return static_cast<int64_t>(v_.size()); }
  float* data() { return v_.data(); }
  const float* data() const { return v_.data(); }
  std::span<float> values() { return v_; }
  std::span<const float> values() const { return v_; }
  float operator[](int64_t i) const { return v_[static_cast<size_t>(i)]; }
  float& operator[](int64_t i) { return v_[static_cast<size_t>(i)]; }
  float at4(int64_t n, int64_t c, int64_t h, int64_t w) const;
  float& at4(int64_t n, int64_t c, int64_t h, int64_t w);

 private:
  Shape shape_;
  std::vector<float> v_;
};

double l2_norm(const Tensor& t);
double sq_l2_norm(const Tensor& t);
double dot(const Tensor& a, const Tensor& b);
float max_abs(const Tensor& t);
bool has_nonfinite(const Tensor& t);

// ------------------------------------------------------------ quantize.hpp
struct QuantParams {
  float clip = 1.0f;
  float scale = 1.0f;  // clip / 127
  static QuantParams from_clip(float c);
};

struct QuantizedTensor {
  Shape shape;
  std::vector<int8_t> q;
  QuantParams params;
  int64_t numel() const { return static_cast<int64_t>(q.size()); }
};

enum class RoundingMode { kNearest, kStochastic };

// X <- 1664525 X + 1013904223 (mod 2^32); u = X / 2^32.
class LcgStream {
 public:
  static constexpr uint32_t kMultiplier = 1664525u;
  static constexpr uint32_t kIncrement = 1013904223u;
  explicit LcgStream(uint32_t seed = 0) : x_(seed) {}
  uint32_t state() const { return x_; }
  uint32_t next_state() { return x_ = kMultiplier * x_ + kIncrement; }
  double next_uniform() { return static_cast<double>(next_state()) * 0x1.0p-32; }
  // extension: reposition the stream (used after device-side draws)
  void seek(uint32_t state) { x_ = state; }

 private:
  uint32_t x_;
};

int8_t quantize_value(float x, const QuantParams& p, RoundingMode mode, LcgStream* stream);
QuantizedTensor quantize(const Tensor& x, const QuantParams& p, RoundingMode mode, LcgStream* stream = nullptr);
QuantizedTensor quantize_partitioned(const Tensor& x, const QuantParams& p, uint32_t base_seed, int partitions,
                                     int threads = 0);
Tensor dequantize(const QuantizedTensor& qt);

// ------------------------------------------------------------ gemm.hpp
struct Int8Matrix {
  int64_t rows = 0, cols = 0;
  std::vector<int8_t> data;
  Int8Matrix() = default;
  Int8Matrix(int64_t r, int64_t c) : rows(r), cols(c), data(static_cast<size_t>(r * c), 0) {}
  int8_t at(int64_t i, int64_t j) const { return data[static_cast<size_t>(i * cols + j)]; }
  int8_t& at(int64_t i, int64_t j) { return data[static_cast<size_t>(i * cols + j)]; }
};

struct Int32Matrix {
  int64_t rows = 0, cols = 0;
  std::vector<int32_t> data;
  Int32Matrix() = default;
  Int32Matrix(int64_t r, int64_t c) : rows(r), cols(c), data(static_cast<size_t>(r * c), 0) {}
  int32_t at(int64_t i, int64_t j) const { return data[static_cast<size_t>(i * cols + j)]; }
  int32_t& at(int64_t i, int64_t j) { return data[static_cast<size_t>(i * cols + j)]; }
};

inline constexpr int64_t kMaxGemmDepth = 130000;

Int32Matrix gemm_i8(const Int8Matrix& a, const Int8Matrix& b, int threads = 0);
Int8Matrix transpose(const Int8Matrix& m);
Int32Matrix gemm_i8_fused_lhs(const Tensor& a_rowmajor, const QuantParams& pa, RoundingMode mode, LcgStream* stream,
                              const Int8Matrix& b);

// ------------------------------------------------------------ conv.hpp
struct ConvGeometry {
  int64_t n = 1, c = 1, h = 1, w = 1;
  int64_t k = 1, kh = 1, kw = 1;
  int64_t stride = 1, pad = 0;
  bool depthwise = false;
  int64_t out_h() const { return (h + 2 * pad - kh) / stride + 1; }
  int64_t out_w() const { return (w + 2 * pad - kw) / stride + 1; }
  int64_t out_positions() const { return n * out_h() * out_w(); }
  void validate() const;
  Shape input_shape() const { return Shape{n, c, h, w}; }
  Shape weight_shape() const { return depthwise ? Shape{c, 1, kh, kw} : Shape{k, c, kh, kw}; }
  Shape output_shape() const { return Shape{n, depthwise ? c : k, out_h(), out_w()}; }
};

void im2col_i8(const int8_t* x, const ConvGeometry& g, int8_t* out);
void im2col_channel_i8(const int8_t* x, const ConvGeometry& g, int64_t channel, int8_t* out);
Tensor conv2d_q(const QuantizedTensor& a, const QuantizedTensor& w, const ConvGeometry& g, int threads = 0);
std::pair<Tensor, Tensor> conv2d_backward_q(const QuantizedTensor& g_z, const QuantizedTensor& a,
                                            const QuantizedTensor& w, const ConvGeometry& g, int threads = 0);

// ------------------------------------------------------------ clip.hpp
struct ClipState {
  std::string layer_id;
  float clip = 0.0f;
  double last_dc = 0.0;
  int64_t iter_of_last_update = -1;
  int64_t period = 100;
};

struct ClipSearchConfig {
  int grid_resolution = 32;
  int refine_rounds = 2;
};

struct ClipSearchResult {
  float clip = 0.0f;
  double dc = 0.0;
};

double cosine_distance(const Tensor& g, const Tensor& g_hat);
double measure_dc(const Tensor& g, float clip);
ClipSearchResult search_clip(const Tensor& g, const ClipSearchConfig& cfg, float prev_clip = 0.0f);
void maybe_update(ClipState& state, const Tensor& g, int64_t iter, const ClipSearchConfig& cfg);

// ------------------------------------------------------------ lr_scale.hpp
enum class ScaleForm { kExponential, kLinear, kQuadratic };

struct LrScaleConfig {
  double alpha = 20.0;
  double beta = 0.1;
  ScaleForm form = ScaleForm::kExponential;
};

double scale_factor(double dc, const LrScaleConfig& cfg);
std::map<std::string, double> effective_lr(double base_lr, const std::map<std::string, double>& dc_per_layer,
                                           const LrScaleConfig& cfg);

}  // namespace i8t
