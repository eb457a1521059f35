// test_shim.cpp -- the reference's unit-test known answers, compiled against
// the drop-in header (include/i8t/*.hpp) and linked to libi8t.so, i.e. the way
// a reference user would switch libraries.  Exit code = number of failures.
// Built by __graft_entry__.build(); run on a B200 by tests/test_gpu_shim.py.
#include <cmath>
#include <cstdio>
#include <functional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "i8t/clip.hpp"
#include "i8t/conv.hpp"
#include "i8t/gemm.hpp"
#include "i8t/lr_scale.hpp"
#include "i8t/quantize.hpp"
#include "i8t/tensor.hpp"

using namespace i8t;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                     \
  do {                                                                  \
    ++g_checks;                                                         \
    if (!(cond)) {                                                      \
      ++g_fail;                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);       \
    }                                                                   \
  } while (0)
template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

// SplitMix64 for deterministic inputs (test-side only)
struct Rng {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  int8_t i8() { return static_cast<int8_t>(static_cast<int64_t>(next() % 255) - 127); }
};

static void test_quantize() {
  LcgStream s(0);
  CHECK(s.next_state() == 1013904223u);
  QuantParams p = QuantParams::from_clip(127.0f);
  CHECK(p.scale == 1.0f);
  CHECK(quantize(Tensor({1}, {200.0f}), p, RoundingMode::kNearest).q[0] == 127);
  CHECK(quantize(Tensor({1}, {-200.0f}), p, RoundingMode::kNearest).q[0] == -127);
  // 3.4 -> {3, 4} at rate 0.4 for 4 (one tensor of n copies == n single draws in order)
  const int n = 100000;
  LcgStream st(2024);
  auto q = quantize(Tensor::full(Shape{n}, 3.4f), p, RoundingMode::kStochastic, &st);
  double sum = 0;
  bool only34 = true;
  for (int8_t v : q.q) {
    sum += v;
    only34 = only34 && (v == 3 || v == 4);
  }
  CHECK(only34);
  CHECK(std::fabs(sum / n - 3.4) < 3.0 * std::sqrt(0.24) / std::sqrt(double(n)));
  // one draw per element, unconditionally
  LcgStream a(31337), ref(31337);
  quantize(Tensor::full(Shape{257}, 0.25f), QuantParams::from_clip(1.0f), RoundingMode::kStochastic, &a);
  for (int i = 0; i < 257; ++i) ref.next_state();
  CHECK(a.state() == ref.state());
  CHECK(throws<std::domain_error>([] {
    quantize(Tensor({1}, {std::nanf("")}), QuantParams::from_clip(1.0f), RoundingMode::kNearest);
  }));
  CHECK(throws<std::invalid_argument>([] { QuantParams::from_clip(0.0f); }));
  CHECK(throws<std::invalid_argument>([] {
    quantize(Tensor({1}, {0.5f}), QuantParams::from_clip(1.0f), RoundingMode::kStochastic, nullptr);
  }));
  QuantizedTensor qt;
  qt.shape = Shape{2};
  qt.q = {127, 0};
  qt.params = QuantParams::from_clip(1.27f);
  Tensor d = dequantize(qt);
  CHECK(std::fabs(d[0] - 1.27f) < 1e-6f && d[1] == 0.0f);
  // partitioned: chunk 0 draws from LcgStream(base)
  Tensor t(Shape{1000});
  Rng r{3};
  for (int64_t i = 0; i < t.numel(); ++i) t[i] = static_cast<float>(r.uniform() * 2 - 1);
  QuantParams pt = QuantParams::from_clip(max_abs(t));
  auto part = quantize_partitioned(t, pt, 900, 8, 4);
  LcgStream s0(900);
  CHECK(part.q[0] == quantize_value(t[0], pt, RoundingMode::kStochastic, &s0));
}

static void test_gemm_conv() {
  Int8Matrix a(2, 2), b(2, 2);
  a.data = {1, 2, 3, 4};
  b.data = {5, 6, 7, 8};
  CHECK(gemm_i8(a, b).data == (std::vector<int32_t>{19, 22, 43, 50}));
  Int8Matrix row(1, 4), col(4, 1);
  row.data = {127, 127, 127, 127};
  col.data = {127, 127, 127, 127};
  CHECK(gemm_i8(row, col).data[0] == 64516);
  CHECK(throws<std::invalid_argument>([] { gemm_i8(Int8Matrix(2, 3), Int8Matrix(2, 2)); }));
  // conv == direct convolution on random small geometries (test_kernels.cpp:163-200)
  Rng r{101};
  for (int t = 0; t < 12; ++t) {
    ConvGeometry g;
    g.n = 1 + r.next() % 2;
    g.c = 1 + r.next() % 4;
    g.kh = g.kw = 1 + r.next() % 3;
    g.stride = 1 + r.next() % 2;
    g.pad = r.next() % 2;
    g.depthwise = (t % 4 == 3);
    g.k = g.depthwise ? g.c : 1 + r.next() % 4;
    const int64_t oh = 1 + r.next() % 4, ow = 1 + r.next() % 4;
    g.h = (oh - 1) * g.stride + g.kh - 2 * g.pad;
    if (g.h < 1) g.h = g.kh;
    g.w = (ow - 1) * g.stride + g.kw - 2 * g.pad;
    if (g.w < 1) g.w = g.kw;
    try {
      g.validate();
    } catch (...) {
      continue;
    }
    QuantizedTensor qa, qw;
    qa.shape = g.input_shape();
    qw.shape = g.weight_shape();
    qa.q.resize(qa.shape.numel());
    qw.q.resize(qw.shape.numel());
    for (auto& v : qa.q) v = r.i8();
    for (auto& v : qw.q) v = r.i8();
    qa.params = QuantParams::from_clip(1.27f);
    qw.params = QuantParams::from_clip(12.7f);
    Tensor z = conv2d_q(qa, qw, g);
    const double rs = double(qa.params.scale) * double(qw.params.scale);
    const int64_t kout = g.depthwise ? g.c : g.k;
    bool same = true;
    for (int64_t n = 0; n < g.n; ++n)
      for (int64_t ko = 0; ko < kout; ++ko)
        for (int64_t i = 0; i < g.out_h(); ++i)
          for (int64_t j = 0; j < g.out_w(); ++j) {
            int64_t acc = 0;
            const int64_t c0 = g.depthwise ? ko : 0, c1 = g.depthwise ? ko + 1 : g.c;
            for (int64_t c = c0; c < c1; ++c)
              for (int64_t ki = 0; ki < g.kh; ++ki)
                for (int64_t kj = 0; kj < g.kw; ++kj) {
                  const int64_t ih = i * g.stride + ki - g.pad, iw = j * g.stride + kj - g.pad;
                  if (ih < 0 || ih >= g.h || iw < 0 || iw >= g.w) continue;
                  const int64_t widx = ((ko * (g.depthwise ? 1 : g.c) + (g.depthwise ? 0 : c)) * g.kh + ki) * g.kw + kj;
                  acc += int64_t(qa.q[((n * g.c + c) * g.h + ih) * g.w + iw]) * int64_t(qw.q[widx]);
                }
            same = same && z.at4(n, ko, i, j) == static_cast<float>(rs * double(acc));
          }
    CHECK(same);
  }
  // backward 1x1: exact matrix calculus (test_kernels.cpp:271-300)
  ConvGeometry g{.n = 1, .c = 3, .h = 2, .w = 2, .k = 4, .kh = 1, .kw = 1};
  QuantizedTensor qa, qw, qg;
  qa.shape = g.input_shape();
  qw.shape = g.weight_shape();
  qg.shape = g.output_shape();
  for (auto* q : {&qa, &qw, &qg}) {
    q->q.resize(q->shape.numel());
    for (auto& v : q->q) v = r.i8();
    q->params = QuantParams::from_clip(1.27f);
  }
  auto [gw, ga] = conv2d_backward_q(qg, qa, qw, g);
  const double rw = double(qg.params.scale) * double(qa.params.scale);
  bool ok = true;
  for (int64_t k = 0; k < 4; ++k)
    for (int64_t c = 0; c < 3; ++c) {
      int64_t acc = 0;
      for (int64_t p = 0; p < 4; ++p) acc += int64_t(qg.q[k * 4 + p]) * int64_t(qa.q[c * 4 + p]);
      ok = ok && gw[k * 3 + c] == static_cast<float>(rw * double(acc));
    }
  for (int64_t c = 0; c < 3; ++c)
    for (int64_t p = 0; p < 4; ++p) {
      int64_t acc = 0;
      for (int64_t k = 0; k < 4; ++k) acc += int64_t(qw.q[k * 3 + c]) * int64_t(qg.q[k * 4 + p]);
      ok = ok && ga[c * 4 + p] == static_cast<float>(rw * double(acc));
    }
  CHECK(ok);
  ConvGeometry bad{.n = 1, .c = 1, .h = 4, .w = 4, .k = 1, .kh = 3, .kw = 3, .stride = 2, .pad = 0};
  CHECK(throws<std::invalid_argument>([&] { bad.validate(); }));
}

// fused quantize-GEMM == unfused composition bit-exactly, incl. the stream
// (test_kernels.cpp:120-142); a ragged m*k (not a multiple of 4) as well
static void test_fused_lhs() {
  Rng r{31};
  for (auto [m, k, n] : {std::tuple<int64_t, int64_t, int64_t>{9, 40, 13}, {7, 41, 5}, {130, 300, 70}}) {
    Tensor a(Shape{m, k});
    for (int64_t i = 0; i < a.numel(); ++i) a[i] = static_cast<float>(2.0 * r.uniform() - 1.0) * 3.0f;
    Int8Matrix b(k, n);
    for (auto& v : b.data) v = r.i8();
    QuantParams pa = QuantParams::from_clip(max_abs(a));
    LcgStream s1(555), s2(555);
    auto q = quantize(a, pa, RoundingMode::kStochastic, &s1);
    Int8Matrix qa(m, k);
    qa.data = q.q;
    auto unfused = gemm_i8(qa, b);
    auto fused = gemm_i8_fused_lhs(a, pa, RoundingMode::kStochastic, &s2, b);
    CHECK(unfused.data == fused.data);
    CHECK(s1.state() == s2.state());
    auto fused_nearest = gemm_i8_fused_lhs(a, pa, RoundingMode::kNearest, nullptr, b);
    Int8Matrix qn(m, k);
    qn.data = quantize(a, pa, RoundingMode::kNearest).q;
    CHECK(fused_nearest.data == gemm_i8(qn, b).data);
  }
  CHECK(throws<std::invalid_argument>([] {
    LcgStream s(1);
    gemm_i8_fused_lhs(Tensor(Shape{2, 3}), QuantParams::from_clip(1.0f), RoundingMode::kNearest, &s, Int8Matrix(3, 1));
  }));
  Tensor bad(Shape{1, 4}, {1.0f, NAN, 0.0f, 2.0f});
  CHECK(throws<std::domain_error>([&] {
    gemm_i8_fused_lhs(bad, QuantParams::from_clip(1.0f), RoundingMode::kNearest, nullptr, Int8Matrix(4, 2));
  }));
}

// im2col known layouts (test_kernels.cpp:144-161) + a padded strided case vs a direct gather
static void test_im2col() {
  ConvGeometry g{.n = 1, .c = 1, .h = 3, .w = 3, .k = 1, .kh = 2, .kw = 2};
  std::vector<int8_t> x = {1, 2, 3, 4, 5, 6, 7, 8, 9};
  std::vector<int8_t> col(4 * 4);
  im2col_i8(x.data(), g, col.data());
  CHECK(col[0 * 4 + 0] == 1);
  CHECK(col[1 * 4 + 0] == 2);
  CHECK(col[2 * 4 + 0] == 4);
  CHECK(col[3 * 4 + 0] == 5);
  ConvGeometry g2{.n = 1, .c = 1, .h = 3, .w = 3, .k = 1, .kh = 3, .kw = 3};
  std::vector<int8_t> col2(9);
  im2col_i8(x.data(), g2, col2.data());
  CHECK(col2 == x);
  Rng r{7};
  ConvGeometry g3{.n = 2, .c = 3, .h = 7, .w = 7, .k = 4, .kh = 3, .kw = 3, .stride = 2, .pad = 1};
  std::vector<int8_t> x3(2 * 3 * 7 * 7);
  for (auto& v : x3) v = r.i8();
  const int64_t oh = g3.out_h(), ow = g3.out_w(), cols = g3.n * oh * ow;
  std::vector<int8_t> c3(static_cast<size_t>(3 * 9 * cols)), ch1(static_cast<size_t>(9 * cols));
  im2col_i8(x3.data(), g3, c3.data());
  im2col_channel_i8(x3.data(), g3, 1, ch1.data());
  bool same = true;
  for (int64_t c = 0; c < 3; ++c)
    for (int64_t i = 0; i < 3; ++i)
      for (int64_t j = 0; j < 3; ++j)
        for (int64_t n = 0; n < 2; ++n)
          for (int64_t p = 0; p < oh; ++p)
            for (int64_t q = 0; q < ow; ++q) {
              const int64_t y = p * 2 + i - 1, xx = q * 2 + j - 1, row = (c * 3 + i) * 3 + j;
              const int8_t want = (y >= 0 && y < 7 && xx >= 0 && xx < 7) ? x3[((n * 3 + c) * 7 + y) * 7 + xx] : 0;
              const int64_t m = (n * oh + p) * ow + q;
              same = same && c3[row * cols + m] == want;
              if (c == 1) same = same && ch1[(i * 3 + j) * cols + m] == want;
            }
  CHECK(same);
}

static void test_clip_lr() {
  CHECK(std::fabs(cosine_distance(Tensor({3}, {0.5f, -1.0f, 2.0f}), Tensor({3}, {0.5f, -1.0f, 2.0f}))) < 1e-12);
  CHECK(cosine_distance(Tensor({2}, {1, 0}), Tensor({2}, {0, 0})) == 1.0);
  Tensor g(Shape{255});
  for (int i = -127; i <= 127; ++i) g[i + 127] = 0.01f * static_cast<float>(i);
  auto r = search_clip(g, ClipSearchConfig{});
  CHECK(r.clip == max_abs(g));
  CHECK(std::fabs(r.dc) < 1e-12);
  CHECK(throws<std::invalid_argument>([&] { search_clip(g, ClipSearchConfig{.grid_resolution = 4, .refine_rounds = 0}); }));
  ClipState st{.layer_id = "l", .period = 100};
  maybe_update(st, g, 0, ClipSearchConfig{});
  CHECK(st.iter_of_last_update == 0 && st.clip > 0.0f);
  const float c0 = st.clip;
  maybe_update(st, g, 1, ClipSearchConfig{});
  CHECK(st.clip == c0 && st.iter_of_last_update == 0);
  ClipState st5{.layer_id = "l", .period = 1};
  maybe_update(st5, g, 5, ClipSearchConfig{});
  CHECK(throws<std::invalid_argument>([&] { maybe_update(st5, g, 4, ClipSearchConfig{}); }));
  LrScaleConfig cfg;
  CHECK(scale_factor(0.0, cfg) == 1.0);
  CHECK(std::fabs(scale_factor(0.05, cfg) - std::exp(-1.0)) < 1e-12);
  CHECK(scale_factor(1.0, cfg) == 0.1);
  CHECK(throws<std::invalid_argument>([&] { scale_factor(2.5, cfg); }));
  auto lr = effective_lr(0.1, {{"a", 0.0}, {"b", 2.0}}, cfg);
  CHECK(lr["a"] == 0.1 && std::fabs(lr["b"] - 0.01) < 1e-12);
}

int main() {
  std::vector<std::pair<const char*, std::function<void()>>> suites = {
      {"quantize", test_quantize}, {"gemm_conv", test_gemm_conv}, {"fused_lhs", test_fused_lhs},
      {"im2col", test_im2col},     {"clip_lr", test_clip_lr}};
  for (auto& [name, fn] : suites) {
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("FAIL suite %s threw: %s\n", name, e.what());
    }
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail;
}
