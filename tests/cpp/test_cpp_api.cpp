// C++ drop-in API test (include/xbarsim/layers.hpp over the C ABI), written
// the way the reference's doctest cases use the API (reference
// proj/tests/unit/test_nn.cpp): CrossbarLinear, lin.core()->gradient(),
// lin.core()->weights().implied_weights(), exception types.
//
//   test_cpp_api cpu   validation errors only (no GPU needed)
//   test_cpp_api gpu   bit-exact parity against the CPU oracle (test
//                      infrastructure, linked here only as the checker)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>

#include "xbarsim/layers.hpp"

extern "C" {  // oracle/xbs_oracle_capi.cpp (orc_options has xbs_layer_options' layout)
int orc_core_create(const void* o, int snapped, const double* W, long K, long N, void** out);
void orc_core_destroy(void* h);
int orc_core_forward(void* h, const double* x, long M, long K, int training, double* y);
int orc_core_backward(void* h, const double* dy, long M, long N, double gd, double* dx);
int orc_core_gradient(void* h, double* out);
int orc_core_set_nonideal(void* h, int s, int p, int t, const double* g);
int orc_core_master(void* h, int s, double* u);
int orc_core_apply_updates(void* h, uint64_t it);
int orc_conv2d_create(const void* o, int snapped, const double* W, long K, long N, int in_c, int out_c, int k,
                      int stride, int pad, void** out);
void orc_conv2d_destroy(void* h);
int orc_conv2d_forward(void* h, const double* x, long batch, int c, int hh, int ww, int training, double* y,
                       int* dims3);
int orc_conv2d_backward(void* h, const double* dy, long batch, long feat, double* dx);
int orc_conv2d_apply_updates(void* h, uint64_t it);
}

using xbarsim::MatrixXd;
using namespace xbarsim::nn;

static int failures = 0;
#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

template <class E>
static bool throws(const std::function<void()>& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static MatrixXd seeded(long r, long c, unsigned seed, double lo, double hi) {
  MatrixXd m(r, c);
  unsigned long long s = 0x9e3779b97f4a7c15ull ^ seed;
  for (long j = 0; j < c; ++j)
    for (long i = 0; i < r; ++i) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      m(i, j) = lo + (hi - lo) * double(s >> 11) * 0x1.0p-53;
    }
  return m;
}

static CrossbarLayerOptions aam_options() {
  CrossbarLayerOptions o;
  o.engine = xbarsim::EngineKind::aam;
  o.crossbar.rows = o.crossbar.cols = 64;
  o.map.tile_rows = o.map.tile_cols = 64;
  o.map.weight_bits = 8;
  o.map.device_bits = 2;
  o.map.variation_sigma = 0.1;
  o.map.seed = 3;
  o.adc.bits = 6;
  o.adc.i_fs = 6e-5;
  o.update.lr = 0.2;
  o.update.v = 0.5;
  o.update.gamma = 1.0;
  o.update.seed = 9;
  return o;
}

static void cpu_cases() {
  MatrixXd W = seeded(10, 6, 1, -0.1, 0.1);
  CrossbarLayerOptions o = aam_options();
  o.act_bits = 0;  // layers.cpp:17-47: 1 <= act_bits <= 24
  CHECK(throws<xbarsim::ConfigError>([&] { CrossbarLinear lin(W, o); }));
  o = aam_options();
  o.dac.bits = 2;  // dac.bits must equal stream_bits
  CHECK(throws<xbarsim::ConfigError>([&] { CrossbarLinear lin(W, o); }));
  o = aam_options();
  o.map.tile_rows = 128;  // tile larger than the crossbar (mapping.cpp:20-21)
  CHECK(throws<std::exception>([&] { CrossbarLinear lin(W, o); }));
}

static void gpu_cases() {
  const long K = 150, N = 90, M = 7;
  const CrossbarLayerOptions o = aam_options();
  const MatrixXd W = seeded(K, N, 2, -0.1, 0.1);
  CrossbarLinear lin(W, o);
  CHECK(lin.name() == "linear");
  CHECK(lin.core()->in_features() == K && lin.core()->out_features() == N);

  // backward before forward -> StateError (test_nn.cpp:240-244)
  Tensor dy0;
  dy0.values = MatrixXd(M, N);
  CHECK(throws<xbarsim::StateError>([&] { lin.backward(dy0); }));

  const xbs_layer_options co = o.to_c();
  void* orc = nullptr;
  CHECK(orc_core_create(&co, 1, W.data(), K, N, &orc) == 0);
  // feed the GPU's snapped conductances to the oracle (libm ulp flips only)
  const auto w = lin.core()->weights();
  const int T = w.grid_rows() * w.grid_cols();
  for (int s = 0; s < w.num_slices(); ++s)
    for (int p = 0; p < 2; ++p)
      for (int t = 0; t < T; ++t)
        CHECK(orc_core_set_nonideal(orc, s, p, t,
                                    lin.core()->nonideal(s, xbarsim::mapping::Polarity(p), t).data()) == 0);

  Tensor x;
  x.values = seeded(M, K, 3, -0.2, 1.2);
  x.dims = {int(K)};
  const Tensor y = lin.forward(x, true);
  MatrixXd y_o(M, N);
  CHECK(orc_core_forward(orc, x.values.data(), M, K, 1, y_o.data()) == 0);
  CHECK(y.values == y_o);
  CHECK(y.dims.size() == 1 && y.dims[0] == N);

  Tensor dy;
  dy.values = seeded(M, N, 4, -1.0, 1.0);
  const Tensor dx = lin.backward(dy);
  MatrixXd dx_o(M, K), dw_o(K, N);
  CHECK(orc_core_backward(orc, dy.values.data(), M, N, 1.0, dx_o.data()) == 0);
  CHECK(orc_core_gradient(orc, dw_o.data()) == 0);
  CHECK(dx.values == dx_o);
  CHECK(lin.core()->gradient() == dw_o);

  lin.apply_updates(0);
  CHECK(orc_core_apply_updates(orc, 0) == 0);
  const MatrixXd u = lin.core()->weights().master_diff(1);
  MatrixXd u_o(u.rows(), u.cols());
  CHECK(orc_core_master(orc, 1, u_o.data()) == 0);
  double err = 0.0, mx = 0.0;
  for (long j = 0; j < u.cols(); ++j)
    for (long i = 0; i < u.rows(); ++i) {
      err = std::fmax(err, std::fabs(u(i, j) - u_o(i, j)));
      mx = std::fmax(mx, std::fabs(u_o(i, j)));
    }
  CHECK(err <= 1e-12 * mx);
  CHECK(lin.core()->refresh_count() == 2);
  CHECK(lin.core()->grad_abs_max_seen() == dw_o.absMax());

  // shape errors -> std::invalid_argument (layers.cpp:216-217)
  Tensor bad;
  bad.values = MatrixXd(M, K + 1);
  CHECK(throws<std::invalid_argument>([&] { lin.forward(bad, false); }));
  orc_core_destroy(orc);
}

// CrossbarConv2d through the C++ API (test_nn.cpp's conv cases use the same
// calls): y, dx, dW bit-exact against the oracle's conv over two steps.
static void gpu_conv_cases() {
  const int in_c = 3, out_c = 8, k = 3, stride = 2, pad = 1, H = 9, Wd = 7;
  const long B = 2;
  const CrossbarLayerOptions o = aam_options();
  const MatrixXd W = seeded(in_c * k * k, out_c, 5, -0.2, 0.2);
  CHECK(throws<std::invalid_argument>([&] { CrossbarConv2d bad(W, in_c, out_c + 1, k, stride, pad, o); }));
  CrossbarConv2d conv(W, in_c, out_c, k, stride, pad, o);
  CHECK(conv.name() == "conv2d");
  CHECK(conv.core()->in_features() == in_c * k * k);
  const xbs_layer_options co = o.to_c();
  void* orc = nullptr;
  CHECK(orc_conv2d_create(&co, 1, W.data(), W.rows(), W.cols(), in_c, out_c, k, stride, pad, &orc) == 0);
  Tensor x;
  x.values = seeded(B, in_c * H * Wd, 6, -0.3, 1.1);
  x.dims = {in_c, H, Wd};
  for (int it = 0; it < 2; ++it) {
    const Tensor y = conv.forward(x, true);
    int dims[3] = {0, 0, 0};
    MatrixXd y_o(B, y.values.cols());
    CHECK(orc_conv2d_forward(orc, x.values.data(), B, in_c, H, Wd, 1, y_o.data(), dims) == 0);
    CHECK(y.dims.size() == 3 && y.dims[0] == dims[0] && y.dims[1] == dims[1] && y.dims[2] == dims[2]);
    CHECK(y.values == y_o);
    Tensor dy;
    dy.values = seeded(B, y.values.cols(), 7 + it, -1.0, 1.0);
    dy.dims = y.dims;
    const Tensor dx = conv.backward(dy);
    MatrixXd dx_o(B, x.values.cols());
    CHECK(orc_conv2d_backward(orc, dy.values.data(), B, dy.values.cols(), dx_o.data()) == 0);
    CHECK(dx.values == dx_o);
    CHECK(dx.dims == x.dims);
    conv.apply_updates(it);
    CHECK(orc_conv2d_apply_updates(orc, it) == 0);
  }
  Tensor bad;
  bad.values = MatrixXd(B, 2 * H * Wd);
  bad.dims = {2, H, Wd};
  CHECK(throws<std::invalid_argument>([&] { conv.forward(bad, false); }));
  orc_conv2d_destroy(orc);
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  cpu_cases();
  if (mode == "gpu") {
    gpu_cases();
    gpu_conv_cases();
  }
  std::printf("%s: %d failure(s)\n", mode.c_str(), failures);
  return failures == 0 ? 0 : 1;
}
