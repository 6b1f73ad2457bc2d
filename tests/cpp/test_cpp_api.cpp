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

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  cpu_cases();
  if (mode == "gpu") gpu_cases();
  std::printf("%s: %d failure(s)\n", mode.c_str(), failures);
  return failures == 0 ? 0 : 1;
}
