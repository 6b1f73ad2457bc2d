// The reference's update and mapping unit tests (proj/tests/unit/
// test_update.cpp, test_mapping.cpp) restated against the drop-in headers
// include/xbarsim/{update,mapping}.hpp: every free function runs on the GPU
// through the C ABI (map_weights, apply_variation, apply_update,
// scale_gradient, nonlinear_update, write_noise, reconstruct_output).
// Random matrices come from std::mt19937_64 (Eigen::MatrixXd::Random is not
// available); the known answers, seeds and tolerances are the reference's.
//
//   test_update_mapping          all cases (needs a B200)
//   test_update_mapping cpu      validation-only cases (no device work)
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "xbarsim/layers.hpp"
#include "xbarsim/update.hpp"

using namespace xbarsim;
using mapping::MappingSpec;
using mapping::Polarity;
using update::UpdateSpec;

static int failures = 0;
#define CHECK(c)                                                                 \
  do {                                                                           \
    if (!(c)) {                                                                  \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
      ++failures;                                                                \
    }                                                                            \
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

static bool approx(double a, double b, double eps) {
  return std::abs(a - b) <= eps * (1.0 + std::max(std::abs(a), std::abs(b)));
}

static MatrixXd uniform(int r, int c, std::mt19937_64& rng, double amp = 1.0) {
  std::uniform_real_distribution<double> d(-amp, amp);
  MatrixXd m(r, c);
  for (int j = 0; j < c; ++j)
    for (int i = 0; i < r; ++i) m(i, j) = d(rng);
  return m;
}

static double abs_max(const MatrixXd& m) { return m.absMax(); }

// ------------------------------------------------------------ test_update.cpp
static circuit::CrossbarConfig device_cfg() {  // test_update.cpp:16-23
  circuit::CrossbarConfig cfg;
  cfg.rows = cfg.cols = 4;
  cfg.g_min = 1e-6;
  cfg.g_max = 1e-5;
  return cfg;
}

static mapping::TiledLayerWeights tiny_layer(const MatrixXd& W, const circuit::CrossbarConfig& cfg, int wb = 8,
                                             int db = 8, double w_max = 1.0) {  // test_update.cpp:26-36
  MappingSpec spec;
  spec.weight_bits = wb;
  spec.device_bits = db;
  spec.tile_rows = cfg.rows;
  spec.tile_cols = cfg.cols;
  spec.w_max = w_max;
  return mapping::map_weights(W, spec, cfg);
}

static void update_cases() {
  {  // scale_gradient: definition, linearity, failure on zero scale (:41-60)
    auto cfg = device_cfg();
    UpdateSpec spec;
    spec.layer_scale = 0.5;
    spec.lr = 0.1;
    CHECK(abs_max(update::scale_gradient(MatrixXd::Zero(3, 3), spec, cfg)) == 0.0);
    auto dg = update::scale_gradient(MatrixXd::Constant(2, 2, 0.5), spec, cfg);
    CHECK(approx(dg(0, 0), cfg.g_max - cfg.g_min, 1e-15));
    std::mt19937_64 rng(3);
    MatrixXd r = uniform(4, 4, rng), r2(4, 4);
    for (int j = 0; j < 4; ++j)
      for (int i = 0; i < 4; ++i) r2(i, j) = 2.0 * r(i, j);
    auto a = update::scale_gradient(r2, spec, cfg), b = update::scale_gradient(r, spec, cfg);
    bool lin = true;
    for (int j = 0; j < 4; ++j)
      for (int i = 0; i < 4; ++i) lin = lin && a(i, j) == 2.0 * b(i, j);
    CHECK(lin);
    spec.layer_scale = 0.0;
    CHECK(throws<ConfigError>([&] { update::scale_gradient(MatrixXd::Constant(2, 2, 0.5), spec, cfg); }));
    MatrixXd bad = MatrixXd::Zero(2, 2);
    bad(1, 0) = std::nan("");
    spec.layer_scale = 1.0;
    CHECK(throws<std::invalid_argument>([&] { update::scale_gradient(bad, spec, cfg); }));
  }
  {  // nonlinear_update: closed-form checks (:62-78)
    auto cfg = device_cfg();
    UpdateSpec spec;
    spec.v = 0.0;
    CHECK(update::nonlinear_update(5e-6, 3e-7, spec, cfg) == 3e-7);
    CHECK(update::nonlinear_update(5e-6, -3e-7, spec, cfg) == -3e-7);
    spec.v = 2.5;
    CHECK(update::nonlinear_update(cfg.g_min, 1e-7, spec, cfg) == 1e-7);
    spec.v = 1.0;
    CHECK(approx(update::nonlinear_update(cfg.g_max, 1e-7, spec, cfg), 1e-7 * std::exp(-1.0), 1e-14));
    CHECK(throws<std::invalid_argument>([&] { update::nonlinear_update(2e-5, 1e-7, spec, cfg); }));
  }
  {  // nonlinear_update: attenuation bound and sign preservation (:80-95)
    auto cfg = device_cfg();
    std::mt19937_64 rng(5);
    std::uniform_real_distribution<double> gd(cfg.g_min, cfg.g_max), dgd(-1e-6, 1e-6), vd(0.0, 4.0);
    bool ok = true;
    for (int t = 0; t < 2000; ++t) {
      UpdateSpec spec;
      spec.v = vd(rng);
      const double g = gd(rng), dg = dgd(rng);
      const double out = update::nonlinear_update(g, dg, spec, cfg);
      ok = ok && std::abs(out) <= std::abs(dg) * (1.0 + 1e-15) && out * dg >= 0.0;
    }
    CHECK(ok);
  }
  {  // write_noise: exact zeros and empirical sigma (:97-122)
    auto cfg = device_cfg();
    UpdateSpec spec;
    CounterRng rng(1, 2, 3);
    spec.gamma = 0.0;
    CHECK(update::write_noise(1e-7, spec, cfg, rng) == 0.0);
    spec.gamma = 5.0;
    CHECK(update::write_noise(0.0, spec, cfg, rng) == 0.0);
    CHECK(rng.counter() == 0);  // a zero deviation draws nothing
    const double dg = 1e-9, expect = 5.0 * std::sqrt((cfg.g_max - cfg.g_min) * dg);
    double sum = 0.0, sq = 0.0;
    const int n = 100000;
    for (int k = 0; k < n; ++k) {
      CounterRng r(42, static_cast<std::uint64_t>(k), 0);
      const double x = update::write_noise(dg, spec, cfg, r);
      sum += x;
      sq += x * x;
    }
    const double mean = sum / n, sd = std::sqrt(sq / n - mean * mean);
    CHECK(approx(sd, expect, 0.02));
    CHECK(std::abs(mean) <= 3.0 * expect / std::sqrt(double(n)));
    // the device draw equals the host CounterRng's own gaussian() bit for bit
    // up to libm (cos / log / sqrt ulps): same counters, same key
    CounterRng h(42, 7, 0), d(42, 7, 0);
    const double host = 5.0 * std::sqrt((cfg.g_max - cfg.g_min) * dg) * h.gaussian();
    const double dev = update::write_noise(dg, spec, cfg, d);
    CHECK(approx(dev, host, 1e-13));
    CHECK(d.counter() == 2);
  }
  {  // apply_update: zero gradient with zero noise is a no-op (:124-136)
    auto cfg = device_cfg();
    std::mt19937_64 rng(7);
    auto t = tiny_layer(uniform(4, 4, rng), cfg);
    const MatrixXd before = t.master_diff(0);
    UpdateSpec spec;
    spec.lr = 0.5;
    spec.layer_scale = 1.0;
    update::apply_update(t, MatrixXd::Zero(4, 4), spec, 0);
    CHECK(t.master_diff(0) == before);
  }
  {  // apply_update: linear noiseless update is SGD in conductance space (:138-158)
    auto cfg = device_cfg();
    circuit::CrossbarConfig c1 = cfg;
    c1.rows = c1.cols = 1;
    auto t = tiny_layer(MatrixXd::Constant(1, 1, 0.25), c1);
    UpdateSpec spec;
    spec.lr = 1.0;
    spec.layer_scale = 1.0;
    const MatrixXd dW = MatrixXd::Constant(1, 1, 0.125);
    const double u_before = t.master_diff(0)(0, 0);
    update::apply_update(t, dW, spec, 0);
    const double u_after = t.master_diff(0)(0, 0);
    CHECK(approx(u_before - u_after, update::scale_gradient(dW, spec, c1)(0, 0), 1e-15));
  }
  {  // apply_update: polarity switches when the magnitude crosses zero (:160-181)
    auto cfg = device_cfg();
    circuit::CrossbarConfig c1 = cfg;
    c1.rows = c1.cols = 1;
    auto t = tiny_layer(MatrixXd::Constant(1, 1, 0.1), c1);
    CHECK(t.master_polarity(0, Polarity::pos)(0, 0) > c1.g_min);
    UpdateSpec spec;
    spec.lr = 1.0;
    spec.layer_scale = 1.0;
    update::apply_update(t, MatrixXd::Constant(1, 1, 0.3), spec, 0);
    CHECK(t.master_polarity(0, Polarity::pos)(0, 0) == c1.g_min);
    CHECK(t.master_polarity(0, Polarity::neg)(0, 0) > c1.g_min);
    CHECK(approx(t.implied_weights()(0, 0), 26.0 / 255.0 - 0.3, 1e-12));
  }
  {  // apply_update: conductances stay railed into [g_min, g_max] (:183-211)
    auto cfg = device_cfg();
    std::mt19937_64 rng(11);
    std::normal_distribution<double> nd(0.0, 1.0);
    auto t = tiny_layer(uniform(4, 4, rng), cfg, 8, 2);
    UpdateSpec spec;
    spec.lr = 0.05;
    spec.layer_scale = 1.0;
    spec.v = 0.3;
    spec.gamma = 5.0;
    spec.seed = 9;
    for (int iter = 0; iter < 10000; ++iter) {
      MatrixXd dW(4, 4);
      for (int j = 0; j < 4; ++j)
        for (int i = 0; i < 4; ++i) dW(i, j) = nd(rng);
      update::apply_update(t, dW, spec, static_cast<std::uint64_t>(iter));
    }
    bool railed = true;
    for (int s = 0; s < t.num_slices(); ++s)
      for (Polarity p : {Polarity::pos, Polarity::neg}) {
        const MatrixXd g = t.master_polarity(s, p);
        for (std::int64_t k = 0; k < g.size(); ++k)
          railed = railed && g.data()[k] >= cfg.g_min && g.data()[k] <= cfg.g_max;
      }
    CHECK(railed);
  }
  {  // apply_update: bit-identical for identical seeds (:213-239)
    auto cfg = device_cfg();
    std::mt19937_64 rng(13);
    const MatrixXd W = uniform(4, 4, rng), dW = uniform(4, 4, rng);
    UpdateSpec spec;
    spec.lr = 0.1;
    spec.layer_scale = 1.0;
    spec.v = 0.1;
    spec.gamma = 2.0;
    spec.seed = 1234;
    auto a = tiny_layer(W, cfg, 8, 2), b = tiny_layer(W, cfg, 8, 2);
    for (int iter = 0; iter < 5; ++iter) {
      update::apply_update(a, dW, spec, static_cast<std::uint64_t>(iter));
      update::apply_update(b, dW, spec, static_cast<std::uint64_t>(iter));
    }
    for (int s = 0; s < a.num_slices(); ++s) CHECK(a.master_diff(s) == b.master_diff(s));
    auto c = tiny_layer(W, cfg, 8, 2);
    UpdateSpec other = spec;
    other.seed = 4321;
    update::apply_update(c, dW, other, 0);
    update::apply_update(a, dW, spec, 5);
    CHECK(a.master_diff(0) != c.master_diff(0));
  }
  {  // apply_update: shape mismatch rejected (:241-248)
    auto cfg = device_cfg();
    auto t = tiny_layer(MatrixXd::Zero(4, 4), cfg);
    UpdateSpec spec;
    spec.layer_scale = 1.0;
    CHECK(throws<std::invalid_argument>([&] { update::apply_update(t, MatrixXd::Zero(3, 4), spec, 0); }));
    spec.lr = 0.0;  // UpdateSpec::validate runs first (update.cpp:45)
    CHECK(throws<std::invalid_argument>([&] { update::apply_update(t, MatrixXd::Zero(4, 4), spec, 0); }));
  }
  {  // mutable_master_diff (mapping.hpp:56) edits feed the next update
    auto cfg = device_cfg();
    auto t = tiny_layer(MatrixXd::Zero(4, 4), cfg, 8, 8);
    t.mutable_master_diff(0)(1, 2) = 2e-6;
    UpdateSpec spec;
    spec.lr = 1.0;
    spec.layer_scale = 1.0;
    MatrixXd dW = MatrixXd::Zero(4, 4);
    dW(1, 2) = 1e-3;
    update::apply_update(t, dW, spec, 0);
    CHECK(approx(t.master_diff(0)(1, 2), 2e-6 - 1e-3 * (cfg.g_max - cfg.g_min), 1e-15));
    CHECK(t.master_diff(0)(0, 0) == 0.0);
  }
}

// ----------------------------------------------------------- test_mapping.cpp
static circuit::CrossbarConfig base_cfg() {  // test_mapping.cpp:14-24
  circuit::CrossbarConfig cfg;
  cfg.rows = cfg.cols = 64;
  cfg.r_row = 1.0;
  cfg.r_col = 4.6;
  cfg.g_min = 1e-6;
  cfg.g_max = 1e-5;
  cfg.v_fs = 1.0;
  return cfg;
}

// independent sign-magnitude fixed-point value of w (test_mapping.cpp:28-35)
static double quantize_ref(double w, double scale, int wb) {
  const double levels = std::pow(2.0, wb) - 1.0;
  double q = double(std::llround(std::abs(w) / scale * levels));
  if (q > levels) q = levels;
  return (w < 0 ? -1.0 : 1.0) * q * (scale / levels);
}

static MappingSpec spec_of(int wb, int db, int tr, int tc, double w_max = 0.0) {
  MappingSpec s;
  s.weight_bits = wb;
  s.device_bits = db;
  s.tile_rows = tr;
  s.tile_cols = tc;
  s.w_max = w_max;
  return s;
}

static bool all_equal(const MatrixXd& m, double v) {
  for (std::int64_t k = 0; k < m.size(); ++k)
    if (m.data()[k] != v) return false;
  return true;
}

static void mapping_validation_cases() {  // test_mapping.cpp:124-144 (validation precedes any device work)
  auto cfg = base_cfg();
  auto spec = spec_of(8, 3, 8, 8);
  CHECK(throws<std::invalid_argument>([&] { mapping::map_weights(MatrixXd::Zero(4, 4), spec, cfg); }));
  spec.device_bits = 2;
  spec.tile_rows = 128;
  CHECK(throws<std::invalid_argument>([&] { mapping::map_weights(MatrixXd::Zero(4, 4), spec, cfg); }));
  MappingSpec rs = spec_of(4, 2, 8, 8);
  std::vector<VectorXd> missing(1, VectorXd::Zero(3)), neg(2, VectorXd::Zero(3));
  CHECK(throws<std::invalid_argument>([&] { mapping::reconstruct_output(missing, neg, rs, 1.0); }));
  nn::CrossbarLayerOptions o;  // CrossbarLayerOptions::validate (layers.cpp:17-47)
  o.validate();
  o.dac.bits = 2;
  CHECK(throws<ConfigError>([&] { o.validate(); }));
  o.dac.bits = 1;
  o.update.lr = 0.0;
  CHECK(throws<std::invalid_argument>([&] { o.validate(); }));
}

static void mapping_cases() {
  {  // zero matrix parks every device pair at g_min (:46-59)
    auto cfg = base_cfg();
    auto t = mapping::map_weights(MatrixXd::Zero(8, 8), spec_of(8, 2, 8, 8), cfg);
    for (int s = 0; s < t.num_slices(); ++s) {
      CHECK(abs_max(t.master_diff(s)) == 0.0);
      CHECK(all_equal(t.master_polarity(s, Polarity::pos), cfg.g_min));
      CHECK(all_equal(t.master_polarity(s, Polarity::neg), cfg.g_min));
    }
  }
  {  // full-scale positive weight saturates the pos device (:61-74)
    auto cfg = base_cfg();
    auto t = mapping::map_weights(MatrixXd::Constant(1, 1, 1.0), spec_of(2, 2, 1, 1, 1.0), cfg);
    CHECK(t.master_polarity(0, Polarity::pos)(0, 0) == cfg.g_max);
    CHECK(t.master_polarity(0, Polarity::neg)(0, 0) == cfg.g_min);
  }
  {  // 100x80 over 64x64 tiles: 2x2 grid and exact unmap (:76-101)
    auto cfg = base_cfg();
    std::mt19937_64 rng(7);
    const MatrixXd W = uniform(100, 80, rng);
    auto t = mapping::map_weights(W, spec_of(8, 2, 64, 64), cfg);
    CHECK(t.grid_rows() == 2 && t.grid_cols() == 2);
    CHECK(t.padded_rows() == 128 && t.padded_cols() == 128);
    CHECK(t.num_slices() == 4);
    const MatrixXd back = t.implied_weights();
    CHECK(back.rows() == 100 && back.cols() == 80);
    bool ok = true;
    for (int i = 0; i < 100; ++i)
      for (int j = 0; j < 80; ++j) ok = ok && approx(back(i, j), quantize_ref(W(i, j), t.layer_scale(), 8), 1e-12);
    CHECK(ok);
  }
  {  // differential exclusivity on every slice (:103-122)
    auto cfg = base_cfg();
    std::mt19937_64 rng(11);
    auto t = mapping::map_weights(uniform(30, 20, rng), spec_of(6, 3, 16, 16), cfg);
    bool ok = true;
    for (int s = 0; s < t.num_slices(); ++s) {
      const MatrixXd gp = t.master_polarity(s, Polarity::pos), gn = t.master_polarity(s, Polarity::neg);
      for (std::int64_t k = 0; k < gp.size(); ++k) ok = ok && !(gp.data()[k] > cfg.g_min && gn.data()[k] > cfg.g_min);
    }
    CHECK(ok);
  }
  {  // validation errors, non-finite weight (:140-143)
    auto cfg = base_cfg();
    MatrixXd bad = MatrixXd::Zero(2, 2);
    bad(1, 1) = std::nan("");
    CHECK(throws<std::invalid_argument>([&] { mapping::map_weights(bad, spec_of(8, 2, 8, 8), cfg); }));
  }
  {  // apply_variation: identity at sigma 0, deterministic per seed (:146-166)
    auto cfg = base_cfg();
    std::mt19937_64 rng(13);
    auto t = mapping::map_weights(uniform(16, 16, rng), spec_of(4, 2, 16, 16), cfg);
    auto same = mapping::apply_variation(t, 0.0, 99);
    CHECK(same.ideal_working(0, Polarity::pos) == t.master_polarity(0, Polarity::pos));
    auto a = mapping::apply_variation(t, 0.1, 42), b = mapping::apply_variation(t, 0.1, 42);
    CHECK(a.ideal_working(1, Polarity::neg) == b.ideal_working(1, Polarity::neg));
    auto c = mapping::apply_variation(t, 0.1, 43);
    CHECK(a.ideal_working(1, Polarity::neg) != c.ideal_working(1, Polarity::neg));
    CHECK(throws<std::invalid_argument>([&] { mapping::apply_variation(t, -0.1, 1); }));
  }
  {  // apply_variation: empirical spread within 2% (:168-190)
    auto cfg = base_cfg();
    cfg.rows = 400;
    cfg.cols = 250;
    cfg.g_max = 1e-4;
    auto t = mapping::apply_variation(
        mapping::map_weights(MatrixXd::Constant(400, 250, 0.1), spec_of(2, 2, 400, 250, 1.0), cfg), 0.1, 7);
    const MatrixXd base = t.master_polarity(0, Polarity::pos), varied = t.ideal_working(0, Polarity::pos);
    const double n = double(base.size());
    double sum = 0.0;
    for (std::int64_t k = 0; k < base.size(); ++k) sum += varied.data()[k] / base.data()[k];
    const double mean = sum / n;
    double var = 0.0;
    for (std::int64_t k = 0; k < base.size(); ++k) {
      const double d = varied.data()[k] / base.data()[k] - mean;
      var += d * d;
    }
    var /= n - 1.0;
    CHECK(approx(std::sqrt(var), 0.1, 0.02));
    CHECK(approx(mean, 1.0, 0.002));
  }
  {  // master state survives variation untouched (:192-208; the standalone
     // fcm_convert of the reference test is not part of this path's API)
    auto cfg = base_cfg();
    std::mt19937_64 rng(17);
    auto t = mapping::map_weights(uniform(10, 6, rng), spec_of(4, 2, 8, 8), cfg);
    const MatrixXd before = t.master_diff(0);
    auto varied = mapping::apply_variation(t, 0.2, 5);
    (void)varied.ideal_tile(0, Polarity::pos, 0, 0);
    CHECK(varied.master_diff(0) == before);
    CHECK(t.master_diff(0) == before);
  }
  {  // padding cells sit at g_min in every tile (:210-225)
    auto cfg = base_cfg();
    std::mt19937_64 rng(19);
    auto t = mapping::map_weights(uniform(5, 3, rng), spec_of(2, 2, 4, 4), cfg);
    CHECK(t.grid_rows() == 2 && t.grid_cols() == 1);
    const auto tile = t.ideal_tile(0, Polarity::pos, 1, 0);
    bool ok = true;
    for (int j = 0; j < 4; ++j)
      for (int i = 1; i < 4; ++i) ok = ok && tile.g(i, j) == cfg.g_min;
    CHECK(ok);
  }
  {  // reconstruct_output: recombination and cancellation (:227-249)
    const MappingSpec spec = spec_of(4, 2, 8, 8);
    std::vector<VectorXd> zeros(2, VectorXd::Zero(3));
    auto out = mapping::reconstruct_output(zeros, zeros, spec, 2.5);
    CHECK(out == VectorXd::Zero(3));
    std::vector<VectorXd> codes = {VectorXd::Constant(3, 7.0), VectorXd::Constant(3, 2.0)};
    CHECK(mapping::reconstruct_output(codes, codes, spec, 1.0) == VectorXd::Zero(3));
    std::vector<VectorXd> neg(2, VectorXd::Zero(3));
    const auto val = mapping::reconstruct_output(codes, neg, spec, 0.5);
    for (int k = 0; k < 3; ++k) CHECK(approx(val[k], 0.5 * (7.0 + 4.0 * 2.0), 1e-15));
  }
  {  // reconstruct_output inverts the slice decomposition (:251-279)
    auto cfg = base_cfg();
    std::mt19937_64 rng(23);
    const MatrixXd W = uniform(1, 8, rng);
    const MappingSpec spec = spec_of(8, 2, 8, 8);
    auto t = mapping::map_weights(W, spec, cfg);
    std::vector<VectorXd> pos(4, VectorXd(8)), neg(4, VectorXd(8));
    for (int s = 0; s < 4; ++s) {
      const MatrixXd gp = t.master_polarity(s, Polarity::pos), gn = t.master_polarity(s, Polarity::neg);
      for (int j = 0; j < 8; ++j) {
        pos[s][j] = std::round((gp(0, j) - cfg.g_min) / t.level_step());
        neg[s][j] = std::round((gn(0, j) - cfg.g_min) / t.level_step());
      }
    }
    const auto w_back = mapping::reconstruct_output(pos, neg, spec, t.layer_scale() / 255.0);
    bool ok = true;
    for (int j = 0; j < 8; ++j) ok = ok && approx(w_back[j], quantize_ref(W(0, j), t.layer_scale(), 8), 1e-12);
    CHECK(ok);
  }
  {  // a core's weights are a view: same master as the core, not updatable
    nn::CrossbarLayerOptions o;
    o.engine = EngineKind::aam;
    o.adc.i_fs = 1e-4;
    std::mt19937_64 rng(29);
    const MatrixXd W = uniform(64, 64, rng, 0.1);
    nn::CrossbarCore core(W, o);
    auto w = core.weights();
    auto m = mapping::map_weights(W, o.map, o.crossbar);
    CHECK(w.master_diff(2) == m.master_diff(2));
    CHECK(w.implied_weights() == m.implied_weights());
    UpdateSpec spec;
    CHECK(throws<std::invalid_argument>([&] { update::apply_update(w, MatrixXd::Zero(64, 64), spec, 0); }));
  }
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "gpu";
  mapping_validation_cases();
  if (mode == "gpu") {
    update_cases();
    mapping_cases();
  }
  std::printf("%s: %d failure(s)\n", mode.c_str(), failures);
  return failures == 0 ? 0 : 1;
}
