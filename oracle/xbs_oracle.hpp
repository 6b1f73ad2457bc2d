// =============================================================================
//  xbs_oracle — CPU restatement of the xbarsim crossbar-evaluation hot path.
//
//  TEST INFRASTRUCTURE ONLY.  This file is the *checker*: it is linked by the
//  tests under tests/, by __graft_entry__.smoke() and by bench.py's
//  cpu_baseline / --impl reference legs, and by nothing else.  The product
//  (paper_2002_11151_b200/, include/) never includes or links it.
//
//  What it restates (all paths relative to /root/reference/proj/core):
//    rng.hpp:12-48            CounterRng (splitmix64 keyed counter RNG)
//    crossbar.hpp:17-61       CrossbarConfig / ConductanceTile validation
//    aam.cpp:5-35             AAM closed-form direct-path conversion
//    converters.cpp:11-111    DAC encode, stream slices, ADC quantise, calibrator
//    tensor.cpp:8-51          unsigned / signed activation & error quantisers
//    mapping.cpp:10-160       weight mapping, polarity, variation, implied W
//    update.cpp:10-88         gradient scaling, non-linear update, write noise
//    layers.cpp:17-413        CrossbarLayerOptions::validate, CrossbarCore
//                             (regenerate, sense, forward, backward,
//                             apply_updates) and CrossbarLinear
//
//  The reference itself cannot be built in this image (Eigen3 and doctest are
//  absent), so this restatement is pinned against the known
//  answers of the reference's own unit tests (oracle/tests/kat_*.cpp).
//
//  Two current-evaluation modes:
//    literal : I = sum_r V[m,r] * G[r,c] in ascending r (fp64, no FMA);
//              this is the reference with Eigen's summation order fixed.
//    snapped : after conversion every non-ideal conductance is snapped to the
//              grid q * 2^-e (q integer, q <= Q_MAX), which makes every column
//              current an exact fp64 integer multiple of 2^-e.  This is the
//              exactness contract the GPU path implements bit for bit.
//  The only structural change vs. the reference is that regenerate() builds
//  the working (variation-applied) conductances once per (slice, polarity)
//  instead of once per tile job (layers.cpp:171 -> mapping.cpp:64); values
//  are identical.
// =============================================================================
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- errors.hpp
struct StateError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };

// -------------------------------------------------------- column-major matrix
// Stand-in for Eigen::MatrixXd / MatrixXi (the reference stores column-major).
template <class T>
struct Mat {
  long rows = 0, cols = 0;
  std::vector<T> v;
  Mat() = default;
  Mat(long r, long c, T fill = T(0)) : rows(r), cols(c), v(size_t(r) * size_t(c), fill) {}
  T& operator()(long i, long j) { return v[size_t(j) * size_t(rows) + size_t(i)]; }
  const T& operator()(long i, long j) const { return v[size_t(j) * size_t(rows) + size_t(i)]; }
  T* data() { return v.data(); }
  const T* data() const { return v.data(); }
  size_t size() const { return v.size(); }
};
using Matrix = Mat<double>;
using IMatrix = Mat<int>;

double max_abs(const Matrix& m);

// ------------------------------------------------------------------- rng.hpp
// rng.hpp:12-48
class CounterRng {
 public:
  CounterRng(uint64_t seed, uint64_t a, uint64_t b = 0, uint64_t c = 0)
      : key_(mix(mix(mix(mix(0x9e3779b97f4a7c15ull ^ seed, a), b), c), 0)) {}
  double uniform() { return to_unit(next()); }
  double gaussian() {
    double u1 = 1.0 - to_unit(next());
    double u2 = to_unit(next());
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925287 * u2);
  }
  uint64_t next() { return mix(key_, ++counter_); }
  uint64_t key() const { return key_; }
  static uint64_t mix(uint64_t h, uint64_t v) {
    h += 0x9e3779b97f4a7c15ull + v;
    h = (h ^ (h >> 30)) * 0xbf58476d1ce4e5b9ull;
    h = (h ^ (h >> 27)) * 0x94d049bb133111ebull;
    return h ^ (h >> 31);
  }
  static double to_unit(uint64_t x) { return double(x >> 11) * 0x1.0p-53; }

 private:
  uint64_t key_;
  uint64_t counter_ = 0;
};

// -------------------------------------------------------------- crossbar.hpp
struct CrossbarConfig {  // crossbar.hpp:17-40
  int rows = 64, cols = 64;
  double r_row = 1.0, r_col = 4.6, r_source = 0.0, r_sense = 0.0;
  double g_min = 1e-6, g_max = 1e-5, v_fs = 1.0;
  void validate() const;
};

enum class EngineKind { ideal = 0, oracle = 1, fcm = 2, aam = 3, interp_fcm = 4 };

// ------------------------------------------------------------ converters.hpp
struct DacSpec {  // converters.hpp:14-22
  int bits = 1;
  double v_fs = 1.0;
  std::vector<double> transfer;
  int stream_bits = 1;
  bool ideal_linear() const { return transfer.empty(); }
  void validate() const;
};
double dac_encode(uint64_t x, const DacSpec& spec);
struct StreamSlice { uint64_t value, weight; };
std::vector<StreamSlice> stream_slices(uint64_t x, int total_bits, int stream_bits);

struct AdcSpec {  // converters.hpp:37-45
  int bits = 8;
  double i_fs = 0.0;
  std::vector<double> transfer;
  double clip_percentile = 0.999;
  bool passthrough() const { return bits == 0; }
  void validate() const;
};
uint64_t adc_quantize(double i, const AdcSpec& spec);

class AdcCalibrator {  // converters.hpp:55-66
 public:
  void observe(double i);
  size_t sample_count() const { return samples_.size(); }
  double calibrate(double clip_percentile) const;

 private:
  std::vector<double> samples_;
};

// ---------------------------------------------------------------- tensor.hpp
IMatrix quantize_unsigned_codes(const Matrix& x, int bits, double full_scale);
Matrix codes_to_values(const IMatrix& codes, int bits, double full_scale);
struct SignedCodes { IMatrix magnitude, sign; };
SignedCodes quantize_signed_codes(const Matrix& x, int bits, double scale);

// --------------------------------------------------------------- mapping.hpp
enum class Polarity { pos = 0, neg = 1 };

struct MappingSpec {  // mapping.hpp:14-25
  int weight_bits = 8, device_bits = 2, tile_rows = 64, tile_cols = 64;
  double variation_sigma = 0.0;
  uint64_t seed = 0;
  double w_max = 0.0;
  int num_slices() const { return weight_bits / device_bits; }
  void validate(const CrossbarConfig& cfg) const;
};

class TiledLayerWeights {  // mapping.hpp:39-90
 public:
  int rows() const { return rows_; }
  int cols() const { return cols_; }
  int padded_rows() const { return grid_rows_ * spec_.tile_rows; }
  int padded_cols() const { return grid_cols_ * spec_.tile_cols; }
  int grid_rows() const { return grid_rows_; }
  int grid_cols() const { return grid_cols_; }
  int num_slices() const { return spec_.num_slices(); }
  double layer_scale() const { return layer_scale_; }
  const MappingSpec& spec() const { return spec_; }
  const CrossbarConfig& tile_config() const { return tile_cfg_; }
  double variation_sigma() const { return variation_sigma_; }
  uint64_t variation_seed() const { return variation_seed_; }
  const Matrix& master_diff(int s) const { return master_.at(size_t(s)); }
  Matrix& mutable_master_diff(int s) { return master_.at(size_t(s)); }
  Matrix master_polarity(int slice, Polarity p) const;
  Matrix ideal_working(int slice, Polarity p) const;
  Matrix ideal_tile(int slice, Polarity p, int tr, int tc) const;
  Matrix implied_weights() const;
  double level_step() const { return level_step_; }

  friend TiledLayerWeights map_weights(const Matrix&, const MappingSpec&, const CrossbarConfig&);
  friend TiledLayerWeights apply_variation(const TiledLayerWeights&, double, uint64_t);

 private:
  MappingSpec spec_;
  CrossbarConfig tile_cfg_;
  int rows_ = 0, cols_ = 0, grid_rows_ = 0, grid_cols_ = 0;
  double layer_scale_ = 1.0, level_step_ = 0.0, variation_sigma_ = 0.0;
  uint64_t variation_seed_ = 0;
  std::vector<Matrix> master_;
};

TiledLayerWeights map_weights(const Matrix& W, const MappingSpec& spec, const CrossbarConfig& cfg);
TiledLayerWeights apply_variation(const TiledLayerWeights& t, double sigma, uint64_t seed);
std::vector<double> reconstruct_output(const std::vector<std::vector<double>>& codes_pos,
                                       const std::vector<std::vector<double>>& codes_neg,
                                       const MappingSpec& spec, double scale);
double variation_multiplier(uint64_t seed, int slice, Polarity p, int64_t linear_index, double sigma);

// ------------------------------------------------------------------- aam.hpp
// aam.cpp:5-35; `g` is a tile of cfg.rows x cfg.cols.
Matrix aam_convert(const CrossbarConfig& cfg, const Matrix& g);

// ----------------------------------------------------- fcm.hpp / ladder.hpp
// fcm.cpp:14-224: block Gauss-Seidel over the row and column ladders, each
// line solved exactly by the Thomas algorithm, to a fixed point.
struct ConvergenceError : std::runtime_error {
  double residual;
  int iterations;
  ConvergenceError(const std::string& m, double r, int it) : std::runtime_error(m), residual(r), iterations(it) {}
};
struct StaleCacheError : std::runtime_error { using std::runtime_error::runtime_error; };
struct FcmOptions {  // fcm.hpp:9-16
  std::vector<double> v_cal;  // empty: all rows at v_fs
  double tol = 1e-6;
  int max_iter = 1000;
};
struct LadderResult {  // ladder.hpp:11-17
  Matrix v_top, v_bot;
  int sweeps = 0;
  double residual = 0.0;
  bool converged = false;
};
LadderResult solve_ladder(const CrossbarConfig& cfg, const Matrix& g, const std::vector<double>& v_in, double tol,
                          int max_iter);
Matrix fcm_convert(const CrossbarConfig& cfg, const Matrix& g, const FcmOptions& opt = {});

// ----------------------------------------------------------------- nodal.hpp
// nodal.cpp:14-176: the exact parasitic network (KCL at every top and bottom
// node) -- dense Cholesky up to 32x32 tiles, the ladder relaxation to 1e-10
// above.  CPU-only validation of FCM / AAM.
struct DegenerateCircuitError : std::runtime_error { using std::runtime_error::runtime_error; };
struct NodalSolution {
  Matrix v_top, v_bot;
  std::vector<double> i_col;
};
NodalSolution solve_nodal_oracle(const CrossbarConfig& cfg, const Matrix& g, const std::vector<double>& v_in);

// ------------------------------------------------------------ distortion.hpp
// distortion.cpp:10-48: interp_fcm's cached per-device distortion profile.
struct DistortionCache {
  Matrix d, g_at_refresh, g_non_at_refresh;
  int age = 0;
  int refresh_interval = 10;
};
void refresh_distortion(DistortionCache& cache, const CrossbarConfig& cfg, const Matrix& ideal, int engine_kind,
                        const FcmOptions& fcm_opt);
Matrix apply_distortion(DistortionCache& cache, const Matrix& ideal);

// ---------------------------------------------------------------- update.hpp
struct UpdateSpec {  // update.hpp:13-23
  double v = 0.0, gamma = 0.0, lr = 0.01;
  uint64_t seed = 0;
  double layer_scale = 0.0;
  void validate() const;
};
Matrix scale_gradient(const Matrix& dW, const UpdateSpec& spec, const CrossbarConfig& cfg);
double nonlinear_update(double g, double dg_ideal, const UpdateSpec& spec, const CrossbarConfig& cfg);
double write_noise(double dg_ideal, const UpdateSpec& spec, const CrossbarConfig& cfg, CounterRng& rng);
void apply_update(TiledLayerWeights& t, const Matrix& dW, const UpdateSpec& spec, uint64_t iteration);

// ------------------------------------------------------- snapped exactness grid
// Q_MAX = 255^3 - 1: the largest snapped level (three radix-255 u8 digits,
// the GPU's tensor-core limbs).
constexpr double kQMax = 16581374.0;  // 255.0 * 255.0 * 255.0 - 1
// Largest e with g_max * 2^e <= Q_MAX (radix-255 variant).
int snap_exponent(double g_max);
double snap_conductance(double g, int e);  // nearbyint(g * 2^e) * 2^-e

// ---------------------------------------------------------------- layers.hpp
struct CrossbarLayerOptions {  // layers.hpp:19-37
  MappingSpec map;
  CrossbarConfig crossbar;
  DacSpec dac;
  AdcSpec adc;
  UpdateSpec update;
  EngineKind engine = EngineKind::fcm;
  EngineKind interp_base = EngineKind::fcm;
  int interp_interval = 10;
  double fcm_tol = 1e-6;
  int fcm_max_iter = 1000;
  int act_bits = 8;
  double act_full_scale = 1.0;
  int error_bits = 8;
  int adc_cal_batches = 20;
  int threads = 1;
  // oracle-only: true -> snapped current mode, false -> literal
  bool snapped = true;
  void validate() const;
};

class CrossbarCore {  // layers.hpp:49-111
 public:
  // tiles: convert only these tiles (tr * grid_cols + tc) at construction and
  // at every regeneration (sampled parity runs on layers too large to convert)
  CrossbarCore(const Matrix& W0, const CrossbarLayerOptions& opt, const std::vector<int>* tiles = nullptr);
  Matrix forward(const Matrix& x, bool training);
  Matrix backward(const Matrix& dy, double grad_divisor);
  void apply_updates(uint64_t iteration);

  // Tile-sampled evaluation (same arithmetic as forward/backward, restricted
  // to a subset of output tiles; used for C4/C5 parity).  Columns/rows not
  // in the sample are left 0.  Neither changes the cached state except as
  // forward/backward would.
  Matrix forward_tiles(const Matrix& x, bool training, const std::vector<int>& tcs);
  Matrix backward_tiles(const Matrix& dy, double grad_divisor, const std::vector<int>& trs,
                        bool compute_dw);

  int in_features() const { return weights_.rows(); }
  int out_features() const { return weights_.cols(); }
  const TiledLayerWeights& weights() const { return weights_; }
  TiledLayerWeights& mutable_weights() { return weights_; }
  const Matrix& gradient() const { return dW_; }
  // parity harness: feed a gradient for the next apply_updates (the GPU's
  // xbs_core_set_gradient)
  void set_gradient(const Matrix& dW) {
    dW_ = dW;
    have_grad_ = true;
  }
  long refresh_count() const { return refreshes_; }
  double weight_abs_max_seen() const { return wmax_seen_; }
  double grad_abs_max_seen() const { return dwmax_seen_; }
  double forward_adc_full_scale() const { return adc_fwd_.i_fs; }
  double backward_adc_full_scale() const { return adc_bwd_.i_fs; }
  const Matrix& nonideal(int slice, Polarity p, int tile) const;
  int snap_e() const { return snap_e_; }
  bool fully_ideal() const;
  // all ADC codes produced by the last forward/backward (for flip counting);
  // only recorded when record_codes is set.
  bool record_codes = false;
  std::vector<uint16_t> last_codes;
  // regenerate using conductances restricted to a subset of tiles (cheap
  // sampled regeneration for huge layers); empty = all tiles.
  std::vector<int> regen_tiles;
  void regenerate();
  // overwrite one non-ideal tile (parity harness: feed GPU-produced state)
  void set_nonideal(int slice, Polarity p, int tile, const Matrix& g);

 private:
  void maybe_freeze_adc();
  Matrix sense(const Matrix& currents, const AdcSpec& spec, AdcCalibrator& cal, bool observe);
  Matrix currents(const Matrix& V, long col0, const Matrix& G, bool transpose) const;
  Matrix convert_tile(const Matrix& tile, int slice, int pol, int tile_index);
  double k_out_fwd() const;
  double k_out_bwd(double step_e) const;

  CrossbarLayerOptions opt_;
  TiledLayerWeights weights_;
  Matrix wimp_;
  std::vector<std::vector<std::vector<Matrix>>> nonideal_;
  std::vector<std::vector<std::vector<DistortionCache>>> caches_;  // interp_fcm
  AdcSpec adc_fwd_, adc_bwd_;
  AdcCalibrator cal_fwd_, cal_bwd_;
  bool adc_auto_ = false, adc_frozen_ = false;
  long training_batches_ = 0;
  std::vector<double> dac_lut_;
  Matrix x_values_;
  IMatrix x_codes_;
  bool have_forward_ = false;
  Matrix dW_;
  bool have_grad_ = false;
  uint64_t update_count_ = 0;
  long refreshes_ = 0;
  double wmax_seen_ = 0.0, dwmax_seen_ = 0.0;
  int snap_e_ = 0;
};

// Minimal tensor + layer wrappers (layers.hpp:113-134, tensor.hpp:13-21)
struct Tensor {
  Matrix values;
  std::vector<int> dims;
  int bits = 0;
  double full_scale = 0.0;
};

class CrossbarLinear {  // layers.cpp:393-413
 public:
  CrossbarLinear(const Matrix& W0, const CrossbarLayerOptions& opt) : core_(W0, opt) {}
  Tensor forward(const Tensor& x, bool training);
  Tensor backward(const Tensor& dy);
  void apply_updates(uint64_t iteration) { core_.apply_updates(iteration); }
  CrossbarCore* core() { return &core_; }

 private:
  CrossbarCore core_;
};

class CrossbarConv2d {  // layers.cpp:415-505 (im2col lowering onto one core)
 public:
  CrossbarConv2d(const Matrix& W0, int in_c, int out_c, int kernel, int stride, int padding,
                 const CrossbarLayerOptions& opt);
  Tensor forward(const Tensor& x, bool training);
  Tensor backward(const Tensor& dy);
  void apply_updates(uint64_t iteration) { core_.apply_updates(iteration); }
  CrossbarCore* core() { return &core_; }

 private:
  CrossbarCore core_;
  int in_c_, out_c_, kernel_, stride_, padding_;
  int in_h_ = 0, in_w_ = 0, out_h_ = 0, out_w_ = 0;
  long batch_ = 0;
};

// train.cpp:11-33
double softmax_cross_entropy(const Matrix& logits, const std::vector<int>& labels, Matrix& dlogits);
// layers.cpp:510-522: y = x * (x > 0), dx = dy * mask (IEEE products: -0.0 kept)
Matrix relu_forward(const Matrix& x, Matrix& mask);
Matrix relu_backward(const Matrix& dy, const Matrix& mask);
// layers.cpp:524-575: (c, h, w) feature order per batch row, strict '>'
// keeps the first maximum in (ky, kx) order; arg = input feature index
Matrix maxpool2d_forward(const Matrix& x, int c, int h, int w, int kernel, int stride, std::vector<int>& arg);
Matrix maxpool2d_backward(const Matrix& dy, int c, int h, int w, const std::vector<int>& arg);

}  // namespace orc
