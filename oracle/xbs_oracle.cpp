// TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.
// See xbs_oracle.hpp for scope.  Every function cites the reference
// file:line (relative to /root/reference/proj/core) it restates.
// Build with -ffp-contract=off: the reference build (Release, no -march)
// never contracts a*b+c into an FMA on x86-64.
#include "xbs_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <limits>

namespace orc {

double max_abs(const Matrix& m) {
  double r = 0.0;
  for (double x : m.v) r = std::max(r, std::abs(x));
  return r;
}

static bool all_finite(const Matrix& m) {
  for (double x : m.v)
    if (!std::isfinite(x)) return false;
  return true;
}

// ------------------------------------------------------------ crossbar.hpp:31-39
void CrossbarConfig::validate() const {
  if (rows < 1 || cols < 1) throw std::invalid_argument("CrossbarConfig: rows and cols must be >= 1");
  if (r_row < 0 || r_col < 0 || r_source < 0 || r_sense < 0)
    throw std::invalid_argument("CrossbarConfig: resistances must be >= 0");
  if (!(g_min > 0) || !(g_max > g_min)) throw std::invalid_argument("CrossbarConfig: need 0 < g_min < g_max");
  if (!(v_fs > 0)) throw std::invalid_argument("CrossbarConfig: v_fs must be > 0");
}

// ---------------------------------------------------------- converters.cpp:11-26
void DacSpec::validate() const {
  if (bits < 1 || bits > 32) throw std::invalid_argument("DacSpec: bits must be in [1, 32]");
  if (!(v_fs > 0)) throw std::invalid_argument("DacSpec: v_fs must be > 0");
  if (stream_bits < 1) throw std::invalid_argument("DacSpec: stream_bits must be >= 1");
  if (!transfer.empty()) {
    if (transfer.size() != (size_t{1} << bits))
      throw std::invalid_argument("DacSpec: transfer table must have 2^bits entries");
    if (transfer.front() != 0.0) throw std::invalid_argument("DacSpec: transfer[0] must be 0");
    if (transfer.back() > v_fs) throw std::invalid_argument("DacSpec: transfer must not exceed v_fs");
    if (!std::is_sorted(transfer.begin(), transfer.end()))
      throw std::invalid_argument("DacSpec: transfer table must be monotone");
  }
}

// converters.cpp:28-35
double dac_encode(uint64_t x, const DacSpec& spec) {
  const uint64_t levels = (uint64_t{1} << spec.bits) - 1;
  if (x > levels) throw std::invalid_argument("dac_encode: code out of range for DAC precision");
  if (!spec.transfer.empty()) return spec.transfer[size_t(x)];
  if (x == 0) return 0.0;
  return double(x) / double(levels) * spec.v_fs;
}

// converters.cpp:37-55
std::vector<StreamSlice> stream_slices(uint64_t x, int total_bits, int stream_bits) {
  if (total_bits < 1 || total_bits > 63 || stream_bits < 1)
    throw std::invalid_argument("stream_slices: invalid bit widths");
  if (total_bits % stream_bits != 0)
    throw std::invalid_argument("stream_slices: total_bits must be divisible by stream_bits");
  if (total_bits < 63 && x >= (uint64_t{1} << total_bits))
    throw std::invalid_argument("stream_slices: value does not fit in total_bits");
  const int n = total_bits / stream_bits;
  const uint64_t mask = (uint64_t{1} << stream_bits) - 1;
  std::vector<StreamSlice> out(static_cast<size_t>(n));
  for (int k = 0; k < n; ++k) {
    out[size_t(k)] = {x & mask, uint64_t{1} << (k * stream_bits)};
    x >>= stream_bits;
  }
  return out;
}

// converters.cpp:57-68
void AdcSpec::validate() const {
  if (bits < 0 || bits > 32) throw std::invalid_argument("AdcSpec: bits must be in [0, 32]");
  if (!(clip_percentile > 0.0) || clip_percentile > 1.0)
    throw std::invalid_argument("AdcSpec: clip_percentile must be in (0, 1]");
  if (!transfer.empty()) {
    if (bits == 0) throw std::invalid_argument("AdcSpec: transfer table with pass-through ADC");
    if (!std::is_sorted(transfer.begin(), transfer.end()))
      throw std::invalid_argument("AdcSpec: transfer thresholds must be monotone");
  }
}

// converters.cpp:70-88
uint64_t adc_quantize(double i, const AdcSpec& spec) {
  if (spec.passthrough()) throw StateError("adc_quantize: pass-through ADC has no codes");
  if (i < 0.0 || !std::isfinite(i)) throw std::invalid_argument("adc_quantize: current must be finite and >= 0");
  const uint64_t max_code = (uint64_t{1} << spec.bits) - 1;
  if (!spec.transfer.empty()) {
    auto it = std::upper_bound(spec.transfer.begin(), spec.transfer.end(), i);
    if (it == spec.transfer.begin()) return 0;
    uint64_t code = uint64_t((it - spec.transfer.begin()) - 1);
    return std::min(code, max_code);
  }
  if (!(spec.i_fs > 0)) throw StateError("adc_quantize: i_fs not set (calibrate first)");
  const double scaled = i / spec.i_fs * double(max_code);
  if (scaled >= double(max_code)) return max_code;
  return uint64_t(std::llround(scaled));
}

// converters.cpp:90-107
void AdcCalibrator::observe(double i) {
  if (!std::isfinite(i) || i < 0.0) throw std::invalid_argument("AdcCalibrator: current must be finite and >= 0");
  samples_.push_back(i);
}
double AdcCalibrator::calibrate(double clip_percentile) const {
  if (samples_.empty()) throw StateError("AdcCalibrator: no observations to calibrate from");
  if (!(clip_percentile > 0.0) || clip_percentile > 1.0)
    throw std::invalid_argument("AdcCalibrator: clip_percentile must be in (0, 1]");
  std::vector<double> sorted = samples_;
  std::sort(sorted.begin(), sorted.end());
  const auto n = sorted.size();
  auto rank = size_t(clip_percentile * double(n));
  if (rank >= n) rank = n - 1;
  return sorted[rank];
}

// ------------------------------------------------------------- tensor.cpp:8-51
IMatrix quantize_unsigned_codes(const Matrix& x, int bits, double full_scale) {
  if (bits < 1 || bits > 30) throw std::invalid_argument("quantize_unsigned_codes: bits must be in [1, 30]");
  if (!(full_scale > 0)) throw std::invalid_argument("quantize_unsigned_codes: full_scale must be > 0");
  const double levels = double((1 << bits) - 1);
  const double step = full_scale / levels;
  IMatrix codes(x.rows, x.cols);
  for (long j = 0; j < x.cols; ++j)
    for (long i = 0; i < x.rows; ++i) {
      double q = double(std::llround(x(i, j) / step));
      if (q < 0) q = 0;
      if (q > levels) q = levels;
      codes(i, j) = int(q);
    }
  return codes;
}

Matrix codes_to_values(const IMatrix& codes, int bits, double full_scale) {
  const double step = full_scale / double((1 << bits) - 1);
  Matrix v(codes.rows, codes.cols);
  for (size_t k = 0; k < v.v.size(); ++k) v.v[k] = double(codes.v[k]) * step;
  return v;
}

SignedCodes quantize_signed_codes(const Matrix& x, int bits, double scale) {
  if (bits < 1 || bits > 30) throw std::invalid_argument("quantize_signed_codes: bits must be in [1, 30]");
  SignedCodes out;
  out.magnitude = IMatrix(x.rows, x.cols, 0);
  out.sign = IMatrix(x.rows, x.cols, 0);
  if (!(scale > 0)) return out;
  const double levels = double((1 << bits) - 1);
  const double step = scale / levels;
  for (long j = 0; j < x.cols; ++j)
    for (long i = 0; i < x.rows; ++i) {
      const double v = x(i, j);
      double q = double(std::llround(std::abs(v) / step));
      if (q > levels) q = levels;
      out.magnitude(i, j) = int(q);
      out.sign(i, j) = q == 0 ? 0 : (v < 0 ? -1 : 1);
    }
  return out;
}

// ------------------------------------------------------------- mapping.cpp:10-160
void MappingSpec::validate(const CrossbarConfig& cfg) const {
  if (weight_bits < 1 || weight_bits > 24) throw std::invalid_argument("MappingSpec: weight_bits must be in [1, 24]");
  if (device_bits < 1 || device_bits > weight_bits)
    throw std::invalid_argument("MappingSpec: device_bits must be in [1, weight_bits]");
  if (weight_bits % device_bits != 0)
    throw std::invalid_argument("MappingSpec: weight_bits must be divisible by device_bits");
  if (tile_rows < 1 || tile_cols < 1) throw std::invalid_argument("MappingSpec: tile dims must be >= 1");
  if (tile_rows > cfg.rows || tile_cols > cfg.cols)
    throw std::invalid_argument("MappingSpec: tile dims exceed crossbar dims");
  if (variation_sigma < 0) throw std::invalid_argument("MappingSpec: variation_sigma must be >= 0");
}

// mapping.cpp:28-35
double variation_multiplier(uint64_t seed, int slice, Polarity p, int64_t linear_index, double sigma) {
  CounterRng rng(seed, uint64_t(slice) * 2 + (p == Polarity::neg ? 1 : 0), uint64_t(linear_index));
  double m = 1.0 + sigma * rng.gaussian();
  return m > 1e-12 ? m : 1e-12;
}

// mapping.cpp:39-45
Matrix TiledLayerWeights::master_polarity(int slice, Polarity p) const {
  const Matrix& u = master_.at(size_t(slice));
  const double g_min = tile_cfg_.g_min;
  Matrix g(u.rows, u.cols);
  for (size_t k = 0; k < u.v.size(); ++k)
    g.v[k] = (p == Polarity::pos ? std::max(u.v[k], 0.0) : std::max(-u.v[k], 0.0)) + g_min;
  return g;
}

// mapping.cpp:47-58
Matrix TiledLayerWeights::ideal_working(int slice, Polarity p) const {
  Matrix g = master_polarity(slice, p);
  if (variation_sigma_ == 0.0) return g;
  const double g_max = tile_cfg_.g_max;
  for (long j = 0; j < g.cols; ++j)
    for (long i = 0; i < g.rows; ++i) {
      const int64_t idx = int64_t(i) * padded_cols() + j;
      double m = variation_multiplier(variation_seed_, slice, p, idx, variation_sigma_);
      g(i, j) = std::min(g(i, j) * m, g_max);
    }
  return g;
}

// mapping.cpp:60-68
Matrix TiledLayerWeights::ideal_tile(int slice, Polarity p, int tr, int tc) const {
  if (tr < 0 || tr >= grid_rows_ || tc < 0 || tc >= grid_cols_)
    throw std::invalid_argument("TiledLayerWeights: tile index out of range");
  // Only the requested block is needed; element values equal the reference's
  // full-layer ideal_working() block (deduplicated, Appendix C.1).
  const int R = spec_.tile_rows, C = spec_.tile_cols;
  const Matrix& u = master_.at(size_t(slice));
  Matrix g(R, C);
  for (int j = 0; j < C; ++j)
    for (int i = 0; i < R; ++i) {
      const long gi = long(tr) * R + i, gj = long(tc) * C + j;
      const double uu = u(gi, gj);
      double v = (p == Polarity::pos ? std::max(uu, 0.0) : std::max(-uu, 0.0)) + tile_cfg_.g_min;
      if (variation_sigma_ != 0.0) {
        const int64_t idx = int64_t(gi) * padded_cols() + gj;
        double m = variation_multiplier(variation_seed_, slice, p, idx, variation_sigma_);
        v = std::min(v * m, tile_cfg_.g_max);
      }
      g(i, j) = v;
    }
  return g;
}

// mapping.cpp:70-81
Matrix TiledLayerWeights::implied_weights() const {
  const int slices = num_slices();
  Matrix acc(padded_rows(), padded_cols(), 0.0);
  const double base = double(uint64_t{1} << spec_.device_bits);
  for (int s = slices - 1; s >= 0; --s)
    for (size_t k = 0; k < acc.v.size(); ++k) acc.v[k] = acc.v[k] * base + master_[size_t(s)].v[k];
  const double levels = double((uint64_t{1} << spec_.weight_bits) - 1);
  const double slice_levels = double((uint64_t{1} << spec_.device_bits) - 1);
  const double factor = (layer_scale_ / (tile_cfg_.g_max - tile_cfg_.g_min)) * (slice_levels / levels);
  Matrix out(rows_, cols_);
  for (int j = 0; j < cols_; ++j)
    for (int i = 0; i < rows_; ++i) out(i, j) = factor * acc(i, j);
  return out;
}

// mapping.cpp:83-131
TiledLayerWeights map_weights(const Matrix& W, const MappingSpec& spec, const CrossbarConfig& cfg) {
  cfg.validate();
  spec.validate(cfg);
  if (!all_finite(W)) throw std::invalid_argument("map_weights: weights must be finite");
  if (W.rows == 0 || W.cols == 0) throw std::invalid_argument("map_weights: empty weight matrix");
  TiledLayerWeights t;
  t.spec_ = spec;
  t.tile_cfg_ = cfg;
  t.tile_cfg_.rows = spec.tile_rows;
  t.tile_cfg_.cols = spec.tile_cols;
  t.rows_ = int(W.rows);
  t.cols_ = int(W.cols);
  t.grid_rows_ = (t.rows_ + spec.tile_rows - 1) / spec.tile_rows;
  t.grid_cols_ = (t.cols_ + spec.tile_cols - 1) / spec.tile_cols;
  t.variation_sigma_ = spec.variation_sigma;
  t.variation_seed_ = spec.seed;
  double scale = spec.w_max > 0 ? spec.w_max : max_abs(W);
  if (scale == 0.0) scale = 1.0;
  t.layer_scale_ = scale;
  const int slices = spec.num_slices();
  const uint64_t q_levels = (uint64_t{1} << spec.weight_bits) - 1;
  const uint64_t d_levels = (uint64_t{1} << spec.device_bits) - 1;
  t.level_step_ = (cfg.g_max - cfg.g_min) / double(d_levels);
  t.master_.assign(size_t(slices), Matrix(t.padded_rows(), t.padded_cols(), 0.0));
  for (int i = 0; i < t.rows_; ++i)
    for (int j = 0; j < t.cols_; ++j) {
      const double w = W(i, j);
      const double mag = std::abs(w) / scale * double(q_levels);
      uint64_t q = uint64_t(std::llround(mag));
      if (q > q_levels) q = q_levels;
      const double sign = w < 0 ? -1.0 : 1.0;
      for (int s = 0; s < slices; ++s) {
        const uint64_t digit = (q >> (s * spec.device_bits)) & d_levels;
        if (digit != 0) t.master_[size_t(s)](i, j) = sign * (double(digit) * t.level_step_);
      }
    }
  return t;
}

// mapping.cpp:133-140
TiledLayerWeights apply_variation(const TiledLayerWeights& t, double sigma, uint64_t seed) {
  if (sigma < 0) throw std::invalid_argument("apply_variation: sigma must be >= 0");
  TiledLayerWeights out = t;
  out.variation_sigma_ = sigma;
  out.variation_seed_ = seed;
  return out;
}

// mapping.cpp:142-160
std::vector<double> reconstruct_output(const std::vector<std::vector<double>>& codes_pos,
                                       const std::vector<std::vector<double>>& codes_neg,
                                       const MappingSpec& spec, double scale) {
  const size_t slices = size_t(spec.num_slices());
  if (codes_pos.size() != slices || codes_neg.size() != slices)
    throw std::invalid_argument("reconstruct_output: need codes for every slice");
  const size_t n = codes_pos.empty() ? 0 : codes_pos[0].size();
  for (size_t s = 0; s < slices; ++s)
    if (codes_pos[s].size() != n || codes_neg[s].size() != n)
      throw std::invalid_argument("reconstruct_output: inconsistent code lengths");
  std::vector<double> acc(n, 0.0);
  double w = 1.0;
  for (size_t s = 0; s < slices; ++s) {
    for (size_t k = 0; k < n; ++k) acc[k] += w * (codes_pos[s][k] - codes_neg[s][k]);
    w *= double(uint64_t{1} << spec.device_bits);
  }
  for (double& a : acc) a = scale * a;
  return acc;
}

// ------------------------------------------------------------------ aam.cpp:5-35
Matrix aam_convert(const CrossbarConfig& cfg, const Matrix& g) {
  cfg.validate();
  if (g.rows != cfg.rows || g.cols != cfg.cols)
    throw std::invalid_argument("AamModel: tile dims do not match model geometry");
  Matrix gn(cfg.rows, cfg.cols);
  for (int j = 0; j < cfg.cols; ++j)
    for (int i = 0; i < cfg.rows; ++i) {
      const double rp = cfg.r_source + (j + 1) * cfg.r_row + (cfg.rows - i) * cfg.r_col + cfg.r_sense;
      const double gij = g(i, j);
      if (gij == 0.0) gn(i, j) = 0.0;
      else if (rp == 0.0) gn(i, j) = gij;
      else gn(i, j) = 1.0 / (1.0 / gij + rp);
    }
  return gn;
}

// --------------------------------------------------------------- update.cpp:10-88
void UpdateSpec::validate() const {
  if (v < 0) throw std::invalid_argument("UpdateSpec: v must be >= 0");
  if (gamma < 0) throw std::invalid_argument("UpdateSpec: gamma must be >= 0");
  if (!(lr > 0)) throw std::invalid_argument("UpdateSpec: lr must be > 0");
}

Matrix scale_gradient(const Matrix& dW, const UpdateSpec& spec, const CrossbarConfig& cfg) {
  if (!all_finite(dW)) throw std::invalid_argument("scale_gradient: gradient must be finite");
  if (spec.layer_scale == 0.0) throw ConfigError("scale_gradient: layer_scale must be nonzero");
  const double factor = (cfg.g_max - cfg.g_min) / spec.layer_scale;
  Matrix out(dW.rows, dW.cols);
  for (size_t k = 0; k < dW.v.size(); ++k) out.v[k] = dW.v[k] * factor;
  return out;
}

double nonlinear_update(double g, double dg_ideal, const UpdateSpec& spec, const CrossbarConfig& cfg) {
  if (g < cfg.g_min || g > cfg.g_max) throw std::invalid_argument("nonlinear_update: g outside device range");
  const double range = cfg.g_max - cfg.g_min;
  const double x = dg_ideal >= 0.0 ? (g - cfg.g_min) / range : (cfg.g_max - g) / range;
  return dg_ideal * std::exp(-spec.v * x);
}

double write_noise(double dg_ideal, const UpdateSpec& spec, const CrossbarConfig& cfg, CounterRng& rng) {
  const double sigma = spec.gamma * std::sqrt((cfg.g_max - cfg.g_min) * std::abs(dg_ideal));
  if (sigma == 0.0) return 0.0;
  return sigma * rng.gaussian();
}

void apply_update(TiledLayerWeights& t, const Matrix& dW, const UpdateSpec& spec, uint64_t iteration) {
  spec.validate();
  if (dW.rows != t.rows() || dW.cols != t.cols())
    throw std::invalid_argument("apply_update: gradient shape does not match layer");
  const CrossbarConfig& cfg = t.tile_config();
  const double range = cfg.g_max - cfg.g_min;
  UpdateSpec eff = spec;
  if (eff.layer_scale == 0.0) eff.layer_scale = t.layer_scale();
  const Matrix dg_ideal = scale_gradient(dW, eff, cfg);
  const int slices = t.num_slices();
  const bool linear = spec.v == 0.0;
  for (int s = 0; s < slices; ++s) {
    Matrix& u = t.mutable_master_diff(s);
    for (int j = 0; j < t.cols(); ++j)
      for (int i = 0; i < t.rows(); ++i) {
        const double dg = dg_ideal(i, j);
        double du = dg;
        if (!linear && dg != 0.0) {
          const double ui = u(i, j);
          const bool pos_active = ui > 0.0 || (ui == 0.0 && dg < 0.0);
          const double dev_arg = pos_active ? -dg : dg;
          const double nl = nonlinear_update(cfg.g_min + std::abs(ui), dev_arg, eff, cfg);
          du = pos_active ? -nl : nl;
        }
        double noise = 0.0;
        if (spec.gamma != 0.0 && dg != 0.0) {
          const int64_t idx = int64_t(i) * t.cols() + j;
          CounterRng rng(eff.seed, iteration, uint64_t(s), uint64_t(idx));
          noise = write_noise(dg, eff, cfg, rng);
        }
        double nu = u(i, j) - eff.lr * (du + noise);
        if (nu > range) nu = range;
        if (nu < -range) nu = -range;
        u(i, j) = nu;
      }
  }
}

// ------------------------------------------------------------------- snapping
int snap_exponent(double g_max) {
  // largest e with g_max * 2^e <= kQMax; ldexp is exact so the comparisons are.
  int e;
  (void)std::frexp(kQMax / g_max, &e);
  e += 2;
  while (std::ldexp(g_max, e) > kQMax) --e;
  return e;
}

double snap_conductance(double g, int e) { return std::ldexp(std::nearbyint(std::ldexp(g, e)), -e); }

// ------------------------------------------------------------- layers.cpp:17-47
void CrossbarLayerOptions::validate() const {
  crossbar.validate();
  map.validate(crossbar);
  dac.validate();
  adc.validate();
  update.validate();
  if (dac.bits != dac.stream_bits)
    throw ConfigError("dac.bits (" + std::to_string(dac.bits) + ") must equal dac.stream_bits (" +
                      std::to_string(dac.stream_bits) + "): the streamed slice is the physical converter");
  if (act_bits < 1 || act_bits > 24) throw ConfigError("act_bits must be in [1, 24]");
  if (error_bits < 1 || error_bits > 24) throw ConfigError("error_bits must be in [1, 24]");
  if (act_bits % dac.stream_bits != 0) throw ConfigError("activation_bits must be divisible by dac.stream_bits");
  if (error_bits % dac.stream_bits != 0) throw ConfigError("error_bits must be divisible by dac.stream_bits");
  if (!(act_full_scale > 0)) throw ConfigError("act_full_scale must be > 0");
  if (interp_interval < 1) throw ConfigError("interp_interval must be >= 1");
  if (engine == EngineKind::interp_fcm && interp_base != EngineKind::fcm && interp_base != EngineKind::aam)
    throw ConfigError("interp_base must be fcm or aam");
  if (adc_cal_batches < 1) throw ConfigError("adc_cal_batches must be >= 1");
  if (threads < 1) throw ConfigError("threads must be >= 1");
}

// layers.cpp:52-64 (digit_plane + lut_volts fused)
static Matrix plane_volts(const IMatrix& codes, int k, int sb, const std::vector<double>& lut) {
  const int shift = k * sb, mask = (1 << sb) - 1;
  Matrix v(codes.rows, codes.cols);
  for (size_t q = 0; q < v.v.size(); ++q) v.v[q] = lut[size_t((codes.v[q] >> shift) & mask)];
  return v;
}

// layers.cpp:68-83
CrossbarCore::CrossbarCore(const Matrix& W0, const CrossbarLayerOptions& opt, const std::vector<int>* tiles)
    : opt_(opt), weights_(map_weights(W0, opt.map, opt.crossbar)) {
  if (tiles) regen_tiles = *tiles;  // sampled parity runs convert only these tiles
  opt_.validate();
  adc_fwd_ = opt_.adc;
  adc_bwd_ = opt_.adc;
  adc_auto_ = opt_.adc.bits > 0 && !(opt_.adc.i_fs > 0) && opt_.adc.transfer.empty();
  const int digits = 1 << opt_.dac.bits;
  dac_lut_.resize(size_t(digits));
  for (int d = 0; d < digits; ++d) dac_lut_[size_t(d)] = dac_encode(uint64_t(d), opt_.dac);
  snap_e_ = snap_exponent(opt_.crossbar.g_max);
  regenerate();
}

// layers.cpp:85-88
bool CrossbarCore::fully_ideal() const {
  return opt_.engine == EngineKind::ideal && weights_.variation_sigma() == 0.0 && opt_.dac.ideal_linear() &&
         opt_.adc.bits == 0;
}

// ------------------------------------------------------------------- fcm.cpp
namespace {

// fcm.cpp:18-46: Thomas algorithm for the top nodes of row i, bottom nodes
// fixed; the driver reaches T(i, 0) through r_source plus one row segment.
void solve_row_tridiag(const CrossbarConfig& cfg, const Matrix& g, long i, double v_drive, const Matrix& v_bot,
                       Matrix& v_top, std::vector<double>& cw, std::vector<double>& dw) {
  const long C = cfg.cols;
  const double g_seg = 1.0 / cfg.r_row;
  const double g_drv = 1.0 / (cfg.r_source + cfg.r_row);
  double prev_c = 0.0, prev_d = 0.0;
  for (long j = 0; j < C; ++j) {
    const double gl = (j == 0) ? g_drv : g_seg;
    const double gr = (j < C - 1) ? g_seg : 0.0;
    const double diag = gl + gr + g(i, j);
    double rhs = g(i, j) * v_bot(i, j);
    if (j == 0) rhs += gl * v_drive;
    const double denom = diag - gl * prev_c;
    prev_c = gr / denom;
    prev_d = (rhs + gl * prev_d) / denom;
    cw[size_t(j)] = prev_c;
    dw[size_t(j)] = prev_d;
  }
  double x = dw[size_t(C - 1)];
  v_top(i, C - 1) = x;
  for (long j = C - 2; j >= 0; --j) {
    x = dw[size_t(j)] + cw[size_t(j)] * x;
    v_top(i, j) = x;
  }
}

// fcm.cpp:48-76: bottom nodes of column j, top nodes fixed; the foot drains
// to ground through one column segment plus r_sense.
void solve_col_tridiag(const CrossbarConfig& cfg, const Matrix& g, long j, const Matrix& v_top, Matrix& v_bot,
                       std::vector<double>& cw, std::vector<double>& dw) {
  const long R = cfg.rows;
  const double g_seg = 1.0 / cfg.r_col;
  const double g_foot = 1.0 / (cfg.r_col + cfg.r_sense);
  double prev_c = 0.0, prev_d = 0.0;
  for (long i = 0; i < R; ++i) {
    const double gu = (i > 0) ? g_seg : 0.0;
    const double gd = (i < R - 1) ? g_seg : g_foot;
    const double diag = gu + gd + g(i, j);
    const double rhs = g(i, j) * v_top(i, j);
    const double denom = diag - gu * prev_c;
    prev_c = gd / denom;
    prev_d = (rhs + gu * prev_d) / denom;
    cw[size_t(i)] = prev_c;
    dw[size_t(i)] = prev_d;
  }
  double x = dw[size_t(R - 1)];
  v_bot(R - 1, j) = x;
  for (long i = R - 2; i >= 0; --i) {
    x = dw[size_t(i)] + cw[size_t(i)] * x;
    v_bot(i, j) = x;
  }
}

// fcm.cpp:78-108: rows / columns collapsed to one node (zero wire resistance)
void solve_row_collapsed(const CrossbarConfig& cfg, const Matrix& g, long i, double v_drive, const Matrix& v_bot,
                         Matrix& v_top) {
  if (cfg.r_source == 0.0) {
    for (long j = 0; j < cfg.cols; ++j) v_top(i, j) = v_drive;
    return;
  }
  double num = v_drive / cfg.r_source;
  double den = 1.0 / cfg.r_source;
  for (long j = 0; j < cfg.cols; ++j) {
    num += g(i, j) * v_bot(i, j);
    den += g(i, j);
  }
  for (long j = 0; j < cfg.cols; ++j) v_top(i, j) = num / den;
}

void solve_col_collapsed(const CrossbarConfig& cfg, const Matrix& g, long j, const Matrix& v_top, Matrix& v_bot) {
  if (cfg.r_sense == 0.0) {
    for (long i = 0; i < cfg.rows; ++i) v_bot(i, j) = 0.0;
    return;
  }
  double num = 0.0;
  double den = 1.0 / cfg.r_sense;
  for (long i = 0; i < cfg.rows; ++i) {
    num += g(i, j) * v_top(i, j);
    den += g(i, j);
  }
  for (long i = 0; i < cfg.rows; ++i) v_bot(i, j) = num / den;
}

}  // namespace

// fcm.cpp:112-153
LadderResult solve_ladder(const CrossbarConfig& cfg, const Matrix& g, const std::vector<double>& v_in, double tol,
                          int max_iter) {
  const long R = cfg.rows, C = cfg.cols;
  LadderResult res;
  res.v_top = Matrix(R, C);
  for (long j = 0; j < C; ++j)
    for (long i = 0; i < R; ++i) res.v_top(i, j) = v_in[size_t(i)];
  res.v_bot = Matrix(R, C, 0.0);
  std::vector<double> cw(size_t(std::max(R, C))), dw(size_t(std::max(R, C)));
  for (int sweep = 1; sweep <= max_iter; ++sweep) {
    const Matrix top_prev = res.v_top, bot_prev = res.v_bot;
    for (long i = 0; i < R; ++i) {
      if (cfg.r_row == 0.0) solve_row_collapsed(cfg, g, i, v_in[size_t(i)], res.v_bot, res.v_top);
      else solve_row_tridiag(cfg, g, i, v_in[size_t(i)], res.v_bot, res.v_top, cw, dw);
    }
    for (long j = 0; j < C; ++j) {
      if (cfg.r_col == 0.0) solve_col_collapsed(cfg, g, j, res.v_top, res.v_bot);
      else solve_col_tridiag(cfg, g, j, res.v_top, res.v_bot, cw, dw);
    }
    double delta = 0.0;
    for (size_t k = 0; k < res.v_top.v.size(); ++k) delta = std::max(delta, std::fabs(res.v_top.v[k] - top_prev.v[k]));
    for (size_t k = 0; k < res.v_bot.v.size(); ++k) delta = std::max(delta, std::fabs(res.v_bot.v[k] - bot_prev.v[k]));
    res.sweeps = sweep;
    res.residual = delta / cfg.v_fs;
    if (res.residual <= tol) {
      res.converged = true;
      return res;
    }
  }
  return res;
}

// fcm.cpp:169-224
Matrix fcm_convert(const CrossbarConfig& cfg, const Matrix& g, const FcmOptions& opt) {
  if (!(opt.tol > 0.0) || !std::isfinite(opt.tol))
    throw std::invalid_argument("fcm_convert: tol must be positive and finite");
  if (opt.max_iter < 1) throw std::invalid_argument("fcm_convert: max_iter must be >= 1");
  std::vector<double> v_cal = opt.v_cal;
  if (v_cal.empty()) v_cal.assign(size_t(cfg.rows), cfg.v_fs);
  if (long(v_cal.size()) != cfg.rows) throw std::invalid_argument("fcm_convert: v_cal length does not match tile rows");
  for (double v : v_cal)
    if (!std::isfinite(v) || v < 0.0 || v > cfg.v_fs)
      throw std::invalid_argument("fcm_convert: v_cal entries must lie in [0, v_fs]");
  if (cfg.r_row == 0.0 && cfg.r_col == 0.0 && cfg.r_source == 0.0 && cfg.r_sense == 0.0) return g;
  auto run = [&](const std::vector<double>& v) {
    LadderResult r = solve_ladder(cfg, g, v, opt.tol, opt.max_iter);
    if (!r.converged)
      throw ConvergenceError("fcm_convert: no fixed point after " + std::to_string(opt.max_iter) +
                                 " sweeps (residual " + std::to_string(r.residual) + ")",
                             r.residual, r.sweeps);
    return r;
  };
  LadderResult sol = run(v_cal);
  Matrix gn(cfg.rows, cfg.cols);
  bool any_zero = false;
  for (long i = 0; i < cfg.rows; ++i) {
    if (v_cal[size_t(i)] == 0.0) {
      any_zero = true;
      continue;
    }
    for (long j = 0; j < cfg.cols; ++j) {
      const double gij = g(i, j);
      const double v_dev = sol.v_top(i, j) - sol.v_bot(i, j);
      const double eff = gij * v_dev / v_cal[size_t(i)];
      gn(i, j) = std::min(std::max(eff, 0.0), gij);
    }
  }
  if (any_zero) {
    std::vector<double> v_fb = v_cal;
    for (double& v : v_fb)
      if (v == 0.0) v = cfg.v_fs;
    LadderResult fb = run(v_fb);
    for (long i = 0; i < cfg.rows; ++i) {
      if (v_cal[size_t(i)] != 0.0) continue;
      for (long j = 0; j < cfg.cols; ++j) {
        const double gij = g(i, j);
        const double eff = gij * (fb.v_top(i, j) - fb.v_bot(i, j)) / cfg.v_fs;
        gn(i, j) = std::min(std::max(eff, 0.0), gij);
      }
    }
  }
  return gn;
}

// ------------------------------------------------------------------ nodal.cpp
namespace {

std::vector<double> column_currents(const Matrix& g, const Matrix& v_top, const Matrix& v_bot) {
  std::vector<double> i_col(size_t(g.cols));
  for (long j = 0; j < g.cols; ++j) {
    double acc = 0.0;
    for (long i = 0; i < g.rows; ++i) acc += g(i, j) * (v_top(i, j) - v_bot(i, j));
    i_col[size_t(j)] = acc;
  }
  return i_col;
}

struct NodeRef {
  long index = -1;  // >= 0: unknown
  double value = 0.0;
  bool fixed() const { return index < 0; }
};

// nodal.cpp:41-143 with zero-resistance chains collapsed onto supernodes (or
// onto the driver / ground); the SPD system is factorised by a plain
// row-oriented Cholesky (Eigen's LLT order is not reproducible here anyway).
NodalSolution solve_dense(const CrossbarConfig& cfg, const Matrix& g, const std::vector<double>& v_in) {
  const long R = cfg.rows, C = cfg.cols;
  const bool rows_chain = cfg.r_row > 0.0, rows_super = !rows_chain && cfg.r_source > 0.0;
  const bool cols_chain = cfg.r_col > 0.0, cols_super = !cols_chain && cfg.r_sense > 0.0;
  long n = 0;
  std::vector<long> top_idx, bot_idx, row_super(size_t(R), -1), col_super(size_t(C), -1);
  if (rows_chain) {
    top_idx.resize(size_t(R * C));
    for (long i = 0; i < R; ++i)
      for (long j = 0; j < C; ++j) top_idx[size_t(i * C + j)] = n++;
  } else if (rows_super) {
    for (long i = 0; i < R; ++i) row_super[size_t(i)] = n++;
  }
  if (cols_chain) {
    bot_idx.resize(size_t(R * C));
    for (long i = 0; i < R; ++i)
      for (long j = 0; j < C; ++j) bot_idx[size_t(i * C + j)] = n++;
  } else if (cols_super) {
    for (long j = 0; j < C; ++j) col_super[size_t(j)] = n++;
  }
  auto top = [&](long i, long j) -> NodeRef {
    if (rows_chain) return {top_idx[size_t(i * C + j)], 0.0};
    if (rows_super) return {row_super[size_t(i)], 0.0};
    return {-1, v_in[size_t(i)]};
  };
  auto bot = [&](long i, long j) -> NodeRef {
    if (cols_chain) return {bot_idx[size_t(i * C + j)], 0.0};
    if (cols_super) return {col_super[size_t(j)], 0.0};
    return {-1, 0.0};
  };
  std::vector<double> A(size_t(n * n), 0.0), b(size_t(n), 0.0);
  auto stamp = [&](NodeRef a, NodeRef c, double gamma) {
    if (gamma == 0.0) return;
    if (!a.fixed() && !c.fixed()) {
      if (a.index == c.index) return;
      A[size_t(a.index * n + a.index)] += gamma;
      A[size_t(c.index * n + c.index)] += gamma;
      A[size_t(a.index * n + c.index)] -= gamma;
      A[size_t(c.index * n + a.index)] -= gamma;
    } else if (!a.fixed()) {
      A[size_t(a.index * n + a.index)] += gamma;
      b[size_t(a.index)] += gamma * c.value;
    } else if (!c.fixed()) {
      A[size_t(c.index * n + c.index)] += gamma;
      b[size_t(c.index)] += gamma * a.value;
    }
  };
  for (long i = 0; i < R; ++i)
    for (long j = 0; j < C; ++j) stamp(top(i, j), bot(i, j), g(i, j));
  if (rows_chain) {
    for (long i = 0; i < R; ++i) {
      stamp({-1, v_in[size_t(i)]}, top(i, 0), 1.0 / (cfg.r_source + cfg.r_row));
      for (long j = 0; j + 1 < C; ++j) stamp(top(i, j), top(i, j + 1), 1.0 / cfg.r_row);
    }
  } else if (rows_super) {
    for (long i = 0; i < R; ++i) stamp({-1, v_in[size_t(i)]}, {row_super[size_t(i)], 0.0}, 1.0 / cfg.r_source);
  }
  if (cols_chain) {
    for (long j = 0; j < C; ++j) {
      for (long i = 0; i + 1 < R; ++i) stamp(bot(i, j), bot(i + 1, j), 1.0 / cfg.r_col);
      stamp(bot(R - 1, j), {-1, 0.0}, 1.0 / (cfg.r_col + cfg.r_sense));
    }
  } else if (cols_super) {
    for (long j = 0; j < C; ++j) stamp({col_super[size_t(j)], 0.0}, {-1, 0.0}, 1.0 / cfg.r_sense);
  }
  std::vector<double> x(size_t(n), 0.0);
  if (n > 0) {
    // Cholesky A = L L^T (L stored in the lower triangle of A)
    for (long k = 0; k < n; ++k) {
      double d = A[size_t(k * n + k)];
      for (long m = 0; m < k; ++m) d -= A[size_t(k * n + m)] * A[size_t(k * n + m)];
      if (!(d > 0.0)) throw DegenerateCircuitError("solve_nodal_oracle: singular nodal system");
      const double lkk = std::sqrt(d);
      A[size_t(k * n + k)] = lkk;
      for (long r = k + 1; r < n; ++r) {
        double v = A[size_t(r * n + k)];
        for (long m = 0; m < k; ++m) v -= A[size_t(r * n + m)] * A[size_t(k * n + m)];
        A[size_t(r * n + k)] = v / lkk;
      }
    }
    std::vector<double> y(static_cast<size_t>(n));
    for (long r = 0; r < n; ++r) {
      double v = b[size_t(r)];
      for (long m = 0; m < r; ++m) v -= A[size_t(r * n + m)] * y[size_t(m)];
      y[size_t(r)] = v / A[size_t(r * n + r)];
    }
    for (long r = n - 1; r >= 0; --r) {
      double v = y[size_t(r)];
      for (long m = r + 1; m < n; ++m) v -= A[size_t(m * n + r)] * x[size_t(m)];
      x[size_t(r)] = v / A[size_t(r * n + r)];
    }
    for (double v : x)
      if (!std::isfinite(v)) throw DegenerateCircuitError("solve_nodal_oracle: non-finite nodal solution");
  }
  NodalSolution sol;
  sol.v_top = Matrix(R, C);
  sol.v_bot = Matrix(R, C);
  for (long i = 0; i < R; ++i)
    for (long j = 0; j < C; ++j) {
      const NodeRef t = top(i, j), c = bot(i, j);
      sol.v_top(i, j) = t.fixed() ? t.value : x[size_t(t.index)];
      sol.v_bot(i, j) = c.fixed() ? c.value : x[size_t(c.index)];
    }
  sol.i_col = column_currents(g, sol.v_top, sol.v_bot);
  return sol;
}

}  // namespace

// nodal.cpp:147-176
NodalSolution solve_nodal_oracle(const CrossbarConfig& cfg, const Matrix& g, const std::vector<double>& v_in) {
  if (long(v_in.size()) != cfg.rows) throw std::invalid_argument("solve_nodal_oracle: v_in length does not match rows");
  for (double v : v_in)
    if (!std::isfinite(v) || v < 0.0 || v > cfg.v_fs)
      throw std::invalid_argument("solve_nodal_oracle: v_in entries must lie in [0, v_fs]");
  const bool no_par = cfg.r_row == 0.0 && cfg.r_col == 0.0 && cfg.r_source == 0.0 && cfg.r_sense == 0.0;
  bool all_zero = true;
  for (double x : g.v) all_zero = all_zero && x == 0.0;
  if (no_par && all_zero) throw DegenerateCircuitError("solve_nodal_oracle: all conductances zero with zero parasitics");
  if (cfg.rows <= 32 && cfg.cols <= 32) return solve_dense(cfg, g, v_in);
  LadderResult r = solve_ladder(cfg, g, v_in, 1e-10, 50000);
  if (!r.converged) throw ConvergenceError("solve_nodal_oracle: relaxation did not converge", r.residual, r.sweeps);
  NodalSolution sol;
  sol.v_top = r.v_top;
  sol.v_bot = r.v_bot;
  sol.i_col = column_currents(g, sol.v_top, sol.v_bot);
  return sol;
}

// ------------------------------------------------------------ distortion.cpp
void refresh_distortion(DistortionCache& cache, const CrossbarConfig& cfg, const Matrix& ideal, int engine_kind,
                        const FcmOptions& fcm_opt) {
  if (cache.refresh_interval < 1) throw std::invalid_argument("refresh_distortion: refresh_interval must be >= 1");
  if (engine_kind != int(EngineKind::fcm) && engine_kind != int(EngineKind::aam))
    throw std::invalid_argument("refresh_distortion: engine must be fcm or aam");
  Matrix non = engine_kind == int(EngineKind::fcm) ? fcm_convert(cfg, ideal, fcm_opt) : aam_convert(cfg, ideal);
  cache.d = Matrix(ideal.rows, ideal.cols);
  for (long j = 0; j < ideal.cols; ++j)
    for (long i = 0; i < ideal.rows; ++i) {
      const double gi = ideal(i, j);
      cache.d(i, j) = (gi == 0.0) ? 0.0 : (gi - non(i, j)) / gi;
    }
  cache.g_at_refresh = ideal;
  cache.g_non_at_refresh = non;
  cache.age = 0;
}

Matrix apply_distortion(DistortionCache& cache, const Matrix& ideal) {
  if (cache.d.v.empty()) throw StateError("apply_distortion: cache never refreshed");
  if (cache.d.rows != ideal.rows || cache.d.cols != ideal.cols)
    throw std::invalid_argument("apply_distortion: cache dims do not match tile");
  if (cache.age >= cache.refresh_interval)
    throw StaleCacheError("apply_distortion: cache age " + std::to_string(cache.age) + " reached refresh interval " +
                          std::to_string(cache.refresh_interval));
  ++cache.age;
  if (ideal.v == cache.g_at_refresh.v) return cache.g_non_at_refresh;  // unchanged tile: stored conversion
  Matrix gn(ideal.rows, ideal.cols);
  for (size_t k = 0; k < gn.v.size(); ++k) gn.v[k] = ideal.v[k] * (1.0 - cache.d.v[k]);
  return gn;
}

// layers.cpp:90-127 (ideal, aam, fcm, interp_fcm, and the oracle engine
// through the nodal solve, §8f row 4: CPU-only), then the snapped-mode grid.
Matrix CrossbarCore::convert_tile(const Matrix& tile, int slice, int pol, int tile_index) {
  const CrossbarConfig& cfg = weights_.tile_config();
  FcmOptions fo;
  fo.tol = opt_.fcm_tol;
  fo.max_iter = opt_.fcm_max_iter;
  const bool zero_par = cfg.r_row == 0.0 && cfg.r_col == 0.0 && cfg.r_source == 0.0 && cfg.r_sense == 0.0;
  Matrix g;
  switch (opt_.engine) {
    case EngineKind::ideal: g = tile; break;
    case EngineKind::aam: g = aam_convert(cfg, tile); break;
    case EngineKind::fcm: g = fcm_convert(cfg, tile, fo); break;
    case EngineKind::interp_fcm: {
      DistortionCache& cache = caches_[size_t(slice)][size_t(pol)][size_t(tile_index)];
      if (update_count_ % uint64_t(opt_.interp_interval) == 0)
        refresh_distortion(cache, cfg, tile, int(opt_.interp_base), fo);
      g = apply_distortion(cache, tile);
      break;
    }
    case EngineKind::oracle: {  // layers.cpp:104-117: effective g from the nodal solve at v_fs
      if (zero_par) {
        g = tile;
        break;
      }
      const NodalSolution sol = solve_nodal_oracle(cfg, tile, std::vector<double>(size_t(cfg.rows), cfg.v_fs));
      g = Matrix(cfg.rows, cfg.cols);
      for (int j = 0; j < cfg.cols; ++j)
        for (int i = 0; i < cfg.rows; ++i) {
          const double eff = tile(i, j) * (sol.v_top(i, j) - sol.v_bot(i, j)) / cfg.v_fs;
          g(i, j) = std::min(std::max(eff, 0.0), tile(i, j));
        }
      break;
    }
  }
  if (opt_.snapped)
    for (double& x : g.v) x = snap_conductance(x, snap_e_);
  return g;
}

// layers.cpp:129-179
void CrossbarCore::regenerate() {
  if (opt_.engine == EngineKind::ideal) {
    wimp_ = weights_.implied_weights();
    if (opt_.dac.ideal_linear() && opt_.adc.bits == 0 && weights_.variation_sigma() == 0.0) return;
  }
  const int slices = weights_.num_slices();
  const int tiles = weights_.grid_rows() * weights_.grid_cols();
  const bool interp = opt_.engine == EngineKind::interp_fcm;
  const bool refresh_now = !interp || update_count_ % uint64_t(opt_.interp_interval) == 0;
  if (nonideal_.empty()) {
    nonideal_.assign(size_t(slices), std::vector<std::vector<Matrix>>(2, std::vector<Matrix>(size_t(tiles))));
    if (interp) {
      caches_.assign(size_t(slices),
                     std::vector<std::vector<DistortionCache>>(2, std::vector<DistortionCache>(size_t(tiles))));
      for (auto& ps : caches_)
        for (auto& pp : ps)
          for (auto& c : pp) c.refresh_interval = opt_.interp_interval;
    }
  }
  std::vector<int> which = regen_tiles;
  if (which.empty())
    for (int t = 0; t < tiles; ++t) which.push_back(t);
  for (int s = 0; s < slices; ++s)
    for (int p = 0; p < 2; ++p)
      for (int t : which) {
        const int tr = t / weights_.grid_cols(), tc = t % weights_.grid_cols();
        nonideal_[size_t(s)][size_t(p)][size_t(t)] =
            convert_tile(weights_.ideal_tile(s, p == 0 ? Polarity::pos : Polarity::neg, tr, tc), s, p, t);
      }
  if (refresh_now && opt_.engine != EngineKind::ideal) ++refreshes_;
}

const Matrix& CrossbarCore::nonideal(int slice, Polarity p, int tile) const {
  if (nonideal_.empty()) throw StateError("CrossbarCore: no non-ideal state for the ideal fast path");
  return nonideal_.at(size_t(slice)).at(p == Polarity::pos ? 0 : 1).at(size_t(tile));
}

void CrossbarCore::set_nonideal(int slice, Polarity p, int tile, const Matrix& g) {
  nonideal_.at(size_t(slice)).at(p == Polarity::pos ? 0 : 1).at(size_t(tile)) = g;
}

// layers.cpp:189-197
void CrossbarCore::maybe_freeze_adc() {
  if (!adc_auto_ || adc_frozen_) return;
  if (training_batches_ < opt_.adc_cal_batches) return;
  if (cal_fwd_.sample_count() > 0) adc_fwd_.i_fs = cal_fwd_.calibrate(adc_fwd_.clip_percentile);
  if (cal_bwd_.sample_count() > 0) adc_bwd_.i_fs = cal_bwd_.calibrate(adc_bwd_.clip_percentile);
  adc_frozen_ = true;
}

// layers.cpp:199-213
Matrix CrossbarCore::sense(const Matrix& currents, const AdcSpec& spec, AdcCalibrator& cal, bool observe) {
  if (spec.bits == 0) return currents;
  const bool calibrating = adc_auto_ && !adc_frozen_;
  if (calibrating) {
    if (observe)
      for (double i : currents.v) cal.observe(i);
    return currents;
  }
  Matrix out(currents.rows, currents.cols);
  for (size_t k = 0; k < out.v.size(); ++k) {
    const uint64_t c = adc_quantize(currents.v[k], spec);
    out.v[k] = double(c);
    if (record_codes) last_codes.push_back(uint16_t(c));
  }
  return out;
}

// I = V[:, col0 : col0+G.rows] * G (transpose=false) or * G^T (transpose=true),
// ascending reduction index, plain multiply-add (layers.cpp:260-262, 356-361).
Matrix CrossbarCore::currents(const Matrix& V, long col0, const Matrix& G, bool transpose) const {
  const long Kr = transpose ? G.cols : G.rows;
  const long Nc = transpose ? G.rows : G.cols;
  Matrix I(V.rows, Nc, 0.0);
  for (long n = 0; n < Nc; ++n)
    for (long r = 0; r < Kr; ++r) {
      const double g = transpose ? G(n, r) : G(r, n);
      const double* vcol = &V.v[size_t(col0 + r) * size_t(V.rows)];
      double* icol = &I.v[size_t(n) * size_t(V.rows)];
      for (long m = 0; m < V.rows; ++m) icol[m] += vcol[m] * g;
    }
  return I;
}

double CrossbarCore::k_out_fwd() const {  // layers.cpp:272-281
  const double vu = opt_.dac.v_fs / (std::pow(2.0, opt_.dac.bits) - 1.0);
  const double sx = opt_.act_full_scale / (std::pow(2.0, opt_.act_bits) - 1.0);
  const double levels = std::pow(2.0, weights_.spec().weight_bits) - 1.0;
  const double slice_levels = std::pow(2.0, weights_.spec().device_bits) - 1.0;
  const double F = (weights_.layer_scale() / (opt_.crossbar.g_max - opt_.crossbar.g_min)) * (slice_levels / levels);
  double k_out = sx * F / vu;
  if (adc_fwd_.bits > 0 && (adc_frozen_ || !adc_auto_) && adc_fwd_.transfer.empty())
    k_out *= adc_fwd_.i_fs / (std::pow(2.0, adc_fwd_.bits) - 1.0);
  return k_out;
}

double CrossbarCore::k_out_bwd(double step_e) const {  // layers.cpp:369-377
  const double vu = opt_.dac.v_fs / (std::pow(2.0, opt_.dac.bits) - 1.0);
  const double levels = std::pow(2.0, weights_.spec().weight_bits) - 1.0;
  const double slice_levels = std::pow(2.0, weights_.spec().device_bits) - 1.0;
  const double F = (weights_.layer_scale() / (opt_.crossbar.g_max - opt_.crossbar.g_min)) * (slice_levels / levels);
  double k_out = step_e * F / vu;
  if (adc_bwd_.bits > 0 && (adc_frozen_ || !adc_auto_) && adc_bwd_.transfer.empty())
    k_out *= adc_bwd_.i_fs / (std::pow(2.0, adc_bwd_.bits) - 1.0);
  return k_out;
}

Matrix CrossbarCore::forward(const Matrix& x, bool training) {
  std::vector<int> all;
  for (int tc = 0; tc < weights_.grid_cols(); ++tc) all.push_back(tc);
  return forward_tiles(x, training, all);
}

// layers.cpp:215-284
Matrix CrossbarCore::forward_tiles(const Matrix& x, bool training, const std::vector<int>& tcs) {
  if (x.cols != weights_.rows()) throw std::invalid_argument("CrossbarCore::forward: feature count mismatch");
  maybe_freeze_adc();
  const long batch = x.rows;
  IMatrix codes = quantize_unsigned_codes(x, opt_.act_bits, opt_.act_full_scale);
  x_values_ = codes_to_values(codes, opt_.act_bits, opt_.act_full_scale);
  x_codes_ = codes;
  have_forward_ = true;
  if (training) ++training_batches_;
  last_codes.clear();

  if (fully_ideal()) {  // x_values_ * wimp_, ascending k
    Matrix y(batch, wimp_.cols, 0.0);
    for (long j = 0; j < wimp_.cols; ++j)
      for (long k = 0; k < wimp_.rows; ++k) {
        const double w = wimp_(k, j);
        for (long i = 0; i < batch; ++i) y(i, j) += x_values_(i, k) * w;
      }
    return y;
  }
  const int in = weights_.rows(), out = weights_.cols();
  const int tile_rows = weights_.spec().tile_rows, tile_cols = weights_.spec().tile_cols;
  const int slices = weights_.num_slices();
  const int sb = opt_.dac.stream_bits;
  const int n_streams = opt_.act_bits / sb;
  IMatrix codes_pad(batch, weights_.padded_rows(), 0);
  for (long j = 0; j < in; ++j)
    for (long i = 0; i < batch; ++i) codes_pad(i, j) = codes(i, j);
  std::vector<Matrix> volts(static_cast<size_t>(n_streams));
  for (int k = 0; k < n_streams; ++k) volts[size_t(k)] = plane_volts(codes_pad, k, sb, dac_lut_);
  const double slice_base = std::pow(2.0, weights_.spec().device_bits);
  const double stream_base = std::pow(2.0, sb);

  Matrix out_pad(batch, weights_.padded_cols(), 0.0);
  for (int tc : tcs)
    for (int tr = 0; tr < weights_.grid_rows(); ++tr) {
      const int t = tr * weights_.grid_cols() + tc;
      Matrix tile_out(batch, tile_cols, 0.0);
      for (int s = 0; s < slices; ++s) {
        const double sw = std::pow(slice_base, s);
        for (int p = 0; p < 2; ++p) {
          const Matrix& G = nonideal_[size_t(s)][size_t(p)][size_t(t)];
          Matrix acc(batch, tile_cols, 0.0);
          double wk = 1.0;
          for (int k = 0; k < n_streams; ++k) {
            Matrix cur = currents(volts[size_t(k)], long(tr) * tile_rows, G, false);
            Matrix sensed = sense(cur, adc_fwd_, cal_fwd_, training);
            for (size_t q = 0; q < acc.v.size(); ++q) acc.v[q] += wk * sensed.v[q];
            wk *= stream_base;
          }
          const double sgn = p == 0 ? sw : -sw;
          for (size_t q = 0; q < acc.v.size(); ++q) tile_out.v[q] += sgn * acc.v[q];
        }
      }
      for (long j = 0; j < tile_cols; ++j)
        for (long i = 0; i < batch; ++i) out_pad(i, long(tc) * tile_cols + j) += tile_out(i, j);
    }
  const double k_out = k_out_fwd();
  Matrix y(batch, out);
  for (long j = 0; j < out; ++j)
    for (long i = 0; i < batch; ++i) y(i, j) = out_pad(i, j) * k_out;
  return y;
}

Matrix CrossbarCore::backward(const Matrix& dy, double grad_divisor) {
  std::vector<int> all;
  for (int tr = 0; tr < weights_.grid_rows(); ++tr) all.push_back(tr);
  return backward_tiles(dy, grad_divisor, all, true);
}

// layers.cpp:286-380
Matrix CrossbarCore::backward_tiles(const Matrix& dy, double grad_divisor, const std::vector<int>& trs,
                                    bool compute_dw) {
  if (!have_forward_) throw StateError("CrossbarCore::backward: no cached forward activations");
  if (dy.cols != weights_.cols() || dy.rows != x_values_.rows)
    throw std::invalid_argument("CrossbarCore::backward: gradient shape mismatch");
  maybe_freeze_adc();
  last_codes.clear();
  const long batch = dy.rows;
  const int in = weights_.rows(), out = weights_.cols();
  const int eb = opt_.error_bits;
  const double se = max_abs(dy);
  SignedCodes sc = quantize_signed_codes(dy, eb, se);
  const double step_e = se > 0 ? se / (std::pow(2.0, eb) - 1.0) : 0.0;
  Matrix dy_q(batch, out);
  for (size_t q = 0; q < dy_q.v.size(); ++q)
    dy_q.v[q] = double(sc.sign.v[q]) * double(sc.magnitude.v[q]) * step_e;

  if (compute_dw) {
    dW_ = Matrix(in, out, 0.0);
    if (opt_.snapped) {
      // Snapped-mode dW contract: exact integer outer
      // product, then ((S * sx) * step_e) / grad_divisor.
      const double sx = opt_.act_full_scale / (std::pow(2.0, opt_.act_bits) - 1.0);
      for (long j = 0; j < out; ++j)
        for (long i = 0; i < in; ++i) {
          int64_t S = 0;
          for (long b = 0; b < batch; ++b)
            S += int64_t(x_codes_(b, i)) * int64_t(sc.sign(b, j) * sc.magnitude(b, j));
          dW_(i, j) = ((double(S) * sx) * step_e) / grad_divisor;
        }
    } else {  // x_values_^T * dy_q / grad_divisor, ascending batch index
      for (long j = 0; j < out; ++j)
        for (long i = 0; i < in; ++i) {
          double a = 0.0;
          for (long b = 0; b < batch; ++b) a += x_values_(b, i) * dy_q(b, j);
          dW_(i, j) = a / grad_divisor;
        }
    }
    have_grad_ = true;
  }

  if (fully_ideal()) {  // dy_q * wimp_^T
    Matrix dx(batch, in, 0.0);
    for (long j = 0; j < in; ++j)
      for (long k = 0; k < out; ++k) {
        const double w = wimp_(j, k);
        for (long i = 0; i < batch; ++i) dx(i, j) += dy_q(i, k) * w;
      }
    return dx;
  }
  if (!(se > 0)) return Matrix(batch, in, 0.0);

  const int tile_rows = weights_.spec().tile_rows, tile_cols = weights_.spec().tile_cols;
  const int slices = weights_.num_slices();
  const int sb = opt_.dac.stream_bits;
  const int n_streams = eb / sb;
  IMatrix plus(batch, weights_.padded_cols(), 0), minus(batch, weights_.padded_cols(), 0);
  for (long j = 0; j < out; ++j)
    for (long i = 0; i < batch; ++i) {
      if (sc.sign(i, j) > 0) plus(i, j) = sc.magnitude(i, j);
      else if (sc.sign(i, j) < 0) minus(i, j) = sc.magnitude(i, j);
    }
  std::vector<Matrix> vp(static_cast<size_t>(n_streams)), vm(static_cast<size_t>(n_streams));
  for (int k = 0; k < n_streams; ++k) {
    vp[size_t(k)] = plane_volts(plus, k, sb, dac_lut_);
    vm[size_t(k)] = plane_volts(minus, k, sb, dac_lut_);
  }
  const double slice_base = std::pow(2.0, weights_.spec().device_bits);
  const double stream_base = std::pow(2.0, sb);
  Matrix dx_pad(batch, weights_.padded_rows(), 0.0);
  for (int tr : trs)
    for (int tc = 0; tc < weights_.grid_cols(); ++tc) {
      const int t = tr * weights_.grid_cols() + tc;
      Matrix tile_dx(batch, tile_rows, 0.0);
      for (int s = 0; s < slices; ++s) {
        const double sw = std::pow(slice_base, s);
        const Matrix& gp = nonideal_[size_t(s)][0][size_t(t)];
        const Matrix& gn = nonideal_[size_t(s)][1][size_t(t)];
        Matrix acc_pos(batch, tile_rows, 0.0), acc_neg(batch, tile_rows, 0.0);
        double wk = 1.0;
        for (int k = 0; k < n_streams; ++k) {
          const long c0 = long(tc) * tile_cols;
          Matrix a = sense(currents(vp[size_t(k)], c0, gp, true), adc_bwd_, cal_bwd_, true);
          Matrix b = sense(currents(vm[size_t(k)], c0, gn, true), adc_bwd_, cal_bwd_, true);
          Matrix c = sense(currents(vp[size_t(k)], c0, gn, true), adc_bwd_, cal_bwd_, true);
          Matrix d = sense(currents(vm[size_t(k)], c0, gp, true), adc_bwd_, cal_bwd_, true);
          for (size_t q = 0; q < acc_pos.v.size(); ++q) {
            acc_pos.v[q] += wk * (a.v[q] + b.v[q]);
            acc_neg.v[q] += wk * (c.v[q] + d.v[q]);
          }
          wk *= stream_base;
        }
        for (size_t q = 0; q < tile_dx.v.size(); ++q) tile_dx.v[q] += sw * (acc_pos.v[q] - acc_neg.v[q]);
      }
      for (long j = 0; j < tile_rows; ++j)
        for (long i = 0; i < batch; ++i) dx_pad(i, long(tr) * tile_rows + j) += tile_dx(i, j);
    }
  const double k_out = k_out_bwd(step_e);
  Matrix dx(batch, in);
  for (long j = 0; j < in; ++j)
    for (long i = 0; i < batch; ++i) dx(i, j) = dx_pad(i, j) * k_out;
  return dx;
}

// layers.cpp:382-391
void CrossbarCore::apply_updates(uint64_t iteration) {
  if (!have_grad_) return;
  dwmax_seen_ = std::max(dwmax_seen_, max_abs(dW_));
  apply_update(weights_, dW_, opt_.update, iteration);
  wmax_seen_ = std::max(wmax_seen_, max_abs(weights_.implied_weights()));
  ++update_count_;
  regenerate();
  have_grad_ = false;
  have_forward_ = false;
}

// layers.cpp:397-409
// layers.cpp:415-429
CrossbarConv2d::CrossbarConv2d(const Matrix& W0, int in_c, int out_c, int kernel, int stride, int padding,
                               const CrossbarLayerOptions& opt)
    : core_(W0, opt), in_c_(in_c), out_c_(out_c), kernel_(kernel), stride_(stride), padding_(padding) {
  if (W0.rows != long(in_c) * kernel * kernel || W0.cols != out_c)
    throw std::invalid_argument("CrossbarConv2d: kernel matrix must be (in_c*k*k) x out_c");
  if (stride < 1 || kernel < 1 || padding < 0) throw std::invalid_argument("CrossbarConv2d: bad geometry");
}

// layers.cpp:431-469: im2col (one row per output position per sample), the
// dense pipeline, then (b, oc, oy, ox) order
Tensor CrossbarConv2d::forward(const Tensor& x, bool training) {
  if (x.dims.size() != 3 || x.dims[0] != in_c_) throw std::invalid_argument("CrossbarConv2d: expected (c, h, w) input");
  in_h_ = x.dims[1];
  in_w_ = x.dims[2];
  out_h_ = (in_h_ + 2 * padding_ - kernel_) / stride_ + 1;
  out_w_ = (in_w_ + 2 * padding_ - kernel_) / stride_ + 1;
  if (out_h_ < 1 || out_w_ < 1) throw std::invalid_argument("CrossbarConv2d: kernel does not fit the input");
  batch_ = x.values.rows;
  const long rows = batch_ * out_h_ * out_w_;
  Matrix patches(rows, long(in_c_) * kernel_ * kernel_, 0.0);
  for (long b = 0; b < batch_; ++b)
    for (int oy = 0; oy < out_h_; ++oy)
      for (int ox = 0; ox < out_w_; ++ox) {
        const long r = (b * out_h_ + oy) * out_w_ + ox;
        for (int c = 0; c < in_c_; ++c)
          for (int ky = 0; ky < kernel_; ++ky)
            for (int kx = 0; kx < kernel_; ++kx) {
              const int iy = oy * stride_ + ky - padding_, ix = ox * stride_ + kx - padding_;
              if (iy < 0 || iy >= in_h_ || ix < 0 || ix >= in_w_) continue;
              patches(r, (c * kernel_ + ky) * kernel_ + kx) = x.values(b, (long(c) * in_h_ + iy) * in_w_ + ix);
            }
      }
  const Matrix flat = core_.forward(patches, training);
  Tensor y;
  y.dims = {out_c_, out_h_, out_w_};
  y.values = Matrix(batch_, long(out_c_) * out_h_ * out_w_);
  for (long b = 0; b < batch_; ++b)
    for (int oc = 0; oc < out_c_; ++oc)
      for (int oy = 0; oy < out_h_; ++oy)
        for (int ox = 0; ox < out_w_; ++ox)
          y.values(b, (long(oc) * out_h_ + oy) * out_w_ + ox) = flat((b * out_h_ + oy) * out_w_ + ox, oc);
  return y;
}

// layers.cpp:471-500: col2im accumulates in (b, oy, ox, c, ky, kx) order
Tensor CrossbarConv2d::backward(const Tensor& dy) {
  const long rows = batch_ * out_h_ * out_w_;
  Matrix flat(rows, out_c_);
  for (long b = 0; b < batch_; ++b)
    for (int oc = 0; oc < out_c_; ++oc)
      for (int oy = 0; oy < out_h_; ++oy)
        for (int ox = 0; ox < out_w_; ++ox)
          flat((b * out_h_ + oy) * out_w_ + ox, oc) = dy.values(b, (long(oc) * out_h_ + oy) * out_w_ + ox);
  const Matrix dp = core_.backward(flat, 1.0);
  Tensor dx;
  dx.dims = {in_c_, in_h_, in_w_};
  dx.values = Matrix(batch_, long(in_c_) * in_h_ * in_w_, 0.0);
  for (long b = 0; b < batch_; ++b)
    for (int oy = 0; oy < out_h_; ++oy)
      for (int ox = 0; ox < out_w_; ++ox) {
        const long r = (b * out_h_ + oy) * out_w_ + ox;
        for (int c = 0; c < in_c_; ++c)
          for (int ky = 0; ky < kernel_; ++ky)
            for (int kx = 0; kx < kernel_; ++kx) {
              const int iy = oy * stride_ + ky - padding_, ix = ox * stride_ + kx - padding_;
              if (iy < 0 || iy >= in_h_ || ix < 0 || ix >= in_w_) continue;
              dx.values(b, (long(c) * in_h_ + iy) * in_w_ + ix) += dp(r, (c * kernel_ + ky) * kernel_ + kx);
            }
      }
  return dx;
}

Tensor CrossbarLinear::forward(const Tensor& x, bool training) {
  Tensor y;
  y.values = core_.forward(x.values, training);
  y.dims = {core_.out_features()};
  return y;
}
Tensor CrossbarLinear::backward(const Tensor& dy) {
  Tensor dx;
  dx.values = core_.backward(dy.values, 1.0);
  dx.dims = {core_.in_features()};
  return dx;
}

// train.cpp:11-33
double softmax_cross_entropy(const Matrix& logits, const std::vector<int>& labels, Matrix& dlogits) {
  const long n = logits.rows, c = logits.cols;
  if (long(labels.size()) != n) throw std::invalid_argument("softmax_cross_entropy: label count mismatch");
  dlogits = Matrix(n, c);
  double total = 0.0;
  for (long i = 0; i < n; ++i) {
    double m = -std::numeric_limits<double>::infinity();
    for (long j = 0; j < c; ++j) m = std::max(m, logits(i, j));
    double z = 0.0;
    for (long j = 0; j < c; ++j) z += std::exp(logits(i, j) - m);
    const int y = labels[size_t(i)];
    total += -(logits(i, y) - m - std::log(z));
    for (long j = 0; j < c; ++j) {
      double p = std::exp(logits(i, j) - m) / z;
      dlogits(i, j) = (p - (j == y ? 1.0 : 0.0)) / double(n);
    }
  }
  return total / double(n);
}

// layers.cpp:510-522
Matrix relu_forward(const Matrix& x, Matrix& mask) {
  mask = Matrix(x.rows, x.cols);
  Matrix y(x.rows, x.cols);
  for (size_t k = 0; k < x.v.size(); ++k) {
    mask.v[k] = x.v[k] > 0.0 ? 1.0 : 0.0;
    y.v[k] = x.v[k] * mask.v[k];
  }
  return y;
}
Matrix relu_backward(const Matrix& dy, const Matrix& mask) {
  Matrix dx(dy.rows, dy.cols);
  for (size_t k = 0; k < dy.v.size(); ++k) dx.v[k] = dy.v[k] * mask.v[k];
  return dx;
}

// layers.cpp:524-563
Matrix maxpool2d_forward(const Matrix& x, int c, int h, int w, int kernel, int stride, std::vector<int>& arg) {
  if (kernel < 1 || stride < 1) throw std::invalid_argument("MaxPool2d: bad kernel/stride");
  const int oh = (h - kernel) / stride + 1, ow = (w - kernel) / stride + 1;
  const long batch = x.rows;
  Matrix y(batch, long(c) * oh * ow);
  arg.assign(size_t(batch * c * oh * ow), 0);
  for (long b = 0; b < batch; ++b)
    for (int ch = 0; ch < c; ++ch)
      for (int oy = 0; oy < oh; ++oy)
        for (int ox = 0; ox < ow; ++ox) {
          double best = -std::numeric_limits<double>::infinity();
          int best_idx = 0;
          for (int ky = 0; ky < kernel; ++ky)
            for (int kx = 0; kx < kernel; ++kx) {
              const int idx = (ch * h + oy * stride + ky) * w + ox * stride + kx;
              const double v = x(b, idx);
              if (v > best) {
                best = v;
                best_idx = idx;
              }
            }
          const long o = (long(ch) * oh + oy) * ow + ox;
          y(b, o) = best;
          arg[size_t(b * c * oh * ow + o)] = best_idx;
        }
  return y;
}

// layers.cpp:565-575
Matrix maxpool2d_backward(const Matrix& dy, int c, int h, int w, const std::vector<int>& arg) {
  Matrix dx(dy.rows, long(c) * h * w, 0.0);
  const long per = dy.cols;
  for (long b = 0; b < dy.rows; ++b)
    for (long o = 0; o < per; ++o) dx(b, arg[size_t(b * per + o)]) += dy(b, o);
  return dx;
}

}  // namespace orc
