// TEST INFRASTRUCTURE ONLY — flat C API over the CPU oracle so the Python
// parity tests (tests/) and bench.py's cpu_baseline leg can drive it through
// ctypes.  The options POD mirrors include/xbarsim_b200.h's xbs_layer_options
// field for field (same order, same types) so one Python dataclass fills both.
#include <cstring>
#include <memory>
#include <string>

#include "xbs_oracle.hpp"

extern "C" {

typedef struct orc_options {
  int32_t weight_bits, device_bits, tile_rows, tile_cols;
  double variation_sigma;
  uint64_t variation_seed;
  double w_max;
  int32_t xbar_rows, xbar_cols;
  double r_row, r_col, r_source, r_sense, g_min, g_max, v_fs;
  int32_t dac_bits, dac_stream_bits;
  double dac_v_fs;
  const double* dac_transfer;
  int32_t dac_transfer_len;
  int32_t adc_bits;
  double adc_i_fs;
  const double* adc_transfer;
  int32_t adc_transfer_len;
  double adc_clip_percentile;
  double upd_v, upd_gamma, upd_lr;
  uint64_t upd_seed;
  double upd_layer_scale;
  int32_t engine, interp_base, interp_interval;
  double fcm_tol;
  int32_t fcm_max_iter;
  int32_t act_bits;
  double act_full_scale;
  int32_t error_bits, adc_cal_batches, threads;
} orc_options;

}  // extern "C"

namespace {
thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 StateError, 3 ConfigError, 9 other
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const orc::StateError& e) {
    g_err = e.what();
    return 2;
  } catch (const orc::ConfigError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

orc::CrossbarLayerOptions to_opts(const orc_options* o, int snapped) {
  orc::CrossbarLayerOptions r;
  r.map.weight_bits = o->weight_bits;
  r.map.device_bits = o->device_bits;
  r.map.tile_rows = o->tile_rows;
  r.map.tile_cols = o->tile_cols;
  r.map.variation_sigma = o->variation_sigma;
  r.map.seed = o->variation_seed;
  r.map.w_max = o->w_max;
  r.crossbar.rows = o->xbar_rows;
  r.crossbar.cols = o->xbar_cols;
  r.crossbar.r_row = o->r_row;
  r.crossbar.r_col = o->r_col;
  r.crossbar.r_source = o->r_source;
  r.crossbar.r_sense = o->r_sense;
  r.crossbar.g_min = o->g_min;
  r.crossbar.g_max = o->g_max;
  r.crossbar.v_fs = o->v_fs;
  r.dac.bits = o->dac_bits;
  r.dac.stream_bits = o->dac_stream_bits;
  r.dac.v_fs = o->dac_v_fs;
  if (o->dac_transfer && o->dac_transfer_len > 0)
    r.dac.transfer.assign(o->dac_transfer, o->dac_transfer + o->dac_transfer_len);
  r.adc.bits = o->adc_bits;
  r.adc.i_fs = o->adc_i_fs;
  if (o->adc_transfer && o->adc_transfer_len > 0)
    r.adc.transfer.assign(o->adc_transfer, o->adc_transfer + o->adc_transfer_len);
  r.adc.clip_percentile = o->adc_clip_percentile;
  r.update.v = o->upd_v;
  r.update.gamma = o->upd_gamma;
  r.update.lr = o->upd_lr;
  r.update.seed = o->upd_seed;
  r.update.layer_scale = o->upd_layer_scale;
  r.engine = orc::EngineKind(o->engine);
  r.interp_base = orc::EngineKind(o->interp_base);
  r.interp_interval = o->interp_interval;
  r.fcm_tol = o->fcm_tol;
  r.fcm_max_iter = o->fcm_max_iter;
  r.act_bits = o->act_bits;
  r.act_full_scale = o->act_full_scale;
  r.error_bits = o->error_bits;
  r.adc_cal_batches = o->adc_cal_batches;
  r.threads = o->threads;
  r.snapped = snapped != 0;
  return r;
}

orc::Matrix wrap(const double* p, long r, long c) {
  orc::Matrix m(r, c);
  if (r * c != 0) std::memcpy(m.data(), p, sizeof(double) * size_t(r * c));
  return m;
}
void unwrap(const orc::Matrix& m, double* out) {
  if (m.size()) std::memcpy(out, m.data(), sizeof(double) * m.size());
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

int orc_core_create(const orc_options* o, int snapped, const double* W, long K, long N, void** out) {
  return guard([&] { *out = new orc::CrossbarCore(wrap(W, K, N), to_opts(o, snapped)); });
}
// Sampled construction: only `tiles` are converted (now and at every
// regeneration); forward_tiles / backward_tiles must stay inside them.
int orc_core_create_tiles(const orc_options* o, int snapped, const double* W, long K, long N, const int* tiles, int n,
                          void** out) {
  return guard([&] {
    const std::vector<int> t(tiles, tiles + n);
    *out = new orc::CrossbarCore(wrap(W, K, N), to_opts(o, snapped), &t);
  });
}
void orc_core_destroy(void* h) { delete static_cast<orc::CrossbarCore*>(h); }

// CrossbarConv2d (layers.cpp:415-505); x: batch x (c*h*w) column-major
int orc_conv2d_create(const orc_options* o, int snapped, const double* W, long K, long N, int in_c, int out_c,
                      int kernel, int stride, int padding, void** out) {
  return guard([&] {
    *out = new orc::CrossbarConv2d(wrap(W, K, N), in_c, out_c, kernel, stride, padding, to_opts(o, snapped));
  });
}
void orc_conv2d_destroy(void* h) { delete static_cast<orc::CrossbarConv2d*>(h); }
int orc_conv2d_forward(void* h, const double* x, long batch, int c, int hh, int ww, int training, double* y,
                       int* dims3) {
  return guard([&] {
    orc::Tensor t;
    t.values = wrap(x, batch, long(c) * hh * ww);
    t.dims = {c, hh, ww};
    orc::Tensor r = static_cast<orc::CrossbarConv2d*>(h)->forward(t, training != 0);
    for (int k = 0; k < 3; ++k) dims3[k] = r.dims[size_t(k)];
    if (y) unwrap(r.values, y);
  });
}
int orc_conv2d_backward(void* h, const double* dy, long batch, long feat, double* dx) {
  return guard([&] {
    orc::Tensor t;
    t.values = wrap(dy, batch, feat);
    unwrap(static_cast<orc::CrossbarConv2d*>(h)->backward(t).values, dx);
  });
}
int orc_conv2d_apply_updates(void* h, uint64_t it) {
  return guard([&] { static_cast<orc::CrossbarConv2d*>(h)->apply_updates(it); });
}
void* orc_conv2d_core(void* h) { return static_cast<orc::CrossbarConv2d*>(h)->core(); }


static orc::CrossbarCore* C(void* h) { return static_cast<orc::CrossbarCore*>(h); }

int orc_core_forward(void* h, const double* x, long M, long K, int training, double* y) {
  return guard([&] { unwrap(C(h)->forward(wrap(x, M, K), training != 0), y); });
}
int orc_core_forward_tiles(void* h, const double* x, long M, long K, int training, const int* tcs, int n,
                           double* y) {
  return guard([&] {
    unwrap(C(h)->forward_tiles(wrap(x, M, K), training != 0, std::vector<int>(tcs, tcs + n)), y);
  });
}
int orc_core_backward(void* h, const double* dy, long M, long N, double gd, double* dx) {
  return guard([&] { unwrap(C(h)->backward(wrap(dy, M, N), gd), dx); });
}
int orc_core_backward_tiles(void* h, const double* dy, long M, long N, double gd, const int* trs, int n,
                            int compute_dw, double* dx) {
  return guard([&] {
    unwrap(C(h)->backward_tiles(wrap(dy, M, N), gd, std::vector<int>(trs, trs + n), compute_dw != 0), dx);
  });
}
int orc_core_apply_updates(void* h, uint64_t it) {
  return guard([&] { C(h)->apply_updates(it); });
}
int orc_core_gradient(void* h, double* out) {
  return guard([&] { unwrap(C(h)->gradient(), out); });
}
int orc_core_set_gradient(void* h, const double* dW) {
  return guard([&] {
    const auto& w = C(h)->weights();
    C(h)->set_gradient(wrap(dW, w.rows(), w.cols()));
  });
}
int orc_core_nonideal(void* h, int s, int p, int t, double* out) {
  return guard([&] { unwrap(C(h)->nonideal(s, p ? orc::Polarity::neg : orc::Polarity::pos, t), out); });
}
int orc_core_set_nonideal(void* h, int s, int p, int t, const double* g) {
  return guard([&] {
    const auto& w = C(h)->weights();
    C(h)->set_nonideal(s, p ? orc::Polarity::neg : orc::Polarity::pos, t,
                       wrap(g, w.spec().tile_rows, w.spec().tile_cols));
  });
}
int orc_core_master(void* h, int s, double* out) {
  return guard([&] { unwrap(C(h)->weights().master_diff(s), out); });
}
int orc_core_set_master(void* h, int s, const double* u) {
  return guard([&] {
    auto& m = C(h)->mutable_weights().mutable_master_diff(s);
    std::memcpy(m.data(), u, sizeof(double) * m.size());
  });
}
int orc_core_implied_weights(void* h, double* out) {
  return guard([&] { unwrap(C(h)->weights().implied_weights(), out); });
}
int orc_core_regenerate(void* h, const int* tiles, int n) {
  return guard([&] {
    C(h)->regen_tiles.assign(tiles, tiles + n);
    C(h)->regenerate();
  });
}
// geometry: rows, cols, grid_rows, grid_cols, padded_rows, padded_cols, slices, snap_e
int orc_core_geometry(void* h, long* out8) {
  return guard([&] {
    const auto& w = C(h)->weights();
    out8[0] = w.rows();
    out8[1] = w.cols();
    out8[2] = w.grid_rows();
    out8[3] = w.grid_cols();
    out8[4] = w.padded_rows();
    out8[5] = w.padded_cols();
    out8[6] = w.num_slices();
    out8[7] = C(h)->snap_e();
  });
}
// stats: layer_scale, wmax_seen, dwmax_seen, fwd i_fs, bwd i_fs, refresh_count, level_step
int orc_core_stats(void* h, double* out7) {
  return guard([&] {
    auto* c = C(h);
    out7[0] = c->weights().layer_scale();
    out7[1] = c->weight_abs_max_seen();
    out7[2] = c->grad_abs_max_seen();
    out7[3] = c->forward_adc_full_scale();
    out7[4] = c->backward_adc_full_scale();
    out7[5] = double(c->refresh_count());
    out7[6] = c->weights().level_step();
  });
}
int orc_core_record_codes(void* h, int on) {
  C(h)->record_codes = on != 0;
  return 0;
}
long orc_core_last_codes(void* h, uint16_t* out, long cap) {
  const auto& v = C(h)->last_codes;
  long n = long(v.size());
  if (out && cap > 0) std::memcpy(out, v.data(), sizeof(uint16_t) * size_t(std::min(n, cap)));
  return n;
}

// ---- free functions used by the KAT / pin tests
void orc_rng_draws(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, long n, uint64_t* out) {
  orc::CounterRng r(seed, a, b, c);
  for (long i = 0; i < n; ++i) out[i] = r.next();
}
double orc_rng_gaussian(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  orc::CounterRng r(seed, a, b, c);
  return r.gaussian();
}
int orc_snap_exponent(double g_max) { return orc::snap_exponent(g_max); }
int orc_adc_quantize(double i, int bits, double i_fs, uint64_t* code) {
  return guard([&] {
    orc::AdcSpec s;
    s.bits = bits;
    s.i_fs = i_fs;
    *code = orc::adc_quantize(i, s);
  });
}
int orc_aam_convert(int rows, int cols, double r_row, double r_col, double r_source, double r_sense,
                    const double* g, double* out) {
  return guard([&] {
    orc::CrossbarConfig cfg;
    cfg.rows = rows;
    cfg.cols = cols;
    cfg.r_row = r_row;
    cfg.r_col = r_col;
    cfg.r_source = r_source;
    cfg.r_sense = r_sense;
    unwrap(orc::aam_convert(cfg, wrap(g, rows, cols)), out);
  });
}
// Step glue of the reference's training loop (train.cpp:11-33,
// layers.cpp:510-575), column-major batch x features like every matrix here.
int orc_softmax_ce(const double* logits, long n, long c, const int* labels, long nlab, double* dlogits,
                   double* loss) {
  return guard([&] {
    orc::Matrix d;
    *loss = orc::softmax_cross_entropy(wrap(logits, n, c), std::vector<int>(labels, labels + nlab), d);
    unwrap(d, dlogits);
  });
}
int orc_relu(const double* x, long n, long f, const double* dy, double* y, double* dx) {
  return guard([&] {
    orc::Matrix mask;
    unwrap(orc::relu_forward(wrap(x, n, f), mask), y);
    unwrap(orc::relu_backward(wrap(dy, n, f), mask), dx);
  });
}
int orc_maxpool2d(const double* x, long n, int c, int h, int w, int kernel, int stride, const double* dy, double* y,
                  double* dx) {
  return guard([&] {
    std::vector<int> arg;
    const orc::Matrix ym = orc::maxpool2d_forward(wrap(x, n, long(c) * h * w), c, h, w, kernel, stride, arg);
    unwrap(ym, y);
    unwrap(orc::maxpool2d_backward(wrap(dy, n, ym.cols), c, h, w, arg), dx);
  });
}
// ADC-calibrator quantile over a sample (converters.cpp:96-107) -- used to
// pick the explicit i_fs each parity config pins.
double orc_calibrate(const double* samples, long n, double pct) {
  orc::AdcCalibrator c;
  for (long i = 0; i < n; ++i) c.observe(samples[i]);
  return c.calibrate(pct);
}

}  // extern "C"
