// TEST INFRASTRUCTURE ONLY — flat C API over the REFERENCE ITSELF: the
// reference's own core sources (/root/reference/proj/core/src/*.cpp,
// unchanged) compiled against oracle/eigen_shim into oracle/_ref/libxbsref.so
// by oracle/ref/Makefile.  tests/test_ref_pin_cpu.py drives it through ctypes
// to pin the restated oracle (oracle/xbs_oracle.cpp, literal mode) to the
// reference's own code on the same inputs.  The options POD is the oracle
// C API's (xbs_oracle_capi.cpp), field for field.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "xbarsim/errors.hpp"
#include "xbarsim/layers.hpp"
#include "xbarsim/train.hpp"

extern "C" {
typedef struct ref_options {
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
} ref_options;
}

namespace {
using namespace xbarsim;
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const StateError& e) {
    g_err = e.what();
    return 2;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

nn::CrossbarLayerOptions convert(const ref_options& o) {
  nn::CrossbarLayerOptions r;
  r.map.weight_bits = o.weight_bits;
  r.map.device_bits = o.device_bits;
  r.map.tile_rows = o.tile_rows;
  r.map.tile_cols = o.tile_cols;
  r.map.variation_sigma = o.variation_sigma;
  r.map.seed = o.variation_seed;
  r.map.w_max = o.w_max;
  r.crossbar.rows = o.xbar_rows;
  r.crossbar.cols = o.xbar_cols;
  r.crossbar.r_row = o.r_row;
  r.crossbar.r_col = o.r_col;
  r.crossbar.r_source = o.r_source;
  r.crossbar.r_sense = o.r_sense;
  r.crossbar.g_min = o.g_min;
  r.crossbar.g_max = o.g_max;
  r.crossbar.v_fs = o.v_fs;
  r.dac.bits = o.dac_bits;
  r.dac.stream_bits = o.dac_stream_bits;
  r.dac.v_fs = o.dac_v_fs;
  if (o.dac_transfer_len > 0) r.dac.transfer.assign(o.dac_transfer, o.dac_transfer + o.dac_transfer_len);
  r.adc.bits = o.adc_bits;
  r.adc.i_fs = o.adc_i_fs;
  if (o.adc_transfer_len > 0) r.adc.transfer.assign(o.adc_transfer, o.adc_transfer + o.adc_transfer_len);
  r.adc.clip_percentile = o.adc_clip_percentile;
  r.update.v = o.upd_v;
  r.update.gamma = o.upd_gamma;
  r.update.lr = o.upd_lr;
  r.update.seed = o.upd_seed;
  r.update.layer_scale = o.upd_layer_scale;
  r.engine = static_cast<EngineKind>(o.engine);
  r.interp_base = static_cast<EngineKind>(o.interp_base);
  r.interp_interval = o.interp_interval;
  r.fcm_tol = o.fcm_tol;
  r.fcm_max_iter = o.fcm_max_iter;
  r.act_bits = o.act_bits;
  r.act_full_scale = o.act_full_scale;
  r.error_bits = o.error_bits;
  r.adc_cal_batches = o.adc_cal_batches;
  r.threads = o.threads;
  return r;
}

Eigen::MatrixXd wrap(const double* p, long r, long c) {
  Eigen::MatrixXd m(r, c);
  if (r * c) std::memcpy(m.data(), p, sizeof(double) * size_t(r * c));
  return m;
}
void unwrap(const Eigen::MatrixXd& m, double* out) {
  if (m.size()) std::memcpy(out, m.data(), sizeof(double) * size_t(m.size()));
}
nn::CrossbarCore* C(void* h) { return static_cast<nn::CrossbarCore*>(h); }
}  // namespace

extern "C" {
const char* ref_last_error() { return g_err.c_str(); }

int ref_core_create(const ref_options* o, const double* W, long K, long N, void** out) {
  return guard([&] { *out = new nn::CrossbarCore(wrap(W, K, N), convert(*o)); });
}
void ref_core_destroy(void* h) { delete C(h); }
int ref_core_forward(void* h, const double* x, long M, long K, int training, double* y) {
  return guard([&] { unwrap(C(h)->forward(wrap(x, M, K), training != 0), y); });
}
int ref_core_backward(void* h, const double* dy, long M, long N, double gd, double* dx) {
  return guard([&] { unwrap(C(h)->backward(wrap(dy, M, N), gd), dx); });
}
int ref_core_apply_updates(void* h, uint64_t it) {
  return guard([&] { C(h)->apply_updates(it); });
}
int ref_core_gradient(void* h, double* out) {
  return guard([&] { unwrap(C(h)->gradient(), out); });
}
int ref_core_nonideal(void* h, int s, int p, int t, double* out) {
  return guard([&] { unwrap(C(h)->nonideal(s, p == 0 ? mapping::Polarity::pos : mapping::Polarity::neg, t), out); });
}
int ref_core_master(void* h, int s, double* out) {
  return guard([&] { unwrap(C(h)->weights().master_diff(s), out); });
}
int ref_core_stats(void* h, double* out) {  // refresh count, |W| / |dW| maxima, forward ADC full scale
  return guard([&] {
    out[0] = double(C(h)->refresh_count());
    out[1] = C(h)->weight_abs_max_seen();
    out[2] = C(h)->grad_abs_max_seen();
    out[3] = C(h)->forward_adc_full_scale();
  });
}
int ref_softmax_ce(const double* logits, long n, long c, const int* labels, long nlab, double* dlogits,
                   double* loss) {
  return guard([&] {
    Eigen::MatrixXd d;
    *loss = nn::softmax_cross_entropy(wrap(logits, n, c), std::vector<int>(labels, labels + nlab), d);
    unwrap(d, dlogits);
  });
}
}  // extern "C"
