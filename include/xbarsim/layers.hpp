// xbarsim/layers.hpp — the drop-in for the reference's
// proj/core/include/xbarsim/layers.hpp:19-134 (CrossbarLayerOptions,
// CrossbarCore, Layer, CrossbarLinear) over the C ABI in xbarsim_b200.h.
// Same namespaces, class and method names, argument meanings and exception
// types; Eigen::MatrixXd becomes xbarsim::MatrixXd (column-major fp64).
// Every call is synchronous at return, like the reference.  Beyond the
// reference surface: the *_device entry points (HBM pointers, async on the
// core's CUDA stream) for callers that keep activations on the GPU.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "xbarsim/converters.hpp"
#include "xbarsim/crossbar.hpp"
#include "xbarsim/engine.hpp"
#include "xbarsim/mapping.hpp"
#include "xbarsim/status.hpp"
#include "xbarsim/tensor.hpp"
#include "xbarsim/update.hpp"

namespace xbarsim::nn {

struct CrossbarLayerOptions {
  mapping::MappingSpec map;
  circuit::CrossbarConfig crossbar;
  converters::DacSpec dac;
  converters::AdcSpec adc;
  update::UpdateSpec update;
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

  /// Flat POD for the C ABI; pointers borrow this object's vectors.
  xbs_layer_options to_c() const {
    xbs_layer_options o;
    xbs_options_init(&o);
    o.weight_bits = map.weight_bits;
    o.device_bits = map.device_bits;
    o.tile_rows = map.tile_rows;
    o.tile_cols = map.tile_cols;
    o.variation_sigma = map.variation_sigma;
    o.variation_seed = map.seed;
    o.w_max = map.w_max;
    o.xbar_rows = crossbar.rows;
    o.xbar_cols = crossbar.cols;
    o.r_row = crossbar.r_row;
    o.r_col = crossbar.r_col;
    o.r_source = crossbar.r_source;
    o.r_sense = crossbar.r_sense;
    o.g_min = crossbar.g_min;
    o.g_max = crossbar.g_max;
    o.v_fs = crossbar.v_fs;
    o.dac_bits = dac.bits;
    o.dac_stream_bits = dac.stream_bits;
    o.dac_v_fs = dac.v_fs;
    o.dac_transfer = dac.transfer.empty() ? nullptr : dac.transfer.data();
    o.dac_transfer_len = static_cast<int32_t>(dac.transfer.size());
    o.adc_bits = adc.bits;
    o.adc_i_fs = adc.i_fs;
    o.adc_transfer = adc.transfer.empty() ? nullptr : adc.transfer.data();
    o.adc_transfer_len = static_cast<int32_t>(adc.transfer.size());
    o.adc_clip_percentile = adc.clip_percentile;
    o.upd_v = update.v;
    o.upd_gamma = update.gamma;
    o.upd_lr = update.lr;
    o.upd_seed = update.seed;
    o.upd_layer_scale = update.layer_scale;
    o.engine = static_cast<int32_t>(engine);
    o.interp_base = static_cast<int32_t>(interp_base);
    o.interp_interval = interp_interval;
    o.fcm_tol = fcm_tol;
    o.fcm_max_iter = fcm_max_iter;
    o.act_bits = act_bits;
    o.act_full_scale = act_full_scale;
    o.error_bits = error_bits;
    o.adc_cal_batches = adc_cal_batches;
    o.threads = threads;
    return o;
  }
};

/// reference layers.hpp:49-111 (layers.cpp:68-391).
class CrossbarCore {
 public:
  CrossbarCore(const MatrixXd& W0, const CrossbarLayerOptions& opt) {
    const xbs_layer_options o = opt.to_c();
    xbs_core* h = nullptr;
    detail::check(xbs_core_create(&o, W0.data(), W0.rows(), W0.cols(), W0.rows() > 0 ? W0.rows() : 1, &h));
    h_.reset(h);
  }

  MatrixXd forward(const MatrixXd& x, bool training) {
    MatrixXd y(x.rows(), out_features());
    detail::check(xbs_core_forward(h_.get(), x.data(), x.rows(), x.cols(), ld(x), training ? 1 : 0, y.data(), ld(y)));
    return y;
  }
  MatrixXd backward(const MatrixXd& dy, double grad_divisor) {
    MatrixXd dx(dy.rows(), in_features());
    detail::check(xbs_core_backward(h_.get(), dy.data(), dy.rows(), dy.cols(), ld(dy), grad_divisor, dx.data(), ld(dx)));
    grad_valid_ = false;
    return dx;
  }
  void apply_updates(std::uint64_t iteration) {
    detail::check(xbs_core_apply_updates(h_.get(), iteration));
    grad_valid_ = false;
  }

  int in_features() const { return info().in_features; }
  int out_features() const { return info().out_features; }
  mapping::TiledLayerWeights weights() const { return mapping::TiledLayerWeights(h_.get()); }
  const MatrixXd& gradient() const {
    if (!grad_valid_) {
      dW_.resize(in_features(), out_features());
      detail::check(xbs_core_gradient(h_.get(), dW_.data(), ld(dW_)));
      grad_valid_ = true;
    }
    return dW_;
  }
  long refresh_count() const { return static_cast<long>(info().refresh_count); }
  double conversion_seconds() const { return info().conversion_seconds; }
  double weight_abs_max_seen() const { return info().weight_abs_max_seen; }
  double grad_abs_max_seen() const { return info().grad_abs_max_seen; }
  double forward_adc_full_scale() const { return info().forward_adc_full_scale; }

  /// Snapped non-ideal conductances of tile (tr * grid_cols + tc).
  const MatrixXd& nonideal(int slice, mapping::Polarity p, int tile) const {
    const xbs_core_info i = info();  // tile dims = padded dims / grid
    tile_.resize(i.padded_rows / i.grid_rows, i.padded_cols / i.grid_cols);
    detail::check(xbs_core_nonideal(h_.get(), slice, static_cast<int32_t>(p), tile, tile_.data(), ld(tile_)));
    return tile_;
  }

  // ---- B200 extensions: device-resident calls (column-major, ld = M) ----
  void forward_device(const double* d_x, std::int64_t M, bool training, double* d_y) {
    detail::check(xbs_core_forward_device(h_.get(), d_x, M, training ? 1 : 0, d_y));
  }
  void backward_device(const double* d_dy, std::int64_t M, double grad_divisor, double* d_dx) {
    detail::check(xbs_core_backward_device(h_.get(), d_dy, M, grad_divisor, d_dx));
    grad_valid_ = false;
  }
  void apply_updates_device(std::uint64_t iteration) {
    detail::check(xbs_core_apply_updates_device(h_.get(), iteration));
    grad_valid_ = false;
  }
  void synchronize() { detail::check(xbs_core_synchronize(h_.get())); }
  /// Enqueue on the caller's cudaStream_t (nullptr: a private stream).
  void set_stream(void* stream) { detail::check(xbs_core_set_stream(h_.get(), stream)); }
  xbs_core* handle() const { return h_.get(); }

 private:
  struct Deleter {
    void operator()(xbs_core* c) const { xbs_core_destroy(c); }
  };
  static std::int64_t ld(const MatrixXd& m) { return m.rows() > 0 ? m.rows() : 1; }
  xbs_core_info info() const {
    xbs_core_info i{};
    detail::check(xbs_core_get_info(h_.get(), &i));
    return i;
  }
  std::unique_ptr<xbs_core, Deleter> h_;
  mutable MatrixXd dW_, tile_;
  mutable bool grad_valid_ = false;
};

/// reference layers.hpp:113-121
class Layer {
 public:
  virtual ~Layer() = default;
  virtual Tensor forward(const Tensor& x, bool training) = 0;
  virtual Tensor backward(const Tensor& dy) = 0;
  virtual void apply_updates(std::uint64_t /*iteration*/) {}
  virtual CrossbarCore* core() { return nullptr; }
  virtual std::string name() const = 0;
};

/// reference layers.hpp:123-134 (layers.cpp:393-413): grad_divisor 1.0.
class CrossbarLinear : public Layer {
 public:
  CrossbarLinear(const MatrixXd& W0, const CrossbarLayerOptions& opt) : core_(W0, opt) {}
  Tensor forward(const Tensor& x, bool training) override {
    Tensor y;
    y.values = core_.forward(x.values, training);
    y.dims = {core_.out_features()};
    return y;
  }
  Tensor backward(const Tensor& dy) override {
    Tensor dx;
    dx.values = core_.backward(dy.values, 1.0);
    dx.dims = {core_.in_features()};
    return dx;
  }
  void apply_updates(std::uint64_t iteration) override { core_.apply_updates(iteration); }
  CrossbarCore* core() override { return &core_; }
  std::string name() const override { return "linear"; }

 private:
  CrossbarCore core_;
};

}  // namespace xbarsim::nn
