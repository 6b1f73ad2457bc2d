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
#include "xbarsim/rng.hpp"
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

  /// layers.cpp:17-47 (the reference's checks and exception classes)
  void validate() const {
    const xbs_layer_options o = to_c();
    detail::check(xbs_options_validate(&o));
  }

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

namespace core_detail {
struct CoreDeleter {
  bool owns = true;  // false: a view of a core owned by a CrossbarConv2d
  void operator()(xbs_core* c) const {
    if (owns) xbs_core_destroy(c);
  }
};
}  // namespace core_detail

/// reference layers.hpp:49-111 (layers.cpp:68-391).
class CrossbarCore {
 public:
  CrossbarCore(const MatrixXd& W0, const CrossbarLayerOptions& opt) {
    const xbs_layer_options o = opt.to_c();
    xbs_core* h = nullptr;
    detail::check(xbs_core_create(&o, W0.data(), W0.rows(), W0.cols(), W0.rows() > 0 ? W0.rows() : 1, &h));
    h_.reset(h);
  }
  /// View of a core owned by another object (CrossbarConv2d's core).
  static CrossbarCore borrow(xbs_core* h) { return CrossbarCore(h); }

  MatrixXd forward(const MatrixXd& x, bool training) {
    MatrixXd y(x.rows(), out_features());
    detail::check(xbs_core_forward(h_.get(), x.data(), x.rows(), x.cols(), ld(x), training ? 1 : 0, y.data(), ld(y)));
    return y;
  }
  MatrixXd backward(const MatrixXd& dy, double grad_divisor) {
    MatrixXd dx(dy.rows(), in_features());
    detail::check(xbs_core_backward(h_.get(), dy.data(), dy.rows(), dy.cols(), ld(dy), grad_divisor, dx.data(), ld(dx)));
    return dx;
  }
  void apply_updates(std::uint64_t iteration) {
    detail::check(xbs_core_apply_updates(h_.get(), iteration));
  }

  int in_features() const { return info().in_features; }
  int out_features() const { return info().out_features; }
  mapping::TiledLayerWeights weights() const { return mapping::TiledLayerWeights(h_.get()); }
  /// Fetched on every call: a conv layer, set_gradient or a raw handle()
  /// caller can replace dW behind this wrapper's back.  The reference stays
  /// valid until the next mutating call; this copy until the next gradient().
  const MatrixXd& gradient() const {
    dW_.resize(in_features(), out_features());
    detail::check(xbs_core_gradient(h_.get(), dW_.data(), ld(dW_)));
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
  }
  void apply_updates_device(std::uint64_t iteration) {
    detail::check(xbs_core_apply_updates_device(h_.get(), iteration));
  }
  void synchronize() { detail::check(xbs_core_synchronize(h_.get())); }
  /// Enqueue on the caller's cudaStream_t (nullptr: a private stream).
  void set_stream(void* stream) { detail::check(xbs_core_set_stream(h_.get(), stream)); }
  xbs_core* handle() const { return h_.get(); }

 private:
  explicit CrossbarCore(xbs_core* borrowed) : h_(borrowed, core_detail::CoreDeleter{false}) {}
  static std::int64_t ld(const MatrixXd& m) { return m.rows() > 0 ? m.rows() : 1; }
  xbs_core_info info() const {
    xbs_core_info i{};
    detail::check(xbs_core_get_info(h_.get(), &i));
    return i;
  }
  std::unique_ptr<xbs_core, core_detail::CoreDeleter> h_;
  mutable MatrixXd dW_, tile_;
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

/// reference layers.hpp:136-152 (layers.cpp:415-505): im2col lowering onto
/// one core, done on the device; features ordered (c, y, x).
class CrossbarConv2d : public Layer {
 public:
  CrossbarConv2d(const MatrixXd& W0, int in_c, int out_c, int kernel, int stride, int padding,
                 const CrossbarLayerOptions& opt)
      : h_(make(W0, in_c, out_c, kernel, stride, padding, opt)), core_(CrossbarCore::borrow(xbs_conv2d_core(h_.get()))) {}
  Tensor forward(const Tensor& x, bool training) override {
    if (x.dims.size() != 3) throw std::invalid_argument("CrossbarConv2d: expected (c, h, w) input");
    std::int32_t oh = 0, ow = 0;
    detail::check(xbs_conv2d_output_dims(h_.get(), x.dims[1], x.dims[2], &oh, &ow));
    Tensor y;
    y.values.resize(x.values.rows(), static_cast<MatrixXd::Index>(core_.out_features()) * oh * ow);
    detail::check(xbs_conv2d_forward(h_.get(), x.values.data(), x.values.rows(), x.dims[0], x.dims[1], x.dims[2],
                                     ld(x.values), training ? 1 : 0, y.values.data(), ld(y.values)));
    y.dims = {core_.out_features(), oh, ow};
    in_dims_ = x.dims;
    return y;
  }
  Tensor backward(const Tensor& dy) override {
    Tensor dx;
    if (in_dims_.size() != 3) throw StateError("CrossbarConv2d::backward before forward");
    dx.values.resize(dy.values.rows(), static_cast<MatrixXd::Index>(in_dims_[0]) * in_dims_[1] * in_dims_[2]);
    detail::check(xbs_conv2d_backward(h_.get(), dy.values.data(), dy.values.rows(), ld(dy.values), dx.values.data(),
                                      ld(dx.values)));
    dx.dims = in_dims_;
    return dx;
  }
  void apply_updates(std::uint64_t iteration) override { detail::check(xbs_conv2d_apply_updates(h_.get(), iteration)); }
  CrossbarCore* core() override { return &core_; }
  std::string name() const override { return "conv2d"; }

 private:
  struct Deleter {
    void operator()(xbs_conv2d* c) const { xbs_conv2d_destroy(c); }
  };
  static xbs_conv2d* make(const MatrixXd& W0, int in_c, int out_c, int kernel, int stride, int padding,
                          const CrossbarLayerOptions& opt) {
    if (W0.rows() != static_cast<MatrixXd::Index>(in_c) * kernel * kernel || W0.cols() != out_c)
      throw std::invalid_argument("CrossbarConv2d: kernel matrix must be (in_c*k*k) x out_c");
    const xbs_layer_options o = opt.to_c();
    xbs_conv2d* h = nullptr;
    detail::check(xbs_conv2d_create(&o, W0.data(), W0.rows() > 0 ? W0.rows() : 1, in_c, out_c, kernel, stride, padding,
                                    &h));
    return h;
  }
  static std::int64_t ld(const MatrixXd& m) { return m.rows() > 0 ? m.rows() : 1; }
  std::unique_ptr<xbs_conv2d, Deleter> h_;
  CrossbarCore core_;
  std::vector<int> in_dims_;
};

}  // namespace xbarsim::nn
