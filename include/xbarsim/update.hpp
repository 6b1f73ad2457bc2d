// xbarsim/update.hpp — UpdateSpec and the update free functions (reference
// update.hpp:13-52) over the C ABI.  update::apply_update changes the master
// only, on the device (update.cpp:43-88; the caller regenerates, as in the
// reference).  The elementwise helpers run the same device arithmetic as
// the fused core update (xbs_kernels.cu k_update).
#pragma once

#include <cstdint>
#include <stdexcept>

#include "xbarsim/crossbar.hpp"
#include "xbarsim/mapping.hpp"
#include "xbarsim/matrix.hpp"
#include "xbarsim/rng.hpp"
#include "xbarsim/status.hpp"

namespace xbarsim::update {

struct UpdateSpec {
  double v = 0.0;
  double gamma = 0.0;
  double lr = 0.01;
  std::uint64_t seed = 0;
  double layer_scale = 0.0;  // 0: the mapping's layer scale
  /// update.cpp:10-14
  void validate() const {
    if (v < 0) throw std::invalid_argument("UpdateSpec: v must be >= 0");
    if (gamma < 0) throw std::invalid_argument("UpdateSpec: gamma must be >= 0");
    if (!(lr > 0)) throw std::invalid_argument("UpdateSpec: lr must be > 0");
  }
};

/// update.cpp:16-24
inline MatrixXd scale_gradient(const MatrixXd& dW, const UpdateSpec& spec, const circuit::CrossbarConfig& cfg) {
  MatrixXd out(dW.rows(), dW.cols());
  const std::int64_t ld = dW.rows() > 0 ? dW.rows() : 1;
  detail::check(
      xbs_scale_gradient(dW.data(), dW.rows(), dW.cols(), ld, spec.layer_scale, cfg.g_min, cfg.g_max, out.data(), ld));
  return out;
}

/// update.cpp:26-33
inline double nonlinear_update(double g, double dg_ideal, const UpdateSpec& spec, const circuit::CrossbarConfig& cfg) {
  double out = 0.0;
  detail::check(xbs_nonlinear_update(&g, &dg_ideal, 1, spec.v, cfg.g_min, cfg.g_max, &out));
  return out;
}

/// update.cpp:35-41: draws one Gaussian from rng unless the deviation is 0.
inline double write_noise(double dg_ideal, const UpdateSpec& spec, const circuit::CrossbarConfig& cfg,
                          CounterRng& rng) {
  const std::uint64_t key = rng.key(), ctr = rng.counter();
  double out = 0.0;
  std::int32_t drew = 0;
  detail::check(xbs_write_noise(&dg_ideal, 1, spec.gamma, cfg.g_min, cfg.g_max, &key, &ctr, &out, &drew));
  if (drew) rng.advance(2);
  return out;
}

/// update.cpp:43-88: the master of t only (the caller regenerates).
inline void apply_update(mapping::TiledLayerWeights& t, const MatrixXd& dW, const UpdateSpec& spec,
                         std::uint64_t iteration) {
  const xbs_update_spec s{spec.v, spec.gamma, spec.lr, spec.seed, spec.layer_scale};
  detail::check(
      xbs_apply_update(t.handle(), dW.data(), dW.rows(), dW.cols(), dW.rows() > 0 ? dW.rows() : 1, &s, iteration));
}

}  // namespace xbarsim::update
