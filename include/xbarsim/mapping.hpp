// xbarsim/mapping.hpp — Polarity, MappingSpec (reference mapping.hpp:12-25)
// and a read-through TiledLayerWeights (mapping.hpp:39-89) over a device-
// resident core: the master lives in HBM, so the accessors copy it out on
// call and return by value (a const& binding still works).
#pragma once

#include <cstdint>

#include "xbarsim/matrix.hpp"
#include "xbarsim/status.hpp"

namespace xbarsim::mapping {

enum class Polarity { pos = 0, neg = 1 };

struct MappingSpec {
  int weight_bits = 8;
  int device_bits = 2;
  int tile_rows = 64;
  int tile_cols = 64;
  double variation_sigma = 0.0;
  std::uint64_t seed = 0;
  double w_max = 0.0;
  int num_slices() const { return weight_bits / device_bits; }
};

class TiledLayerWeights {
 public:
  explicit TiledLayerWeights(xbs_core* core) : core_(core) {}
  int rows() const { return info().in_features; }
  int cols() const { return info().out_features; }
  int padded_rows() const { return info().padded_rows; }
  int padded_cols() const { return info().padded_cols; }
  int grid_rows() const { return info().grid_rows; }
  int grid_cols() const { return info().grid_cols; }
  int num_slices() const { return info().num_slices; }
  double layer_scale() const { return info().layer_scale; }
  double level_step() const { return info().level_step; }
  /// Signed differential master of one slice (padded dims).
  MatrixXd master_diff(int slice) const {
    const xbs_core_info i = info();
    MatrixXd u(i.padded_rows, i.padded_cols);
    detail::check(xbs_core_master(core_, slice, u.data(), u.rows()));
    return u;
  }
  void set_master_diff(int slice, const MatrixXd& u) {
    detail::check(xbs_core_set_master(core_, slice, u.data(), u.rows()));
  }
  /// mapping.cpp:70-81
  MatrixXd implied_weights() const {
    const xbs_core_info i = info();
    MatrixXd w(i.in_features, i.out_features);
    detail::check(xbs_core_implied_weights(core_, w.data(), w.rows()));
    return w;
  }

 private:
  xbs_core_info info() const {
    xbs_core_info i{};
    detail::check(xbs_core_get_info(core_, &i));
    return i;
  }
  xbs_core* core_;
};

}  // namespace xbarsim::mapping
