// xbarsim/mapping.hpp — Polarity, MappingSpec and TiledLayerWeights
// (reference mapping.hpp:12-109) over the C ABI.  The master lives in HBM
// (an xbs_weights handle): map_weights() owns one, CrossbarCore::weights()
// is a view of the core's.  master_diff() copies a slice out into a host
// mirror and returns a reference to it; mutable_master_diff() hands out the
// mirror for editing and writes it back before the next device operation on
// these weights (value semantics as in the reference; copies are deep).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <vector>

#include "xbarsim/crossbar.hpp"
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

class TiledLayerWeights;
TiledLayerWeights map_weights(const MatrixXd& W, const MappingSpec& spec, const circuit::CrossbarConfig& cfg);
TiledLayerWeights apply_variation(const TiledLayerWeights& t, double sigma, std::uint64_t seed);

class TiledLayerWeights {
 public:
  /// View of a core's weights (CrossbarCore::weights()).
  explicit TiledLayerWeights(xbs_core* core) {
    xbs_weights* w = nullptr;
    detail::check(xbs_core_weights(core, &w));
    h_.reset(w, xbs_weights_destroy);
  }
  TiledLayerWeights(const TiledLayerWeights& o) { *this = o; }
  TiledLayerWeights& operator=(const TiledLayerWeights& o) {
    if (this == &o) return *this;
    o.flush();
    if (o.is_view()) {  // a view stays a view of the same core
      h_ = o.h_;
    } else {            // value semantics: a deep copy of the master
      const xbs_weights_info i = o.info();
      xbs_weights* w = nullptr;
      detail::check(xbs_weights_apply_variation(o.h_.get(), i.variation_sigma, i.variation_seed, &w));
      h_.reset(w, xbs_weights_destroy);
    }
    view_ = o.view_;
    mirror_.clear();
    dirty_.clear();
    return *this;
  }
  TiledLayerWeights(TiledLayerWeights&&) = default;
  TiledLayerWeights& operator=(TiledLayerWeights&&) = default;

  int rows() const { return info().rows; }
  int cols() const { return info().cols; }
  int padded_rows() const { return info().padded_rows; }
  int padded_cols() const { return info().padded_cols; }
  int grid_rows() const { return info().grid_rows; }
  int grid_cols() const { return info().grid_cols; }
  int num_slices() const { return info().num_slices; }
  double layer_scale() const { return info().layer_scale; }
  double level_step() const { return info().level_step; }
  double variation_sigma() const { return info().variation_sigma; }
  std::uint64_t variation_seed() const { return info().variation_seed; }
  MappingSpec spec() const {
    const xbs_weights_info i = info();
    MappingSpec s;
    s.weight_bits = i.weight_bits;
    s.device_bits = i.device_bits;
    s.tile_rows = i.tile_rows;
    s.tile_cols = i.tile_cols;
    s.variation_sigma = i.variation_sigma;
    s.seed = i.variation_seed;
    s.w_max = i.layer_scale;
    return s;
  }

  /// Signed differential master of one slice (padded dims), mapping.hpp:55.
  const MatrixXd& master_diff(int slice) const {
    MatrixXd& m = mirror(slice);
    if (!dirty_[static_cast<size_t>(slice)]) fetch(slice, m);
    return m;
  }
  /// mapping.hpp:56: edits are written back before the next device use.
  MatrixXd& mutable_master_diff(int slice) {
    MatrixXd& m = mirror(slice);
    if (!dirty_[static_cast<size_t>(slice)]) fetch(slice, m);
    dirty_[static_cast<size_t>(slice)] = true;
    return m;
  }
  /// For a core view: writes one slice and regenerates the core.
  void set_master_diff(int slice, const MatrixXd& u) {
    flush();
    detail::check(xbs_weights_set_master(h_.get(), slice, u.data(), ld(u)));
    if (static_cast<size_t>(slice) < mirror_.size()) dirty_[static_cast<size_t>(slice)] = false;
  }
  /// mapping.cpp:39-45
  MatrixXd master_polarity(int slice, Polarity p) const { return padded(slice, p, xbs_weights_master_polarity); }
  /// mapping.cpp:47-58 (variation from the counter RNG, on the device)
  MatrixXd ideal_working(int slice, Polarity p) const { return padded(slice, p, xbs_weights_ideal_working); }
  /// mapping.cpp:60-68: one working tile with tile-sized geometry.
  circuit::ConductanceTile ideal_tile(int slice, Polarity p, int tr, int tc) const {
    const xbs_weights_info i = info();
    if (tr < 0 || tr >= i.grid_rows || tc < 0 || tc >= i.grid_cols)
      throw std::invalid_argument("TiledLayerWeights: tile index out of range");
    const MatrixXd w = ideal_working(slice, p);
    circuit::ConductanceTile t;
    t.config.rows = i.tile_rows;
    t.config.cols = i.tile_cols;
    t.config.g_min = i.g_min;
    t.config.g_max = i.g_max;
    t.g = MatrixXd(i.tile_rows, i.tile_cols);
    for (int c = 0; c < i.tile_cols; ++c)
      for (int r = 0; r < i.tile_rows; ++r) t.g(r, c) = w(std::int64_t(tr) * i.tile_rows + r, std::int64_t(tc) * i.tile_cols + c);
    return t;
  }
  /// mapping.cpp:70-81
  MatrixXd implied_weights() const {
    flush();
    const xbs_weights_info i = info();
    MatrixXd w(i.rows, i.cols);
    detail::check(xbs_weights_implied(h_.get(), w.data(), i.rows > 0 ? i.rows : 1));
    return w;
  }

  /// The C handle, with pending mutable_master_diff edits written back.
  xbs_weights* handle() const {
    flush();
    return h_.get();
  }
  bool is_view() const { return view_; }

 private:
  friend TiledLayerWeights map_weights(const MatrixXd&, const MappingSpec&, const circuit::CrossbarConfig&);
  friend TiledLayerWeights apply_variation(const TiledLayerWeights&, double, std::uint64_t);
  TiledLayerWeights(xbs_weights* owned, bool) : h_(owned, xbs_weights_destroy), view_(false) {}
  xbs_weights_info info() const {
    xbs_weights_info i{};
    detail::check(xbs_weights_get_info(h_.get(), &i));
    return i;
  }
  static std::int64_t ld(const MatrixXd& m) { return m.rows() > 0 ? m.rows() : 1; }
  MatrixXd& mirror(int slice) const {
    const int S = num_slices();
    if (slice < 0 || slice >= S) throw std::out_of_range("TiledLayerWeights: slice out of range");
    if (mirror_.size() != static_cast<size_t>(S)) {
      mirror_.assign(static_cast<size_t>(S), MatrixXd());
      dirty_.assign(static_cast<size_t>(S), false);
    }
    return mirror_[static_cast<size_t>(slice)];
  }
  void fetch(int slice, MatrixXd& m) const {
    const xbs_weights_info i = info();
    m.resize(i.padded_rows, i.padded_cols);
    detail::check(xbs_weights_master(h_.get(), slice, m.data(), ld(m)));
  }
  void flush() const {
    for (size_t s = 0; s < dirty_.size(); ++s)
      if (dirty_[s]) {
        detail::check(xbs_weights_set_master(h_.get(), static_cast<int>(s), mirror_[s].data(), ld(mirror_[s])));
        dirty_[s] = false;
      }
  }
  template <class F>
  MatrixXd padded(int slice, Polarity p, F fn) const {
    flush();
    const xbs_weights_info i = info();
    MatrixXd g(i.padded_rows, i.padded_cols);
    detail::check(fn(h_.get(), slice, static_cast<int32_t>(p), g.data(), ld(g)));
    return g;
  }

  std::shared_ptr<xbs_weights> h_;
  bool view_ = true;
  mutable std::vector<MatrixXd> mirror_;
  mutable std::vector<bool> dirty_;
};

namespace detail_map {
inline xbs_layer_options options(const MappingSpec& spec, const circuit::CrossbarConfig& cfg) {
  xbs_layer_options o;
  xbs_options_init(&o);
  o.weight_bits = spec.weight_bits;
  o.device_bits = spec.device_bits;
  o.tile_rows = spec.tile_rows;
  o.tile_cols = spec.tile_cols;
  o.variation_sigma = spec.variation_sigma;
  o.variation_seed = spec.seed;
  o.w_max = spec.w_max;
  o.xbar_rows = cfg.rows;
  o.xbar_cols = cfg.cols;
  o.r_row = cfg.r_row;
  o.r_col = cfg.r_col;
  o.r_source = cfg.r_source;
  o.r_sense = cfg.r_sense;
  o.g_min = cfg.g_min;
  o.g_max = cfg.g_max;
  o.v_fs = cfg.v_fs;
  return o;
}
}  // namespace detail_map

/// mapping.cpp:83-131, on the device.
inline TiledLayerWeights map_weights(const MatrixXd& W, const MappingSpec& spec, const circuit::CrossbarConfig& cfg) {
  const xbs_layer_options o = detail_map::options(spec, cfg);
  xbs_weights* w = nullptr;
  detail::check(xbs_map_weights(&o, W.data(), W.rows(), W.cols(), W.rows() > 0 ? W.rows() : 1, &w));
  return TiledLayerWeights(w, true);
}

/// mapping.cpp:133-140: a copy with new variation parameters.
inline TiledLayerWeights apply_variation(const TiledLayerWeights& t, double sigma, std::uint64_t seed) {
  xbs_weights* w = nullptr;
  detail::check(xbs_weights_apply_variation(t.handle(), sigma, seed, &w));
  return TiledLayerWeights(w, true);
}

/// mapping.cpp:142-160: scale * sum_s 2^(s*device_bits) (pos[s] - neg[s]).
inline VectorXd reconstruct_output(const std::vector<VectorXd>& codes_pos, const std::vector<VectorXd>& codes_neg,
                                   const MappingSpec& spec, double scale) {
  const size_t slices = static_cast<size_t>(spec.num_slices());
  if (codes_pos.size() != slices || codes_neg.size() != slices)
    throw std::invalid_argument("reconstruct_output: need codes for every slice");
  const VectorXd::Index n = codes_pos.empty() ? 0 : codes_pos[0].size();
  for (size_t s = 0; s < slices; ++s)
    if (codes_pos[s].size() != n || codes_neg[s].size() != n)
      throw std::invalid_argument("reconstruct_output: inconsistent code lengths");
  std::vector<double> pos(slices * static_cast<size_t>(n)), neg(pos.size());
  for (size_t s = 0; s < slices; ++s)
    for (VectorXd::Index k = 0; k < n; ++k) {
      pos[s * static_cast<size_t>(n) + static_cast<size_t>(k)] = codes_pos[s](k);
      neg[s * static_cast<size_t>(n) + static_cast<size_t>(k)] = codes_neg[s](k);
    }
  VectorXd out(n);
  detail::check(xbs_reconstruct_output(pos.data(), neg.data(), static_cast<int32_t>(slices), n, spec.device_bits,
                                       scale, out.data()));
  return out;
}

}  // namespace xbarsim::mapping
