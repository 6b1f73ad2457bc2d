// xbarsim/matrix.hpp — minimal stand-in for Eigen::MatrixXd (Eigen is not in
// this image): column-major fp64, element (i, j) at
// data()[j * rows() + i], value semantics, exact == comparison.  Code written
// against the reference compiles after `using MatrixXd = xbarsim::MatrixXd`.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace xbarsim {

class MatrixXd {
 public:
  using Index = std::int64_t;
  MatrixXd() = default;
  MatrixXd(Index rows, Index cols, double fill = 0.0)
      : rows_(check(rows)), cols_(check(cols)), v_(static_cast<size_t>(rows * cols), fill) {}
  static MatrixXd Zero(Index rows, Index cols) { return MatrixXd(rows, cols, 0.0); }
  static MatrixXd Constant(Index rows, Index cols, double v) { return MatrixXd(rows, cols, v); }

  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  Index size() const { return rows_ * cols_; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(Index i, Index j) { return v_[static_cast<size_t>(j * rows_ + i)]; }
  double operator()(Index i, Index j) const { return v_[static_cast<size_t>(j * rows_ + i)]; }
  void resize(Index rows, Index cols) {
    rows_ = check(rows);
    cols_ = check(cols);
    v_.assign(static_cast<size_t>(rows * cols), 0.0);
  }
  void setZero() { std::fill(v_.begin(), v_.end(), 0.0); }
  double absMax() const {
    double m = 0.0;
    for (double x : v_) m = std::max(m, std::fabs(x));
    return m;
  }
  bool operator==(const MatrixXd& o) const { return rows_ == o.rows_ && cols_ == o.cols_ && v_ == o.v_; }
  bool operator!=(const MatrixXd& o) const { return !(*this == o); }

 private:
  static Index check(Index n) {
    if (n < 0) throw std::invalid_argument("MatrixXd: negative dimension");
    return n;
  }
  Index rows_ = 0, cols_ = 0;
  std::vector<double> v_;
};

/// Minimal stand-in for Eigen::VectorXd (reconstruct_output's codes).
class VectorXd {
 public:
  using Index = std::int64_t;
  VectorXd() = default;
  explicit VectorXd(Index n, double fill = 0.0) : v_(static_cast<size_t>(n < 0 ? 0 : n), fill) {
    if (n < 0) throw std::invalid_argument("VectorXd: negative dimension");
  }
  static VectorXd Zero(Index n) { return VectorXd(n, 0.0); }
  static VectorXd Constant(Index n, double v) { return VectorXd(n, v); }
  Index size() const { return static_cast<Index>(v_.size()); }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(Index i) { return v_[static_cast<size_t>(i)]; }
  double operator()(Index i) const { return v_[static_cast<size_t>(i)]; }
  double& operator[](Index i) { return v_[static_cast<size_t>(i)]; }
  double operator[](Index i) const { return v_[static_cast<size_t>(i)]; }
  void resize(Index n) { v_.assign(static_cast<size_t>(n), 0.0); }
  bool operator==(const VectorXd& o) const { return v_ == o.v_; }
  bool operator!=(const VectorXd& o) const { return !(*this == o); }

 private:
  std::vector<double> v_;
};

}  // namespace xbarsim
