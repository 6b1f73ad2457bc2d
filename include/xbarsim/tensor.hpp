// xbarsim/tensor.hpp — nn::Tensor (reference tensor.hpp:13-21).
#pragma once

#include <vector>

#include "xbarsim/matrix.hpp"

namespace xbarsim::nn {

struct Tensor {
  MatrixXd values;
  std::vector<int> dims;
  int bits = 0;
  double full_scale = 0.0;
  MatrixXd::Index batch() const { return values.rows(); }
  MatrixXd::Index features() const { return values.cols(); }
};

}  // namespace xbarsim::nn
