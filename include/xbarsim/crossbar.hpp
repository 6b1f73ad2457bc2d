// xbarsim/crossbar.hpp — CrossbarConfig (reference crossbar.hpp:17-40).
// Validation happens behind the C ABI (xbs_core_create), in the reference's
// order and with its messages.
#pragma once

namespace xbarsim::circuit {

struct CrossbarConfig {
  int rows = 64;
  int cols = 64;
  double r_row = 1.0;
  double r_col = 4.6;
  double r_source = 0.0;
  double r_sense = 0.0;
  double g_min = 1e-6;
  double g_max = 1e-5;
  double v_fs = 1.0;
  double on_off_ratio() const { return g_max / g_min; }
};

}  // namespace xbarsim::circuit

#include "xbarsim/matrix.hpp"

namespace xbarsim::circuit {

/// reference crossbar.hpp:46-61: a tile's geometry and conductances (g(i, j)).
struct ConductanceTile {
  CrossbarConfig config;
  MatrixXd g;
};

}  // namespace xbarsim::circuit
