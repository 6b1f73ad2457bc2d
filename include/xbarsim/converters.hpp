// xbarsim/converters.hpp — DacSpec / AdcSpec (reference converters.hpp:11-45).
#pragma once

#include <vector>

namespace xbarsim::converters {

struct DacSpec {
  int bits = 1;
  double v_fs = 1.0;
  std::vector<double> transfer;  // empty -> ideal linear
  int stream_bits = 1;
  bool ideal_linear() const { return transfer.empty(); }
};

struct AdcSpec {
  int bits = 8;
  double i_fs = 0.0;             // > 0: explicit full scale (the path's contract)
  std::vector<double> transfer;  // optional code thresholds
  double clip_percentile = 0.999;
  bool passthrough() const { return bits == 0; }
};

}  // namespace xbarsim::converters
