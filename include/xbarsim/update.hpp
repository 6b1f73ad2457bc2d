// xbarsim/update.hpp — UpdateSpec (reference update.hpp:13-23).  The update
// itself (update.cpp:43-88) runs on the GPU inside CrossbarCore::apply_updates.
#pragma once

#include <cstdint>

namespace xbarsim::update {

struct UpdateSpec {
  double v = 0.0;
  double gamma = 0.0;
  double lr = 0.01;
  std::uint64_t seed = 0;
  double layer_scale = 0.0;  // 0: the mapping's layer scale
};

}  // namespace xbarsim::update
