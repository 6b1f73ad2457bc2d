// xbarsim/status.hpp — xbs_status -> the reference's exception types
// (SURVEY.md §8b "Errors": one status per exception class; device faults
// surface as StateError carrying the CUDA message).
#pragma once

#include <stdexcept>
#include <string>

#include "xbarsim/errors.hpp"
#include "xbarsim_b200.h"

namespace xbarsim::detail {

inline void check(int rc) {
  if (rc == XBS_OK) return;
  const std::string m = xbs_last_error();
  switch (rc) {
    case XBS_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case XBS_STATE_ERROR:
    case XBS_CUDA_ERROR: throw StateError(m);
    case XBS_CONFIG_ERROR:
    case XBS_UNSUPPORTED: throw ConfigError(m);
    case XBS_CONVERGENCE_ERROR: throw ConvergenceError(m, 0.0, 0);
    case XBS_STALE_CACHE_ERROR: throw StaleCacheError(m);
    case XBS_DEGENERATE_CIRCUIT_ERROR: throw DegenerateCircuitError(m);
    default: throw std::runtime_error(m);
  }
}

}  // namespace xbarsim::detail
