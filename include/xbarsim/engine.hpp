// xbarsim/engine.hpp — EngineKind (reference engine.hpp:15).  This path
// evaluates ideal, aam, fcm and interp_fcm (either base) on the GPU, and the
// oracle engine in its zero-parasitic identity case; the dense nodal solve
// with parasitics is CPU-only and rejected with ConfigError.
#pragma once

namespace xbarsim {
enum class EngineKind { ideal = 0, oracle = 1, fcm = 2, aam = 3, interp_fcm = 4 };
}  // namespace xbarsim
