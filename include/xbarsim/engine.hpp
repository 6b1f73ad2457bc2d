// xbarsim/engine.hpp — EngineKind (reference engine.hpp:15).  This path
// evaluates ideal, aam, and zero-parasitic fcm / oracle / interp_fcm (which
// reduce to the identity); circuit solves with parasitics are out of scope
// and rejected with ConfigError.
#pragma once

namespace xbarsim {
enum class EngineKind { ideal = 0, oracle = 1, fcm = 2, aam = 3, interp_fcm = 4 };
}  // namespace xbarsim
