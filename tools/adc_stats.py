"""Dev tool: fraction of ADC conversions that took the exact fp64 path."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2002_11151_b200.configs import CONFIGS
from paper_2002_11151_b200 import xbarsim as xb
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2-512"]
L = cfg.layers[0]
core = xb.CrossbarCore(cfg.weights(L), cfg.options())
e0, _ = core.adc_counters()
y = core.forward(cfg.inputs(L), True)
e1, _ = core.adc_counters()
conv = L.M * 8 * ((L.N + cfg.tile - 1) // cfg.tile * cfg.tile) * ((L.K + cfg.tile - 1) // cfg.tile) * (cfg.weight_bits // cfg.device_bits) * 2
print(cfg.name, "exact-path conversions", e1 - e0, "of", conv, "=", (e1 - e0) / conv)
