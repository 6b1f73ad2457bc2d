#!/usr/bin/env python3
"""CPU oracle (the restated reference path, one thread) per BASELINE.json
config, for BASELINE.md section 5: each config's first layer as a bounded
K = N = one-crossbar-tile slice (bench.cpu_sample), and the whole config's
step time extrapolated linearly in MACs (the oracle's VMM cost is linear in
tile count and batch rows).  Run on the GPU box's host:

  python tools/cpu_table.py > gpurun_out/cpu_table.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]

import bench  # noqa: E402
from paper_2002_11151_b200.configs import CONFIGS  # noqa: E402

out = {}
for name in ("c1", "c2-512", "c2-1024", "c2-2048", "c2-4096", "c3", "c4", "c5"):
    cfg = CONFIGS[name]
    rate, dt, desc = bench.cpu_sample(cfg, cfg.tile, 1, 0, rows=256)
    total = sum(cfg.macs(L)["total"] for L in cfg.layers)
    out[cfg.name] = {"mac_per_s": rate, "sample_s": dt, "sample": desc, "config_macs": total,
                     "extrapolated_s_per_step": total / rate, "threads": 1}
    print(json.dumps({cfg.name: out[cfg.name]}), file=sys.stderr)
print(json.dumps(out))
