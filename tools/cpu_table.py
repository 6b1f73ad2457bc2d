#!/usr/bin/env python3
"""CPU time of the reference path per BASELINE.json config (BASELINE.md
section 5): the reference's own core sources (oracle/_ref, one thread: its
forward / backward / update are serial, layers.hpp:34) step each distinct
layer shape of the config at full K x N on a bounded number of batch rows;
the config's step time is the sum over its layers of (seconds per row x M),
the reference's VMM cost being linear in batch rows.  C5 (8192^2, too large
to regenerate whole on one core in a bounded time) is timed on a one-tile
slice and scaled by tile count (bench.cpu_sample).  Prints one JSON object.

  python tools/cpu_table.py > profiles/r02/cpu_table.json
"""
import collections
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]

import bench  # noqa: E402
from paper_2002_11151_b200.configs import CONFIGS, Layer  # noqa: E402

ROWS = 32


def layer_seconds_per_row(cfg, L, idx):
    opt = cfg.options()
    rows = min(L.M, ROWS)
    sl = Layer(L.name, rows, L.K, L.N)
    W, x, dy = cfg.weights(sl, idx), cfg.inputs(sl, idx), cfg.errors(sl, idx)
    core = bench.cpu_core(W, opt)
    t0 = time.perf_counter()
    core.forward(x, True)
    core.backward(dy, 1.0)
    core.apply_updates(0)
    return (time.perf_counter() - t0) / rows


out = {"kind": bench.cpu_kind(), "threads": 1, "rows_sampled": ROWS, "host": os.uname().nodename}
for name in ("c1", "c2-512", "c2-1024", "c2-2048", "c2-4096", "c3", "c4"):
    cfg = CONFIGS[name]
    shapes = collections.Counter((L.K, L.N) for L in cfg.layers)
    per_shape, total = {}, 0.0
    for i, L in enumerate(cfg.layers):
        key = (L.K, L.N)
        if key not in per_shape:
            per_shape[key] = layer_seconds_per_row(cfg, L, i)
        total += per_shape[key] * L.M
    out[cfg.name] = {"s_per_step": total, "distinct_layer_shapes": len(shapes)}
    print(json.dumps({cfg.name: out[cfg.name]}), file=sys.stderr, flush=True)
cfg = CONFIGS["c5"]
rate, dt, desc = bench.cpu_sample(cfg, cfg.tile, 1, 0, rows=ROWS)
total = sum(cfg.macs(L)["total"] for L in cfg.layers)
out[cfg.name] = {"s_per_step": total / rate, "sample": desc}
print(json.dumps(out))
