#!/usr/bin/env python3
"""ADC flips of the snapped contract vs the literal fp64 model, all configs.

Runs the CPU oracle in `literal` and `snapped` mode on the same seeded
inputs of every BASELINE.json config (tests/flips.py) on larger samples than
the -m gpu test, and writes the table BASELINE.md section 5 and bench.py's
`parity` field quote.  The GPU side of the claim (GPU == snapped oracle, bit
for bit) is tests/test_adc_flips_gpu.py / test_parity*_gpu.py.  Oracle only:
runs on any host (no GPU), one process per case.

  python tools/flip_report.py --out profiles/r02/adc_flips.json
"""
import argparse
import json
import multiprocessing as mp
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

# (config, layer index, sampled batch rows, tile columns, tile rows)
CASES = [("c1", 0, 64, 4, 13), ("c1", 1, 64, 1, 4), ("c2-512", 0, 256, 4, 4), ("c2-1024", 0, 256, 2, 2),
         ("c2-2048", 0, 256, 1, 1), ("c2-4096", 0, 256, 1, 1), ("c3", 0, 512, 1, 1), ("c3", 1, 512, 1, 2),
         ("c3", 8, 256, 1, 3), ("c3", 14, 256, 1, 5), ("c3", 19, 128, 1, 1), ("c4", 0, 64, 1, 2),
         ("c4", 1, 64, 1, 2), ("c4", 10, 64, 1, 2), ("c4", 19, 48, 1, 1), ("c4", 20, 32, 2, 2), ("c5", 0, 48, 1, 1)]


def run(case):
    from paper_2002_11151_b200 import configs
    import flips

    name, li, n_rows, n_tc, n_tr = case
    cfg = configs.CONFIGS[name]
    L = cfg.layers[li]
    opt = cfg.options()
    W, x, dy = cfg.weights(L, li), cfg.inputs(L, li), cfg.errors(L, li)
    rows = flips.sample_rows(x, dy, n_rows, 17)
    GR, GC = -(-L.K // cfg.tile), -(-L.N // cfg.tile)
    rng = np.random.default_rng(23)
    tcs = sorted(rng.choice(GC, size=min(n_tc, GC), replace=False).tolist())
    trs = sorted(rng.choice(GR, size=min(n_tr, GR), replace=False).tolist())
    t0 = time.time()
    r = flips.flip_stats(W, opt, x[rows], dy[rows], tcs, trs)
    r.update({"config": cfg.name, "layer": L.name, "M": L.M, "K": L.K, "N": L.N, "adc_bits": cfg.adc_bits,
              "seconds": round(time.time() - t0, 1)})
    print(json.dumps({k: r[k] for k in ("config", "layer", "forward", "backward", "seconds")}), flush=True)
    return r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "adc_flips.json"))
    ap.add_argument("--procs", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    with mp.get_context("fork").Pool(a.procs) as pool:
        res = pool.map(run, CASES, chunksize=1)
    tot = {d: {"conversions": sum(r[d]["conversions"] for r in res), "flips": sum(r[d]["flips"] for r in res)}
           for d in ("forward", "backward")}
    for d in tot.values():
        d["rate"] = d["flips"] / max(1, d["conversions"])
    out = {"what": "ADC codes of the snapped contract (GPU == snapped oracle bit for bit) vs the literal unsnapped "
                   "fp64 oracle (ascending-row current sums, layers.cpp:260-263 / converters.cpp:79-87) on the same "
                   "seeded inputs; sampled batch rows (incl. the max|x| / max|dy| rows) and crossbar tiles",
           "max_abs_code_delta": max(max(r["forward"]["max_abs_code_delta"], r["backward"]["max_abs_code_delta"])
                                     for r in res),
           "total": tot, "cases": res}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps({"total": tot, "max_abs_code_delta": out["max_abs_code_delta"]}))


if __name__ == "__main__":
    main()
