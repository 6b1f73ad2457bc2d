"""Generates the committed golden fixtures (tests/golden/*.npz) from the CPU
oracle (snapped mode, the GPU's exactness contract: since
round 2 the 24-bit grid of three radix-255 limbs, q <= 255^3 - 1).

The oracle itself is pinned on the reference's own known answers
(oracle/tests/kat_oracle.cpp, restating test_nn.cpp / test_update.cpp /
test_mapping.cpp / test_converters.cpp / test_circuit.cpp); the reference
cannot be built here (Eigen3 absent), so these fixtures carry
that pin to the GPU box, where neither /root/reference nor a rebuild of the
checker is needed.  Cases avoid transcendental functions (sigma = 0, v = 0,
gamma = 0) so every value is bit-exact across glibc and CUDA libm:
x / W / dy are seeded numpy draws; one training step of CrossbarCore
(layers.cpp:215-391): y0 = forward(x, training), dx = backward(dy, 1.0),
dW = gradient(), apply_updates(0), y1 = forward(x, false).

    python tests/golden/make_golden.py        # rewrites the .npz files
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import aam_options  # noqa: E402

CASES = {
    # C1-like (BASELINE configs[0] crossbar): 64x64 tiles, ragged K and N,
    # 4 two-bit slices, 6-bit ADC, 1 kOhm source / sense resistances
    "c1_ragged": dict(M=24, K=150, N=70, seed=11,
                      opt=dict(tile=64, wb=8, db=2, adc_bits=6, i_fs=1.7e-4, r_row=1.0, r_col=1.0,
                               r_source=1000.0, r_sense=1000.0, lr=0.1),
                      x=(0.0, 1.0), wsd=0.05),
    # C2-like (configs[1] crossbar): 128x128 tiles, 7-bit ADC, defaults r_row = 1, r_col = 4.6
    "c2_tile128": dict(M=32, K=256, N=200, seed=12,
                       opt=dict(tile=128, wb=8, db=2, adc_bits=7, i_fs=1.8e-4, r_row=1.0, r_col=4.6, lr=0.1),
                       x=(-1.0, 1.0), wsd=0.02),
    # C3-like narrow layer: 16 outputs of a 128-column tile, 4-bit slices, 8-bit ADC
    "c3_narrow": dict(M=40, K=144, N=16, seed=13,
                      opt=dict(tile=128, wb=8, db=4, adc_bits=8, i_fs=2.0e-4, r_row=1.0, r_col=4.6, lr=0.1),
                      x=(-1.0, 1.0), wsd=0.1),
}


def inputs(c):
    rng = np.random.default_rng(c["seed"])
    x = rng.uniform(c["x"][0], c["x"][1], (c["M"], c["K"]))
    W = rng.normal(0.0, c["wsd"], (c["K"], c["N"]))
    dy = rng.uniform(-1.0, 1.0, (c["M"], c["N"]))
    return x, W, dy


def run_oracle(name):
    import oracle_py

    c = CASES[name]
    x, W, dy = inputs(c)
    o = oracle_py.OracleCore(W, aam_options(**c["opt"]), snapped=True)
    y0 = o.forward(x, training=True)
    dx = o.backward(dy, 1.0)
    dW = o.gradient()
    o.apply_updates(0)
    y1 = o.forward(x, training=False)
    return dict(y0=y0, dx=dx, dW=dW, y1=y1)


def main():
    for name in CASES:
        out = run_oracle(name)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, {k: (v.shape, float(np.abs(v).max())) for k, v in out.items()})


if __name__ == "__main__":
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    main()
