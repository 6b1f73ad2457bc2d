"""Golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py
from the KAT-pinned oracle): the CPU oracle must still reproduce them bit for
bit, and the CUDA path (C ABI, both VMM kernels) must match them bit for bit
through one training step of CrossbarCore (layers.cpp:215-391)."""
import os
import sys

import numpy as np
import pytest

from helpers import ROOT, aam_options, xb

sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import make_golden  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
NAMES = sorted(make_golden.CASES)


def _load(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_golden(name, oracle_build):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    want = _load(name)
    got = make_golden.run_oracle(name)
    for k in ("y0", "dx", "dW", "y1"):
        assert np.array_equal(got[k], want[k]), (name, k)


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", [0, 1])  # tcgen05, SIMT cross-check
@pytest.mark.parametrize("name", NAMES)
def test_cuda_path_matches_golden(name, kernel):
    c = make_golden.CASES[name]
    x, W, dy = make_golden.inputs(c)
    want = _load(name)
    core = xb.CrossbarCore(W, aam_options(**c["opt"]))
    core.select_kernel(kernel)
    got = {"y0": core.forward(x, True), "dx": core.backward(dy, 1.0), "dW": core.gradient()}
    core.apply_updates(0)
    got["y1"] = core.forward(x, False)
    for k in ("y0", "dx", "dW", "y1"):
        assert np.array_equal(np.asarray(got[k]), want[k]), (name, kernel, k,
                                                            float(np.abs(np.asarray(got[k]) - want[k]).max()))
