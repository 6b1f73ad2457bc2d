"""Pins the restated CPU oracle to the REFERENCE'S OWN CODE (CPU, no GPU).

oracle/ref/Makefile compiles the reference's core sources unchanged, in
place under /root/reference, against a minimal Eigen-API shim
(oracle/eigen_shim: eager evaluation, matrix products summed over the inner
index in ascending order -- the order the oracle's `literal` mode defines,
since Eigen's is unspecified), into oracle/_ref/libxbsref.so.  On the same
seeded inputs the oracle's literal mode must then reproduce the reference
bit for bit: forward y, backward dx, dW, every non-ideal conductance tile,
the per-slice master after non-linear / noisy updates, the running
statistics and the softmax loss.  Where the reference tree is absent (the
GPU box) the test skips."""
import numpy as np
import pytest

import oracle_py
import ref_py
from helpers import aam_options, normal, rand, xb

pytestmark = pytest.mark.skipif(not ref_py.available(), reason="reference build (oracle/_ref) absent")


def _case(name):
    E = xb.EngineKind
    if name == "c1_aam_sigma":
        o = aam_options(tile=64, adc_bits=6, i_fs=1.7e-4, sigma=0.1, r_source=1000.0, r_sense=1000.0, vseed=4001)
        return o, (100, 70, 6)
    if name == "c2_aam":
        return aam_options(tile=128, adc_bits=7, i_fs=1.8e-4, r_col=4.6), (200, 150, 5)
    if name == "c3_nonlinear_noise":
        o = aam_options(tile=64, wb=8, db=4, adc_bits=8, i_fs=2e-4, v=1.0, gamma=0.05, useed=5003)
        return o, (90, 40, 4)
    if name == "c5_like":
        o = aam_options(tile=64, wb=8, db=1, adc_bits=8, i_fs=4e-4, r_row=2.5, r_col=2.5, sigma=0.2, vseed=7)
        return o, (80, 70, 3)
    if name == "fcm":
        o = aam_options(tile=16, adc_bits=7, i_fs=3e-5, r_col=4.6, engine=E.fcm)
        return o, (40, 30, 3)
    if name == "interp_fcm":
        o = aam_options(tile=16, adc_bits=7, i_fs=3e-5, r_col=4.6, engine=E.interp_fcm)
        o.interp_interval = 2
        return o, (30, 20, 3)
    if name == "nodal_oracle":
        o = aam_options(tile=8, adc_bits=8, i_fs=2e-5, r_col=4.6, engine=E.oracle)
        return o, (16, 12, 3)
    if name == "passthrough":
        return aam_options(tile=32, adc_bits=0, r_col=4.6), (50, 40, 3)
    if name == "ideal_fast_path":
        o = aam_options(tile=32, adc_bits=0, engine=E.ideal)
        return o, (50, 40, 3)
    if name == "dac2_adc_table":
        o = aam_options(tile=32, adc_bits=6, i_fs=1e-4, r_col=4.6)
        o.dac.bits = o.dac.stream_bits = 2
        o.adc.transfer = list(np.linspace(0.0, 1.2e-4, 64))
        return o, (50, 40, 3)
    raise KeyError(name)


CASES = ["c1_aam_sigma", "c2_aam", "c3_nonlinear_noise", "c5_like", "fcm", "interp_fcm", "nodal_oracle",
         "passthrough", "ideal_fast_path", "dac2_adc_table"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_literal_mode_is_the_reference(name):
    opt, (K, N, M) = _case(name)
    W = normal((K, N), 11, 0.05)
    orc = oracle_py.OracleCore(W, opt, snapped=False)
    ref = ref_py.RefCore(W, opt, opt.map.tile_rows, opt.map.tile_cols, opt.map.num_slices(),
                         orc.grid_rows * orc.grid_cols)
    S, T = opt.map.num_slices(), orc.grid_rows * orc.grid_cols
    for it in range(3):
        if opt.engine != xb.EngineKind.ideal:
            for s in range(S):
                for p in range(2):
                    for t in range(T):
                        assert np.array_equal(orc.nonideal(s, p, t), ref.nonideal(s, p, t)), (name, it, s, p, t)
        x = rand((M, K), 20 + it, -0.2, 1.2)
        dy = rand((M, N), 30 + it, -1.0, 1.0)
        assert np.array_equal(orc.forward(x, True), ref.forward(x, True)), (name, it)
        assert np.array_equal(orc.backward(dy, 1.0), ref.backward(dy, 1.0)), (name, it)
        assert np.array_equal(orc.gradient(), ref.gradient()), (name, it)
        orc.apply_updates(it)
        ref.apply_updates(it)
        for s in range(S):
            assert np.array_equal(orc.master(s), ref.master(s, orc.padded_rows, orc.padded_cols)), (name, it, s)
    so, sr = orc.stats(), ref.stats()
    assert so["wmax_seen"] == sr["weight_abs_max_seen"] and so["dwmax_seen"] == sr["grad_abs_max_seen"]
    assert so["refresh_count"] == sr["refresh_count"]


def test_softmax_cross_entropy_is_the_reference():
    rng = np.random.default_rng(5)
    logits = rng.normal(0.0, 3.0, (32, 10))
    labels = rng.integers(0, 10, 32)
    lo, do = oracle_py.softmax_cross_entropy(logits, labels)
    lr, dr = ref_py.softmax_cross_entropy(logits, labels)
    assert lo == lr and np.array_equal(do, dr)
