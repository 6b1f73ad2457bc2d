"""ADC auto-calibration (layers.cpp:74, 189-213,
converters.cpp:90-107) on the device against the oracle's restatement.

While calibrating, the VMMs pass currents through and record them; after
adc_cal_batches training forwards the next forward or backward freezes each
direction's i_fs at the nearest-rank clip_percentile quantile of what it
observed.  Checked: y and dx bit-exact at every call (pass-through during
calibration, quantised after), the frozen forward i_fs equal to the oracle's,
and the freeze landing on the same call (a backward can be the first
quantised call)."""
import numpy as np
import pytest

from helpers import aam_options, normal, rand, xb

pytestmark = pytest.mark.gpu

oracle_py = pytest.importorskip("oracle_py")

CASES = [
    # K, N, M, tile, cal_batches, clip_percentile, opt kwargs
    (100, 80, 7, 64, 2, 0.999, dict(adc_bits=6)),
    (256, 128, 16, 128, 3, 0.999, dict(adc_bits=7, r_col=4.6)),
    (300, 140, 5, 128, 2, 1.0, dict(adc_bits=8, sigma=0.1, vseed=4)),
    (90, 200, 9, 64, 2, 0.5, dict(adc_bits=5, act_bits=6, error_bits=5)),
]


def _sync(gpu, orc, opt):
    for s in range(opt.map.num_slices()):
        orc.set_master(s, gpu.master_diff(s))
    orc.regenerate()
    for s in range(opt.map.num_slices()):
        for p in range(2):
            for t in range(orc.grid_rows * orc.grid_cols):
                orc.set_nonideal(s, p, t, gpu.nonideal(s, p, t))


@pytest.mark.parametrize("kernel", [1, 0])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_auto_calibration_matches_oracle(case, kernel):
    K, N, M, tile, cal, pct, kw = CASES[case]
    opt = aam_options(tile=tile, i_fs=0.0, lr=0.2, useed=3, **kw)
    opt.adc.clip_percentile = pct
    opt.adc_cal_batches = cal
    W = normal((K, N), 5 + case, 0.1)
    gpu = xb.CrossbarCore(W, opt)
    gpu.select_kernel(kernel)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    _sync(gpu, orc, opt)
    x = rand((M, K), 6 + case, -0.1, 1.1)
    for it in range(cal + 2):
        if it == 0:  # an evaluation forward: pass-through, not observed
            assert np.array_equal(gpu.forward(x, False), orc.forward(x, False))
        y = gpu.forward(x, True)
        y_o = orc.forward(x, True)
        assert np.array_equal(y, y_o), (it, np.max(np.abs(y - y_o)))
        dy = rand((M, N), 7 + it)
        dx = gpu.backward(dy, 1.0)
        dx_o = orc.backward(dy, 1.0)
        assert np.array_equal(dx, dx_o), (it, np.max(np.abs(dx - dx_o)))
        assert np.array_equal(gpu.gradient(), orc.gradient())
        st = orc.stats()
        assert gpu.forward_adc_full_scale() == st["fwd_i_fs"]
        frozen = it + 1 >= cal  # the backward of batch `cal` freezes both directions
        assert (st["fwd_i_fs"] > 0) == frozen
        assert (st["bwd_i_fs"] > 0) == frozen
        gpu.apply_updates(it)
        orc.apply_updates(it)
        _sync(gpu, orc, opt)


def test_direction_without_observations_stays_unset():
    """layers.cpp:189-197 + converters.cpp:83-84: a direction that saw no
    currents keeps i_fs unset and its ADC throws StateError when used; a zero
    error never reaches the ADC."""
    opt = aam_options(tile=64, adc_bits=6, i_fs=0.0)
    opt.adc_cal_batches = 1
    W = normal((70, 50), 2, 0.1)
    gpu = xb.CrossbarCore(W, opt)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    x = rand((4, 70), 3, 0.0, 1.0)
    assert np.array_equal(gpu.forward(x, True), orc.forward(x, True))  # observed; the next call freezes
    assert np.array_equal(gpu.forward(x, True), orc.forward(x, True))
    assert gpu.forward_adc_full_scale() == orc.stats()["fwd_i_fs"] > 0
    assert np.array_equal(gpu.backward(np.zeros((4, 50)), 1.0), orc.backward(np.zeros((4, 50)), 1.0))
    with pytest.raises(xb.StateError):
        gpu.backward(rand((4, 50), 4), 1.0)
    with pytest.raises(oracle_py.OracleError):
        orc.backward(rand((4, 50), 4), 1.0)


def test_backward_right_after_the_only_calibration_batch():
    """adc_cal_batches = 1: the first backward already freezes, with no
    backward observations, so it raises StateError (as the reference does)."""
    opt = aam_options(tile=64, adc_bits=6, i_fs=0.0)
    opt.adc_cal_batches = 1
    W = normal((70, 50), 8, 0.1)
    gpu = xb.CrossbarCore(W, opt)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    x, dy = rand((4, 70), 9, 0.0, 1.0), rand((4, 50), 10)
    assert np.array_equal(gpu.forward(x, True), orc.forward(x, True))
    with pytest.raises(xb.StateError):
        gpu.backward(dy, 1.0)
    with pytest.raises(oracle_py.OracleError):
        orc.backward(dy, 1.0)
    assert gpu.forward_adc_full_scale() == orc.stats()["fwd_i_fs"] > 0


def test_auto_calibration_at_c1_scale():
    """C1's fc1 geometry (784 x 256, 64 x 64 crossbars, 4 slices): millions
    of observations per batch, quantile selected on the device equal to the
    oracle's sorted nearest rank."""
    opt = aam_options(tile=64, adc_bits=8, i_fs=0.0, r_col=4.6, lr=0.1)
    opt.adc_cal_batches = 2
    W = normal((784, 256), 11, 0.05)
    gpu = xb.CrossbarCore(W, opt)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    _sync(gpu, orc, opt)
    x = rand((32, 784), 12, -0.2, 1.0)
    for it in range(3):
        y, y_o = gpu.forward(x, True), orc.forward(x, True)
        assert np.array_equal(y, y_o), it
        dy = rand((32, 256), 13 + it)
        assert np.array_equal(gpu.backward(dy, 1.0), orc.backward(dy, 1.0)), it
        gpu.apply_updates(it)
        orc.apply_updates(it)
        _sync(gpu, orc, opt)
    st = orc.stats()
    assert st["fwd_i_fs"] > 0 and st["bwd_i_fs"] > 0
    assert gpu.forward_adc_full_scale() == st["fwd_i_fs"]
