"""General converters on the GPU: multi-bit DAC
streams (layers.cpp:52-64, 236-241), non-linear DAC transfer tables
(converters.cpp:28-35), ADC threshold tables (converters.cpp:76-82), ADCs
wider than 16 bits and non-power-of-two DAC full scales.  These currents are
not integers on the snapped grid, so the layer runs the exact fp64
CUDA-core VMMs (k_fwd_volts / k_bwd_volts), which follow the reference's
fp64 order term by term: y and dx bit-exact against the snapped oracle,
before and after an update, plus dW; ADC auto-calibration on the same
converters."""
import numpy as np
import pytest

from helpers import aam_options, normal, rand, xb

pytestmark = pytest.mark.gpu

oracle_py = pytest.importorskip("oracle_py")
from test_parity_gpu import _sync_conductances  # noqa: E402


def _dac_curve(bits):
    n = 1 << bits  # monotone, transfer[0] = 0, <= v_fs: a compressive DAC
    return [0.0] + [float((d / (n - 1)) ** 0.7) for d in range(1, n)]


CASES = {
    "dac2": dict(dac_bits=2),
    "dac4_table": dict(dac_bits=4, dac_table=True),
    "adc_table": dict(adc_table=64),
    "adc20": dict(adc_bits=20),
    "vfs_0.8": dict(v_fs=0.8),
    "dac2_passthrough": dict(dac_bits=2, adc_bits=0),
    "dac2_sigma": dict(dac_bits=2, sigma=0.1, r_source=1000.0, r_sense=1000.0),
    "dac4_tile128": dict(dac_bits=4, tile=128, K=300, N=150),
}


def _options(case):
    c = CASES[case]
    o = aam_options(tile=c.get("tile", 64), adc_bits=c.get("adc_bits", 7), i_fs=1e-4, sigma=c.get("sigma", 0.0),
                    r_source=c.get("r_source", 0.0), r_sense=c.get("r_sense", 0.0), r_col=4.6)
    sb = c.get("dac_bits", 1)
    o.dac.bits = o.dac.stream_bits = sb
    o.dac.v_fs = c.get("v_fs", 1.0)
    if c.get("dac_table"):
        o.dac.transfer = _dac_curve(sb)
    if c.get("adc_table"):
        o.adc.transfer = list(np.linspace(0.0, 2.5e-4, c["adc_table"]))
    return o, c.get("K", 100), c.get("N", 80)


@pytest.mark.parametrize("case", sorted(CASES))
def test_general_converters_bit_exact(case):
    opt, K, N = _options(case)
    M = 6
    W = normal((K, N), 31, 0.05)
    gpu = xb.CrossbarCore(W, opt)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    _sync_conductances(gpu, orc, opt)
    for it in range(2):
        x = rand((M, K), 40 + it, -0.2, 1.2)
        dy = rand((M, N), 50 + it, -1.0, 1.0)
        y_g, y_o = gpu.forward(x, True), orc.forward(x, True)
        assert np.count_nonzero(y_o) > 0
        assert np.array_equal(y_g, y_o), (case, it, np.max(np.abs(y_g - y_o)))
        dx_g, dx_o = gpu.backward(dy, 1.0), orc.backward(dy, 1.0)
        assert np.array_equal(dx_g, dx_o), (case, it, np.max(np.abs(dx_g - dx_o)))
        assert np.array_equal(gpu.gradient(), orc.gradient())
        gpu.apply_updates(it)
        orc.apply_updates(it)
        _sync_conductances(gpu, orc, opt)  # libm ulps of the update, as in test_parity_gpu
    assert gpu.info().tc_fallbacks == 0  # this path is by design, not a fallback


AUTOCAL = {
    "dac2": dict(dac_bits=2),
    "dac4_table": dict(dac_bits=4, dac_table=True),
    "vfs_0.8": dict(v_fs=0.8),
    "adc20": dict(adc_bits=20),
    "codes20": dict(act_bits=20, error_bits=20),
}


@pytest.mark.parametrize("case", sorted(AUTOCAL))
def test_general_converters_auto_calibrate(case):
    """layers.cpp:74, 189-213 with the general converters: the calibration
    batches pass the fp64 currents through and record them (as bit patterns:
    non-negative doubles order as integers); the freeze picks the reference's
    nearest-rank quantile (converters.cpp:96-107).  y, dx bit-exact at every
    call, the frozen forward i_fs equal to the oracle's."""
    c = AUTOCAL[case]
    o = aam_options(tile=64, adc_bits=c.get("adc_bits", 7), i_fs=0.0, r_col=4.6, act_bits=c.get("act_bits", 8),
                    error_bits=c.get("error_bits", 8), lr=0.2, useed=3)
    sb = c.get("dac_bits", 1)
    o.dac.bits = o.dac.stream_bits = sb
    o.dac.v_fs = c.get("v_fs", 1.0)
    if c.get("dac_table"):
        o.dac.transfer = _dac_curve(sb)
    o.adc.clip_percentile = 0.995
    o.adc_cal_batches = cal = 2
    K, N, M = 100, 80, 5
    W = normal((K, N), 11, 0.05)
    gpu = xb.CrossbarCore(W, o)
    orc = oracle_py.OracleCore(W, o, snapped=True)
    _sync_conductances(gpu, orc, o)
    x = rand((M, K), 12, -0.1, 1.1)
    for it in range(cal + 1):
        y, y_o = gpu.forward(x, True), orc.forward(x, True)
        assert np.array_equal(y, y_o), (case, it, np.max(np.abs(y - y_o)))
        dy = rand((M, N), 13 + it)
        dx, dx_o = gpu.backward(dy, 1.0), orc.backward(dy, 1.0)
        assert np.array_equal(dx, dx_o), (case, it, np.max(np.abs(dx - dx_o)))
        assert np.array_equal(gpu.gradient(), orc.gradient())
        st = orc.stats()
        assert gpu.forward_adc_full_scale() == st["fwd_i_fs"]
        assert (st["fwd_i_fs"] > 0) == (it + 1 >= cal)
        gpu.apply_updates(it)
        orc.apply_updates(it)
        _sync_conductances(gpu, orc, o)
