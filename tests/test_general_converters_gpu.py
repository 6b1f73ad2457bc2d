"""General converters on the GPU: multi-bit DAC
streams (layers.cpp:52-64, 236-241), non-linear DAC transfer tables
(converters.cpp:28-35), ADC threshold tables (converters.cpp:76-82), ADCs
wider than 16 bits and non-power-of-two DAC full scales.  These currents are
not integers on the snapped grid, so the layer runs the exact fp64
CUDA-core VMMs (k_fwd_volts / k_bwd_volts), which follow the reference's
fp64 order term by term: y and dx bit-exact against the snapped oracle,
before and after an update, plus dW."""
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


def test_general_converters_refuse_auto_calibration():
    opt, K, N = _options("dac2")
    opt.adc.i_fs = 0.0  # auto-calibration with a multi-bit DAC
    with pytest.raises(xb.UnsupportedConfigError):
        xb.CrossbarCore(normal((K, N), 1, 0.05), opt)
