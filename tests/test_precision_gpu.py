"""Activation / error precisions up to the path's 16-bit limit (the
reference accepts 1..24, layers.cpp:28-31; 17..24 are refused loudly here):
16-bit activations and errors on the tensor-core path (16 bit planes per
stream) and on the general-converter path (4-bit DAC streams), bit-exact
against the snapped oracle, dW included."""
import numpy as np
import pytest

from helpers import aam_options, normal, rand, xb

pytestmark = pytest.mark.gpu

oracle_py = pytest.importorskip("oracle_py")
from test_parity_gpu import _sync_conductances  # noqa: E402


@pytest.mark.parametrize("bits,dac,tile", [(16, 1, 128), (12, 1, 64), (16, 4, 64), (15, 3, 64)])
@pytest.mark.parametrize("kernel", [0, 1])
def test_wide_activation_and_error_codes(bits, dac, tile, kernel):
    opt = aam_options(tile=tile, adc_bits=8, i_fs=1.2e-4, act_bits=bits, error_bits=bits, r_col=4.6)
    opt.dac.bits = opt.dac.stream_bits = dac
    K, N, M = 150, 130, 5
    W = normal((K, N), 7 + bits, 0.05)
    gpu = xb.CrossbarCore(W, opt)
    gpu.select_kernel(kernel)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    _sync_conductances(gpu, orc, opt)
    x = rand((M, K), 3, -0.1, 1.1)
    dy = rand((M, N), 4, -1.0, 1.0)
    assert np.array_equal(gpu.forward(x, True), orc.forward(x, True))
    assert np.array_equal(gpu.backward(dy, 1.0), orc.backward(dy, 1.0))
    assert np.array_equal(gpu.gradient(), orc.gradient())
    assert gpu.info().tc_fallbacks == 0


def test_precisions_above_16_bits_are_refused():
    opt = aam_options(tile=64, act_bits=20, error_bits=8)
    with pytest.raises(xb.UnsupportedConfigError):
        xb.CrossbarCore(normal((64, 64), 1, 0.05), opt)
