"""Activation / error precisions over the reference's whole range (1..24,
layers.cpp:28-31): up to 16-bit activations and errors on the tensor-core
path (16 bit planes per stream) and on the general-converter path (4-bit
DAC streams); 17..24 bits on the general-converter path (u32 codes, exact
fp64 CUDA-core VMMs).  Bit-exact against the snapped oracle, dW included."""
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


@pytest.mark.parametrize("act,err,dac", [(20, 8, 1), (24, 24, 1), (8, 18, 1), (24, 24, 4), (18, 18, 2)])
def test_codes_above_16_bits(act, err, dac):
    """17- to 24-bit activation / error codes (layers.cpp:28-31): u32 codes
    on the exact fp64 CUDA-core VMMs (the general-converter path), bit-exact
    against the snapped oracle over forward, backward, dW and an update."""
    opt = aam_options(tile=64, adc_bits=8, i_fs=1.2e-4, act_bits=act, error_bits=err, r_col=4.6, lr=0.2)
    opt.dac.bits = opt.dac.stream_bits = dac
    K, N, M = 100, 70, 4
    W = normal((K, N), 3 + act, 0.05)
    gpu = xb.CrossbarCore(W, opt)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    _sync_conductances(gpu, orc, opt)
    for it in range(2):
        x = rand((M, K), 5 + it, -0.1, 1.1)
        dy = rand((M, N), 6 + it, -1.0, 1.0)
        assert np.array_equal(gpu.forward(x, True), orc.forward(x, True))
        assert np.array_equal(gpu.backward(dy, 1.0), orc.backward(dy, 1.0))
        assert np.array_equal(gpu.gradient(), orc.gradient())
        gpu.apply_updates(it)
        orc.apply_updates(it)
        _sync_conductances(gpu, orc, opt)
    assert gpu.info().tc_fallbacks == 0  # by design, not a fallback


def test_codes_above_16_bits_fully_ideal():
    """The fully-ideal fast path (layers.cpp:226, 307) reads the same u32 codes."""
    opt = aam_options(tile=64, adc_bits=0, act_bits=22, error_bits=20)
    opt.engine = xb.EngineKind.ideal
    W = normal((90, 60), 2, 0.05)
    gpu = xb.CrossbarCore(W, opt)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    x, dy = rand((5, 90), 3, -0.1, 1.1), rand((5, 60), 4)
    assert np.array_equal(gpu.forward(x, True), orc.forward(x, True))
    assert np.array_equal(gpu.backward(dy, 1.0), orc.backward(dy, 1.0))
    assert np.array_equal(gpu.gradient(), orc.gradient())
