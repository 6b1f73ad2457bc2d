"""Layers past the single-pass exactness bounds of the tcgen05 VMMs stay on
the tensor cores (split into crossbar-tile ranges with exact int64 totals)
and stay bit-exact against the snapped oracle.

C5 crossbar options (256x256 crossbars, eight 1-bit slices, 8-bit ADC): a
forward over 130 row tiles passes the int32 bit-plane combine bound
(130 * 255 * 255 * 255 >= 2^31), a backward over 66 column tiles passes it
too (66 * 2 * 255 * 255 * 255).  Before the split these shapes ran on the
CUDA-core cross-check kernels (counted in tc_fallbacks)."""
import numpy as np
import pytest

from helpers import aam_options, xb

pytestmark = pytest.mark.gpu

oracle_py = pytest.importorskip("oracle_py")


def _c5_options():
    return aam_options(tile=256, wb=8, db=1, adc_bits=8, i_fs=4e-4, r_row=2.5, r_col=2.5)


@pytest.mark.parametrize("K,N", [(33280, 256), (256, 16896)])
def test_deep_and_wide_layers_stay_on_tensor_cores(K, N):
    opt = _c5_options()
    rng = np.random.default_rng(K + N)
    W = rng.normal(0.0, 0.02, (K, N))
    x = rng.uniform(0.0, 1.0, (4, K))
    dy = rng.uniform(-1.0, 1.0, (4, N))
    gpu = xb.CrossbarCore(W, opt)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    y = gpu.forward(x, True)
    dx = gpu.backward(dy, 1.0)
    assert gpu.info().tc_fallbacks == 0
    y_o = orc.forward(x, True)
    dx_o = orc.backward(dy, 1.0)
    assert np.count_nonzero(y) > 0 and np.count_nonzero(dx) > 0
    assert np.array_equal(y, y_o), np.max(np.abs(y - y_o))
    assert np.array_equal(dx, dx_o), np.max(np.abs(dx - dx_o))
