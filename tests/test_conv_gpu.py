"""CrossbarConv2d (layers.cpp:415-505) on the device -- im2col gather, the
crossbar core, col2im gather in the reference's summation order -- against
the oracle's restatement: y, dx and dW bit-exact over a few training steps
(C3-like 3x3 layers, stride 1 and 2, padding 0 and 1)."""
import numpy as np
import pytest

from helpers import aam_options, normal, rand, xb

pytestmark = pytest.mark.gpu

oracle_py = pytest.importorskip("oracle_py")

GEOMS = [
    # in_c, out_c, k, stride, pad, h, w, batch
    (3, 16, 3, 1, 1, 8, 8, 2),
    (16, 32, 3, 2, 1, 8, 8, 3),
    (2, 5, 3, 1, 0, 7, 6, 2),
]


@pytest.mark.parametrize("gi", range(len(GEOMS)))
def test_conv2d_matches_oracle(gi):
    in_c, out_c, k, s, p, h, w, b = GEOMS[gi]
    opt = aam_options(tile=64, adc_bits=7, i_fs=1e-4, sigma=0.1, vseed=2, lr=0.2)
    W = normal((in_c * k * k, out_c), 11 + gi, 0.2)
    conv = xb.CrossbarConv2d(W, in_c, out_c, k, s, p, opt)
    orc = oracle_py.OracleConv2d(W, in_c, out_c, k, s, p, opt)
    x = rand((b, in_c * h * w), 12 + gi, -0.5, 1.2)
    for it in range(3):
        y = conv.forward(xb.Tensor(x, [in_c, h, w]), True)
        y_o, dims = orc.forward(x, in_c, h, w, True)
        assert tuple(y.dims) == dims
        assert np.array_equal(y.values, y_o), (it, np.max(np.abs(y.values - y_o)))
        dy = rand(y.values.shape, 13 + gi + it)
        dx = conv.backward(xb.Tensor(dy, y.dims))
        dx_o = orc.backward(dy)
        assert np.array_equal(dx.values, dx_o), (it, np.max(np.abs(dx.values - dx_o)))
        assert dx.dims == [in_c, h, w]
        conv.apply_updates(it)
        orc.apply_updates(it)
    # keep the comparison meaningful: the conv really moved
    assert np.any(conv.core().gradient() != 0)


def test_conv2d_geometry_errors():
    opt = aam_options(tile=64, adc_bits=6, i_fs=1e-4)
    with pytest.raises(ValueError):
        xb.CrossbarConv2d(np.zeros((10, 4)), 1, 4, 3, 1, 0, opt)  # not (in_c*k*k) x out_c
    conv = xb.CrossbarConv2d(normal((9, 4), 1, 0.1), 1, 4, 3, 1, 0, opt)
    with pytest.raises(ValueError):
        conv.forward(xb.Tensor(np.zeros((2, 4)), [1, 2, 2]), False)  # kernel does not fit
    with pytest.raises(xb.StateError):
        conv.backward(xb.Tensor(np.zeros((2, 16)), [4, 2, 2]))  # backward before forward
