"""The Python mirror's digital step glue (ReLU, MaxPool2d, Flatten, softmax
cross-entropy) against the oracle's C++ restatement of the reference
(layers.cpp:510-587, train.cpp:11-33), so the end-to-end step tests
(test_mlp_step_gpu.py, test_convnet_step_gpu.py) do not check the product's
glue against itself.

Bars: ReLU / MaxPool2d / Flatten bit-identical (signed zeros included:
the reference multiplies by a 0/1 mask); softmax cross-entropy within
4 ulp (numpy's exp/log against glibc's)."""
import numpy as np
import oracle_py
import pytest

from helpers import xb


def _relu_case(rng, n, f):
    x = rng.normal(0.0, 1.0, (n, f))
    x[rng.random((n, f)) < 0.1] = 0.0  # exact zeros take the mask's 0 branch
    return x, rng.normal(0.0, 1.0, (n, f))


def test_relu_matches_oracle_bit_for_bit():
    rng = np.random.default_rng(1)
    x, dy = _relu_case(rng, 7, 33)
    r = xb.ReLU()
    y = r.forward(xb.Tensor(x, [33]), True).values
    dx = r.backward(xb.Tensor(dy, [33])).values
    y_o, dx_o = oracle_py.relu(x, dy)
    for a, b in ((y, y_o), (dx, dx_o)):
        assert np.array_equal(a, b)
        assert np.array_equal(np.signbit(a), np.signbit(b))  # -0.0 where the reference has it


@pytest.mark.parametrize("c,h,w,k,s", [(3, 8, 8, 2, 2), (2, 7, 9, 3, 2), (4, 6, 6, 3, 1), (1, 5, 5, 5, 1)])
def test_maxpool2d_matches_oracle_bit_for_bit(c, h, w, k, s):
    rng = np.random.default_rng(c * 100 + h * 10 + k)
    n = 5
    # coarse values force ties inside windows: the first maximum in (ky, kx)
    # order must win on both sides, and dx scatters onto it
    x = np.round(rng.normal(0.0, 1.0, (n, c * h * w)) * 2.0) / 2.0
    mp = xb.MaxPool2d(k, s)
    y = mp.forward(xb.Tensor(x, [c, h, w]), True)
    dy = rng.normal(0.0, 1.0, y.values.shape)
    dx = mp.backward(xb.Tensor(dy, list(y.dims))).values
    y_o, dx_o = oracle_py.maxpool2d(x, c, h, w, k, s, dy)
    assert y.dims == [c, (h - k) // s + 1, (w - k) // s + 1]
    assert np.array_equal(y.values, y_o)
    assert np.array_equal(dx, dx_o)


def test_flatten_keeps_values_and_restores_dims():
    x = np.arange(2 * 3 * 4 * 5, dtype=np.float64).reshape(2, 60)
    f = xb.Flatten()
    y = f.forward(xb.Tensor(x, [3, 4, 5]), True)
    assert y.dims == [60] and np.array_equal(y.values, x)
    dx = f.backward(xb.Tensor(x * 2.0, [60]))
    assert dx.dims == [3, 4, 5] and np.array_equal(dx.values, x * 2.0)


def test_softmax_cross_entropy_matches_oracle():
    rng = np.random.default_rng(3)
    for n, c in ((64, 10), (5, 1000), (1, 3)):
        logits = rng.normal(0.0, 3.0, (n, c))
        labels = rng.integers(0, c, n)
        loss, d = xb.softmax_cross_entropy(logits, labels)
        loss_o, d_o = oracle_py.softmax_cross_entropy(logits, labels)
        assert abs(loss - loss_o) <= 4 * np.spacing(abs(loss_o))
        assert np.all(np.abs(d - d_o) <= 4 * np.spacing(np.maximum(np.abs(d_o), 1e-300)))
    with pytest.raises(ValueError):
        xb.softmax_cross_entropy(np.zeros((2, 3)), [0])
    with pytest.raises(oracle_py.OracleError):
        oracle_py.softmax_cross_entropy(np.zeros((2, 3)), [0])
