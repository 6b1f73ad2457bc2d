"""BASELINE configs[0] end to end: the MLP 784-256-10
train step at full size (batch 64, 64x64 crossbars, 4 two-bit slices, 6-bit
ADC, 1 kOhm source / sense, variation sigma = 0.1) through the reference's
layer stack -- CrossbarLinear -> ReLU -> CrossbarLinear -> softmax CE
(train.cpp:11-33) -> backward x2 -> apply_updates (train.cpp:93-144) -- on
the GPU (C ABI) against the same stack on the snapped CPU oracle, for three
iterations.  Bar: logits, loss, dW and dx bit-exact; the non-ideal
conductances regenerated after each update equal the oracle's up to libm
ulp flips in the variation Gaussian (CUDA vs glibc), which are counted and
fed back so the trajectories stay comparable (as in test_parity_gpu).

The oracle stack's digital glue is the oracle's own C++ restatement
(ReLU layers.cpp:510-522, softmax CE train.cpp:11-33), not the Python
mirror's; the mirror's loss and dlogits are checked against it within 4 ulp
(numpy vs glibc exp/log), and both stacks then back-propagate the oracle's
dlogits so the crossbar layers compare bit for bit."""
import numpy as np
import pytest

from helpers import xb

pytestmark = pytest.mark.gpu
oracle_py = pytest.importorskip("oracle_py")

from paper_2002_11151_b200.configs import CONFIGS  # noqa: E402
from test_parity_gpu import _sync_conductances  # noqa: E402


class _OracleLinear(xb.Layer):
    def __init__(self, W, opt):
        self.c = oracle_py.OracleCore(W, opt, snapped=True)

    def forward(self, x, training):
        return xb.Tensor(self.c.forward(x.values, training), [self.c.N])

    def backward(self, dy):
        return xb.Tensor(self.c.backward(dy.values, 1.0), [self.c.K])

    def apply_updates(self, it):
        self.c.apply_updates(it)


class _OracleReLU(xb.Layer):
    def forward(self, x, training):
        self._x = x.values
        return xb.Tensor(oracle_py.relu(x.values, np.zeros_like(x.values))[0], list(x.dims))

    def backward(self, dy):
        return xb.Tensor(oracle_py.relu(self._x, dy.values)[1], list(dy.dims))


def _forward(net, x):
    h = xb.Tensor(x, [x.shape[1]])
    for layer in net:
        h = layer.forward(h, True)
    return h.values.copy()


def _backward(net, d, it):
    g = xb.Tensor(d, [d.shape[1]])
    grads = []
    for layer in reversed(net):
        g = layer.backward(g)
        grads.append(g.values.copy())
    for layer in net:
        layer.apply_updates(it)
    return grads


def test_c1_mlp_train_step_matches_oracle():
    cfg = CONFIGS["c1"]
    opt = cfg.options()
    L1, L2 = cfg.layers
    W1, W2 = cfg.weights(L1, 0), cfg.weights(L2, 1)
    x = cfg.inputs(L1)
    labels = np.random.default_rng(6000 + cfg.cid).integers(0, 10, size=L1.M)
    gpu = [xb.CrossbarLinear(W1, opt), xb.ReLU(), xb.CrossbarLinear(W2, opt)]
    orc = [_OracleLinear(W1, opt), _OracleReLU(), _OracleLinear(W2, opt)]
    flips = 0
    for g, o in ((gpu[0], orc[0]), (gpu[2], orc[2])):
        flips += _sync_conductances(g.core(), o.c, opt)
    for it in range(3):
        lg, lo = _forward(gpu, x), _forward(orc, x)
        assert np.array_equal(lg, lo), it
        loss_g, d_g = xb.softmax_cross_entropy(lg, labels)
        loss_o, d_o = oracle_py.softmax_cross_entropy(lo, labels)
        assert abs(loss_g - loss_o) <= 4 * np.spacing(loss_o), it
        assert np.all(np.abs(d_g - d_o) <= 4 * np.spacing(np.abs(d_o))), it
        grads_g, grads_o = _backward(gpu, d_o, it), _backward(orc, d_o, it)
        for a, b in zip(grads_g, grads_o):
            assert np.array_equal(a, b), it
        for g, o in ((gpu[0], orc[0]), (gpu[2], orc[2])):
            assert np.array_equal(g.core().gradient(), o.c.gradient()), it
            flips += _sync_conductances(g.core(), o.c, opt)
    # libm flips are rare (a snapped value one grid step off at a tie)
    n_dev = 2 * opt.map.num_slices() * (832 * 256 + 256 * 64)
    assert flips <= 1e-4 * n_dev * 4
