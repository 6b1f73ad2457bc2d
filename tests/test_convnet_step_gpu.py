"""C3-shaped network step in the reference's own layer set (SURVEY.md §8d
C3 "optional end-to-end step": conv -> ReLU chain, Flatten -> FC, softmax CE;
layers.cpp:415-587, train.cpp:11-33) with C3's crossbar options verbatim
(128x128 crossbars, 4-bit slices, 8-bit ADC, v = 1.0, gamma = 0.05) at a
reduced spatial size so the oracle finishes in seconds: GPU (C ABI) against
the snapped CPU oracle.  Before the first update every value is bit-exact;
the update's exp / log / cos come from CUDA's libm on one side and glibc on
the other (<= 1e-12 relative on the master), so the second
forward is compared within the one-ADC-LSB effect a flipped conductance
grid step can have."""
import numpy as np
import pytest

from helpers import xb

pytestmark = pytest.mark.gpu
oracle_py = pytest.importorskip("oracle_py")

from paper_2002_11151_b200.configs import CONFIGS  # noqa: E402

B, H = 16, 16  # batch, image side (C3: 128, 32)


def _net_weights(rng):
    k1 = rng.normal(0.0, np.sqrt(2.0 / 27), (27, 16))       # conv1 3->16, Kaiming
    k2 = rng.normal(0.0, np.sqrt(2.0 / 144), (144, 16))     # conv2 16->16 stride 2
    fc = rng.normal(0.0, np.sqrt(2.0 / 1024), (1024, 10))   # 16 x 8 x 8 -> 10
    return k1, k2, fc


def _gpu_step(net, x, labels, it, d_ref=None):
    """d_ref: back-propagate these dlogits (the oracle's) instead of the
    mirror's, so the crossbar backward compares bit for bit."""
    h = xb.Tensor(x, [3, H, H])
    for layer in net:
        h = layer.forward(h, True)
    loss, d = xb.softmax_cross_entropy(h.values, labels)
    if d_ref is not None:
        assert np.all(np.abs(d - d_ref) <= 4 * np.spacing(np.abs(d_ref)))
        d = d_ref
    g = xb.Tensor(d, [10])
    grads = []
    for layer in reversed(net):
        g = layer.backward(g)
        grads.append(g.values.copy())
    for layer in net:
        layer.apply_updates(it)
    return h.values.copy(), loss, grads


def _orc_step(c1, c2, fc, x, labels, it):
    """The oracle's own restatement of the digital glue (ReLU layers.cpp:510-522,
    softmax CE train.cpp:11-33) around the oracle crossbar layers."""
    y1, d1 = c1.forward(x, 3, H, H, True)
    a1 = oracle_py.relu(y1, np.zeros_like(y1))[0]
    y2, d2 = c2.forward(a1, d1[0], d1[1], d1[2], True)
    a2 = oracle_py.relu(y2, np.zeros_like(y2))[0]
    logits = fc.forward(a2, True)
    loss, d = oracle_py.softmax_cross_entropy(logits, labels)
    g_fc = fc.backward(d)
    g_r2 = oracle_py.relu(y2, g_fc)[1]
    g_c2 = c2.backward(g_r2)
    g_r1 = oracle_py.relu(y1, g_c2)[1]
    g_c1 = c1.backward(g_r1)
    for layer in (c1, c2, fc):
        layer.apply_updates(it)
    # same order as the GPU stack's reversed walk (fc, flatten, relu, conv2, relu, conv1)
    return logits, loss, [g_fc, g_fc, g_r2, g_c2, g_r1, g_c1], d


def test_c3_convnet_step_matches_oracle():
    opt = CONFIGS["c3"].options()
    rng = np.random.default_rng(7003)
    k1, k2, wfc = _net_weights(rng)
    x = rng.normal(0.0, 1.0, (B, 3 * H * H))
    labels = rng.integers(0, 10, size=B)
    gpu = [xb.CrossbarConv2d(k1, 3, 16, 3, 1, 1, opt), xb.ReLU(), xb.CrossbarConv2d(k2, 16, 16, 3, 2, 1, opt),
           xb.ReLU(), xb.Flatten(), xb.CrossbarLinear(wfc, opt)]
    c1 = oracle_py.OracleConv2d(k1, 3, 16, 3, 1, 1, opt)
    c2 = oracle_py.OracleConv2d(k2, 16, 16, 3, 2, 1, opt)
    fc = oracle_py.OracleCore(wfc, opt, snapped=True)

    lo, loss_o, grads_o, d_o = _orc_step(c1, c2, fc, x, labels, 0)
    lg, loss_g, grads_g = _gpu_step(gpu, x, labels, 0, d_ref=d_o)
    assert np.array_equal(lg, lo)
    assert abs(loss_g - loss_o) <= 4 * np.spacing(loss_o)
    for a, b in zip(grads_g, grads_o):
        assert np.array_equal(a, b)
    assert np.array_equal(gpu[5].core().gradient(), fc.gradient())

    # after the non-linear, noisy update (libm on both sides)
    h = xb.Tensor(x, [3, H, H])
    for layer in gpu:
        h = layer.forward(h, False)
    y1, d1 = c1.forward(x, 3, H, H, False)
    y2, d2 = c2.forward(oracle_py.relu(y1, np.zeros_like(y1))[0], d1[0], d1[1], d1[2], False)
    lo2 = fc.forward(oracle_py.relu(y2, np.zeros_like(y2))[0], False)
    same = np.mean(h.values == lo2)
    assert same >= 0.9, same
    assert np.all(np.isfinite(h.values))
