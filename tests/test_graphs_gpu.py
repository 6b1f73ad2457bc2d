"""CUDA-graph replay of repeated forward / backward calls.

A call that repeats the previous call's buffers and shape is captured once
and replayed (xbs_core.cu run_graphed); every step must give the same bits as
the eager launches, with new data in the same buffers each step, through the
device API, the host API and a conv layer, and across the update (which runs
eagerly between replays).
"""
import numpy as np
import pytest

from helpers import aam_options, normal, rand, xb

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _dev(a):
    """M x K column-major device copy (a K x M C-order tensor)."""
    return torch.from_numpy(np.ascontiguousarray(a.T)).cuda()


@pytest.mark.parametrize("kernel", [0, 1])
def test_device_api_graph_replay_bit_identical(kernel):
    K, N, M = 300, 260, 33
    opt = aam_options(tile=128, adc_bits=7, i_fs=2e-4, sigma=0.1, v=0.3, gamma=0.5, lr=0.2, useed=5, vseed=2)
    W = normal((K, N), 7, 0.05)
    cores = [xb.CrossbarCore(W, opt) for _ in range(2)]
    cores[1].use_graphs(False)
    for c in cores:
        c.select_kernel(kernel)
    bufs = [(torch.zeros((K, M), dtype=torch.float64, device="cuda"), torch.zeros((N, M), dtype=torch.float64,
                                                                                   device="cuda"),
             torch.zeros((N, M), dtype=torch.float64, device="cuda"),
             torch.zeros((K, M), dtype=torch.float64, device="cuda")) for _ in cores]
    launches = [0, 0]
    for it in range(5):  # eager, capture, then replays
        x = rand((M, K), 100 + it, -0.2, 1.2)
        dy = rand((M, N), 200 + it)
        res = []
        for i, (c, (dx_in, ddy, dyout, ddx)) in enumerate(zip(cores, bufs)):
            dx_in.copy_(torch.from_numpy(np.ascontiguousarray(x.T)))
            ddy.copy_(torch.from_numpy(np.ascontiguousarray(dy.T)))
            l0 = c.launch_count()
            c.forward_device(dx_in.data_ptr(), M, True, dyout.data_ptr())
            c.backward_device(ddy.data_ptr(), M, 1.0, ddx.data_ptr())
            c.apply_updates_device(it)
            c.synchronize()
            launches[i] += c.launch_count() - l0
            res.append((dyout.cpu().numpy().copy(), ddx.cpu().numpy().copy(), c.gradient(), c.master_diff(0)))
        for a, b in zip(res[0], res[1]):
            assert np.array_equal(a, b)
    assert launches[0] == launches[1]  # the replayed graphs hold the same kernels


def test_host_api_graph_replay_bit_identical():
    K, N, M = 200, 130, 20
    opt = aam_options(tile=64, adc_bits=6, i_fs=6e-5)
    W = normal((K, N), 8, 0.05)
    g, e = xb.CrossbarCore(W, opt), xb.CrossbarCore(W, opt)
    e.use_graphs(False)
    for it in range(4):
        x = rand((M, K), 300 + it, -0.2, 1.2)
        dy = rand((M, N), 400 + it)
        assert np.array_equal(g.forward(x, True), e.forward(x, True))
        assert np.array_equal(g.backward(dy, 2.0), e.backward(dy, 2.0))
        assert np.array_equal(g.gradient(), e.gradient())
        g.apply_updates(it)
        e.apply_updates(it)


def test_conv_graph_replay_bit_identical():
    opt = aam_options(tile=64, adc_bits=6, i_fs=6e-5)
    W = normal((3 * 3 * 3, 8), 9, 0.1)
    a = xb.CrossbarConv2d(W, 3, 8, 3, 1, 1, opt)
    b = xb.CrossbarConv2d(W, 3, 8, 3, 1, 1, opt)
    b.core().use_graphs(False)  # the conv layer's own core
    for it in range(4):
        x = normal((2, 3 * 6 * 6), 500 + it)
        ya = a.forward(xb.Tensor(x, [3, 6, 6]), True)
        yb = b.forward(xb.Tensor(x, [3, 6, 6]), True)
        assert np.array_equal(ya.values, yb.values)
        dy = normal(ya.values.shape, 600 + it)
        assert np.array_equal(a.backward(xb.Tensor(dy, ya.dims)).values, b.backward(xb.Tensor(dy, yb.dims)).values)
        a.apply_updates(it)
        b.apply_updates(it)
