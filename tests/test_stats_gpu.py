"""Statistics and error semantics of apply_updates on the GPU.

Reference: CrossbarCore::apply_updates (layers.cpp:382-391) keeps running
maxima of |dW| and |implied W| over every update; scale_gradient refuses a
non-finite gradient before the master changes (update.cpp:18-19).  The
device-resident path (*_device, the path bench.py times) must keep the same
running statistics across back-to-back steps, and an error must surface
exactly once.
"""
import numpy as np
import pytest

from helpers import aam_options, normal, rand, xb

pytestmark = pytest.mark.gpu

oracle_py = pytest.importorskip("oracle_py")
torch = pytest.importorskip("torch")


def _dev(a):  # M x K column-major on the device
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64).T)).cuda()


def test_device_path_running_statistics():
    """5 device-path steps, one synchronize: |W| / |dW| maxima equal the
    oracle's running maxima; conversion_seconds accumulates every update."""
    K, N, M = 192, 160, 24
    opt = aam_options(tile=64, adc_bits=6, i_fs=6e-5)  # sigma = v = gamma = 0: no libm on either side
    W = normal((K, N), 3, 0.05)
    gpu = xb.CrossbarCore(W, opt)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    t0 = gpu.conversion_seconds()
    ys = []
    for it in range(5):
        x, dy = rand((M, K), 10 + it, 0.0, 1.0), rand((M, N), 20 + it) * (0.2 + it)
        dx_, dy_ = _dev(x), _dev(dy)
        y_, dxo = torch.empty((N, M), dtype=torch.float64, device="cuda"), torch.empty((K, M), dtype=torch.float64,
                                                                                         device="cuda")
        gpu.forward_device(dx_.data_ptr(), M, True, y_.data_ptr())
        gpu.backward_device(dy_.data_ptr(), M, 1.0, dxo.data_ptr())
        gpu.apply_updates_device(it)
        ys.append((y_, orc.forward(x, True)))
        orc.backward(dy, 1.0)
        orc.apply_updates(it)
    gpu.synchronize()
    for y_, yo in ys:
        assert np.array_equal(y_.cpu().numpy().T, yo)
    st = orc.stats()
    assert gpu.grad_abs_max_seen() == st["dwmax_seen"]
    assert gpu.weight_abs_max_seen() == st["wmax_seen"]
    assert gpu.conversion_seconds() > t0
    for s in range(opt.map.num_slices()):
        assert np.array_equal(gpu.master_diff(s), orc.master(s))


@pytest.mark.parametrize("device_path", [False, True])
def test_nonfinite_gradient_is_refused_once(device_path):
    """grad_divisor = 0 makes dW non-finite: the update raises ValueError
    (std::invalid_argument, update.cpp:18-19), the master is unchanged, and
    the error does not resurface on later calls."""
    K, N, M = 128, 96, 8
    opt = aam_options(tile=64, adc_bits=6, i_fs=6e-5)
    W = normal((K, N), 5, 0.05)
    gpu = xb.CrossbarCore(W, opt)
    before = [gpu.master_diff(s) for s in range(opt.map.num_slices())]
    x, dy = rand((M, K), 1, 0.0, 1.0), rand((M, N), 2)
    gpu.forward(x, True)
    gpu.backward(dy, 0.0)
    assert not np.all(np.isfinite(gpu.gradient()))
    if device_path:
        gpu.apply_updates_device(0)
        with pytest.raises(ValueError, match="finite"):
            gpu.synchronize()
        gpu.synchronize()  # read once, then cleared
    else:
        with pytest.raises(ValueError, match="finite"):
            gpu.apply_updates(0)
    for s, u in enumerate(before):
        assert np.array_equal(gpu.master_diff(s), u)
    # the next step runs normally
    gpu.forward(x, True)
    gpu.backward(dy, 1.0)
    gpu.apply_updates(1)
    gpu.synchronize()
    assert np.isfinite(gpu.weight_abs_max_seen())


def test_set_gradient_nonfinite_refused():
    K, N = 64, 64
    opt = aam_options(tile=64, adc_bits=6, i_fs=6e-5)
    gpu = xb.CrossbarCore(normal((K, N), 7, 0.05), opt)
    before = gpu.master_diff(0)
    dW = normal((K, N), 8, 0.01)
    dW[3, 5] = np.inf
    gpu.set_gradient(dW)
    with pytest.raises(ValueError, match="finite"):
        gpu.apply_updates(0)
    assert np.array_equal(gpu.master_diff(0), before)
    dW[3, 5] = 0.0
    gpu.set_gradient(dW)
    gpu.apply_updates(0)
    assert not np.array_equal(gpu.master_diff(0), before)


def test_tc_fallback_is_counted():
    """16-bit weights as sixteen 1-bit slices with an 8-bit ADC pass the
    one-tile fp32 bound only per crossbar tile: the forward splits the row
    tiles (split-K) and stays on the tensor cores.  With a 16-bit ADC a single
    tile's shift-add total (maxc * sum 2^s >= 2^24) is outside the tcgen05
    kernels' exact fp32 accumulators, so the exact SIMT kernel runs, and the
    C ABI counts it so callers (bench.py) can refuse it."""
    K, N, M = 300, 40, 6
    x = rand((M, K), 4, 0.0, 1.0)
    W = normal((K, N), 9, 0.05)
    for adc_bits, i_fs, fallback in ((8, 4e-4, False), (16, 4e-4, True)):
        opt = aam_options(tile=256, wb=16, db=1, adc_bits=adc_bits, i_fs=i_fs, r_row=2.5, r_col=2.5)
        gpu = xb.CrossbarCore(W, opt)
        orc = oracle_py.OracleCore(W, opt, snapped=True)
        assert gpu.info().tc_fallbacks == 0
        assert np.array_equal(gpu.forward(x, True), orc.forward(x, True))
        assert (gpu.info().tc_fallbacks >= 1) == fallback
