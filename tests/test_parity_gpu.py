"""GPU-vs-oracle parity through the C ABI (small seeded layers the oracle
finishes in seconds).  Bar:
  * non-ideal conductances: bit-identical snapped grid values (any mismatch
    would come from a CUDA-vs-glibc libm ulp in the variation Gaussian and is
    counted; tolerance 1e-5 max-rel as in the north star);
  * forward y, backward dx: bit-exact fp64 (integer ADC totals x the same
    k_out) given the same conductances;
  * dW: bit-exact (exact integer contract);
  * updated master: 1e-12 max-rel (CUDA exp/log/cos vs glibc, ulp level).
"""
import numpy as np
import pytest

from helpers import aam_options, dyadic_ideal_options, normal, rand, xb

pytestmark = pytest.mark.gpu

oracle_py = pytest.importorskip("oracle_py")

KERNELS = [1, 0]  # SIMT cross-check, tcgen05


def _pair(W, opt, kernel):
    gpu = xb.CrossbarCore(W, opt)
    gpu.select_kernel(kernel)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    return gpu, orc


def _sync_conductances(gpu, orc, opt):
    """Feeds the GPU's regenerated conductances to the oracle; returns the
    number of snapped values that differed (libm ulp flips)."""
    flips = 0
    S = opt.map.num_slices()
    T = orc.grid_rows * orc.grid_cols
    for s in range(S):
        for p in range(2):
            for t in range(T):
                g = gpu.nonideal(s, p, t)
                o = orc.nonideal(s, p, t)
                flips += int(np.count_nonzero(g != o))
                assert np.all(np.abs(g - o) <= 1e-5 * np.abs(o))
                orc.set_nonideal(s, p, t, g)
    return flips


CASES = [
    # (K, N, M, tile, opt kwargs)
    (100, 80, 7, 64, dict(adc_bits=6, i_fs=6e-5)),
    (130, 257, 5, 64, dict(adc_bits=8, i_fs=1e-4, sigma=0.1, r_source=1000.0, r_sense=1000.0, i_fs_scale=0.2)),
    (256, 128, 16, 128, dict(adc_bits=7, i_fs=2e-4, r_col=4.6)),
    (96, 96, 3, 32, dict(adc_bits=5, i_fs=5e-5, wb=8, db=1, act_bits=6, error_bits=5)),
    # 256-row / 256-column crossbars (C5 geometry: two 128-row k-blocks per
    # accumulation), mixed shapes and a ragged 200-row tile padded to 256
    (520, 300, 9, 256, dict(adc_bits=8, i_fs=4e-4, wb=8, db=1, sigma=0.2, r_row=2.5, r_col=2.5)),
    (300, 260, 6, None, dict(rows=256, cols=128, adc_bits=7, i_fs=3e-4)),
    (260, 300, 6, None, dict(rows=128, cols=256, adc_bits=7, i_fs=2e-4)),
    (410, 150, 4, None, dict(rows=200, cols=72, adc_bits=6, i_fs=3e-4, act_bits=4, error_bits=6)),
]


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("case", range(len(CASES)))
def test_forward_backward_dw_bit_exact(case, kernel):
    K, N, M, tile, kw = CASES[case]
    kw = dict(kw)
    kw.pop("i_fs_scale", None)
    opt = aam_options(tile=tile, **kw)
    W = normal((K, N), 10 + case, 0.05)
    gpu, orc = _pair(W, opt, kernel)
    flips = _sync_conductances(gpu, orc, opt)
    assert flips == 0
    x = rand((M, K), 20 + case, -0.2, 1.2)
    y_g = gpu.forward(x, True)
    y_o = orc.forward(x, True)
    assert np.array_equal(y_g, y_o), np.max(np.abs(y_g - y_o))
    dy = rand((M, N), 30 + case, -1.0, 1.0)
    dx_g = gpu.backward(dy, 1.0)
    dx_o = orc.backward(dy, 1.0)
    assert np.array_equal(dx_g, dx_o), np.max(np.abs(dx_g - dx_o))
    assert np.array_equal(gpu.gradient(), orc.gradient())


UPDATE_CASES = [
    # (K, N, opt kwargs): each hits a different specialisation of K3b
    (100, 70, dict(sigma=0.1, v=0.5, gamma=2.0)),          # 2 weights/thread, variation + nonlinear + noise
    (100, 72, dict(sigma=0.0, v=0.5, gamma=2.0)),          # 4 weights/thread, qmin table + nonlinear + noise
    (50, 33, dict(sigma=0.1, v=0.5, gamma=2.0)),           # odd N: generic one-weight-per-thread kernel
    (96, 64, dict(sigma=0.0, wb=8, db=1, lr=0.5)),         # S = 8, linear, sigma = 0
    (80, 128, dict(sigma=0.2, wb=8, db=4, lr=0.5)),        # S = 2, linear, variation
]


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("ucase", range(len(UPDATE_CASES)))
def test_update_and_regeneration(kernel, ucase):
    K, N, kw = UPDATE_CASES[ucase]
    kw = dict(dict(lr=0.3), **kw)
    opt = aam_options(tile=64, adc_bits=6, i_fs=6e-5, useed=7, vseed=3, **kw)
    W = normal((K, N), 1, 0.05)
    gpu, orc = _pair(W, opt, kernel)
    x = rand((6, K), 2, 0.0, 1.0)
    dy = rand((6, N), 3)
    for it in range(3):
        gpu.forward(x, True)
        orc.forward(x, True)
        gpu.backward(dy, 1.0)
        orc.backward(dy, 1.0)
        assert np.array_equal(gpu.gradient(), orc.gradient())
        gpu.apply_updates(it)
        orc.apply_updates(it)
        for s in range(opt.map.num_slices()):
            ug, uo = gpu.master_diff(s), orc.master(s)
            assert np.max(np.abs(ug - uo)) <= 1e-12 * max(1e-30, np.max(np.abs(uo)))
            orc.set_master(s, ug)  # continue from the GPU state
        orc.regenerate()
        flips = _sync_conductances(gpu, orc, opt)
        assert flips <= 2
        st = orc.stats()
        assert gpu.grad_abs_max_seen() == st["dwmax_seen"]
        assert abs(gpu.weight_abs_max_seen() - st["wmax_seen"]) <= 1e-12 * st["wmax_seen"]
    assert gpu.refresh_count() == 4


def test_fully_ideal_fast_path_matches_digital_reference():
    """test_nn.cpp:89-108 through the GPU: y, dx bit-identical on the dyadic grid."""
    opt = dyadic_ideal_options(9, 5)
    W = rand((9, 5), 2, -0.9, 0.9)
    gpu = xb.CrossbarCore(W, opt)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    x = np.abs(rand((7, 9), 3))
    assert np.array_equal(gpu.forward(x, True), orc.forward(x, True))
    dy = rand((7, 5), 4, -0.3, 0.3)
    assert np.array_equal(gpu.backward(dy, 1.0), orc.backward(dy, 1.0))
    assert np.array_equal(gpu.gradient(), orc.gradient())
    with pytest.raises(xb.StateError):
        gpu.nonideal(0, 0, 0)


def test_passthrough_adc_streamed_equals_oracle():
    opt = aam_options(tile=8, adc_bits=0, r_row=1.0, r_col=4.6)
    W = rand((8, 8), 4, -0.9, 0.9)
    gpu = xb.CrossbarCore(W, opt)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    x = np.abs(rand((4, 8), 5))
    assert np.array_equal(gpu.forward(x, False), orc.forward(x, False))
    dy = rand((4, 8), 6, -0.2, 0.2)
    assert np.array_equal(gpu.backward(dy, 1.0), orc.backward(dy, 1.0))


def test_backward_before_forward_and_zero_error():
    opt = aam_options(tile=64, adc_bits=6, i_fs=6e-5)
    gpu = xb.CrossbarCore(normal((20, 10), 1, 0.05), opt)
    with pytest.raises(xb.StateError):
        gpu.backward(np.zeros((2, 10)), 1.0)
    with pytest.raises(xb.StateError):  # state before shape (layers.cpp:287-290)
        gpu.backward(np.zeros((2, 11)), 1.0)
    with pytest.raises(ValueError):
        gpu.forward(np.zeros((2, 21)), False)
    gpu.forward(np.ones((2, 20)) * 0.5, True)
    dx = gpu.backward(np.zeros((2, 10)), 1.0)
    assert np.all(dx == 0.0) and not np.any(np.signbit(dx))
    assert np.all(gpu.gradient() == 0.0)
    with pytest.raises(ValueError):
        gpu.backward(np.zeros((3, 10)), 1.0)


def test_zero_input_zero_output_and_empty_batch():
    opt = aam_options(tile=64, adc_bits=8, i_fs=1e-4, r_col=4.6)
    gpu = xb.CrossbarCore(normal((6, 4), 1, 0.3), opt)
    assert np.all(gpu.forward(np.zeros((3, 6)), False) == 0.0)
    assert gpu.forward(np.zeros((0, 6)), False).shape == (0, 4)


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("gd", [4.0, 3.0, 0.125, 1e-310])
def test_grad_divisor(kernel, gd):
    """dW = x_values^T dy_q / grad_divisor (layers.cpp:304): power-of-two
    divisors take an exact reciprocal multiply on the GPU, others divide;
    both bit-identical to the oracle's division (subnormal divisor included)."""
    K, N, M = 150, 140, 300
    opt = aam_options(tile=128, adc_bits=7, i_fs=2e-4)
    W = normal((K, N), 41, 0.05)
    gpu, orc = _pair(W, opt, kernel)
    x = rand((M, K), 42, -0.2, 1.2)
    dy = rand((M, N), 43)
    gpu.forward(x, True)
    orc.forward(x, True)
    assert np.array_equal(gpu.backward(dy, gd), orc.backward(dy, gd))
    assert np.array_equal(gpu.gradient(), orc.gradient())
