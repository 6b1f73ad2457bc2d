"""Host-pointer C ABI with pinned caller buffers.

xbs_core_forward / xbs_core_backward write y and dx straight into a pinned,
mapped host buffer from the tcgen05 epilogues (the D2H transfer overlaps the
VMM), and through a staging buffer + copy otherwise (pageable memory, the
SIMT kernels).  Every route must return the same bits, for contiguous and
strided (ld > M) outputs, and agree with the snapped oracle.
"""
import ctypes

import numpy as np
import pytest

from helpers import aam_options, normal, rand, xb

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
oracle_py = pytest.importorskip("oracle_py")

_D = ctypes.POINTER(ctypes.c_double)


def _pinned(rows, cols, ld):
    """(ld x cols) column-major view of pinned host memory (kept alive by t)."""
    t = torch.zeros((cols, ld), dtype=torch.float64, pin_memory=True)
    return t, t.numpy().T


def _p(a):
    return a.ctypes.data_as(_D)


@pytest.mark.parametrize("kernel", [0, 1])
@pytest.mark.parametrize("pad", [0, 5])
def test_pinned_outputs_bit_identical(kernel, pad):
    K, N, M = 300, 260, 37
    opt = aam_options(tile=128, adc_bits=7, i_fs=2e-4, r_col=4.6)
    W = normal((K, N), 4, 0.05)
    x = np.asfortranarray(rand((M, K), 5, -0.2, 1.2))
    dy = np.asfortranarray(rand((M, N), 6))
    ref = xb.CrossbarCore(W, opt)  # pageable numpy buffers: staging + copy
    ref.select_kernel(kernel)
    y_ref = ref.forward(x, True)
    dx_ref = ref.backward(dy, 1.0)

    gpu = xb.CrossbarCore(W, opt)
    gpu.select_kernel(kernel)
    lib = xb.load_library()
    ty, y = _pinned(M, N, M + pad)
    tx, dx = _pinned(M, K, M + pad)
    y[:] = np.nan
    dx[:] = np.nan
    xb._check(lib.xbs_core_forward(gpu._h, _p(x), M, K, M, 1, _p(y), M + pad))
    xb._check(lib.xbs_core_backward(gpu._h, _p(dy), M, N, M, 1.0, _p(dx), M + pad))
    assert np.array_equal(y[:M], y_ref)
    assert np.array_equal(dx[:M], dx_ref)
    if pad:  # rows beyond M of the caller's buffer are not touched
        assert np.all(np.isnan(y[M:])) and np.all(np.isnan(dx[M:]))

    orc = oracle_py.OracleCore(W, opt, snapped=True)
    assert np.array_equal(y[:M], orc.forward(x, True))
    assert np.array_equal(dx[:M], orc.backward(dy, 1.0))
