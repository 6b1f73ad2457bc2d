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


def test_deferred_update_matches_synchronous():
    """Host apply_updates on an AAM / linear-update core returns before the
    update finishes; every later call settles it first.  The
    trajectory, the statistics and the next forward (whose input copy
    overlaps the pending update) equal those of the synchronous path
    (profiling on keeps apply_updates synchronous)."""
    from helpers import aam_options, normal, rand, xb

    W = normal((300, 200), 71, 0.05)
    x = rand((48, 300), 72, 0.0, 1.0)
    dy = rand((48, 200), 73)
    opt = aam_options(tile=128, adc_bits=7, i_fs=1.8e-4, r_col=4.6)
    runs = []
    for sync_path in (False, True):
        c = xb.CrossbarCore(W, opt)
        if sync_path:
            c.profile(True)
        ys, stats = [], []
        for it in range(3):
            ys.append(c.forward(x, True).copy())
            c.backward(dy, 1.0)
            c.apply_updates(it)
            stats.append((c.weight_abs_max_seen(), c.grad_abs_max_seen(), c.refresh_count()))
        ys.append(c.forward(x, False).copy())
        assert c.conversion_seconds() > 0.0
        runs.append((ys, stats, [c.master_diff(s).copy() for s in range(opt.map.num_slices())]))
    (ya, sa, ma), (yb, sb, mb) = runs
    for a, b in zip(ya, yb):
        assert np.array_equal(a, b)
    assert sa == sb
    for a, b in zip(ma, mb):
        assert np.array_equal(a, b)
