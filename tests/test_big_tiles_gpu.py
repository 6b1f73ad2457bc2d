"""Crossbar tiles above 256 x 256 (the reference puts no bound on
CrossbarConfig rows / cols, crossbar.hpp:31-39): a 256-row crossbar is the
most one TMEM accumulator pair sums exactly, so these layers run the exact
integer CUDA-core VMMs by design (not counted as a tensor-core fallback).
Conductances bit-identical, y / dx / dW bit-exact against the snapped oracle,
across an update with variation; auto-calibration on the same geometry."""
import numpy as np
import pytest

from helpers import aam_options, normal, rand, xb

pytestmark = pytest.mark.gpu

oracle_py = pytest.importorskip("oracle_py")
from test_parity_gpu import _sync_conductances  # noqa: E402

CASES = [
    # K, N, M, rows, cols, opt kwargs
    (700, 400, 4, 320, 320, dict(adc_bits=8, i_fs=4e-4)),
    (600, 500, 3, 512, 384, dict(adc_bits=7, i_fs=6e-4, sigma=0.1, vseed=2, r_col=2.5)),
    (1100, 1030, 2, 1024, 1024, dict(adc_bits=8, i_fs=1.5e-3, wb=8, db=1, r_row=0.5, r_col=0.5)),
    (400, 300, 3, 300, 260, dict(adc_bits=0)),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_big_tiles_bit_exact(case):
    K, N, M, rows, cols, kw = CASES[case]
    opt = aam_options(tile=None, rows=rows, cols=cols, lr=0.2, useed=5, **kw)
    W = normal((K, N), 60 + case, 0.05)
    gpu = xb.CrossbarCore(W, opt)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    assert _sync_conductances(gpu, orc, opt) == 0
    for it in range(2):
        x = rand((M, K), 70 + it, -0.2, 1.2)
        dy = rand((M, N), 80 + it, -1.0, 1.0)
        y_g, y_o = gpu.forward(x, True), orc.forward(x, True)
        assert np.count_nonzero(y_o) > 0
        assert np.array_equal(y_g, y_o), (case, it, np.max(np.abs(y_g - y_o)))
        dx_g, dx_o = gpu.backward(dy, 1.0), orc.backward(dy, 1.0)
        assert np.array_equal(dx_g, dx_o), (case, it, np.max(np.abs(dx_g - dx_o)))
        assert np.array_equal(gpu.gradient(), orc.gradient())
        gpu.apply_updates(it)
        orc.apply_updates(it)
        _sync_conductances(gpu, orc, opt)
    assert gpu.info().tc_fallbacks == 0


def test_big_tiles_auto_calibration():
    opt = aam_options(tile=None, rows=320, cols=288, adc_bits=6, i_fs=0.0, lr=0.2)
    opt.adc_cal_batches = 2  # the second batch's backward freezes both directions
    W = normal((500, 300), 9, 0.05)
    gpu = xb.CrossbarCore(W, opt)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    _sync_conductances(gpu, orc, opt)
    x = rand((3, 500), 10, -0.1, 1.1)
    for it in range(3):
        assert np.array_equal(gpu.forward(x, True), orc.forward(x, True))
        dy = rand((3, 300), 11 + it)
        assert np.array_equal(gpu.backward(dy, 1.0), orc.backward(dy, 1.0))
        assert gpu.forward_adc_full_scale() == orc.stats()["fwd_i_fs"]
    assert gpu.forward_adc_full_scale() > 0


def test_big_tiles_fcm_refused():
    """The FCM kernels run one thread per crossbar line (<= 256 per CTA):
    circuit engines on larger tiles fail loudly, never approximated."""
    opt = aam_options(tile=None, rows=288, cols=272, adc_bits=7, i_fs=3e-4, engine=xb.EngineKind.fcm, r_col=2.0)
    with pytest.raises(xb.UnsupportedConfigError):
        xb.CrossbarCore(normal((300, 280), 12, 0.05), opt)
