"""GPU FCM / interp-FCM regeneration against the oracle's restatement of
fcm.cpp:18-224 and distortion.cpp:10-48 (same Thomas recurrences, same
operation order): converted conductances bit-identical up to libm ulp flips
of the variation multipliers (counted), then y / dx / dW bit-exact, and
regeneration after updates (the interp engine refreshing every
interp_interval updates) tracked over several iterations."""
import numpy as np
import pytest

from helpers import aam_options, normal, rand, xb

pytestmark = pytest.mark.gpu

oracle_py = pytest.importorskip("oracle_py")


def _opts(engine, base=None, interval=10, sigma=0.0, **kw):
    o = aam_options(tile=64, adc_bits=6, i_fs=6e-5, sigma=sigma, r_row=1.0, r_col=4.6, vseed=5, useed=9, **kw)
    o.engine = engine
    if base is not None:
        o.interp_base = base
    o.interp_interval = interval
    return o


def _compare_tiles(gpu, orc, opt, sync=True):
    flips, worst = 0, 0.0
    for s in range(opt.map.num_slices()):
        for p in range(2):
            for t in range(orc.grid_rows * orc.grid_cols):
                g, o = gpu.nonideal(s, p, t), orc.nonideal(s, p, t)
                flips += int(np.count_nonzero(g != o))
                worst = max(worst, float(np.max(np.abs(g - o) / np.maximum(np.abs(o), 1e-300))))
                if sync:
                    orc.set_nonideal(s, p, t, g)
    return flips, worst


ENGINES = [
    (xb.EngineKind.fcm, None),
    (xb.EngineKind.interp_fcm, xb.EngineKind.fcm),
    (xb.EngineKind.interp_fcm, xb.EngineKind.aam),
]


@pytest.mark.parametrize("sigma", [0.0, 0.1])
@pytest.mark.parametrize("eng", range(len(ENGINES)))
def test_circuit_engine_vmm_and_regeneration(eng, sigma):
    engine, base = ENGINES[eng]
    opt = _opts(engine, base, interval=2, sigma=sigma, v=0.5, gamma=1.0, lr=0.3)
    K, N, M = 100, 72, 6
    W = normal((K, N), 3, 0.05)
    gpu = xb.CrossbarCore(W, opt)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    flips, worst = _compare_tiles(gpu, orc, opt)
    assert worst <= 1e-12 and flips <= 4, (flips, worst)
    x = rand((M, K), 4, 0.0, 1.0)
    dy = rand((M, N), 5)
    for it in range(4):  # interp: refresh at 0, 2, 4; apply at 1, 3
        y_g, y_o = gpu.forward(x, True), orc.forward(x, True)
        assert np.array_equal(y_g, y_o), (it, np.max(np.abs(y_g - y_o)))
        dx_g, dx_o = gpu.backward(dy, 1.0), orc.backward(dy, 1.0)
        assert np.array_equal(dx_g, dx_o), (it, np.max(np.abs(dx_g - dx_o)))
        assert np.array_equal(gpu.gradient(), orc.gradient())
        gpu.apply_updates(it)
        orc.apply_updates(it)
        for s in range(opt.map.num_slices()):  # continue from the GPU master (libm ulps in exp/log/cos)
            ug, uo = gpu.master_diff(s), orc.master(s)
            assert np.max(np.abs(ug - uo)) <= 1e-12 * max(1e-30, np.max(np.abs(uo)))
            orc.set_master(s, ug)
        # each side regenerated from its own master inside apply_updates (an
        # extra regenerate would age the interp cache past its interval)
        flips, worst = _compare_tiles(gpu, orc, opt)
        assert worst <= 1e-9 and flips <= 8, (it, flips, worst)
    # layers.cpp:145-176: one refresh at construction, then every update
    # (fcm) or every interp_interval-th update (interp_fcm)
    expect = 1 + (4 if engine == xb.EngineKind.fcm else sum(1 for u in range(1, 5) if u % 2 == 0))
    assert gpu.refresh_count() == expect


def test_fcm_distortion_grows_with_column_index_on_gpu():
    """test_circuit.cpp:179-190 through the GPU engine: a uniform g_min tile."""
    opt = _opts(xb.EngineKind.fcm)
    gpu = xb.CrossbarCore(np.zeros((64, 64)), opt)  # zero weights: every device at g_min
    g = gpu.nonideal(0, 0, 0)
    d = 1.0 - g / opt.crossbar.g_min
    assert np.all(d > 0) and np.all(np.diff(d, axis=1) > 0)


def test_fcm_non_convergence_raises():
    """test_circuit.cpp:209-237: a starved iteration budget on a strongly coupled tile."""
    opt = _opts(xb.EngineKind.fcm)
    opt.crossbar.g_min, opt.crossbar.g_max = 1e-3, 1e-2
    opt.crossbar.r_row = opt.crossbar.r_col = 50.0
    opt.crossbar.rows = opt.crossbar.cols = opt.map.tile_rows = opt.map.tile_cols = 16
    opt.fcm_tol, opt.fcm_max_iter = 1e-12, 1
    with pytest.raises(xb.ConvergenceError):
        xb.CrossbarCore(normal((16, 16), 1, 0.05), opt)
