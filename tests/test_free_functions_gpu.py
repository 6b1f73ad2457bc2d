"""The free-function half of the operator API (mapping.hpp:92-109,
update.hpp:25-52) on the GPU against the oracle: map_weights,
apply_variation, update::apply_update (master only), scale_gradient,
nonlinear_update, write_noise, reconstruct_output, CrossbarCore.weights().
The C++ restatement of the reference's test_update.cpp / test_mapping.cpp
runs through tests/test_cpp_api.py."""
import numpy as np
import pytest

from helpers import aam_options, normal, rand, xb

pytestmark = pytest.mark.gpu

oracle_py = pytest.importorskip("oracle_py")


def test_map_weights_matches_core_and_oracle():
    opt = aam_options(tile=64, wb=8, db=2, sigma=0.1, vseed=3)
    W = normal((100, 80), 1, 0.05)
    t = xb.map_weights(W, opt.map, opt.crossbar)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    core = xb.CrossbarCore(W, opt)
    assert (t.grid_rows(), t.grid_cols(), t.num_slices()) == (2, 2, 4)
    for s in range(4):
        assert np.array_equal(t.master_diff(s), orc.master(s))
        assert np.array_equal(core.weights().master_diff(s), orc.master(s))
    assert np.array_equal(t.implied_weights(), orc.implied_weights())
    # variation: the device Gaussian vs glibc, ulp level
    g = t.ideal_working(1, xb.Polarity.neg)
    for tr in range(2):
        for tc in range(2):
            blk = g[tr * 64:(tr + 1) * 64, tc * 64:(tc + 1) * 64]
            assert np.allclose(blk, t.ideal_tile(1, xb.Polarity.neg, tr, tc), rtol=0, atol=0)
    assert np.all(g >= opt.crossbar.g_min * 1e-12) and np.all(g <= opt.crossbar.g_max)
    v = xb.apply_variation(t, 0.0, 9)
    assert np.array_equal(v.ideal_working(0, xb.Polarity.pos), t.master_polarity(0, xb.Polarity.pos))
    assert np.array_equal(v.master_diff(2), t.master_diff(2))


@pytest.mark.parametrize("v,gamma", [(0.0, 0.0), (0.5, 0.0), (0.3, 2.0)])
def test_apply_update_master_only_vs_oracle(v, gamma):
    """update.cpp:43-88: the GPU free function equals the oracle's
    apply_updates master (same dW) -- 1e-12 relative (CUDA vs glibc libm in
    exp / log / cos) -- and changes nothing else."""
    opt = aam_options(tile=64, wb=8, db=2, v=v, gamma=gamma, lr=0.1, useed=77)
    W = normal((96, 72), 2, 0.05)
    dW = normal((96, 72), 3, 0.02)
    t = xb.map_weights(W, opt.map, opt.crossbar)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    for it in range(3):
        xb.apply_update(t, dW, opt.update, it)
        orc.set_gradient(dW)
        orc.apply_updates(it)
        for s in range(opt.map.num_slices()):
            ug, uo = t.master_diff(s), orc.master(s)
            assert np.max(np.abs(ug - uo)) <= 1e-12 * np.max(np.abs(uo))
            if v == 0.0 and gamma == 0.0:
                assert np.array_equal(ug, uo)
    with pytest.raises(ValueError):
        xb.apply_update(t, dW[:, :10], opt.update, 9)
    bad = dW.copy()
    bad[0, 0] = np.nan
    before = t.master_diff(0)
    with pytest.raises(ValueError, match="finite"):
        xb.apply_update(t, bad, opt.update, 9)
    assert np.array_equal(t.master_diff(0), before)


def test_elementwise_helpers():
    cfg = xb.CrossbarConfig(g_min=1e-6, g_max=1e-5)
    spec = xb.UpdateSpec(v=1.0, layer_scale=0.5)
    dW = rand((5, 7), 4)
    assert np.array_equal(xb.scale_gradient(dW, spec, cfg), dW * ((cfg.g_max - cfg.g_min) / 0.5))
    with pytest.raises(xb.ConfigError):
        xb.scale_gradient(dW, xb.UpdateSpec(layer_scale=0.0), cfg)
    g = np.linspace(cfg.g_min, cfg.g_max, 11)
    dg = np.linspace(-1e-6, 1e-6, 11)
    out = xb.nonlinear_update(g, dg, spec, cfg)
    x = np.where(dg >= 0, (g - cfg.g_min) / 9e-6, (cfg.g_max - g) / 9e-6)
    assert np.allclose(out, dg * np.exp(-1.0 * x), rtol=1e-15, atol=0)
    with pytest.raises(ValueError):
        xb.nonlinear_update(2e-5, 1e-7, spec, cfg)
    r = xb.CounterRng(42, 7)
    h = xb.CounterRng(42, 7)
    n = xb.write_noise(1e-9, xb.UpdateSpec(gamma=5.0), cfg, r)
    assert r.counter == 2
    assert abs(n - 5.0 * np.sqrt(9e-6 * 1e-9) * h.gaussian()) <= 1e-13 * abs(n)
    assert xb.write_noise(0.0, xb.UpdateSpec(gamma=5.0), cfg, r) == 0.0 and r.counter == 2
    spec2 = xb.MappingSpec(weight_bits=4, device_bits=2)
    pos = [np.full(3, 7.0), np.full(3, 2.0)]
    assert np.array_equal(xb.reconstruct_output(pos, [np.zeros(3)] * 2, spec2, 0.5), np.full(3, 0.5 * 15.0))
