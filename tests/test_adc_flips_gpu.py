"""ADC-code flips of the GPU's snapped contract against the literal fp64
model of the reference, on all five BASELINE.json configs (north star:
"any ADC code flips at threshold boundaries counted and reported").

The GPU runs each layer at full size; on sampled batch rows and crossbar
tiles the oracle is run twice on the same inputs -- `snapped` (holding the
GPU's own conductances) and `literal` (unsnapped fp64 sums in ascending row
order, layers.cpp:260-263 / converters.cpp:79-87):
  * GPU y / dx == snapped oracle, bit for bit (the exactness contract);
  * literal vs snapped: flip rate <= 1e-5 per conversion, and a flipped code
    moves by exactly one LSB.  (Each snapped conductance is within half a
    2^-e grid step, ~2^-33 g_max, of the literal one, so a column current
    moves by < 1e-6 of an ADC LSB at these resolutions.)
A 16-bit-ADC sensitivity case shows the counter is not vacuous.
"""
import numpy as np
import pytest

from helpers import aam_options, normal, rand, xb

pytestmark = pytest.mark.gpu

oracle_py = pytest.importorskip("oracle_py")
flips = pytest.importorskip("flips")
from paper_2002_11151_b200 import configs  # noqa: E402

RATE_BOUND = 1e-5


def _check(gpu, W, opt, x, dy, y, dx, rows, tcs, trs):
    r = flips.flip_stats(W, opt, x[rows], dy[rows], tcs, trs, gpu=gpu)
    T_r, T_c = opt.map.tile_rows, opt.map.tile_cols
    for tc in tcs:
        cs = slice(tc * T_c, min((tc + 1) * T_c, W.shape[1]))
        assert np.array_equal(y[rows][:, cs], r["y_snapped"][:, cs])
    for tr in trs:
        rs = slice(tr * T_r, min((tr + 1) * T_r, W.shape[0]))
        assert np.array_equal(dx[rows][:, rs], r["dx_snapped"][:, rs])
    for d in ("forward", "backward"):
        assert r[d]["rate"] <= RATE_BOUND, r
        assert r[d]["max_abs_code_delta"] <= 1, r
    assert r["libm_conductance_flips"] <= 4
    return r


@pytest.mark.parametrize("cfg_name,layer_idx,n_rows", [("c1", 0, 32), ("c1", 1, 32), ("c2-4096", 0, 32), ("c3", 1, 24),
                                                        ("c3", 13, 24), ("c4", 0, 12), ("c4", -2, 16), ("c5", 0, 6)])
def test_flips_vs_literal(cfg_name, layer_idx, n_rows):
    cfg = configs.CONFIGS[cfg_name]
    L = cfg.layers[layer_idx]
    opt = cfg.options()
    W, x, dy = cfg.weights(L, layer_idx % len(cfg.layers)), cfg.inputs(L), cfg.errors(L)
    gpu = xb.CrossbarCore(W, opt)
    y = gpu.forward(x, True)
    dx = gpu.backward(dy, 1.0)
    rows = flips.sample_rows(x, dy, n_rows, 3)
    GR, GC = -(-L.K // cfg.tile), -(-L.N // cfg.tile)
    rng = np.random.default_rng(5)
    tcs = sorted(set(rng.choice(GC, size=1).tolist()))
    trs = sorted(set(rng.choice(GR, size=1).tolist()))
    _check(gpu, W, opt, x, dy, y, dx, rows, tcs, trs)


def test_flip_counter_sensitivity_16bit_adc():
    """At 16 ADC bits the LSB is ~2^9 times finer than at 7, so the snap
    (< 1e-6 LSB at 7 bits) flips a measurable fraction of codes: the counter
    must see them, each one LSB, while the GPU stays bit-exact against the
    snapped oracle."""
    K, N, M = 512, 256, 64
    opt = aam_options(tile=128, adc_bits=16, i_fs=1.8e-4, r_col=4.6)
    W = normal((K, N), 1, 0.02)
    x, dy = rand((M, K), 2), rand((M, N), 3)
    gpu = xb.CrossbarCore(W, opt)
    y = gpu.forward(x, True)
    dx = gpu.backward(dy, 1.0)
    r = flips.flip_stats(W, opt, x, dy, [0, 1], [0, 1, 2, 3], gpu=gpu)
    assert np.array_equal(y[:, :256], r["y_snapped"][:, :256])
    assert np.array_equal(dx, r["dx_snapped"])
    assert r["forward"]["flips"] + r["backward"]["flips"] > 0
    assert r["forward"]["max_abs_code_delta"] == 1 or r["forward"]["flips"] == 0
    assert r["backward"]["max_abs_code_delta"] <= 1


def test_polarity_ties_after_one_update():
    """update.cpp:66-72: a device at u == 0 takes its active polarity from the
    sign of dg (the tie rule).  After one non-linear, noisy C3-style update
    (v = 1, gamma = 0.05: exp / log / cos on both sides), every device's
    polarity (sign of u) on the GPU equals the oracle's; ties and sign
    changes are counted."""
    cfg = configs.CONFIGS["c3"]
    L = cfg.layers[9]  # s2.2: 32768 x 288 x 32
    opt = cfg.options()
    W, x, dy = cfg.weights(L, 9), cfg.inputs(L, 9)[:2048], cfg.errors(L, 9)[:2048]
    gpu = xb.CrossbarCore(W, opt)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    S = opt.map.num_slices()
    u0 = [orc.master(s)[:L.K, :L.N] for s in range(S)]
    gpu.forward(x, True)
    orc.forward(x, True)
    gpu.backward(dy, 1.0)
    orc.backward(dy, 1.0)
    dW = gpu.gradient()
    assert np.array_equal(dW, orc.gradient())
    gpu.apply_updates(0)
    orc.apply_updates(0)
    ties = changed = mismatched = 0
    for s in range(S):
        ug, uo = gpu.master_diff(s)[:L.K, :L.N], orc.master(s)[:L.K, :L.N]
        ties += int(np.count_nonzero((u0[s] == 0) & (dW != 0)))
        changed += int(np.count_nonzero(np.sign(uo) != np.sign(u0[s])))
        mismatched += int(np.count_nonzero(np.sign(ug) != np.sign(uo)))
    print(f"u=0 ties {ties}, polarity changes {changed}, GPU/oracle polarity mismatches {mismatched}")
    assert ties > 0 and changed > 0
    assert mismatched == 0
