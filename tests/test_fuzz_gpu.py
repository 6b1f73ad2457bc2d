"""Seeded random-configuration sweep of the crossbar path against the
oracle (both VMM kernels): tile shapes 32..256 (ragged and rectangular),
weight/device bit splits, 1..12-bit ADCs with full scales across three
decades (saturating and near-empty codes), 1..8-bit input / error streams,
variation on and off.  y, dx and dW bit-exact given the same conductances
(DESIGN.md §2)."""
import numpy as np
import pytest

from helpers import aam_options, normal, rand, xb

pytestmark = pytest.mark.gpu

oracle_py = pytest.importorskip("oracle_py")

N_CASES = 64


def _case(seed):
    g = np.random.default_rng(9000 + seed)
    rows = int(g.choice([32, 64, 96, 128, 200, 256]))
    cols = int(g.choice([32, 64, 128, 72, 256]))
    wb, db = [(8, 2), (8, 1), (8, 4), (6, 2), (4, 4), (8, 8), (6, 3)][int(g.integers(7))]
    kw = dict(rows=rows, cols=cols, wb=wb, db=db, adc_bits=int(g.integers(1, 13)),
              i_fs=float(10 ** g.uniform(-5.3, -2.7)), act_bits=int(g.integers(1, 9)),
              error_bits=int(g.integers(1, 9)), sigma=float(g.choice([0.0, 0.1])), vseed=seed,
              r_row=float(g.choice([0.0, 1.0, 2.5])), r_col=float(g.choice([0.0, 1.0, 4.6])))
    K, N, M = int(g.integers(1, 521)), int(g.integers(1, 401)), int(g.integers(1, 34))
    return K, N, M, kw


@pytest.mark.parametrize("kernel", [0, 1])
@pytest.mark.parametrize("seed", range(N_CASES))
def test_random_configuration_bit_exact(seed, kernel):
    K, N, M, kw = _case(seed)
    opt = aam_options(**kw)
    W = normal((K, N), 100 + seed, 0.05)
    gpu = xb.CrossbarCore(W, opt)
    gpu.select_kernel(kernel)
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    for s in range(opt.map.num_slices()):
        for p in range(2):
            for t in range(orc.grid_rows * orc.grid_cols):
                orc.set_nonideal(s, p, t, gpu.nonideal(s, p, t))
    x = rand((M, K), 200 + seed, -0.2, 1.2)
    y_g, y_o = gpu.forward(x, True), orc.forward(x, True)
    assert np.array_equal(y_g, y_o), (kw, np.max(np.abs(y_g - y_o)))
    dy = rand((M, N), 300 + seed, -1.0, 1.0)
    dx_g, dx_o = gpu.backward(dy, 1.0), orc.backward(dy, 1.0)
    assert np.array_equal(dx_g, dx_o), (kw, np.max(np.abs(dx_g - dx_o)))
    assert np.array_equal(gpu.gradient(), orc.gradient())
