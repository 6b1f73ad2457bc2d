"""Full-size parity: the GPU runs BASELINE.json's workloads at their real
sizes; the oracle checks them on samples it can finish in seconds.

Sampling is exact, not statistical:
  * forward y[b, j] depends on x row b, the conductance column block of j and
    the batch-wide activation scale max|x|; backward dx[b, i] on dy row b,
    the conductance row block of i and max|dy|.  The sampled batch rows
    always include the rows holding max|x| and max|dy|, so the oracle's
    quantizer scales equal the full batch's;
  * a sampled tile column / row block is checked on an oracle core built from
    that block of W (which holds the global max|W|, so the layer scale is the
    same) with the GPU's conductances copied in tile by tile;
  * dW needs the whole batch: the oracle computes it alone (forward_tiles /
    backward_tiles with no tiles = quantize + dW contract only).
Bars as in test_parity_gpu.py: y, dx and dW bit-exact.
"""
import numpy as np
import pytest

from helpers import xb

pytestmark = pytest.mark.gpu

oracle_py = pytest.importorskip("oracle_py")
flips = pytest.importorskip("flips")
from paper_2002_11151_b200 import configs  # noqa: E402


def _rows(x, dy, n, seed):
    rng = np.random.default_rng(seed)
    rows = set(rng.choice(x.shape[0], size=min(n, x.shape[0]), replace=False).tolist())
    rows.add(int(np.unravel_index(np.argmax(np.abs(x)), x.shape)[0]))
    rows.add(int(np.unravel_index(np.argmax(np.abs(dy)), dy.shape)[0]))
    return np.array(sorted(rows))


def _copy_tiles(gpu, orc, opt, gpu_tiles, same_numbering=True):
    """gpu_tiles[t_oracle] = t_gpu; returns how many snapped values the GPU's
    regeneration produced differently (libm ulp flips), after copying.  A
    block core numbers its tiles differently, so its own variation draws
    differ and only the copy is meaningful."""
    flips = 0
    for s in range(opt.map.num_slices()):
        for p in range(2):
            for to, tg in enumerate(gpu_tiles):
                g = gpu.nonideal(s, p, tg)
                o = orc.nonideal(s, p, to)
                if same_numbering:
                    assert np.all(np.abs(g - o) <= 1e-5 * np.abs(o))
                flips += int(np.count_nonzero(g != o))
                orc.set_nonideal(s, p, to, g)
    return flips


def _run_gpu(cfg, layer, kernel=0):
    opt = cfg.options()
    W = cfg.weights(layer)
    x = cfg.inputs(layer)
    dy = cfg.errors(layer)
    gpu = xb.CrossbarCore(W, opt)
    gpu.select_kernel(kernel)
    y = gpu.forward(x, True)
    dx = gpu.backward(dy, 1.0)
    return opt, W, x, dy, gpu, y, dx


def _check_dw(gpu, W, x, dy, opt):
    orc = oracle_py.OracleCore(W, opt, snapped=True)
    orc.forward_tiles(x, [], True)
    orc.backward_tiles(dy, [], 1.0, compute_dw=True)
    dw_o = orc.gradient()
    dw_g = gpu.gradient()
    assert np.array_equal(dw_g, dw_o), np.max(np.abs(dw_g - dw_o))


def _check_blocks(cfg, opt, W, x, dy, gpu, y, dx, n_rows=12, n_blocks=2):
    """Forward on sampled tile columns, backward on sampled tile rows, each
    through an oracle core built from that block of W."""
    T = opt.map.tile_rows
    GR = (W.shape[0] + T - 1) // T
    GC = (W.shape[1] + T - 1) // T
    rows = _rows(x, dy, n_rows, 7)
    imax, jmax = np.unravel_index(np.argmax(np.abs(W)), W.shape)
    rng = np.random.default_rng(11)
    # forward: tile columns holding max|W| (exact layer scale) + random others
    # through the FULL-width core when it is small, else per-block cores
    tcs = sorted({int(jmax // T)} | set(rng.choice(GC, size=min(n_blocks, GC), replace=False).tolist()))
    trs = sorted({int(imax // T)} | set(rng.choice(GR, size=min(n_blocks, GR), replace=False).tolist()))
    if W.size <= 4096 * 4096:
        orc = oracle_py.OracleCore(W, opt, snapped=True)
        n_flips = _copy_tiles(gpu, orc, opt, range(GR * GC))
        n_vals = GR * GC * 2 * opt.map.num_slices() * T * T
        print(f"\n{cfg.name}: {n_flips} snapped conductances of {n_vals} differ (libm)")
        assert n_flips <= max(4, 1e-6 * n_vals)
        y_o = orc.forward_tiles(x[rows], tcs, True)
        dx_o = orc.backward_tiles(dy[rows], trs, 1.0)
        for tc in tcs:
            cs = slice(tc * T, min((tc + 1) * T, W.shape[1]))
            assert np.array_equal(y[rows][:, cs], y_o[:, cs]), (tc, np.max(np.abs(y[rows][:, cs] - y_o[:, cs])))
        for tr in trs:
            rs = slice(tr * T, min((tr + 1) * T, W.shape[0]))
            assert np.array_equal(dx[rows][:, rs], dx_o[:, rs]), (tr, np.max(np.abs(dx[rows][:, rs] - dx_o[:, rs])))
        return
    # per-block oracle cores; only the blocks holding max|W| keep the layer scale
    tc = int(jmax // T)
    cs = slice(tc * T, min((tc + 1) * T, W.shape[1]))
    orc = oracle_py.OracleCore(W[:, cs], opt, snapped=True)
    _copy_tiles(gpu, orc, opt, [tr * GC + tc for tr in range(GR)], False)
    y_o = orc.forward(x[rows], True)
    assert np.array_equal(y[rows][:, cs], y_o), np.max(np.abs(y[rows][:, cs] - y_o))
    tr = int(imax // T)
    rs = slice(tr * T, min((tr + 1) * T, W.shape[0]))
    orc = oracle_py.OracleCore(W[rs, :], opt, snapped=True)
    _copy_tiles(gpu, orc, opt, [tr * GC + c for c in range(GC)], False)
    orc.forward_tiles(x[rows][:, rs], [], True)
    dx_o = orc.backward(dy[rows], 1.0)
    assert np.array_equal(dx[rows][:, rs], dx_o), np.max(np.abs(dx[rows][:, rs] - dx_o))


def test_c2_4096_full_size():
    """configs[1] at the bench size: M=256, K=N=4096, 128x128 tiles."""
    cfg = configs.CONFIGS["c2-4096"]
    layer = cfg.layers[0]
    opt, W, x, dy, gpu, y, dx = _run_gpu(cfg, layer)
    _check_blocks(cfg, opt, W, x, dy, gpu, y, dx)
    _check_dw(gpu, W, x, dy, opt)


def test_c5_stress_8192_sampled_blocks():
    """C5: M=4096, K=N=8192, 256x256 crossbars, 1-bit devices, sigma 20%.

    The oracle holds the whole 8192^2 layer but converts only the sampled
    crossbar tiles (three tile columns for y, three tile rows for dx, each
    set including the one holding max|W|), so its variation draws and AAM
    use the layer's own device indices: the GPU's regenerated conductances
    are compared (libm flips counted and bounded) before they are fed back.
    dW: every batch row, on the tile column holding max|dy| (so the error
    quantizer's scale is the layer's), through a column-block oracle core."""
    cfg = configs.CONFIGS["c5"]
    layer = cfg.layers[0]
    opt, W, x, dy, gpu, y, dx = _run_gpu(cfg, layer)
    T = opt.map.tile_rows
    GR, GC = -(-W.shape[0] // T), -(-W.shape[1] // T)
    rows = _rows(x, dy, 6, 7)
    imax, jmax = np.unravel_index(np.argmax(np.abs(W)), W.shape)
    rng = np.random.default_rng(13)
    tcs = sorted({int(jmax // T)} | set(rng.choice(GC, size=2, replace=False).tolist()))
    trs = sorted({int(imax // T)} | set(rng.choice(GR, size=2, replace=False).tolist()))
    tiles = sorted({tr * GC + tc for tc in tcs for tr in range(GR)} | {tr * GC + tc for tr in trs for tc in range(GC)})
    orc = oracle_py.OracleCore(W, opt, snapped=True, tiles=tiles)
    n_flips = flips.copy_gpu_tiles(gpu, orc, opt, tiles)
    n_vals = len(tiles) * 2 * opt.map.num_slices() * T * T
    print(f"\nC5: {len(tiles)} tiles compared, {n_flips} snapped conductances of {n_vals} differ (libm)")
    assert n_flips <= max(4, 1e-6 * n_vals)
    y_o = orc.forward_tiles(x[rows], tcs, True)
    dx_o = orc.backward_tiles(dy[rows], trs, 1.0)
    for tc in tcs:
        cs = slice(tc * T, (tc + 1) * T)
        assert np.array_equal(y[rows][:, cs], y_o[:, cs]), tc
    for tr in trs:
        rs = slice(tr * T, (tr + 1) * T)
        assert np.array_equal(dx[rows][:, rs], dx_o[:, rs]), tr
    del orc
    # dW[:, j] needs every batch row but only column j of dy
    jd = int(np.unravel_index(np.argmax(np.abs(dy)), dy.shape)[1])
    cs = slice((jd // T) * T, (jd // T + 1) * T)
    ob = oracle_py.OracleCore(W[:, cs], opt, snapped=True, tiles=[])
    ob.forward_tiles(x, [], True)
    ob.backward_tiles(dy[:, cs], [], 1.0, compute_dw=True)
    dw_g = gpu.gradient()[:, cs]
    assert np.array_equal(dw_g, ob.gradient()), np.max(np.abs(dw_g - ob.gradient()))


@pytest.mark.parametrize("cfg_name,layer_idx", [("c4", 0), ("c4", -1), ("c3", 1), ("c3", 13), ("c1", 0)])
def test_im2col_and_mlp_layers_full_size(cfg_name, layer_idx):
    """C3/C4 im2col GEMMs at full M (131072 / 401408 patch rows, ragged N=16,
    K=27/147) and the C1 MLP layer: sampled rows for y/dx, full-batch dW."""
    cfg = configs.CONFIGS[cfg_name]
    layer = cfg.layers[layer_idx]
    opt, W, x, dy, gpu, y, dx = _run_gpu(cfg, layer)
    _check_blocks(cfg, opt, W, x, dy, gpu, y, dx)
    _check_dw(gpu, W, x, dy, opt)
