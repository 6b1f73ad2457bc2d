"""ADC-code flips of the snapped exactness contract against the literal model.

TEST INFRASTRUCTURE (imported by tests/ and tools/flip_report.py only).

The reference sums I = V.G over unsnapped fp64 conductances
(/root/reference/proj/core/src/layers.cpp:260-263, 356-361) and quantises
scaled = I / i_fs * maxc with llround (converters.cpp:79-87).  The GPU
evaluates the same formula on conductances snapped to a 2^-e grid
(DESIGN.md section 2), bit-exact against the oracle's `snapped` mode.  This
module runs the oracle in both modes on identical seeded inputs and counts
the conversions whose code differs: the only place the GPU contract and the
reference's arithmetic part ways.

For a sampled layer both oracle cores convert only the crossbar tiles the
sample needs (tile column tc for the forward, tile row tr for the backward);
variation and AAM are evaluated per tile with the layer's global device
index, so those tiles equal the full layer's.
"""
from __future__ import annotations

import numpy as np

import oracle_py


def sample_rows(x, dy, n, seed):
    """n random batch rows plus the rows holding max|x| and max|dy| (the
    batch-wide quantizer scales then equal the full batch's)."""
    rng = np.random.default_rng(seed)
    rows = set(rng.choice(x.shape[0], size=min(n, x.shape[0]), replace=False).tolist())
    rows.add(int(np.unravel_index(np.argmax(np.abs(x)), x.shape)[0]))
    rows.add(int(np.unravel_index(np.argmax(np.abs(dy)), dy.shape)[0]))
    return np.array(sorted(rows))


def _k_out(opt, layer_scale, step):
    """layers.cpp:272-281 / 369-377: the fp64 factor one ADC LSB of the
    shift-added total is worth (step = sx forward, step_e backward)."""
    vu = opt.dac.v_fs / (2.0 ** opt.dac.bits - 1.0)
    F = (layer_scale / (opt.crossbar.g_max - opt.crossbar.g_min)) * (
        (2.0 ** opt.map.device_bits - 1.0) / (2.0 ** opt.map.weight_bits - 1.0))
    return step * F / vu * (opt.adc.i_fs / (2.0 ** opt.adc.bits - 1.0))


def _cmp(cl, cs):
    d = cl.astype(np.int64) - cs.astype(np.int64)
    nz = np.count_nonzero(d)
    return {"conversions": int(cl.size), "flips": int(nz), "rate": float(nz / max(1, cl.size)),
            "max_abs_code_delta": int(np.max(np.abs(d))) if cl.size else 0}


def copy_gpu_tiles(gpu, orc, opt, tiles):
    """Feeds the GPU's snapped conductances of `tiles` to a snapped oracle
    core; returns how many values its own regeneration produced differently
    (CUDA vs glibc libm in the variation Gaussian: at most one grid step)."""
    flips = 0
    for s in range(opt.map.num_slices()):
        for p in range(2):
            for t in tiles:
                g = gpu.nonideal(s, p, t)
                o = orc.nonideal(s, p, t)
                assert np.all(np.abs(g - o) <= 1e-5 * np.abs(o))
                flips += int(np.count_nonzero(g != o))
                orc.set_nonideal(s, p, t, g)
    return flips


def flip_stats(W, opt, x, dy, tcs, trs, gpu=None):
    """Literal vs snapped oracle on the same inputs: forward on tile columns
    tcs, backward on tile rows trs (x, dy: the sampled batch rows).  Returns
    per-direction flip counts and the output deviation in k_out units (one
    ADC LSB of the integer total).  With `gpu` (a CrossbarCore over the same
    W and options) the snapped core first takes the GPU's conductances, and
    the snapped outputs are returned under "y_snapped" / "dx_snapped" for a
    bit-exact comparison with the GPU's."""
    T_r, T_c = opt.map.tile_rows, opt.map.tile_cols
    GR, GC = -(-W.shape[0] // T_r), -(-W.shape[1] // T_c)
    tiles = sorted({tr * GC + tc for tc in tcs for tr in range(GR)} | {tr * GC + tc for tr in trs for tc in range(GC)})
    out = {}
    ys, dxs, codes = {}, {}, {}
    for mode in ("literal", "snapped"):
        orc = oracle_py.OracleCore(W, opt, snapped=(mode == "snapped"), tiles=tiles)
        if gpu is not None and mode == "snapped":
            out["libm_conductance_flips"] = copy_gpu_tiles(gpu, orc, opt, tiles)
        orc.record_codes(True)
        ys[mode] = orc.forward_tiles(x, tcs, True)
        cf = orc.last_codes()
        dxs[mode] = orc.backward_tiles(dy, trs, 1.0)
        cb = orc.last_codes()
        codes[mode] = (cf, cb)
        scale = orc.stats()["layer_scale"]
    fwd = _cmp(codes["literal"][0], codes["snapped"][0])
    bwd = _cmp(codes["literal"][1], codes["snapped"][1])
    sx = opt.act_full_scale / (2.0 ** opt.act_bits - 1.0)
    se = float(np.max(np.abs(dy)))
    step_e = se / (2.0 ** opt.error_bits - 1.0) if se > 0 else 0.0
    cols = np.concatenate([np.arange(tc * T_c, min((tc + 1) * T_c, W.shape[1])) for tc in tcs])
    rows = np.concatenate([np.arange(tr * T_r, min((tr + 1) * T_r, W.shape[0])) for tr in trs])
    kf, kb = _k_out(opt, scale, sx), _k_out(opt, scale, step_e)
    dyv = np.abs(ys["literal"][:, cols] - ys["snapped"][:, cols])
    dxv = np.abs(dxs["literal"][:, rows] - dxs["snapped"][:, rows])
    fwd["max_abs_dy_lsb"] = float(np.max(dyv) / kf) if dyv.size else 0.0
    bwd["max_abs_dx_lsb"] = float(np.max(dxv) / kb) if dxv.size and kb > 0 else 0.0
    fwd["outputs_changed"] = int(np.count_nonzero(dyv))
    bwd["outputs_changed"] = int(np.count_nonzero(dxv))
    out["forward"], out["backward"] = fwd, bwd
    if gpu is not None:
        out["y_snapped"], out["dx_snapped"] = ys["snapped"], dxs["snapped"]
    out["sample"] = {"batch_rows": int(x.shape[0]), "tile_cols": list(map(int, tcs)), "tile_rows": list(map(int, trs)),
                     "tiles_converted": len(tiles)}
    return out
