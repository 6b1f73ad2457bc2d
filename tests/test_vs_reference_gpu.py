"""The GPU against the REFERENCE'S OWN CODE (oracle/_ref: the reference's
core sources compiled unchanged against the Eigen-API shim; built in the
development container, shipped with the snapshot).  The GPU evaluates the
snapped-grid contract bit-exactly (test_parity*_gpu.py); this measures what
that contract costs against the reference itself, on BASELINE configs[0]
(C1, both layers at full size) and configs[1] (C2-512), one training step:
  * non-ideal conductances within half a snap-grid step of the reference's;
  * ADC-code flips: y / dx elements that differ at all, each by at most one
    ADC code at one stream / slice weight, no more than 1e-5 of the ADC
    conversions behind them;
  * dW within 1e-12 max|dW| (exact-integer contract vs fp64 sums)."""
import numpy as np
import pytest

from helpers import xb

pytestmark = pytest.mark.gpu
ref_py = pytest.importorskip("ref_py")
if not ref_py.available():
    pytest.skip("reference build (oracle/_ref) absent", allow_module_level=True)

from paper_2002_11151_b200.configs import CONFIGS  # noqa: E402


def _k_out(opt, layer_scale, step):
    vu = opt.dac.v_fs / (2.0 ** opt.dac.bits - 1.0)
    F = (layer_scale / (opt.crossbar.g_max - opt.crossbar.g_min)) * (
        (2.0 ** opt.map.device_bits - 1.0) / (2.0 ** opt.map.weight_bits - 1.0))
    return step * F / vu * (opt.adc.i_fs / (2.0 ** opt.adc.bits - 1.0))


@pytest.mark.parametrize("cfg_name,layer_idx", [("c1", 0), ("c1", 1), ("c2-512", 0)])
def test_gpu_against_the_reference_code(cfg_name, layer_idx):
    cfg = CONFIGS[cfg_name]
    L = cfg.layers[layer_idx]
    opt = cfg.options()
    W, x, dy = cfg.weights(L, layer_idx), cfg.inputs(L, layer_idx), cfg.errors(L, layer_idx)
    gpu = xb.CrossbarCore(W, opt)
    T = opt.map.tile_rows
    GR, GC = -(-L.K // T), -(-L.N // T)
    ref = ref_py.RefCore(W, opt, T, opt.map.tile_cols, opt.map.num_slices(), GR * GC)
    g_rel = g_abs = 0.0
    for s in range(opt.map.num_slices()):
        for p in range(2):
            for t in range(GR * GC):
                a, b = gpu.nonideal(s, p, t), ref.nonideal(s, p, t)
                g_abs = max(g_abs, float(np.max(np.abs(a - b))))
                g_rel = max(g_rel, float(np.max(np.abs(a - b) / b)))
    # the snap moves each conductance by at most half a grid step 2^-e, e the
    # largest exponent with g_max 2^e <= 255^3 - 1
    e = int(np.floor(np.log2((255.0 ** 3 - 1) / opt.crossbar.g_max)))
    while opt.crossbar.g_max * 2.0 ** (e + 1) <= 255.0 ** 3 - 1:
        e += 1
    while opt.crossbar.g_max * 2.0 ** e > 255.0 ** 3 - 1:
        e -= 1
    half_step = 0.5 * 2.0 ** -e
    y_g, y_r = gpu.forward(x, True), ref.forward(x, True)
    dx_g, dx_r = gpu.backward(dy, 1.0), ref.backward(dy, 1.0)
    dw_g, dw_r = gpu.gradient(), ref.gradient()
    scale = float(np.max(np.abs(W)))
    kf = _k_out(opt, scale, opt.act_full_scale / (2.0 ** opt.act_bits - 1.0))
    kb = _k_out(opt, scale, float(np.max(np.abs(dy))) / (2.0 ** opt.error_bits - 1.0))
    fy, fx = int(np.count_nonzero(y_g != y_r)), int(np.count_nonzero(dx_g != dx_r))
    # one flipped code moves an output by one LSB times its stream / slice weight
    wmax = (2.0 ** opt.act_bits - 1.0) * (2.0 ** (opt.map.weight_bits - opt.map.device_bits))
    # ADC conversions behind each output: a flip rate <= 1e-5
    # per conversion bounds the outputs that may differ
    conv = cfg.adc_conversions(L)
    print(f"\n{cfg.name}/{L.name}: conductance max diff {g_abs:.3e} S = {g_abs / half_step:.3f} half grid steps "
          f"(max rel {g_rel:.2e}); y differs in {fy} of {y_g.size} ({conv['fwd']:.3g} conversions), dx in {fx} of "
          f"{dx_g.size} ({conv['bwd']:.3g}); max |dy| {np.max(np.abs(y_g - y_r)) / kf:.1f} LSB-weights, "
          f"max |ddx| {np.max(np.abs(dx_g - dx_r)) / kb:.1f}")
    assert g_abs <= half_step * (1 + 1e-6)  # + libm ulps of the variation multiplier
    assert fy <= max(2, 1e-5 * conv["fwd"]) and fx <= max(2, 1e-5 * conv["bwd"])
    assert np.max(np.abs(y_g - y_r)) <= wmax * kf * (1 + 1e-9)
    assert np.max(np.abs(dx_g - dx_r)) <= 2 * wmax * kb * (1 + 1e-9)
    assert np.max(np.abs(dw_g - dw_r)) <= 1e-12 * np.max(np.abs(dw_r))
