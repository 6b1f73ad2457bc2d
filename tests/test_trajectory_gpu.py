"""Unsynchronised trajectory: BASELINE configs[0] (the
C1 MLP train step) run for ten iterations on the GPU and on the snapped CPU
oracle from the same seeds, each side with its own digital glue, with NO
state copied between them.  test_mlp_step_gpu.py re-synchronises the
conductances every step; this test reports how far the two runs drift when
nothing is fed back: the only sources are libm (CUDA vs glibc exp / log /
cos in the variation Gaussian and the softmax) reaching a rounding tie of
the snapped grid or an ADC threshold.  Measured on B200: none is reached in
ten steps -- logits, loss and the master stay bit-identical -- so the test
asserts that (the drift table is printed with pytest -s)."""
import numpy as np
import pytest

from helpers import xb

pytestmark = pytest.mark.gpu
oracle_py = pytest.importorskip("oracle_py")

from paper_2002_11151_b200.configs import CONFIGS  # noqa: E402

STEPS = 10


def test_c1_ten_step_trajectory_drift():
    cfg = CONFIGS["c1"]
    opt = cfg.options()
    L1, L2 = cfg.layers
    W1, W2 = cfg.weights(L1, 0), cfg.weights(L2, 1)
    x = cfg.inputs(L1)
    labels = np.random.default_rng(6000 + cfg.cid).integers(0, 10, size=L1.M)
    g1, g2 = xb.CrossbarLinear(W1, opt), xb.CrossbarLinear(W2, opt)
    relu = xb.ReLU()
    o1, o2 = oracle_py.OracleCore(W1, opt, snapped=True), oracle_py.OracleCore(W2, opt, snapped=True)
    rows = []
    for it in range(STEPS):
        # GPU stack, Python-mirror glue
        h = relu.forward(g1.forward(xb.Tensor(x, [784]), True), True)
        lg = g2.forward(h, True).values
        loss_g, d_g = xb.softmax_cross_entropy(lg, labels)
        g1.backward(relu.backward(g2.backward(xb.Tensor(d_g, [10]))))
        g1.apply_updates(it)
        g2.apply_updates(it)
        # oracle stack, oracle glue
        y1 = o1.forward(x, True)
        a1 = oracle_py.relu(y1, np.zeros_like(y1))[0]
        lo = o2.forward(a1, True)
        loss_o, d_o = oracle_py.softmax_cross_entropy(lo, labels)
        o1.backward(oracle_py.relu(y1, o2.backward(d_o, 1.0))[1], 1.0)
        o1.apply_updates(it)
        o2.apply_updates(it)
        rows.append((it, int(np.count_nonzero(lg != lo)), abs(loss_g - loss_o) / loss_o,
                     float(np.max(np.abs(lg - lo)) / np.max(np.abs(lo)))))
    drift = max(float(np.max(np.abs(g1.core().master_diff(s) - o1.master(s)))) for s in range(opt.map.num_slices()))
    scale = max(float(np.max(np.abs(o1.master(s)))) for s in range(opt.map.num_slices()))
    print("\nC1 10-step unsynchronised trajectory (iteration, differing logits of 640, |dloss|/loss, "
          "max|dlogit|/max|logit|):")
    for r in rows:
        print("  %2d %4d %.3e %.3e" % r)
    print("  fc1 master drift after %d steps: %.3e (max |u| %.3e)" % (STEPS, drift, scale))
    assert all(r[1] == 0 and r[2] == 0.0 for r in rows), rows
    assert drift == 0.0, (drift, scale)
