"""The forward VMM has two epilogue loops (8 warps x 32 columns, 16 warps x
16 columns) chosen per layer shape; XBS_FWD_EW forces one.  Both must give
the same bits on every shape: the golden-fixture and precision tests (small
layers the heuristic sends to the 8-warp loop) are re-run in a subprocess with
each loop forced (the switch is read once per process)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("ew", ["8", "16"])
def test_forward_epilogue_variants_bit_exact(ew):
    env = dict(os.environ, XBS_FWD_EW=ew)
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_golden.py", "tests/test_precision_gpu.py",
                        "-m", "gpu", "-q", "-x", "-k", "not codes_above"], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
