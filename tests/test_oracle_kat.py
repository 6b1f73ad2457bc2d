"""Pins the CPU oracle to the reference's own known answers.

Runs oracle/tests/kat_oracle.cpp: a restatement of the reference unit tests
(test_converters.cpp, test_mapping.cpp, test_update.cpp, test_nn.cpp,
test_circuit.cpp AAM cases) against the oracle, same known answers and
tolerances, deviations marked in the source.
"""
import os
import subprocess


def test_oracle_known_answers(oracle_build):
    exe = os.path.join(oracle_build, "kat_oracle")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
