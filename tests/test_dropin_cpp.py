"""The C++ drop-in (include/rnntsim_cuda.hpp) run through the reference's own
acceptance checks in one binary (tests/cpp/test_dropin.cpp), built in the
build container by tests/cpp/Makefile (needs /root/reference headers) and
executed here on the B200."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def test_dropin_binary_built_or_buildable():
    if os.path.exists(BIN):
        return
    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("drop-in binary not built and the reference headers are absent")
    subprocess.run(["make", "-s", "-f", os.path.join(ROOT, "tests", "cpp", "Makefile")], check=True)
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_dropin_acceptance_on_gpu():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/test_dropin not built (needs the reference headers)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") >= 8
