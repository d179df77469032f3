"""C++ link-level drop-in: a program written against the reference API, swapped onto
prlab::gpu:: (oracle/dropin_test.cpp, built here by oracle/Makefile), run on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "dropin_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="dropin_test not built (needs /root/reference at build time)")
def test_cpp_dropin_program():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "DROPIN OK" in r.stdout
