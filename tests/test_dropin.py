"""GPU: the C++ drop-in (deconv_b200.cpp replacing the reference's deconv.cpp,
over libvkrl.so) vs the unmodified reference in the same process.  The binary
is assembled by tests/dropin/Makefile (run by __graft_entry__.build())."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "dropin", "_build", "test_dropin")


@pytest.mark.gpu
def test_cpp_dropin_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("tests/dropin/_build/test_dropin not built (needs the reference headers: run build())")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
