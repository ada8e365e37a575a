"""GPU: run the C++ parity tests (tests/cpp/test_parity.cpp) built against the C++ host
mirror (include/uniprefill_b200.hpp) and the unmodified reference (oracle/_ref)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_build", "test_parity")


def test_cpp_parity_suite(up):
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build/test_parity not built (needs oracle/_ref)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
