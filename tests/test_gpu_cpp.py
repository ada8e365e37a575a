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


def test_cpp_host_driver_runs_the_layer_loop(up):
    """examples/drop_layer_bench: score -> select -> compact driven from C++ only (the host
    mirror over the C ABI), graph-captured; it must run and drop tokens in the planted regime."""
    import json
    exe = os.path.join(ROOT, "examples", "_build", "drop_layer_bench")
    if not os.path.exists(exe):
        pytest.skip("examples/_build/drop_layer_bench not built")
    r = subprocess.run([exe, "--requests", "2", "--len", "8192", "--layers", "3", "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["tokens_per_s"] > 0 and 0.05 < line["retention_rho"] < 0.8
    assert line["launches_per_layer"] >= 6
