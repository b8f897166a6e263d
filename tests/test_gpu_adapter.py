"""The C++ drop-in adapter (include/topopt_gpu.hpp) against the reference's
own functions: runs tests/cpp/_build/test_adapter (built from the reference
headers by __graft_entry__.build() in the build container)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "cpp", "_build", "test_adapter")
DRV = os.path.join(os.path.dirname(__file__), "cpp", "_build", "test_driver")


def test_cpp_adapter_matches_reference():
    if not os.path.exists(BIN):
        pytest.skip("adapter test binary not built (needs the reference headers at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout


def test_cpp_device_loop_matches_reference_driver():
    # gpu::run_optimization (state solve on the device) vs driver.hpp's loop
    if not os.path.exists(DRV):
        pytest.skip("driver test binary not built (needs the reference headers at build time)")
    r = subprocess.run([DRV], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout
