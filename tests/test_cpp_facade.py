"""The C++ entry points (include/hankel_b200.hpp, namespace hankel::b200) that
keep the reference's proj/include/hankel API over the C ABI: the reference's
own unit-test cases (test_ldlt / test_inversion / test_jacobi / test_pipeline /
test_moments), compiled as tests/cpp/test_facade.cpp.  On CPU the host-only
cases run and the device cases report themselves skipped; on the GPU every
case must run (--require-gpu)."""
import subprocess

import pytest


def test_facade_host_cases(facade_bin):
    out = subprocess.run([facade_bin], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failed" in out.stdout


@pytest.mark.gpu
def test_facade_device_cases(facade_bin):
    out = subprocess.run([facade_bin, "--require-gpu"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "skipped" not in out.stdout and "0 failed" in out.stdout
