import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    # torch first: its NCCL (libnccl.so.2) is then the one the library's dlopen
    # resolves to; the other order binds torch to an older NCCL and fails its import
    import torch  # noqa: F401


def _ensure_built(target):
    if not os.path.exists(os.path.join(ROOT, target)):
        subprocess.run(["make", "-C", ROOT, target], check=True, capture_output=True)


@pytest.fixture(scope="session")
def emu_bin():
    _ensure_built("build/emu_mp")
    return os.path.join(ROOT, "build", "emu_mp")


@pytest.fixture(scope="session")
def ref_driver():
    path = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
    if not os.path.exists(path):
        if not os.path.isdir("/root/reference"):
            pytest.skip("oracle/_ref not built and /root/reference absent")
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, capture_output=True)
    return path


@pytest.fixture(scope="session")
def facade_bin():
    """tests/cpp/test_facade.cpp: the reference's unit cases through include/hankel_b200.hpp."""
    _ensure_built("build/test_facade")
    return os.path.join(ROOT, "build", "test_facade")
