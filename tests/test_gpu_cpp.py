"""The C++ mirror of the reference API (include/srtt_b200.hpp) drives the
engine end to end from a compiled C++ program."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def test_cpp_client():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)
    out = subprocess.run([os.path.join(HERE, "cpp", "test_capi")], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "tucker rel error" in out.stdout and "invalid_argument" in out.stdout
