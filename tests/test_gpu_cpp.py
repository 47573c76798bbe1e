"""Runs the C++ host-API parity suite (tests/cpp/test_cobs_b200.cpp) on the
device: the reference-shaped C++ tests over include/cobs_b200.hpp."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_cpp_host_api_suite(gpu):
    subprocess.run(["make", "-C", ROOT, "cpptest"], check=True, capture_output=True)
    r = subprocess.run([os.path.join(ROOT, "tests", "cpp", "test_cobs_b200")], capture_output=True,
                       text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_cpp_suite_compiles():
    """The C++ API header and the suite compile (no device needed)."""
    subprocess.run(["make", "-C", ROOT, "cpptest"], check=True, capture_output=True)
    assert os.path.exists(os.path.join(ROOT, "tests", "cpp", "test_cobs_b200"))
