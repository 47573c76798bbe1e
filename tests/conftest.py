import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")


def _ensure_built():
    lib = os.path.join(ROOT, "paper_1905_09624_b200", "_lib", "libcobs_gpu.so")
    synth = os.path.join(ROOT, "workloads", "_lib", "libcobs_synth.so")
    orc = os.path.join(ROOT, "oracle", "_build", "libcobs_oracle.so")
    if not (os.path.exists(lib) and os.path.exists(synth)):
        subprocess.run(["make", "-C", ROOT, "-j8", "lib"], check=True)
    if not os.path.exists(orc):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)


_ensure_built()


def have_gpu() -> bool:
    return os.path.exists("/dev/nvidiactl") or os.path.exists("/dev/nvidia0")


@pytest.fixture(scope="session")
def gpu():
    if not have_gpu():
        pytest.skip("no CUDA device")
    return 0
