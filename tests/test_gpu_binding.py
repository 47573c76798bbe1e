"""The reference's own callers over the B200 path: integration/check_binding
(built against the reference sources, see integration/Makefile) runs
cobs::write_index, cobs::query, cobs::run_validation, cobs::oracle_query and
cobs::open_resident over cobs::gpu::DeviceIndexView (a cobs::IndexView whose
payload lives in HBM) and compares them with the device engine and the
device build from TermSets."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "check_binding")


@pytest.mark.gpu
def test_reference_callers_over_device_view(gpu):
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/check_binding not built (needs the reference sources)")
    r = subprocess.run([BIN, str(gpu)], capture_output=True, text=True, timeout=900)
    lines = r.stdout.splitlines()
    failed = [l for l in lines if l.startswith("[FAIL]")]
    assert r.returncode == 0 and not failed, r.stdout[-4000:] + r.stderr[-2000:]
    assert sum(l.startswith("[PASS]") for l in lines) >= 30


def test_binding_header_compiles_without_gpu():
    """The binding's header parses against the reference headers here (no
    GPU needed) -- skipped where the reference is absent."""
    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc):
        pytest.skip("reference headers absent")
    src = '#include "cobs_gpu_binding.hpp"\nint main() { return 0; }\n'
    r = subprocess.run(["g++", "-std=gnu++20", "-fsyntax-only", "-x", "c++", "-", "-I" + ref_inc,
                        "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(ROOT, "integration")],
                       input=src, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
