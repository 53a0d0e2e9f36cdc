"""The reference-side C++ shim (integration/tileq_gpu.cpp) driven by ported
reference tests (integration/test_gpu_shim.cpp: test_infer.cpp:117-231,320-357,
test_io.cpp:220-280, test_moe.cpp:110-191) through libtileq_b200.so.

The binary is built where /root/reference exists (`make -C integration`,
run by __graft_entry__.build()) and travels with the repo snapshot."""
import os
import subprocess

import pytest

from conftest import REPO

BIN = os.path.join(REPO, "integration", "_build", "test_gpu_shim")


@pytest.mark.gpu
def test_reference_tests_through_the_shim():
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/test_gpu_shim not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600, cwd=os.path.dirname(BIN))
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout or "failures 0" in r.stdout, r.stdout[-2000:]


def test_shim_links_and_rejects_bad_layers_without_a_gpu():
    """Host-side checks of the shim (FormatError for an out-of-grid placement)
    run before any device call; the binary links against the product library."""
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/test_gpu_shim not built")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libtileq_b200.so" in out and "not found" not in out, out
