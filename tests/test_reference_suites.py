"""The reference's own C-ABI test suite (/root/reference/proj/tests/
test_capi.cpp, compiled unchanged against include/phfem.h and libphfem.so by
tests/reference_suites/Makefile) run on the B200: the drop-in claim, tested
by the reference's tests rather than ours."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "ref_test_capi")


@pytest.mark.gpu
def test_reference_capi_suite_passes():
    if not os.path.exists(BIN):
        pytest.skip("build/ref_test_capi not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(r.stdout)
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "| 0 failed |" in r.stdout


def test_reference_capi_suite_links_our_library():
    if not os.path.exists(BIN):
        pytest.skip("build/ref_test_capi not built")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    line = [l for l in out.splitlines() if "libphfem.so" in l]
    assert line and "paper_2509_11133_b200/lib/libphfem.so" in line[0], out
