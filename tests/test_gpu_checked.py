"""The parity suite against the bounds-checked build of the library
(paper_2509_11133_b200/lib/checked/libphfem.so, compiled with -DPHG_CHECKS:
device asserts on star positions, hash-probe counts, first-occurrence slots,
midpoint node ids, CG columns and segmented-sort positions; common.cuh).
compute-sanitizer is closed on the GPU pool (it left GPUs needing a reset),
so these checks stand in for its memcheck: an out-of-range index traps the
kernel and fails the run.  Cases: the config parity set (1 full, 3/4/5
scaled), the high-valence fans, error paths, the cube ladder."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2509_11133_b200", "lib", "checked", "libphfem.so")


def test_parity_suite_under_bounds_checks():
    if not os.path.exists(CHECKED):
        pytest.fail("checked build missing (build() makes lib/checked/libphfem.so)")
    env = dict(os.environ, PHFEM_LIB=CHECKED)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "test_gpu_parity.py")],
                       capture_output=True, text=True, env=env, cwd=ROOT, timeout=1500)
    print(r.stdout[-3000:])
    print(r.stderr[-3000:])
    assert r.returncode == 0, r.stdout[-3000:]
    assert "passed" in r.stdout and "failed" not in r.stdout
