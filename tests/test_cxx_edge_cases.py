"""The C++ API on edge cases (an element-less mesh, one element with all
faces Dirichlet / all Neumann (L = 0) / mixed through solve_direct, an element
repeating a node id, the level-1 cube), run through this library on the B200
and compared with the reference's own report of the same program
(tests/cxx_diff/edge_cases.cpp, built against the reference by
tests/cxx_diff/Makefile -> tests/golden/cxx_edge_cases.txt): tables, element
and Schur data and error messages exactly, solutions and error norms ('~'
lines) to 1e-9 relative."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "cxx_edge_cases")
GOLDEN = os.path.join(ROOT, "tests", "golden", "cxx_edge_cases.txt")


def test_cxx_edge_cases_match_reference():
    if not os.path.exists(BIN):
        pytest.skip("build/cxx_edge_cases not built (make -C tests/cxx_diff)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    got = out.stdout.splitlines()
    ref = open(GOLDEN).read().splitlines()
    assert len(got) == len(ref), (len(got), len(ref))
    for g, r in zip(got, ref):
        if r.startswith("~"):
            gk, *gv = g.split()
            rk, *rv = r.split()
            assert gk == rk and len(gv) == len(rv), (g, r)
            for a, b in zip(gv, rv):
                a, b = float(a), float(b)
                assert abs(a - b) <= 1e-9 * max(abs(b), 1e-300), (g, r)
        else:
            assert g == r, (g, r)
