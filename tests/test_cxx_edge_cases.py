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
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def _compare(got, ref):
    assert len(got) == len(ref), (len(got), len(ref), got[-5:])
    for g, r in zip(got, ref):
        if r.startswith("~"):
            gt, rt = g.split(), r.split()
            assert len(gt) == len(rt), (g, r)
            for a, b in zip(gt, rt):
                try:
                    x, y = float(a), float(b)
                except ValueError:
                    assert a == b, (g, r)
                    continue
                assert abs(x - y) <= 1e-9 * max(abs(y), 1e-300), (g, r)
        else:
            assert g == r, (g, r)


def _run(name, args=()):
    exe = os.path.join(ROOT, "build", name)
    if not os.path.exists(exe):
        pytest.skip(f"build/{name} not built (make -C tests/cxx_diff)")
    out = subprocess.run([exe, *args], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.splitlines()


def test_cxx_edge_cases_match_reference():
    _compare(_run("cxx_edge_cases"), open(os.path.join(GOLDEN_DIR, "cxx_edge_cases.txt")).read().splitlines())


def test_capi_edge_cases_match_reference(tmp_path):
    """The C ABI on meshes read from the reference's text format (one
    element all Dirichlet / all Neumann / mixed, no elements, a repeated node
    id, a bad index, a boundary face missing from the lists): counts, sizes,
    diameter, both solvers, every output file (byte checksums; solution
    files by value norm) and the error statuses and messages."""
    _compare(_run("capi_edge_cases", [str(tmp_path)]),
             open(os.path.join(GOLDEN_DIR, "capi_edge_cases.txt")).read().splitlines())
