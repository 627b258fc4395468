"""The reference's own test suites run against this repository's library on
the B200: the drop-in claim, tested by the reference's tests rather than
ours.

tests/reference_suites/Makefile compiles, unchanged and from where they lie
in /root/reference/proj/tests,
* test_capi.cpp against include/phfem.h (the C ABI), and
* test_mesh / test_connectivity / test_refine / test_quadrature /
  test_assembly / test_solver / test_analysis / acceptance.cpp against
  include/phfem_cxx/*.hpp (the C++ API of proj/src/*.hpp),
each linked with libphfem.so only (no reference source is compiled into
them).  The binaries travel to the GPU box with the repo.

acceptance.cpp reports two criteria FAILED by design in the reference
itself (the paper's printed 8x8 matrix and Table 4; SURVEY finding 7); the
test checks every criterion's verdict and the measured error table against
the reference's own run (tests/golden/reference_acceptance.txt, made by
tools/gen_reference_acceptance.sh from the unmodified reference objects)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "build")
UNIT_SUITES = ["test_capi", "test_mesh", "test_connectivity", "test_refine", "test_quadrature", "test_assembly",
               "test_solver", "test_analysis"]


def _bin(name):
    p = os.path.join(BUILD, "ref_" + name)
    if not os.path.exists(p):
        pytest.skip(f"build/ref_{name} not built (needs /root/reference at build time)")
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("suite", UNIT_SUITES)
def test_reference_suite_passes(suite):
    r = subprocess.run([_bin(suite)], capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-2000:])
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "| 0 failed |" in r.stdout


def _criteria(text):
    out = []
    for line in text.splitlines():
        m = re.match(r"\[(PASS|FAIL)\] criterion (\d+): (.*?)(?: -- (.*))?$", line)
        if m:
            out.append((m.group(1), int(m.group(2)), m.group(3).strip(), m.group(4) or ""))
    return out


@pytest.mark.gpu
def test_reference_acceptance_matches_reference_run():
    r = subprocess.run([_bin("acceptance")], capture_output=True, text=True, timeout=1800, cwd=ROOT)
    print(r.stdout)
    print(r.stderr[-3000:])
    with open(os.path.join(ROOT, "tests", "golden", "reference_acceptance.txt")) as f:
        want = _criteria(f.read())
    got = _criteria(r.stdout)
    assert [(v, n, w) for v, n, w, _ in got] == [(v, n, w) for v, n, w, _ in want]
    # the two by-design failures, with the reference's measured values
    fails = [(n, d) for v, n, _, d in got if v == "FAIL"]
    assert [n for n, _ in fails] == [3, 4]
    nums = lambda d: re.findall(r"\{[^}]*\}", d)  # noqa: E731
    assert nums(fails[1][1]) == nums([d for v, n, _, d in want if v == "FAIL"][1])
    assert r.returncode == 2


def test_reference_suites_link_our_library():
    for s in UNIT_SUITES + ["acceptance"]:
        out = subprocess.run(["ldd", _bin(s)], capture_output=True, text=True).stdout
        line = [l for l in out.splitlines() if "libphfem.so" in l]
        assert line and "paper_2509_11133_b200/lib/libphfem.so" in line[0], (s, out)
        # no reference object is linked in: every phfem:: symbol is undefined
        # in the binary and resolved by libphfem.so
        syms = subprocess.run(["nm", "-C", _bin(s)], capture_output=True, text=True).stdout
        defined = [l for l in syms.splitlines() if " T phfem::" in l]
        assert not defined, (s, defined[:5])
