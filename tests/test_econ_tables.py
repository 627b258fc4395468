"""The economised series tables of problems.cuh (econ_trig / econ_exp) are
the ones tools/econ_tables.py derives, and their truncation error on each
class interval is below half an ulp (one ulp for the N = 5 class) (CPU, mpmath)."""
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytest.importorskip("mpmath")


def test_tables_match_generator():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "econ_tables.py")], capture_output=True,
                         text=True, check=True).stdout.splitlines()
    trig = [ln for ln in out if ln.startswith("trig")]
    exp = [ln for ln in out if ln.startswith("exp")]
    gen = [float.fromhex(v) for v in re.findall(r"0x[0-9a-f.]+p[+-]\d+", "\n".join(trig + exp))]
    src = open(os.path.join(ROOT, "paper_2509_11133_b200", "csrc", "problems.cuh")).read()
    body = src[src.index("econ_trig(int n)"):src.index("taylor_order(double r)")]
    shipped = [float.fromhex(v) if v.startswith("0x") else float(v)
               for v in re.findall(r"(0x[0-9a-f.]+p[+-]\d+|1\.0(?=[,}]))", body)]
    assert gen == shipped
    for ln in out:
        if ln.startswith("//"):
            errs = [float(x) for x in re.findall(r"(?:cos|sin|exp) ([0-9.e+-]+)", ln)]
            # half an ulp of 1 for N >= 6; one ulp (2.2e-16, +5%) for the N = 5 class
            bound = 2.35e-16 if ln.startswith("// N = 5,") else 5.6e-17
            assert len(errs) == 3 and max(errs) < bound, ln
