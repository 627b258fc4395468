"""The face solve's two SpMV paths on the same element-major system give the
same iterates bit for bit: cg_spmv_em (the default: S read element-major
through each row's two slots) and the SELL-32 copy of elem_to_sell
(PHFEM_CG_SELL=1), whose row order and zero padding cg_spmv_em reproduces
(cg.cu).  The switch is read once per process, so each path runs in its own
interpreter; Lambda, the iteration count and the relative residual are
compared exactly on scaled configs 3 and 5 (Neumann faces: rows with one
element and slots without rows) and config 4 (Dirichlet on z = 0 only).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_2509_11133_b200 import configs
cfg = configs.CONFIGS[{cid}].scaled({factor})
m = cfg.build()
m.pipeline(cfg.problem, False)
lam, st = m.solve_faces(cfg.problem, tol=cfg.tol)
np.savez({out!r}, lam=lam, it=st["iterations"], rel=st["rel_residual"])
"""


def _run(tmp_path, cid, factor, sell):
    out = str(tmp_path / f"cg_{cid}_{int(sell)}.npz")
    env = dict(os.environ)
    env["PHFEM_CG_SELL"] = "1" if sell else "0"
    code = SCRIPT.format(root=ROOT, cid=cid, factor=factor, out=out)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


@pytest.mark.parametrize("cid,factor", [(3, 4), (5, 4), (4, 8)])
def test_element_major_spmv_matches_sell(tmp_path, cid, factor):
    a = _run(tmp_path, cid, factor, sell=False)
    b = _run(tmp_path, cid, factor, sell=True)
    assert int(a["it"]) == int(b["it"]) and int(a["it"]) > 0
    assert np.array_equal(a["lam"].view(np.uint64), b["lam"].view(np.uint64))
    assert float(a["rel"]) == float(b["rel"])
