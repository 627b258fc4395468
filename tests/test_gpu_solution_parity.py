"""Solution parity at the BASELINE.json sizes (configs 3, 4 and 5): the GPU
Schur path's Lambda, U, error norms, iteration count and verify verdict
against the CPU oracle's full solve of the same system.

The oracle's serial CG (the reference's own arithmetic, pinned bit for bit
to it in test_oracle_pins.py) takes 20-35 min per config, so its result is
cached in tests/golden/solution_cfg<N>.npz by tools/gen_solution_fixtures.py
(SURVEY.md 8(c) "Limits"): scalars plus Lambda and U at 32768 seeded random
indices each.  Bars (BASELINE.json north_star):

* Lambda, U: rel_l2 <= 1e-9 over the sampled entries, and the full norms
  ||Lambda||, ||U|| within 1e-9;
* L2 error (and the y-norm / multiplier-norm errors) to 3 significant
  digits;
* CG iterations within 2% (dot products are summed in a different order);
* verify_solution's verdict equal to the reference's (the reference itself
  refuses configs 3 and 5 at tol 1e-10, SURVEY finding 8); where the
  reference's deciding residual sits within 2% of its limit (config 3:
  1.011e-10 against 1e-10) a rounding-level difference may flip the verdict,
  and then the GPU's deciding residual must sit within 2% of the limit too;
* the face solve on the bit-identical S: the CG stops on its recursively
  updated residual, as the reference's does (sparse.cpp:187-192); the true
  residual ||S Lambda - rhs_neg|| drifts above that stop level on these
  ill-conditioned systems (measured: 5x on config 3 after 41.7k
  iterations, 1.3x on config 5), equally for the reference's own iterates
  (Lambda agrees to ~1e-11), so it is reported and bounded by 100 tol
  ||rhs_neg||.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ph = pytest.importorskip("paper_2509_11133_b200.phfem")
from paper_2509_11133_b200 import configs  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _fixture(cid):
    p = os.path.join(GOLDEN, f"solution_cfg{cid}.npz")
    if not os.path.exists(p):
        pytest.fail(f"missing fixture {p} (tools/gen_solution_fixtures.py {cid})")
    z = np.load(p)
    return json.loads(str(z["meta"])), z


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("cid", [3, 4, 5])
def test_full_size_solution_parity(cid):
    meta, z = _fixture(cid)
    cfg = configs.CONFIGS[cid]
    g = cfg.build()
    assert g.sizes()[1] == meta["ne"]
    u, lam, st = g.solve_unverified(cfg.problem, tol=cfg.tol)
    assert len(lam) == meta["l"]
    # Lambda and U at the sampled entries and in norm
    rl = _rel(lam[z["idx_lambda"]], z["lam"])
    ru = _rel(u[z["idx_u"]], z["u"])
    nl = abs(np.linalg.norm(lam) / meta["norm_lambda"] - 1.0)
    nu = abs(np.linalg.norm(u) / meta["norm_u"] - 1.0)
    print(json.dumps({"config": cfg.name, "rel_l2_lambda_sample": rl, "rel_l2_u_sample": ru, "norm_lambda_rel": nl,
                      "norm_u_rel": nu, "iterations": st["iterations"], "iterations_ref": meta["iterations"],
                      "err_l2": st["err_l2"], "err_l2_ref": meta["err_l2"], "accepted": st["accepted"],
                      "verify_ref": meta["verify_msg"] or "accepted"}))
    assert rl <= 1e-9 and ru <= 1e-9, (rl, ru)
    assert nl <= 1e-9 and nu <= 1e-9, (nl, nu)
    # error norms to 3 significant digits
    for k in ("err_y", "err_kappa", "err_l2"):
        assert abs(st[k] - meta[k]) <= 5e-4 * abs(meta[k]), (k, st[k], meta[k])
    assert abs(st["iterations"] - meta["iterations"]) <= 0.02 * meta["iterations"]
    # the same verify_solution verdict as the reference (solver.cpp:68-69)
    assert st["converged"]
    tol = cfg.tol
    margins = {"combined": st["residual"] / tol, "primal": st["r1"] / (tol * max(st["norm_rhs"], 1e-300)),
               "constraint": st["r2"] / (tol * (1.0 + st["norm_bd"]))}
    print(json.dumps({"verify_margins_gpu": margins, "reference_residual_over_tol": meta["residual"] / tol}))
    if st["accepted"] != (meta["verify_rc"] == 0):
        assert abs(meta["residual"] / tol - 1.0) <= 0.02 and abs(max(margins.values()) - 1.0) <= 0.02, (
            margins, meta["verify_msg"])
    elif meta["verify_rc"]:
        with pytest.raises(ph.SolverError, match="missed the residual target"):
            g.solve_ex(cfg.problem, tol=cfg.tol)
    # the reference's stopping rule on S (bit-identical to the oracle's,
    # test_gpu_fullsize_parity.py)
    sysg = g.assemble(cfg.problem)
    import scipy.sparse as sp

    S = sp.csr_matrix((sysg["s_val"], sysg["s_col"], sysg["s_rowptr"]), shape=(meta["l"], meta["l"]))
    res = np.linalg.norm(S @ lam - sysg["rhs_neg"])
    stop = min(cfg.tol * np.linalg.norm(sysg["rhs_neg"]),
               0.2 * cfg.tol * np.hypot(np.linalg.norm(sysg["rhs"]), np.linalg.norm(sysg["bd"])))
    print(json.dumps({"true_residual": float(res), "stop_level": float(stop), "ratio": float(res / stop)}))
    assert res <= 100 * cfg.tol * np.linalg.norm(sysg["rhs_neg"]), (res, stop)
