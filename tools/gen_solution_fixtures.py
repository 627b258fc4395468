"""Generate the full-size solution fixtures of configs 3, 4 and 5 (TEST
INFRASTRUCTURE; the GPU parity test tests/test_gpu_solution_parity.py reads
them).

For each config at its BASELINE.json size this runs the CPU oracle
(oracle/phfem_oracle.c, pinned bit-for-bit to the reference incl. the CG
iterates, tests/test_oracle_pins.py) through the reference's Schur path:

  Kuhn mesh -> face table -> assemble_system + build_schur -> pcg_jacobi with
  inner_cg_options (solver.cpp:78-86, sparse.cpp:163-212) -> element-local
  recovery -> verify_solution (solver.cpp:44-76) -> error norms + L2.

The oracle's serial CG is the reference's own arithmetic; config 4 takes
~30 min on one core, which is why the result is cached instead of re-run in
every GPU test (SURVEY.md 8(c) "Limits").  Lambda and U are too large to
commit (200-400 MB), so the fixture keeps:

* scalars: iterations, relative/constraint residuals, the verify verdict and
  message, norms of Lambda/U/rhs/b_D/rhs_neg, the three error norms;
* Lambda and U at 32768 seeded random indices each (counter RNG, seed 7),
  from which the test estimates rel_l2(GPU - oracle) over the sample.

Usage: python tools/gen_solution_fixtures.py 3 4 5   (writes
tests/golden/solution_cfg<N>.npz).  Run in the repo container (62 GB RAM);
the oracle is deterministic IEEE code built with -ffp-contract=off, so the
result does not depend on the host.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle_bind import Oracle  # noqa: E402
from paper_2509_11133_b200 import configs  # noqa: E402

NSAMPLE = 32768
SAMPLE_SEED = 7


def sample_indices(n: int, k: int = NSAMPLE, seed: int = SAMPLE_SEED) -> np.ndarray:
    """sorted distinct indices in [0, n) from the counter RNG"""
    u = configs.uniform(seed, np.arange(4 * k))
    idx = np.unique((u * n).astype(np.int64))
    return idx[:k] if idx.size >= k else idx


def run(cid: int, out_dir: str) -> dict:
    O = Oracle()
    cfg = configs.CONFIGS[cid]
    t0 = time.time()
    m = O.kuhn(cfg.nx, cfg.ny, cfg.nz, lx=cfg.lx, ly=cfg.ly, lz=cfg.lz, jitter=cfg.jitter,
               seed=configs.SEED_JITTER, dmask=cfg.dirichlet_mask)
    k = cfg.coefficients(m.ne)
    ft = O.faces(m)
    sysd = O.assemble(m, ft, cfg.problem, cfg.c, k["a_elem"], k["a_diag"])
    t_asm = time.time() - t0
    t1 = time.time()
    u, lam, st, rc, msg = _solve_keep(O, m, sysd, cfg, k)
    t_solve = time.time() - t1
    errs = O.errors(m, ft, u, lam, cfg.problem, cfg.c, k["a_elem"], k["a_diag"])
    iu = sample_indices(u.size)
    il = sample_indices(lam.size)
    meta = dict(config=cfg.name, cid=cid, ne=m.ne, l=int(ft["l"]), tol=cfg.tol,
                iterations=st["iterations"], residual=st["residual"],
                constraint_residual=st["constraint_residual"], verify_rc=rc, verify_msg=msg,
                norm_lambda=float(np.linalg.norm(lam)), norm_u=float(np.linalg.norm(u)),
                norm_rhs=float(np.linalg.norm(sysd["rhs"])), norm_bd=float(np.linalg.norm(sysd["bd"])),
                norm_rhs_neg=float(np.linalg.norm(sysd["rhs_neg"])),
                err_y=float(errs[0]), err_kappa=float(errs[1]), err_l2=float(errs[2]),
                seconds_assemble=t_asm, seconds_solve=t_solve, sample_seed=SAMPLE_SEED)
    path = os.path.join(out_dir, f"solution_cfg{cid}.npz")
    np.savez_compressed(path, meta=json.dumps(meta), idx_u=iu, u=u[iu], idx_lambda=il, lam=lam[il])
    print(json.dumps(meta), flush=True)
    return meta


def _solve_keep(O, m, sysd, cfg, k):
    """or_solve_schur fills U/Lambda/stats before verify_solution decides;
    call it raw so a refused solve still yields its iterates."""
    import ctypes as C
    from oracle_bind import _ptr
    pr = O._prob(cfg.problem, cfg.c, k["a_elem"], k["a_diag"])
    l = len(sysd["bd"])
    u = np.zeros(4 * m.ne)
    lam = np.zeros(l)
    st = np.zeros(3)
    rc = O.L.or_solve_schur(m.nc, m.ne, _ptr(m.coords), _ptr(m.tets), C.byref(pr), l, _ptr(sysd["slot_coef"]),
                       _ptr(sysd["slot_mrow"]), _ptr(sysd["rhs"]), _ptr(sysd["bd"]), _ptr(sysd["c_rowptr"]),
                       _ptr(sysd["c_col"]), _ptr(sysd["c_val"]), _ptr(sysd["s_rowptr"]), _ptr(sysd["s_col"]),
                       _ptr(sysd["s_val"]), _ptr(sysd["rhs_neg"]), cfg.tol, -1, _ptr(u), _ptr(lam), _ptr(st))
    msg = O.L.or_last_error().decode() if rc else ""
    return u, lam, dict(iterations=int(st[0]), residual=st[1], constraint_residual=st[2]), rc, msg


if __name__ == "__main__":
    out = os.path.join(ROOT, "tests", "golden")
    for a in sys.argv[1:]:
        run(int(a), out)
